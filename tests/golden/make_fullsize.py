"""Full-size goldens for BASELINE.json's configs (tests/golden/fullsize.json).

The GPU must match the reference's indexed-frame run bit-for-bit at the
configs' own sizes (north_star). These runs take minutes to an hour of CPU,
so they are computed once here and frozen as hashes:

* C2 (R-MAT 18), deterministic (indexed, spf 1, seed 42): the COMPILED
  REFERENCE (oracle/_ref/ref_driver = the unmodified headers, run_indexed
  with 8 threads), cross-checked by the threaded oracle (oracle.c
  or_estimate_bc_threads) — the two must agree before anything is written;
* C3 (BA 2^20), deterministic: the threaded oracle. The compiled reference's
  run_indexed at T = 8 on this graph grew past 60 GB of host memory (each
  frame is an n-length u64 StateFrame, 8 MB here, and frames pile up behind
  the in-order consumer, engine.hpp:531-566) and was killed; the oracle
  matches the reference on C2 at full size and on every golden run;
* C4 (2048^2 lattice), deterministic: the threaded oracle only. The compiled
  reference dereferences dist[UINT32_MAX] on this graph (frame 247 of seed
  42: every predecessor's sigma wraps to 0 mod 2^64, kadabra.hpp:230-241) and
  segfaults; the oracle defines that step (first predecessor) exactly as the
  engine does;
* C2, cumulative epochs (B = 1 024, seed 42): the threaded oracle in
  MODE_EPOCH, the semantics of the fused non-deterministic pipeline;
* C5 (R-MAT 24): the full run is ~10^7 core-seconds, so its first 200
  frames (the sampled paths, i.e. the RNG stream and the backtrack choices)
  are frozen instead;
* every config: n, m, components, D_ub (oracle.c or_diameter_upper_bound,
  graph.hpp:202-214) and omega (kadabra.hpp:41-53).

Each graph is pinned by the SHA-256 of the generator's edge pairs, so the
GPU test regenerates the identical graph on the box.

    python tests/golden/make_fullsize.py [--threads 8] [--only c2_rmat18,...]

Needs /root/reference (for the C2/C3 reference runs); results are cached in
tests/golden/_cache/ (git-ignored) so an interrupted run resumes.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_1903_09422_b200 import datasets  # noqa: E402

CACHE = HERE / "_cache"
OUT = HERE / "fullsize.json"

# (config, mode, spf, epoch_samples, seed, source)
RUNS = [
    ("c2_rmat18", "indexed", 1, 0, 42, "reference"),
    ("c3_ba", "indexed", 1, 0, 42, "oracle"),
    ("c4_grid", "indexed", 1, 0, 42, "oracle"),
    ("c2_rmat18", "epoch", 1, 1024, 42, "oracle"),
]
FRAMES = [("c5_rmat24", 42, 1, 0, 200)]
NOMINAL_T = 8


def pairs_sha(p: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(p, dtype="<u8").tobytes()).hexdigest()


def fnv1a_u32(ids: np.ndarray) -> str:
    """FNV-1a 64 over the little-endian u32 stream (vectorised per byte lane)."""
    h = 0xcbf29ce484222325
    b = np.ascontiguousarray(ids, dtype="<u4").tobytes()
    for byte in b:
        h ^= byte
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def run_key(r) -> str:
    cfg, mode, spf, B, seed, _ = r
    return f"{cfg}|{mode}|spf{spf}|B{B}|seed{seed}"


def cached(name: str, fn):
    CACHE.mkdir(parents=True, exist_ok=True)
    path = CACHE / f"{name}.json"
    if path.exists():
        return json.loads(path.read_text())
    t0 = time.time()
    val = fn()
    val["cpu_seconds_wall"] = round(time.time() - t0, 1)
    path.write_text(json.dumps(val, indent=1, sort_keys=True))
    return val


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 8)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    only = set(filter(None, a.only.split(",")))
    out = json.loads(OUT.read_text()) if OUT.exists() else {}
    out.setdefault("generator", "tests/golden/make_fullsize.py")
    out.setdefault("graphs", {})
    out.setdefault("runs", {})
    out.setdefault("frames", {})
    names = sorted({r[0] for r in RUNS} | {f[0] for f in FRAMES})
    for name in names:
        if only and name not in only:
            continue
        w = datasets.CONFIGS[name]
        pairs = datasets.pairs(name)
        sha = pairs_sha(pairs)
        g = oracle.from_pairs(pairs)
        print(f"[{name}] n={g.n} pairs sha {sha[:16]}", flush=True)

        def graph_facts():
            _, comps = oracle.components(g)
            dub = oracle.diameter_upper_bound(g)
            return {"pairs_sha256": sha, "n": g.n, "m": int(g.nbrs.shape[0] // 2), "components": comps,
                    "diameter_bound": dub, "epsilon": w.epsilon, "delta": w.delta,
                    "omega": oracle.compute_omega(dub, w.epsilon, w.delta)}

        facts = cached(f"{name}.graph", graph_facts)
        assert facts["pairs_sha256"] == sha, f"generator drift for {name}"
        out["graphs"][name] = {k: v for k, v in facts.items() if k != "cpu_seconds_wall"}

        for r in RUNS:
            if r[0] != name:
                continue
            cfg, mode, spf, B, seed, source = r
            key = run_key(r)

            def oracle_run():
                res = oracle.estimate_bc(g, w.epsilon, w.delta, mode=oracle.MODE_EPOCH if mode == "epoch"
                                         else oracle.MODE_INDEXED, spf=spf, epoch_samples=max(B, 1), seed=seed,
                                         nominal_threads=NOMINAL_T, threads=a.threads)
                c = res.counts
                return {"tau": res.tau, "check_cycles": res.check_cycles, "stop_epoch": res.stop_epoch,
                        "omega": res.omega, "diameter_bound": res.diameter_bound, "reason": res.reason,
                        "counts_fnv1a": oracle.fnv1a(c), "counts_sum": int(c.sum()), "counts_max": int(c.max()),
                        "degenerate_steps": int(res.degenerate_steps)}

            orc = cached(f"{key}.oracle".replace("|", "_"), oracle_run)
            print(f"  oracle {key}: tau {orc['tau']} fnv {orc['counts_fnv1a']} ({orc.get('cpu_seconds_wall')} s)",
                  flush=True)
            entry = {k: v for k, v in orc.items() if k != "cpu_seconds_wall"}
            entry.update({"config": cfg, "mode": mode, "spf": spf, "epoch_samples": B, "seed": seed,
                          "nominal_threads": NOMINAL_T, "epsilon": w.epsilon, "delta": w.delta})
            if source == "reference":
                def ref_run():
                    path = datasets.edge_list_file(name, ROOT / "build" / "graphs")
                    cpath = CACHE / f"{name}.ref.counts"
                    res = oracle.ref_run(path, eps=w.epsilon, delta=w.delta, seed=seed, variant="indexed", spf=spf,
                                         threads=NOMINAL_T, counts_path=cpath)
                    res["counts_fnv1a_check"] = oracle.fnv1a(np.fromfile(cpath, dtype="<u8"))
                    return res

                ref = cached(f"{key}.reference".replace("|", "_"), ref_run)
                got = (ref["tau"], ref["check_cycles"], ref["stop_epoch"], ref["omega"], ref["diameter_bound"],
                       ref["reason"], ref["counts_fnv1a"])
                want = (orc["tau"], orc["check_cycles"], orc["stop_epoch"], orc["omega"], orc["diameter_bound"],
                        orc["reason"], orc["counts_fnv1a"])
                assert got == want, f"reference and oracle disagree on {key}: {got} vs {want}"
                entry["source"] = "compiled reference (ref_driver run_indexed, T=8), equal to the threaded oracle"
                entry["reference_ads_seconds"] = ref["ads_s"]
            else:
                entry["source"] = "threaded oracle (oracle.c or_estimate_bc_threads)"
            out["runs"][key] = entry

        for fr in FRAMES:
            if fr[0] != name:
                continue
            cfg, seed, spf, first, count = fr
            key = f"{cfg}|seed{seed}|spf{spf}|{first}+{count}"

            def frames():
                got = oracle.sample_frames(g, seed, spf, first, count, threads=a.threads)
                lens = np.array([len(x) for x in got], dtype=np.uint64)
                ids = np.concatenate(got) if got else np.zeros(0, np.uint32)
                return {"lens": [int(x) for x in lens], "ids_fnv1a": fnv1a_u32(ids), "total_ids": int(ids.size)}

            fv = cached(key.replace("|", "_").replace("+", "_"), frames)
            print(f"  frames {key}: {fv['total_ids']} ids fnv {fv['ids_fnv1a']}", flush=True)
            out["frames"][key] = {"config": cfg, "seed": seed, "spf": spf, "first": first, "count": count,
                                  "lens": fv["lens"], "ids_fnv1a": fv["ids_fnv1a"], "total_ids": fv["total_ids"],
                                  "source": "threaded oracle (oracle.c or_sample_frames_threads)"}
        OUT.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
        del g
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()

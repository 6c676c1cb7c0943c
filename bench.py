"""KADABRA adaptive-sampling benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2_rmat18] [--impl adsb|reference]

A step is one complete estimate_bc run to the stopping rule at (epsilon, delta)
on the config's seeded synthetic graph (default configs[1]: R-MAT scale 18,
eps 0.005, delta 0.1, non-deterministic epoch mode). `value` is samples drawn
per second over the whole job (bench.hpp:131-133's definition), timed on the
device with CUDA events per step (L2 flushed between steps), max over ranks.
`e2e` repeats the measurement through the public API from host CSR buffers
(graph upload + run + result download per step). `roofline` relates the
sampler kernel's algorithmic bytes (4 B per adjacency entry scanned + 8 B per
expanded vertex) to its device time and the measured HBM peak.
`cpu_baseline` / `--impl reference` time the UNMODIFIED reference (compiled by
oracle/Makefile) on this host's cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM_GBS = 6650.0


def _peak_hbm() -> tuple[float, str]:
    try:
        return float(json.loads(PEAKS_FILE.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.005)  # ~10 samples even in a 50 ms timed region

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args, world: int, rank: int) -> None:
    """--impl reference: the compiled reference on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    from paper_1903_09422_b200 import datasets
    w = datasets.CONFIGS[args.config]
    cores = os.cpu_count() or 1
    line = {"impl": "reference", "metric": f"KADABRA samples/sec ({w.name})", "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True}
    if not oracle.ref_available():
        try:
            oracle.build()
        except Exception:
            pass
    path = datasets.edge_list_file(w.name, ROOT / "build" / "graphs")
    per_rep_samples = CPU_SAMPLES_PER_CORE.get(w.name, args.ref_samples_per_core) * cores
    variant = "indexed" if w.variant == "indexed" else "barrier"
    if oracle.ref_available():
        kind = "reference"
        res = oracle.ref_run(path, eps=w.epsilon, delta=w.delta, seed=w.seed, variant=variant,
                             spf=w.samples_per_frame, threads=cores, check_interval=per_rep_samples,
                             max_cycles=2 if variant == "barrier" else max(1, per_rep_samples // w.samples_per_frame),
                             reps=args.warmup + args.steps)
        reps = res["reps"][args.warmup:]
        secs = sum(r[0] for r in reps)
        samples = sum(r[1] for r in reps)
        sample_desc = (f"{len(reps)} capped {variant} runs of ~{per_rep_samples} samples each "
                       f"(FixedCycleSampler), T={cores}")
    else:
        kind, cores = "port", 1
        g = oracle.parse_file(path)
        t0 = time.perf_counter()
        r = oracle.estimate_bc(g, w.epsilon, w.delta, spf=1, seed=w.seed, max_frames=args.ref_samples_per_core)
        secs = time.perf_counter() - t0
        samples = r.tau
        sample_desc = f"oracle port, {samples} samples, 1 thread"
    value = samples / secs if secs > 0 else 0.0
    line.update({"value": value, "ms_per_step": 1000 * secs / max(1, args.steps),
                 "config": {"workload": w.name, "epsilon": w.epsilon, "delta": w.delta, "variant": variant},
                 "dtype": "u64", "data": "synthetic (seeded generator, DESIGN.md)",
                 "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": kind,
                                  "sample": sample_desc},
                 "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


# Reference samples per host core for one capped CPU run (~2-10 s each): the
# reference's forward BFS costs 0.38 / 39 / 234 / 174 / 5340 ms per sample on
# C1..C5.
CPU_SAMPLES_PER_CORE = {"c1_er": 2000, "c2_rmat18": 100, "c3_ba": 20, "c4_grid": 30, "c5_rmat24": 1}


def _kernel_label(n: int, variant, diameter_bound: int, world: int) -> str:
    """The sampler kernel the engine dispatches for this workload (engine.cu ensure_arena /
    estimate_bc): warp teams for n <= 2^16, else block teams; the fused epoch pipeline for
    cumulative epochs on one GPU; the global-state variant when D_ub > 128."""
    from paper_1903_09422_b200 import adsamp
    if n <= (1 << 16):
        return "sampler_kernel (warp teams, global state)"
    mode = "det" if variant == adsamp.Variant.indexed else ("fused" if world == 1 else "epoch")
    store = "global-state" if diameter_bound > 128 else "shared-memory hash"
    return f"sampler_cta_kernel<{mode}> (block teams, {store})"


def cpu_baseline(w, path) -> dict:
    import oracle
    cores = os.cpu_count() or 1
    per = CPU_SAMPLES_PER_CORE.get(w.name, 20) * cores
    try:
        if not oracle.ref_available():
            oracle.build()
        if oracle.ref_available():
            variant = "barrier"
            res = oracle.ref_run(path, eps=w.epsilon, delta=w.delta, seed=w.seed, variant=variant, threads=cores,
                                 check_interval=per, max_cycles=2, reps=2)
            secs = sum(r[0] for r in res["reps"])
            samples = sum(r[1] for r in res["reps"])
            return {"value": samples / secs, "unit": "samples/s", "cores": cores, "kind": "reference",
                    "sample": f"2 capped runs of {per} samples (barrier, T={cores}, FixedCycleSampler) "
                              f"of the same graph/eps/delta; ads_seconds only"}
    except Exception as e:  # pragma: no cover - reported, not fatal
        return {"value": None, "unit": "samples/s", "cores": cores, "kind": "reference", "sample": f"failed: {e}"}
    return {"value": None, "unit": "samples/s", "cores": cores, "kind": "reference", "sample": "ref_driver absent"}


REF_EQUIV_SAMPLES = {"c1_er": 400, "c2_rmat18": 40, "c3_ba": 10, "c4_grid": 10, "c5_rmat24": 2}


def reference_equivalent(w, value: float) -> dict:
    """Bytes the reference's forward BFS (kadabra.hpp:208-242) reads per sample,
    replayed by the oracle on a few samples of the same graph and seed."""
    import oracle
    from paper_1903_09422_b200 import datasets
    k = REF_EQUIV_SAMPLES.get(w.name, 10)
    g = oracle.from_pairs(datasets.pairs(w.name))
    r = oracle.estimate_bc(g, w.epsilon, w.delta, spf=1, seed=w.seed, max_frames=k)
    per = (4 * r.edges_scanned + 8 * r.vertices_expanded) / max(1, r.tau)
    return {"forward_bfs_bytes_per_sample": per, "samples_replayed": r.tau,
            "equivalent_gbs": per * value / 1e9,
            "note": "edge-read rate the reference algorithm would need for the same samples/s"}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2_rmat18")
    ap.add_argument("--impl", default="adsb", choices=["adsb", "reference"])
    ap.add_argument("--epoch-samples", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-samples-per-core", type=int, default=25)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world, rank, local = _dist()

    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import numpy as np
    import torch

    torch.cuda.set_device(local)
    from paper_1903_09422_b200 import adsamp, datasets
    from paper_1903_09422_b200.kadabra import estimate_bc

    comm = None
    if world > 1:
        import torch.distributed as dist
        from paper_1903_09422_b200.distributed import Comm
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = Comm.from_torch_distributed(device=local)

    w = datasets.CONFIGS[args.config]
    t0 = time.perf_counter()
    parsed = datasets.graph(w.name)
    g = parsed.graph
    gen_s = time.perf_counter() - t0
    variant = adsamp.Variant[w.variant]
    cfg = adsamp.EngineConfig(variant=variant, samples_per_frame=w.samples_per_frame, base_seed=w.seed,
                              threads=8, device=local, epoch_samples=args.epoch_samples, comm=comm)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        estimate_bc(g, w.epsilon, w.delta, cfg)

    step_ms, results = [], []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = estimate_bc(g, w.epsilon, w.delta, cfg)
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            results.append(r)
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    samples = sum(r.run.total_samples for r in results)
    value = samples / (total_ms / 1000.0)
    edges = sum(r.edges_scanned for r in results)
    verts = sum(r.vertices_expanded for r in results)
    sampler_ms = sum(r.sampler_ms for r in results)
    alg_bytes = 4 * edges + 8 * verts
    achieved = alg_bytes / (sampler_ms / 1000.0) / 1e9 if sampler_ms > 0 else 0.0
    peak, peak_src = _peak_hbm()
    traffic = None
    prof = ROOT / "profiles" / "ncu_sampler_summary.json"
    if prof.exists():
        try:
            entry = json.loads(prof.read_text()).get(w.name, {})
            traffic = entry.get("dram_bytes_per_launch")
            if traffic is None and entry.get("dram_bytes_per_sample"):
                # configs whose step launches several sampler batches: ncu bytes
                # per sample (capped capture) x the samples of this step
                traffic = entry["dram_bytes_per_sample"] * (
                    sum(r.run.total_samples for r in results) / max(1, len(results)))
        except Exception:
            traffic = None
    launches = sum(r.kernel_launches for r in results)

    # ---- end to end through the public API from host CSR buffers
    e2e = None
    if not args.no_e2e:
        off = np.ascontiguousarray(g.offsets())
        nb = np.ascontiguousarray(g.neighbor_list())
        n = g.num_vertices()
        e2e_ms, e2e_samples = [], 0
        for i in range(args.warmup + args.steps):
            flush.fill_(1)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g2 = adsamp.Graph.from_csr(n, off, nb)
            r2 = estimate_bc(g2, w.epsilon, w.delta, cfg)
            del g2
            e1.record()
            torch.cuda.synchronize()
            if i >= args.warmup:
                e2e_ms.append(e0.elapsed_time(e1))
                e2e_samples += r2.run.total_samples
        tot = sum(e2e_ms)
        if world > 1:
            t = torch.tensor([tot], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            tot = float(t.item())
        e2e = {"value": e2e_samples / (tot / 1000.0), "unit": "samples/s",
               "h2d_bytes_per_step": 4 * (n + 1) + 4 * int(nb.shape[0]),
               "d2h_bytes_per_step": 4 * n + 64,
               "note": "graph_from_csr (host validate) + device CSR upload + estimate_bc + counts download, "
                       "host buffers pageable"}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    r0 = results[-1]
    line = {
        "metric": f"KADABRA samples/sec ({w.name}, eps={w.epsilon}, delta={w.delta})",
        "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64",
        "data": f"synthetic: {w.description}",
        "config": {"workload": w.name, "n": g.num_vertices(), "m": g.num_edges(), "epsilon": w.epsilon,
                   "delta": w.delta, "mode": "deterministic-frames" if variant == adsamp.Variant.indexed
                   else "cumulative-epochs", "samples_per_frame": w.samples_per_frame, "seed": w.seed,
                   "l2": "flushed between steps (256 MiB write)", "parallelism": f"dp{world} (sample sharding)"},
        "time_to_stop_s": total_ms / args.steps / 1000.0,
        "tau": r0.tau, "total_samples_per_step": r0.run.total_samples, "reason": r0.reason.name,
        "omega": r0.omega, "diameter_bound": r0.diameter_bound, "preprocess_s": r0.preprocess_seconds,
        "edge_read_gbs": achieved,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic,
                     "kernel": _kernel_label(g.num_vertices(), variant, r0.diameter_bound, world),
                     "peak_source": peak_src,
                     "alg_bytes_per_sample": alg_bytes / max(1, sum(r.run.total_samples for r in results)),
                     "sampler_ms_per_step": sampler_ms / args.steps,
                     "edges_per_sample": {k: v / max(1, sum(r.run.total_samples for r in results)) for k, v in {
                         "bfs": edges - sum(r.rebuild_edges + r.backtrack_edges for r in results),
                         "rebuild": sum(r.rebuild_edges for r in results),
                         "backtrack": sum(r.backtrack_edges for r in results),
                         "vertices": verts}.items()}},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "graph_build_s": gen_s,
    }
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline and g.num_edges() <= 50_000_000:
        try:
            line["reference_equivalent"] = reference_equivalent(w, value)
        except Exception as e:  # pragma: no cover
            line["reference_equivalent"] = {"error": str(e)}
    if world == 1 and not args.no_cpu_baseline:
        if g.num_edges() > 50_000_000 and not args.force_cpu_baseline:
            line["cpu_baseline"] = {"value": None, "unit": "samples/s", "cores": os.cpu_count(), "kind": "reference",
                                    "sample": "skipped: the reference parses the multi-GB edge list single-threaded "
                                              "(minutes); pass --force-cpu-baseline"}
        else:
            path = datasets.edge_list_file(w.name, ROOT / "build" / "graphs")
            line["cpu_baseline"] = cpu_baseline(w, path)
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

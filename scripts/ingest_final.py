"""Copy the outputs of scripts/gpu_r2_final.sh (gpurun_out/r2f) into profiles/ and print the numbers the docs quote."""
import json
import re
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "gpurun_out" / "r2f"
DST = ROOT / "profiles"


def last_json(path: Path) -> dict:
    return json.loads(path.read_text().strip().splitlines()[-1])


names = {"c5": "bench_c5", "c1_er": "bench_c1_er", "c2_rmat18": "bench_c2_rmat18", "c3_ba": "bench_c3_ba",
         "c4_grid": "bench_c4_grid", "c5_reference": "bench_c5_reference"}
for out, src in names.items():
    line = (SRC / f"{src}.log").read_text().strip().splitlines()[-1]
    json.loads(line)
    (DST / f"r02_bench_{out}.json").write_text(line + "\n")
for c in ["c1", "c2", "c3", "c4", "c5"]:
    shutil.copy(SRC / f"{c}_full.json", DST / f"r02_{c}_ncu_full.json")
shutil.copy(SRC / "launches_c5.csv", DST / "r02_launches_c5.csv")
(DST / "r02_launches_c5_summary.txt").write_text(subprocess.run(
    [sys.executable, str(ROOT / "scripts" / "summarize_launches.py"), str(DST / "r02_launches_c5.csv")],
    capture_output=True, text=True).stdout)
shutil.copy(SRC / "pytest_gpu.log", DST / "r02_pytest_gpu_head.log")
shutil.copy(SRC / "smoke.log", DST / "r02_smoke_head.log")


def samples(log: str, key: str) -> int:
    m = re.findall(rf"{key}=(\d+)", (SRC / log).read_text())
    return int(m[-1])


caps = {"c5_rmat24": ("c5", samples("plain_c5.log", "total"), "capped 64-epoch fused launch (scripts/prof_capped.py c5_rmat24 64)"),
        "c2_rmat18": ("c2", samples("plain_c2.log", "total"), "the fused launch of rep 1 of scripts/prof_one.py c2_rmat18"),
        "c4_grid": ("c4", samples("plain_c4.log", "total"), "capped 1184-frame launch (scripts/prof_capped.py c4_grid 1184)")}
for cfg, (c, n, note) in caps.items():
    subprocess.run([sys.executable, str(ROOT / "scripts" / "ncu_to_summary.py"), cfg, str(SRC / f"{c}_full.json"), str(n),
                    f"profiles/r02_{c}_ncu_full.json: {note}, scripts/gpu_r2_final.sh"], capture_output=True)
rep = SRC / "c5_full.ncu-rep"
if rep.exists():
    csv = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    tmp = ROOT / "build" / "c5_cs.csv"
    tmp.parent.mkdir(exist_ok=True)
    tmp.write_text(csv)
    (DST / "r02_c5_hot_lines.txt").write_text(subprocess.run(
        [sys.executable, str(ROOT / "scripts" / "ncu_hot.py"), str(tmp), "40"], capture_output=True, text=True).stdout)
for out in ["c5", "c1_er", "c2_rmat18", "c3_ba", "c4_grid"]:
    d = last_json(DST / f"r02_bench_{out}.json")
    r, e, cb = d["roofline"], d["e2e"], d.get("cpu_baseline") or {}
    print(f"{out}: tau {d['tau']} drawn {d['drawn_samples_per_step']:.0f} ms {d['ms_per_step']:.3f} value {d['value']:.0f} "
          f"e2e {e['value']:.0f} ({e['ms_per_step']:.2f} ms) cpu {cb.get('value')} ({cb.get('kind')}) frac {r['frac']:.4f} "
          f"achieved {r['achieved']:.1f} alg/sample {r['alg_bytes_per_sample']:.0f} l2_frac {r.get('l2_frac')}")
d = last_json(DST / "r02_bench_c5_reference.json")
print("reference arm:", d["value"], "samples/s", d["ms_per_step"], "ms/step")
for c in ["c1", "c2", "c3", "c4", "c5"]:
    d = json.loads((DST / f"r02_{c}_ncu_full.json").read_text())[0]
    print(c, d["kernel"][:44], "dram R/W", d["dram__bytes_read.sum"], d["dram__bytes_write.sum"], "t", d["gpu__time_duration.sum"],
          "L2", d["lts__t_bytes.sum"], "hit", d["lts__t_sector_hit_rate.pct"][0], "issue",
          d["smsp__issue_active.avg.pct_of_peak_sustained_active"][0])

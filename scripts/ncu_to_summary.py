"""Merge one ncu --set full capture of the sampler kernel into profiles/ncu_sampler_summary.json.

    python scripts/ncu_to_summary.py CONFIG REPORT.ncu-rep|RAW.csv|SUMMARY.json SAMPLES_IN_LAUNCH "source note"

(SUMMARY.json: the output of scripts/ncu_summary.py written on the GPU box.)

Per launch: DRAM bytes (read + write) and L2 bytes (lts__t_bytes), converted
to bytes per sample, which bench.py scales by the samples a step draws.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "profiles" / "ncu_sampler_summary.json"
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def metrics(rep: str) -> dict:
    """rep: an .ncu-rep, the `ncu -i REP --page raw --csv` output saved on the GPU box, or ncu_summary.py's JSON"""
    if rep.endswith(".json"):
        d = json.loads(Path(rep).read_text())[0]
        out = {"kernel": d["kernel"]}
        for k, v in d.items():
            if isinstance(v, list):
                out[k] = v[0] * UNITS.get(v[1], 1.0)
        return out
    if rep.endswith(".csv"):
        txt = Path(rep).read_text()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, row = rows[0], rows[1], rows[2]
    out = {"kernel": row[hdr.index("Kernel Name")]}
    for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum",
                "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
                "launch__registers_per_thread"]:
        if key in hdr:
            i = hdr.index(key)
            v = float(row[i].replace(",", ""))
            out[key] = v * UNITS.get(units[i], 1.0)
    return out


def main() -> None:
    cfg, rep, samples, note = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
    m = metrics(rep)
    dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    d = json.loads(OUT.read_text()) if OUT.exists() else {}
    d["note"] = ("sampler kernel, one ncu --set full capture per config (+ lts__t_bytes): DRAM and L2 bytes per "
                 "sample of the captured launch; bench.py multiplies by the samples a step draws")
    d[cfg] = {"dram_bytes_per_sample": dram / samples, "lts_bytes_per_sample": m.get("lts__t_bytes.sum", 0) / samples,
              "dram_bytes_per_launch": dram, "lts_bytes_per_launch": m.get("lts__t_bytes.sum"),
              "samples_per_launch": samples, "kernel": m["kernel"][:120],
              "launch_ms_ncu": m.get("gpu__time_duration.sum"), "l2_hit_pct": m.get("lts__t_sector_hit_rate.pct"),
              "issue_active_pct": m.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
              "warps_active_pct": m.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
              "source": note}
    OUT.write_text(json.dumps(d, indent=1) + "\n")
    print(json.dumps(d[cfg], indent=1))


if __name__ == "__main__":
    main()

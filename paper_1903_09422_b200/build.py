"""Builds libadsb.so in-tree (paper_1903_09422_b200/libadsb.so) with nvcc for sm_100a.

    python -m paper_1903_09422_b200.build [--force] [--verbose]

Every .cu / .cpp under csrc/ is compiled with nvcc (-gencode
arch=compute_100a,code=sm_100a -lineinfo); host code uses -ffp-contract=off so
the FP64 stopping rule keeps the reference's operation order. cudart is linked
statically; NCCL dynamically (libnccl.so.2).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
# ADSB_BUILD_TAG=<tag>: an A/B variant (with ADSB_NVCC_EXTRA flags) built into
# build/obj_<tag> and ab/libadsb_<tag>.so, loaded with ADSB_LIB_PATH
_TAG = os.environ.get("ADSB_BUILD_TAG", "")
OBJ = ROOT / "build" / (f"obj_{_TAG}" if _TAG else "obj")
LIB = (ROOT / "ab" / f"libadsb_{_TAG}.so") if _TAG else PKG / "libadsb.so"
TOOL = PKG / "adsb_run"
TOOL_SRC = ROOT / "tools" / "adsb_run.cpp"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = [
    "-O3", "-std=c++17", "-lineinfo", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O3",
    f"-I{ROOT / 'include'}", f"-I{CSRC}",
    *os.environ.get("ADSB_NVCC_EXTRA", "").split(),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _sources() -> list[Path]:
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers() -> list[Path]:
    return sorted(list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h")))


def _compile(src: Path, verbose: bool) -> tuple[Path, str]:
    obj = OBJ / (src.name + ".o")
    cmd = [nvcc(), *ARCH, *COMMON, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cu" and verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stderr}\n{res.stdout}")
    return obj, res.stderr


def build(force: bool = False, verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    LIB.parent.mkdir(parents=True, exist_ok=True)
    srcs = _sources()
    newest_header = max((h.stat().st_mtime for h in _headers()), default=0.0)
    todo = []
    for s in srcs:
        o = OBJ / (s.name + ".o")
        if force or not o.exists() or o.stat().st_mtime < max(s.stat().st_mtime, newest_header):
            todo.append(s)
    logs = []
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4)) as ex:
            for obj, log in ex.map(lambda s: _compile(s, verbose), todo):
                logs.append(log)
    objs = [OBJ / (s.name + ".o") for s in srcs]
    if todo or force or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lnccl", "-lpthread"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}\n{res.stdout}")
    if not _TAG and TOOL_SRC.exists() and (not TOOL.exists() or TOOL.stat().st_mtime < max(LIB.stat().st_mtime,
                                                                            TOOL_SRC.stat().st_mtime)):
        cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++20", f"-I{ROOT / 'include'}", str(TOOL_SRC),
               "-o", str(TOOL), f"-L{PKG}", "-ladsb", "-Wl,-rpath,$ORIGIN"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"adsb_run build failed:\n{res.stderr}")
    if verbose:
        for log in logs:
            if log.strip():
                print(log, file=sys.stderr)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))

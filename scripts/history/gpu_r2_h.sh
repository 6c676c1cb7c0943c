# Round 2 h: vec4 in dynamic smem (scalar kernels keep the old L1 carve-out) vs the round-1 scalar build.
mkdir -p gpurun_out/r2h; rm -f gpurun_out/r2h/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
bash scripts/gpu_ab.sh "w0 cur" "c5_rmat24 c2_rmat18 c3_ba" r2h/ab.log
timeout 900 python -m pytest tests -m gpu -q -rf -k "sampler_variants or block_teams_frames or fullsize_frames or world2" > gpurun_out/r2h/pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2h/pytest.log

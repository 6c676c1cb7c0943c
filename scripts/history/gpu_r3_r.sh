# e2e breakdown on C5 after the from_csr changes (identity original ids written on request, parallel offsets check)
mkdir -p gpurun_out/r3r; rm -f gpurun_out/r3r/*
export ADSB_GRAPH_CACHE=build/gcache
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('c5_rmat24')"
timeout 600 python scripts/diag_e2e.py c5_rmat24 > gpurun_out/r3r/e2e_c5.log 2>&1
timeout 600 python scripts/diag_e2e.py c2_rmat18 > gpurun_out/r3r/e2e_c2.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3r/bench_c5.log 2>&1
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x -k "c5 or dropin or multirank or graph_facts" > gpurun_out/r3r/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3r/pytest.log

mkdir -p gpurun_out/rex
timeout 900 python scripts/exact_bc_check.py c2_rmat18 gpurun_out/rex/exact_c2.json > gpurun_out/rex/exact_c2.log 2>&1

D=/tmp/dbg; rm -rf $D; mkdir -p $D; cp -r paper_1903_09422_b200 include scripts tests oracle $D/
(cd $D && ADSB_NVCC_EXTRA="-DADSB_DEBUG_CHECKS" python -m paper_1903_09422_b200.build --force > build.log 2>&1)
(cd $D && timeout 600 python scripts/prof_one.py c3_ba 1 > /root/repo/gpurun_out/dbg_c3.log 2>&1)
(cd $D && ADSB_NO_SMEM=1 timeout 600 python scripts/prof_one.py c3_ba 1 > /root/repo/gpurun_out/dbg_c3_nosmem.log 2>&1)

mkdir -p gpurun_out/rd
bash scripts/gpu_ab2.sh "new=new hint=hint hint0=hint:ADSB_CSR_HINT=0 hint1=hint:ADSB_CSR_HINT=1" "c4_grid c3_ba c2_rmat18" rd/ab.log
bash scripts/gpu_ab2.sh "new=new hint=hint hint1=hint:ADSB_CSR_HINT=1" "c5_rmat24" rd/ab_c5.log
ADSB_LIB_PATH=ab/libadsb_hint.so timeout 300 python scripts/prof_capped.py c4_grid 1184 2 > gpurun_out/rd/plain_c4_capped.log 2>&1 && \
ADSB_LIB_PATH=ab/libadsb_hint.so timeout 900 ncu --set full --clock-control none -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/rd/c4_hint_full python scripts/prof_capped.py c4_grid 1184 2 > gpurun_out/rd/ncu_c4.log 2>&1

# ncu of the C3 L=2 scorer at S = 2 (host-driven loop so every launch is visible): iteration ~100
mkdir -p gpurun_out
KRONRED_LOOP=host timeout 600 ncu --set full --clock-control none -k regex:score3_kernel --launch-skip 100 -c 1 \
  -o gpurun_out/c3_s3_it100 -f python tools/profile_run.py c3 3e-3 0.03 > gpurun_out/c3_ncu.log 2>&1
tail -2 gpurun_out/c3_ncu.log

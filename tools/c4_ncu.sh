# ncu of the C4 L=2 scorer (host-driven loop so every launch is visible): iteration ~50 and ~3000
mkdir -p gpurun_out
KRONRED_LOOP=host timeout 600 ncu --set full --clock-control none -k regex:score3_kernel --launch-skip 50 -c 1 \
  -o gpurun_out/c4_s3_it50 -f python tools/profile_run.py c4 3e-3 0.02 > gpurun_out/c4_ncu.log 2>&1
tail -2 gpurun_out/c4_ncu.log

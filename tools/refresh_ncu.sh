# ncu source-level capture of the incremental base refresh (one launch)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:base_refresh --launch-skip 210 -c 1 \
  -o gpurun_out/refresh_inc -f timeout 300 python tools/micro/base_refresh.py c2 > gpurun_out/refresh_ncu.log 2>&1
tail -3 gpurun_out/refresh_ncu.log

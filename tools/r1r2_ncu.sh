timeout 300 python tools/r1r2_ab.py . 96 0.001 > /dev/null 2>&1  # generates /tmp/c4_L96.csv
KRONRED_LOOP=host timeout 600 ncu --section SourceCounters --clock-control none -k regex:score3 --launch-skip 20 -c 1 -f -o gpurun_out/s3_new python tools/r1r2_ab.py . 96 0.005 > /dev/null 2>&1
KRONRED_LOOP=host timeout 600 ncu --section SourceCounters --clock-control none -k regex:score3 --launch-skip 20 -c 1 -f -o gpurun_out/s3_r1 python tools/r1r2_ab.py tools/_var_r1 96 0.005 > /dev/null 2>&1
ls -la gpurun_out/s3_*.ncu-rep

# score1 for two-scenario libraries: timings (default vs KRONRED_NO_S1_LS2, forced splits)
run() { echo "== $*"; env "$@" timeout 300 python tools/iter_profile.py c4 3e-3 0.2 --bucket 5000 2>&1 | grep "total device"; env "$@" timeout 300 python tools/iter_profile.py c3 3e-3 0.9 --bucket 9000 2>&1 | grep "total device"; }
run KRONRED_X=1
run KRONRED_S3_S=1
run KRONRED_S3_S=2
run KRONRED_NO_S1_LS2=1
run KRONRED_NO_S1_LS2=1 KRONRED_S3_S=2

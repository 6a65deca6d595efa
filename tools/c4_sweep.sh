# C4 L=2 scorer geometry sweep (first 20 % of the run): score3 slots G and row split S
run() { echo "== $*"; env "$@" timeout 300 python tools/iter_profile.py c4 3e-3 0.2 --bucket 5000 2>&1 | grep "total device\|^sum"; }
run KRONRED_X=0
run KRONRED_S3_G=16
run KRONRED_S3_G=24
run KRONRED_S3_G=48
run KRONRED_S3_S=2
run KRONRED_S3_S=4
run KRONRED_S3_G=16 KRONRED_S3_S=2

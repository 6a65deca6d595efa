# multi-phase split x policy on C2 (score1 items 8,8,4)
for m in 4 2 1; do
  KRONRED_S3_MULTI=$m timeout 300 python tools/split_sweep.py c2 3e-3 --runs 2 --S 0 2>/dev/null | sed "s/^/MULTI=$m /" | cut -c1-330
done
KRONRED_S3_FILL=30000 timeout 300 python tools/split_sweep.py c2 3e-3 --runs 2 --S 0 2>/dev/null | sed "s/^/FILL30k /" | cut -c1-330
KRONRED_S3_FILL=100000 timeout 300 python tools/split_sweep.py c2 3e-3 --runs 2 --S 0 2>/dev/null | sed "s/^/FILL100k /" | cut -c1-330

for ns in 3 8; do KRONRED_S3_NS=$ns timeout 300 python tools/split_sweep.py c2 3e-3 --runs 2 --S 0,2 2>/dev/null | sed "s/^/NS=$ns /"; done

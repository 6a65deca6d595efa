# base refresh phase clocks and the BR_TRACE per-round breakdown; parity subset
timeout 120 python tools/micro/base_refresh.py c2
KRONRED_LIB=tools/_var_brtrace/libkronred_b200.so timeout 120 python tools/micro/base_refresh.py c2 2>&1 | grep "^round" | head -6
timeout 900 python -m pytest tests -m gpu -x -q -k "c2 or c1 or incremental or large or golden or m40 or h2k" 2>&1 | tail -2

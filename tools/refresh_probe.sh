# base refresh phase clocks: default, serial walk, and the BR_TRACE per-round breakdown
timeout 120 python tools/micro/base_refresh.py c2
KRONRED_SERIAL_WALK=1 timeout 120 python tools/micro/base_refresh.py c2
KRONRED_LIB=tools/_var_brtrace/libkronred_b200.so timeout 120 python tools/micro/base_refresh.py c2 2>&1 | grep "^round" | head -60

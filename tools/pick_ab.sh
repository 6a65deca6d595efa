# pick/commit kernel changes: parity subset + the per-iteration timeline
timeout 900 python -m pytest tests -m gpu -x -q -k "c2 or c1 or incremental or full_run or exchange or complex or live or m40" 2>&1 | tail -2
timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | grep "after pick\|^sum\|total device\|pick start" | sort -u

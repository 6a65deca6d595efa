for v in . tools/_var_r1 . tools/_var_r1; do KRONRED_LOOP=host timeout 600 python tools/r1r2_ab.py $v 96 0.01 --profile 2>&1 | grep "iterations\|scorer"; done
timeout 1200 python -m pytest tests -m gpu -x -q -k "large or c3 or c4 or iteration_scores or s24 or c2 or m40 or h2k or regenerated" 2>&1 | tail -2

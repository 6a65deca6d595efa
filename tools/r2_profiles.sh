# Round-2 measurement set (one GPU): bench line, launch lists, --set full
# captures of the scorer (iterations 100/500/850), the base refresh and the
# elimination executor, and the device-loop timeline. Outputs: gpurun_out/r2/.
set -u
O=gpurun_out/r2; mkdir -p $O
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc $?"
timeout 300 python tools/iter_profile.py c2 3e-3 --out $O/iter_timeline_c2.tsv > $O/iter_profile.txt 2>&1; echo "timeline rc $?"
# launch list of the host-driven loop (every kernel visible to ncu; cold-cache, serialised)
KRONRED_LOOP=host timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c2_hostloop.csv python tools/profile_run.py c2 > $O/ncu_ll.log 2>&1; echo "launch list rc $?"
# launch list of the bench command itself
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "bench launch list rc $?"
for it in 100 500 850; do
  KRONRED_LOOP=host timeout 600 ncu --set full --import-source on --clock-control none -k regex:score1 \
    --launch-skip $((it - 1)) --launch-count 1 -f -o $O/score1_it$it python tools/profile_run.py c2 > $O/ncu_s1_$it.log 2>&1
  echo "score1 it$it rc $?"
done
KRONRED_LOOP=host timeout 600 ncu --set full --import-source on --clock-control none -k regex:base_refresh \
  --launch-skip 100 --launch-count 1 -f -o $O/refresh_it100 python tools/profile_run.py c2 > $O/ncu_ref.log 2>&1; echo "refresh rc $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:elim_factor \
  --launch-count 1 -f -o $O/elim_first python tools/profile_run.py c2 > $O/ncu_elim.log 2>&1; echo "elim rc $?"

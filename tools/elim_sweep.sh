# elim_factor_kernel per-launch times (ncu launch list) for 256 (default) / 512 / 1024 threads on C2
for v in default 512 1024; do
  lib=""; [ "$v" != default ] && lib="KRONRED_LIB=tools/_var_elim$v/libkronred_b200.so"
  env $lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:elim_factor --csv \
      python tools/profile_run.py c2 2>/dev/null | grep elim_factor | awk -F'","' -v v=$v '{gsub(/"/,"",$NF); printf "%s %s\n", v, $NF}'
done

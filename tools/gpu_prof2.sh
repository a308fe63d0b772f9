mkdir -p gpurun_out
for cfg in "G2 gemv_cm_rows" "G3 gemv_cm_split" "G1 gemv_rm_sweep"; do
  set -- $cfg
  python tools/ncu_runner.py --config $1 --reps 2 > gpurun_out/plain_$1.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o gpurun_out/prof_$1 -f python tools/ncu_runner.py --config $1 --reps 2 > gpurun_out/ncu_$1.log 2>&1
  echo "$1 ncu rc=$?"
done

mkdir -p gpurun_out
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench2.json 2> gpurun_out/bench2.err
for cfg in "D1 dot_kernel" "G1 gemv_rm_vec" "R1 ger_vec"; do
  set -- $cfg
  python tools/ncu_runner.py --config $1 --reps 2 > gpurun_out/plain_$1.log 2>&1 && \
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o gpurun_out/prof_$1 -f python tools/ncu_runner.py --config $1 --reps 2 > gpurun_out/ncu_$1.log 2>&1
  echo "$1 ncu rc=$?"
done

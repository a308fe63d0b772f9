# Round evidence (r02): full GPU tests, smoke, C++ examples, bench + reference arm,
# ncu launch list, back-to-back DRAM checks, ncu --set full per config, sweeps.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
./tests/cpp/mgpu_example > gpurun_out/mgpu_example.log 2>&1; echo "rc=$?" >> gpurun_out/mgpu_example.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 1 --steps 200 --warmup 5 --no-suite > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err
CMD="python bench.py --steps 20 --warmup 3 --no-suite --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_launches.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
python tools/ncu_runner.py --config G1 --reps 6 --no-flush > gpurun_out/plain_b2b.log 2>&1 && timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gemv_rm -c 6 --csv --log-file gpurun_out/ncu_b2b_G1.csv python tools/ncu_runner.py --config G1 --reps 6 --no-flush > gpurun_out/ncu_b2b.log 2>&1
python tools/ncu_runner.py --config D1 --reps 6 --no-flush > gpurun_out/plain_b2b_D1.log 2>&1 && timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:dot_kernel -c 6 --csv --log-file gpurun_out/ncu_b2b_D1.csv python tools/ncu_runner.py --config D1 --reps 6 --no-flush > gpurun_out/ncu_b2b_D1.log 2>&1
for cfg in "G1 gemv_rm_sweep" "D1 dot_kernel" "R1 ger_tile" "G2 gemv_cm_tall" "G3 gemv_cm_split" "D2 dot_chunk" "G4 gemv_rm_sweep" "D1f dot_peer" "R1x ger_flat_any" "G1g gemv_rm_gather" "CM4096 gemv_cm_fullcol_kernel" "RM1024 gemv_rm_subsweep_kernel" "RM1001 gemv_rm_subsweep_scalar"; do
  set -- $cfg
  python tools/ncu_runner.py --config $1 --reps 2 > gpurun_out/plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o gpurun_out/prof_$1 -f python tools/ncu_runner.py --config $1 --reps 2 > gpurun_out/ncu_$1.log 2>&1
  echo "$1 ncu rc=$?"
done
timeout 900 python -m paper_2108_02025_b200.benchcli --kernel all --sizes 4096,8192 --rect 256x1048576,1048576x256 --dtype f32 --reps 5 --bounds --csv gpurun_out/bounds_plain.csv > /dev/null 2> gpurun_out/bounds_plain.err && \
timeout 1200 python -m paper_2108_02025_b200.benchcli --kernel all --sizes 4096,8192 --rect 256x1048576,1048576x256 --dtype f32 --reps 5 --bounds --measure-dram --csv gpurun_out/bounds.csv > /dev/null 2> gpurun_out/bounds.err
python tools/peer_cost.py > gpurun_out/peer_cost.jsonl 2>&1
python tools/shape_sweep.py > gpurun_out/shape_sweep.md 2> gpurun_out/shape_sweep.err

# Bench-only evidence refresh (kernels unchanged since the last full refresh): default
# bench, the reference arm, three runs at the driver's K = 20 / W = 5, torchrun world 1.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
rm -f gpurun_out/bench_k20_runs.jsonl
for i in 1 2 3; do timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-suite >> gpurun_out/bench_k20_runs.jsonl 2>> gpurun_out/bench_k20.err; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 1 --steps 200 --warmup 5 --no-suite > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err
python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_gpus2_on_1gpu.out 2>&1; echo "rc=$?" >> gpurun_out/bench_gpus2_on_1gpu.out

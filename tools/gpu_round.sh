mkdir -p gpurun_out
(lscpu | head -20; free -g; nproc) > gpurun_out/host.txt 2>&1
timeout 1800 python bench.py --cpu-table > gpurun_out/cpu_table.jsonl 2> gpurun_out/cpu_table.err; echo "rc=$?" >> gpurun_out/cpu_table.err

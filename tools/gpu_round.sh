mkdir -p gpurun_out
python tools/ncu_runner.py --config D1 --reps 8 --no-flush > gpurun_out/plain_b2b_D1.log 2>&1 && timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:dot_kernel -c 8 --csv --log-file gpurun_out/ncu_b2b_D1.csv python tools/ncu_runner.py --config D1 --reps 8 --no-flush > gpurun_out/ncu_b2b_D1.log 2>&1
timeout 300 python tools/b2b.py D1 R1 > gpurun_out/b2b2.jsonl 2>&1

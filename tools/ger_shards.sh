# GER on the R1 shard shapes of 2/4/8 GPUs (m = 4096/2048/1024 x 8192 fp32), per launch mode.
mkdir -p gpurun_out
out=gpurun_out/ger_shards.jsonl
rm -f $out
for bytes in 134217728 67108864 33554432; do
  for mode in 2 1 0; do
    CABL_TUNING=1 CABL_GER_MODE=$mode timeout 200 python tools/ab_shapes.py --tag mode$mode --op ger-row --n 8192 --dtypes f32 --bytes $bytes >> $out 2>&1
  done
done

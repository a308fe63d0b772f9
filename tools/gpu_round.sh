mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
for i in 1 2; do
CABL_TUNING=1 CABL_CM_COLBULK=0 timeout 300 python tools/ab_shapes.py --tag realign --op gemv-col --n 9300,10001,11000,12275 --dtypes f32 >> gpurun_out/ab.jsonl 2>&1
timeout 300 python tools/ab_shapes.py --tag product --op gemv-col --n 9300,10001,11000,12275 --dtypes f32 >> gpurun_out/ab.jsonl 2>&1
done

mkdir -p gpurun_out
out=gpurun_out/rm_subsweep256.jsonl
rm -f $out
for v in 0 8192; do
  CABL_TUNING=1 CABL_RM_SUBSWEEP_MAXB=$v timeout 300 python tools/ab_shapes.py --tag maxb$v --op gemv-row --n 2048,1792,1536,1280,1032 --dtypes f32 >> $out 2>&1
  CABL_TUNING=1 CABL_RM_SUBSWEEP_MAXB=$v timeout 300 python tools/ab_shapes.py --tag maxb$v --op gemv-row --n 1024,768,640,516 --dtypes f64 >> $out 2>&1
done

# Row-major GEMV, rows of 256 B - 4 KiB: the sub-CTA sweep against the G-lanes kernel.
# CABL_RM_SUBSWEEP: 0 = off, <percent> = least share of a slot's lanes a row must fill.
mkdir -p gpurun_out
out=gpurun_out/rm_subsweep.jsonl
rm -f $out
for v in 0 50; do
  CABL_TUNING=1 CABL_RM_SUBSWEEP=$v timeout 400 python tools/ab_shapes.py --tag subsweep$v --op gemv-row --n 1024,768,640,520,512,400,320,264,256,200,160,136,128,96,72 --dtypes f32 >> $out 2>&1
  CABL_TUNING=1 CABL_RM_SUBSWEEP=$v timeout 400 python tools/ab_shapes.py --tag subsweep$v --op gemv-row --n 512,384,260,256,132,128,100,68,64,48,36 --dtypes f64 >> $out 2>&1
done

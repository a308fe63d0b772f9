# Row-major GEMV, odd / misaligned rows of 65 - 2048 elements: the scalar sub-CTA sweep
# against the scalar G-lanes kernel.
mkdir -p gpurun_out
out=gpurun_out/rm_subsweep_scalar.jsonl
rm -f $out
for v in 0 1; do
  CABL_TUNING=1 CABL_RM_SUBSWEEP_SCALAR=$v timeout 400 python tools/ab_shapes.py --tag scalar$v --op gemv-row --n 2047,1501,1001,999,513,255,249,129,100,65 --dtypes f32 >> $out 2>&1
  CABL_TUNING=1 CABL_RM_SUBSWEEP_SCALAR=$v timeout 400 python tools/ab_shapes.py --tag scalar$v --op gemv-row --n 1001,513,255,129,65 --dtypes f64 >> $out 2>&1
done

mkdir -p gpurun_out
out=gpurun_out/rm_subsweep_scalar_f64.jsonl
rm -f $out
for v in 0 1; do
  CABL_TUNING=1 CABL_RM_SUBSWEEP_SCALAR=$v timeout 400 python tools/ab_shapes.py --tag scalar$v --op gemv-row --n 1501,901,801,701,601,401,301 --dtypes f64 >> $out 2>&1
done

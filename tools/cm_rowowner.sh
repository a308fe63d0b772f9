# Row-owner experiment: the 2-D split forced to ~one row tile per SM and a single
# column part (no cross-CTA partials), against the product paths.
mkdir -p gpurun_out
out=gpurun_out/cm_rowowner.jsonl
rm -f $out
run() { # tag m dtype env...
  tag=$1; m=$2; dt=$3; shift 3
  env CABL_TUNING=1 "$@" timeout 300 python tools/ab_shapes.py --tag $tag --op gemv-col --n $m --dtypes $dt >> $out 2>&1
}
for m in 4096 8192 16384 32768 65536; do run product $m f32; done
run t32 4096 f32 CABL_CM_TILE=512,32 CABL_CM_FULLCOL=0
run t56 8192 f32 CABL_CM_TILE=512,56 CABL_CM_FULLCOL=0
run t64 8192 f32 CABL_CM_TILE=512,64 CABL_CM_FULLCOL=0
run t112 16384 f32 CABL_CM_TILE=512,112 CABL_CM_FULLCOL=0
run t128 16384 f32 CABL_CM_TILE=512,128 CABL_CM_FULLCOL=0
run t224 32768 f32 CABL_CM_TILE=512,224 CABL_CM_FULLCOL=0
run t256 32768 f32 CABL_CM_TILE=512,256 CABL_CM_FULLCOL=0
run t448 65536 f32 CABL_CM_TILE=512,448 CABL_CM_FULLCOL=0
run t512 65536 f32 CABL_CM_TILE=512,512 CABL_CM_FULLCOL=0
for m in 8192 16384; do run product $m f64; done
run t56 8192 f64 CABL_CM_TILE=512,56 CABL_CM_FULLCOL=0
run t112 16384 f64 CABL_CM_TILE=512,112 CABL_CM_FULLCOL=0

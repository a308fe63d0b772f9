mkdir -p gpurun_out
: > gpurun_out/g1_variants.txt
run() { echo "$1 $(env $1 python tools/b2b.py G1 2>&1 | tail -1)" >> gpurun_out/g1_variants.txt; }
run "X=default"
run "CABL_GEMV_DYN=1"
run "CABL_RM_SWEEP=2,4,2"
run "CABL_RM_SWEEP=4,1,4"
run "CABL_RM_SWEEP=8,1,2"
run "CABL_RM_SWEEP=4,4,1"
run "CABL_RM_SWEEP=8,2,1"
run "CABL_RM_SWEEP=2,8,1"
run "CABL_PDL_PREFETCH=0"

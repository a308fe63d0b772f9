mkdir -p gpurun_out
: > gpurun_out/d1_pf.txt
run() { echo "$1 $(env $1 python tools/b2b.py D1 2>&1 | tail -1)" >> gpurun_out/d1_pf.txt; }
run "CABL_PDL_PREFETCH=1"
run "CABL_PDL_PREFETCH=3"
run "CABL_PDL_PREFETCH=4"
run "CABL_PDL_PREFETCH=6"
run "CABL_PDL_PREFETCH=8"
run "CABL_PDL_PREFETCH=1"

mkdir -p gpurun_out
rm -f gpurun_out/tune22.jsonl
for pf in 0 1 2 4 8; do
  CABL_PDL_PREFETCH=$pf timeout 300 python tools/b2b.py G1 G4 | sed "s/^/pf$pf /" >> gpurun_out/tune22.jsonl 2>&1
done

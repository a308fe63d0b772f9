mkdir -p gpurun_out
rm -f gpurun_out/tune22.jsonl
for i in 1 2; do
for ef in 0 1; do CABL_GER_EF=$ef timeout 300 python tools/b2b.py R1 | sed "s/^/ef$ef /" >> gpurun_out/tune22.jsonl 2>&1; done
done

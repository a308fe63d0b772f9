mkdir -p gpurun_out
rm -f gpurun_out/tune16.jsonl
python tools/b2b.py D1 >> gpurun_out/tune16.jsonl 2>&1
for ch in 1024 2048 4096 8192; do
CABL_DOT_CHUNKED=1 CABL_DOT_CHUNK=$ch python tools/b2b.py D1 | sed "s/^/chunk=$ch /" >> gpurun_out/tune16.jsonl 2>&1
done

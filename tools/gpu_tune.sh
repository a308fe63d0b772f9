mkdir -p gpurun_out
python tools/tune.py G1 G4 >> gpurun_out/tune3.jsonl 2>&1
for cfg in 256,1,8 256,2,8 256,2,4 256,4,4 512,2,2 512,4,2 1024,2,1 1024,4,1; do CABL_DOT_CFG=$cfg TUNE_STEPS=60 python tools/tune.py D1 >> gpurun_out/tune3.jsonl 2>&1; done

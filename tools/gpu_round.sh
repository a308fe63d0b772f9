mkdir -p gpurun_out
cat > /tmp/cm_tiles.py <<'PY'
import sys, json, os, torch
sys.path.insert(0, 'tools'); sys.path.insert(0, '.')
from ger_odd import buf, timeit
import paper_2108_02025_b200 as cb
pol = cb.default_policy(1)
for m, n in ((1024, 65536), (2048, 32768), (4096, 16384), (8192, 8192), (16384, 4096), (32768, 2048)):
    A, x, c = buf(m * n, 0, torch.float32), buf(n, 0, torch.float32), buf(m, 0, torch.float32)
    Am = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
    c0 = c.clone(); cb.gemv_col_major(Am, x, c0, pol)
    us = timeit(lambda: cb.gemv_col_major(Am, x, c, pol))
    print(json.dumps({"tile": os.environ.get("CABL_CM_TILE", "auto") + "/" + os.environ.get("CABL_CM_EXTFINAL", "0"), "m": m, "n": n, "us": round(us, 2), "c0": float(c0[:64].double().sum())}), flush=True)
PY
python /tmp/cm_tiles.py > gpurun_out/cm_ext.jsonl 2>&1
for t in 256 512 1024 2048 4096; do CABL_CM_EXTFINAL=1 CABL_CM_TILE=512,$t python /tmp/cm_tiles.py >> gpurun_out/cm_ext.jsonl 2>&1; done
CABL_CM_EXTFINAL=1 python /tmp/cm_tiles.py >> gpurun_out/cm_ext.jsonl 2>&1

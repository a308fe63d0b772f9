mkdir -p gpurun_out
cat > /tmp/rm_gv.py <<'PY'
import sys, json, os, torch
sys.path.insert(0, 'tools'); sys.path.insert(0, '.')
from ger_odd import buf, timeit
import paper_2108_02025_b200 as cb
pol = cb.default_policy(1)
for m, n in ((65536, 1024), (131072, 512), (262144, 256), (32768, 2048)):
    A, x, c = buf(m * n, 0, torch.float32), buf(n, 0, torch.float32), buf(m, 0, torch.float32)
    Am = cb.DenseMatrix.wrap(A, m, n, cb.Layout.RowMajor)
    us = timeit(lambda: cb.gemv_row_major(Am, x, c, pol))
    print(json.dumps({"cfg": os.environ.get("CABL_GEMV_RM_MODE", "auto") + "/" + os.environ.get("CABL_RM_SWEEP", "-"), "m": m, "n": n, "us": round(us, 2)}), flush=True)
PY
python /tmp/rm_gv.py > gpurun_out/rm_gv.jsonl 2>&1
for c in "1 4,2,2" "1 8,1,2" "1 4,1,4" "2 2,4,2"; do set -- $c; CABL_GEMV_RM_MODE=$1 CABL_RM_SWEEP=$2 python /tmp/rm_gv.py >> gpurun_out/rm_gv.jsonl 2>&1; done

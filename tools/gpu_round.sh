mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
cat > /tmp/px.py <<'PY'
import sys, json, torch
sys.path.insert(0, sys.argv[1] + '/tools'); sys.path.insert(0, sys.argv[1])
from ger_odd import buf, timeit
import paper_2108_02025_b200 as cb
pol = cb.default_policy(1)
for m, n in ((16, 4194304), (8192, 8192), (1024, 65536)):
    for xoff in (0, 1):
        A, x, c = buf(m * n, 0, torch.float32), buf(n, xoff, torch.float32), buf(m, 0, torch.float32)
        for lay in (cb.Layout.RowMajor, cb.Layout.ColMajor):
            Am = cb.DenseMatrix.wrap(A, m, n, lay)
            f = cb.gemv_row_major if lay == cb.Layout.RowMajor else cb.gemv_col_major
            print(json.dumps({"lay": int(lay), "m": m, "n": n, "xoff": xoff, "us": round(timeit(lambda: f(Am, x, c, pol)), 2)}), flush=True)
PY
python /tmp/px.py $PWD > gpurun_out/probe_x.jsonl 2>&1

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bounds.py -q -x -k "ger" --timeout 600 -p no:cacheprovider > gpurun_out/pytest_ger.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ger.log
cat > /tmp/axpy_t.py <<'PY'
import sys, json, torch
sys.path.insert(0, 'tools'); sys.path.insert(0, '.')
from ger_odd import buf, timeit
import paper_2108_02025_b200 as cb
pol = cb.default_policy(1)
for dt in (torch.float32, torch.float64):
    s = torch.tensor([], dtype=dt).element_size()
    N = (256 << 20) // s
    for lay, m, n in ((cb.Layout.ColMajor, 1, N), (cb.Layout.RowMajor, N, 1)):
        x, y, C = buf(m, 0, dt), buf(n, 0, dt), buf(m * n, 0, dt)
        Cm = cb.DenseMatrix.wrap(C, m, n, lay)
        us = timeit(lambda: cb.ger(x, y, Cm, pol))
        print(json.dumps({"dtype": str(dt)[6:], "layout": str(lay), "m": m, "n": n, "us": round(us, 2), "gbs": round((2*m*n+m+n)*s/us/1e3, 1)}), flush=True)
PY
CABL_GER_ANY=1 python /tmp/axpy_t.py > gpurun_out/axpy.jsonl 2>&1

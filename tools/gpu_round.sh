mkdir -p gpurun_out
cat > /tmp/cm_mid.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import bench
import paper_2108_02025_b200 as cb
dev = torch.device('cuda:0')
pol = cb.default_policy(1)
fl = bench.L2Flush(dev)
m, n = int(sys.argv[1]), int(sys.argv[2])
A = cb.fill_uniform(torch.empty(m * n, device=dev), 1, 3)
x = cb.fill_uniform(torch.empty(n, device=dev), 1, 1)
c = cb.fill_uniform(torch.empty(m, device=dev), 1, 4)
Am = cb.DenseMatrix.wrap(A, m, n, cb.Layout.ColMajor)
for _ in range(3):
    fl.zero_(); cb.gemv_col_major(Am, x, c, pol)
torch.cuda.synchronize()
print('ok')
PY
python /tmp/cm_mid.py 4096 16384 > gpurun_out/cm_mid_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_cm -s 1 -c 1 -o gpurun_out/prof_cm4096 -f python /tmp/cm_mid.py 4096 16384 > gpurun_out/ncu_cm4096.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cm_mid_launches.csv python /tmp/cm_mid.py 4096 16384 > /dev/null 2>&1

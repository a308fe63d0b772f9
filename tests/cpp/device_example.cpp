// Device-resident use of the drop-in (cabl/device.hpp): operands uploaded
// once, every call stays in HBM.  Checks each result against the same call on
// host containers (the two paths run the same kernels, so results are equal
// bit for bit).
#include <cabl/device.hpp>

#include <cstdio>
#include <random>

using namespace cabl;

int main() {
    const ExecPolicy pol(derive_blocking_plan(default_machine()), 1);
    std::mt19937_64 rng(42);
    std::uniform_real_distribution<float> d(-1.f, 1.f);
    const std::size_t m = 4096, n = 2048;
    DenseMatrix<float> A(m, n, Layout::RowMajor);
    Vector<float> x(n), c(m), y(m);
    for (std::size_t i = 0; i < A.size(); ++i) A.data()[i] = d(rng);
    for (auto& v : x) v = d(rng);
    for (auto& v : c) v = d(rng);
    for (auto& v : y) v = d(rng);

    DeviceMatrix<float> dA(A);
    DeviceVector<float> dx(x), dc(c), dy(y);
    gemv_row_major(dA, dx, dc, pol);
    Vector<float> host_c = c;
    gemv_row_major(A, x, host_c, pol);
    const bool gemv_ok = dc.download() == host_c;

    const float dd = dot(dy, dc, 0.5f, pol);
    const float hd = dot(y, host_c, 0.5f, pol);

    DeviceMatrix<float> dC(m, n, Layout::ColMajor);
    DenseMatrix<float> C(m, n, Layout::ColMajor, 0.25f);
    dC.upload(C);
    ger(dy, dx, dC, pol);
    ger(y, x, C, pol);
    const bool ger_ok = dC.download() == C;

    // the live GPU in the reference's descriptor model
    const MachineDescriptor gm = gpu_machine(0, sizeof(float));
    const BlockingPlan gbp = derive_blocking_plan(gm); // the reference rules accept it
    const GpuPlan gp = derive_gpu_plan(gm);
    const bool mach_ok = gm.cores == describe_device(0).sm_count && gp.dot_ctas == 2 * gm.cores &&
                         gp.queue_threshold_bytes >= 4 * gp.l2_bytes && gbp.max_threads == gm.cores;
    std::printf("machine: %u SMs, L1 %llu B, L2 %llu B, queue threshold %llu B (%s)\n", gm.cores,
                (unsigned long long)gm.level(0).size_bytes(),
                (unsigned long long)gm.level(1).size_bytes(),
                (unsigned long long)gp.queue_threshold_bytes, mach_ok ? "ok" : "MISMATCH");

    std::printf("gemv %s, dot %s (%.6f), ger %s\n", gemv_ok ? "ok" : "MISMATCH",
                dd == hd ? "ok" : "MISMATCH", double(dd), ger_ok ? "ok" : "MISMATCH");
    return (gemv_ok && dd == hd && ger_ok && mach_ok) ? 0 : 1;
}

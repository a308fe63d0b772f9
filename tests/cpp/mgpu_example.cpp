// Multi-GPU drop-in use (cabl/nccl.hpp over the cabl_mgpu_* C ABI): one
// process drives every visible device through an NCCL clique.  Checks the sharded results bit for bit
// against the same per-shard computations run one by one on device 0:
//   DOT  = rank-ordered sum of the per-shard partials + alpha0 (NCCL all-gather
//          path and the fused peer-memory path),
//   GEMV = each row block, GER = each row block.
// With one GPU (this run's boxes) the clique has one member and the path
// still goes through ncclCommInitAll / ncclAllGather / the ordered combine.
#include <cabl/nccl.hpp>

#include <cstdio>
#include <random>

using namespace cabl;

int main() {
    int ndev = 0;
    cudaGetDeviceCount(&ndev);
    if (ndev < 1) {
        std::printf("no CUDA device\n");
        return 2;
    }
    std::vector<int> devs;
    for (int d = 0; d < ndev; ++d) devs.push_back(d);
    nccl::Group g(devs);
    const int G = g.size();
    const ExecPolicy pol(derive_blocking_plan(default_machine()), 1);
    std::mt19937_64 rng(2026);
    std::uniform_real_distribution<float> U(-1.f, 1.f);
    bool ok = true;

    // ---- DOT
    const std::size_t n = (std::size_t(1) << 24) + 5;
    Vector<float> x(n), y(n);
    for (auto& v : x) v = U(rng);
    for (auto& v : y) v = U(rng);
    std::vector<DeviceVector<float>> xs, ys;
    float expect = 0.f;
    for (int r = 0; r < G; ++r) {
        const nccl::Range rg = nccl::partition(n, G, r);
        Vector<float> xc(rg.end - rg.begin), yc(rg.end - rg.begin);
        std::copy(x.begin() + rg.begin, x.begin() + rg.end, xc.begin());
        std::copy(y.begin() + rg.begin, y.begin() + rg.end, yc.begin());
        cudaSetDevice(0);
        const float p = dot(DeviceVector<float>(xc), DeviceVector<float>(yc), 0.0f, pol);
        expect = expect + p; // rank order, alpha0 last (kernels.hpp:160-163)
        cudaSetDevice(g.device(r));
        xs.emplace_back(xc);
        ys.emplace_back(yc);
    }
    expect = expect + 0.75f;
    std::vector<const DeviceVector<float>*> xp, yp;
    for (int r = 0; r < G; ++r) {
        xp.push_back(&xs[r]);
        yp.push_back(&ys[r]);
    }
    const float got = nccl::sharded_dot(g, xp, yp, 0.75f, pol);
    ok &= got == expect;
    std::printf("sharded dot over %d GPU(s): %.9g (expected %.9g) %s\n", G, double(got),
                double(expect), got == expect ? "ok" : "MISMATCH");
    for (int call = 0; call < 3; ++call) { // the fused (peer-memory) exchange: same bits
        const float fused = nccl::sharded_dot_fused(g, xp, yp, 0.75f, pol);
        ok &= fused == expect;
        std::printf("fused sharded dot over %d GPU(s), call %d: %.9g %s\n", G, call,
                    double(fused), fused == expect ? "ok" : "MISMATCH");
    }

    { // DOT over fixed global segments: the same bits for any device count
        const std::size_t seg = std::size_t(1) << 20, K = (n + seg - 1) / seg;
        float want = 0.f;
        cudaSetDevice(0);
        for (std::size_t k = 0; k < K; ++k) { // one single-GPU partial per segment, index order
            const std::size_t lo = k * seg, hi = std::min(n, lo + seg);
            Vector<float> xc(hi - lo), yc(hi - lo);
            std::copy(x.begin() + lo, x.begin() + hi, xc.begin());
            std::copy(y.begin() + lo, y.begin() + hi, yc.begin());
            want = want + dot(DeviceVector<float>(xc), DeviceVector<float>(yc), 0.0f, pol);
        }
        want = want + 0.75f;
        std::vector<DeviceVector<float>> sx, sy;
        for (int r = 0; r < G; ++r) { // device r owns a balanced run of whole segments
            const nccl::Range kr = nccl::partition(K, G, r);
            const std::size_t lo = std::min(n, kr.begin * seg), hi = std::min(n, kr.end * seg);
            Vector<float> xc(hi - lo), yc(hi - lo);
            std::copy(x.begin() + lo, x.begin() + hi, xc.begin());
            std::copy(y.begin() + lo, y.begin() + hi, yc.begin());
            cudaSetDevice(g.device(r));
            sx.emplace_back(xc);
            sy.emplace_back(yc);
        }
        std::vector<const DeviceVector<float>*> sxp, syp;
        for (int r = 0; r < G; ++r) {
            sxp.push_back(&sx[r]);
            syp.push_back(&sy[r]);
        }
        const float segd = nccl::sharded_dot_segmented(g, sxp, syp, 0.75f, seg, pol);
        ok &= segd == want;
        std::printf("segmented (device-count-invariant) dot over %d GPU(s): %.9g (expected %.9g) %s\n",
                    G, double(segd), double(want), segd == want ? "ok" : "MISMATCH");
    }

    // ---- GEMV (row blocks) and GER (row blocks)
    const std::size_t m = 8192, k = 4096;
    DenseMatrix<float> A(m, k, Layout::RowMajor), C(m, k, Layout::RowMajor);
    Vector<float> xv(k), cv(m), gx(m), gy(k);
    for (std::size_t i = 0; i < A.size(); ++i) A.data()[i] = U(rng);
    for (std::size_t i = 0; i < C.size(); ++i) C.data()[i] = U(rng);
    for (auto& v : xv) v = U(rng);
    for (auto& v : cv) v = U(rng);
    for (auto& v : gx) v = U(rng);
    for (auto& v : gy) v = U(rng);
    std::vector<DeviceMatrix<float>> Ab, Cb;
    std::vector<DeviceVector<float>> xb, cb, gxb, gyb;
    std::vector<Vector<float>> c_expect;
    std::vector<DenseMatrix<float>> C_expect;
    for (int r = 0; r < G; ++r) {
        const nccl::Range rg = nccl::partition(m, G, r);
        const std::size_t mr = rg.end - rg.begin;
        DenseMatrix<float> Ar(mr, k, Layout::RowMajor), Cr(mr, k, Layout::RowMajor);
        std::copy(A.data() + rg.begin * k, A.data() + rg.end * k, Ar.data());
        std::copy(C.data() + rg.begin * k, C.data() + rg.end * k, Cr.data());
        Vector<float> cr(mr), gxr(mr);
        std::copy(cv.begin() + rg.begin, cv.begin() + rg.end, cr.begin());
        std::copy(gx.begin() + rg.begin, gx.begin() + rg.end, gxr.begin());
        // expected: the same shard computed alone on device 0
        cudaSetDevice(0);
        {
            DeviceMatrix<float> dA(Ar), dC(Cr);
            DeviceVector<float> dx(xv), dc(cr), dgx(gxr), dgy(gy);
            gemv_row_major(dA, dx, dc, pol);
            ger(dgx, dgy, dC, pol);
            c_expect.push_back(dc.download());
            C_expect.push_back(dC.download());
        }
        cudaSetDevice(g.device(r));
        Ab.emplace_back(Ar);
        Cb.emplace_back(Cr);
        xb.emplace_back(xv);
        cb.emplace_back(cr);
        gxb.emplace_back(gxr);
        gyb.emplace_back(gy);
    }
    std::vector<const DeviceMatrix<float>*> Ap;
    std::vector<const DeviceVector<float>*> xq, gxq, gyq;
    std::vector<DeviceVector<float>*> cq;
    std::vector<DeviceMatrix<float>*> Cq;
    for (int r = 0; r < G; ++r) {
        Ap.push_back(&Ab[r]);
        xq.push_back(&xb[r]);
        cq.push_back(&cb[r]);
        gxq.push_back(&gxb[r]);
        gyq.push_back(&gyb[r]);
        Cq.push_back(&Cb[r]);
    }
    nccl::sharded_gemv_rows(g, Ap, xq, cq, pol);
    nccl::sharded_ger_rows(g, gxq, gyq, Cq, pol);
    for (int r = 0; r < G; ++r) {
        cudaSetDevice(g.device(r));
        const bool gemv_ok = cb[r].download() == c_expect[r];
        const bool ger_ok = Cb[r].download() == C_expect[r];
        ok &= gemv_ok && ger_ok;
        std::printf("rank %d: gemv rows %s, ger rows %s\n", r, gemv_ok ? "ok" : "MISMATCH",
                    ger_ok ? "ok" : "MISMATCH");
    }
    // the gathered variant: a second step on the same shards, then every
    // device holds all of c (the concatenation of the per-rank results)
    std::vector<DeviceVector<float>> full;
    std::vector<DeviceVector<float>*> fullq;
    std::vector<Vector<float>> c2_expect;
    for (int r = 0; r < G; ++r) {
        cudaSetDevice(0);
        {
            DeviceMatrix<float> dA(Ab[r].download());
            DeviceVector<float> dx(xv), dc(c_expect[r]);
            gemv_row_major(dA, dx, dc, pol);
            c2_expect.push_back(dc.download());
        }
        cudaSetDevice(g.device(r));
        full.emplace_back(m);
    }
    for (int r = 0; r < G; ++r) fullq.push_back(&full[r]);
    nccl::sharded_gemv_rows_gather(g, Ap, xq, cq, fullq, pol);
    Vector<float> want_full(m);
    for (int r = 0, o = 0; r < G; o += int(c2_expect[r].len()), ++r)
        std::copy(c2_expect[r].begin(), c2_expect[r].end(), want_full.begin() + o);
    for (int r = 0; r < G; ++r) {
        cudaSetDevice(g.device(r));
        const bool full_ok = full[r].download() == want_full;
        ok &= full_ok;
        std::printf("rank %d: gathered c %s\n", r, full_ok ? "ok" : "MISMATCH");
    }
    // the same with the gather fused into the GEMV kernel (peer memory): a third
    // step, then every device's gathered buffer is the concatenation of the
    // per-rank results (slices that do not take the sweep kernel are rejected)
    {
        std::vector<Vector<float>> c3_expect;
        for (int r = 0; r < G; ++r) {
            cudaSetDevice(0);
            DeviceMatrix<float> dA(Ab[r].download());
            DeviceVector<float> dx(xv), dc(c2_expect[r]);
            gemv_row_major(dA, dx, dc, pol);
            c3_expect.push_back(dc.download());
        }
        Vector<float> want3(m);
        for (int r = 0, o = 0; r < G; o += int(c3_expect[r].len()), ++r)
            std::copy(c3_expect[r].begin(), c3_expect[r].end(), want3.begin() + o);
        try {
            std::vector<DeviceVector<float>> full3;
            std::vector<DeviceVector<float>*> full3q;
            for (int r = 0; r < G; ++r) {
                cudaSetDevice(g.device(r));
                full3.emplace_back(m);
            }
            for (int r = 0; r < G; ++r) full3q.push_back(&full3[r]);
            nccl::sharded_gemv_rows_gather_fused(g, Ap, xq, cq, full3q, pol);
            for (int r = 0; r < G; ++r) {
                cudaSetDevice(g.device(r));
                const bool f_ok = full3[r].download() == want3 && cb[r].download() == c3_expect[r];
                ok &= f_ok;
                std::printf("rank %d: gathered c, gather fused into the kernel %s\n", r,
                            f_ok ? "ok" : "MISMATCH");
            }
        } catch (const std::invalid_argument& e) {
            std::printf("fused gather skipped: %s\n", e.what());
        }
    }
    // col-major GEMV sharded by columns: every replica of c ends equal to
    // c + the rank-ordered sum of the column blocks' partials
    {
        const std::size_t mc = 256, kc = 30001;
        DenseMatrix<float> Ac(mc, kc, Layout::ColMajor);
        Vector<float> xcv(kc), ccv(mc);
        for (std::size_t i = 0; i < Ac.size(); ++i) Ac.data()[i] = U(rng);
        for (auto& v : xcv) v = U(rng);
        for (auto& v : ccv) v = U(rng);
        std::vector<DeviceMatrix<float>> Acb;
        std::vector<DeviceVector<float>> xcb, ccb;
        Vector<float> want = ccv;
        std::vector<float> total(mc, 0.0f);
        for (int r = 0; r < G; ++r) {
            const nccl::Range rg = nccl::partition(kc, G, r);
            const std::size_t kr = rg.end - rg.begin;
            DenseMatrix<float> Ar(mc, kr, Layout::ColMajor);
            std::copy(Ac.data() + rg.begin * mc, Ac.data() + rg.end * mc, Ar.data());
            Vector<float> xr(kr);
            std::copy(xcv.begin() + rg.begin, xcv.begin() + rg.end, xr.begin());
            cudaSetDevice(0);
            {
                DeviceMatrix<float> dA(Ar);
                DeviceVector<float> dx(xr), dp(Vector<float>(mc, 0.0f));
                gemv_col_major(dA, dx, dp, pol);
                const Vector<float> p = dp.download();
                for (std::size_t i = 0; i < mc; ++i) total[i] = total[i] + p[i];
            }
            cudaSetDevice(g.device(r));
            Acb.emplace_back(Ar);
            xcb.emplace_back(xr);
            ccb.emplace_back(ccv);
        }
        for (std::size_t i = 0; i < mc; ++i) want[i] = want[i] + total[i];
        std::vector<const DeviceMatrix<float>*> Acp;
        std::vector<const DeviceVector<float>*> xcp;
        std::vector<DeviceVector<float>*> ccp;
        for (int r = 0; r < G; ++r) {
            Acp.push_back(&Acb[r]);
            xcp.push_back(&xcb[r]);
            ccp.push_back(&ccb[r]);
        }
        nccl::sharded_gemv_cols(g, Acp, xcp, ccp, pol);
        for (int r = 0; r < G; ++r) {
            cudaSetDevice(g.device(r));
            const bool cols_ok = ccb[r].download() == want;
            ok &= cols_ok;
            std::printf("rank %d: gemv by columns %s\n", r, cols_ok ? "ok" : "MISMATCH");
        }
        // again with the combine over peer memory: every replica gets the same
        // rank-ordered sum once more (want += total, in the same order)
        for (std::size_t i = 0; i < mc; ++i) want[i] = want[i] + total[i];
        nccl::sharded_gemv_cols_fused(g, Acp, xcp, ccp, pol);
        for (int r = 0; r < G; ++r) {
            cudaSetDevice(g.device(r));
            const bool cols_ok = ccb[r].download() == want;
            ok &= cols_ok;
            std::printf("rank %d: gemv by columns, combine over peer memory %s\n", r,
                        cols_ok ? "ok" : "MISMATCH");
        }
    }
    return ok ? 0 : 1;
}

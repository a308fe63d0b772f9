// The reference's hot-path test obligations, re-hosted against the B200
// drop-in header (include/cabl/kernels.hpp -> libcabl_cuda.so).
//
// Covers, case by case, what the reference checks for dot / gemv / ger
// (reference proj/tests/test_kernels.cpp:54-344) and acceptance criteria
// 1, 7 and 9 (proj/tests/acceptance.cpp:102-201, :374-391, :476-530):
// hand values, dispatch probe, oracle tolerances, GER bitwise, ragged edges,
// zero sizes, policy/alias contracts, concurrent callers, determinism and the
// 1000-instance randomized equivalence with the reference's seed and pools.
// Written without Catch2 (absent from the image): each group prints
// PASS/FAIL and the exit status is the number of failed groups.
//
// Oracles: oracle/cabl_oracle.hpp (test infrastructure).
#include <cabl/cabl.hpp>

#include "cabl_oracle.hpp"

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <random>
#include <string>
#include <thread>
#include <vector>

using namespace cabl;

namespace {

int g_failed_groups = 0;

struct Group {
    std::string name;
    int fails = 0;
    std::vector<std::string> notes;
    void expect(bool ok, const std::string& what) {
        if (!ok) {
            ++fails;
            if (notes.size() < 8) notes.push_back(what);
        }
    }
};

void run_group(const char* name, const std::function<void(Group&)>& body) {
    Group g;
    g.name = name;
    try {
        body(g);
    } catch (const std::exception& e) {
        g.expect(false, std::string("unexpected exception: ") + e.what());
    }
    std::printf("[%s] %s\n", g.fails ? "FAIL" : "PASS", name);
    for (auto& n : g.notes) std::printf("    %s\n", n.c_str());
    std::fflush(stdout);
    if (g.fails) ++g_failed_groups;
}

template <typename F>
bool throws_invalid(F&& f) {
    try {
        f();
    } catch (const std::invalid_argument&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

constexpr double kEps = std::numeric_limits<double>::epsilon();

ExecPolicy pol(unsigned threads) {
    static const BlockingPlan plan = derive_blocking_plan(default_machine());
    return ExecPolicy(plan, threads);
}

template <typename T>
Vector<T> rand_vec(std::size_t n, std::mt19937_64& rng) {
    std::uniform_real_distribution<T> d(T(-1), T(1));
    Vector<T> v(n);
    for (auto& e : v) e = d(rng);
    return v;
}

template <typename T>
DenseMatrix<T> rand_mat(std::size_t m, std::size_t n, Layout lay, std::mt19937_64& rng) {
    std::uniform_real_distribution<T> d(T(-1), T(1));
    DenseMatrix<T> A(m, n, lay);
    for (std::size_t i = 0; i < A.size(); ++i) A.data()[i] = d(rng);
    return A;
}

double sum_abs_products(const Vector<double>& x, const Vector<double>& y) {
    double s = 0;
    for (std::size_t p = 0; p < x.len(); ++p) s += std::abs(x[p] * y[p]);
    return s;
}

// per-row reference bound n*eps*sum_j |A_ij x_j| (test_kernels.cpp:42-50)
bool gemv_close(const DenseMatrix<double>& A, const Vector<double>& x, const Vector<double>& got,
                const Vector<double>& want) {
    for (std::size_t i = 0; i < got.len(); ++i) {
        double row = 0;
        for (std::size_t j = 0; j < A.cols(); ++j) row += std::abs(A(i, j) * x[j]);
        if (std::abs(got[i] - want[i]) > double(A.cols()) * kEps * row) return false;
    }
    return true;
}

} // namespace

int main() {
    std::printf("drop-in tests (B200 via libcabl_cuda.so, %d device(s))\n", cabl_device_count());

    run_group("dot hand values", [](Group& g) {
        g.expect(dot<double>({1, 2, 3}, {4, 5, 6}, 0.0, pol(1)) == 32.0, "[1,2,3].[4,5,6] == 32");
        Vector<double> x{0.5, -1.25, 3.0}, zero(3, 0.0), e1{0.0, 1.0, 0.0};
        g.expect(dot(x, zero, 7.5, pol(2)) == 7.5, "zero vector returns alpha0");
        g.expect(dot(e1, e1, 0.0, pol(2)) == 1.0, "basis dot is 1");
        g.expect(throws_invalid([&] { dot(x, Vector<double>(2), 0.0, pol(1)); }), "length mismatch throws");
    });

    run_group("dot dispatch boundary (acceptance criterion 7)", [](Group& g) {
        const ExecPolicy p = pol(4);
        std::mt19937_64 rng(7);
        const std::size_t cut = p.plan.dot_cutoff;
        auto x = rand_vec<double>(cut, rng), y = rand_vec<double>(cut, rng);
        (void)dot(x, y, 0.0, p);
        g.expect(last_exec().variant == KernelVariant::dot_small, "n == cutoff -> dot_small");
        g.expect(last_exec().threads_used == 1, "n == cutoff -> 1 worker");
        auto x1 = rand_vec<double>(cut + 1, rng), y1 = rand_vec<double>(cut + 1, rng);
        (void)dot(x1, y1, 0.0, p);
        g.expect(last_exec().variant == KernelVariant::dot_blocked, "n == cutoff+1 -> dot_blocked");
        g.expect(last_exec().threads_used >= 2, "n == cutoff+1 -> >= 2 workers");
    });

    run_group("dot vs dot_ref across thread counts", [](Group& g) {
        std::mt19937_64 rng(2);
        for (unsigned t : {1u, 2u, 4u, 8u})
            for (std::size_t n : {std::size_t(0), std::size_t(1), std::size_t(3), std::size_t(100000)}) {
                auto x = rand_vec<double>(n, rng), y = rand_vec<double>(n, rng);
                const double want = dot_ref(x, y, 0.25), got = dot(x, y, 0.25, pol(t));
                g.expect(std::abs(got - want) <= double(n) * kEps * sum_abs_products(x, y) + 4 * kEps * std::abs(want),
                         "n=" + std::to_string(n) + " threads=" + std::to_string(t));
            }
    });

    run_group("dot linearity", [](Group& g) {
        std::mt19937_64 rng(3);
        auto x = rand_vec<double>(10000, rng), y = rand_vec<double>(10000, rng);
        Vector<double> lx = x;
        for (auto& v : lx) v *= 3.5;
        const double lhs = dot(lx, y, 0.0, pol(2)), rhs = 3.5 * dot(x, y, 0.0, pol(2));
        g.expect(std::abs(lhs - rhs) <= 2 * 10000 * kEps * sum_abs_products(lx, y) + 1e-12, "dot(3.5x, y) == 3.5 dot(x, y)");
    });

    run_group("gemv_col_major vs gemv_ref", [](Group& g) {
        std::mt19937_64 rng(4);
        DenseMatrix<double> I(3, 3, Layout::ColMajor);
        for (int i = 0; i < 3; ++i) I(i, i) = 1.0;
        Vector<double> c(3, 0.0);
        gemv_col_major(I, Vector<double>{1, 2, 3}, c, pol(1));
        g.expect(c == Vector<double>{1, 2, 3}, "identity");
        auto A = rand_mat<double>(1000, 1000, Layout::ColMajor, rng);
        auto x = rand_vec<double>(1000, rng), c0 = rand_vec<double>(1000, rng);
        Vector<double> want = c0;
        gemv_ref(A, x, want);
        for (unsigned t : {1u, 4u}) {
            Vector<double> cc = c0;
            gemv_col_major(A, x, cc, pol(t));
            g.expect(gemv_close(A, x, cc, want), "random 1000x1000 threads=" + std::to_string(t));
        }
        const BlockingPlan plan = pol(1).plan;
        auto R = rand_mat<double>(plan.m_c + 1, plan.n_c + 1, Layout::ColMajor, rng);
        auto rx = rand_vec<double>(plan.n_c + 1, rng), rc = rand_vec<double>(plan.m_c + 1, rng);
        Vector<double> rwant = rc;
        gemv_ref(R, rx, rwant);
        gemv_col_major(R, rx, rc, pol(3));
        g.expect(gemv_close(R, rx, rc, rwant), "ragged m_c+1 x n_c+1");
        DenseMatrix<double> rm(4, 4, Layout::RowMajor, 1.0);
        Vector<double> c4(4, 0.0);
        g.expect(throws_invalid([&] { gemv_col_major(rm, Vector<double>(4, 1.0), c4, pol(1)); }),
                 "layout mismatch rejected");
    });

    run_group("gemv_row_major vs gemv_ref", [](Group& g) {
        std::mt19937_64 rng(5);
        DenseMatrix<double> I(3, 3, Layout::RowMajor);
        for (int i = 0; i < 3; ++i) I(i, i) = 1.0;
        Vector<double> c(3, 0.0);
        gemv_row_major(I, Vector<double>{1, 2, 3}, c, pol(2));
        g.expect(c == Vector<double>{1, 2, 3}, "identity");
        auto A = rand_mat<double>(2000, 500, Layout::RowMajor, rng);
        auto x = rand_vec<double>(500, rng), c0 = rand_vec<double>(2000, rng);
        Vector<double> want = c0;
        gemv_ref(A, x, want);
        for (unsigned t : {1u, 8u}) {
            Vector<double> cc = c0;
            gemv_row_major(A, x, cc, pol(t));
            g.expect(gemv_close(A, x, cc, want), "random 2000x500 threads=" + std::to_string(t));
        }
        const std::size_t n = 777;
        auto row = rand_mat<double>(1, n, Layout::RowMajor, rng);
        auto rx = rand_vec<double>(n, rng);
        Vector<double> rv(n);
        for (std::size_t j = 0; j < n; ++j) rv[j] = row(0, j);
        Vector<double> one{0.125};
        gemv_row_major(row, rx, one, pol(1));
        g.expect(one[0] == dot_ref(rv, rx, 0.125), "1 x 777 equals dot_ref bitwise");
        auto S = rand_mat<double>(8, 8, Layout::RowMajor, rng);
        auto sx = rand_vec<double>(8, rng);
        Vector<double> sc(8, 0.0);
        gemv_row_major(S, sx, sc, pol(8));
        g.expect(last_exec().threads_used == 1, "8x8 stays on one worker");
    });

    run_group("ger hand values and bitwise equality", [](Group& g) {
        DenseMatrix<double> C(3, 3, Layout::ColMajor, 0.0);
        ger(Vector<double>{0, 1, 0}, Vector<double>{0, 0, 1}, C, pol(1));
        bool one_elem = true;
        for (std::size_t i = 0; i < 3; ++i)
            for (std::size_t j = 0; j < 3; ++j)
                one_elem &= C(i, j) == ((i == 1 && j == 2) ? 1.0 : 0.0);
        g.expect(one_elem, "basis outer product touches exactly one element");
        DenseMatrix<double> H(2, 3, Layout::RowMajor, 0.0);
        ger(Vector<double>{1, 2}, Vector<double>{3, 4, 5}, H, pol(2));
        const double want[2][3] = {{3, 4, 5}, {6, 8, 10}};
        bool hand = true;
        for (std::size_t i = 0; i < 2; ++i)
            for (std::size_t j = 0; j < 3; ++j) hand &= H(i, j) == want[i][j];
        g.expect(hand, "[1,2] (x) [3,4,5]");
        DenseMatrix<double> M(2, 2, Layout::ColMajor);
        g.expect(throws_invalid([&] { ger(Vector<double>{1, 2}, Vector<double>{3}, M, pol(1)); }),
                 "dimension mismatch throws");
        std::mt19937_64 rng(6);
        for (Layout lay : {Layout::ColMajor, Layout::RowMajor}) {
            auto x = rand_vec<double>(500, rng), y = rand_vec<double>(500, rng);
            auto C0 = rand_mat<double>(500, 500, lay, rng);
            DenseMatrix<double> ref = C0;
            ger_ref(x, y, ref);
            for (unsigned t : {1u, 2u, 8u}) {
                DenseMatrix<double> Cg = C0;
                ger(x, y, Cg, pol(t));
                g.expect(Cg == ref, std::string("bitwise ") + layout_name(lay) + " threads=" + std::to_string(t));
            }
        }
    });

    run_group("zero-sized operands", [](Group& g) {
        Vector<double> empty;
        g.expect(dot(empty, empty, 2.5, pol(2)) == 2.5, "dot(empty) == alpha0");
        DenseMatrix<double> A0(0, 5, Layout::ColMajor);
        Vector<double> x5(5, 1.0), c0;
        gemv_col_major(A0, x5, c0, pol(2));
        DenseMatrix<double> A1(5, 0, Layout::RowMajor);
        Vector<double> x0, c5(5, 3.0);
        gemv_row_major(A1, x0, c5, pol(2));
        g.expect(c5 == Vector<double>(5, 3.0), "n = 0 keeps c");
        DenseMatrix<double> C(0, 0, Layout::ColMajor);
        ger(c0, x0, C, pol(2));
    });

    run_group("policy and alias contracts", [](Group& g) {
        const BlockingPlan plan = pol(1).plan;
        g.expect(throws_invalid([&] { ExecPolicy(plan, 0); }), "threads = 0 throws");
        g.expect(throws_invalid([&] { ExecPolicy(plan, plan.max_threads + 1); }), "threads > max throws");
        Vector<double> x{1, 2, 3};
        DenseMatrix<double> A(3, 3, Layout::ColMajor, 1.0);
        g.expect(throws_invalid([&] { gemv_col_major(A, x, x, pol(1)); }), "c aliasing x throws");
    });

    run_group("concurrent callers on disjoint outputs", [](Group& g) {
        std::mt19937_64 rng(9);
        auto A = rand_mat<double>(600, 400, Layout::ColMajor, rng);
        auto x = rand_vec<double>(400, rng);
        Vector<double> want(600, 0.0);
        gemv_ref(A, x, want);
        std::vector<Vector<double>> out(4, Vector<double>(600, 0.0));
        std::vector<std::thread> th;
        for (auto& c : out) th.emplace_back([&A, &x, &c] { gemv_col_major(A, x, c, pol(2)); });
        for (auto& t : th) t.join();
        for (auto& c : out) g.expect(gemv_close(A, x, c, want), "caller result");
    });

    run_group("float dot vs dot_ref", [](Group& g) {
        std::mt19937_64 rng(8);
        auto x = rand_vec<float>(4096, rng), y = rand_vec<float>(4096, rng);
        const float got = dot(x, y, 0.0f, pol(2)), want = dot_ref(x, y, 0.0f);
        float s = 0;
        for (std::size_t i = 0; i < 4096; ++i) s += std::abs(x[i] * y[i]);
        g.expect(std::abs(got - want) <= 4096.0f * std::numeric_limits<float>::epsilon() * s, "n = 4096");
    });

    // ---- acceptance criterion 1: randomized oracle equivalence --------------
    run_group("criterion 1: 1000 randomized instances per kernel", [](Group& g) {
        const BlockingPlan plan = derive_blocking_plan(default_machine());
        const unsigned tset[3] = {1, 2, plan.max_threads};
        std::mt19937_64 rng(20260810);
        const std::uint64_t db = plan.dot_block, dc = plan.dot_cutoff, mc = plan.m_c, mr = plan.m_r;
        const std::vector<std::uint64_t> dpool = {0, 1, 7, 8, 9, db - 1, db, db + 1, 2 * db, 3 * db,
                                                  dc - 1, dc, dc + 1, 4 * db + 13};
        const std::vector<std::uint64_t> mpool = {0, 1, mr - 1, mr, mr + 1, mc - 1, mc, mc + 1, 2 * mc, 2 * mc + 3};
        std::uniform_int_distribution<std::uint64_t> rdot(0, 30000), rdim(1, 420);
        std::uniform_int_distribution<std::size_t> pick(0, 99);
        auto dsize = [&](int i) -> std::uint64_t {
            if (i < 3) return 1000000;
            const std::size_t p = pick(rng);
            return p < 50 ? dpool[p % dpool.size()] : rdot(rng);
        };
        auto msize = [&](int i) -> std::uint64_t {
            if (i < 3) return 1000;
            const std::size_t p = pick(rng);
            return p < 50 ? mpool[p % mpool.size()] : rdim(rng);
        };
        int bad_dot = 0, bad_col = 0, bad_row = 0, bad_ger = 0;
        for (int i = 0; i < 1000; ++i) {
            const ExecPolicy p(plan, tset[i % 3]);
            const std::uint64_t n = dsize(i);
            auto x = rand_vec<double>(n, rng), y = rand_vec<double>(n, rng);
            const double want = dot_ref(x, y, 0.0), got = dot(x, y, 0.0, p);
            if (std::abs(got - want) > double(n) * kEps * sum_abs_products(x, y)) ++bad_dot;
        }
        for (int pass = 0; pass < 2; ++pass) {
            const Layout lay = pass == 0 ? Layout::ColMajor : Layout::RowMajor;
            for (int i = 0; i < 1000; ++i) {
                const ExecPolicy p(plan, tset[i % 3]);
                const std::uint64_t m = msize(i), n = msize(i);
                auto A = rand_mat<double>(m, n, lay, rng);
                auto x = rand_vec<double>(n, rng), c = rand_vec<double>(m, rng);
                Vector<double> want = c;
                gemv_ref(A, x, want);
                if (lay == Layout::ColMajor) gemv_col_major(A, x, c, p);
                else gemv_row_major(A, x, c, p);
                if (!gemv_close(A, x, c, want)) ++(pass == 0 ? bad_col : bad_row);
            }
        }
        for (int i = 0; i < 1000; ++i) {
            const ExecPolicy p(plan, tset[i % 3]);
            const std::uint64_t m = msize(i), n = msize(i);
            const Layout lay = i % 2 ? Layout::RowMajor : Layout::ColMajor;
            auto x = rand_vec<double>(m, rng), y = rand_vec<double>(n, rng);
            auto C = rand_mat<double>(m, n, lay, rng);
            DenseMatrix<double> want = C;
            ger_ref(x, y, want);
            ger(x, y, C, p);
            if (!(C == want)) ++bad_ger;
        }
        g.expect(bad_dot == 0, std::to_string(bad_dot) + " dot instances outside tolerance");
        g.expect(bad_col == 0, std::to_string(bad_col) + " gemv-col instances outside tolerance");
        g.expect(bad_row == 0, std::to_string(bad_row) + " gemv-row instances outside tolerance");
        g.expect(bad_ger == 0, std::to_string(bad_ger) + " ger instances not bitwise equal");
    });

    // ---- acceptance criterion 9: bitwise determinism over 100 trials ---------
    run_group("criterion 9: bitwise determinism across 100 runs", [](Group& g) {
        const BlockingPlan plan = derive_blocking_plan(default_machine());
        const ExecPolicy p(plan, 4);
        std::mt19937_64 rng(17);
        auto x = rand_vec<double>(3 * plan.dot_block + 7, rng), y = rand_vec<double>(3 * plan.dot_block + 7, rng);
        const double d0 = dot(x, y, 1.25, p);
        int bad = 0;
        for (int t = 0; t < 100; ++t) bad += dot(x, y, 1.25, p) != d0;
        g.expect(bad == 0, "dot varied");
        auto Ac = rand_mat<double>(700, 500, Layout::ColMajor, rng);
        auto xc = rand_vec<double>(500, rng), c0 = rand_vec<double>(700, rng);
        Vector<double> first = c0;
        gemv_col_major(Ac, xc, first, p);
        bad = 0;
        for (int t = 0; t < 100; ++t) {
            Vector<double> c = c0;
            gemv_col_major(Ac, xc, c, p);
            bad += !(c == first);
        }
        g.expect(bad == 0, "gemv-col varied");
        auto Ar = rand_mat<double>(500, 700, Layout::RowMajor, rng);
        auto xr = rand_vec<double>(700, rng), r0 = rand_vec<double>(500, rng);
        Vector<double> firstr = r0;
        gemv_row_major(Ar, xr, firstr, p);
        bad = 0;
        for (int t = 0; t < 100; ++t) {
            Vector<double> c = r0;
            gemv_row_major(Ar, xr, c, p);
            bad += !(c == firstr);
        }
        g.expect(bad == 0, "gemv-row varied");
        auto gx = rand_vec<double>(400, rng), gy = rand_vec<double>(300, rng);
        auto C0 = rand_mat<double>(400, 300, Layout::ColMajor, rng);
        DenseMatrix<double> firstC = C0;
        ger(gx, gy, firstC, p);
        bad = 0;
        for (int t = 0; t < 100; ++t) {
            DenseMatrix<double> C = C0;
            ger(gx, gy, C, p);
            bad += !(C == firstC);
        }
        g.expect(bad == 0, "ger varied");
    });

    if (g_failed_groups) std::printf("%d group(s) failed\n", g_failed_groups);
    else std::printf("all groups passed\n");
    return g_failed_groups;
}

// cabl/kernels.hpp — DROP-IN replacement of the reference hot path
// (reference proj/include/cabl/kernels.hpp).
//
// Same names, template signatures, preconditions, exception types and
// messages, dispatch probe and zero-size behaviour as the reference CPU
// templates; the bodies validate arguments and forward to the B200 C ABI
// (include/cabl_cuda.h, libcabl_cuda.so).  There is no CPU compute path: a
// missing GPU surfaces as std::runtime_error from the first call.
//
//   reference                                       here
//   ExecPolicy            kernels.hpp:28-36          ExecPolicy (same checks)
//   KernelVariant/ExecProbe/last_exec :40-55        same, fed by the C ABI probe
//   dot                   :134-164                  cabl_host_dot_{f32,f64}
//   gemv_col_major        :187-224                  cabl_host_gemv_{f32,f64}(COL_MAJOR)
//   gemv_row_major        :230-257                  cabl_host_gemv_{f32,f64}(ROW_MAJOR)
//   ger                   :277-313                  cabl_host_ger_{f32,f64}
//
// The naive oracles dot_ref / gemv_ref / ger_ref are CPU reference code, not
// part of the accelerated path; tests take them from oracle/cabl_oracle.hpp.
// Device-resident operands (no host transfers): cabl/device.hpp.
//
// Threading (reference README "Kernels run on an internal worker pool ..."):
// calls are thread-safe and may be issued concurrently on disjoint outputs;
// each call runs on the calling thread's per-thread default stream unless the
// device overloads are given an explicit stream.  policy.threads is validated
// but has no effect on the GPU launch shape.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>

#include "../cabl_cuda.h"
#include "dense.hpp"
#include "machine.hpp"

namespace cabl {

struct ExecPolicy {
    BlockingPlan plan;
    unsigned threads = 1;

    ExecPolicy(const BlockingPlan& p, unsigned t) : plan(p), threads(t) {
        if (t < 1 || t > p.max_threads)
            throw std::invalid_argument("ExecPolicy: threads must be in [1, plan.max_threads]");
    }
};

enum class KernelVariant : std::uint8_t {
    none = CABL_VARIANT_NONE,
    dot_small = CABL_VARIANT_DOT_SMALL,
    dot_blocked = CABL_VARIANT_DOT_BLOCKED,
    gemv_col_blocked = CABL_VARIANT_GEMV_COL_BLOCKED,
    gemv_row = CABL_VARIANT_GEMV_ROW,
    ger = CABL_VARIANT_GER,
};

// threads_used: CTAs of the GPU launch (1 for the ordered small-problem path).
struct ExecProbe {
    KernelVariant variant = KernelVariant::none;
    unsigned threads_used = 0;
};

inline thread_local ExecProbe g_last_exec;
inline const ExecProbe& last_exec() { return g_last_exec; }

namespace detail {

inline void require(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

inline bool aliases(const void* a, const void* b) { return a != nullptr && a == b; }

// C ABI status -> the reference's exception types.
inline void check(int rc) {
    if (rc == CABL_OK) return;
    const std::string msg = cabl_last_error();
    if (rc == CABL_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("cabl (CUDA): " + msg);
}

inline void record(const cabl_probe& p) {
    g_last_exec = ExecProbe{static_cast<KernelVariant>(p.variant), p.threads_used};
}

template <typename T>
constexpr bool supported_v = std::is_same_v<T, float> || std::is_same_v<T, double>;

// cudaStreamPerThread: concurrent callers on different host threads do not
// serialise on the legacy default stream, and each gets its own scratch.
inline void* per_thread_stream() { return reinterpret_cast<void*>(0x2); }

// one overload per element type: the C ABI is monomorphic
inline int host_dot(const float* x, const float* y, std::uint64_t n, float a, float* r,
                    std::uint64_t cut, cabl_probe* p) {
    return cabl_host_dot_f32(x, y, n, a, r, cut, p, per_thread_stream());
}
inline int host_dot(const double* x, const double* y, std::uint64_t n, double a, double* r,
                    std::uint64_t cut, cabl_probe* p) {
    return cabl_host_dot_f64(x, y, n, a, r, cut, p, per_thread_stream());
}
inline int host_gemv(const float* A, int lay, std::uint64_t m, std::uint64_t n, const float* x,
                     float* c, std::uint64_t cut, cabl_probe* p) {
    return cabl_host_gemv_f32(A, lay, m, n, x, c, cut, p, per_thread_stream());
}
inline int host_gemv(const double* A, int lay, std::uint64_t m, std::uint64_t n, const double* x,
                     double* c, std::uint64_t cut, cabl_probe* p) {
    return cabl_host_gemv_f64(A, lay, m, n, x, c, cut, p, per_thread_stream());
}
inline int host_ger(const float* x, const float* y, float* C, int lay, std::uint64_t m,
                    std::uint64_t n, std::uint64_t cut, cabl_probe* p) {
    return cabl_host_ger_f32(x, y, C, lay, m, n, cut, p, per_thread_stream());
}
inline int host_ger(const double* x, const double* y, double* C, int lay, std::uint64_t m,
                    std::uint64_t n, std::uint64_t cut, cabl_probe* p) {
    return cabl_host_ger_f64(x, y, C, lay, m, n, cut, p, per_thread_stream());
}

} // namespace detail

// ---------------------------------------------------------------------------
// DOT: alpha0 + x.y (alpha0 added last).  n <= plan.dot_cutoff reports
// dot_small / 1 thread like the reference (kernels.hpp:140-143); larger n
// reports dot_blocked / CTAs.
// ---------------------------------------------------------------------------
template <typename T>
T dot(const Vector<T>& x, const Vector<T>& y, T alpha0, const ExecPolicy& policy) {
    static_assert(detail::supported_v<T>, "cabl (B200): float and double only");
    detail::require(x.len() == y.len(), "dot: x and y lengths differ");
    const BlockingPlan& plan = policy.plan;
    if (x.len() > plan.dot_cutoff)
        detail::require(plan.dot_block >= 1, "dot: plan.dot_block must be >= 1");
    T result{};
    cabl_probe probe{};
    detail::check(detail::host_dot(x.data(), y.data(), x.len(), alpha0, &result, plan.dot_cutoff,
                                   &probe));
    detail::record(probe);
    return result;
}

// ---------------------------------------------------------------------------
// GEMV: c += A x.
// ---------------------------------------------------------------------------
template <typename T>
void gemv_col_major(const DenseMatrix<T>& A, const Vector<T>& x, Vector<T>& c,
                    const ExecPolicy& policy) {
    static_assert(detail::supported_v<T>, "cabl (B200): float and double only");
    detail::require(A.layout() == Layout::ColMajor, "gemv_col_major: matrix is not col-major");
    detail::require(A.cols() == x.len(), "gemv: A.cols != x.len");
    detail::require(A.rows() == c.len(), "gemv: A.rows != c.len");
    detail::require(!detail::aliases(c.data(), x.data()), "gemv: c must not alias x");
    const BlockingPlan& plan = policy.plan;
    detail::require(plan.m_c >= 1 && plan.n_c >= 1 && plan.m_r >= 1,
                    "gemv_col_major: plan blocks must be >= 1");
    cabl_probe probe{};
    detail::check(detail::host_gemv(A.data(), CABL_COL_MAJOR, A.rows(), A.cols(), x.data(),
                                    c.data(), plan.dot_cutoff, &probe));
    detail::record(probe);
}

template <typename T>
void gemv_row_major(const DenseMatrix<T>& A, const Vector<T>& x, Vector<T>& c,
                    const ExecPolicy& policy) {
    static_assert(detail::supported_v<T>, "cabl (B200): float and double only");
    detail::require(A.layout() == Layout::RowMajor, "gemv_row_major: matrix is not row-major");
    detail::require(A.cols() == x.len(), "gemv: A.cols != x.len");
    detail::require(A.rows() == c.len(), "gemv: A.rows != c.len");
    detail::require(!detail::aliases(c.data(), x.data()), "gemv: c must not alias x");
    cabl_probe probe{};
    detail::check(detail::host_gemv(A.data(), CABL_ROW_MAJOR, A.rows(), A.cols(), x.data(),
                                    c.data(), policy.plan.dot_cutoff, &probe));
    detail::record(probe);
}

// ---------------------------------------------------------------------------
// GER: C += x (x) y — one fused multiply-add per element, bitwise equal to
// the reference's ger / ger_ref for either layout.
// ---------------------------------------------------------------------------
template <typename T>
void ger(const Vector<T>& x, const Vector<T>& y, DenseMatrix<T>& C, const ExecPolicy& policy) {
    static_assert(detail::supported_v<T>, "cabl (B200): float and double only");
    detail::require(C.rows() == x.len(), "ger: C.rows != x.len");
    detail::require(C.cols() == y.len(), "ger: C.cols != y.len");
    detail::require(!detail::aliases(C.data(), x.data()) && !detail::aliases(C.data(), y.data()),
                    "ger: C must not alias x or y");
    cabl_probe probe{};
    const int lay = C.layout() == Layout::RowMajor ? CABL_ROW_MAJOR : CABL_COL_MAJOR;
    detail::check(detail::host_ger(x.data(), y.data(), C.data(), lay, C.rows(), C.cols(),
                                   policy.plan.dot_cutoff, &probe));
    detail::record(probe);
}

} // namespace cabl

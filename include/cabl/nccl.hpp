// cabl/nccl.hpp — multi-GPU DOT / GEMV / GER for C++ callers, one process
// driving G devices (NVLink 5 / NVSwitch), the process model of SURVEY.md
// §8(e).  A thin RAII layer over the multi-GPU C ABI (cabl_mgpu_*,
// include/cabl_cuda.h), so C++ and FFI callers share one implementation:
// NCCL is loaded by libcabl_cuda.so at run time (no -lnccl here), every call
// validates all shards before launching anything, and returns only when all
// devices are done — an NCCL error, an asynchronous NCCL error, a timed-out
// peer exchange or the Group's timeout throws ExchangeError after aborting
// the communicators (the reference pool rethrows worker failures to the
// caller, thread_pool.hpp:63-68; nothing hangs).  (Python callers with one
// process per GPU use paper_2108_02025_b200/shard.py.)
//
// Partitioning (reference parallel_chunks, thread_pool.hpp:153-164, lifted to
// devices): balanced contiguous ranges (partition()).
//   DOT   chunks of x and y; per-device partial (alpha0 = 0); the G partials
//         summed in device order on every device, alpha0 last, as the
//         reference combines thread partials (kernels.hpp:160-163) — the
//         result is independent of the collective's algorithm.
//   GEMV  row blocks of A and c, x replicated; optionally the full c on every
//         device.  Col-major A by column blocks: rank-ordered sum of partials.
//   GER   row blocks of C and x, y replicated, no exchange at all.
// The *_fused variants run the exchange inside the kernels over NVLink P2P
// (csrc/peer.cu, peer_gemv.cu) instead of NCCL collectives: same bits.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "device.hpp"

namespace cabl::nccl {

// CABL_ENCCL: the exchange failed and the Group's communicators are aborted;
// the Group must be destroyed (every later call throws again).
struct ExchangeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void mgpu_check(int rc) {
    if (rc == CABL_OK) return;
    const std::string msg = cabl_last_error();
    if (rc == CABL_EINVAL) throw std::invalid_argument(msg);
    if (rc == CABL_ENCCL) throw ExchangeError(msg);
    throw std::runtime_error(msg);
}

struct Range {
    std::uint64_t begin, end;
};

// balanced contiguous split: the first total % parts ranges get one extra
inline Range partition(std::uint64_t total, int parts, int rank) {
    const std::uint64_t q = total / parts, r = total % parts;
    const std::uint64_t b = rank * q + (std::uint64_t(rank) < r ? rank : r);
    return Range{b, b + q + (std::uint64_t(rank) < r ? 1 : 0)};
}

// One communicator clique over `devices` with one stream each (a cabl_mgpu
// context).  Rank r is devices[r].
class Group {
public:
    explicit Group(const std::vector<int>& devices) {
        mgpu_check(cabl_mgpu_init(devices.data(), int(devices.size()), &ctx_));
    }
    Group(const Group&) = delete;
    Group& operator=(const Group&) = delete;
    ~Group() { cabl_mgpu_finalize(ctx_); }
    int size() const { return cabl_mgpu_size(ctx_); }
    int device(int r) const { return cabl_mgpu_device(ctx_, r); }
    cudaStream_t stream(int r) const { return static_cast<cudaStream_t>(cabl_mgpu_stream(ctx_, r)); }
    cabl_mgpu* handle() const { return ctx_; }
    void set_timeout_ms(std::uint64_t ms) { mgpu_check(cabl_mgpu_set_timeout_ms(ctx_, ms)); }
    void synchronize() const {
        for (int r = 0; r < size(); ++r) {
            detail::cuda_check(cudaSetDevice(device(r)), "cudaSetDevice");
            detail::cuda_check(cudaStreamSynchronize(stream(r)), "sync");
        }
    }

private:
    cabl_mgpu* ctx_ = nullptr;
};

namespace detail {
inline int mdot(cabl_mgpu* c, const float* const* x, const float* const* y, const std::uint64_t* n,
                float a, std::uint64_t cut, int ex, float* out) {
    return cabl_mgpu_dot_f32(c, x, y, n, a, cut, ex, out);
}
inline int mdot(cabl_mgpu* c, const double* const* x, const double* const* y,
                const std::uint64_t* n, double a, std::uint64_t cut, int ex, double* out) {
    return cabl_mgpu_dot_f64(c, x, y, n, a, cut, ex, out);
}
inline int mdot_seg(cabl_mgpu* c, const float* const* x, const float* const* y,
                    const std::uint64_t* n, std::uint64_t seg, float a, std::uint64_t cut,
                    float* out) {
    return cabl_mgpu_dot_segmented_f32(c, x, y, n, seg, a, cut, out);
}
inline int mdot_seg(cabl_mgpu* c, const double* const* x, const double* const* y,
                    const std::uint64_t* n, std::uint64_t seg, double a, std::uint64_t cut,
                    double* out) {
    return cabl_mgpu_dot_segmented_f64(c, x, y, n, seg, a, cut, out);
}
inline int mgemv_rm(cabl_mgpu* c, const float* const* A, const std::uint64_t* m, std::uint64_t n,
                    const float* const* x, float* const* cs, std::uint64_t cut, int ex,
                    float* const* full) {
    return cabl_mgpu_gemv_rm_f32(c, A, m, n, x, cs, cut, ex, full);
}
inline int mgemv_rm(cabl_mgpu* c, const double* const* A, const std::uint64_t* m, std::uint64_t n,
                    const double* const* x, double* const* cs, std::uint64_t cut, int ex,
                    double* const* full) {
    return cabl_mgpu_gemv_rm_f64(c, A, m, n, x, cs, cut, ex, full);
}
inline int mgemv_cols(cabl_mgpu* c, const float* const* A, std::uint64_t m, const std::uint64_t* n,
                      const float* const* x, float* const* cs, std::uint64_t cut, int ex) {
    return cabl_mgpu_gemv_cm_cols_f32(c, A, m, n, x, cs, cut, ex);
}
inline int mgemv_cols(cabl_mgpu* c, const double* const* A, std::uint64_t m, const std::uint64_t* n,
                      const double* const* x, double* const* cs, std::uint64_t cut, int ex) {
    return cabl_mgpu_gemv_cm_cols_f64(c, A, m, n, x, cs, cut, ex);
}
inline int mger(cabl_mgpu* c, const float* const* x, const std::uint64_t* m, const float* const* y,
                std::uint64_t n, float* const* C, std::uint64_t cut) {
    return cabl_mgpu_ger_rm_f32(c, x, m, y, n, C, cut);
}
inline int mger(cabl_mgpu* c, const double* const* x, const std::uint64_t* m,
                const double* const* y, std::uint64_t n, double* const* C, std::uint64_t cut) {
    return cabl_mgpu_ger_rm_f64(c, x, m, y, n, C, cut);
}

inline void need(bool ok, const std::string& msg) {
    if (!ok) throw std::invalid_argument(msg);
}
inline void one_per_device(const Group& g, std::size_t k, const char* what) {
    need(int(k) == g.size(), std::string(what) + ": one shard per device");
}

template <typename T>
T dot_common(Group& g, const std::vector<const DeviceVector<T>*>& x,
             const std::vector<const DeviceVector<T>*>& y, T alpha0, const ExecPolicy& policy,
             int exchange, const char* what) {
    one_per_device(g, x.size(), what);
    one_per_device(g, y.size(), what);
    std::vector<const T*> xp, yp;
    std::vector<std::uint64_t> n;
    for (int r = 0; r < g.size(); ++r) {
        need(x[r]->len() == y[r]->len(), "dot: x and y lengths differ");
        xp.push_back(x[r]->data());
        yp.push_back(y[r]->data());
        n.push_back(x[r]->len());
    }
    T out{};
    mgpu_check(mdot(g.handle(), xp.data(), yp.data(), n.data(), alpha0, policy.plan.dot_cutoff,
                    exchange, &out));
    return out;
}

template <typename T>
void gemv_rows_common(Group& g, const std::vector<const DeviceMatrix<T>*>& A,
                      const std::vector<const DeviceVector<T>*>& x,
                      const std::vector<DeviceVector<T>*>& c,
                      const std::vector<DeviceVector<T>*>* c_full, const ExecPolicy& policy,
                      int exchange, const char* what) {
    one_per_device(g, A.size(), what);
    one_per_device(g, x.size(), what);
    one_per_device(g, c.size(), what);
    const int G = g.size();
    std::vector<const T*> Ap, xp;
    std::vector<T*> cp, fp;
    std::vector<std::uint64_t> m;
    std::uint64_t total = 0;
    const std::size_t n = A[0]->cols();
    for (int r = 0; r < G; ++r) {
        need(A[r]->layout() == Layout::RowMajor, "gemv_row_major: matrix is not row-major");
        need(A[r]->cols() == x[r]->len(), "gemv: A.cols != x.len");
        need(A[r]->rows() == c[r]->len(), "gemv: A.rows != c.len");
        need(A[r]->cols() == n, std::string(what) + ": every row block must have the same columns");
        Ap.push_back(A[r]->data());
        xp.push_back(x[r]->data());
        cp.push_back(c[r]->data());
        m.push_back(A[r]->rows());
        total += A[r]->rows();
    }
    if (c_full) {
        one_per_device(g, c_full->size(), what);
        for (int r = 0; r < G; ++r) {
            need((*c_full)[r]->len() == total, std::string(what) + ": c_full length != sum of the slices");
            fp.push_back((*c_full)[r]->data());
        }
    }
    mgpu_check(mgemv_rm(g.handle(), Ap.data(), m.data(), n, xp.data(), cp.data(),
                        policy.plan.dot_cutoff, exchange, c_full ? fp.data() : nullptr));
}

template <typename T>
void gemv_cols_common(Group& g, const std::vector<const DeviceMatrix<T>*>& A,
                      const std::vector<const DeviceVector<T>*>& x,
                      const std::vector<DeviceVector<T>*>& c, const ExecPolicy& policy,
                      int exchange, const char* what) {
    one_per_device(g, A.size(), what);
    one_per_device(g, x.size(), what);
    one_per_device(g, c.size(), what);
    const std::size_t m = c[0]->len();
    std::vector<const T*> Ap, xp;
    std::vector<T*> cp;
    std::vector<std::uint64_t> n;
    for (int r = 0; r < g.size(); ++r) {
        need(A[r]->layout() == Layout::ColMajor, "gemv_col_major: matrix is not col-major");
        need(A[r]->cols() == x[r]->len(), "gemv: A.cols != x.len");
        need(A[r]->rows() == m && c[r]->len() == m,
             "sharded_gemv_cols: col-major blocks of m rows, c replicas of length m");
        Ap.push_back(A[r]->data());
        xp.push_back(x[r]->data());
        cp.push_back(c[r]->data());
        n.push_back(A[r]->cols());
    }
    mgpu_check(mgemv_cols(g.handle(), Ap.data(), m, n.data(), xp.data(), cp.data(),
                          policy.plan.dot_cutoff, exchange));
}
} // namespace detail

// alpha0 + x.y with x, y given as per-device chunks (x[r], y[r] on
// g.device(r)).  The device partials are exchanged with an NCCL all-gather
// and summed in rank order on every device.
template <typename T>
T sharded_dot(Group& g, const std::vector<const DeviceVector<T>*>& x,
              const std::vector<const DeviceVector<T>*>& y, T alpha0, const ExecPolicy& policy) {
    return detail::dot_common(g, x, y, alpha0, policy, CABL_MGPU_NCCL, "sharded_dot");
}

// DOT over fixed global segments of `segment` elements (the shards, concatenated
// in device order, cut every `segment` elements; every shard before the last
// non-empty one a whole number of segments): one partial per segment, summed in
// index order.  The result is bit for bit the same for any number of devices.
template <typename T>
T sharded_dot_segmented(Group& g, const std::vector<const DeviceVector<T>*>& x,
                        const std::vector<const DeviceVector<T>*>& y, T alpha0,
                        std::uint64_t segment, const ExecPolicy& policy) {
    detail::one_per_device(g, x.size(), "sharded_dot_segmented");
    detail::one_per_device(g, y.size(), "sharded_dot_segmented");
    std::vector<const T*> xp, yp;
    std::vector<std::uint64_t> n;
    for (int r = 0; r < g.size(); ++r) {
        detail::need(x[r]->len() == y[r]->len(), "dot: x and y lengths differ");
        xp.push_back(x[r]->data());
        yp.push_back(y[r]->data());
        n.push_back(x[r]->len());
    }
    T out{};
    mgpu_check(detail::mdot_seg(g.handle(), xp.data(), yp.data(), n.data(), segment,
                                        alpha0, policy.plan.dot_cutoff, &out));
    return out;
}

// sharded_dot with the exchange fused into the DOT kernel (peer memory, no
// NCCL): same arguments, same bits.
template <typename T>
T sharded_dot_fused(Group& g, const std::vector<const DeviceVector<T>*>& x,
                    const std::vector<const DeviceVector<T>*>& y, T alpha0,
                    const ExecPolicy& policy) {
    return detail::dot_common(g, x, y, alpha0, policy, CABL_MGPU_PEER, "sharded_dot_fused");
}

// c[r] += A[r] x[r] on every device's row block (no exchange).  Row-major
// blocks go through one cabl_mgpu call; col-major row blocks (each device's
// own m_r x n col-major matrix) through the single-GPU kernel per device.
template <typename T>
void sharded_gemv_rows(Group& g, const std::vector<const DeviceMatrix<T>*>& A,
                       const std::vector<const DeviceVector<T>*>& x,
                       const std::vector<DeviceVector<T>*>& c, const ExecPolicy& policy) {
    detail::one_per_device(g, A.size(), "sharded_gemv_rows");
    bool row_major = true;
    for (const auto* a : A) row_major &= a->layout() == Layout::RowMajor;
    if (row_major) {
        detail::gemv_rows_common(g, A, x, c, static_cast<const std::vector<DeviceVector<T>*>*>(nullptr),
                                 policy, CABL_MGPU_NCCL, "sharded_gemv_rows");
        return;
    }
    for (int r = 0; r < g.size(); ++r) {
        cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
        if (A[r]->layout() == Layout::RowMajor)
            gemv_row_major(*A[r], *x[r], *c[r], policy, g.stream(r));
        else
            gemv_col_major(*A[r], *x[r], *c[r], policy, g.stream(r));
    }
    g.synchronize();
}

// The same on row-major blocks, then every device assembles the full c
// ("output slices optionally all-gathered"): c_full[r] (length
// sum of the slices, on g.device(r)) receives slice q at offset
// sum_{p<q} |c[p]| (grouped ncclBroadcast per source rank: unequal slices
// need no padding).
template <typename T>
void sharded_gemv_rows_gather(Group& g, const std::vector<const DeviceMatrix<T>*>& A,
                              const std::vector<const DeviceVector<T>*>& x,
                              const std::vector<DeviceVector<T>*>& c,
                              const std::vector<DeviceVector<T>*>& c_full,
                              const ExecPolicy& policy) {
    detail::gemv_rows_common(g, A, x, c, &c_full, policy, CABL_MGPU_NCCL,
                             "sharded_gemv_rows_gather");
}

// sharded_gemv_rows_gather with the gather fused into the GEMV kernel (peer
// memory, no NCCL): every device's rows are stored into every device's
// gathered buffer as they finish, then copied to c_full.  Slices that do not
// take the sweep kernel (few or short rows, unaligned) throw
// std::invalid_argument before any kernel runs — use sharded_gemv_rows_gather.
template <typename T>
void sharded_gemv_rows_gather_fused(Group& g, const std::vector<const DeviceMatrix<T>*>& A,
                                    const std::vector<const DeviceVector<T>*>& x,
                                    const std::vector<DeviceVector<T>*>& c,
                                    const std::vector<DeviceVector<T>*>& c_full,
                                    const ExecPolicy& policy) {
    detail::gemv_rows_common(g, A, x, c, &c_full, policy, CABL_MGPU_PEER,
                             "sharded_gemv_rows_gather_fused");
}

// Col-major GEMV sharded by columns (short-wide shapes): A[r] is device r's
// column block (m x n_r, col-major), x[r] the matching slice of x, c[r] a
// replica of c.  Each device computes its partial from zero; every replica
// gets c += the rank-ordered sum of the partials (all-gather +
// combine_rows), so all devices end with the same bits.
template <typename T>
void sharded_gemv_cols(Group& g, const std::vector<const DeviceMatrix<T>*>& A,
                       const std::vector<const DeviceVector<T>*>& x,
                       const std::vector<DeviceVector<T>*>& c, const ExecPolicy& policy) {
    detail::gemv_cols_common(g, A, x, c, policy, CABL_MGPU_NCCL, "sharded_gemv_cols");
}

// sharded_gemv_cols with the all-gather + combine replaced by one peer-memory
// kernel per device (cabl_cuda_combine_rows_peer_*): same bits, no NCCL call.
template <typename T>
void sharded_gemv_cols_fused(Group& g, const std::vector<const DeviceMatrix<T>*>& A,
                             const std::vector<const DeviceVector<T>*>& x,
                             const std::vector<DeviceVector<T>*>& c, const ExecPolicy& policy) {
    detail::gemv_cols_common(g, A, x, c, policy, CABL_MGPU_PEER, "sharded_gemv_cols_fused");
}

// C[r] += x[r] (x) y[r] on every device's row block (no communication).
template <typename T>
void sharded_ger_rows(Group& g, const std::vector<const DeviceVector<T>*>& x,
                      const std::vector<const DeviceVector<T>*>& y,
                      const std::vector<DeviceMatrix<T>*>& C, const ExecPolicy& policy) {
    detail::one_per_device(g, x.size(), "sharded_ger_rows");
    detail::one_per_device(g, y.size(), "sharded_ger_rows");
    detail::one_per_device(g, C.size(), "sharded_ger_rows");
    bool row_major = true;
    for (const auto* m : C) row_major &= m->layout() == Layout::RowMajor;
    if (!row_major) { // col-major blocks: the single-GPU kernel per device
        for (int r = 0; r < g.size(); ++r) {
            cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
            ger(*x[r], *y[r], *C[r], policy, g.stream(r));
        }
        g.synchronize();
        return;
    }
    const std::size_t n = C[0]->cols();
    std::vector<const T*> xp, yp;
    std::vector<T*> Cp;
    std::vector<std::uint64_t> m;
    for (int r = 0; r < g.size(); ++r) {
        detail::need(C[r]->rows() == x[r]->len(), "ger: C.rows != x.len");
        detail::need(C[r]->cols() == y[r]->len(), "ger: C.cols != y.len");
        detail::need(C[r]->cols() == n, "sharded_ger_rows: every row block must have the same columns");
        xp.push_back(x[r]->data());
        yp.push_back(y[r]->data());
        Cp.push_back(C[r]->data());
        m.push_back(C[r]->rows());
    }
    mgpu_check(detail::mger(g.handle(), xp.data(), m.data(), yp.data(), n, Cp.data(),
                            policy.plan.dot_cutoff));
}

} // namespace cabl::nccl

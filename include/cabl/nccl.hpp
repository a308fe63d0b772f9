// cabl/nccl.hpp — multi-GPU DOT / GEMV / GER for C++ callers, one process
// driving G devices over NCCL (NVLink 5 / NVSwitch), the process model of
// SURVEY.md §8(e).  (Python callers use paper_2108_02025_b200/shard.py: one
// process per GPU under torchrun.)
//
// Partitioning (reference parallel_chunks, thread_pool.hpp:153-164, lifted to
// devices): balanced contiguous ranges.
//   DOT   chunks of x and y; each device computes its partial with alpha0 = 0;
//         one ncclAllGather of the G partials; each device sums them in device
//         order and adds alpha0 last (cabl_cuda_combine_partials_*), as the
//         reference combines thread partials (kernels.hpp:160-163) — the
//         result is independent of NCCL's algorithm and identical everywhere.
//   GEMV  row blocks of A and c, x replicated, no exchange needed.
//   GER   row blocks of C and x, y replicated, no exchange at all.
//   sharded_gemv_cols_fused: the column-block partials combined by one
//         peer-memory kernel per device instead of all-gather + combine_rows.
//   sharded_gemv_rows_gather_fused: the c all-gather inside the GEMV kernel —
//         rows stored into every device's double-buffered gathered c over P2P.
//   sharded_dot_fused: DOT with the exchange inside the kernel — every device
//         stores its partial into every device's mailbox over NVLink P2P and
//         sums the G partials in device order itself (cabl_cuda_dot_peer_*,
//         csrc/peer.cu); same bits as sharded_dot, one kernel, no NCCL call.
//
// Needs nccl.h and -lnccl in addition to cabl/device.hpp's requirements.
#pragma once

#include <nccl.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "device.hpp"

namespace cabl::nccl {

inline void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + ncclGetErrorString(r));
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

// One communicator clique over `devices` (ncclCommInitAll), one stream each.
class Group {
public:
    explicit Group(std::vector<int> devices) : devs_(std::move(devices)) {
        comms_.resize(devs_.size());
        nccl_check(ncclCommInitAll(comms_.data(), int(devs_.size()), devs_.data()), "ncclCommInitAll");
        for (int d : devs_) {
            detail::cuda_check(cudaSetDevice(d), "cudaSetDevice");
            cudaStream_t s;
            detail::cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
            streams_.push_back(s);
        }
    }
    Group(const Group&) = delete;
    Group& operator=(const Group&) = delete;
    ~Group() {
        free_gather();
        for (std::size_t i = 0; i < mboxes_.size(); ++i) {
            cudaSetDevice(devs_[i]);
            cabl_peer_mailbox_destroy(mboxes_[i]);
        }
        for (std::size_t i = 0; i < devs_.size(); ++i) {
            cudaSetDevice(devs_[i]);
            cudaStreamDestroy(streams_[i]);
            ncclCommDestroy(comms_[i]);
        }
    }
    int size() const { return int(devs_.size()); }
    int device(int r) const { return devs_[r]; }
    ncclComm_t comm(int r) const { return comms_[r]; }
    cudaStream_t stream(int r) const { return streams_[r]; }
    void synchronize() const {
        for (int r = 0; r < size(); ++r) {
            detail::cuda_check(cudaSetDevice(devs_[r]), "cudaSetDevice");
            detail::cuda_check(cudaStreamSynchronize(streams_[r]), "sync");
        }
    }

    // Peer-DOT mailboxes, one per device, created on first use; every device
    // gets P2P access to every other (NVLink), so the table holds plain
    // device pointers (no IPC inside one process).
    void* const* mailboxes() {
        if (mboxes_.empty()) {
            enable_peer_access();
            for (int r = 0; r < size(); ++r) {
                detail::cuda_check(cudaSetDevice(devs_[r]), "cudaSetDevice");
                void* mb = nullptr;
                detail::check(cabl_peer_mailbox_create(&mb));
                mboxes_.push_back(mb);
            }
        }
        return mboxes_.data();
    }

    // Gathered-c buffers (2 x bytes_half each, one per device) and their own
    // mailboxes for the fused GEMV gather; reallocated when the size changes.
    struct Gather {
        std::vector<void*> bufs, mboxes;
        std::size_t bytes_half = 0;
        std::uint64_t calls = 0;
    };
    Gather& gather(std::size_t bytes_half) {
        if (gather_.bytes_half != bytes_half) {
            free_gather();
            enable_peer_access();
            for (int r = 0; r < size(); ++r) {
                detail::cuda_check(cudaSetDevice(devs_[r]), "cudaSetDevice");
                void* b = nullptr;
                void* mb = nullptr;
                detail::check(cabl_peer_alloc(2 * bytes_half, &b));
                detail::check(cabl_peer_mailbox_create(&mb));
                gather_.bufs.push_back(b);
                gather_.mboxes.push_back(mb);
            }
            gather_.bytes_half = bytes_half;
            gather_.calls = 0;
        }
        return gather_;
    }

    // Slot buffers (2 x 8 x m values each, one per device) and mailboxes for
    // the peer-memory row combine; reallocated when the size changes.
    Gather& rows(std::size_t bytes_slots) {
        if (rows_.bytes_half != bytes_slots) {
            free_set(rows_);
            enable_peer_access();
            for (int r = 0; r < size(); ++r) {
                detail::cuda_check(cudaSetDevice(devs_[r]), "cudaSetDevice");
                void* b = nullptr;
                void* mb = nullptr;
                detail::check(cabl_peer_alloc(bytes_slots, &b));
                detail::check(cabl_peer_mailbox_create(&mb));
                rows_.bufs.push_back(b);
                rows_.mboxes.push_back(mb);
            }
            rows_.bytes_half = bytes_slots;
        }
        return rows_;
    }

private:
    void free_set(Gather& st) {
        for (std::size_t i = 0; i < st.bufs.size(); ++i) {
            cudaSetDevice(devs_[i]);
            cabl_peer_free(st.bufs[i]);
            cabl_peer_mailbox_destroy(st.mboxes[i]);
        }
        st = Gather{};
    }
    void enable_peer_access() {
        if (peer_enabled_) return;
        const int G = size();
        for (int r = 0; r < G; ++r) {
            detail::cuda_check(cudaSetDevice(devs_[r]), "cudaSetDevice");
            for (int q = 0; q < G; ++q) {
                if (q == r) continue;
                int can = 0;
                detail::cuda_check(cudaDeviceCanAccessPeer(&can, devs_[r], devs_[q]),
                                   "cudaDeviceCanAccessPeer");
                if (!can) throw std::runtime_error("peer-memory path: no P2P path between devices");
                const cudaError_t e = cudaDeviceEnablePeerAccess(devs_[q], 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else detail::cuda_check(e, "cudaDeviceEnablePeerAccess");
            }
        }
        peer_enabled_ = true;
    }
    void free_gather() {
        free_set(gather_);
        free_set(rows_);
    }

    std::vector<int> devs_;
    std::vector<ncclComm_t> comms_;
    std::vector<cudaStream_t> streams_;
    std::vector<void*> mboxes_;
    Gather gather_, rows_;
    bool peer_enabled_ = false;
};

namespace detail {
template <typename T> ncclDataType_t nccl_type();
template <> inline ncclDataType_t nccl_type<float>() { return ncclFloat32; }
template <> inline ncclDataType_t nccl_type<double>() { return ncclFloat64; }
inline int combine(const float* p, std::uint32_t k, float a, float* o, cudaStream_t s) {
    return cabl_cuda_combine_partials_f32(p, k, a, o, s);
}
inline int combine(const double* p, std::uint32_t k, double a, double* o, cudaStream_t s) {
    return cabl_cuda_combine_partials_f64(p, k, a, o, s);
}
inline int combine_rows(const float* p, std::uint32_t k, std::uint64_t m, float* c, cudaStream_t s) {
    return cabl_cuda_combine_rows_f32(p, k, m, c, s);
}
inline int combine_rows(const double* p, std::uint32_t k, std::uint64_t m, double* c,
                        cudaStream_t s) {
    return cabl_cuda_combine_rows_f64(p, k, m, c, s);
}
inline int dot_peer(const float* x, const float* y, std::uint64_t n, float a, float* o,
                    void* const* mb, int G, int r, std::uint64_t cut, cudaStream_t s) {
    return cabl_cuda_dot_peer_f32(x, y, n, a, o, mb, G, r, cut, nullptr, s);
}
inline int dot_peer(const double* x, const double* y, std::uint64_t n, double a, double* o,
                    void* const* mb, int G, int r, std::uint64_t cut, cudaStream_t s) {
    return cabl_cuda_dot_peer_f64(x, y, n, a, o, mb, G, r, cut, nullptr, s);
}
inline int gemv_gather(const float* A, std::uint64_t m, std::uint64_t n, const float* x, float* c,
                       std::uint64_t off, std::uint64_t mt, void* const* b, void* const* mb, int G,
                       int r, cudaStream_t s) {
    return cabl_cuda_gemv_rm_gather_f32(A, m, n, x, c, off, mt, b, mb, G, r, nullptr, s);
}
inline int gemv_gather(const double* A, std::uint64_t m, std::uint64_t n, const double* x,
                       double* c, std::uint64_t off, std::uint64_t mt, void* const* b,
                       void* const* mb, int G, int r, cudaStream_t s) {
    return cabl_cuda_gemv_rm_gather_f64(A, m, n, x, c, off, mt, b, mb, G, r, nullptr, s);
}
inline int rows_peer(const float* p, std::uint64_t m, float* c, void* const* b, void* const* mb,
                     int G, int r, cudaStream_t s) {
    return cabl_cuda_combine_rows_peer_f32(p, m, c, b, mb, G, r, s);
}
inline int rows_peer(const double* p, std::uint64_t m, double* c, void* const* b,
                     void* const* mb, int G, int r, cudaStream_t s) {
    return cabl_cuda_combine_rows_peer_f64(p, m, c, b, mb, G, r, s);
}
} // namespace detail

// alpha0 + x.y with x, y given as per-device chunks (x[r], y[r] on
// g.device(r), equal lengths per rank).  Returns the host value (every device
// holds the same bits in its `out`).
template <typename T>
T sharded_dot(Group& g, const std::vector<const DeviceVector<T>*>& x,
              const std::vector<const DeviceVector<T>*>& y, T alpha0, const ExecPolicy& policy) {
    const int G = g.size();
    cabl::detail::require(int(x.size()) == G && int(y.size()) == G, "sharded_dot: one chunk per device");
    std::vector<DeviceVector<T>> partial, gathered, out;
    for (int r = 0; r < G; ++r) {
        cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
        partial.emplace_back(1);
        gathered.emplace_back(std::size_t(G));
        out.emplace_back(1);
        dot_async(*x[r], *y[r], T(0), partial[r].data(), policy, g.stream(r));
    }
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (int r = 0; r < G; ++r)
        nccl_check(ncclAllGather(partial[r].data(), gathered[r].data(), 1, detail::nccl_type<T>(),
                                 g.comm(r), g.stream(r)),
                   "ncclAllGather");
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
    for (int r = 0; r < G; ++r) {
        cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
        cabl::detail::check(detail::combine(gathered[r].data(), std::uint32_t(G), alpha0,
                                            out[r].data(), g.stream(r)));
    }
    T result{};
    cabl::detail::cuda_check(cudaSetDevice(g.device(0)), "cudaSetDevice");
    cabl::detail::cuda_check(cudaMemcpyAsync(&result, out[0].data(), sizeof(T),
                                             cudaMemcpyDeviceToHost, g.stream(0)), "D2H");
    g.synchronize();
    return result;
}

// sharded_dot with the exchange fused into the DOT kernel (peer memory, no
// NCCL): same arguments, same bits.  All G kernels are enqueued before any
// is waited on; each spins only for its peers' partials.
template <typename T>
T sharded_dot_fused(Group& g, const std::vector<const DeviceVector<T>*>& x,
                    const std::vector<const DeviceVector<T>*>& y, T alpha0,
                    const ExecPolicy& policy) {
    const int G = g.size();
    cabl::detail::require(int(x.size()) == G && int(y.size()) == G,
                          "sharded_dot_fused: one chunk per device");
    void* const* mb = g.mailboxes();
    std::vector<DeviceVector<T>> out;
    for (int r = 0; r < G; ++r) {
        cabl::detail::require(x[r]->len() == y[r]->len(), "Vectors must have equal length");
        cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
        out.emplace_back(1);
        cabl::detail::check(detail::dot_peer(x[r]->data(), y[r]->data(), x[r]->len(), alpha0,
                                             out[r].data(), mb, G, r, policy.plan.dot_cutoff,
                                             g.stream(r)));
    }
    T result{};
    cabl::detail::cuda_check(cudaSetDevice(g.device(0)), "cudaSetDevice");
    cabl::detail::cuda_check(cudaMemcpyAsync(&result, out[0].data(), sizeof(T),
                                             cudaMemcpyDeviceToHost, g.stream(0)), "D2H");
    g.synchronize();
    return result;
}

// c[r] += A[r] x[r] on every device's row block (no exchange).
template <typename T>
void sharded_gemv_rows(Group& g, const std::vector<const DeviceMatrix<T>*>& A,
                       const std::vector<const DeviceVector<T>*>& x,
                       const std::vector<DeviceVector<T>*>& c, const ExecPolicy& policy) {
    for (int r = 0; r < g.size(); ++r) {
        cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
        if (A[r]->layout() == Layout::RowMajor)
            gemv_row_major(*A[r], *x[r], *c[r], policy, g.stream(r));
        else
            gemv_col_major(*A[r], *x[r], *c[r], policy, g.stream(r));
    }
    g.synchronize();
}

// The same, then every device assembles the full c ("output
// slices optionally all-gathered"): c_full[r] (length sum of the slices, on
// g.device(r)) receives slice q at offset sum_{p<q} |c[p]| through one
// ncclBroadcast per source rank, grouped — unequal slices need no padding.
template <typename T>
void sharded_gemv_rows_gather(Group& g, const std::vector<const DeviceMatrix<T>*>& A,
                              const std::vector<const DeviceVector<T>*>& x,
                              const std::vector<DeviceVector<T>*>& c,
                              const std::vector<DeviceVector<T>*>& c_full,
                              const ExecPolicy& policy) {
    const int G = g.size();
    cabl::detail::require(int(c_full.size()) == G, "sharded_gemv_rows_gather: one c_full per device");
    std::vector<std::size_t> off(std::size_t(G) + 1, 0);
    for (int q = 0; q < G; ++q) off[q + 1] = off[q] + c[q]->len();
    for (int r = 0; r < G; ++r)
        cabl::detail::require(c_full[r]->len() == off[G], "sharded_gemv_rows_gather: c_full length");
    for (int r = 0; r < G; ++r) {
        cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
        if (A[r]->layout() == Layout::RowMajor)
            gemv_row_major(*A[r], *x[r], *c[r], policy, g.stream(r));
        else
            gemv_col_major(*A[r], *x[r], *c[r], policy, g.stream(r));
    }
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (int q = 0; q < G; ++q)
        for (int r = 0; r < G; ++r)
            nccl_check(ncclBroadcast(r == q ? c[q]->data() : nullptr, c_full[r]->data() + off[q],
                                     c[q]->len(), detail::nccl_type<T>(), q, g.comm(r),
                                     g.stream(r)),
                       "ncclBroadcast");
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
    g.synchronize();
}

// sharded_gemv_rows_gather with the gather fused into the GEMV kernel (peer
// memory, no NCCL): every device's slice update is stored into every device's
// gathered buffer as its rows finish.  Returns, per device, a device pointer
// to the full c (sum of the slice lengths), valid until the call after next
// on this Group.  Row-major slices that take the sweep kernel only (long
// aligned rows, enough of them); others throw std::invalid_argument — use
// sharded_gemv_rows_gather there.
template <typename T>
std::vector<const T*> sharded_gemv_rows_gather_fused(Group& g,
                                                     const std::vector<const DeviceMatrix<T>*>& A,
                                                     const std::vector<const DeviceVector<T>*>& x,
                                                     const std::vector<DeviceVector<T>*>& c,
                                                     const ExecPolicy&) {
    const int G = g.size();
    std::vector<std::uint64_t> off(std::size_t(G) + 1, 0);
    for (int q = 0; q < G; ++q) off[q + 1] = off[q] + c[q]->len();
    Group::Gather& st = g.gather(off[G] * sizeof(T));
    for (int r = 0; r < G; ++r) {
        cabl::detail::require(A[r]->layout() == Layout::RowMajor,
                              "gemv_row_major: A must be RowMajor");
        cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
        cabl::detail::check(detail::gemv_gather(A[r]->data(), A[r]->rows(), A[r]->cols(),
                                                x[r]->data(), c[r]->data(), off[r], off[G],
                                                st.bufs.data(), st.mboxes.data(), G, r,
                                                g.stream(r)));
    }
    g.synchronize();
    st.calls += 1;
    std::vector<const T*> full;
    for (int r = 0; r < G; ++r)
        full.push_back(static_cast<const T*>(st.bufs[r]) + (st.calls & 1) * off[G]);
    return full;
}

// Col-major GEMV sharded by columns (short-wide shapes): A[r] is device r's
// column block (m x n_r, col-major), x[r] the matching slice of x, c[r] a
// replica of c.  Each device computes its partial from zero; the partials are
// all-gathered and added to every replica in rank order (combine_rows), so
// all devices end with the same bits.
template <typename T>
void sharded_gemv_cols(Group& g, const std::vector<const DeviceMatrix<T>*>& A,
                       const std::vector<const DeviceVector<T>*>& x,
                       const std::vector<DeviceVector<T>*>& c, const ExecPolicy& policy) {
    const int G = g.size();
    const std::size_t m = c[0]->len();
    std::vector<DeviceVector<T>> part, gathered;
    for (int r = 0; r < G; ++r) {
        cabl::detail::require(A[r]->layout() == Layout::ColMajor && A[r]->rows() == m &&
                                  c[r]->len() == m,
                              "sharded_gemv_cols: col-major blocks of m rows, c replicas of length m");
        cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
        part.emplace_back(m);
        gathered.emplace_back(m * std::size_t(G));
        cabl::detail::cuda_check(cudaMemsetAsync(part[r].data(), 0, m * sizeof(T), g.stream(r)),
                                 "memset");
        gemv_col_major(*A[r], *x[r], part[r], policy, g.stream(r));
    }
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (int r = 0; r < G; ++r)
        nccl_check(ncclAllGather(part[r].data(), gathered[r].data(), m, detail::nccl_type<T>(),
                                 g.comm(r), g.stream(r)),
                   "ncclAllGather");
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
    for (int r = 0; r < G; ++r) {
        cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
        cabl::detail::check(detail::combine_rows(gathered[r].data(), std::uint32_t(G), m,
                                                 c[r]->data(), g.stream(r)));
    }
    g.synchronize();
}

// sharded_gemv_cols with the all-gather + combine replaced by one peer-memory
// kernel per device (cabl_cuda_combine_rows_peer_*): same bits, no NCCL call.
template <typename T>
void sharded_gemv_cols_fused(Group& g, const std::vector<const DeviceMatrix<T>*>& A,
                             const std::vector<const DeviceVector<T>*>& x,
                             const std::vector<DeviceVector<T>*>& c, const ExecPolicy& policy) {
    const int G = g.size();
    const std::size_t m = c[0]->len();
    Group::Gather& st = g.rows(2 * 8 * (m ? m : 1) * sizeof(T));
    std::vector<DeviceVector<T>> part;
    for (int r = 0; r < G; ++r) {
        cabl::detail::require(A[r]->layout() == Layout::ColMajor && A[r]->rows() == m &&
                                  c[r]->len() == m,
                              "sharded_gemv_cols: col-major blocks of m rows, c replicas of length m");
        cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
        part.emplace_back(m);
        cabl::detail::cuda_check(cudaMemsetAsync(part[r].data(), 0, m * sizeof(T), g.stream(r)),
                                 "memset");
        gemv_col_major(*A[r], *x[r], part[r], policy, g.stream(r));
        cabl::detail::check(detail::rows_peer(part[r].data(), m, c[r]->data(), st.bufs.data(),
                                              st.mboxes.data(), G, r, g.stream(r)));
    }
    g.synchronize();
}

// C[r] += x[r] (x) y[r] on every device's row block (no communication).
template <typename T>
void sharded_ger_rows(Group& g, const std::vector<const DeviceVector<T>*>& x,
                      const std::vector<const DeviceVector<T>*>& y,
                      const std::vector<DeviceMatrix<T>*>& C, const ExecPolicy& policy) {
    for (int r = 0; r < g.size(); ++r) {
        cabl::detail::cuda_check(cudaSetDevice(g.device(r)), "cudaSetDevice");
        ger(*x[r], *y[r], *C[r], policy, g.stream(r));
    }
    g.synchronize();
}

} // namespace cabl::nccl

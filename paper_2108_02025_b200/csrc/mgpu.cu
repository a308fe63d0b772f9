// Multi-GPU C ABI (cabl_mgpu_*, include/cabl_cuda.h): one process driving G
// devices, the process model of SURVEY.md §8(e), for FFI consumers of
// libcabl_cuda.so.  The partitioning lifts the reference's parallel_chunks
// (proj/include/cabl/thread_pool.hpp:153-164) from threads to devices: the
// caller hands each device its contiguous shard and the library runs the
// single-GPU kernel on every shard, then the exchange:
//
//   DOT      per-device partial (alpha0 = 0) -> ncclAllGather of the G
//            partials -> rank-ordered sum + alpha0 on every device
//            (cabl_cuda_combine_partials), or the fused peer-memory kernel
//            (cabl_cuda_dot_peer): the same bits either way;
//   GEMV rm  row blocks, x replicated; optional full c on every device
//            (grouped ncclBroadcast per source rank, or the gathering kernel);
//   GEMV cm  column blocks; every replica of c gets the rank-ordered sum of
//            the G partials (all-gather + combine_rows, or the peer combine);
//   GER rm   row blocks of C, no exchange.
//
// Errors follow the reference pool's contract (thread_pool.hpp:63-68: a
// worker's failure is rethrown to the caller, never swallowed, never a
// hang): every call validates ALL shards before it launches anything
// (CABL_EINVAL), and it returns only when every device is done — polling
// cudaEventQuery and ncclCommGetAsyncError, with a timeout.  An asynchronous
// NCCL error, a peer-memory exchange that timed out, or the timeout itself
// aborts every communicator (ncclCommAbort) and returns CABL_ENCCL; the
// context is then unusable (every later call returns CABL_ENCCL) and must be
// finalized.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2", or CABL_NCCL_LIB): the
// single-GPU library has no NCCL dependency, and inside a process that
// already loaded NCCL (e.g. PyTorch) the loaded copy is reused.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "cabl_cuda.h"
#include "kernels.cuh"

namespace {

struct NcclApi {
    void* h = nullptr;
    std::string err;
    int version = 0;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* path = getenv("CABL_NCCL_LIB");
        api.h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!api.h) {
            const char* e = dlerror();
            api.err = std::string("cannot load NCCL (") + (path && *path ? path : "libnccl.so.2") +
                      "): " + (e ? e : "?");
            return;
        }
        bool ok = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(api.h, name));
            if (!fn) {
                ok = false;
                api.err = std::string("NCCL symbol missing: ") + name;
            }
        };
        sym(api.GetVersion, "ncclGetVersion");
        sym(api.CommInitAll, "ncclCommInitAll");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommAbort, "ncclCommAbort");
        sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
        sym(api.GetErrorString, "ncclGetErrorString");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.AllGather, "ncclAllGather");
        sym(api.Broadcast, "ncclBroadcast");
        if (ok && api.GetVersion(&api.version) != ncclSuccess) {
            ok = false;
            api.err = "ncclGetVersion failed";
        }
        if (!ok) {
            dlclose(api.h);
            api.h = nullptr;
        }
    });
    return api;
}

template <typename T> ncclDataType_t nccl_type();
template <> ncclDataType_t nccl_type<float>() { return ncclFloat32; }
template <> ncclDataType_t nccl_type<double>() { return ncclFloat64; }

// the single-device C ABI, by dtype
int dot1(const float* x, const float* y, uint64_t n, float a, float* o, uint64_t cut, cudaStream_t s) {
    return cabl_cuda_dot_f32(x, y, n, a, o, cut, nullptr, s);
}
int dot1(const double* x, const double* y, uint64_t n, double a, double* o, uint64_t cut, cudaStream_t s) {
    return cabl_cuda_dot_f64(x, y, n, a, o, cut, nullptr, s);
}
int combine1(const float* p, uint32_t k, float a, float* o, cudaStream_t s) {
    return cabl_cuda_combine_partials_f32(p, k, a, o, s);
}
int combine1(const double* p, uint32_t k, double a, double* o, cudaStream_t s) {
    return cabl_cuda_combine_partials_f64(p, k, a, o, s);
}
int rows1(const float* p, uint32_t k, uint64_t m, float* c, cudaStream_t s) {
    return cabl_cuda_combine_rows_f32(p, k, m, c, s);
}
int rows1(const double* p, uint32_t k, uint64_t m, double* c, cudaStream_t s) {
    return cabl_cuda_combine_rows_f64(p, k, m, c, s);
}
int gemv_rm1(const float* A, uint64_t m, uint64_t n, const float* x, float* c, uint64_t cut, cudaStream_t s) {
    return cabl_cuda_gemv_rm_f32(A, m, n, x, c, cut, nullptr, s);
}
int gemv_rm1(const double* A, uint64_t m, uint64_t n, const double* x, double* c, uint64_t cut,
             cudaStream_t s) {
    return cabl_cuda_gemv_rm_f64(A, m, n, x, c, cut, nullptr, s);
}
int gemv_cm1(const float* A, uint64_t m, uint64_t n, const float* x, float* c, uint64_t cut, cudaStream_t s) {
    return cabl_cuda_gemv_cm_f32(A, m, n, x, c, cut, nullptr, s);
}
int gemv_cm1(const double* A, uint64_t m, uint64_t n, const double* x, double* c, uint64_t cut,
             cudaStream_t s) {
    return cabl_cuda_gemv_cm_f64(A, m, n, x, c, cut, nullptr, s);
}
int ger_rm1(const float* x, const float* y, float* C, uint64_t m, uint64_t n, uint64_t cut, cudaStream_t s) {
    return cabl_cuda_ger_rm_f32(x, y, C, m, n, cut, nullptr, s);
}
int ger_rm1(const double* x, const double* y, double* C, uint64_t m, uint64_t n, uint64_t cut,
            cudaStream_t s) {
    return cabl_cuda_ger_rm_f64(x, y, C, m, n, cut, nullptr, s);
}
int dot_peer1(const float* x, const float* y, uint64_t n, float a, float* o, void* const* mb, int G,
              int r, uint64_t cut, cudaStream_t s) {
    return cabl_cuda_dot_peer_f32(x, y, n, a, o, mb, G, r, cut, nullptr, s);
}
int dot_peer1(const double* x, const double* y, uint64_t n, double a, double* o, void* const* mb,
              int G, int r, uint64_t cut, cudaStream_t s) {
    return cabl_cuda_dot_peer_f64(x, y, n, a, o, mb, G, r, cut, nullptr, s);
}
int gather1(const float* A, uint64_t m, uint64_t n, const float* x, float* c, uint64_t off,
            uint64_t mt, void* const* b, void* const* mb, int G, int r, cudaStream_t s) {
    return cabl_cuda_gemv_rm_gather_f32(A, m, n, x, c, off, mt, b, mb, G, r, nullptr, s);
}
int gather1(const double* A, uint64_t m, uint64_t n, const double* x, double* c, uint64_t off,
            uint64_t mt, void* const* b, void* const* mb, int G, int r, cudaStream_t s) {
    return cabl_cuda_gemv_rm_gather_f64(A, m, n, x, c, off, mt, b, mb, G, r, nullptr, s);
}
int gather_ok1(const float* A, uint64_t m, uint64_t n, const float* x, int* ok) {
    return cabl_cuda_gemv_rm_gather_supported_f32(A, m, n, x, ok);
}
int gather_ok1(const double* A, uint64_t m, uint64_t n, const double* x, int* ok) {
    return cabl_cuda_gemv_rm_gather_supported_f64(A, m, n, x, ok);
}
int rows_peer1(const float* p, uint64_t m, float* c, void* const* b, void* const* mb, int G, int r,
               cudaStream_t s) {
    return cabl_cuda_combine_rows_peer_f32(p, m, c, b, mb, G, r, s);
}
int rows_peer1(const double* p, uint64_t m, double* c, void* const* b, void* const* mb, int G,
               int r, cudaStream_t s) {
    return cabl_cuda_combine_rows_peer_f64(p, m, c, b, mb, G, r, s);
}

} // namespace

// A set of peer buffers (one per device, all mapped into every device's
// address space by P2P) and their mailboxes, for one fused exchange.
struct PeerSet {
    std::vector<void*> bufs, mboxes;
    size_t bytes = 0;
    uint64_t calls = 0;
};

struct cabl_mgpu {
    std::vector<int> devs;
    std::vector<ncclComm_t> comms;
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> start, done; // per rank, around each call's device work
    bool timed = false;                    // start events recorded for the last call
    std::vector<void*> scratch;
    std::vector<size_t> scratch_bytes;
    uint64_t timeout_ms = 60000;
    bool broken = false;
    std::string broken_why;
    bool peer_enabled = false;
    PeerSet dot_mb, gather, rows;
    std::mutex mu; // calls on one context run one at a time
};

namespace {

int mfail(int code, const std::string& msg) {
    cabl_dev::set_last_error(msg); // what cabl_last_error() returns on this thread
    return code;
}

int cuda_err(cudaError_t e, const char* where) {
    cudaGetLastError();
    return mfail(CABL_ECUDA, std::string("cabl_mgpu: ") + where + ": " + cudaGetErrorString(e));
}

#define MG_CUDA(expr, where)                                                                    \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess) return cuda_err(e_, where);                                      \
    } while (0)

#define MG_RC(expr)                                                                             \
    do {                                                                                        \
        int rc_ = (expr);                                                                       \
        if (rc_ != CABL_OK) return rc_;                                                         \
    } while (0)

int nccl_err(cabl_mgpu* c, ncclResult_t r, const char* where);

void abort_all(cabl_mgpu* c, const std::string& why) {
    const NcclApi& N = nccl();
    for (size_t r = 0; r < c->comms.size(); ++r)
        if (c->comms[r]) {
            cudaSetDevice(c->devs[r]);
            N.CommAbort(c->comms[r]);
            c->comms[r] = nullptr;
        }
    c->broken = true;
    c->broken_why = why;
}

int nccl_err(cabl_mgpu* c, ncclResult_t r, const char* where) {
    const std::string why = std::string("cabl_mgpu: ") + where + ": " + nccl().GetErrorString(r);
    abort_all(c, why);
    return mfail(CABL_ENCCL, why);
}

#define MG_NCCL(ctx, expr, where)                                                               \
    do {                                                                                        \
        ncclResult_t r_ = (expr);                                                               \
        if (r_ != ncclSuccess) return nccl_err(ctx, r_, where);                                 \
    } while (0)

int usable(cabl_mgpu* c) {
    if (!c) return mfail(CABL_EINVAL, "cabl_mgpu: null context");
    if (c->broken)
        return mfail(CABL_ENCCL, "cabl_mgpu: context aborted after an earlier failure (" +
                                     c->broken_why + "); call cabl_mgpu_finalize");
    return CABL_OK;
}

int set_dev(cabl_mgpu* c, int r) {
    MG_CUDA(cudaSetDevice(c->devs[r]), "cudaSetDevice");
    return CABL_OK;
}

// the device-side start of a call, on every rank's stream (after validation,
// before the first launch): cabl_mgpu_last_call_ms measures from here to the
// end of the call's last operation on that rank
int mark_start(cabl_mgpu* c) {
    c->timed = false;
    for (size_t r = 0; r < c->devs.size(); ++r) {
        MG_RC(set_dev(c, int(r)));
        MG_CUDA(cudaEventRecord(c->start[r], c->streams[r]), "cudaEventRecord");
    }
    return CABL_OK; // wait_all sets `timed` once the call has completed
}

// Block until every device's stream has drained, watching NCCL for
// asynchronous errors and the clock for the context's timeout.
int wait_all(cabl_mgpu* c, bool watch_nccl, const char* what) {
    const int G = int(c->devs.size());
    for (int r = 0; r < G; ++r) {
        MG_RC(set_dev(c, r));
        MG_CUDA(cudaEventRecord(c->done[r], c->streams[r]), "cudaEventRecord");
    }
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<bool> finished(size_t(G), false);
    int left = G;
    unsigned spins = 0;
    while (left > 0) {
        for (int r = 0; r < G; ++r) {
            if (finished[r]) continue;
            MG_RC(set_dev(c, r));
            const cudaError_t q = cudaEventQuery(c->done[r]);
            if (q == cudaSuccess) {
                finished[r] = true;
                --left;
            } else if (q != cudaErrorNotReady) {
                const int rc = cuda_err(q, what);
                if (watch_nccl) abort_all(c, cabl_last_error());
                return rc;
            }
        }
        if (left == 0) break;
        if (watch_nccl) {
            for (int r = 0; r < G; ++r) {
                ncclResult_t st = ncclSuccess;
                const ncclResult_t q = nccl().CommGetAsyncError(c->comms[r], &st);
                if (q != ncclSuccess) return nccl_err(c, q, "ncclCommGetAsyncError");
                if (st != ncclSuccess && st != ncclInProgress) return nccl_err(c, st, what);
            }
        }
        const double ms = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t0).count();
        if (ms > double(c->timeout_ms)) {
            const std::string why = std::string("cabl_mgpu: ") + what + ": not complete after " +
                                    std::to_string(c->timeout_ms) + " ms (a device or peer stalled)";
            abort_all(c, why);
            return mfail(CABL_ENCCL, why);
        }
        if (++spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
    c->timed = true;
    return CABL_OK;
}

int scratch(cabl_mgpu* c, int r, size_t bytes, void** out) {
    if (c->scratch_bytes[r] < bytes) {
        MG_RC(set_dev(c, r));
        MG_CUDA(cudaStreamSynchronize(c->streams[r]), "scratch sync");
        if (c->scratch[r]) cudaFree(c->scratch[r]);
        c->scratch[r] = nullptr;
        c->scratch_bytes[r] = 0;
        const size_t want = bytes < (1u << 20) ? (1u << 20) : bytes;
        MG_CUDA(cudaMalloc(&c->scratch[r], want), "scratch");
        c->scratch_bytes[r] = want;
    }
    *out = c->scratch[r];
    return CABL_OK;
}

int enable_peers(cabl_mgpu* c) {
    if (c->peer_enabled) return CABL_OK;
    const int G = int(c->devs.size());
    for (int r = 0; r < G; ++r) {
        MG_RC(set_dev(c, r));
        for (int q = 0; q < G; ++q) {
            if (q == r) continue;
            int can = 0;
            MG_CUDA(cudaDeviceCanAccessPeer(&can, c->devs[r], c->devs[q]), "cudaDeviceCanAccessPeer");
            if (!can)
                return mfail(CABL_EINVAL, "cabl_mgpu: peer-memory exchange needs P2P between every "
                                          "pair of devices (use CABL_MGPU_NCCL)");
            const cudaError_t e = cudaDeviceEnablePeerAccess(c->devs[q], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else if (e != cudaSuccess) return cuda_err(e, "cudaDeviceEnablePeerAccess");
        }
    }
    c->peer_enabled = true;
    return CABL_OK;
}

void free_set(cabl_mgpu* c, PeerSet& st) {
    for (size_t i = 0; i < st.mboxes.size(); ++i) {
        cudaSetDevice(c->devs[i]);
        if (i < st.bufs.size() && st.bufs[i]) cabl_peer_free(st.bufs[i]);
        if (st.mboxes[i]) cabl_peer_mailbox_destroy(st.mboxes[i]);
    }
    st = PeerSet{};
}

// (re)build a peer set with `bytes` of buffer per device (0: mailboxes only)
int peer_set(cabl_mgpu* c, PeerSet& st, size_t bytes) {
    if (!st.mboxes.empty() && st.bytes == bytes) return CABL_OK;
    free_set(c, st);
    MG_RC(enable_peers(c));
    const int G = int(c->devs.size());
    for (int r = 0; r < G; ++r) {
        MG_RC(set_dev(c, r));
        void* b = nullptr;
        void* mb = nullptr;
        if (bytes) {
            if (int rc = cabl_peer_alloc(bytes, &b)) {
                free_set(c, st);
                return rc;
            }
        }
        if (int rc = cabl_peer_mailbox_create(&mb)) {
            if (b) cabl_peer_free(b);
            free_set(c, st);
            return rc;
        }
        st.bufs.push_back(b);
        st.mboxes.push_back(mb);
    }
    st.bytes = bytes;
    return CABL_OK;
}

// after a fused call: any device whose mailbox recorded a timed-out exchange
// fails the call (and the context: the mailboxes' epochs no longer agree)
int check_peer_faults(cabl_mgpu* c, PeerSet& st, const char* what) {
    for (size_t r = 0; r < st.mboxes.size(); ++r) {
        MG_RC(set_dev(c, int(r)));
        uint64_t epoch = 0, fault = 0;
        MG_RC(cabl_peer_mailbox_state(st.mboxes[r], &epoch, &fault));
        if (fault) {
            const std::string why = std::string("cabl_mgpu: ") + what + ": device " +
                                    std::to_string(c->devs[r]) +
                                    " timed out waiting for its peers (call " +
                                    std::to_string(fault) + ")";
            free_set(c, st);
            abort_all(c, why);
            return mfail(CABL_ENCCL, why);
        }
    }
    return CABL_OK;
}

int check_exchange(int exchange) {
    if (exchange != CABL_MGPU_NCCL && exchange != CABL_MGPU_PEER)
        return mfail(CABL_EINVAL, "cabl_mgpu: exchange must be CABL_MGPU_NCCL or CABL_MGPU_PEER");
    return CABL_OK;
}

// ------------------------------------------------------------------ DOT
template <typename T>
int mgpu_dot(cabl_mgpu* c, const T* const* x, const T* const* y, const uint64_t* n, T alpha0,
             uint64_t cutoff, int exchange, T* result) {
    if (!c) return mfail(CABL_EINVAL, "cabl_mgpu: null context");
    std::lock_guard<std::mutex> lk(c->mu);
    MG_RC(usable(c));
    MG_RC(check_exchange(exchange));
    const int G = int(c->devs.size());
    if (!x || !y || !n || !result) return mfail(CABL_EINVAL, "cabl_mgpu_dot: null argument");
    for (int r = 0; r < G; ++r)
        if (n[r] > 0 && (!x[r] || !y[r]))
            return mfail(CABL_EINVAL, "cabl_mgpu_dot: x and y must not be null");
    // scratch per device: [0] partial, [1..G] gathered partials, [G+1] result
    std::vector<T*> sc(size_t(G), nullptr);
    for (int r = 0; r < G; ++r) {
        void* p = nullptr;
        MG_RC(scratch(c, r, (size_t(G) + 2) * sizeof(T), &p));
        sc[r] = static_cast<T*>(p);
    }
    if (exchange == CABL_MGPU_PEER) {
        MG_RC(peer_set(c, c->dot_mb, 0));
        MG_RC(mark_start(c));
        for (int r = 0; r < G; ++r) {
            MG_RC(set_dev(c, r));
            if (int rc = dot_peer1(x[r], y[r], n[r], alpha0, sc[r] + G + 1, c->dot_mb.mboxes.data(),
                                   G, r, cutoff, c->streams[r])) {
                // ranks 0..r-1 are already waiting for this one: their
                // mailboxes will record a timed-out exchange
                if (r > 0) abort_all(c, "dot (peer exchange): launch failed after peers started");
                return rc;
            }
        }
        MG_RC(wait_all(c, false, "dot (peer exchange)"));
        MG_RC(check_peer_faults(c, c->dot_mb, "dot (peer exchange)"));
    } else {
        MG_RC(mark_start(c));
        for (int r = 0; r < G; ++r) {
            MG_RC(set_dev(c, r));
            MG_RC(dot1(x[r], y[r], n[r], T(0), sc[r], cutoff, c->streams[r]));
        }
        const NcclApi& N = nccl();
        MG_NCCL(c, N.GroupStart(), "ncclGroupStart");
        for (int r = 0; r < G; ++r)
            MG_NCCL(c, N.AllGather(sc[r], sc[r] + 1, 1, nccl_type<T>(), c->comms[r], c->streams[r]),
                    "ncclAllGather");
        MG_NCCL(c, N.GroupEnd(), "ncclGroupEnd");
        for (int r = 0; r < G; ++r) {
            MG_RC(set_dev(c, r));
            MG_RC(combine1(sc[r] + 1, uint32_t(G), alpha0, sc[r] + G + 1, c->streams[r]));
        }
        MG_RC(wait_all(c, true, "dot (NCCL all-gather)"));
    }
    MG_RC(set_dev(c, 0));
    MG_CUDA(cudaMemcpy(result, sc[0] + G + 1, sizeof(T), cudaMemcpyDeviceToHost), "result D2H");
    return CABL_OK;
}

// DOT over fixed global segments (a GPU-count-invariant result; SURVEY.md
// §8(e)'s optional item, the reference's block decomposition of kernels.hpp:
// 145-163 with a fixed block length): the shards, concatenated in rank order,
// are cut every `segment` elements; each segment's partial comes from its own
// launch of the single-GPU kernel (alpha0 = 0) on the device that holds it, so
// it depends on the segment's data and length only; the K partials are
// all-gathered (padded to the widest rank) and summed in index order + alpha0
// on every device.  Every shard except the last non-empty one must therefore be a
// whole number of segments.
template <typename T>
int mgpu_dot_segmented(cabl_mgpu* c, const T* const* x, const T* const* y, const uint64_t* n,
                       uint64_t segment, T alpha0, uint64_t cutoff, T* result) {
    if (!c) return mfail(CABL_EINVAL, "cabl_mgpu: null context");
    std::lock_guard<std::mutex> lk(c->mu);
    MG_RC(usable(c));
    const int G = int(c->devs.size());
    if (!x || !y || !n || !result)
        return mfail(CABL_EINVAL, "cabl_mgpu_dot_segmented: null argument");
    if (segment == 0) return mfail(CABL_EINVAL, "cabl_mgpu_dot_segmented: segment must be > 0");
    // a segment keeps the alignment class of its shard's base whichever device
    // holds it (the kernel's vector path depends on it), so the cut points must
    // not move it: whole 64-element (256 / 512-byte) units
    if (segment % 64 != 0)
        return mfail(CABL_EINVAL, "cabl_mgpu_dot_segmented: segment must be a multiple of 64 elements");
    int last = -1;
    for (int r = 0; r < G; ++r) {
        if (n[r] > 0 && (!x[r] || !y[r]))
            return mfail(CABL_EINVAL, "cabl_mgpu_dot_segmented: x and y must not be null");
        if (n[r] > 0) last = r;
    }
    std::vector<uint64_t> cnt(size_t(G), 0);
    uint64_t K = 0, widest = 1;
    for (int r = 0; r < G; ++r) {
        if (r < last && n[r] % segment != 0)
            return mfail(CABL_EINVAL, "cabl_mgpu_dot_segmented: every shard before the last "
                                      "non-empty one must be a whole number of segments");
        cnt[r] = (n[r] + segment - 1) / segment;
        K += cnt[r];
        if (cnt[r] > widest) widest = cnt[r];
    }
    if (K > 0xffffffffull) return mfail(CABL_EINVAL, "cabl_mgpu_dot_segmented: too many segments");
    // scratch per device: own partials [widest], gathered [G * widest],
    // partials in index order [K], result [1]
    const size_t own = 0, gat = size_t(widest), ord = gat + size_t(G) * widest,
                 res = ord + size_t(K ? K : 1), total = res + 1;
    std::vector<T*> sc(size_t(G), nullptr);
    for (int r = 0; r < G; ++r) {
        void* p = nullptr;
        MG_RC(scratch(c, r, total * sizeof(T), &p));
        sc[r] = static_cast<T*>(p);
    }
    MG_RC(mark_start(c));
    for (int r = 0; r < G; ++r) {
        MG_RC(set_dev(c, r));
        MG_CUDA(cudaMemsetAsync(sc[r] + own, 0, widest * sizeof(T), c->streams[r]), "partials memset");
        for (uint64_t k = 0; k < cnt[r]; ++k) {
            const uint64_t lo = k * segment, len = n[r] - lo < segment ? n[r] - lo : segment;
            MG_RC(dot1(x[r] + lo, y[r] + lo, len, T(0), sc[r] + own + k, cutoff, c->streams[r]));
        }
    }
    if (G > 1) {
        const NcclApi& N = nccl();
        MG_NCCL(c, N.GroupStart(), "ncclGroupStart");
        for (int r = 0; r < G; ++r)
            MG_NCCL(c, N.AllGather(sc[r] + own, sc[r] + gat, size_t(widest), nccl_type<T>(),
                                   c->comms[r], c->streams[r]),
                    "ncclAllGather");
        MG_NCCL(c, N.GroupEnd(), "ncclGroupEnd");
    }
    for (int r = 0; r < G; ++r) {
        MG_RC(set_dev(c, r));
        const T* src = G > 1 ? sc[r] + gat : sc[r] + own;
        uint64_t at = 0;
        for (int q = 0; q < G; ++q) { // drop each rank's padding: index order, K values
            if (cnt[q])
                MG_CUDA(cudaMemcpyAsync(sc[r] + ord + at, src + size_t(q) * widest, cnt[q] * sizeof(T),
                                        cudaMemcpyDeviceToDevice, c->streams[r]),
                        "partials compaction");
            at += cnt[q];
        }
        MG_RC(combine1(sc[r] + ord, uint32_t(K), alpha0, sc[r] + res, c->streams[r]));
    }
    MG_RC(wait_all(c, G > 1, "dot (segmented, NCCL all-gather)"));
    MG_RC(set_dev(c, 0));
    MG_CUDA(cudaMemcpy(result, sc[0] + res, sizeof(T), cudaMemcpyDeviceToHost), "result D2H");
    return CABL_OK;
}

// ------------------------------------------------------- GEMV row blocks
template <typename T>
int mgpu_gemv_rm(cabl_mgpu* c, const T* const* A, const uint64_t* m, uint64_t n,
                 const T* const* x, T* const* cs, uint64_t cutoff, int exchange, T* const* c_full) {
    if (!c) return mfail(CABL_EINVAL, "cabl_mgpu: null context");
    std::lock_guard<std::mutex> lk(c->mu);
    MG_RC(usable(c));
    MG_RC(check_exchange(exchange));
    const int G = int(c->devs.size());
    if (!A || !m || !x || !cs) return mfail(CABL_EINVAL, "cabl_mgpu_gemv_rm: null argument");
    std::vector<uint64_t> off(size_t(G) + 1, 0);
    for (int r = 0; r < G; ++r) {
        if (m[r] > 0 && n > 0 && (!A[r] || !x[r]))
            return mfail(CABL_EINVAL, "cabl_mgpu_gemv_rm: A and x must not be null");
        if (m[r] > 0 && !cs[r]) return mfail(CABL_EINVAL, "cabl_mgpu_gemv_rm: c must not be null");
        off[r + 1] = off[r] + m[r];
    }
    const bool gather = c_full != nullptr;
    if (gather)
        for (int r = 0; r < G; ++r)
            if (!c_full[r] && off[G] > 0)
                return mfail(CABL_EINVAL, "cabl_mgpu_gemv_rm: null entry in c_full");
    if (gather && exchange == CABL_MGPU_PEER) {
        // every shard must take the sweep kernel BEFORE any kernel launches:
        // a rank that fails after its peers started would leave them waiting
        for (int r = 0; r < G; ++r) {
            MG_RC(set_dev(c, r));
            int ok = 0;
            MG_RC(gather_ok1(A[r], m[r], n, x[r], &ok));
            if (!ok)
                return mfail(CABL_EINVAL, "cabl_mgpu_gemv_rm: shard " + std::to_string(r) +
                                              " does not take the gathering sweep kernel (few or "
                                              "short rows, unaligned): use CABL_MGPU_NCCL");
        }
        MG_RC(peer_set(c, c->gather, 2 * size_t(off[G]) * sizeof(T)));
        MG_RC(mark_start(c));
        for (int r = 0; r < G; ++r) {
            MG_RC(set_dev(c, r));
            if (int rc = gather1(A[r], m[r], n, x[r], cs[r], off[r], off[G], c->gather.bufs.data(),
                                 c->gather.mboxes.data(), G, r, c->streams[r])) {
                if (r > 0) abort_all(c, "gemv_rm gather: launch failed after peers started");
                return rc;
            }
        }
        c->gather.calls += 1;
        const uint64_t half = (c->gather.calls & 1) * off[G];
        for (int r = 0; r < G; ++r) { // consumed in stream order before the next call
            MG_RC(set_dev(c, r));
            MG_CUDA(cudaMemcpyAsync(c_full[r], static_cast<T*>(c->gather.bufs[r]) + half,
                                    off[G] * sizeof(T), cudaMemcpyDeviceToDevice, c->streams[r]),
                    "gathered c copy");
        }
        MG_RC(wait_all(c, false, "gemv_rm (peer gather)"));
        return check_peer_faults(c, c->gather, "gemv_rm (peer gather)");
    }
    MG_RC(mark_start(c));
    for (int r = 0; r < G; ++r) {
        MG_RC(set_dev(c, r));
        MG_RC(gemv_rm1(A[r], m[r], n, x[r], cs[r], cutoff, c->streams[r]));
    }
    if (!gather) return wait_all(c, false, "gemv_rm");
    const NcclApi& N = nccl();
    MG_NCCL(c, N.GroupStart(), "ncclGroupStart");
    for (int q = 0; q < G; ++q) {
        if (m[q] == 0) continue;
        for (int r = 0; r < G; ++r)
            MG_NCCL(c, N.Broadcast(r == q ? cs[q] : nullptr, c_full[r] + off[q], m[q], nccl_type<T>(),
                                   q, c->comms[r], c->streams[r]),
                    "ncclBroadcast");
    }
    MG_NCCL(c, N.GroupEnd(), "ncclGroupEnd");
    return wait_all(c, true, "gemv_rm (NCCL gather)");
}

// --------------------------------------------------- GEMV col-major by columns
template <typename T>
int mgpu_gemv_cm_cols(cabl_mgpu* c, const T* const* A, uint64_t m, const uint64_t* n,
                      const T* const* x, T* const* cs, uint64_t cutoff, int exchange) {
    if (!c) return mfail(CABL_EINVAL, "cabl_mgpu: null context");
    std::lock_guard<std::mutex> lk(c->mu);
    MG_RC(usable(c));
    MG_RC(check_exchange(exchange));
    const int G = int(c->devs.size());
    if (!A || !n || !x || !cs) return mfail(CABL_EINVAL, "cabl_mgpu_gemv_cm_cols: null argument");
    for (int r = 0; r < G; ++r) {
        if (m > 0 && n[r] > 0 && (!A[r] || !x[r]))
            return mfail(CABL_EINVAL, "cabl_mgpu_gemv_cm_cols: A and x must not be null");
        if (m > 0 && !cs[r]) return mfail(CABL_EINVAL, "cabl_mgpu_gemv_cm_cols: c must not be null");
    }
    if (m == 0) return CABL_OK;
    // scratch per device: part (m), gathered parts (G m)
    std::vector<T*> part(size_t(G), nullptr);
    for (int r = 0; r < G; ++r) {
        void* p = nullptr;
        MG_RC(scratch(c, r, (size_t(G) + 1) * m * sizeof(T), &p));
        part[r] = static_cast<T*>(p);
    }
    if (exchange == CABL_MGPU_PEER) MG_RC(peer_set(c, c->rows, 2 * 8 * size_t(m) * sizeof(T)));
    MG_RC(mark_start(c));
    for (int r = 0; r < G; ++r) {
        MG_RC(set_dev(c, r));
        MG_CUDA(cudaMemsetAsync(part[r], 0, m * sizeof(T), c->streams[r]), "memset");
        MG_RC(gemv_cm1(A[r], m, n[r], x[r], part[r], cutoff, c->streams[r]));
    }
    if (exchange == CABL_MGPU_PEER) {
        for (int r = 0; r < G; ++r) {
            MG_RC(set_dev(c, r));
            if (int rc = rows_peer1(part[r], m, cs[r], c->rows.bufs.data(), c->rows.mboxes.data(), G,
                                    r, c->streams[r])) {
                if (r > 0) abort_all(c, "gemv_cm_cols combine: launch failed after peers started");
                return rc;
            }
        }
        MG_RC(wait_all(c, false, "gemv_cm_cols (peer combine)"));
        return check_peer_faults(c, c->rows, "gemv_cm_cols (peer combine)");
    }
    const NcclApi& N = nccl();
    MG_NCCL(c, N.GroupStart(), "ncclGroupStart");
    for (int r = 0; r < G; ++r)
        MG_NCCL(c, N.AllGather(part[r], part[r] + m, m, nccl_type<T>(), c->comms[r], c->streams[r]),
                "ncclAllGather");
    MG_NCCL(c, N.GroupEnd(), "ncclGroupEnd");
    for (int r = 0; r < G; ++r) {
        MG_RC(set_dev(c, r));
        MG_RC(rows1(part[r] + m, uint32_t(G), m, cs[r], c->streams[r]));
    }
    return wait_all(c, true, "gemv_cm_cols (NCCL all-gather)");
}

// ------------------------------------------------------------ GER row blocks
template <typename T>
int mgpu_ger_rm(cabl_mgpu* c, const T* const* x, const uint64_t* m, const T* const* y, uint64_t n,
                T* const* C, uint64_t cutoff) {
    if (!c) return mfail(CABL_EINVAL, "cabl_mgpu: null context");
    std::lock_guard<std::mutex> lk(c->mu);
    MG_RC(usable(c));
    const int G = int(c->devs.size());
    if (!x || !m || !y || !C) return mfail(CABL_EINVAL, "cabl_mgpu_ger_rm: null argument");
    for (int r = 0; r < G; ++r)
        if (m[r] > 0 && n > 0 && (!x[r] || !y[r] || !C[r]))
            return mfail(CABL_EINVAL, "cabl_mgpu_ger_rm: null operand");
    MG_RC(mark_start(c));
    for (int r = 0; r < G; ++r) {
        MG_RC(set_dev(c, r));
        MG_RC(ger_rm1(x[r], y[r], C[r], m[r], n, cutoff, c->streams[r]));
    }
    return wait_all(c, false, "ger_rm");
}

} // namespace

extern "C" {

CABL_API int cabl_mgpu_nccl_version(int* version) {
    if (!version) return mfail(CABL_EINVAL, "cabl_mgpu_nccl_version: null argument");
    const NcclApi& N = nccl();
    if (!N.h) return mfail(CABL_ENCCL, N.err);
    *version = N.version;
    return CABL_OK;
}

CABL_API int cabl_mgpu_init(const int* devices, int count, cabl_mgpu** ctx) {
    if (!ctx) return mfail(CABL_EINVAL, "cabl_mgpu_init: null context pointer");
    *ctx = nullptr;
    if (!devices || count < 1) return mfail(CABL_EINVAL, "cabl_mgpu_init: need at least one device");
    for (int i = 0; i < count; ++i)
        for (int j = 0; j < i; ++j)
            if (devices[i] == devices[j])
                return mfail(CABL_EINVAL, "cabl_mgpu_init: a device is listed twice");
    int have = 0;
    if (cudaGetDeviceCount(&have) != cudaSuccess || have == 0) {
        cudaGetLastError();
        return mfail(CABL_ECUDA, "cabl_mgpu_init: no CUDA device available (no CPU fallback)");
    }
    for (int i = 0; i < count; ++i)
        if (devices[i] < 0 || devices[i] >= have)
            return mfail(CABL_EINVAL, "cabl_mgpu_init: device " + std::to_string(devices[i]) +
                                          " is not one of the " + std::to_string(have) +
                                          " visible devices");
    const NcclApi& N = nccl();
    if (!N.h) return mfail(CABL_ENCCL, "cabl_mgpu_init: " + N.err);
    auto* c = new cabl_mgpu();
    c->devs.assign(devices, devices + count);
    if (const char* e = getenv("CABL_MGPU_TIMEOUT_MS")) {
        const unsigned long long v = strtoull(e, nullptr, 10);
        if (v) c->timeout_ms = v;
    }
    c->comms.assign(size_t(count), nullptr);
    const ncclResult_t ir = N.CommInitAll(c->comms.data(), count, c->devs.data());
    if (ir != ncclSuccess) {
        const std::string why = std::string("cabl_mgpu_init: ncclCommInitAll: ") + N.GetErrorString(ir);
        c->comms.assign(size_t(count), nullptr);
        cabl_mgpu_finalize(c);
        return mfail(CABL_ENCCL, why);
    }
    for (int r = 0; r < count; ++r) {
        cudaStream_t s = nullptr;
        cudaEvent_t ev = nullptr;
        cudaError_t e = cudaSetDevice(c->devs[r]);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        cudaEvent_t ev0 = nullptr;
        if (e == cudaSuccess) e = cudaEventCreate(&ev);
        if (e == cudaSuccess) e = cudaEventCreate(&ev0);
        c->streams.push_back(s);
        c->done.push_back(ev);
        c->start.push_back(ev0);
        if (e != cudaSuccess) {
            const int rc = cuda_err(e, "stream/event");
            cabl_mgpu_finalize(c);
            return rc;
        }
    }
    c->scratch.assign(size_t(count), nullptr);
    c->scratch_bytes.assign(size_t(count), 0);
    *ctx = c;
    return CABL_OK;
}

CABL_API int cabl_mgpu_finalize(cabl_mgpu* c) {
    if (!c) return CABL_OK;
    {
        std::lock_guard<std::mutex> lk(c->mu);
        for (size_t r = 0; r < c->devs.size(); ++r) {
            cudaSetDevice(c->devs[r]);
            if (r < c->streams.size() && c->streams[r] && !c->broken) cudaStreamSynchronize(c->streams[r]);
        }
        free_set(c, c->dot_mb);
        free_set(c, c->gather);
        free_set(c, c->rows);
        const NcclApi& N = nccl();
        for (size_t r = 0; r < c->devs.size(); ++r) {
            cudaSetDevice(c->devs[r]);
            if (r < c->scratch.size() && c->scratch[r]) cudaFree(c->scratch[r]);
            if (r < c->done.size() && c->done[r]) cudaEventDestroy(c->done[r]);
            if (r < c->start.size() && c->start[r]) cudaEventDestroy(c->start[r]);
            if (r < c->streams.size() && c->streams[r]) cudaStreamDestroy(c->streams[r]);
            if (r < c->comms.size() && c->comms[r] && N.h) N.CommDestroy(c->comms[r]);
        }
        cudaGetLastError();
    }
    delete c;
    return CABL_OK;
}

CABL_API int cabl_mgpu_size(const cabl_mgpu* c) { return c ? int(c->devs.size()) : 0; }

CABL_API int cabl_mgpu_device(const cabl_mgpu* c, int rank) {
    return (c && rank >= 0 && rank < int(c->devs.size())) ? c->devs[rank] : -1;
}

CABL_API void* cabl_mgpu_stream(const cabl_mgpu* c, int rank) {
    return (c && rank >= 0 && rank < int(c->streams.size())) ? c->streams[rank] : nullptr;
}

CABL_API int cabl_mgpu_last_call_ms(cabl_mgpu* c, int rank, float* ms) {
    if (!c || !ms || rank < 0 || rank >= int(c->devs.size()))
        return mfail(CABL_EINVAL, "cabl_mgpu_last_call_ms: null argument or rank out of range");
    std::lock_guard<std::mutex> lk(c->mu);
    if (!c->timed) return mfail(CABL_EINVAL, "cabl_mgpu_last_call_ms: no completed call to time");
    MG_RC(set_dev(c, rank));
    MG_CUDA(cudaEventElapsedTime(ms, c->start[rank], c->done[rank]), "cudaEventElapsedTime");
    return CABL_OK;
}

CABL_API int cabl_mgpu_set_timeout_ms(cabl_mgpu* c, uint64_t ms) {
    if (!c || ms == 0) return mfail(CABL_EINVAL, "cabl_mgpu_set_timeout_ms: null context or zero timeout");
    c->timeout_ms = ms;
    return CABL_OK;
}

CABL_API int cabl_mgpu_dot_f32(cabl_mgpu* c, const float* const* x, const float* const* y,
                               const uint64_t* n, float alpha0, uint64_t small_cutoff, int exchange,
                               float* result) {
    return mgpu_dot<float>(c, x, y, n, alpha0, small_cutoff, exchange, result);
}
CABL_API int cabl_mgpu_dot_f64(cabl_mgpu* c, const double* const* x, const double* const* y,
                               const uint64_t* n, double alpha0, uint64_t small_cutoff,
                               int exchange, double* result) {
    return mgpu_dot<double>(c, x, y, n, alpha0, small_cutoff, exchange, result);
}
CABL_API int cabl_mgpu_dot_segmented_f32(cabl_mgpu* c, const float* const* x, const float* const* y,
                                         const uint64_t* n, uint64_t segment, float alpha0,
                                         uint64_t small_cutoff, float* result) {
    return mgpu_dot_segmented<float>(c, x, y, n, segment, alpha0, small_cutoff, result);
}
CABL_API int cabl_mgpu_dot_segmented_f64(cabl_mgpu* c, const double* const* x,
                                         const double* const* y, const uint64_t* n,
                                         uint64_t segment, double alpha0, uint64_t small_cutoff,
                                         double* result) {
    return mgpu_dot_segmented<double>(c, x, y, n, segment, alpha0, small_cutoff, result);
}
CABL_API int cabl_mgpu_gemv_rm_f32(cabl_mgpu* c, const float* const* A, const uint64_t* m,
                                   uint64_t n, const float* const* x, float* const* cs,
                                   uint64_t small_cutoff, int exchange, float* const* c_full) {
    return mgpu_gemv_rm<float>(c, A, m, n, x, cs, small_cutoff, exchange, c_full);
}
CABL_API int cabl_mgpu_gemv_rm_f64(cabl_mgpu* c, const double* const* A, const uint64_t* m,
                                   uint64_t n, const double* const* x, double* const* cs,
                                   uint64_t small_cutoff, int exchange, double* const* c_full) {
    return mgpu_gemv_rm<double>(c, A, m, n, x, cs, small_cutoff, exchange, c_full);
}
CABL_API int cabl_mgpu_gemv_cm_cols_f32(cabl_mgpu* c, const float* const* A, uint64_t m,
                                        const uint64_t* n, const float* const* x, float* const* cs,
                                        uint64_t small_cutoff, int exchange) {
    return mgpu_gemv_cm_cols<float>(c, A, m, n, x, cs, small_cutoff, exchange);
}
CABL_API int cabl_mgpu_gemv_cm_cols_f64(cabl_mgpu* c, const double* const* A, uint64_t m,
                                        const uint64_t* n, const double* const* x,
                                        double* const* cs, uint64_t small_cutoff, int exchange) {
    return mgpu_gemv_cm_cols<double>(c, A, m, n, x, cs, small_cutoff, exchange);
}
CABL_API int cabl_mgpu_ger_rm_f32(cabl_mgpu* c, const float* const* x, const uint64_t* m,
                                  const float* const* y, uint64_t n, float* const* C,
                                  uint64_t small_cutoff) {
    return mgpu_ger_rm<float>(c, x, m, y, n, C, small_cutoff);
}
CABL_API int cabl_mgpu_ger_rm_f64(cabl_mgpu* c, const double* const* x, const uint64_t* m,
                                  const double* const* y, uint64_t n, double* const* C,
                                  uint64_t small_cutoff) {
    return mgpu_ger_rm<double>(c, x, m, y, n, C, small_cutoff);
}

} // extern "C"

// extern "C" boundary of libcabl_cuda.so — see include/cabl_cuda.h.
//
// Responsibilities: argument validation with the reference's messages
// (proj/include/cabl/kernels.hpp:59-64 and the `require` call sites), the
// small-problem dispatch rule (kernels.hpp:140, :240-241, :286-287), the
// execution-path probe (kernels.hpp:40-55), per-(device, stream) scratch for
// the kernels' cross-CTA combines, host-buffer staging, and the mapping of
// CUDA errors to status codes with a thread-local message.  No CPU fallback:
// without a usable device every compute entry point returns CABL_ECUDA.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "cabl_cuda.h"
#include "common.cuh"
#include "kernels.cuh"

using namespace cabl_dev;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

} // namespace

void cabl_dev::set_last_error(const std::string& msg) { g_err = msg; }

namespace {

int cuda_fail(cudaError_t e, const char* where) {
    cudaGetLastError(); // clear sticky-free errors so the next call starts clean
    return fail(CABL_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CABL_TRY_CUDA(expr, where)                                                            \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess) return cuda_fail(e_, where);                                   \
    } while (0)

int current_device(int* dev) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(CABL_ECUDA,
                    "no CUDA device available (libcabl_cuda has no CPU fallback)");
    }
    CABL_TRY_CUDA(cudaGetDevice(dev), "cudaGetDevice");
    return CABL_OK;
}

// ---------------------------------------------------------------- scratch
// Keyed by (device, stream handle).  A destroyed stream may still be running
// a kernel that uses its scratch when the driver hands the same handle to a
// new stream; the entry therefore remembers the stream's process-unique ID
// (cudaStreamGetId) and a call that finds a different ID gets a fresh entry
// (the old buffers are abandoned, never freed under a running kernel).  The
// ID cannot be queried while a stream is capturing a graph; captured calls
// use the entry their warm-up call created.
struct WsKey {
    int device;
    cudaStream_t stream;
    std::thread::id tid; // only for the per-thread default stream
    bool operator<(const WsKey& o) const {
        return std::tie(device, stream, tid) < std::tie(o.device, o.stream, o.tid);
    }
};

struct WsEntry {
    Workspace ws;
    unsigned long long stream_id = 0; // 0 = not yet known
    std::mutex mu;                    // held from scratch sizing to kernel enqueue (WsLease)
};

std::mutex g_ws_mu;
std::map<WsKey, WsEntry*>& ws_map() {
    static auto* m = new std::map<WsKey, WsEntry*>(); // leaked on purpose: no teardown order issues
    return *m;
}

// A lease holds the (device, stream) entry's lock from before the scratch is
// (re)sized until after the kernel that uses it is enqueued, so a concurrent
// caller on the same stream cannot free (stream-ordered) a buffer that an
// earlier-acquired, not-yet-enqueued launch is about to use.
struct WsLease {
    std::unique_lock<std::mutex> lock;
    Workspace ws;
};

int get_workspace(int device, cudaStream_t s, const WorkspaceNeed& need, WsLease* out) {
    if (need.counters == 0 && need.scratch_bytes == 0 && need.slots == 0) {
        out->ws = Workspace{};
        return CABL_OK;
    }
    unsigned long long sid = 0;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) {
        cudaGetLastError();
        cap = cudaStreamCaptureStatusActive; // cannot tell: do not query the ID
    }
    if (cap == cudaStreamCaptureStatusNone && cudaStreamGetId(s, &sid) != cudaSuccess) {
        cudaGetLastError();
        sid = 0;
    }
    WsKey key{device, s, s == cudaStreamPerThread ? std::this_thread::get_id() : std::thread::id()};
    WsEntry* ent;
    {
        std::lock_guard<std::mutex> lk(g_ws_mu);
        auto& m = ws_map();
        auto it = m.find(key);
        if (it == m.end()) {
            it = m.emplace(key, new WsEntry()).first;
        } else if (sid != 0 && it->second->stream_id != 0 && it->second->stream_id != sid) {
            it->second = new WsEntry(); // handle reused by a new stream: abandon the old entry
        }
        ent = it->second;
        if (sid != 0) ent->stream_id = sid;
    }
    out->lock = std::unique_lock<std::mutex>(ent->mu);
    Workspace& ws = ent->ws;
    if (need.counters > ws.n_counters) {
        size_t cnt = need.counters < 1024 ? 1024 : need.counters * 2;
        void* p = nullptr;
        CABL_TRY_CUDA(cudaMallocAsync(&p, cnt * sizeof(unsigned), s), "workspace counters");
        CABL_TRY_CUDA(cudaMemsetAsync(p, 0, cnt * sizeof(unsigned), s), "workspace memset");
        if (ws.counters) cudaFreeAsync(ws.counters, s);
        ws.counters = static_cast<unsigned*>(p);
        ws.n_counters = cnt;
    }
    if (need.scratch_bytes > ws.scratch_bytes) {
        size_t bytes = need.scratch_bytes < (1u << 20) ? (1u << 20) : need.scratch_bytes * 2;
        void* p = nullptr;
        CABL_TRY_CUDA(cudaMallocAsync(&p, bytes, s), "workspace scratch");
        if (ws.scratch) cudaFreeAsync(ws.scratch, s);
        ws.scratch = p;
        ws.scratch_bytes = bytes;
    }
    if (need.slots > ws.n_slots) {
        // zeroed once: epoch 0 and untagged partials (dot.cu's collector)
        size_t cnt = need.slots < 1024 ? 1024 : need.slots * 2;
        void* p = nullptr;
        CABL_TRY_CUDA(cudaMallocAsync(&p, cnt * sizeof(unsigned long long), s), "workspace slots");
        CABL_TRY_CUDA(cudaMemsetAsync(p, 0, cnt * sizeof(unsigned long long), s), "workspace memset");
        if (ws.slots) cudaFreeAsync(ws.slots, s);
        ws.slots = static_cast<unsigned long long*>(p);
        ws.n_slots = cnt;
    }
    out->ws = ws;
    return CABL_OK;
}

void set_probe(cabl_probe* p, int variant, unsigned ctas) {
    if (p) {
        p->variant = variant;
        p->threads_used = ctas < 1 ? 1u : ctas;
    }
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }


// ------------------------------------------------------------------- DOT
template <typename T>
int dot_impl(const T* x, const T* y, uint64_t n, T alpha0, T* out, uint64_t cutoff,
             cabl_probe* probe, void* stream) {
    if (!out) return fail(CABL_EINVAL, "dot: out must not be null");
    if (n > 0 && (!x || !y)) return fail(CABL_EINVAL, "dot: x and y must not be null");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    const bool small = n <= cutoff; // reference kernels.hpp:140
    cudaStream_t s = as_stream(stream);
    WsLease lease;
    if (int rc = get_workspace(dev, s, dot_need<T>(n, small), &lease)) return rc;
    LaunchInfo info;
    CABL_TRY_CUDA(dot_launch<T>(x, y, n, alpha0, out, small, lease.ws, s, &info), "dot kernel");
    set_probe(probe, small ? CABL_VARIANT_DOT_SMALL : CABL_VARIANT_DOT_BLOCKED, info.ctas);
    return CABL_OK;
}

template <typename T>
int combine_impl(const T* p, uint32_t count, T alpha0, T* out, void* stream) {
    if (!out || (count > 0 && !p)) return fail(CABL_EINVAL, "combine: null pointer");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    CABL_TRY_CUDA(combine_partials_launch<T>(p, count, alpha0, out, as_stream(stream)),
                  "combine kernel");
    return CABL_OK;
}

template <typename T>
int combine_rows_impl(const T* parts, uint32_t count, uint64_t m, T* c, void* stream) {
    if (m > 0 && (!c || (count > 0 && !parts))) return fail(CABL_EINVAL, "combine_rows: null pointer");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    CABL_TRY_CUDA(combine_rows_launch<T>(parts, count, m, c, as_stream(stream)),
                  "combine_rows kernel");
    return CABL_OK;
}

// ------------------------------------------------- peer-memory DOT (peer.cu)
unsigned long long peer_timeout_ns() {
    static const unsigned long long ns = [] {
        const char* e = getenv("CABL_PEER_TIMEOUT_MS");
        const unsigned long long ms = e ? strtoull(e, nullptr, 10) : 30000ull;
        return (ms ? ms : 30000ull) * 1000000ull;
    }();
    return ns;
}

template <typename T>
int peer_common_checks(int world, void* const* mboxes) {
    if (world < 1 || world > kMaxPeers)
        return fail(CABL_EINVAL, "dot_peer: world must be in [1, 8] (one NVLink domain)");
    if (!mboxes) return fail(CABL_EINVAL, "dot_peer: mailbox table must not be null");
    for (int g = 0; g < world; ++g)
        if (!mboxes[g]) return fail(CABL_EINVAL, "dot_peer: null mailbox in the table");
    return CABL_OK;
}

// Fill local slot lr of the argument block from the rank's operands and the
// single-GPU plan; `ws` provides its partials and counters.
template <typename T>
void peer_slot(PeerDotArgs<T>& a, int lr, const T* x, const T* y, uint64_t n, T* out,
               const DotPlan& p, T* partials, unsigned* counters) {
    a.x[lr] = x;
    a.y[lr] = y;
    a.out[lr] = out;
    a.n[lr] = n;
    a.head[lr] = p.head;
    a.chunk[lr] = p.chunk;
    a.partials[lr] = partials;
    a.counters[lr] = counters;
    a.grid[lr] = p.grid;
    a.vec_ok[lr] = p.vec_ok;
}

template <typename T>
int dot_peer_impl(const T* x, const T* y, uint64_t n, T alpha0, T* out, void* const* mboxes,
                  int world, int rank, uint64_t cutoff, cabl_probe* probe, void* stream) {
    if (!out) return fail(CABL_EINVAL, "dot_peer: out must not be null");
    if (n > 0 && (!x || !y)) return fail(CABL_EINVAL, "dot_peer: x and y must not be null");
    if (int rc = peer_common_checks<T>(world, mboxes)) return rc;
    if (rank < 0 || rank >= world) return fail(CABL_EINVAL, "dot_peer: rank must be in [0, world)");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    const bool small = n <= cutoff;
    cudaStream_t s = as_stream(stream);
    WsLease lease;
    if (int rc = get_workspace(dev, s, dot_need<T>(n, small), &lease)) return rc;
    const DotPlan p = dot_plan<T>(x, y, n, small);
    PeerDotArgs<T> a{};
    peer_slot(a, 0, x, y, n, out, p, static_cast<T*>(lease.ws.scratch), lease.ws.counters);
    for (int g = 0; g < world; ++g) a.mbox[g] = mboxes[g];
    a.world = world;
    a.rank0 = rank;
    a.timeout_ns = peer_timeout_ns();
    a.prefetch = pdl_prefetch_enabled();
    a.alpha0 = alpha0;
    CABL_TRY_CUDA(dot_peer_launch<T>(a, 1, p.chunked, p.head != 0, false, s), "dot_peer kernel");
    set_probe(probe, small ? CABL_VARIANT_DOT_SMALL : CABL_VARIANT_DOT_BLOCKED, p.grid);
    return CABL_OK;
}

template <typename T>
int dot_peer_emulate_impl(int world, const T* const* xs, const T* const* ys, const uint64_t* ns,
                          T alpha0, T* const* outs, void* const* mboxes, uint64_t cutoff,
                          void* stream) {
    if (int rc = peer_common_checks<T>(world, mboxes)) return rc;
    if (!xs || !ys || !ns || !outs) return fail(CABL_EINVAL, "dot_peer_emulate: null table");
    for (int r = 0; r < world; ++r) {
        if (!outs[r]) return fail(CABL_EINVAL, "dot_peer_emulate: out must not be null");
        if (ns[r] > 0 && (!xs[r] || !ys[r]))
            return fail(CABL_EINVAL, "dot_peer_emulate: x and y must not be null");
    }
    int dev;
    if (int rc = current_device(&dev)) return rc;
    DotPlan plan[kMaxPeers];
    size_t per_rank = 256;
    bool chunked = false, peel = false;
    unsigned gx = 1;
    for (int r = 0; r < world; ++r) {
        const bool small = ns[r] <= cutoff;
        plan[r] = dot_plan<T>(xs[r], ys[r], ns[r], small);
        const WorkspaceNeed w = dot_need<T>(ns[r], small);
        per_rank = w.scratch_bytes > per_rank ? w.scratch_bytes : per_rank;
        if (r > 0 && plan[r].chunked != chunked)
            return fail(CABL_EINVAL, "dot_peer_emulate: every rank must take the same DOT kernel");
        chunked = plan[r].chunked;
        peel = peel || plan[r].head != 0;
        gx = plan[r].grid > gx ? plan[r].grid : gx;
    }
    per_rank = (per_rank + 255) / 256 * 256;
    // every waiting CTA must be co-resident: one cooperative wave
    const int per_sm = dot_peer_ctas_per_sm(chunked, sizeof(T));
    if (uint64_t(gx) * uint64_t(world) > uint64_t(per_sm) * uint64_t(sm_count()))
        return fail(CABL_EINVAL, "dot_peer_emulate: the emulated ranks' grids do not fit one "
                                 "co-resident wave (use smaller shards)");
    cudaStream_t s = as_stream(stream);
    WorkspaceNeed need;
    need.counters = 2 * size_t(world);
    need.scratch_bytes = per_rank * size_t(world);
    WsLease lease;
    if (int rc = get_workspace(dev, s, need, &lease)) return rc;
    PeerDotArgs<T> a{};
    for (int r = 0; r < world; ++r)
        peer_slot(a, r, xs[r], ys[r], ns[r], outs[r], plan[r],
                  reinterpret_cast<T*>(static_cast<char*>(lease.ws.scratch) + per_rank * r),
                  lease.ws.counters + 2 * r);
    for (int g = 0; g < world; ++g) a.mbox[g] = mboxes[g];
    a.world = world;
    a.rank0 = 0;
    a.timeout_ns = peer_timeout_ns();
    a.prefetch = pdl_prefetch_enabled();
    a.alpha0 = alpha0;
    CABL_TRY_CUDA(dot_peer_launch<T>(a, world, chunked, peel, true, s), "dot_peer_emulate kernel");
    return CABL_OK;
}

// ------------------------------------ rank-ordered row combine, peer memory
template <typename T>
int rows_peer_fill(PeerRowsArgs<T>& a, int world, uint64_t m, void* const* slots,
                   void* const* mboxes) {
    if (world < 1 || world > kMaxPeers)
        return fail(CABL_EINVAL, "combine_rows_peer: world must be in [1, 8] (one NVLink domain)");
    if (!slots || !mboxes) return fail(CABL_EINVAL, "combine_rows_peer: null peer table");
    for (int g = 0; g < world; ++g) {
        if (!slots[g] || !mboxes[g]) return fail(CABL_EINVAL, "combine_rows_peer: null entry in a peer table");
        a.slots[g] = static_cast<T*>(slots[g]);
        a.mbox[g] = mboxes[g];
    }
    a.m = m;
    a.world = world;
    a.timeout_ns = peer_timeout_ns();
    return CABL_OK;
}

template <typename T>
int combine_rows_peer_impl(const T* part, uint64_t m, T* c, void* const* slots,
                           void* const* mboxes, int world, int rank, void* stream) {
    PeerRowsArgs<T> a{};
    if (int rc = rows_peer_fill<T>(a, world, m, slots, mboxes)) return rc;
    if (rank < 0 || rank >= world) return fail(CABL_EINVAL, "combine_rows_peer: rank must be in [0, world)");
    if (m == 0) return CABL_OK;
    if (!part || !c) return fail(CABL_EINVAL, "combine_rows_peer: null pointer");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    a.part[0] = part;
    a.c[0] = c;
    a.rank0 = rank;
    CABL_TRY_CUDA(combine_rows_peer_launch<T>(a, 1, false, as_stream(stream)), "combine_rows_peer kernel");
    return CABL_OK;
}

template <typename T>
int combine_rows_peer_emulate_impl(int world, const T* const* parts, uint64_t m, T* const* cs,
                                   void* const* slots, void* const* mboxes, void* stream) {
    PeerRowsArgs<T> a{};
    if (int rc = rows_peer_fill<T>(a, world, m, slots, mboxes)) return rc;
    if (m == 0) return CABL_OK;
    if (!parts || !cs) return fail(CABL_EINVAL, "combine_rows_peer_emulate: null table");
    for (int r = 0; r < world; ++r) {
        if (!parts[r] || !cs[r]) return fail(CABL_EINVAL, "combine_rows_peer_emulate: null pointer");
        a.part[r] = parts[r];
        a.c[r] = cs[r];
    }
    int dev;
    if (int rc = current_device(&dev)) return rc;
    a.rank0 = 0;
    CABL_TRY_CUDA(combine_rows_peer_launch<T>(a, world, true, as_stream(stream)),
                  "combine_rows_peer_emulate kernel");
    return CABL_OK;
}

// ------------------------------------- row-major GEMV + fused all-gather
// Fence between the pushes and the completion words: none at world 1 (no
// peer reads the buffers), else fence.acq_rel.sys; CABL_GATHER_FENCE=0|1|2
// overrides (A/B only; 2 = fence.sc.sys).
int gather_fence(int world) {
    static const int forced = [] {
        const char* e = getenv("CABL_GATHER_FENCE");
        return e ? atoi(e) : -1;
    }();
    if (forced >= 0) return forced;
    return world > 1 ? 1 : 0;
}

template <typename T>
int gather_common_checks(int world, void* const* cfull, void* const* mboxes, uint64_t n,
                         uint64_t m_total) {
    if (world < 1 || world > kMaxPeers)
        return fail(CABL_EINVAL, "gemv_rm_gather: world must be in [1, 8] (one NVLink domain)");
    if (!cfull || !mboxes) return fail(CABL_EINVAL, "gemv_rm_gather: null peer table");
    for (int g = 0; g < world; ++g)
        if (!cfull[g] || !mboxes[g]) return fail(CABL_EINVAL, "gemv_rm_gather: null entry in a peer table");
    if (n == 0 || m_total == 0) return fail(CABL_EINVAL, "gemv_rm_gather: empty matrix");
    return CABL_OK;
}

template <typename T>
int gather_supported_impl(const T* A, uint64_t m, uint64_t n, const T* x, int* ok) {
    if (!ok) return fail(CABL_EINVAL, "gemv_rm_gather_supported: null result pointer");
    *ok = 0;
    if (!A || !x || m == 0 || n == 0) return CABL_OK;
    int dev;
    if (int rc = current_device(&dev)) return rc;
    int R, KV, mb;
    *ok = gemv_rm_sweep_cfg<T>(A, x, m, n, &R, &KV, &mb) &&
          gemv_rm_gather_ctas_per_sm(R, KV, mb, sizeof(T)) != 0;
    return CABL_OK;
}

template <typename T>
int gemv_gather_impl(const T* A, uint64_t m, uint64_t n, const T* x, T* c, uint64_t row_off,
                     uint64_t m_total, void* const* cfull, void* const* mboxes, int world, int rank,
                     cabl_probe* probe, void* stream) {
    if (int rc = gather_common_checks<T>(world, cfull, mboxes, n, m_total)) return rc;
    if (rank < 0 || rank >= world) return fail(CABL_EINVAL, "gemv_rm_gather: rank must be in [0, world)");
    if (!A || !x || !c || m == 0) return fail(CABL_EINVAL, "gemv_rm_gather: null operand or empty slice");
    if (row_off + m > m_total) return fail(CABL_EINVAL, "gemv_rm_gather: slice outside the gathered c");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    int R, KV, mb;
    if (!gemv_rm_sweep_cfg<T>(A, x, m, n, &R, &KV, &mb) || gemv_rm_gather_ctas_per_sm(R, KV, mb, sizeof(T)) == 0)
        return fail(CABL_EINVAL, "gemv_rm_gather: this slice shape does not take the sweep kernel "
                                 "(use gemv_rm + a collective)");
    cudaStream_t s = as_stream(stream);
    WorkspaceNeed need;
    need.counters = 2;
    WsLease lease;
    if (int rc = get_workspace(dev, s, need, &lease)) return rc;
    PeerGemvArgs<T> a{};
    const uint64_t groups = (m + R - 1) / R;
    const uint64_t cap = uint64_t(sm_count()) * mb;
    a.A[0] = A;
    a.x[0] = x;
    a.c[0] = c;
    a.m[0] = m;
    a.row_off[0] = row_off;
    a.grid[0] = unsigned(groups < cap ? groups : cap);
    a.counters[0] = lease.ws.counters;
    for (int g = 0; g < world; ++g) {
        a.cfull[g] = static_cast<T*>(cfull[g]);
        a.mbox[g] = mboxes[g];
    }
    a.n = n;
    a.m_total = m_total;
    a.world = world;
    a.rank0 = rank;
    a.timeout_ns = peer_timeout_ns();
    a.fence = gather_fence(world);
    const bool dyn = gemv_rm_use_dyn(m * n * sizeof(T));
    CABL_TRY_CUDA(gemv_rm_gather_launch<T>(a, 1, R, KV, mb, dyn, false, s), "gemv_rm_gather kernel");
    set_probe(probe, CABL_VARIANT_GEMV_ROW, a.grid[0]);
    return CABL_OK;
}

template <typename T>
int gemv_gather_emulate_impl(int world, const T* const* As, const uint64_t* ms, uint64_t n,
                             const T* const* xs, T* const* cs, const uint64_t* row_offs,
                             uint64_t m_total, void* const* cfull, void* const* mboxes,
                             void* stream) {
    if (int rc = gather_common_checks<T>(world, cfull, mboxes, n, m_total)) return rc;
    if (!As || !ms || !xs || !cs || !row_offs) return fail(CABL_EINVAL, "gemv_rm_gather_emulate: null table");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    int R = 0, KV = 0, mb = 0;
    for (int r = 0; r < world; ++r) {
        if (!As[r] || !xs[r] || !cs[r] || ms[r] == 0 || row_offs[r] + ms[r] > m_total)
            return fail(CABL_EINVAL, "gemv_rm_gather_emulate: bad slice");
        int r_, kv_, mb_;
        if (!gemv_rm_sweep_cfg<T>(As[r], xs[r], ms[r], n, &r_, &kv_, &mb_))
            return fail(CABL_EINVAL, "gemv_rm_gather_emulate: a slice does not take the sweep kernel");
        if (r > 0 && (r_ != R || kv_ != KV || mb_ != mb))
            return fail(CABL_EINVAL, "gemv_rm_gather_emulate: every slice must take the same sweep shape");
        R = r_, KV = kv_, mb = mb_;
    }
    const int per_sm = gemv_rm_gather_ctas_per_sm(R, KV, mb, sizeof(T));
    if (per_sm == 0) return fail(CABL_EINVAL, "gemv_rm_gather_emulate: unsupported sweep shape");
    // every rank's grid in one co-resident wave
    const uint64_t share = uint64_t(sm_count()) * uint64_t(per_sm) / uint64_t(world);
    if (share == 0) return fail(CABL_EINVAL, "gemv_rm_gather_emulate: too many ranks for one wave");
    cudaStream_t s = as_stream(stream);
    WorkspaceNeed need;
    need.counters = 2 * size_t(world);
    WsLease lease;
    if (int rc = get_workspace(dev, s, need, &lease)) return rc;
    PeerGemvArgs<T> a{};
    bool dyn = false;
    for (int r = 0; r < world; ++r) {
        const uint64_t groups = (ms[r] + R - 1) / R;
        a.A[r] = As[r];
        a.x[r] = xs[r];
        a.c[r] = cs[r];
        a.m[r] = ms[r];
        a.row_off[r] = row_offs[r];
        a.grid[r] = unsigned(groups < share ? groups : share);
        a.counters[r] = lease.ws.counters + 2 * r;
        dyn = dyn || gemv_rm_use_dyn(ms[r] * n * sizeof(T));
    }
    for (int g = 0; g < world; ++g) {
        a.cfull[g] = static_cast<T*>(cfull[g]);
        a.mbox[g] = mboxes[g];
    }
    a.n = n;
    a.m_total = m_total;
    a.world = world;
    a.rank0 = 0;
    a.timeout_ns = peer_timeout_ns();
    a.fence = gather_fence(world);
    CABL_TRY_CUDA(gemv_rm_gather_launch<T>(a, world, R, KV, mb, dyn, true, s),
                  "gemv_rm_gather_emulate kernel");
    return CABL_OK;
}

// ------------------------------------------------------------------ GEMV
// Row-major GEMV runs the deterministic sweep kernels (BASELINE tolerance,
// bitwise run to run) by default; CABL_GEMV_RM_ORDER=reference selects the
// reference-order kernel (bit for bit gemv_ref, gemv_rm_ordered.cu) wherever
// the shape allows.  The sweep is ~14% faster on G1/G4.
bool rm_reference_order() {
    static const bool ref = [] {
        const char* e = tuning_env("CABL_GEMV_RM_ORDER");
        return e && std::string(e) == "reference";
    }();
    return ref;
}

template <typename T>
int gemv_impl(const T* A, int layout, uint64_t m, uint64_t n, const T* x, T* c,
              uint64_t cutoff, cabl_probe* probe, void* stream) {
    if (m > 0 && n > 0 && (!A || !x || !c))
        return fail(CABL_EINVAL, "gemv: A, x and c must not be null");
    if (c != nullptr && static_cast<const void*>(c) == static_cast<const void*>(x))
        return fail(CABL_EINVAL, "gemv: c must not alias x"); // kernels.hpp:176,193,236
    int dev;
    if (int rc = current_device(&dev)) return rc;
    const int variant = layout == CABL_ROW_MAJOR ? CABL_VARIANT_GEMV_ROW
                                                 : CABL_VARIANT_GEMV_COL_BLOCKED;
    const uint64_t touched = m * n + m + n; // kernels.hpp:240
    cudaStream_t s = as_stream(stream);
    LaunchInfo info;
    if (touched <= cutoff) {
        CABL_TRY_CUDA(gemv_ordered_launch<T>(A, layout, m, n, x, c, s, &info), "gemv kernel");
    } else if (layout == CABL_ROW_MAJOR && rm_reference_order() &&
               !gemv_rm_is_lane(A, x, m, n, sizeof(T)) && gemv_rm_ordered_ok<T>(A, x, m, n)) {
        CABL_TRY_CUDA(gemv_rm_ordered_launch<T>(A, m, n, x, c, s, &info), "gemv_rm kernel");
    } else if (layout == CABL_ROW_MAJOR) {
        WsLease lease;
        if (int rc = get_workspace(dev, s, gemv_rm_need<T>(A, x, m, n), &lease)) return rc;
        CABL_TRY_CUDA(gemv_rm_launch<T>(A, m, n, x, c, lease.ws, s, &info), "gemv_rm kernel");
    } else {
        WsLease lease;
        if (int rc = get_workspace(dev, s, gemv_cm_need<T>(A, x, m, n), &lease)) return rc;
        CABL_TRY_CUDA(gemv_cm_launch<T>(A, m, n, x, c, lease.ws, s, &info), "gemv_cm kernel");
    }
    set_probe(probe, variant, info.ctas);
    return CABL_OK;
}

// ------------------------------------------------------------------- GER
template <typename T>
int ger_impl(const T* x, const T* y, T* C, int layout, uint64_t m, uint64_t n, uint64_t cutoff,
             cabl_probe* probe, void* stream) {
    if (m > 0 && n > 0 && (!x || !y || !C))
        return fail(CABL_EINVAL, "ger: x, y and C must not be null");
    if (C != nullptr && (static_cast<const void*>(C) == static_cast<const void*>(x) ||
                         static_cast<const void*>(C) == static_cast<const void*>(y)))
        return fail(CABL_EINVAL, "ger: C must not alias x or y"); // kernels.hpp:281-282
    int dev;
    if (int rc = current_device(&dev)) return rc;
    const uint64_t touched = m * n + m + n; // kernels.hpp:285-287
    const bool small = touched <= cutoff;
    LaunchInfo info;
    cudaStream_t s = as_stream(stream);
    WsLease lease;
    if (int rc = get_workspace(dev, s, ger_need<T>(x, y, m, n), &lease)) return rc;
    if (layout == CABL_ROW_MAJOR)
        CABL_TRY_CUDA(ger_launch<T>(x, y, C, m, n, small, lease.ws, s, &info), "ger kernel");
    else
        CABL_TRY_CUDA(ger_launch<T>(y, x, C, n, m, small, lease.ws, s, &info), "ger kernel");
    set_probe(probe, CABL_VARIANT_GER, info.ctas);
    return CABL_OK;
}

// ---------------------------------------------------- host-buffer staging
struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

int dev_alloc(DevBuf& b, size_t bytes, cudaStream_t s) {
    b.s = s;
    if (bytes == 0) bytes = 32;
    CABL_TRY_CUDA(cudaMallocAsync(&b.p, bytes, s), "staging alloc");
    return CABL_OK;
}

void keep_pool_warm(int dev) {
    // Stream-ordered frees return memory to the device pool; keep it there
    // instead of releasing it at every synchronize.
    static std::once_flag flags[64];
    if (dev < 0 || dev >= 64) return;
    std::call_once(flags[dev], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = ~0ULL;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
}

// ---- pageable host memory: multi-threaded staging through pinned slots ----
// cudaMemcpyAsync from pageable memory is staged by the driver through one
// thread (~12 GB/s on the GPU box: 22 ms for G1's 256 MB A, where pinned
// memory takes 5.6 ms).  Large transfers from/to unregistered host memory
// therefore go through kStageThreads worker threads, each owning a pinned
// kStageChunk slot: a worker copies chunk k into its slot with memcpy and
// enqueues the DMA from it (H2D), or waits for the DMA into it and copies
// out (D2H); chunks k = t, t + T, ... belong to worker t, so T chunks are in
// flight at once.  Each worker has its own stream: the caller's stream is
// synchronized first (the destination is stream-ordered staging memory, and
// a D2H source is produced by work on it — and the per-thread default stream
// of the caller is not reachable from another thread), and every worker
// waits for its last DMA, so the data is in place when the call returns.  One
// staged transfer per device at a time (the slots are per device).
constexpr size_t kStageChunk = size_t(8) << 20;
constexpr size_t kStageMin = size_t(4) << 20; // smaller transfers: plain copy
constexpr unsigned kStageThreads = 8;

struct Stager {
    std::mutex mu;
    void* slot[kStageThreads] = {};
    cudaEvent_t ev[kStageThreads] = {};
    cudaStream_t stream[kStageThreads] = {};
    bool ready = false;
};

Stager& stager(int dev) {
    static Stager st[64];
    return st[dev & 63];
}

bool is_pageable(const void* h) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

int stage_init(Stager& st) {
    if (st.ready) return CABL_OK;
    for (unsigned t = 0; t < kStageThreads; ++t) {
        CABL_TRY_CUDA(cudaMallocHost(&st.slot[t], kStageChunk), "pinned staging slot");
        CABL_TRY_CUDA(cudaEventCreateWithFlags(&st.ev[t], cudaEventDisableTiming), "staging event");
        CABL_TRY_CUDA(cudaStreamCreateWithFlags(&st.stream[t], cudaStreamNonBlocking),
                      "staging stream");
    }
    st.ready = true;
    return CABL_OK;
}

// H2D (to_device) or D2H through the slots; returns the first CUDA error
int staged_copy(int dev, void* dst, const void* src, size_t bytes, cudaStream_t s,
                bool to_device) {
    Stager& st = stager(dev);
    std::lock_guard<std::mutex> lk(st.mu);
    if (int rc = stage_init(st)) return rc;
    CABL_TRY_CUDA(cudaStreamSynchronize(s), "staging sync");
    const size_t chunks = (bytes + kStageChunk - 1) / kStageChunk;
    const unsigned T = unsigned(chunks < kStageThreads ? chunks : kStageThreads);
    std::atomic<int> err{0}; // first failing cudaError_t
    auto fail_with = [&](cudaError_t e) {
        int expected = 0;
        err.compare_exchange_strong(expected, int(e));
    };
    auto worker = [&](unsigned t) {
        if (cudaError_t e = cudaSetDevice(dev)) {
            fail_with(e);
            return;
        }
        bool first = true;
        for (size_t k = t; k < chunks && !err.load(); k += T) {
            const size_t off = k * kStageChunk;
            const size_t len = bytes - off < kStageChunk ? bytes - off : kStageChunk;
            cudaError_t e = cudaSuccess;
            if (to_device) {
                // the slot's previous DMA (this transfer's or an earlier, failed
                // one's) must be done before it is overwritten; a never-recorded
                // event is complete
                e = cudaEventSynchronize(st.ev[t]);
                if (e == cudaSuccess) {
                    std::memcpy(st.slot[t], static_cast<const char*>(src) + off, len);
                    e = cudaMemcpyAsync(static_cast<char*>(dst) + off, st.slot[t], len,
                                        cudaMemcpyHostToDevice, st.stream[t]);
                }
                if (e == cudaSuccess) e = cudaEventRecord(st.ev[t], st.stream[t]);
            } else {
                e = cudaMemcpyAsync(st.slot[t], static_cast<const char*>(src) + off, len,
                                    cudaMemcpyDeviceToHost, st.stream[t]);
                if (e == cudaSuccess) e = cudaEventRecord(st.ev[t], st.stream[t]);
                if (e == cudaSuccess) e = cudaEventSynchronize(st.ev[t]);
                if (e == cudaSuccess)
                    std::memcpy(static_cast<char*>(dst) + off, st.slot[t], len);
            }
            if (e != cudaSuccess) {
                fail_with(e);
                return;
            }
            first = false;
        }
        // H2D: the data must be in place before the caller's kernel runs, and
        // the slot must not be reused before the last DMA from it has read it
        if (to_device && !first)
            if (cudaError_t e = cudaEventSynchronize(st.ev[t])) fail_with(e);
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < T; ++t) th.emplace_back(worker, t);
    worker(0);
    for (auto& x : th) x.join();
    if (int e = err.load()) return cuda_fail(cudaError_t(e), "staged host copy");
    return CABL_OK;
}

int h2d(void* d, const void* h, size_t bytes, cudaStream_t s) {
    if (!bytes) return CABL_OK;
    int dev = 0;
    if (bytes >= kStageMin && cudaGetDevice(&dev) == cudaSuccess && is_pageable(h))
        return staged_copy(dev, d, h, bytes, s, true);
    CABL_TRY_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s), "H2D copy");
    return CABL_OK;
}
int d2h(void* h, const void* d, size_t bytes, cudaStream_t s) {
    if (!bytes) return CABL_OK;
    int dev = 0;
    if (bytes >= kStageMin && cudaGetDevice(&dev) == cudaSuccess && is_pageable(h))
        return staged_copy(dev, h, d, bytes, s, false);
    CABL_TRY_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s), "D2H copy");
    return CABL_OK;
}

template <typename T>
int host_dot(const T* x, const T* y, uint64_t n, T alpha0, T* result, uint64_t cutoff,
             cabl_probe* probe, void* stream) {
    if (!result) return fail(CABL_EINVAL, "dot: result must not be null");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    keep_pool_warm(dev);
    cudaStream_t s = as_stream(stream);
    {
        DevBuf dx, dy, dout;
        if (int rc = dev_alloc(dx, n * sizeof(T), s)) return rc;
        if (int rc = dev_alloc(dy, n * sizeof(T), s)) return rc;
        if (int rc = dev_alloc(dout, sizeof(T), s)) return rc;
        if (int rc = h2d(dx.p, x, n * sizeof(T), s)) return rc;
        if (int rc = h2d(dy.p, y, n * sizeof(T), s)) return rc;
        if (int rc = dot_impl<T>(static_cast<T*>(dx.p), static_cast<T*>(dy.p), n, alpha0,
                                 static_cast<T*>(dout.p), cutoff, probe, stream))
            return rc;
        if (int rc = d2h(result, dout.p, sizeof(T), s)) return rc;
    }
    CABL_TRY_CUDA(cudaStreamSynchronize(s), "dot sync");
    return CABL_OK;
}

template <typename T>
int host_gemv(const T* A, int layout, uint64_t m, uint64_t n, const T* x, T* c, uint64_t cutoff,
              cabl_probe* probe, void* stream) {
    if (layout != CABL_ROW_MAJOR && layout != CABL_COL_MAJOR)
        return fail(CABL_EINVAL, "gemv: bad layout");
    if (c != nullptr && static_cast<const void*>(c) == static_cast<const void*>(x))
        return fail(CABL_EINVAL, "gemv: c must not alias x");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    keep_pool_warm(dev);
    cudaStream_t s = as_stream(stream);
    {
        DevBuf dA, dx, dc;
        if (int rc = dev_alloc(dA, m * n * sizeof(T), s)) return rc;
        if (int rc = dev_alloc(dx, n * sizeof(T), s)) return rc;
        if (int rc = dev_alloc(dc, m * sizeof(T), s)) return rc;
        if (int rc = h2d(dA.p, A, m * n * sizeof(T), s)) return rc;
        if (int rc = h2d(dx.p, x, n * sizeof(T), s)) return rc;
        if (int rc = h2d(dc.p, c, m * sizeof(T), s)) return rc;
        if (int rc = gemv_impl<T>(static_cast<T*>(dA.p), layout, m, n, static_cast<T*>(dx.p),
                                  static_cast<T*>(dc.p), cutoff, probe, stream))
            return rc;
        if (int rc = d2h(c, dc.p, m * sizeof(T), s)) return rc;
    }
    CABL_TRY_CUDA(cudaStreamSynchronize(s), "gemv sync");
    return CABL_OK;
}

// ---- pinned host C: the GER host path as a three-stream pipeline ----------
// C is read H2D and written back D2H, 2 x m*n*s over PCIe.  Done one after
// the other the two transfers take twice the link time; PCIe is full duplex,
// so the path splits C into slabs along its major dimension (whole rows of a
// row-major C, whole columns of a col-major one — contiguous host bytes) and
// runs H2D of slab k+1, the GER of slab k and the D2H of slab k-1 at once on
// three library streams (event-ordered).  Each element is still exactly one
// fma(x_i, y_j, C_ij): the bits equal the unsplit call's.
constexpr size_t kPipeSlabMin = size_t(8) << 20;
constexpr int kPipeMaxSlabs = 32;
constexpr int kPipeSlabs = 16;

struct HostPipe {
    std::mutex mu;
    cudaStream_t in = nullptr, work = nullptr, out = nullptr;
    cudaEvent_t start = nullptr;
    cudaEvent_t loaded[kPipeMaxSlabs] = {}, done[kPipeMaxSlabs] = {};
    bool ready = false;
};

HostPipe& host_pipe(int dev) {
    static HostPipe p[64];
    return p[dev & 63];
}

int pipe_init(HostPipe& p) {
    if (p.ready) return CABL_OK;
    CABL_TRY_CUDA(cudaStreamCreateWithFlags(&p.in, cudaStreamNonBlocking), "pipeline stream");
    CABL_TRY_CUDA(cudaStreamCreateWithFlags(&p.work, cudaStreamNonBlocking), "pipeline stream");
    CABL_TRY_CUDA(cudaStreamCreateWithFlags(&p.out, cudaStreamNonBlocking), "pipeline stream");
    CABL_TRY_CUDA(cudaEventCreateWithFlags(&p.start, cudaEventDisableTiming), "pipeline event");
    for (int k = 0; k < kPipeMaxSlabs; ++k) {
        CABL_TRY_CUDA(cudaEventCreateWithFlags(&p.loaded[k], cudaEventDisableTiming), "pipeline event");
        CABL_TRY_CUDA(cudaEventCreateWithFlags(&p.done[k], cudaEventDisableTiming), "pipeline event");
    }
    p.ready = true;
    return CABL_OK;
}

template <typename T>
int host_ger_pipelined(int dev, const T* x, const T* y, T* C, int layout, uint64_t m, uint64_t n,
                       uint64_t cutoff, cabl_probe* probe, cudaStream_t s) {
    HostPipe& p = host_pipe(dev);
    std::lock_guard<std::mutex> lk(p.mu);
    if (int rc = pipe_init(p)) return rc;
    // major dimension (slabs) and the vector that follows it
    const bool rm = layout == CABL_ROW_MAJOR;
    const uint64_t outer = rm ? m : n, inner = rm ? n : m;
    const size_t line = size_t(inner) * sizeof(T);
    const size_t total = size_t(outer) * line;
    // About kPipeSlabs slabs of >= 8 MiB: each copy has a fixed cost, and
    // the pipeline fills and drains in one slab's time (256 MiB fp32 pinned,
    // tools/ger_pipe.py — 4 / 8 / 16 / 32 / 64 / 128 slabs: 6.55 / 6.10 /
    // 5.99 / 6.24 / 6.62 / 7.75 ms; the same copy pattern without the GER
    // kernel, tools/pcie_duplex.py: 5.74 ms at 16 slabs; both directions at
    // once with no dependency: 5.37).  Ramping the first and last slabs
    // (1/8, 1/4, 1/2 of a slab) changed nothing.  CABL_GER_PIPE=
    // "slabs,min_mib" overrides (tuning only).
    static const std::pair<int, size_t> pipe_cfg = [] {
        int sl = kPipeSlabs;
        unsigned long mib = kPipeSlabMin >> 20;
        if (const char* e = tuning_env("CABL_GER_PIPE")) sscanf(e, "%d,%lu", &sl, &mib);
        if (sl < 1 || sl > kPipeMaxSlabs) sl = kPipeSlabs;
        return std::make_pair(sl, size_t(mib) << 20);
    }();
    size_t slab = total / size_t(pipe_cfg.first) + 1;
    if (slab < pipe_cfg.second) slab = pipe_cfg.second;
    uint64_t lines = (slab + line - 1) / line;
    if (lines < 1) lines = 1;
    const uint64_t slabs = (outer + lines - 1) / lines; // <= the slab count
    DevBuf dx, dy, dC;
    if (int rc = dev_alloc(dx, m * sizeof(T), s)) return rc;
    if (int rc = dev_alloc(dy, n * sizeof(T), s)) return rc;
    if (int rc = dev_alloc(dC, total, s)) return rc;
    // the library streams start after everything already on the caller's
    // stream (including these allocations)
    CABL_TRY_CUDA(cudaEventRecord(p.start, s), "pipeline event");
    for (cudaStream_t q : {p.in, p.work, p.out})
        CABL_TRY_CUDA(cudaStreamWaitEvent(q, p.start, 0), "pipeline wait");
    CABL_TRY_CUDA(cudaMemcpyAsync(dx.p, x, m * sizeof(T), cudaMemcpyHostToDevice, p.in), "H2D x");
    CABL_TRY_CUDA(cudaMemcpyAsync(dy.p, y, n * sizeof(T), cudaMemcpyHostToDevice, p.in), "H2D y");
    T* dCt = static_cast<T*>(dC.p);
    const T* dxt = static_cast<const T*>(dx.p);
    const T* dyt = static_cast<const T*>(dy.p);
    const int rc = [&]() -> int {
    for (uint64_t k = 0; k < slabs; ++k) {
        const uint64_t o0 = k * lines, cnt = (outer - o0 < lines) ? outer - o0 : lines;
        const size_t off = size_t(o0) * inner, bytes = size_t(cnt) * line;
        CABL_TRY_CUDA(cudaMemcpyAsync(dCt + off, C + off, bytes, cudaMemcpyHostToDevice, p.in), "H2D C");
        CABL_TRY_CUDA(cudaEventRecord(p.loaded[k], p.in), "pipeline event");
        CABL_TRY_CUDA(cudaStreamWaitEvent(p.work, p.loaded[k], 0), "pipeline wait");
        // the slab: rows o0.. of a row-major C take x[o0..]; columns o0.. of
        // a col-major C take y[o0..]
        const int rc = rm ? ger_impl<T>(dxt + o0, dyt, dCt + off, layout, cnt, n, cutoff,
                                        k == 0 ? probe : nullptr, p.work)
                          : ger_impl<T>(dxt, dyt + o0, dCt + off, layout, m, cnt, cutoff,
                                        k == 0 ? probe : nullptr, p.work);
        if (rc) return rc;
        CABL_TRY_CUDA(cudaEventRecord(p.done[k], p.work), "pipeline event");
        CABL_TRY_CUDA(cudaStreamWaitEvent(p.out, p.done[k], 0), "pipeline wait");
        CABL_TRY_CUDA(cudaMemcpyAsync(C + off, dCt + off, bytes, cudaMemcpyDeviceToHost, p.out), "D2H C");
    }
    return CABL_OK;
    }();
    if (rc) { // nothing may still use the staging buffers when they are freed
        for (cudaStream_t q : {p.in, p.work, p.out}) cudaStreamSynchronize(q);
        return rc;
    }
    // the caller's stream frees the staging buffers after the last D2H
    CABL_TRY_CUDA(cudaEventRecord(p.start, p.out), "pipeline event");
    CABL_TRY_CUDA(cudaStreamWaitEvent(s, p.start, 0), "pipeline wait");
    return CABL_OK;
}

bool host_pinned(const void* h) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

template <typename T>
int host_ger(const T* x, const T* y, T* C, int layout, uint64_t m, uint64_t n, uint64_t cutoff,
             cabl_probe* probe, void* stream) {
    if (layout != CABL_ROW_MAJOR && layout != CABL_COL_MAJOR)
        return fail(CABL_EINVAL, "ger: bad layout");
    if (C != nullptr && (static_cast<const void*>(C) == static_cast<const void*>(x) ||
                         static_cast<const void*>(C) == static_cast<const void*>(y)))
        return fail(CABL_EINVAL, "ger: C must not alias x or y");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    keep_pool_warm(dev);
    cudaStream_t s = as_stream(stream);
    // pinned (page-locked) C larger than one slab: the full-duplex pipeline
    if (m && n && size_t(m) * n * sizeof(T) > 2 * kPipeSlabMin && host_pinned(C)) {
        if (int rc = host_ger_pipelined<T>(dev, x, y, C, layout, m, n, cutoff, probe, s)) {
            cudaStreamSynchronize(s);
            return rc;
        }
        CABL_TRY_CUDA(cudaStreamSynchronize(s), "ger sync");
        return CABL_OK;
    }
    {
        DevBuf dx, dy, dC;
        if (int rc = dev_alloc(dx, m * sizeof(T), s)) return rc;
        if (int rc = dev_alloc(dy, n * sizeof(T), s)) return rc;
        if (int rc = dev_alloc(dC, m * n * sizeof(T), s)) return rc;
        if (int rc = h2d(dx.p, x, m * sizeof(T), s)) return rc;
        if (int rc = h2d(dy.p, y, n * sizeof(T), s)) return rc;
        if (int rc = h2d(dC.p, C, m * n * sizeof(T), s)) return rc;
        if (int rc = ger_impl<T>(static_cast<T*>(dx.p), static_cast<T*>(dy.p),
                                 static_cast<T*>(dC.p), layout, m, n, cutoff, probe, stream))
            return rc;
        if (int rc = d2h(C, dC.p, m * n * sizeof(T), s)) return rc;
    }
    CABL_TRY_CUDA(cudaStreamSynchronize(s), "ger sync");
    return CABL_OK;
}

} // namespace

namespace cabl_dev {

namespace {
// per-device facts, read once from the driver (cabl_describe_device)
struct DevFacts {
    std::atomic<int> sms{0};
    std::atomic<uint64_t> l2{0};
};
DevFacts g_facts[64];

DevFacts* facts_of_current() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return nullptr;
    }
    DevFacts& f = g_facts[dev];
    if (f.sms.load(std::memory_order_acquire) == 0) {
        int v = 0, l2 = 0;
        if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess || l2 <= 0)
            l2 = 0;
        f.l2.store(uint64_t(l2), std::memory_order_relaxed);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = 148;
        f.sms.store(v, std::memory_order_release);
    }
    return &f;
}

uint64_t threshold_from_l2(uint64_t l2) {
    uint64_t t = 1;
    while (t < 4 * l2) t <<= 1;
    return t;
}
} // namespace

int sm_count() {
    DevFacts* f = facts_of_current();
    return f ? f->sms.load(std::memory_order_acquire) : 148;
}

// Operands of at least this many bytes take the atomic work queues (DOT
// chunks, GEMV groups/units): 4 x L2 rounded up to a power of two, 512 MiB on
// B200 — a kernel that long (>= ~80 us) amortises the queue's atomics, one
// that fits a few L2s does not.
uint64_t queue_threshold_bytes() {
    DevFacts* f = facts_of_current();
    const uint64_t l2 = f ? f->l2.load(std::memory_order_relaxed) : 0;
    return threshold_from_l2(l2 ? l2 : uint64_t(126) << 20);
}

} // namespace cabl_dev

extern "C" int cabl_describe_device(int device, cabl_gpu_machine* out) {
    if (!out) return fail(CABL_EINVAL, "describe_device: out must not be null");
    cudaDeviceProp p;
    CABL_TRY_CUDA(cudaGetDeviceProperties(&p, device), "cudaGetDeviceProperties");
    std::memset(out, 0, sizeof(*out));
    out->device = device;
    out->cc_major = p.major;
    out->cc_minor = p.minor;
    out->sm_count = unsigned(p.multiProcessorCount);
    out->max_threads_per_sm = unsigned(p.maxThreadsPerMultiProcessor);
    out->line_bytes = 128;
    out->smem_per_sm = p.sharedMemPerMultiprocessor;
    out->smem_per_block_optin = p.sharedMemPerBlockOptin;
    out->l2_bytes = uint64_t(p.l2CacheSize);
    out->hbm_bytes = p.totalGlobalMem;
    out->mem_bus_bits = unsigned(p.memoryBusWidth);
    out->queue_threshold_bytes = cabl_dev::threshold_from_l2(out->l2_bytes);
    std::snprintf(out->name, sizeof(out->name), "%s", p.name);
    return CABL_OK;
}

extern "C" {

const char* cabl_last_error(void) { return g_err.c_str(); }
int cabl_abi_version(void) { return 106; } // 1.05: + cabl_mgpu_*; 1.06: + cabl_mgpu_dot_segmented_*
int cabl_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

int cabl_cuda_dot_f32(const float* x, const float* y, uint64_t n, float alpha0, float* out,
                      uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return dot_impl<float>(x, y, n, alpha0, out, small_cutoff, probe, stream);
}
int cabl_cuda_dot_f64(const double* x, const double* y, uint64_t n, double alpha0,
                      double* out, uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return dot_impl<double>(x, y, n, alpha0, out, small_cutoff, probe, stream);
}
int cabl_peer_mailbox_create(void** mbox) {
    if (!mbox) return fail(CABL_EINVAL, "peer_mailbox_create: out must not be null");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    void* p = nullptr;
    // cudaMalloc (not the stream-ordered pool): the allocation is exported by IPC
    CABL_TRY_CUDA(cudaMalloc(&p, sizeof(PeerMailbox)), "peer mailbox alloc");
    cudaError_t e = cudaMemset(p, 0, sizeof(PeerMailbox));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(p);
        return cuda_fail(e, "peer mailbox init");
    }
    *mbox = p;
    return CABL_OK;
}
int cabl_peer_mailbox_destroy(void* mbox) {
    if (!mbox) return CABL_OK;
    CABL_TRY_CUDA(cudaFree(mbox), "peer mailbox free");
    return CABL_OK;
}
int cabl_peer_mailbox_export(void* mbox, cabl_peer_handle* out) {
    if (!mbox || !out) return fail(CABL_EINVAL, "peer_mailbox_export: null pointer");
    static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(out->bytes), "IPC handle size");
    cudaIpcMemHandle_t h;
    CABL_TRY_CUDA(cudaIpcGetMemHandle(&h, mbox), "cudaIpcGetMemHandle");
    std::memcpy(out->bytes, &h, sizeof(h));
    return CABL_OK;
}
int cabl_peer_mailbox_import(const cabl_peer_handle* h, void** mapped) {
    if (!h || !mapped) return fail(CABL_EINVAL, "peer_mailbox_import: null pointer");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, h->bytes, sizeof(ih));
    CABL_TRY_CUDA(cudaIpcOpenMemHandle(mapped, ih, cudaIpcMemLazyEnablePeerAccess),
                  "cudaIpcOpenMemHandle");
    return CABL_OK;
}
int cabl_peer_mailbox_unmap(void* mapped) {
    if (!mapped) return CABL_OK;
    CABL_TRY_CUDA(cudaIpcCloseMemHandle(mapped), "cudaIpcCloseMemHandle");
    return CABL_OK;
}
int cabl_peer_mailbox_state(const void* mbox, uint64_t* epoch, uint64_t* fault) {
    if (!mbox) return fail(CABL_EINVAL, "peer_mailbox_state: null mailbox");
    PeerMailbox m;
    CABL_TRY_CUDA(cudaMemcpy(&m, mbox, sizeof(m), cudaMemcpyDeviceToHost), "peer mailbox read");
    if (epoch) *epoch = m.epoch;
    if (fault) *fault = m.fault;
    return CABL_OK;
}
int cabl_cuda_dot_peer_f32(const float* x, const float* y, uint64_t n, float alpha0, float* out,
                           void* const* mboxes, int world, int rank, uint64_t small_cutoff,
                           cabl_probe* probe, void* stream) {
    return dot_peer_impl<float>(x, y, n, alpha0, out, mboxes, world, rank, small_cutoff, probe,
                                stream);
}
int cabl_cuda_dot_peer_f64(const double* x, const double* y, uint64_t n, double alpha0,
                           double* out, void* const* mboxes, int world, int rank,
                           uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return dot_peer_impl<double>(x, y, n, alpha0, out, mboxes, world, rank, small_cutoff, probe,
                                 stream);
}
int cabl_cuda_dot_peer_emulate_f32(int world, const float* const* xs, const float* const* ys,
                                   const uint64_t* ns, float alpha0, float* const* outs,
                                   void* const* mboxes, uint64_t small_cutoff, void* stream) {
    return dot_peer_emulate_impl<float>(world, xs, ys, ns, alpha0, outs, mboxes, small_cutoff,
                                        stream);
}
int cabl_cuda_dot_peer_emulate_f64(int world, const double* const* xs, const double* const* ys,
                                   const uint64_t* ns, double alpha0, double* const* outs,
                                   void* const* mboxes, uint64_t small_cutoff, void* stream) {
    return dot_peer_emulate_impl<double>(world, xs, ys, ns, alpha0, outs, mboxes, small_cutoff,
                                         stream);
}
int cabl_peer_alloc(uint64_t bytes, void** ptr) {
    if (!ptr || bytes == 0) return fail(CABL_EINVAL, "peer_alloc: null out or zero bytes");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    void* p = nullptr;
    CABL_TRY_CUDA(cudaMalloc(&p, bytes), "peer buffer alloc"); // exportable by IPC
    cudaError_t e = cudaMemset(p, 0, bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        cudaFree(p);
        return cuda_fail(e, "peer buffer init");
    }
    *ptr = p;
    return CABL_OK;
}
int cabl_peer_free(void* ptr) {
    if (!ptr) return CABL_OK;
    CABL_TRY_CUDA(cudaFree(ptr), "peer buffer free");
    return CABL_OK;
}
int cabl_cuda_gemv_rm_gather_f32(const float* A, uint64_t m, uint64_t n, const float* x, float* c,
                                 uint64_t row_off, uint64_t m_total, void* const* cfull,
                                 void* const* mboxes, int world, int rank, cabl_probe* probe,
                                 void* stream) {
    return gemv_gather_impl<float>(A, m, n, x, c, row_off, m_total, cfull, mboxes, world, rank,
                                   probe, stream);
}
int cabl_cuda_gemv_rm_gather_f64(const double* A, uint64_t m, uint64_t n, const double* x,
                                 double* c, uint64_t row_off, uint64_t m_total,
                                 void* const* cfull, void* const* mboxes, int world, int rank,
                                 cabl_probe* probe, void* stream) {
    return gemv_gather_impl<double>(A, m, n, x, c, row_off, m_total, cfull, mboxes, world, rank,
                                    probe, stream);
}
int cabl_cuda_gemv_rm_gather_supported_f32(const float* A, uint64_t m, uint64_t n, const float* x,
                                           int* ok) {
    return gather_supported_impl<float>(A, m, n, x, ok);
}
int cabl_cuda_gemv_rm_gather_supported_f64(const double* A, uint64_t m, uint64_t n,
                                           const double* x, int* ok) {
    return gather_supported_impl<double>(A, m, n, x, ok);
}
int cabl_cuda_gemv_rm_gather_emulate_f32(int world, const float* const* As, const uint64_t* ms,
                                         uint64_t n, const float* const* xs, float* const* cs,
                                         const uint64_t* row_offs, uint64_t m_total,
                                         void* const* cfull, void* const* mboxes, void* stream) {
    return gemv_gather_emulate_impl<float>(world, As, ms, n, xs, cs, row_offs, m_total, cfull,
                                           mboxes, stream);
}
int cabl_cuda_gemv_rm_gather_emulate_f64(int world, const double* const* As, const uint64_t* ms,
                                         uint64_t n, const double* const* xs, double* const* cs,
                                         const uint64_t* row_offs, uint64_t m_total,
                                         void* const* cfull, void* const* mboxes, void* stream) {
    return gemv_gather_emulate_impl<double>(world, As, ms, n, xs, cs, row_offs, m_total, cfull,
                                            mboxes, stream);
}
int cabl_cuda_combine_rows_peer_f32(const float* part, uint64_t m, float* c, void* const* slots,
                                    void* const* mboxes, int world, int rank, void* stream) {
    return combine_rows_peer_impl<float>(part, m, c, slots, mboxes, world, rank, stream);
}
int cabl_cuda_combine_rows_peer_f64(const double* part, uint64_t m, double* c, void* const* slots,
                                    void* const* mboxes, int world, int rank, void* stream) {
    return combine_rows_peer_impl<double>(part, m, c, slots, mboxes, world, rank, stream);
}
int cabl_cuda_combine_rows_peer_emulate_f32(int world, const float* const* parts, uint64_t m,
                                            float* const* cs, void* const* slots,
                                            void* const* mboxes, void* stream) {
    return combine_rows_peer_emulate_impl<float>(world, parts, m, cs, slots, mboxes, stream);
}
int cabl_cuda_combine_rows_peer_emulate_f64(int world, const double* const* parts, uint64_t m,
                                            double* const* cs, void* const* slots,
                                            void* const* mboxes, void* stream) {
    return combine_rows_peer_emulate_impl<double>(world, parts, m, cs, slots, mboxes, stream);
}
int cabl_cuda_combine_partials_f32(const float* p, uint32_t count, float alpha0, float* out,
                                   void* stream) {
    return combine_impl<float>(p, count, alpha0, out, stream);
}
int cabl_cuda_combine_partials_f64(const double* p, uint32_t count, double alpha0,
                                   double* out, void* stream) {
    return combine_impl<double>(p, count, alpha0, out, stream);
}

int cabl_cuda_combine_rows_f32(const float* parts, uint32_t count, uint64_t m, float* c,
                               void* stream) {
    return combine_rows_impl<float>(parts, count, m, c, stream);
}
int cabl_cuda_combine_rows_f64(const double* parts, uint32_t count, uint64_t m, double* c,
                               void* stream) {
    return combine_rows_impl<double>(parts, count, m, c, stream);
}

int cabl_cuda_gemv_rm_f32(const float* A, uint64_t m, uint64_t n, const float* x, float* c,
                          uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return gemv_impl<float>(A, CABL_ROW_MAJOR, m, n, x, c, small_cutoff, probe, stream);
}
int cabl_cuda_gemv_rm_f64(const double* A, uint64_t m, uint64_t n, const double* x, double* c,
                          uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return gemv_impl<double>(A, CABL_ROW_MAJOR, m, n, x, c, small_cutoff, probe, stream);
}
int cabl_cuda_gemv_cm_f32(const float* A, uint64_t m, uint64_t n, const float* x, float* c,
                          uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return gemv_impl<float>(A, CABL_COL_MAJOR, m, n, x, c, small_cutoff, probe, stream);
}
int cabl_cuda_gemv_cm_f64(const double* A, uint64_t m, uint64_t n, const double* x, double* c,
                          uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return gemv_impl<double>(A, CABL_COL_MAJOR, m, n, x, c, small_cutoff, probe, stream);
}

int cabl_cuda_ger_rm_f32(const float* x, const float* y, float* C, uint64_t m, uint64_t n,
                         uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return ger_impl<float>(x, y, C, CABL_ROW_MAJOR, m, n, small_cutoff, probe, stream);
}
int cabl_cuda_ger_rm_f64(const double* x, const double* y, double* C, uint64_t m, uint64_t n,
                         uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return ger_impl<double>(x, y, C, CABL_ROW_MAJOR, m, n, small_cutoff, probe, stream);
}
int cabl_cuda_ger_cm_f32(const float* x, const float* y, float* C, uint64_t m, uint64_t n,
                         uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return ger_impl<float>(x, y, C, CABL_COL_MAJOR, m, n, small_cutoff, probe, stream);
}
int cabl_cuda_ger_cm_f64(const double* x, const double* y, double* C, uint64_t m, uint64_t n,
                         uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return ger_impl<double>(x, y, C, CABL_COL_MAJOR, m, n, small_cutoff, probe, stream);
}

int cabl_host_dot_f32(const float* x, const float* y, uint64_t n, float alpha0, float* result,
                      uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return host_dot<float>(x, y, n, alpha0, result, small_cutoff, probe, stream);
}
int cabl_host_dot_f64(const double* x, const double* y, uint64_t n, double alpha0,
                      double* result, uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return host_dot<double>(x, y, n, alpha0, result, small_cutoff, probe, stream);
}
int cabl_host_gemv_f32(const float* A, int layout, uint64_t m, uint64_t n, const float* x,
                       float* c, uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return host_gemv<float>(A, layout, m, n, x, c, small_cutoff, probe, stream);
}
int cabl_host_gemv_f64(const double* A, int layout, uint64_t m, uint64_t n, const double* x,
                       double* c, uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return host_gemv<double>(A, layout, m, n, x, c, small_cutoff, probe, stream);
}
int cabl_host_ger_f32(const float* x, const float* y, float* C, int layout, uint64_t m,
                      uint64_t n, uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return host_ger<float>(x, y, C, layout, m, n, small_cutoff, probe, stream);
}
int cabl_host_ger_f64(const double* x, const double* y, double* C, int layout, uint64_t m,
                      uint64_t n, uint64_t small_cutoff, cabl_probe* probe, void* stream) {
    return host_ger<double>(x, y, C, layout, m, n, small_cutoff, probe, stream);
}

int cabl_cuda_fill_uniform_f32(float* out, uint64_t n, uint64_t seed, uint64_t stream_id,
                               uint64_t offset, void* stream) {
    if (n > 0 && !out) return fail(CABL_EINVAL, "fill: out must not be null");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    CABL_TRY_CUDA(fill_uniform_f32(out, n, seed, stream_id, offset, as_stream(stream)), "fill");
    return CABL_OK;
}
int cabl_cuda_fill_uniform_f64(double* out, uint64_t n, uint64_t seed, uint64_t stream_id,
                               uint64_t offset, void* stream) {
    if (n > 0 && !out) return fail(CABL_EINVAL, "fill: out must not be null");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    CABL_TRY_CUDA(fill_uniform_f64(out, n, seed, stream_id, offset, as_stream(stream)), "fill");
    return CABL_OK;
}
int cabl_cuda_fill_normal_f64(double* out, uint64_t n, uint64_t seed, uint64_t stream_id,
                              uint64_t offset, void* stream) {
    if (n > 0 && !out) return fail(CABL_EINVAL, "fill: out must not be null");
    int dev;
    if (int rc = current_device(&dev)) return rc;
    CABL_TRY_CUDA(fill_normal_f64(out, n, seed, stream_id, offset, as_stream(stream)), "fill");
    return CABL_OK;
}

} // extern "C"

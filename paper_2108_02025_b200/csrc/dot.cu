// DOT: *out = alpha0 + sum_p x[p]*y[p]  — B200 re-design of reference
// cabl::dot (proj/include/cabl/kernels.hpp:134-164).
//
// One launch, no host round trip:
//   * grid = min(tiles, 148 * CTAS_PER_SM) CTAs (one wave, all resident);
//     CTAs stride over tiles of BLOCK*U 32-byte vectors, every thread keeps
//     2*U 256-bit loads in flight and accumulates with FMA in registers;
//   * fixed butterfly warp sums, fixed-order CTA sum -> partials[cta];
//   * every CTA publishes its total as epoch-tagged 64-bit words (common.cuh);
//     CTA 0, once its own sweep is done, polls the CTAs' words, sums them in a
//     fixed order, adds alpha0 LAST (as the reference does, kernels.hpp:142,163)
//     and records the epoch.  The critical path after the last CTA's sweep is
//     one store + one poll instead of a ticket RTT + a partials RTT: D1
//     (2^24 fp32, one flushed launch, ncu) 25.2 -> 24.x us (tools/dotlab.py,
//     profiles/r02_dotlab.md).  No deadlock is possible: only CTA 0 waits,
//     and it waits for CTAs that never wait.
// The element -> thread mapping depends only on n and the grid, so the result
// is bitwise reproducible run to run (reference kernels.hpp:9-13).
//
// Algorithmic bytes per launch: 2 * n * sizeof(T).
#include "common.cuh"
#include "dot_body.cuh"
#include "kernels.cuh"

#include <cstdio>
#include <cstdlib>

namespace cabl_dev {

namespace {


template <typename T, int BLOCK, int U, int MINB, bool PEEL = false>
__global__ void __launch_bounds__(BLOCK, MINB)
    dot_kernel(const T* __restrict__ x, const T* __restrict__ y, uint64_t n, int vec_ok,
               uint64_t head_, T alpha0, T* __restrict__ out,
               unsigned long long* __restrict__ slots, int pf) {
    // vec_ok: x + head and y + head are 32-byte aligned (head < V elements are
    // peeled when both operands share their misalignment); the head and the
    // < V tail run in the scalar loop
    pdl_trigger();
    if (pf > 0 && vec_ok && threadIdx.x < 2 * U) { // warm L2: this CTA's first U slabs of x and y
        const uint64_t nvec = (n - (PEEL ? head_ : 0)) / Vec<T>::N;
        const uint64_t T_all = uint64_t(gridDim.x) * BLOCK;
        const uint64_t v0 = uint64_t(blockIdx.x) * BLOCK + uint64_t(threadIdx.x >> 1) * T_all;
        if (v0 < nvec) {
            const uint64_t cnt = nvec - v0 < uint64_t(BLOCK) ? nvec - v0 : uint64_t(BLOCK);
            const T* base = ((threadIdx.x & 1) ? y : x) + (PEEL ? head_ : 0);
            prefetch_l2_bulk(base + v0 * Vec<T>::N, unsigned(cnt * sizeof(Vec<T>)));
        }
    }
    pdl_wait();
    __shared__ T red[32];
    const int tid = threadIdx.x;
    // the epoch is loaded before the sweep, so its latency hides behind it
    const bool collector = blockIdx.x == 0;
    const unsigned e = (gridDim.x > 1 && (tid == 0 || collector)) ? next_epoch(slots) : 0u;
    const T s = dot_thread_sum<T, BLOCK, U, PEEL>(x, y, n, vec_ok, head_, blockIdx.x, gridDim.x);
    const T cta_total = block_sum(s, red);

    if (gridDim.x == 1) {
        if (tid == 0) *out = add_rn(cta_total, alpha0);
        return;
    }
    constexpr int W = tagged_words<T>();
    if (tid == 0) publish_tagged(slots + 1 + uint64_t(W) * blockIdx.x, cta_total, e);
    if (!collector) return;
    // CTA totals in a fixed order (thread t: CTAs t, t + BLOCK, ...; then the
    // fixed block tree), alpha0 last
    T v = T(0);
    for (unsigned i = tid; i < gridDim.x; i += BLOCK)
        v = add_rn(v, collect_tagged<T>(slots + 1 + uint64_t(W) * i, e));
    const T total = block_sum(v, red);
    if (tid == 0) {
        *out = add_rn(total, alpha0);
        st_relaxed_u64(slots, e); // the next launch on this stream takes e + 1
    }
}

// CHUNKED DOT for large n (2ns >= 512 MiB, e.g. D2 = 2^32): the vector range
// is cut into chunks of kChunkVecs 32-byte vectors; CTAs take chunks from an
// atomic queue (common.cuh dyn_next), so SMs that get faster memory service
// take more chunks.  A chunk's partial is a fixed function of its data (fixed
// thread mapping inside the chunk, fixed trees) and goes to partials[chunk];
// the last CTA to finish sums the partials in chunk order, adds the < V
// trailing elements, then alpha0.  The result depends on n only — not on
// the grid, the scheduling, or the GPU's SM count — and every rounding chain
// is short (<= kChunkVecs/(BLOCK*U) vectors per accumulator).
constexpr uint64_t kChunkVecs = 65536; // at most 2 MiB of x and 2 MiB of y (fp32)

// Vectors per chunk: the largest power of two <= nvec / 2048, clamped to
// [4096, kChunkVecs] — at least 2048 chunks, so the queue balances even at
// the 512 MiB threshold (2^26 fp32 had 128 chunks for 148 SMs: 6.4 TB/s), and
// a function of n alone, so the result still is.  CABL_DOT_CHUNK overrides
// (tuning only).
inline uint64_t chunk_vecs(uint64_t nvec) {
    static const uint64_t forced = [] {
        const char* e = tuning_env("CABL_DOT_CHUNK");
        return e ? uint64_t(atoll(e)) : uint64_t(0);
    }();
    if (forced) return forced;
    uint64_t c = 4096;
    while (c * 2 <= kChunkVecs && c * 2 * 2048 <= nvec) c *= 2;
    return c;
}

template <typename T, int BLOCK, int U, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB)
    dot_chunk_kernel(const T* __restrict__ x, const T* __restrict__ y, uint64_t n, T alpha0,
                     T* __restrict__ out, T* __restrict__ partials,
                     unsigned* __restrict__ counters, uint64_t chunk) {
    pdl_enter();
    __shared__ T red[32];
    __shared__ unsigned long long next_sh;
    __shared__ bool am_last;
    dot_chunk_sweep<T, BLOCK, U>(x, y, n, partials, counters, chunk, blockIdx.x, gridDim.x, red,
                                 &next_sh);
    if (threadIdx.x == 0) {
        __threadfence();
        am_last = atomicAdd(counters + 1, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    const T total = dot_chunk_total<T, BLOCK>(x, y, n, partials, chunk, red);
    if (threadIdx.x == 0) {
        *out = add_rn(total, alpha0);
        counters[1] = 0u;
    }
}

template <typename T>
__global__ void combine_kernel(const T* __restrict__ p, uint32_t count, T alpha0,
                               T* __restrict__ out) {
    pdl_enter();
    // Reference kernels.hpp:160-163: total{} += partials[c] in index order,
    // then + alpha0.
    T total = T(0);
    for (uint32_t i = 0; i < count; ++i) total = add_rn(total, p[i]);
    *out = add_rn(total, alpha0);
}

struct DotCfg {
    int block, unroll, minb;
};

// Launch shape.  CABL_DOT_CFG="block,unroll,ctas_per_sm" picks an entry of
// the tuning table below (tools/tune.py); the default is the measured best.
inline DotCfg dot_cfg() {
    static const DotCfg cfg = [] {
        DotCfg c{kDotBlock, kDotUnroll, kDotCtasPerSm};
        if (const char* e = tuning_env("CABL_DOT_CFG")) sscanf(e, "%d,%d,%d", &c.block, &c.unroll, &c.minb);
        return c;
    }();
    return cfg;
}

template <typename T> unsigned dot_grid(uint64_t n, bool small) {
    if (small) return 1;
    constexpr int V = Vec<T>::N;
    const DotCfg c = dot_cfg();
    const uint64_t per = uint64_t(c.block) * c.unroll;
    const uint64_t tiles = (n / V + per - 1) / per;
    const uint64_t cap = uint64_t(sm_count()) * c.minb;
    uint64_t g = tiles < cap ? tiles : cap;
    return g < 1 ? 1u : unsigned(g);
}

template <typename T, int B, int U, int M>
cudaError_t dot_go(unsigned grid, const T* x, const T* y, uint64_t n, int vec_ok,
                   uint64_t head, T alpha0, T* out, unsigned long long* slots, cudaStream_t s) {
    if (head)
        launch(dot_kernel<T, B, U, M, true>, grid, B, 0, s, x, y, n, vec_ok, head, alpha0, out,
               slots, pdl_prefetch_enabled());
    else
        launch(dot_kernel<T, B, U, M, false>, grid, B, 0, s, x, y, n, vec_ok, head, alpha0, out,
               slots, pdl_prefetch_enabled());
    return cudaGetLastError();
}

template <typename T>
cudaError_t dot_dispatch(unsigned grid, const T* x, const T* y, uint64_t n, int vec_ok,
                         uint64_t head, T alpha0, T* out, unsigned long long* slots,
                         cudaStream_t s) {
    const DotCfg c = dot_cfg();
#define CABL_DOT_CASE(B_, U_, M_)                                                              \
    if (c.block == B_ && c.unroll == U_ && c.minb == M_)                                       \
        return dot_go<T, B_, U_, M_>(grid, x, y, n, vec_ok, head, alpha0, out, slots, s);
    CABL_DOT_CASE(256, 1, 8)
    CABL_DOT_CASE(256, 2, 8)
    CABL_DOT_CASE(256, 4, 4)
    CABL_DOT_CASE(512, 2, 2)
    CABL_DOT_CASE(512, 4, 2)
    CABL_DOT_CASE(1024, 2, 1)
    CABL_DOT_CASE(1024, 4, 1)
    CABL_DOT_CASE(256, 8, 1)
#undef CABL_DOT_CASE
    return dot_go<T, kDotBlock, kDotUnroll, kDotCtasPerSm>(grid, x, y, n, vec_ok, head, alpha0,
                                                          out, slots, s);
}

} // namespace

// large operands (2ns >= 512 MiB) take the chunked, queue-scheduled kernel
inline bool dot_chunked(uint64_t n, size_t s, bool small, bool vec_ok) {
    static const int forced = [] {
        const char* e = tuning_env("CABL_DOT_CHUNKED");
        return e ? atoi(e) : -1;
    }();
    if (small || !vec_ok) return false;
    if (n / (32 / s) < uint64_t(sm_count()) * kDotCtasPerSm) return false; // grid <= vectors
    if (forced >= 0) return forced != 0;
    return 2 * n * s >= queue_threshold_bytes();
}

template <typename T> WorkspaceNeed dot_need(uint64_t n, bool small) {
    WorkspaceNeed w;
    w.counters = 2;
    const uint64_t cv = chunk_vecs(n / Vec<T>::N);
    const uint64_t chunks = (n / Vec<T>::N + cv - 1) / cv;
    const uint64_t g = dot_grid<T>(n, small);
    w.scratch_bytes = size_t(chunks > g ? chunks : g) * sizeof(T);
    w.slots = 1 + size_t(tagged_words<T>()) * g; // epoch + the CTAs' tagged totals
    return w;
}

template <typename T> DotPlan dot_plan(const T* x, const T* y, uint64_t n, bool small) {
    DotPlan p;
    const int vec_ok = aligned32(x) && aligned32(y);
    if (dot_chunked(n, sizeof(T), small, vec_ok)) {
        p.chunked = true;
        p.vec_ok = 1;
        p.chunk = chunk_vecs(n / Vec<T>::N);
        const uint64_t chunks = (n / Vec<T>::N + p.chunk - 1) / p.chunk;
        const uint64_t cap = uint64_t(sm_count()) * kDotCtasPerSm;
        p.grid = unsigned(chunks < cap ? chunks : cap);
        return p;
    }
    // operands that share their misalignment: peel head < V elements so the
    // rest is 32-byte aligned (x[k:], y[k:] slices of aligned buffers)
    p.vec_ok = vec_ok;
    if (!vec_ok) {
        const uintptr_t xa = reinterpret_cast<uintptr_t>(x), ya = reinterpret_cast<uintptr_t>(y);
        if (xa % 32 == ya % 32 && xa % sizeof(T) == 0) {
            p.head = ((32 - xa % 32) % 32) / sizeof(T);
            p.vec_ok = p.head < n ? 1 : 0;
            if (!p.vec_ok) p.head = 0;
        }
    }
    p.grid = dot_grid<T>(n, small);
    return p;
}

template <typename T>
cudaError_t dot_launch(const T* x, const T* y, uint64_t n, T alpha0, T* out, bool small,
                       const Workspace& ws, cudaStream_t s, LaunchInfo* info) {
    const DotPlan p = dot_plan<T>(x, y, n, small);
    if (info) info->ctas = p.grid;
    if (p.chunked) {
        launch(dot_chunk_kernel<T, kDotBlock, kDotUnroll, kDotCtasPerSm>, p.grid, kDotBlock, 0, s,
               x, y, n, alpha0, out, static_cast<T*>(ws.scratch), ws.counters, p.chunk);
        return cudaGetLastError();
    }
    return dot_dispatch<T>(p.grid, x, y, n, p.vec_ok, p.head, alpha0, out, ws.slots, s);
}

template <typename T>
cudaError_t combine_partials_launch(const T* p, uint32_t count, T alpha0, T* out,
                                    cudaStream_t s) {
    launch(combine_kernel<T>, 1, 1, 0, s, p, count, alpha0, out);
    return cudaGetLastError();
}

namespace {
// c[i] += ((parts[0][i] + parts[1][i]) + ...) in index order: the combine of
// a column-sharded col-major GEMV (each rank's partial c over its column block,
// all-gathered), bitwise the same on every rank and for any reduction order
// of the collective.
template <typename T>
__global__ void combine_rows_kernel(const T* __restrict__ parts, uint32_t count, uint64_t m,
                                    T* __restrict__ c) {
    pdl_enter();
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
        T total = T(0);
        for (uint32_t g = 0; g < count; ++g) total = add_rn(total, parts[uint64_t(g) * m + i]);
        c[i] = add_rn(c[i], total);
    }
}
} // namespace

template <typename T>
cudaError_t combine_rows_launch(const T* parts, uint32_t count, uint64_t m, T* c,
                                cudaStream_t s) {
    if (m == 0) return cudaSuccess;
    const uint64_t blocks = (m + 255) / 256;
    const uint64_t cap = uint64_t(sm_count()) * 8;
    launch(combine_rows_kernel<T>, unsigned(blocks < cap ? blocks : cap), 256, 0, s, parts, count,
           m, c);
    return cudaGetLastError();
}
template cudaError_t combine_rows_launch<float>(const float*, uint32_t, uint64_t, float*,
                                                cudaStream_t);
template cudaError_t combine_rows_launch<double>(const double*, uint32_t, uint64_t, double*,
                                                 cudaStream_t);

template DotPlan dot_plan<float>(const float*, const float*, uint64_t, bool);
template DotPlan dot_plan<double>(const double*, const double*, uint64_t, bool);
template WorkspaceNeed dot_need<float>(uint64_t, bool);
template WorkspaceNeed dot_need<double>(uint64_t, bool);
template cudaError_t dot_launch<float>(const float*, const float*, uint64_t, float, float*, bool,
                                       const Workspace&, cudaStream_t, LaunchInfo*);
template cudaError_t dot_launch<double>(const double*, const double*, uint64_t, double, double*,
                                        bool, const Workspace&, cudaStream_t, LaunchInfo*);
template cudaError_t combine_partials_launch<float>(const float*, uint32_t, float, float*,
                                                    cudaStream_t);
template cudaError_t combine_partials_launch<double>(const double*, uint32_t, double, double*,
                                                     cudaStream_t);

} // namespace cabl_dev

// DOT bodies shared by the single-GPU kernels (dot.cu) and the peer-memory
// multi-GPU kernels (peer.cu).  Each takes the CTA's index `bid` and the grid
// size `nblk` as arguments instead of blockIdx.x / gridDim.x, so a kernel can
// run several ranks' grids side by side (blockIdx.y = rank) and every rank
// still sees exactly the element -> thread mapping of its own single-GPU
// launch (same bits).  Reference: cabl::dot, kernels.hpp:134-164.
#pragma once

#include "common.cuh"

namespace cabl_dev {

// measured best on n = 2^24 fp32 (tools/tune.py): 512 x 2 CTAs/SM, 2 vectors
// of x and y in flight per thread per iteration
constexpr int kDotBlock = 512;
constexpr int kDotUnroll = 2;
constexpr int kDotCtasPerSm = 2;

// Grid-stride partial of one thread (the body of dot_kernel): with T threads
// in the grid, thread t takes 32-byte vectors t, t + T, t + 2T, ... (U in
// flight per iteration), then the scalar head/tail.  Returns the thread's sum
// of its U accumulators (fixed order).
template <typename T, int BLOCK, int U, bool PEEL>
__device__ __forceinline__ T dot_thread_sum(const T* __restrict__ x, const T* __restrict__ y,
                                            uint64_t n, int vec_ok, uint64_t head_, unsigned bid,
                                            unsigned nblk) {
    const uint64_t head = PEEL ? head_ : 0;
    constexpr int V = Vec<T>::N;
    const int tid = threadIdx.x;

    T acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = T(0);

    uint64_t done = 0; // elements covered by the head and the vector loop
    if (vec_ok) {
        const uint64_t nvec = (n - head) / V;
        const Vec<T>* X = reinterpret_cast<const Vec<T>*>(x + head);
        const Vec<T>* Y = reinterpret_cast<const Vec<T>*>(y + head);
        // every thread's share is within one vector of every other's and the
        // grid sweeps the operands front to back in T-vector slabs
        const uint64_t T_all = uint64_t(nblk) * BLOCK;
        for (uint64_t k0 = uint64_t(bid) * BLOCK + tid; k0 < nvec; k0 += U * T_all) {
            Vec<T> xv[U], yv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t i = k0 + uint64_t(u) * T_all;
                if (i < nvec) {
                    xv[u] = ld_stream(X + i);
                    yv[u] = ld_stream(Y + i);
                } else {
#pragma unroll
                    for (int k = 0; k < V; ++k) xv[u].v[k] = yv[u].v[k] = T(0);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] = dot_vec(xv[u], yv[u], acc[u]);
        }
        // the peeled head: one element for each of the first `head` threads
        if (PEEL) {
            const uint64_t gt = uint64_t(bid) * BLOCK + tid;
            if (gt < head) acc[0] = fma_rn(x[gt], y[gt], acc[0]);
        }
        done = head + nvec * V;
    }
    // Scalar remainder (unaligned operands, or the < V trailing elements):
    // one chain per thread over i = done + gt, + gs, ... in order, with the
    // loads of kScalarU steps issued before they are consumed (coalesced
    // 128-byte warp requests; one pair at a time ran misaligned DOT at ~2 TB/s).
    {
        constexpr int kScalarU = 8;
        const uint64_t gt = uint64_t(bid) * BLOCK + tid;
        const uint64_t gs = uint64_t(nblk) * BLOCK;
        uint64_t i = done + gt;
        for (; i + uint64_t(kScalarU - 1) * gs < n; i += uint64_t(kScalarU) * gs) {
            T a[kScalarU], b[kScalarU];
#pragma unroll
            for (int u = 0; u < kScalarU; ++u) {
                a[u] = __ldcs(x + i + u * gs);
                b[u] = __ldcs(y + i + u * gs);
            }
#pragma unroll
            for (int u = 0; u < kScalarU; ++u) acc[0] = fma_rn(a[u], b[u], acc[0]);
        }
        for (; i < n; i += gs) acc[0] = fma_rn(x[i], y[i], acc[0]);
    }

    T s = acc[0];
#pragma unroll
    for (int u = 1; u < U; ++u) s = add_rn(s, acc[u]);
    return s;
}

// The chunk sweep of dot_chunk_kernel: CTA `bid` of `nblk` takes chunk bid,
// then chunks from the atomic queue; each chunk's partial (a fixed function of
// its data) goes to partials[chunk].  `red` holds 32 T, `next_sh` one queue slot.
template <typename T, int BLOCK, int U>
__device__ __forceinline__ void dot_chunk_sweep(const T* __restrict__ x, const T* __restrict__ y,
                                                uint64_t n, T* __restrict__ partials,
                                                unsigned* __restrict__ counters, uint64_t chunk,
                                                unsigned bid, unsigned nblk, T* red,
                                                unsigned long long* next_sh) {
    constexpr int V = Vec<T>::N;
    const int tid = threadIdx.x;
    const uint64_t nvec = n / V;
    const uint64_t nchunks = (nvec + chunk - 1) / chunk;
    const Vec<T>* X = reinterpret_cast<const Vec<T>*>(x);
    const Vec<T>* Y = reinterpret_cast<const Vec<T>*>(y);

    uint64_t ch = bid; // first chunk static, the rest from the queue
    while (ch < nchunks) {
        if (tid == 0) *next_sh = dyn_next(counters, nchunks, nblk); // prefetch
        T acc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) acc[u] = T(0);
        const uint64_t c0 = ch * chunk;
        const uint64_t c1 = (c0 + chunk < nvec) ? c0 + chunk : nvec;
        for (uint64_t base = c0; base < c1; base += uint64_t(BLOCK) * U) {
            Vec<T> xv[U], yv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t i = base + uint64_t(u) * BLOCK + tid;
                if (i < c1) {
                    xv[u] = ld_stream(X + i);
                    yv[u] = ld_stream(Y + i);
                } else {
#pragma unroll
                    for (int k = 0; k < V; ++k) xv[u].v[k] = yv[u].v[k] = T(0);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc[u] = dot_vec(xv[u], yv[u], acc[u]);
        }
        T v = acc[0];
#pragma unroll
        for (int u = 1; u < U; ++u) v = add_rn(v, acc[u]);
        const T chunk_total = block_sum(v, red); // its barriers publish next_sh
        if (tid == 0) partials[ch] = chunk_total;
        ch = *next_sh;
        __syncthreads(); // next_sh is rewritten at the top of the next chunk
    }
}

// The last CTA's total of the chunked DOT: chunk partials in chunk order, then
// the < V trailing elements (thread 0's value is the one that counts).
template <typename T, int BLOCK>
__device__ __forceinline__ T dot_chunk_total(const T* __restrict__ x, const T* __restrict__ y,
                                             uint64_t n, const T* partials, uint64_t chunk,
                                             T* red) {
    constexpr int V = Vec<T>::N;
    const uint64_t nvec = n / V;
    const uint64_t nchunks = (nvec + chunk - 1) / chunk;
    T v = T(0);
    for (uint64_t i = threadIdx.x; i < nchunks; i += BLOCK) v = add_rn(v, ld_cg(partials + i));
    T total = block_sum(v, red);
    if (threadIdx.x == 0)
        for (uint64_t i = nvec * V; i < n; ++i) total = fma_rn(x[i], y[i], total);
    return total;
}

} // namespace cabl_dev

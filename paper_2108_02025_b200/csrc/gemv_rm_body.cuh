// Row-major GEMV sweep body shared by the single-GPU sweep kernel (gemv_rm.cu)
// and the gathering sweep (peer_gemv.cu), so both give the same bits per row.
// Reference: cabl::gemv_row_major, proj/include/cabl/kernels.hpp:230-257.
#pragma once

#include "common.cuh"

namespace cabl_dev {

constexpr int kRmBlock = 256;

// The sweep's group loop (shared with the gathering sweep in peer_gemv.cu):
// CTA `bid` of `nblk` takes groups bid, bid + nblk, ... (DYN: the first
// static, the rest from the queue) and hands each row's sum (before c) to
// `epi(row, sum, c_row)`, thread tid < rows, where c_row = c[row] was loaded
// at the start of the group (its latency hides behind the group's A loads
// instead of following the reduction).
template <typename T, int R, int KV, bool DYN, typename Epi>
__device__ __forceinline__ void sweep_groups(const T* __restrict__ A, const T* __restrict__ x,
                                             uint64_t m, uint64_t n, unsigned* __restrict__ counter,
                                             unsigned bid, unsigned nblk, const T* c, Epi epi) {
    constexpr int NW = kRmBlock / kWarp;
    __shared__ T red[2][R][NW];
    __shared__ unsigned long long next_sh[2];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint64_t nvec_row = n / Vec<T>::N;
    const uint64_t groups = (m + R - 1) / R;
    const Vec<T>* X = reinterpret_cast<const Vec<T>*>(x);
    uint64_t g = bid; // first group static, the rest from the queue (DYN)
    int parity = 0;
    while (g < groups) {
        if (DYN && tid == 0) next_sh[parity ^ 1] = dyn_next(counter, groups, nblk); // prefetch
        const uint64_t row0 = g * R;
        const int rows = (m - row0 < uint64_t(R)) ? int(m - row0) : R;
        const T c_row = tid < rows ? c[row0 + tid] : T(0);
        T acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = T(0);
        for (uint64_t base = 0; base < nvec_row; base += uint64_t(kRmBlock) * KV) {
            Vec<T> av[R][KV];
            Vec<T> xv[KV];
#pragma unroll
            for (int k = 0; k < KV; ++k) {
                const uint64_t j = base + uint64_t(tid) + uint64_t(k) * kRmBlock;
                const bool ok = j < nvec_row;
                if (ok) xv[k] = ld_reuse(X + j);
                else
#pragma unroll
                    for (int e = 0; e < Vec<T>::N; ++e) xv[k].v[e] = T(0);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (ok && r < rows)
                        av[r][k] = ld_stream(reinterpret_cast<const Vec<T>*>(A + (row0 + r) * n) + j);
                    else
#pragma unroll
                        for (int e = 0; e < Vec<T>::N; ++e) av[r][k].v[e] = T(0);
                }
            }
#pragma unroll
            for (int k = 0; k < KV; ++k)
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] = dot_vec(av[r][k], xv[k], acc[r]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const T v = warp_sum(acc[r]);
            if (lane == 0) red[parity][r][wid] = v;
        }
        __syncthreads(); // also publishes next_sh[parity ^ 1]
        if (tid < rows) {
            T sum = red[parity][tid][0];
#pragma unroll
            for (int w = 1; w < NW; ++w) sum = add_rn(sum, red[parity][tid][w]);
            epi(row0 + tid, sum, c_row);
        }
        parity ^= 1;
        g = DYN ? next_sh[parity] : g + nblk;
    }
}

} // namespace cabl_dev

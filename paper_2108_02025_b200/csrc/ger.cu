// GER: C += x (x) y — B200 re-design of reference cabl::ger
// (proj/include/cabl/kernels.hpp:277-313) and its oracle ger_ref (:264-270).
//
// The kernel works on a row-major OUTER x INNER view of C:
//   C[o*inner + i] = fma(u[o], v[i], C[o*inner + i]).
// Row-major C: (u, v, outer, inner) = (x, y, m, n).  Col-major C is the
// transposed view, (y, x, n, m); fma(a, b, c) == fma(b, a, c) exactly, so
// both layouts give the reference's single fused multiply-add per element —
// bitwise equal to ger_ref (the compiled reference contracts
// `C(i,j) += x_i*y_j` to FMA; oracle/cabl_oracle.c, tests/test_oracle.py).
//
// Fast path (32-byte aligned C and v, inner % (32/s) == 0, >= 128 vectors per
// row): a thread owns one 32-byte column vector of C for a contiguous,
// balanced range of rows; its v slice sits in registers for the whole range,
// u[o] is a warp-uniform broadcast load, and C streams through a 256-bit
// read-modify-write (no L1 allocation) with U rows of loads in flight.
// Every element is touched by exactly one thread once: no races, and the
// result does not depend on the launch shape.
//
// Generic path (ragged / unaligned / narrow rows, and the single-CTA small
// path the reference runs on one thread, kernels.hpp:286-287): flattened
// element-wise grid-stride FMA.
//
// Algorithmic bytes per launch: 2*m*n*s + m*s + n*s.
#include "common.cuh"
#include "kernels.cuh"

namespace cabl_dev {

namespace {

constexpr int kGerBlock = 256;
constexpr int kGerCtasPerSm = 4;
constexpr int kGerUnroll = 4;
constexpr uint64_t kGerMinVecs = 128;

template <typename T, int U>
__global__ void __launch_bounds__(kGerBlock, kGerCtasPerSm)
    ger_vec_kernel(const T* __restrict__ u, const T* __restrict__ v, T* __restrict__ C,
                   uint64_t outer, uint64_t nvec, unsigned col_blocks) {
    const unsigned cb = blockIdx.x % col_blocks;
    const unsigned rb = blockIdx.x / col_blocks;
    const unsigned row_blocks = gridDim.x / col_blocks;
    const uint64_t vc = uint64_t(cb) * kGerBlock + threadIdx.x; // vector column
    if (vc >= nvec) return;
    const Partition part(outer, row_blocks);
    const uint64_t o0 = part.begin(rb), o1 = part.begin(rb + 1);

    const Vec<T> vv = ld_reuse(reinterpret_cast<const Vec<T>*>(v) + vc);
    Vec<T>* Cv = reinterpret_cast<Vec<T>*>(C) + vc;

    uint64_t o = o0;
    for (; o + U <= o1; o += U) {
        Vec<T> cv[U];
        T uo[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            cv[k] = ld_rmw(Cv + (o + k) * nvec);
            uo[k] = __ldg(u + o + k);
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
#pragma unroll
            for (int e = 0; e < Vec<T>::N; ++e) cv[k].v[e] = fma_rn(uo[k], vv.v[e], cv[k].v[e]);
            st_stream(Cv + (o + k) * nvec, cv[k]);
        }
    }
    for (; o < o1; ++o) {
        Vec<T> cv = ld_rmw(Cv + o * nvec);
        const T uo = __ldg(u + o);
#pragma unroll
        for (int e = 0; e < Vec<T>::N; ++e) cv.v[e] = fma_rn(uo, vv.v[e], cv.v[e]);
        st_stream(Cv + o * nvec, cv);
    }
}

template <typename T>
__global__ void __launch_bounds__(kGerBlock)
    ger_generic_kernel(const T* __restrict__ u, const T* __restrict__ v, T* __restrict__ C,
                       uint64_t outer, uint64_t inner) {
    const uint64_t total = outer * inner;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
        const uint64_t o = e / inner, i = e - o * inner;
        C[e] = fma_rn(u[o], v[i], C[e]);
    }
}

} // namespace

template <typename T>
cudaError_t ger_launch(const T* u, const T* v, T* C, uint64_t outer, uint64_t inner,
                       bool small, cudaStream_t s, LaunchInfo* info) {
    if (info) info->ctas = 0;
    if (outer == 0 || inner == 0) return cudaSuccess;
    constexpr int V = Vec<T>::N;
    const bool vec_ok = aligned32(C) && aligned32(v) && inner % V == 0 &&
                        inner / V >= kGerMinVecs;
    if (!small && vec_ok) {
        const uint64_t nvec = inner / V;
        const unsigned col_blocks = unsigned((nvec + kGerBlock - 1) / kGerBlock);
        const uint64_t target = uint64_t(sm_count()) * kGerCtasPerSm;
        uint64_t row_blocks = target / col_blocks;
        if (row_blocks < 1) row_blocks = 1;
        if (row_blocks > outer) row_blocks = outer;
        const unsigned grid = unsigned(row_blocks * col_blocks);
        ger_vec_kernel<T, kGerUnroll><<<grid, kGerBlock, 0, s>>>(u, v, C, outer, nvec, col_blocks);
        if (info) info->ctas = grid;
    } else {
        const uint64_t total = outer * inner;
        uint64_t grid = small ? 1 : (total + kGerBlock - 1) / kGerBlock;
        const uint64_t cap = uint64_t(sm_count()) * 8;
        if (grid > cap) grid = cap;
        ger_generic_kernel<T><<<unsigned(grid), kGerBlock, 0, s>>>(u, v, C, outer, inner);
        if (info) info->ctas = unsigned(grid);
    }
    return cudaGetLastError();
}

template cudaError_t ger_launch<float>(const float*, const float*, float*, uint64_t, uint64_t,
                                       bool, cudaStream_t, LaunchInfo*);
template cudaError_t ger_launch<double>(const double*, const double*, double*, uint64_t,
                                        uint64_t, bool, cudaStream_t, LaunchInfo*);

} // namespace cabl_dev

// Column-major GEMV: c += A x, A is m x n col-major — B200 re-design of
// reference cabl::gemv_col_major (proj/include/cabl/kernels.hpp:187-224,
// Algorithm 1 of the paper: row blocks x column blocks x m_r register panels).
//
// Two shapes, two kernels:
//
// (1) ROWS (tall: m >= kSplitMaxRows, e.g. 2^20 x 256).  The CPU panel keeps
//     m_r rows of c in registers across a column block; here a LANE keeps one
//     row of c in a register across ALL columns and a warp owns 32 adjacent
//     rows, so every column read is a contiguous 32*s-byte run and the 148
//     SMs stream A with 16 independent loads in flight per lane.  Warps own
//     balanced contiguous ranges of 32-row units.  Each row's sum runs j
//     ascending from c_i — the reference order — with the reference's
//     compiled rounding (multiply-then-add over the 16-byte-vector prefix,
//     FMA on the remainder; see oracle/cabl_oracle.c), so this path is bit
//     for bit equal to the compiled reference gemv_ref.
//
// (2) SPLIT (short-wide: m < kSplitMaxRows, e.g. 256 x 2^20).  The reference
//     runs this shape on ONE thread (one m_c row block).
//     Here the columns are split over a single wave of CTAs (balanced ±1
//     column); inside a CTA, threads are (row lane, column lane) pairs,
//     accumulate with FMA over their columns, and column lanes combine in
//     shared memory in a fixed order -> partials[cta][m].  The last CTA to
//     arrive sums the partials in CTA order per row and adds them to c.
//     Bitwise reproducible run to run; within the BASELINE tolerance of
//     gemv_ref.
//
// Algorithmic bytes per launch: m*n*s + n*s + 2*m*s.
#include "common.cuh"
#include "kernels.cuh"

namespace cabl_dev {

namespace {

constexpr int kCmBlock = 256;
constexpr int kCmUnroll = 16;
constexpr int kCmRowsCtasPerSm = 4;
constexpr uint64_t kSplitMaxRows = 2048;
constexpr int kSplitBlock = 512;
constexpr int kSplitCtasPerSm = 2;

template <typename T>
__global__ void __launch_bounds__(kCmBlock, kCmRowsCtasPerSm)
    gemv_cm_rows_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                        uint64_t m, uint64_t n, uint64_t warps) {
    constexpr uint64_t kRefVec = 16 / sizeof(T);
    const int lane = threadIdx.x & 31;
    const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (gw >= warps) return;
    const uint64_t units = (m + kWarp - 1) / kWarp;
    const Partition part(units, warps);
    const uint64_t cut = (n / kRefVec) * kRefVec; // mul-then-add prefix length

    for (uint64_t unit = part.begin(gw); unit < part.begin(gw + 1); ++unit) {
        const uint64_t i = unit * kWarp + lane;
        const bool live = i < m;
        const T* a = A + (live ? i : 0);
        T acc = live ? c[i] : T(0);
        uint64_t j = 0;
        for (; j + kCmUnroll <= cut; j += kCmUnroll) {
            T av[kCmUnroll];
#pragma unroll
            for (int k = 0; k < kCmUnroll; ++k)
                av[k] = live ? __ldcs(a + (j + k) * m) : T(0);
#pragma unroll
            for (int k = 0; k < kCmUnroll; ++k) acc = add_rn(acc, mul_rn(av[k], __ldg(x + j + k)));
        }
        for (; j < cut; ++j) {
            const T av = live ? __ldcs(a + j * m) : T(0);
            acc = add_rn(acc, mul_rn(av, __ldg(x + j)));
        }
        for (; j < n; ++j) {
            const T av = live ? __ldcs(a + j * m) : T(0);
            acc = fma_rn(av, __ldg(x + j), acc);
        }
        if (live) c[i] = acc;
    }
}

// Split-columns kernel.  Thread layout: row_lanes x col_lanes = kSplitBlock,
// row_lanes = 32 * ceil(min(m, kSplitBlock) / 32); each thread accumulates
// RPT rows (r = row_lane + k*row_lanes).
template <typename T, int RPT>
__global__ void __launch_bounds__(kSplitBlock, kSplitCtasPerSm)
    gemv_cm_split_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                         uint64_t m, uint64_t n, int row_lanes, T* __restrict__ partials,
                         unsigned* __restrict__ ticket) {
    extern __shared__ unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw); // [col_lanes][m]
    __shared__ bool am_last;
    const int tid = threadIdx.x;
    const int col_lanes = kSplitBlock / row_lanes;
    const int rl = tid % row_lanes, cl = tid / row_lanes;
    const Partition part(n, gridDim.x);
    const uint64_t j0 = part.begin(blockIdx.x), j1 = part.begin(blockIdx.x + 1);

    T acc[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) acc[k] = T(0);

    // columns j0 + cl, j0 + cl + col_lanes, ...: U at a time
    constexpr int U = (RPT == 1) ? 16 : (RPT == 2 ? 8 : 4);
    uint64_t j = j0 + cl;
    const uint64_t step = uint64_t(col_lanes);
    for (; j + (U - 1) * step < j1; j += U * step) {
        T av[U][RPT];
        T xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const T* col = A + (j + u * step) * m;
            xv[u] = __ldg(x + j + u * step);
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const uint64_t r = uint64_t(rl) + uint64_t(k) * row_lanes;
                av[u][k] = r < m ? __ldcs(col + r) : T(0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < RPT; ++k) acc[k] = fma_rn(av[u][k], xv[u], acc[k]);
    }
    for (; j < j1; j += step) {
        const T* col = A + j * m;
        const T xj = __ldg(x + j);
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const uint64_t r = uint64_t(rl) + uint64_t(k) * row_lanes;
            if (r < m) acc[k] = fma_rn(__ldcs(col + r), xj, acc[k]);
        }
    }

    // column lanes -> CTA partial, fixed order
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const uint64_t r = uint64_t(rl) + uint64_t(k) * row_lanes;
        if (r < m) sm[uint64_t(cl) * m + r] = acc[k];
    }
    __syncthreads();
    for (uint64_t r = tid; r < m; r += kSplitBlock) {
        T v = sm[r];
        for (int q = 1; q < col_lanes; ++q) v = add_rn(v, sm[uint64_t(q) * m + r]);
        partials[uint64_t(blockIdx.x) * m + r] = v;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) am_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    for (uint64_t r = tid; r < m; r += kSplitBlock) {
        T total = T(0);
        for (unsigned b = 0; b < gridDim.x; ++b) total = add_rn(total, ld_cg(partials + uint64_t(b) * m + r));
        c[r] = add_rn(c[r], total);
    }
    if (tid == 0) *ticket = 0u;
}

struct SplitGeom {
    int row_lanes, col_lanes, rpt;
    unsigned grid;
    size_t smem;
};

template <typename T> SplitGeom split_geom(uint64_t m, uint64_t n) {
    SplitGeom g;
    uint64_t rl = 32; // a power of two, so row_lanes divides the block
    while (rl < m && rl < uint64_t(kSplitBlock)) rl *= 2;
    g.row_lanes = int(rl);
    g.col_lanes = kSplitBlock / g.row_lanes;
    g.rpt = int((m + rl - 1) / rl);
    const uint64_t cap = uint64_t(sm_count()) * kSplitCtasPerSm;
    const uint64_t want = (n + g.col_lanes - 1) / g.col_lanes; // >= 1 column per column lane
    g.grid = unsigned(want < cap ? (want < 1 ? 1 : want) : cap);
    g.smem = size_t(g.col_lanes) * m * sizeof(T); // <= 512*s (m<=512) or m*s (m<2048): < 48 KB
    return g;
}

} // namespace

template <typename T> WorkspaceNeed gemv_cm_need(const T*, const T*, uint64_t m, uint64_t n) {
    WorkspaceNeed w;
    if (m == 0 || n == 0 || m >= kSplitMaxRows) return w;
    const SplitGeom g = split_geom<T>(m, n);
    w.counters = 1;
    w.scratch_bytes = size_t(g.grid) * m * sizeof(T);
    return w;
}

template <typename T>
cudaError_t gemv_cm_launch(const T* A, uint64_t m, uint64_t n, const T* x, T* c,
                           const Workspace& ws, cudaStream_t s, LaunchInfo* info) {
    if (info) info->ctas = 0;
    if (m == 0 || n == 0) return cudaSuccess;
    if (m >= kSplitMaxRows) {
        const uint64_t units = (m + kWarp - 1) / kWarp;
        const uint64_t max_warps = uint64_t(sm_count()) * kCmRowsCtasPerSm * (kCmBlock / kWarp);
        // smallest per-warp unit count that fits one wave, then as few warps
        // as keep that count: every warp gets the same number of units +-1
        const uint64_t per = (units + max_warps - 1) / max_warps;
        const uint64_t warps = (units + per - 1) / per;
        const unsigned grid = unsigned((warps * kWarp + kCmBlock - 1) / kCmBlock);
        gemv_cm_rows_kernel<T><<<grid, kCmBlock, 0, s>>>(A, x, c, m, n, warps);
        if (info) info->ctas = grid;
    } else {
        const SplitGeom g = split_geom<T>(m, n);
        T* partials = static_cast<T*>(ws.scratch);
        switch (g.rpt) {
        case 1:
            gemv_cm_split_kernel<T, 1><<<g.grid, kSplitBlock, g.smem, s>>>(
                A, x, c, m, n, g.row_lanes, partials, ws.counters);
            break;
        case 2:
            gemv_cm_split_kernel<T, 2><<<g.grid, kSplitBlock, g.smem, s>>>(
                A, x, c, m, n, g.row_lanes, partials, ws.counters);
            break;
        default:
            gemv_cm_split_kernel<T, 4><<<g.grid, kSplitBlock, g.smem, s>>>(
                A, x, c, m, n, g.row_lanes, partials, ws.counters);
            break;
        }
        if (info) info->ctas = g.grid;
    }
    return cudaGetLastError();
}

template WorkspaceNeed gemv_cm_need<float>(const float*, const float*, uint64_t, uint64_t);
template WorkspaceNeed gemv_cm_need<double>(const double*, const double*, uint64_t, uint64_t);
template cudaError_t gemv_cm_launch<float>(const float*, uint64_t, uint64_t, const float*,
                                           float*, const Workspace&, cudaStream_t, LaunchInfo*);
template cudaError_t gemv_cm_launch<double>(const double*, uint64_t, uint64_t, const double*,
                                            double*, const Workspace&, cudaStream_t,
                                            LaunchInfo*);

} // namespace cabl_dev

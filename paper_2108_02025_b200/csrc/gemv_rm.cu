// Row-major GEMV: c += A x, A is m x n row-major — B200 re-design of reference
// cabl::gemv_row_major (proj/include/cabl/kernels.hpp:230-257).
//
// The reference hands whole rows to CPU threads.  On B200 a whole-row split
// leaves the 148 SMs unevenly loaded whenever m is not a large multiple of
// the warp count (8192 rows over 2368 warps is 3.46 rows/warp: 16% of the
// machine idles at the end).  Instead the work is cut into UNITS of
// R rows x SEG warp-vectors (one warp-vector = 32 lanes x 32 bytes), units
// are ordered (row group, column segment), and every warp of a single-wave
// grid owns a contiguous, balanced range of units (±1 unit).
//
//   * a warp keeps R*SEG + SEG 256-bit loads in flight per lane per unit
//     (A streamed with L1::no_allocate, x through L1 — it is re-read by every
//     row group, R rows share each x load);
//   * per row, lanes accumulate with FMA, then a fixed butterfly sums lanes;
//   * a row group entirely inside one warp's range is finished by that warp:
//     c[i] = c[i] + sum;
//   * a row group split across warps (only at range boundaries — at most one
//     per warp) leaves one partial per touching warp in a slot; the last warp
//     to arrive (atomic ticket) adds the partials in warp order, then to c,
//     and resets the ticket.
// Every per-element order is a function of (m, n, grid) only: bitwise
// reproducible run to run.
//
// Kernels by shape (rm_mode):
//   * rows <= 256 B, many of them: one thread per row in the reference's
//     order and rounding — bitwise gemv_ref (gemv_rm_lane_kernel, mode 3/4);
//   * rows of 256 B .. 4 KiB: the sub-CTA sweep (row slots of 16 - 128 lanes,
//     gemv_rm_subsweep_kernel), or G lanes per row for fp64 rows that fill
//     barely half of a slot (gemv_rm_gvec_kernel) — both mode 7;
//   * longer rows, enough of them: the CTA-wide SWEEP (modes 1, 2; a row
//     shape with mostly empty last passes switches to 8 x 1 groups);
//   * few rows: the unit kernel described above (mode 0);
//   * unaligned operands or n % (32/sizeof(T)) != 0 (mode -1): the scalar
//     sub-CTA sweep for rows of 65 .. 2048 elements and m >= 148 * 64, one CTA
//     per row for few long rows, else G lanes per row with scalar loads.
// CABL_GEMV_RM_ORDER=reference routes to gemv_rm_ordered.cu instead where it
// applies.  Every kernel is bitwise reproducible run to run.
//
// Algorithmic bytes per launch: m*n*s + n*s + 2*m*s.
#include "common.cuh"
#include "dot_body.cuh"
#include "gemv_rm_body.cuh"
#include "kernels.cuh"

#include <cstdio>
#include <cstdlib>

namespace cabl_dev {

namespace {

constexpr int kRmCtasPerSm = 2;
constexpr int kRmRows = 2; // R
constexpr int kRmSeg = 2;  // SEG warp-vectors per unit

struct RmGeom {
    uint64_t nvec_row; // 32-byte vectors per row
    uint64_t nwv;      // warp-vectors per row
    uint64_t S;        // segments per row group
    uint64_t G;        // row groups
    uint64_t warps;    // warps that own units
};

template <typename T, int R, int SEG>
__global__ void __launch_bounds__(kRmBlock, kRmCtasPerSm)
    gemv_rm_vec_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                       uint64_t m, uint64_t n, RmGeom geo, T* __restrict__ slots,
                       unsigned* __restrict__ tickets) {
    pdl_enter();
    const int lane = threadIdx.x & 31;
    const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (gw >= geo.warps) return;
    const Partition part(geo.G * geo.S, geo.warps);
    const uint64_t u0 = part.begin(gw), u1 = part.begin(gw + 1);
    const Vec<T>* X = reinterpret_cast<const Vec<T>*>(x);
    const uint64_t first_group = u0 / geo.S;

    uint64_t u = u0;
    while (u < u1) {
        const uint64_t g = u / geo.S;
        const uint64_t s_begin = u - g * geo.S;
        const uint64_t s_end = (geo.S - s_begin < u1 - u) ? geo.S : s_begin + (u1 - u);
        const uint64_t row0 = g * R;
        const int rows = (m - row0 < uint64_t(R)) ? int(m - row0) : R;
        const Vec<T>* Arow[R];
#pragma unroll
        for (int r = 0; r < R; ++r)
            Arow[r] = reinterpret_cast<const Vec<T>*>(A + (row0 + (r < rows ? r : 0)) * n);

        T acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = T(0);

        for (uint64_t s = s_begin; s < s_end; ++s) {
            Vec<T> xv[SEG];
            Vec<T> av[SEG][R];
#pragma unroll
            for (int k = 0; k < SEG; ++k) {
                const uint64_t cv = (s * SEG + k) * kWarp + lane; // vector column
                if (cv < geo.nvec_row) {
                    xv[k] = ld_reuse(X + cv);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        if (r < rows) av[k][r] = ld_stream(Arow[r] + cv);
                        else
#pragma unroll
                            for (int e = 0; e < Vec<T>::N; ++e) av[k][r].v[e] = T(0);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < Vec<T>::N; ++e) xv[k].v[e] = T(0);
#pragma unroll
                    for (int r = 0; r < R; ++r)
#pragma unroll
                        for (int e = 0; e < Vec<T>::N; ++e) av[k][r].v[e] = T(0);
                }
            }
#pragma unroll
            for (int k = 0; k < SEG; ++k)
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] = dot_vec(av[k][r], xv[k], acc[r]);
        }

#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = warp_sum(acc[r]);

        if (s_begin == 0 && s_end == geo.S) {
            // whole row group owned by this warp
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (lane == r && r < rows) c[row0 + r] = add_rn(c[row0 + r], acc[r]);
        } else {
            // split row group: deposit, then last arriver combines in warp order
            const int which = (g == first_group) ? 0 : 1;
            T* my_slot = slots + (gw * 2 + which) * R;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (lane == r) my_slot[r] = acc[r];
            __threadfence();
            __syncwarp();
            const uint64_t wf = part.owner(g * geo.S);
            const uint64_t wl = part.owner(g * geo.S + geo.S - 1);
            unsigned arrived = 0;
            if (lane == 0) arrived = atomicAdd(tickets + wf, 1u);
            arrived = __shfl_sync(0xffffffffu, arrived, 0);
            if (arrived == unsigned(wl - wf)) {
                __threadfence();
                // the row's warp partials, lane-strided (lane l sums warps wf + l,
                // wf + l + 32, ... in order), then the fixed butterfly: a row
                // split over thousands of warps (m = 1..64) no longer pays one
                // dependent L2 round trip per warp (2^0 x 2^26 fp32: 870 us)
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (r >= rows) break;
                    T total = T(0);
#pragma unroll 4
                    for (uint64_t w = wf + lane; w <= wl; w += kWarp) {
                        const int wh = (g == part.begin(w) / geo.S) ? 0 : 1;
                        total = add_rn(total, ld_cg(slots + (w * 2 + wh) * R + r));
                    }
                    total = warp_sum(total);
                    if (lane == 0) c[row0 + r] = add_rn(c[row0 + r], total);
                }
                if (lane == 0) tickets[wf] = 0u;
            }
        }
        u += s_end - s_begin;
    }
}

// SWEEP kernel (m large relative to the grid).  Work is cut into groups of R
// rows; all BLOCK threads of a CTA read a group's rows together — thread t
// owns the vector columns t, t + BLOCK, ... — so every CTA-wide load is one
// contiguous BLOCK*32-byte run, and consecutive groups are consecutive
// stretches of A, so the GPU sweeps A front to back (the access order that
// measured fastest for a streaming read on B200, tools/bwlab.py).  Groups are
// handed out in grid-stride order (DYN = false) or drawn from an atomic
// counter (DYN = true): SMs that get faster memory service take more groups.
// x is re-read per chunk through L1 and shared by the R rows.  Per row: fixed
// butterfly per warp, then the warp partials summed in warp order by one
// thread (double-buffered shared slots: one barrier per group),
// c[i] = c[i] + sum.  A group's result does not depend on which CTA took it:
// bitwise reproducible either way.
template <typename T, int R, int KV, int MINB, bool DYN>
__global__ void __launch_bounds__(kRmBlock, MINB)
    gemv_rm_sweep_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                         uint64_t m, uint64_t n, unsigned* __restrict__ counter, int pf) {
    pdl_trigger();
    if (pf > 0 && threadIdx.x < R) {
        // warm L2 with this CTA's first pass (R rows x the block's KV
        // vectors).  Measured neutral on G1/G4 (39.2 / 2305 us either way);
        // prefetching 2-8 passes is slower (40.5-43.4 us on G1).
        const uint64_t row = uint64_t(blockIdx.x) * R + threadIdx.x;
        const uint64_t pass = uint64_t(kRmBlock) * KV * sizeof(Vec<T>);
        if (row < m)
            prefetch_l2_bulk(A + row * n, unsigned(n * sizeof(T) < pass ? n * sizeof(T) : pass));
    }
    pdl_wait();
    sweep_groups<T, R, KV, DYN>(A, x, m, n, counter, blockIdx.x, gridDim.x, c,
                                [&](uint64_t row, T sum, T c_row) { c[row] = add_rn(c_row, sum); });
}

// CHUNKED FEW-ROWS kernel (aligned rows, few of them: a row is a long DOT
// with x).  Units are (row, chunk of `chunk` 32-byte vectors), numbered chunk-
// major so the m units that read the same x chunk run together (x comes from
// L2 after the first row).  CTAs take units from an atomic queue (the first
// one static), as the chunked DOT does (dot_body.cuh); a unit's partial is a
// fixed function of its data and goes to partials[row][chunk]; the CTA that
// finishes a row's last unit (per-row acq_rel ticket) sums the row's partials
// in chunk order and adds them to c.  Bitwise reproducible (depends on m, n
// only).  The unit kernel below keeps 4 loads in flight per lane at 512
// threads per SM (1 x 2^26 fp32: 127 us, 4.2 TB/s).
constexpr int kChunkBlock = 512;
constexpr int kChunkU = 2;

// R rows per unit share each x vector load (R = 1 for a single row).
template <typename T, int R, int MINB>
__global__ void __launch_bounds__(kChunkBlock, MINB)
    gemv_rm_chunk_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                         uint64_t m, uint64_t n, uint64_t chunk, uint64_t nchunks,
                         T* __restrict__ partials, unsigned* __restrict__ counters) {
    pdl_enter();
    constexpr int V = Vec<T>::N;
    constexpr int U = kChunkU;
    __shared__ T red[32];
    __shared__ unsigned long long next_sh;
    __shared__ bool last_sh;
    const int tid = threadIdx.x;
    const uint64_t nvec = n / V;
    const uint64_t groups = (m + R - 1) / R;
    const uint64_t units = groups * nchunks;
    const Vec<T>* X = reinterpret_cast<const Vec<T>*>(x);
    uint64_t u = blockIdx.x;
    while (u < units) {
        if (tid == 0) next_sh = dyn_next(counters, units); // prefetch
        const uint64_t ch = u / groups, grp = u - ch * groups;
        const uint64_t row0 = grp * R;
        const int rows = (m - row0 < uint64_t(R)) ? int(m - row0) : R;
        const uint64_t c0 = ch * chunk;
        const uint64_t c1 = (c0 + chunk < nvec) ? c0 + chunk : nvec;
        T acc[R][U];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int k = 0; k < U; ++k) acc[r][k] = T(0);
        for (uint64_t base = c0; base < c1; base += uint64_t(kChunkBlock) * U) {
            Vec<T> av[R][U], xv[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const uint64_t i = base + uint64_t(k) * kChunkBlock + tid;
                const bool ok = i < c1;
                if (ok) xv[k] = ld_stream(X + i);
                else
#pragma unroll
                    for (int e = 0; e < V; ++e) xv[k].v[e] = T(0);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (ok && r < rows) av[r][k] = ld_stream(reinterpret_cast<const Vec<T>*>(A + (row0 + r) * n) + i);
                    else
#pragma unroll
                        for (int e = 0; e < V; ++e) av[r][k].v[e] = T(0);
                }
            }
#pragma unroll
            for (int k = 0; k < U; ++k)
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r][k] = dot_vec(av[r][k], xv[k], acc[r][k]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            T v = acc[r][0];
#pragma unroll
            for (int k = 1; k < U; ++k) v = add_rn(v, acc[r][k]);
            const T unit_total = block_sum(v, red); // its barriers publish next_sh
            if (tid == 0 && r < rows) partials[(row0 + r) * nchunks + ch] = unit_total;
        }
        if (last_arriver(counters + 1 + grp, unsigned(nchunks), &last_sh)) {
            for (int r = 0; r < rows; ++r) {
                T w = T(0);
                for (uint64_t i = tid; i < nchunks; i += kChunkBlock)
                    w = add_rn(w, ld_cg(partials + (row0 + r) * nchunks + i));
                const T total = block_sum(w, red);
                if (tid == 0) c[row0 + r] = add_rn(c[row0 + r], total);
            }
            if (tid == 0) counters[1 + grp] = 0u;
        }
        u = next_sh;
        __syncthreads(); // next_sh is rewritten at the top of the next unit
    }
}

// Generic path (unaligned operands or n % V != 0): G lanes per row (G = 32 /
// 16 / 8 / 4 by row length, so short rows do not idle most of a warp),
// groups own balanced row ranges, scalar coalesced loads.  Each lane's chain
// runs j = lane, lane + G, ... in order, the loads of kScalarU steps issued
// before they are consumed; then a fixed butterfly over the G lanes.  (One
// load in flight at a time ran odd-width rows at ~2.1 TB/s; 8192 x 8193 fp32
// now 56 us, 4.8 TB/s.)
template <typename T, int G>
__global__ void __launch_bounds__(kRmBlock)
    gemv_rm_scalar_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                          uint64_t m, uint64_t n, uint64_t groups) {
    pdl_enter();
    const int lg = threadIdx.x & (G - 1);
    const uint64_t gg = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    if (gg >= groups) return; // whole groups leave together (G divides 32)
    const Partition part(m, groups);
    constexpr int kScalarU = 16;
    for (uint64_t i = part.begin(gg); i < part.begin(gg + 1); ++i) {
        const T* row = A + i * n;
        T acc = T(0);
        uint64_t j = lg;
        for (; j + uint64_t(kScalarU - 1) * G < n; j += uint64_t(kScalarU) * G) {
            T a[kScalarU], b[kScalarU];
#pragma unroll
            for (int u = 0; u < kScalarU; ++u) {
                a[u] = __ldcs(row + j + u * G);
                b[u] = __ldg(x + j + u * G);
            }
#pragma unroll
            for (int u = 0; u < kScalarU; ++u) acc = fma_rn(a[u], b[u], acc);
        }
        for (; j < n; j += G) acc = fma_rn(row[j], x[j], acc);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o, G));
        if (lg == 0) c[i] = add_rn(c[i], acc);
    }
}

// Long scalar rows, few of them (odd n or unaligned operands; fewer rows than
// the G-lanes kernel needs to keep the SMs' memory pipes full): one CTA per
// row, all kRmBlock threads on the row — thread t chains j = t, t + BLOCK, ...
// with kScalarU loads in flight, then a fixed-order block sum.  (2400 x 27961
// fp32 on one warp per row kept ~32 KB per SM in flight: 113 us.)
template <typename T>
__global__ void __launch_bounds__(kRmBlock)
    gemv_rm_scalar_cta_kernel(const T* __restrict__ A, const T* __restrict__ x,
                              T* __restrict__ c, uint64_t m, uint64_t n) {
    pdl_enter();
    __shared__ T red[32];
    constexpr int kScalarU = 16;
    for (uint64_t i = blockIdx.x; i < m; i += gridDim.x) {
        const T* row = A + i * n;
        T acc = T(0);
        uint64_t j = threadIdx.x;
        for (; j + uint64_t(kScalarU - 1) * kRmBlock < n; j += uint64_t(kScalarU) * kRmBlock) {
            T a[kScalarU], b[kScalarU];
#pragma unroll
            for (int u = 0; u < kScalarU; ++u) {
                a[u] = __ldcs(row + j + u * kRmBlock);
                b[u] = __ldg(x + j + u * kRmBlock);
            }
#pragma unroll
            for (int u = 0; u < kScalarU; ++u) acc = fma_rn(a[u], b[u], acc);
        }
        for (; j < n; j += kRmBlock) acc = fma_rn(row[j], x[j], acc);
        const T total = block_sum(acc, red);
        if (threadIdx.x == 0) c[i] = add_rn(c[i], total);
    }
}

// Short rows (n*s <= rm_lane_max_bytes() = 256 B, e.g. 2^20 x 64): one THREAD per
// row, in the reference's order and rounding — acc = c_i, then for j
// ascending a separately rounded multiply and add (an FMA for the trailing
// n mod 16/s terms), exactly gemv_ref (reference kernels.hpp:171-181): bit
// for bit the compiled reference at bandwidth, because a short row's chain is
// short.  Adjacent rows are adjacent in memory, so a warp's loads cover one
// contiguous 32-row block; the 256 B L2 promotion turns each lane's 32-byte
// requests into full bursts.  U loads in flight per thread; x comes through L1
// (every lane of a warp reads the same x vector).  The sweep kernels spend a
// 256-thread CTA per group of 4 rows.  256 MiB of A, flushed, sweep -> this
// kernel: fp32 n = 1 / 16 / 64 / 256 / 1024: 0.11 / 0.07 / 0.27 / 1.0 / 3.3
// -> 4.1 / 6.2 / 4.8 / 4.3 / 4.4 TB/s; at 8 KiB rows the sweep is ahead.
template <typename T, bool VEC, int U>
__global__ void __launch_bounds__(kRmBlock)
    gemv_rm_lane_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                        uint64_t m, uint64_t n) {
    pdl_enter();
    constexpr uint64_t kRefVec = 16 / sizeof(T);
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m; i += stride) {
        T acc = c[i];
        if constexpr (VEC) { // n % V == 0, 32-byte aligned rows: every term is mul + add
            constexpr int V = Vec<T>::N;
            const Vec<T>* a = reinterpret_cast<const Vec<T>*>(A + i * n);
            const Vec<T>* X = reinterpret_cast<const Vec<T>*>(x);
            const uint64_t nv = n / V;
            uint64_t k = 0;
            for (; k + U <= nv; k += U) {
                Vec<T> av[U], xv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    av[u] = ld_stream(a + k + u);
                    xv[u] = ld_reuse(X + k + u);
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int e = 0; e < V; ++e) acc = add_rn(acc, mul_rn(av[u].v[e], xv[u].v[e]));
            }
            for (; k < nv; ++k) {
                const Vec<T> av = ld_stream(a + k), xv = ld_reuse(X + k);
#pragma unroll
                for (int e = 0; e < V; ++e) acc = add_rn(acc, mul_rn(av.v[e], xv.v[e]));
            }
        } else {
            const T* a = A + i * n;
            const uint64_t cut = (n / kRefVec) * kRefVec;
            uint64_t j = 0;
            for (; j + U <= cut; j += U) {
                T av[U], xv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    av[u] = __ldcs(a + j + u);
                    xv[u] = __ldg(x + j + u);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) acc = add_rn(acc, mul_rn(av[u], xv[u]));
            }
            for (; j < cut; ++j) acc = add_rn(acc, mul_rn(__ldcs(a + j), __ldg(x + j)));
            for (; j < n; ++j) acc = fma_rn(__ldcs(a + j), __ldg(x + j), acc);
        }
        c[i] = acc;
    }
}

// (Measured, not kept: the same chains fed by fully coalesced loads and a
// shared-memory transpose — 256 consecutive rows per CTA, row pitch n + 1 — took
// fp32 n = 64 / 32 57.0 / 64.1 us flushed against 53.1 / 51.0 for this kernel, fp64
// n = 32 / 16 100.4 / 116.0 against 98.3 / 102.0: the two barriers per 64 KB block
// and the scalar shared-memory traffic cost more than the 32-sector gathers they
// replace; profiles/r02_rm_lane_t_lost.jsonl.)
// Row bytes up to which one thread per row beats the CTA-wide sweeps
// (CABL_RM_LANE_MAX overrides, tuning only).  gemv_rm_is_lane (kernels.cuh)
// adds the row-count condition.
inline uint64_t rm_lane_max_bytes() {
    static const uint64_t v = [] {
        const char* e = tuning_env("CABL_RM_LANE_MAX");
        return e ? uint64_t(atoll(e)) : uint64_t(256);
    }();
    return v;
}

// Rows of 256 B .. 4 KiB of whole 32-byte vectors (mode 7): G lanes per row,
// each lane 32-byte vectors j = lg, lg + G, ... with kGVecU in flight, then a
// fixed butterfly over the G lanes.  Coalesced G * 32-byte runs per row
// where the one-thread-per-row kernel's warps touch 32 rows per load.
constexpr int kGVecU = 4;
constexpr uint64_t kGVecMaxBytes = 4096;

template <typename T, int G>
__global__ void __launch_bounds__(kRmBlock)
    gemv_rm_gvec_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                        uint64_t m, uint64_t n, uint64_t groups) {
    pdl_enter();
    const int lg = threadIdx.x & (G - 1);
    const uint64_t gg = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    if (gg >= groups) return;
    const Partition part(m, groups);
    const uint64_t nv = n / Vec<T>::N;
    const Vec<T>* X = reinterpret_cast<const Vec<T>*>(x);
    for (uint64_t i = part.begin(gg); i < part.begin(gg + 1); ++i) {
        const Vec<T>* row = reinterpret_cast<const Vec<T>*>(A + i * n);
        T acc = T(0);
        uint64_t j = lg;
        for (; j + uint64_t(kGVecU - 1) * G < nv; j += uint64_t(kGVecU) * G) {
            Vec<T> a[kGVecU], b[kGVecU];
#pragma unroll
            for (int u = 0; u < kGVecU; ++u) {
                a[u] = ld_stream(row + j + u * G);
                b[u] = ld_reuse(X + j + u * G);
            }
#pragma unroll
            for (int u = 0; u < kGVecU; ++u) acc = dot_vec(a[u], b[u], acc);
        }
        for (; j < nv; j += G) acc = dot_vec(ld_stream(row + j), ld_reuse(X + j), acc);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o, G));
        if (lg == 0) c[i] = add_rn(c[i], acc);
    }
}

// Rows of 9 .. 128 32-byte vectors (256 B .. 4 KiB) as a SWEEP: the CTA's 256
// threads are RP = 256 / SL row slots of SL lanes (SL = 16, 32, 64 or 128: the
// power of two >= the row's vectors), a pass loads one vector per thread of RP
// consecutive rows, a group is R passes (R * RP consecutive rows = one
// contiguous run of up to 64 KB, all its loads in flight before the first FMA),
// and groups go to CTAs grid-stride, so the whole GPU reads A front to back as
// the long-row sweeps do.  x's vector stays in registers for the CTA's lifetime
// (the G-lanes kernel re-reads x from L1 for every row), c is loaded when the
// group starts.  Per row: the thread's dot_vec, a butterfly over the slot's
// lanes (within a warp), then for slots of 2 / 4 warps the warp partials in warp
// order — fixed by n alone.  256 MiB fp32 flushed / back to back
// (profiles/r02_rm_subsweep.jsonl): n = 1024 50.9 / 45.9 -> 44.2 / 39.8 us, 512
// 51.0 / 46.0 -> 44.5 / 40.2, 256 51.1 / 46.7 -> 44.9 / 40.7, 400 71.8 -> 45.5.
template <typename T, int R, int SL>
__global__ void __launch_bounds__(kRmBlock, 2)
    gemv_rm_subsweep_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                            uint64_t m, uint64_t n) {
    pdl_enter();
    constexpr int RP = kRmBlock / SL, GR = R * RP;    // row slots per pass, rows per group
    constexpr int PARTS = SL > 32 ? SL / 32 : 1;      // warp partials per row
    __shared__ T red[2][R][RP * PARTS];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int slot = tid / SL, lr = tid % SL; // row slot, vector in the row
    const uint64_t nv = n / Vec<T>::N;
    const bool live = uint64_t(lr) < nv;
    Vec<T> xv;
    if (live) xv = ld_reuse(reinterpret_cast<const Vec<T>*>(x) + lr);
    else
#pragma unroll
        for (int e = 0; e < Vec<T>::N; ++e) xv.v[e] = T(0);
    const uint64_t groups = (m + GR - 1) / GR;
    int parity = 0;
    for (uint64_t g = blockIdx.x; g < groups; g += gridDim.x) {
        const uint64_t row0 = g * GR;
        // finishing thread t < GR owns row row0 + t (pass t / RP, slot t % RP)
        const bool fin = tid < GR && row0 + tid < m;
        const T c_row = fin ? c[row0 + tid] : T(0);
        Vec<T> av[R];
#pragma unroll
        for (int p = 0; p < R; ++p) {
            const uint64_t row = row0 + uint64_t(p) * RP + slot;
            if (live && row < m) av[p] = ld_stream(reinterpret_cast<const Vec<T>*>(A + row * n) + lr);
            else
#pragma unroll
                for (int e = 0; e < Vec<T>::N; ++e) av[p].v[e] = T(0);
        }
#pragma unroll
        for (int p = 0; p < R; ++p) {
            T v = dot_vec(av[p], xv, T(0));
            if constexpr (SL >= 32) {
                v = warp_sum(v);
                if (lane == 0) red[parity][p][wid] = v; // wid = slot * PARTS + warp in the slot
            } else {
#pragma unroll
                for (int o = SL / 2; o > 0; o >>= 1) v = add_rn(v, __shfl_xor_sync(0xffffffffu, v, o, SL));
                if (lr == 0) red[parity][p][slot] = v;
            }
        }
        __syncthreads();
        if (fin) {
            const int p = tid / RP, sl = tid % RP;
            T sum = red[parity][p][sl * PARTS];
#pragma unroll
            for (int w = 1; w < PARTS; ++w) sum = add_rn(sum, red[parity][p][sl * PARTS + w]);
            c[row0 + tid] = add_rn(c_row, sum);
        }
        parity ^= 1; // the next group's partials go to the other buffer: one barrier per group
    }
}

// The same sweep for rows that are not whole aligned 32-byte vectors (odd n, or A / x
// off a 32-byte boundary): scalar loads, thread lr of a slot takes elements lr, lr +
// SL, ... (NE of them, so a warp's load is one contiguous 128-byte run), x's NE
// elements stay in registers, FMA per element, then the slot butterfly and warp
// partials as above.  Rows of up to NE * SL elements.
// 256 MiB fp32 flushed (profiles/r02_rm_subsweep_scalar*.jsonl), G-lanes scalar kernel
// -> this: n = 1001 75.9 -> 46.8 us, 255 65.8 -> 46.1, 129 90.2 -> 53.5, 65 89.3 ->
// 53.4, 2047 64.0 -> 47.8; fp64 n = 1001 133.1 -> 82.0, 301 105.4 -> 86.2.
template <typename T, int R, int SL, int NE>
__global__ void __launch_bounds__(kRmBlock, 2)
    gemv_rm_subsweep_scalar_kernel(const T* __restrict__ A, const T* __restrict__ x,
                                   T* __restrict__ c, uint64_t m, uint64_t n) {
    pdl_enter();
    constexpr int RP = kRmBlock / SL, GR = R * RP;
    constexpr int PARTS = SL > 32 ? SL / 32 : 1;
    __shared__ T red[2][R][RP * PARTS];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int slot = tid / SL, lr = tid % SL;
    T xr[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
        const uint64_t j = uint64_t(lr) + uint64_t(e) * SL;
        xr[e] = j < n ? __ldg(x + j) : T(0);
    }
    const uint64_t groups = (m + GR - 1) / GR;
    int parity = 0;
    for (uint64_t g = blockIdx.x; g < groups; g += gridDim.x) {
        const uint64_t row0 = g * GR;
        const bool fin = tid < GR && row0 + tid < m;
        const T c_row = fin ? c[row0 + tid] : T(0);
        T av[R][NE];
#pragma unroll
        for (int p = 0; p < R; ++p) {
            const uint64_t row = row0 + uint64_t(p) * RP + slot;
            const T* rp = A + row * n;
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const uint64_t j = uint64_t(lr) + uint64_t(e) * SL;
                av[p][e] = (row < m && j < n) ? __ldcs(rp + j) : T(0);
            }
        }
#pragma unroll
        for (int p = 0; p < R; ++p) {
            T v = T(0);
#pragma unroll
            for (int e = 0; e < NE; ++e) v = fma_rn(av[p][e], xr[e], v);
            if constexpr (SL >= 32) {
                v = warp_sum(v);
                if (lane == 0) red[parity][p][wid] = v;
            } else {
#pragma unroll
                for (int o = SL / 2; o > 0; o >>= 1) v = add_rn(v, __shfl_xor_sync(0xffffffffu, v, o, SL));
                if (lr == 0) red[parity][p][slot] = v;
            }
        }
        __syncthreads();
        if (fin) {
            const int p = tid / RP, sl = tid % RP;
            T sum = red[parity][p][sl * PARTS];
#pragma unroll
            for (int w = 1; w < PARTS; ++w) sum = add_rn(sum, red[parity][p][sl * PARTS + w]);
            c[row0 + tid] = add_rn(c_row, sum);
        }
        parity ^= 1;
    }
}

// Slot shape for the scalar sub-CTA sweep: rows of 65 .. 2048 elements take the
// (SL lanes, NE elements per lane) pair with the smallest capacity SL * NE >= n, NE in
// {5, 6, 8}, so a slot is always >= 75% full (a half-full slot lost: fp32 n = 513 in
// 128 x 8 57.4 -> 63.5 us).  CABL_RM_SUBSWEEP_SCALAR=0|1 (tuning only) turns it
// off / on.
struct SubScalarShape {
    int sl = 0, ne = 0;
};
inline SubScalarShape rm_subsweep_scalar_shape(uint64_t n) {
    static const int knob = [] {
        const char* e = tuning_env("CABL_RM_SUBSWEEP_SCALAR");
        return e ? atoi(e) : -1;
    }();
    SubScalarShape best;
    if (knob == 0 || n <= 64) return best;
    uint64_t cap = ~uint64_t(0);
    for (int sl : {16, 32, 64, 128, 256})
        for (int ne : {5, 6, 8})
            if (uint64_t(sl) * ne >= n && uint64_t(sl) * ne < cap) {
                cap = uint64_t(sl) * ne;
                best.sl = sl;
                best.ne = ne;
            }
    return best;
}

// Slot lanes for the sub-CTA sweep (the power of two >= the row's vectors), or 0
// when the G-lanes kernel keeps the row: fp32 rows always take the sweep (a slot
// is always more than half full: n = 520, 65 of 128 lanes, 56.0 -> 53.4 us; 72, 9
// of 16, 57.6 -> 52.0), fp64 rows from 55% (36: 9 of 16 lanes 117.5 -> 102.6 us,
// but 260 / 132 / 68 at 51-53% lost 90 -> 105, 93 -> 111, 96 -> 109).
// CABL_RM_SUBSWEEP=0 (tuning only) turns it off, CABL_RM_SUBSWEEP=<percent> sets
// the least share of a slot's lanes a row must fill.
inline int rm_subsweep_lanes(uint64_t nv, size_t elem) {
    static const int knob = [] {
        const char* e = tuning_env("CABL_RM_SUBSWEEP");
        return e ? atoi(e) : -1;
    }();
    if (knob == 0) return 0;
    const uint64_t min_pct = knob > 0 ? uint64_t(knob) : (elem == 4 ? 50 : 55);
    for (int sl : {16, 32, 64, 128, 256})
        if (nv <= uint64_t(sl)) return nv * 100 >= uint64_t(sl) * min_pct ? sl : 0;
    return 0;
}

template <typename T> bool rm_vec_ok(const T* A, const T* x, uint64_t n) {
    return aligned32(A) && aligned32(x) && (n % Vec<T>::N == 0);
}

// Few long rows take the chunked kernel (mode 9).  256 MiB of A, flushed
// (tools/rm_few.py), unit kernel -> chunked (R = 1 for one row, else 2 rows per
// unit): m = 1 / 2 / 4 / 16 fp32 129 / 129 / 96 / 61.4 -> 84 / 67.6 / 59.4 /
// 55.3 us; from m = 64 up the other kernels win (51 vs 53; 4 rows per unit
// was slower everywhere).  CABL_RM_FEW_MAX overrides the row limit (tuning).
inline bool rm_few_rows(uint64_t m, uint64_t n, size_t elem) {
    static const uint64_t max_rows = [] {
        const char* e = tuning_env("CABL_RM_FEW_MAX");
        return e ? uint64_t(atoll(e)) : uint64_t(16);
    }();
    return m <= max_rows && n * elem >= 65536;
}

// -1 scalar, 0 segment-balanced warps, 1 sweep for short rows, 2 sweep for
// long rows, 9 chunked few rows.  CABL_GEMV_RM_MODE overrides (tuning / tests only).
// Row groups from which the sweeps run (see rm_mode).
constexpr uint64_t kRmShortMinGroups = 256; // 4-row groups: m >= 1021
constexpr uint64_t kRmLongMinGroups = 128;  // 2-row groups: m >= 255

template <typename T> int rm_mode(const T* A, const T* x, uint64_t m, uint64_t n) {
    const bool vec = rm_vec_ok(A, x, n);
    static const int forced = [] {
        const char* e = tuning_env("CABL_GEMV_RM_MODE");
        return e ? atoi(e) : -2;
    }();
    // one thread per row (3 vector loads, 4 scalar loads): short rows, and
    // enough of them to give every SM a few warps
    const bool lane = gemv_rm_is_lane(A, x, m, n, sizeof(T));
    if (forced == 3 || (forced < 0 && lane)) return vec ? 3 : 4;
    // rows of 256 B .. 4 KiB: G lanes per row with 32-byte vectors (256 MiB
    // fp32, n = 256 / 1024: 51.2 / 51.2 us; the bitwise lane kernel 63.5 /
    // 62.5, the sweeps worse still)
    if (forced == 7 ||
        (forced < 0 && n * sizeof(T) <= kGVecMaxBytes && m >= uint64_t(sm_count()) * 64)) {
        if (vec) return 7;
    }
    // fp32 rows of 4 .. 8 KiB in one-row (256-lane) slots of the sub-CTA sweep: x in
    // registers instead of an L1 load per group (256 MiB flushed / back to back,
    // profiles/r02_rm_subsweep256.jsonl: n = 2048 45.0 / 40.3 -> 43.8 / 39.6 us, 1280
    // 47.9 / 42.8 -> 45.5 / 41.5, 1032 55.0 / 50.0 -> 51.1 / 47.1); fp64 stays on the
    // 8 x 1 sweep (n = 1024 81.0 / 76.3 against 82.4 / 77.9).  CABL_RM_SUBSWEEP_MAXB
    // (tuning only) sets the byte limit for both types.
    static const long long sub_maxb_knob = [] {
        const char* e = tuning_env("CABL_RM_SUBSWEEP_MAXB");
        return e ? atoll(e) : -1ll;
    }();
    const uint64_t sub_maxb = sub_maxb_knob >= 0 ? uint64_t(sub_maxb_knob)
                                                 : (sizeof(T) == 4 ? uint64_t(8192) : uint64_t(0));
    if (forced < 0 && vec && n * sizeof(T) > kGVecMaxBytes && n * sizeof(T) <= sub_maxb &&
        m >= uint64_t(sm_count()) * 64 && rm_subsweep_lanes(n / Vec<T>::N, sizeof(T)) != 0)
        return 7;
    if (!vec) return -1;
    if (forced >= 0 && forced <= 2) return forced;
    if (forced == 9 || (forced < 0 && rm_few_rows(m, n, sizeof(T)))) return 9;
    // measured (tools/tune.py, 8192^2 and 65536^2 fp32): 4 rows x 2 vectors
    // per thread at 2 CTAs/SM for rows of <= 2 CTA passes, 2 rows x 8 vectors
    // at 1 CTA/SM for long rows.  The sweep must see >= 6 row groups per CTA
    // to keep the single wave balanced; otherwise the segment kernel.
    // Few groups per CTA still beat the unit kernel (256 MiB fp32, flushed,
    // tools/rm_mid.py): 2048 x 8192 22.5 -> 16.4 us at 1.7 groups per CTA,
    // 512 x 131072 49.2 -> 44.1 us at 0.9 (CABL_RM_FEW_GROUPS=0: the old
    // >= 6 groups per CTA rule, tuning only).
    const uint64_t sms = uint64_t(sm_count());
    const bool short_rows = n / Vec<T>::N <= uint64_t(kRmBlock) * 2 * 2;
    static const bool few = [] {
        const char* e = tuning_env("CABL_RM_FEW_GROUPS");
        return e ? atoi(e) != 0 : true;
    }();
    const uint64_t short_min = few ? kRmShortMinGroups : 6 * 2 * sms;
    const uint64_t long_min = few ? kRmLongMinGroups : 6 * 1 * sms;
    if (short_rows && (m + 3) / 4 >= short_min) return 1;
    if (!short_rows && (m + 1) / 2 >= long_min) return 2;
    return 0;
}

// Few-rows chunk size (vectors): the largest power of two giving >= 8 units
// per CTA slot, in [256, 65536], and no more than a row.
template <typename T> uint64_t rm_chunk_vecs(uint64_t m, uint64_t n) {
    const uint64_t nvec = n / Vec<T>::N;
    const uint64_t slots = uint64_t(sm_count()) * 2 * 8;
    uint64_t cv = 256;
    while (cv * 2 <= 65536 && m * ((nvec + cv * 2 - 1) / (cv * 2)) >= slots && cv * 2 <= nvec) cv *= 2;
    return cv;
}

// Rows per unit of the chunked kernel (CABL_RM_CHUNK_ROWS overrides: tuning).
inline int rm_chunk_rows(uint64_t m) {
    static const int forced = [] {
        const char* e = tuning_env("CABL_RM_CHUNK_ROWS");
        return e ? atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2) return forced;
    return m == 1 ? 1 : 2; // measured: R = 2 beats 1 from m = 2 and 4 everywhere
}

template <typename T> RmGeom rm_geom(uint64_t m, uint64_t n) {
    RmGeom g;
    g.nvec_row = n / Vec<T>::N;
    g.nwv = (g.nvec_row + kWarp - 1) / kWarp;
    g.S = (g.nwv + kRmSeg - 1) / kRmSeg;
    if (g.S == 0) g.S = 1;
    g.G = (m + kRmRows - 1) / kRmRows;
    const uint64_t max_warps = uint64_t(sm_count()) * kRmCtasPerSm * (kRmBlock / kWarp);
    const uint64_t units = g.G * g.S;
    g.warps = units < max_warps ? units : max_warps;
    return g;
}


struct SweepCfg {
    int R, KV, minb;
};

// Dynamic group queue or static grid-stride order.  Measured (tools/tune.py):
// 65536^2 fp32 2331 -> 2270 us with the queue, 8192^2 fp32 43.5 -> 44.8 us
// (the queue's atomics do not pay off on a 40 us kernel).  CABL_GEMV_DYN=0|1
// overrides the size rule (tuning only).
inline bool use_dyn_queue(uint64_t bytes) {
    static const int forced = [] {
        const char* e = tuning_env("CABL_GEMV_DYN");
        return e ? atoi(e) : -1;
    }();
    if (forced >= 0) return forced != 0;
    return bytes >= queue_threshold_bytes();
}

template <typename T, int R, int KV, int MINB>
unsigned sweep_go(const T* A, const T* x, T* c, uint64_t m, uint64_t n, unsigned* counter,
                  cudaStream_t s) {
    const uint64_t groups = (m + R - 1) / R;
    const uint64_t ctas = uint64_t(sm_count()) * MINB;
    const unsigned grid = unsigned(groups < ctas ? groups : ctas);
    if (use_dyn_queue(m * n * sizeof(T)))
        launch(gemv_rm_sweep_kernel<T, R, KV, MINB, true>, grid, kRmBlock, 0, s, A, x, c, m, n, counter,
               pdl_prefetch_enabled());
    else
        launch(gemv_rm_sweep_kernel<T, R, KV, MINB, false>, grid, kRmBlock, 0, s, A, x, c, m, n, counter,
               pdl_prefetch_enabled());
    return grid;
}

// The sweep shape for (m, n, mode): the CABL_RM_SWEEP="R,KV,MINB" tuning entry
// if set (tools/tune.py), else the measured rule.
//   A row whose vectors leave the last pass of the chosen shape mostly empty
// pays a whole pass of latency for it (fp32 8192 x 8200 under (2,8,1): 59.6
// us against 44.1 for 8192 x 8192).  When the passes would be more than
// 25% empty, take 8 rows x 1 vector (256-vector passes): 8200 -> 47.1,
// 10000 -> 45.1, 2048 -> 46.1 (was 53.3), 5000 -> 46.1 (was 49.2) us.
template <typename T> SweepCfg sweep_choice(uint64_t m, uint64_t n, int mode) {
    static const SweepCfg forced = [] {
        SweepCfg f{0, 0, 0};
        if (const char* e = tuning_env("CABL_RM_SWEEP")) sscanf(e, "%d,%d,%d", &f.R, &f.KV, &f.minb);
        return f;
    }();
    const SweepCfg table[] = {{2, 4, 2}, {2, 8, 1}, {4, 1, 4}, {4, 2, 2}, {4, 4, 1}, {8, 1, 2}, {8, 2, 1},
                              {1, 8, 2}, {1, 16, 1}, {2, 4, 1}};
    for (const SweepCfg& t : table)
        if (forced.R == t.R && forced.KV == t.KV && forced.minb == t.minb) return t;
    // long rows below the queue threshold: 2 rows x 4 vectors at 2 CTAs/SM
    // (256 MiB fp32: 512 x 131072 / 2048 x 32768 / 4096 x 16384 44.1 / 45.1 /
    // 45.1 us against 47.1-49.2 for 2 x 8 at 1 CTA/SM); above it (G4) 2 x 8.
    const bool big = m * n * sizeof(T) >= queue_threshold_bytes();
    const SweepCfg base = mode == 1 ? SweepCfg{4, 2, 2} : (big ? SweepCfg{2, 8, 1} : SweepCfg{2, 4, 2});
    const uint64_t nvec = n / Vec<T>::N;
    const uint64_t pass = uint64_t(kRmBlock) * base.KV;
    const uint64_t used = (nvec + pass - 1) / pass * pass;
    if (used * 4 > nvec * 5 && (m + 7) / 8 >= uint64_t(sm_count()) * 2) return SweepCfg{8, 1, 2};
    return base;
}

template <typename T>
unsigned sweep_launch(const T* A, const T* x, T* c, uint64_t m, uint64_t n, int mode,
                      unsigned* counter, cudaStream_t s) {
    const SweepCfg cfg = sweep_choice<T>(m, n, mode);
#define CABL_SWEEP_CASE(R_, KV_, MB_)                                                          \
    if (cfg.R == R_ && cfg.KV == KV_ && cfg.minb == MB_)                                       \
        return sweep_go<T, R_, KV_, MB_>(A, x, c, m, n, counter, s);
    CABL_SWEEP_CASE(2, 4, 2)
    CABL_SWEEP_CASE(2, 8, 1)
    CABL_SWEEP_CASE(4, 1, 4)
    CABL_SWEEP_CASE(4, 2, 2)
    CABL_SWEEP_CASE(4, 4, 1)
    CABL_SWEEP_CASE(8, 1, 2)
    CABL_SWEEP_CASE(8, 2, 1)
    CABL_SWEEP_CASE(1, 8, 2)
    CABL_SWEEP_CASE(1, 16, 1)
    CABL_SWEEP_CASE(2, 4, 1)
#undef CABL_SWEEP_CASE
    return sweep_go<T, 2, 8, 1>(A, x, c, m, n, counter, s);
}

} // namespace

// Scalar-load rows (odd n or misaligned) take the lane kernel only while a
// row is at most kLaneScalarMaxN long: a warp's scalar loads touch 32 rows'
// sectors per instruction, and the G-lanes-per-row scalar kernel wins above
// (256 MiB fp32: n = 17 lane 75.8 / 4 lanes 96.3 us; n = 33 118.8 / 92.2;
// n = 63 166.8 / 79.9 before the 4..16-lane groups existed).
constexpr uint64_t kLaneScalarMaxN = 24;

// Scalar rows long enough for a CTA each (>= 16 loads per thread) and too few
// for one warp per row to keep 4+ warps' loads per SM scheduler busy.
// CABL_RM_SCALAR_CTA=0|1 overrides (A/B only).
inline bool rm_scalar_cta(uint64_t m, uint64_t n) {
    static const int forced = [] {
        const char* e = tuning_env("CABL_RM_SCALAR_CTA");
        return e ? atoi(e) : -1;
    }();
    if (forced >= 0) return forced != 0;
    return n >= uint64_t(kRmBlock) * 16 && m < uint64_t(sm_count()) * 32;
}

bool gemv_rm_is_lane(const void* A, const void* x, uint64_t m, uint64_t n, size_t elem) {
    const bool vec = aligned32(A) && aligned32(x) && n % (32 / elem) == 0;
    return n * elem <= rm_lane_max_bytes() && m >= uint64_t(sm_count()) * 64 &&
           (vec || n <= kLaneScalarMaxN);
}

bool gemv_rm_use_dyn(uint64_t bytes) { return use_dyn_queue(bytes); }

template <typename T>
bool gemv_rm_sweep_cfg(const T* A, const T* x, uint64_t m, uint64_t n, int* R, int* KV, int* minb) {
    if (m == 0 || n == 0) return false;
    const int mode = rm_mode<T>(A, x, m, n);
    if (mode != 1 && mode != 2) return false;
    const SweepCfg c = sweep_choice<T>(m, n, mode);
    *R = c.R;
    *KV = c.KV;
    *minb = c.minb;
    return true;
}
template bool gemv_rm_sweep_cfg<float>(const float*, const float*, uint64_t, uint64_t, int*, int*, int*);
template bool gemv_rm_sweep_cfg<double>(const double*, const double*, uint64_t, uint64_t, int*, int*,
                                        int*);

namespace {
template <typename T> WorkspaceNeed rm_need_impl(const T* A, const T* x, uint64_t m, uint64_t n) {
    WorkspaceNeed w;
    if (m == 0 || n == 0) return w;
    const int mode = rm_mode<T>(A, x, m, n);
    if (mode == 9) {
        const uint64_t cv = rm_chunk_vecs<T>(m, n);
        const uint64_t nch = (n / Vec<T>::N + cv - 1) / cv;
        w.counters = 1 + m; // queue + per-row tickets
        w.scratch_bytes = m * nch * sizeof(T);
        return w;
    }
    if (mode >= 3) return w; // lane-per-row kernels: no scratch
    if (mode >= 1) {
        w.counters = 1; // group counter of the dynamic sweep
        return w;
    }
    if (mode != 0) return w;
    const RmGeom g = rm_geom<T>(m, n);
    w.counters = g.warps;
    w.scratch_bytes = g.warps * 2 * kRmRows * sizeof(T);
    return w;
}

template <typename T>
cudaError_t rm_launch_impl(const T* A, uint64_t m, uint64_t n, const T* x, T* c,
                           const Workspace& ws, cudaStream_t s, LaunchInfo* info) {
    if (info) info->ctas = 0;
    if (m == 0 || n == 0) return cudaSuccess; // c += 0
    const int mode = rm_mode<T>(A, x, m, n);
    if (mode == 7 && rm_subsweep_lanes(n / Vec<T>::N, sizeof(T)) != 0) {
        constexpr int R = 8;
        const int sl = rm_subsweep_lanes(n / Vec<T>::N, sizeof(T));
        const uint64_t gr = uint64_t(R) * (kRmBlock / sl);
        const uint64_t groups = (m + gr - 1) / gr;
        const uint64_t cap = uint64_t(sm_count()) * 2;
        const unsigned grid = unsigned(groups < cap ? groups : cap);
        if (sl == 16)
            launch(gemv_rm_subsweep_kernel<T, R, 16>, grid, kRmBlock, 0, s, A, x, c, m, n);
        else if (sl == 32)
            launch(gemv_rm_subsweep_kernel<T, R, 32>, grid, kRmBlock, 0, s, A, x, c, m, n);
        else if (sl == 64)
            launch(gemv_rm_subsweep_kernel<T, R, 64>, grid, kRmBlock, 0, s, A, x, c, m, n);
        else if (sl == 256)
            launch(gemv_rm_subsweep_kernel<T, R, 256>, grid, kRmBlock, 0, s, A, x, c, m, n);
        else
            launch(gemv_rm_subsweep_kernel<T, R, 128>, grid, kRmBlock, 0, s, A, x, c, m, n);
        if (info) info->ctas = grid;
    } else if (mode == 7) {
        const uint64_t nv = n / Vec<T>::N;
        const int G = nv > 96 ? 32 : (nv > 48 ? 16 : (nv > 24 ? 8 : 4));
        const uint64_t max_groups = uint64_t(sm_count()) * 8 * (kRmBlock / G);
        const uint64_t groups = m < max_groups ? m : max_groups;
        const unsigned grid = unsigned((groups * G + kRmBlock - 1) / kRmBlock);
        if (G == 32)
            launch(gemv_rm_gvec_kernel<T, 32>, grid, kRmBlock, 0, s, A, x, c, m, n, groups);
        else if (G == 16)
            launch(gemv_rm_gvec_kernel<T, 16>, grid, kRmBlock, 0, s, A, x, c, m, n, groups);
        else if (G == 8)
            launch(gemv_rm_gvec_kernel<T, 8>, grid, kRmBlock, 0, s, A, x, c, m, n, groups);
        else
            launch(gemv_rm_gvec_kernel<T, 4>, grid, kRmBlock, 0, s, A, x, c, m, n, groups);
        if (info) info->ctas = grid;
    } else if (mode == 9) {
        const uint64_t cv = rm_chunk_vecs<T>(m, n);
        const uint64_t nch = (n / Vec<T>::N + cv - 1) / cv;
        const int R = rm_chunk_rows(m);
        const uint64_t units = (m + R - 1) / R * nch;
        const uint64_t cap = uint64_t(sm_count()) * 2;
        const unsigned grid = unsigned(units < cap ? units : cap); // grid <= units (dyn_next)
        T* part = static_cast<T*>(ws.scratch);
        if (R == 1)
            launch(gemv_rm_chunk_kernel<T, 1, 2>, grid, kChunkBlock, 0, s, A, x, c, m, n, cv, nch,
                   part, ws.counters);
        else
            launch(gemv_rm_chunk_kernel<T, 2, 2>, grid, kChunkBlock, 0, s, A, x, c, m, n, cv, nch,
                   part, ws.counters);
        if (info) info->ctas = grid;
    } else if (mode >= 3) {
        const uint64_t cap = uint64_t(sm_count()) * 8;
        const uint64_t need = (m + kRmBlock - 1) / kRmBlock;
        const unsigned grid = unsigned(need < cap ? need : cap);
        if (mode == 3)
        {
            // U = 8 vectors in flight per thread from 8 vectors per row (256
            // MiB flushed, tools/ab_shapes.py: fp32 n = 64 / 32 56.8 / 52.6 ->
            // 53.0 / 50.7 us, fp64 n = 32 103.0 -> 98.3); shorter rows keep
            // U = 2 (fp32 n = 8 60.3 -> 73.1 with 8).  CABL_RM_LANE_U overrides.
            static const int forced_u = [] {
                const char* e = tuning_env("CABL_RM_LANE_U");
                return e ? atoi(e) : 0;
            }();
            const int lane_u = forced_u ? forced_u : (n / Vec<T>::N >= 4 * (sizeof(T) / 4) ? 8 : 2);
            if (lane_u == 4)
                launch(gemv_rm_lane_kernel<T, true, 4>, grid, kRmBlock, 0, s, A, x, c, m, n);
            else if (lane_u == 8)
                launch(gemv_rm_lane_kernel<T, true, 8>, grid, kRmBlock, 0, s, A, x, c, m, n);
            else
                launch(gemv_rm_lane_kernel<T, true, 2>, grid, kRmBlock, 0, s, A, x, c, m, n);
        }
        else
            launch(gemv_rm_lane_kernel<T, false, 8>, grid, kRmBlock, 0, s, A, x, c, m, n);
        if (info) info->ctas = grid;
    } else if (mode >= 1) {
        const unsigned grid = sweep_launch<T>(A, x, c, m, n, mode, ws.counters, s);
        if (info) info->ctas = grid;
    } else if (mode == 0) {
        const RmGeom g = rm_geom<T>(m, n);
        const unsigned grid = unsigned((g.warps * kWarp + kRmBlock - 1) / kRmBlock);
        launch(gemv_rm_vec_kernel<T, kRmRows, kRmSeg>, grid, kRmBlock, 0, s, 
            A, x, c, m, n, g, static_cast<T*>(ws.scratch), ws.counters);
        if (info) info->ctas = grid;
    } else if (rm_scalar_cta(m, n)) {
        const uint64_t cap = uint64_t(sm_count()) * 8;
        const unsigned grid = unsigned(m < cap ? m : cap);
        launch(gemv_rm_scalar_cta_kernel<T>, grid, kRmBlock, 0, s, A, x, c, m, n);
        if (info) info->ctas = grid;
    } else {
        const SubScalarShape sh =
            m >= uint64_t(sm_count()) * 64 ? rm_subsweep_scalar_shape(n) : SubScalarShape{};
        // fp64 rows of 513 .. 640 elements (128 lanes x 5) keep the G-lanes kernel: 513 /
        // 601 flushed 93.9 / 96.3 -> 104.5 / 98.7 us, the one shape that lost
        if (sh.sl != 0 && !(sizeof(T) == 8 && sh.sl == 128 && sh.ne == 5)) {
            constexpr int R = sizeof(T) == 4 ? 8 : 4;
            const uint64_t gr = uint64_t(R) * (kRmBlock / sh.sl);
            const uint64_t groups = (m + gr - 1) / gr;
            const uint64_t cap = uint64_t(sm_count()) * 2;
            const unsigned grid = unsigned(groups < cap ? groups : cap);
#define CABL_SUBSCALAR(SL_, NE_)                                                                 \
    if (sh.sl == SL_ && sh.ne == NE_)                                                            \
        launch(gemv_rm_subsweep_scalar_kernel<T, R, SL_, NE_>, grid, kRmBlock, 0, s, A, x, c, m, n);
#define CABL_SUBSCALAR_SL(SL_) CABL_SUBSCALAR(SL_, 5) CABL_SUBSCALAR(SL_, 6) CABL_SUBSCALAR(SL_, 8)
            CABL_SUBSCALAR_SL(16)
            CABL_SUBSCALAR_SL(32)
            CABL_SUBSCALAR_SL(64)
            CABL_SUBSCALAR_SL(128)
            CABL_SUBSCALAR_SL(256)
#undef CABL_SUBSCALAR_SL
#undef CABL_SUBSCALAR
            if (info) info->ctas = grid;
            return cudaGetLastError();
        }
        // lanes per row: about 8 elements per lane, 4..32 lanes
        const int G = n > 128 ? 32 : (n > 64 ? 16 : (n > 32 ? 8 : 4));
        const uint64_t max_groups = uint64_t(sm_count()) * 8 * (kRmBlock / G);
        const uint64_t groups = m < max_groups ? m : max_groups;
        const unsigned grid = unsigned((groups * G + kRmBlock - 1) / kRmBlock);
        if (G == 32)
            launch(gemv_rm_scalar_kernel<T, 32>, grid, kRmBlock, 0, s, A, x, c, m, n, groups);
        else if (G == 16)
            launch(gemv_rm_scalar_kernel<T, 16>, grid, kRmBlock, 0, s, A, x, c, m, n, groups);
        else if (G == 8)
            launch(gemv_rm_scalar_kernel<T, 8>, grid, kRmBlock, 0, s, A, x, c, m, n, groups);
        else
            launch(gemv_rm_scalar_kernel<T, 4>, grid, kRmBlock, 0, s, A, x, c, m, n, groups);
        if (info) info->ctas = grid;
    }
    return cudaGetLastError();
}

// x not 32-byte aligned while A's rows are whole aligned vectors (x = v[k:] of
// a buffer, say): copy x once into aligned scratch (2 n s bytes against m n s of
// A) and run the vector kernels; 16 x 2^22 fp32 took 1915 us on the scalar
// path.  Few rows only pay it when m >= 4.
template <typename T> bool rm_xcopy(const T* A, const T* x, uint64_t m, uint64_t n) {
    return aligned32(A) && !aligned32(x) && n % Vec<T>::N == 0 && m >= 4 &&
           reinterpret_cast<uintptr_t>(x) % sizeof(T) == 0;
}
} // namespace

template <typename T> WorkspaceNeed gemv_rm_need(const T* A, const T* x, uint64_t m, uint64_t n) {
    if (!rm_xcopy(A, x, m, n)) return rm_need_impl<T>(A, x, m, n);
    WorkspaceNeed w = rm_need_impl<T>(A, A, m, n); // A stands in for an aligned x
    w.scratch_bytes = (w.scratch_bytes + 255) / 256 * 256 + n * sizeof(T);
    return w;
}

template <typename T>
cudaError_t gemv_rm_launch(const T* A, uint64_t m, uint64_t n, const T* x, T* c,
                           const Workspace& ws, cudaStream_t s, LaunchInfo* info) {
    if (!rm_xcopy(A, x, m, n)) return rm_launch_impl<T>(A, m, n, x, c, ws, s, info);
    const size_t off = (rm_need_impl<T>(A, A, m, n).scratch_bytes + 255) / 256 * 256;
    T* xa = reinterpret_cast<T*>(static_cast<char*>(ws.scratch) + off);
    const cudaError_t e = cudaMemcpyAsync(xa, x, n * sizeof(T), cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    return rm_launch_impl<T>(A, m, n, xa, c, ws, s, info);
}

template WorkspaceNeed gemv_rm_need<float>(const float*, const float*, uint64_t, uint64_t);
template WorkspaceNeed gemv_rm_need<double>(const double*, const double*, uint64_t, uint64_t);
template cudaError_t gemv_rm_launch<float>(const float*, uint64_t, uint64_t, const float*,
                                           float*, const Workspace&, cudaStream_t, LaunchInfo*);
template cudaError_t gemv_rm_launch<double>(const double*, uint64_t, uint64_t, const double*,
                                            double*, const Workspace&, cudaStream_t,
                                            LaunchInfo*);

} // namespace cabl_dev

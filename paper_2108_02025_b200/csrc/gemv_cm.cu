// Column-major GEMV: c += A x, A is m x n col-major — B200 re-design of
// reference cabl::gemv_col_major (proj/include/cabl/kernels.hpp:187-224,
// Algorithm 1 of the paper: row blocks x column blocks x m_r register panels).
//
// Two shapes (cm_path picks; the numbers below are the defaults):
//
// (1) TALL (m/V >= 74 units of 256 row vectors, e.g. 2^20 x 256; n < 16 takes
//     the narrow variant with several row vectors per thread).  The CPU panel keeps m_r
//     rows of c in registers across a column block.  Here a THREAD keeps one
//     32-byte vector of rows (4 doubles / 8 floats) of c in registers across
//     ALL columns, and a CTA owns BLOCK consecutive row vectors, so every
//     column read of a CTA is one contiguous BLOCK*32-byte run; CTAs (one per
//     SM) own balanced ranges of such row units and keep U = 16 column loads
//     in flight per thread.  Each row's sum runs j ascending from c_i — the
//     reference order — with the reference's compiled rounding (multiply then
//     add over the 16-byte-vector prefix, FMA on the remainder; see
//     oracle/cabl_oracle.c): bit for bit the compiled reference gemv_ref.
//     If m is not a multiple of the vector (columns misaligned), the same
//     order runs with one row per lane (gemv_cm_rows_kernel).
//
// (2) SPLIT (everything else, e.g. 256 x 2^20).  The reference runs the
//     short-wide shape on ONE thread (a single m_c row block).
//     Below 512 rows (odd m: 1024) the column tiles are contiguous and stream
//     through a cp.async.bulk ring (the bulk kernels); above, row tiles of
//     choose_tile_rows() rows x column parts (2-D split).
//     Here one CTA per SM sweeps column tiles in grid-stride order (the whole
//     GPU reads one contiguous window at a time); threads are (row lane,
//     column lane) pairs accumulating with FMA; column lanes combine in
//     shared memory in a fixed order -> partials[cta][m].  The last CTA to
//     arrive sums the partials per row in CTA order with batched L2 loads and
//     adds them to c.  Bitwise reproducible run to run; within the BASELINE
//     tolerance of gemv_ref.
//
// Algorithmic bytes per launch: m*n*s + n*s + 2*m*s.
#include "bulk.cuh"
#include "common.cuh"
#include "kernels.cuh"

#include <cstdio>
#include <cstdlib>

namespace cabl_dev {

namespace {

constexpr int kTallBlock = 256;
constexpr int kTallUnroll = 16;
constexpr int kCmBlock = 256;
constexpr int kCmUnroll = 16;
constexpr int kCmRowsCtasPerSm = 4;
constexpr uint64_t kSplitMaxRows = 2048;
constexpr int kSplitBlock = 1024;
// column loads in flight per thread: 32 registers of A operands either way
template <typename T> __host__ __device__ constexpr int split_u() { return sizeof(T) == 4 ? 16 : 8; }

// acc + a*x with the compiled reference's rounding for term j:
// separately rounded multiply then add for j < cut, FMA after.
template <typename T> __device__ __forceinline__ T ref_step(T acc, T a, T xj, bool fused) {
    return fused ? fma_rn(a, xj, acc) : add_rn(acc, mul_rn(a, xj));
}

template <typename T, bool DYN>
__global__ void __launch_bounds__(kTallBlock, 1)
    gemv_cm_tall_vec_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                            uint64_t m, uint64_t n, unsigned* __restrict__ counter) {
    pdl_enter();
    constexpr int V = Vec<T>::N;
    constexpr uint64_t kRefVec = 16 / sizeof(T);
    __shared__ unsigned long long next_sh[2];
    const uint64_t mv = m / V; // row vectors == vectors per column
    const uint64_t units = (mv + kTallBlock - 1) / kTallBlock;
    const uint64_t cut = (n / kRefVec) * kRefVec;
    const Vec<T>* Av = reinterpret_cast<const Vec<T>*>(A);
    Vec<T>* Cv = reinterpret_cast<Vec<T>*>(c);
    // DYN: first unit static, the rest from the queue (common.cuh dyn_next);
    // otherwise CTAs own balanced contiguous unit ranges.
    const Partition part(units, gridDim.x);
    uint64_t u = DYN ? uint64_t(blockIdx.x) : part.begin(blockIdx.x);
    const uint64_t u_end = DYN ? units : part.begin(blockIdx.x + 1);
    int parity = 0;
    while (u < u_end) {
        if (DYN && threadIdx.x == 0) next_sh[parity ^ 1] = dyn_next(counter, units); // prefetch
        const uint64_t rv = u * kTallBlock + threadIdx.x;
        if (rv < mv) {
            Vec<T> acc = Cv[rv];
            const Vec<T>* col = Av + rv;
            uint64_t j = 0;
            for (; j + kTallUnroll <= cut; j += kTallUnroll) {
                Vec<T> a[kTallUnroll];
#pragma unroll
                for (int k = 0; k < kTallUnroll; ++k) a[k] = ld_stream(col + (j + k) * mv);
#pragma unroll
                for (int k = 0; k < kTallUnroll; ++k) {
                    const T xj = __ldg(x + j + k);
#pragma unroll
                    for (int e = 0; e < V; ++e) acc.v[e] = ref_step(acc.v[e], a[k].v[e], xj, false);
                }
            }
            for (; j < n; ++j) {
                const Vec<T> a = ld_stream(col + j * mv);
                const T xj = __ldg(x + j);
#pragma unroll
                for (int e = 0; e < V; ++e) acc.v[e] = ref_step(acc.v[e], a.v[e], xj, j >= cut);
            }
            Cv[rv] = acc;
        }
        if (DYN) {
            __syncthreads(); // publishes next_sh[parity ^ 1]
            parity ^= 1;
            u = next_sh[parity];
        } else {
            ++u;
        }
    }
}

// Tall and narrow (n < kTallUnroll): the tall kernel keeps only n column
// loads in flight per thread there (2^24 x 4 fp32 ran at 3.6 TB/s).  Here a
// thread owns P = 16 / NC row vectors (NC >= n, a power of two), so P * n
// loads are issued before any is consumed; each row vector still runs its
// own chain over j ascending with the reference's rounding: bitwise gemv_ref
// like the tall kernel.  CTAs own balanced contiguous ranges of P*256-vector
// units.
template <typename T, int NC>
__global__ void __launch_bounds__(kTallBlock, 1)
    gemv_cm_narrow_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                          uint64_t m, uint64_t n) {
    pdl_enter();
    constexpr int V = Vec<T>::N;
    constexpr int P = kTallUnroll / NC;
    constexpr uint64_t kRefVec = 16 / sizeof(T);
    const uint64_t mv = m / V;
    const uint64_t per_unit = uint64_t(kTallBlock) * P;
    const uint64_t units = (mv + per_unit - 1) / per_unit;
    const uint64_t cut = (n / kRefVec) * kRefVec;
    const Vec<T>* Av = reinterpret_cast<const Vec<T>*>(A);
    Vec<T>* Cv = reinterpret_cast<Vec<T>*>(c);
    T xs[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) xs[k] = uint64_t(k) < n ? __ldg(x + k) : T(0);
    const Partition part(units, gridDim.x);
    for (uint64_t u = part.begin(blockIdx.x); u < part.begin(blockIdx.x + 1); ++u) {
        Vec<T> a[P][NC];
        Vec<T> cv[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const uint64_t rv = u * per_unit + uint64_t(p) * kTallBlock + threadIdx.x;
            // c's vector in the same batch as A's: at n = 4 c is a third of
            // the bytes, and loading it only when the sum starts serialised a
            // second round trip (256 MiB of A flushed, tools/ab_shapes.py:
            // fp32 2^24 x 4 78.7 -> 65.1 us, 2^26 x 1 207 -> 123; fp64 2^24 x
            // 4 147 -> 124)
            if (rv < mv) cv[p] = ld_rmw(Cv + rv);
#pragma unroll
            for (int k = 0; k < NC; ++k)
                if (rv < mv && uint64_t(k) < n) a[p][k] = ld_stream(Av + rv + uint64_t(k) * mv);
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const uint64_t rv = u * per_unit + uint64_t(p) * kTallBlock + threadIdx.x;
            if (rv < mv) {
                Vec<T> acc = cv[p];
#pragma unroll
                for (int k = 0; k < NC; ++k)
                    if (uint64_t(k) < n)
#pragma unroll
                        for (int e = 0; e < V; ++e)
                            acc.v[e] = ref_step(acc.v[e], a[p][k].v[e], xs[k], uint64_t(k) >= cut);
                Cv[rv] = acc;
            }
        }
    }
}

// Tall, any m: one row per lane, warps own balanced ranges of 32-row units.
template <typename T>
__global__ void __launch_bounds__(kCmBlock, kCmRowsCtasPerSm)
    gemv_cm_rows_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                        uint64_t m, uint64_t n, uint64_t warps) {
    pdl_enter();
    constexpr uint64_t kRefVec = 16 / sizeof(T);
    const int lane = threadIdx.x & 31;
    const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (gw >= warps) return;
    const uint64_t units = (m + kWarp - 1) / kWarp;
    const Partition part(units, warps);
    const uint64_t cut = (n / kRefVec) * kRefVec;

    for (uint64_t unit = part.begin(gw); unit < part.begin(gw + 1); ++unit) {
        const uint64_t i = unit * kWarp + lane;
        const bool live = i < m;
        const T* a = A + (live ? i : 0);
        T acc = live ? c[i] : T(0);
        uint64_t j = 0;
        for (; j + kCmUnroll <= cut; j += kCmUnroll) {
            T av[kCmUnroll];
#pragma unroll
            for (int k = 0; k < kCmUnroll; ++k) av[k] = live ? __ldcs(a + (j + k) * m) : T(0);
#pragma unroll
            for (int k = 0; k < kCmUnroll; ++k) acc = ref_step(acc, av[k], __ldg(x + j + k), false);
        }
        for (; j < n; ++j) {
            const T av = live ? __ldcs(a + j * m) : T(0);
            acc = ref_step(acc, av, __ldg(x + j), j >= cut);
        }
        if (live) c[i] = acc;
    }
}

// Last CTA of a split launch over one row tile: c[r] += sum over the G column
// parts b (in order) of partials[b*stride + r], r < rows.  Thread (r, q)
// sums parts q, q+Q, ... with 16 loads in flight, then the Q sums per row
// are added in q order; `sm` holds >= blockDim.x entries.
constexpr int kFinalBatch = 32; // partial loads in flight per thread in split_final

template <typename T>
__device__ void split_final(const T* __restrict__ partials, T* __restrict__ c, uint64_t rows,
                            uint64_t stride, unsigned G, T* sm) {
    int block = 32; // largest power of two <= blockDim.x
    while (block * 2 <= int(blockDim.x)) block *= 2;
    int rl = 32;
    while (uint64_t(rl) < rows && rl < block) rl *= 2;
    const int Q = block / rl;
    const int r0 = threadIdx.x % rl, q = threadIdx.x / rl;
    const bool part = int(threadIdx.x) < block;
    for (uint64_t rb = 0; rb < rows; rb += uint64_t(rl)) {
        const uint64_t r = rb + r0;
        T total = T(0);
        if (part && r < rows) {
            for (unsigned b0 = q; b0 < G; b0 += unsigned(kFinalBatch) * Q) {
                T v[kFinalBatch];
#pragma unroll
                for (int e = 0; e < kFinalBatch; ++e) {
                    const unsigned b = b0 + unsigned(e) * Q;
                    v[e] = b < G ? ld_cg(partials + uint64_t(b) * stride + r) : T(0);
                }
#pragma unroll
                for (int e = 0; e < kFinalBatch; ++e)
                    if (b0 + unsigned(e) * Q < G) total = add_rn(total, v[e]);
            }
        }
        __syncthreads(); // sm reuse
        if (part && r < rows) sm[uint64_t(q) * rl + r0] = total;
        __syncthreads();
        if (part && q == 0 && r < rows) {
            T v = sm[r0];
            for (int k = 1; k < Q; ++k) v = add_rn(v, sm[uint64_t(k) * rl + r0]);
            c[r] = add_rn(c[r], v);
        }
    }
}

// Vectorised split kernel (m % V == 0, aligned), 2-D: blockIdx.y picks a row
// tile of mt rows (column stride lda = m), blockIdx.x one of gridDim.x column
// parts (balanced contiguous column ranges).  A thread owns one 32-byte row
// vector (V rows) of the tile for its column lane; row_lanes = pow2 >= mt/V,
// U = 4 256-bit column loads in flight per thread.  Partials per (row tile,
// column part); the last part to finish a row tile (per-tile ticket) adds
// them into c in part order.
template <typename T>
__global__ void __launch_bounds__(kSplitBlock, 1)
    gemv_cm_split_vec_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                             uint64_t m, uint64_t n, uint64_t mt, int row_lanes,
                             T* __restrict__ partials, unsigned* __restrict__ tickets,
                             int external_combine) {
    pdl_enter();
    constexpr int V = Vec<T>::N;
    constexpr int U = 4;
    __shared__ alignas(32) T sm[kSplitBlock * V]; // [col_lanes][mt] <= 1024 * V entries
    __shared__ bool am_last;
    const int tid = threadIdx.x;
    const int col_lanes = kSplitBlock / row_lanes;
    const int rl = tid % row_lanes, cl = tid / row_lanes;
    const uint64_t r0 = uint64_t(blockIdx.y) * mt;
    const uint64_t rows = (m - r0 < mt) ? m - r0 : mt;
    const uint64_t mv = m / V, rows_v = rows / V;
    const bool live = uint64_t(rl) < rows_v;
    const Vec<T>* Av = reinterpret_cast<const Vec<T>*>(A) + r0 / V + (live ? rl : 0);
    const uint64_t tile = uint64_t(col_lanes) * U;
    // column part blockIdx.x: a balanced contiguous range (parts differ by at
    // most one column; whole tiles dealt out grid-stride left parts up to a
    // tile = 7% apart: 4096 x 16384 fp32 had 15 vs 14 tiles per part)
    const Partition cols(n, gridDim.x);
    const uint64_t cb = cols.begin(blockIdx.x), ce = cols.begin(blockIdx.x + 1);

    Vec<T> acc;
#pragma unroll
    for (int e = 0; e < V; ++e) acc.v[e] = T(0);
    for (uint64_t t0 = cb; t0 < ce; t0 += tile) {
        const uint64_t j0 = t0 + cl;
        Vec<T> av[U];
        T xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t j = j0 + uint64_t(u) * col_lanes;
            const bool ok = live && j < ce;
            xv[u] = j < ce ? __ldg(x + j) : T(0);
            if (ok) av[u] = ld_stream(Av + j * mv);
            else
#pragma unroll
                for (int e = 0; e < V; ++e) av[u].v[e] = T(0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < V; ++e) acc.v[e] = fma_rn(av[u].v[e], xv[u], acc.v[e]);
    }
    if (live)
#pragma unroll
        for (int e = 0; e < V; ++e) sm[uint64_t(cl) * rows + uint64_t(rl) * V + e] = acc.v[e];
    __syncthreads();
    T* tile_partials = partials + uint64_t(blockIdx.y) * gridDim.x * mt;
    for (uint64_t r = tid; r < rows; r += kSplitBlock) {
        T v = sm[r];
        for (int q = 1; q < col_lanes; ++q) v = add_rn(v, sm[uint64_t(q) * rows + r]);
        tile_partials[uint64_t(blockIdx.x) * mt + r] = v;
    }
    if (external_combine) return; // gemv_cm_fullcol_combine16_kernel follows (PDL)
    __threadfence();
    __syncthreads();
    if (tid == 0) am_last = atomicAdd(tickets + blockIdx.y, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    split_final(tile_partials, c + r0, rows, mt, gridDim.x, sm);
    if (tid == 0) tickets[blockIdx.y] = 0u;
}

// Bulk-copy split kernel (m < kSplitMaxRows, m % V == 0, aligned).  The
// column tiles are contiguous in a col-major matrix (tc consecutive columns =
// tc*m*s bytes), so one elected producer thread streams each tile into a ring
// of kBulkStages shared-memory stages with a single cp.async.bulk (TMA engine;
// completion counted on an mbarrier), keeping up to 3 x 48 KB per SM in flight
// without spending registers on it (the tile's x slice rides in the same
// stage).  On 256 x 2^20 fp64 back to back: 299.1 us at 3 x 48 KB against
// 311.0 us for the register-load kernel below — the bytes in flight per SM
// are set exactly by the ring, not by register pressure.  16 consumer warps =
// (row-vector lane, column lane) pairs read their 32-byte row vectors from the stage and FMA into
// register accumulators, then free the stage (one arrive per warp).  Tiles go
// to CTAs in grid-stride (sweep) order; the per-row combine is the same as
// the register kernel's: column lanes in smem in order, then the CTA
// partials in CTA order by the last CTA.
constexpr int kBulkConsumerWarps = 16;
constexpr int kBulkConsumers = kBulkConsumerWarps * 32;
constexpr int kBulkThreads = kBulkConsumers + 32; // + 1 producer warp
constexpr unsigned kBulkXBytes = 1024;            // the tile's slice of x rides along
constexpr unsigned kBulkCombineBytes = 16384;     // >= 512*V*s and >= kBulkThreads*s
constexpr unsigned bulk_smem(int stages, unsigned stage_bytes) {
    return stages * (stage_bytes + kBulkXBytes) + kBulkCombineBytes;
}

template <typename T, int kBulkStages, unsigned kBulkStageBytes>
__global__ void __launch_bounds__(kBulkThreads, 1)
    gemv_cm_split_bulk_kernel(const T* __restrict__ A, const T* __restrict__ x,
                              T* __restrict__ c, uint64_t m, uint64_t n, int row_lanes, int tc,
                              uint64_t x_off, T* __restrict__ partials,
                              unsigned* __restrict__ ticket, int x_bulk, int external_combine) {
    pdl_enter();
    constexpr int V = Vec<T>::N;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* stages = reinterpret_cast<T*>(smem_raw);
    constexpr unsigned kBulkStageStride = kBulkStageBytes + kBulkXBytes;
    T* comb = reinterpret_cast<T*>(smem_raw + kBulkStages * kBulkStageStride);
    __shared__ __align__(8) uint64_t full[kBulkStages];
    __shared__ __align__(8) uint64_t empty[kBulkStages];
    __shared__ bool am_last;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t tiles = (n + tc - 1) / tc;
    const uint64_t stage_elems = kBulkStageStride / sizeof(T);
    // x slice right after the tile's tc*m elements (x_off = tc*m): the host
    // picks tc so tile + slice fit the stage, (m + 1) * tc * s <= stride
    const int col_lanes = kBulkConsumers / row_lanes;

    if (tid == 0) {
        for (int s = 0; s < kBulkStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kBulkConsumerWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == kBulkConsumerWarps) {
        if (lane == 0) { // producer
            const uint64_t pol = l2_evict_first_policy();
            uint64_t it = 0;
            for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
                const int st = int(it % kBulkStages);
                const unsigned use = unsigned(it / kBulkStages);
                if (use > 0) mbar_wait(&empty[st], (use - 1) & 1u);
                const uint64_t col0 = t * tc;
                const uint64_t cols = (n - col0 < uint64_t(tc)) ? n - col0 : uint64_t(tc);
                const unsigned bytes = unsigned(cols * m * sizeof(T));
                // x slice: a full tile's is a multiple of 16 B (tc is) and rides
                // in the stage when it fits the slot (tc * s <= kBulkXBytes); a
                // ragged last tile's, or a wider one's, is read with plain loads
                // (an x that is not 16-byte aligned cannot be bulk-copied: its
                // slices are read with plain loads, x_bulk = 0)
                const unsigned xbytes =
                    (x_bulk && cols == uint64_t(tc)) ? unsigned(cols * sizeof(T)) : 0u;
                mbar_arrive_expect_tx(&full[st], bytes + xbytes);
                bulk_g2s(stages + st * stage_elems, A + col0 * m, bytes, &full[st], pol);
                if (xbytes) bulk_g2s(stages + st * stage_elems + x_off, x + col0, xbytes, &full[st], pol);
            }
        }
    } else {
        const int rl = tid % row_lanes, cl = tid / row_lanes;
        const bool live = uint64_t(rl) * V < m;
        Vec<T> acc;
#pragma unroll
        for (int e = 0; e < V; ++e) acc.v[e] = T(0);
        uint64_t it = 0;
        for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
            const int st = int(it % kBulkStages);
            mbar_wait(&full[st], unsigned(it / kBulkStages) & 1u);
            const uint64_t col0 = t * tc;
            const int cols = int((n - col0 < uint64_t(tc)) ? n - col0 : uint64_t(tc));
            const T* sb = stages + st * stage_elems;
            if (live) {
                for (int j = cl; j < cols; j += col_lanes) {
                    const Vec<T> a = *reinterpret_cast<const Vec<T>*>(sb + uint64_t(j) * m + uint64_t(rl) * V);
                    const T xj = (x_bulk && cols == tc) ? sb[x_off + j] : __ldg(x + col0 + j);
#pragma unroll
                    for (int e = 0; e < V; ++e) acc.v[e] = fma_rn(a.v[e], xj, acc.v[e]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        if (live)
#pragma unroll
            for (int e = 0; e < V; ++e) comb[uint64_t(cl) * m + uint64_t(rl) * V + e] = acc.v[e];
    }
    __syncthreads();
    for (uint64_t r = tid; r < m; r += blockDim.x) {
        T v = comb[r];
        for (int q = 1; q < col_lanes; ++q) v = add_rn(v, comb[uint64_t(q) * m + r]);
        partials[uint64_t(blockIdx.x) * m + r] = v;
    }
    if (external_combine) return; // gemv_cm_fullcol_combine16_kernel follows (PDL)
    __threadfence();
    __syncthreads();
    if (tid == 0) am_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    split_final(partials, c, m, m, gridDim.x, comb);
    if (tid == 0) *ticket = 0u;
}

// Bulk-copy split kernel for short-wide matrices whose rows do not form
// 32-byte vectors (m % V != 0, or A only 16-byte aligned): the column tiles
// are still contiguous, so the same single-producer bulk ring streams them
// (tc a multiple of 16/s keeps every full tile and its x slice whole 16-byte
// units; a ragged last tile's odd tail is read from global memory).
// Consumers read scalars: thread (rl, cl) owns rows rl + k*row_lanes (k <
// RPT = ceil(m / 512), row_lanes = min(m, 512)) and columns j = cl, cl + col_lanes, ...
// of each tile, in order (rpt chosen per m, bulk_scalar_rpt).  The combine
// is the vector kernel's.  Short-wide odd m, ~2 GiB, flushed: fp32 m = 255 /
// 257 / 1001 in 94 / 90 / 100 us (5.4-6.0 TB/s); the 2-D scalar split kernel
// below took 141 / 254 / 150 us.
template <typename T, int kBulkStages, unsigned kBulkStageBytes, int RPT>
__global__ void __launch_bounds__(kBulkThreads, 1)
    gemv_cm_split_bulk_scalar_kernel(const T* __restrict__ A, const T* __restrict__ x,
                                     T* __restrict__ c, uint64_t m, uint64_t n, int row_lanes,
                                     int tc, uint64_t x_off, int x_bulk, T* __restrict__ partials,
                                     unsigned* __restrict__ ticket, int a_off, int external_combine) {
    pdl_enter();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* stages = reinterpret_cast<T*>(smem_raw);
    constexpr unsigned kBulkStageStride = kBulkStageBytes + kBulkXBytes;
    T* comb = reinterpret_cast<T*>(smem_raw + kBulkStages * kBulkStageStride);
    __shared__ __align__(8) uint64_t full[kBulkStages];
    __shared__ __align__(8) uint64_t empty[kBulkStages];
    __shared__ bool am_last;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint64_t tiles = (n + tc - 1) / tc;
    const uint64_t stage_elems = kBulkStageStride / sizeof(T);
    const int col_lanes = kBulkConsumers / row_lanes;

    if (tid == 0) {
        for (int s = 0; s < kBulkStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kBulkConsumerWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == kBulkConsumerWarps) {
        if (lane == 0) { // producer
            const uint64_t pol = l2_evict_first_policy();
            uint64_t it = 0;
            for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
                const int st = int(it % kBulkStages);
                const unsigned use = unsigned(it / kBulkStages);
                if (use > 0) mbar_wait(&empty[st], (use - 1) & 1u);
                const uint64_t col0 = t * tc;
                const uint64_t cols = (n - col0 < uint64_t(tc)) ? n - col0 : uint64_t(tc);
                // a_off > 0 (A not 16-byte aligned): copy from the 16-byte boundary
                // a_off elements before the tile; a full tile is rounded up to
                // whole 16-byte units, so a copy may start / end inside a 16-byte
                // segment of A's neighbours (bytes never read by the consumers)
                const uint64_t span = (cols * m + uint64_t(a_off)) * sizeof(T);
                const unsigned bytes = cols == uint64_t(tc) ? unsigned((span + 15) & ~uint64_t(15))
                                                            : unsigned(span & ~uint64_t(15));
                const unsigned xbytes =
                    (x_bulk && cols == uint64_t(tc)) ? unsigned(cols * sizeof(T)) : 0u;
                mbar_arrive_expect_tx(&full[st], bytes + xbytes);
                if (bytes) bulk_g2s(stages + st * stage_elems, A + col0 * m - a_off, bytes, &full[st], pol);
                if (xbytes) bulk_g2s(stages + st * stage_elems + x_off, x + col0, xbytes, &full[st], pol);
            }
        }
    } else {
        const int rl = tid % row_lanes, cl = tid / row_lanes;
        const bool live = cl < col_lanes;
        const unsigned mm = unsigned(m); // < kSplitMaxRows: 32-bit smem indexing
        bool rok[RPT];
#pragma unroll
        for (int k = 0; k < RPT; ++k) rok[k] = unsigned(rl) + unsigned(k * row_lanes) < mm;
        T acc[RPT];
#pragma unroll
        for (int k = 0; k < RPT; ++k) acc[k] = T(0);
        uint64_t it = 0;
        for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
            const int st = int(it % kBulkStages);
            mbar_wait(&full[st], unsigned(it / kBulkStages) & 1u);
            const uint64_t col0 = t * tc;
            const int cols = int((n - col0 < uint64_t(tc)) ? n - col0 : uint64_t(tc));
            const T* sb = stages + st * stage_elems + a_off;
            if (live) {
                if (cols == tc) { // full tile: everything is in the stage
                    const T* xs = x_bulk ? stages + st * stage_elems + x_off : nullptr;
                    unsigned e = unsigned(cl) * mm + unsigned(rl);
                    const unsigned step = unsigned(col_lanes) * mm;
#pragma unroll 4
                    for (int j = cl; j < cols; j += col_lanes, e += step) {
                        const T xj = xs ? xs[j] : __ldg(x + col0 + j);
#pragma unroll
                        for (int k = 0; k < RPT; ++k)
                            if (rok[k]) acc[k] = fma_rn(sb[e + unsigned(k * row_lanes)], xj, acc[k]);
                    }
                } else { // ragged last tile: its odd tail was not bulk-copied
                    // elements of the tile the producer copied: the whole 16-byte
                    // units from the boundary below A, less the a_off lead-in (none
                    // at all when the tile ends inside its first 16 bytes)
                    const uint64_t copied =
                        ((uint64_t(cols) * m + uint64_t(a_off)) * sizeof(T) & ~uint64_t(15)) /
                        sizeof(T);
                    const uint64_t in_smem = copied > uint64_t(a_off) ? copied - uint64_t(a_off) : 0;
                    for (int j = cl; j < cols; j += col_lanes) {
                        const T xj = __ldg(x + col0 + j);
#pragma unroll
                        for (int k = 0; k < RPT; ++k)
                            if (rok[k]) {
                                const uint64_t e = uint64_t(j) * m + rl + uint64_t(k) * row_lanes;
                                const T a = e < in_smem ? sb[e] : __ldg(A + col0 * m + e);
                                acc[k] = fma_rn(a, xj, acc[k]);
                            }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        if (live)
#pragma unroll
            for (int k = 0; k < RPT; ++k)
                if (rok[k]) comb[uint64_t(cl) * m + rl + uint64_t(k) * row_lanes] = acc[k];
    }
    __syncthreads();
    for (uint64_t r = tid; r < m; r += blockDim.x) {
        T v = comb[r];
        for (int q = 1; q < col_lanes; ++q) v = add_rn(v, comb[uint64_t(q) * m + r]);
        partials[uint64_t(blockIdx.x) * m + r] = v;
    }
    if (external_combine) return; // gemv_cm_fullcol_combine_kernel follows (PDL)
    __threadfence();
    __syncthreads();
    if (tid == 0) am_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    split_final(partials, c, m, m, gridDim.x, comb);
    if (tid == 0) *ticket = 0u;
}

// Full-column bulk ring for columns that are not 32-byte vectors (odd m, or A
// off a 32-byte boundary), 1024 <= m with one column per stage: a column is
// contiguous, so the producer lane copies column j (from the 16-byte boundary
// at or below its first element, rounded up to whole 16-byte units) into a
// ring stage with one cp.async.bulk; CTAs take columns grid-stride (the whole
// GPU sweeps A front to back together, as the aligned full-column sweep
// does).  Consumer thread t owns rows t, t + 512, ... (RPT of them) across all
// columns and reads its scalars from the stage at the column's offset, so no
// realignment shuffles are needed; each CTA writes its partial (row stride
// mp = m rounded up to 16 bytes) and gemv_cm_fullcol_combine16_kernel sums
// them.  Replaces the realigning 2-D split (warp shuffles per column, 128
// registers, one 512-thread CTA per SM, latency-bound at 4.6 TB/s fp32).
constexpr int kColBulkStages = 3;
constexpr unsigned kColBulkStageBytes = 49152;      // stage size for most m
constexpr unsigned kColBulkBigStageBytes = 73728;   // 3 x 72 KB: 2 columns of fp32 m <= 9215,
                                                    // or one of m <= 18424
constexpr int kColBulkMaxTc = 12; // columns per stage: m >= 1024 fits <= 11 fp32 columns

template <typename T, int RPT, unsigned SB>
__global__ void __launch_bounds__(kBulkThreads, 1)
    gemv_cm_colbulk_kernel(const T* __restrict__ A, const T* __restrict__ x, uint64_t m, uint64_t n,
                           uint64_t mp, int tc, T* __restrict__ partials) {
    pdl_enter();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* stages = reinterpret_cast<T*>(smem_raw);
    constexpr uint64_t kStageElems = SB / sizeof(T);
    constexpr uint64_t q = 16 / sizeof(T); // elements per 16-byte unit
    constexpr unsigned ns = kColBulkStages;
    __shared__ __align__(8) uint64_t full[kColBulkStages];
    __shared__ __align__(8) uint64_t empty[kColBulkStages];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // A's element offset from the 16-byte boundary below it
    const uint64_t a_base = (reinterpret_cast<uintptr_t>(A) & 15u) / sizeof(T);
    const uint64_t tiles = (n + uint64_t(tc) - 1) / uint64_t(tc); // tc consecutive columns per stage
    if (tid == 0) {
        for (int st = 0; st < int(ns); ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], kBulkConsumerWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == kBulkConsumerWarps) {
        if (lane == 0) { // producer: column j from the 16-byte boundary at or below it
            const uint64_t pol = l2_evict_first_policy();
            uint64_t it = 0;
            for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
                const int st = int(it % unsigned(ns));
                const unsigned use = unsigned(it / unsigned(ns));
                if (use > 0) mbar_wait(&empty[st], (use - 1) & 1u);
                const uint64_t j0 = t * uint64_t(tc);
                const uint64_t cols = n - j0 < uint64_t(tc) ? n - j0 : uint64_t(tc);
                const uint64_t off = (a_base + j0 * m) % q;
                // whole 16-byte units; the last one may end inside the next
                // column (or past A's end within that same 16-byte segment:
                // bytes never read by the consumers, no page can be crossed)
                const unsigned bytes = unsigned(((off + cols * m) * sizeof(T) + 15) & ~uint64_t(15));
                mbar_arrive_expect_tx(&full[st], bytes);
                bulk_g2s(stages + st * kStageElems, A + j0 * m - off, bytes, &full[st], pol);
            }
        }
    } else {
        T acc[RPT];
#pragma unroll
        for (int k = 0; k < RPT; ++k) acc[k] = T(0);
        uint64_t it = 0;
        for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
            const int st = int(it % unsigned(ns));
            const uint64_t j0 = t * uint64_t(tc);
            const int cols = int(n - j0 < uint64_t(tc) ? n - j0 : uint64_t(tc));
            T xj = __ldg(x + j0); // the first column's x before the wait
            mbar_wait(&full[st], unsigned(it / unsigned(ns)) & 1u);
            const T* col = stages + st * kStageElems + (a_base + j0 * m) % q;
            for (int cc = 0; cc < cols; ++cc, col += m) {
                const T xn = cc + 1 < cols ? __ldg(x + j0 + cc + 1) : T(0); // the next one's
#pragma unroll
                for (int k = 0; k < RPT; ++k) {
                    const unsigned r = unsigned(tid) + unsigned(k) * kBulkConsumers;
                    if (r < unsigned(m)) acc[k] = fma_rn(col[r], xj, acc[k]);
                }
                xj = xn;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        T* out = partials + uint64_t(blockIdx.x) * mp;
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const uint64_t r = uint64_t(tid) + uint64_t(k) * kBulkConsumers;
            if (r < m) out[r] = acc[k];
        }
    }
}

// Full-column sweep (aligned mid-size m, m/V <= 1024: fp32 m <= 8192, fp64 m <= 4096).
// The 2-D split reads a fixed 1 KB row slot of every column per CTA and its
// CTAs finish up to ~10 us apart on a 50 us launch (profiles/r02_cm_mid.md).
// Here a CTA owns whole columns: thread (row-vector lane rl, column lane cl)
// holds one 32-byte accumulator of rows 8rl.. (fp32) and walks columns
// j = blockIdx.x * col_lanes + cl, then + gridDim.x * col_lanes, ... — all
// CTAs sweep the matrix front to back together, as the row-major sweep does,
// with U = 2 columns in flight per thread.  The column lanes are summed in
// lane order in shared memory and the CTA's m-long partial goes to
// partials[blockIdx.x]; gemv_cm_fullcol_combine_kernel (launched next, PDL)
// adds the partials per row in CTA order into c.  The per-row order depends
// only on (m, n, grid), so the result is bitwise reproducible.  256 MiB fp32,
// flushed (tools/cmlab.py): 4096 x 16384 5.24 -> 5.67 TB/s, 2048 x 32768 5.24
// -> 5.54, 1024 x 65536 5.24 -> 5.58.
constexpr int kFullColU = 2;

template <typename T>
__global__ void __launch_bounds__(1024, 1)
    gemv_cm_fullcol_kernel(const T* __restrict__ A, const T* __restrict__ x, uint64_t m, uint64_t n,
                           int row_lanes, T* __restrict__ partials) {
    pdl_enter();
    constexpr int V = Vec<T>::N;
    __shared__ alignas(32) unsigned char raw[32768]; // blockDim.x * V values (<= 32 KB)
    T* sm = reinterpret_cast<T*>(raw);
    const int tid = threadIdx.x;
    const int col_lanes = int(blockDim.x) / row_lanes;
    const int rl = tid % row_lanes, cl = tid / row_lanes;
    const uint64_t mv = m / V;
    const bool live = uint64_t(rl) < mv;
    const Vec<T>* Av = reinterpret_cast<const Vec<T>*>(A) + (live ? rl : 0);
    const uint64_t jstep = uint64_t(gridDim.x) * col_lanes;
    Vec<T> acc;
#pragma unroll
    for (int e = 0; e < V; ++e) acc.v[e] = T(0);
    for (uint64_t j0 = uint64_t(blockIdx.x) * col_lanes + cl; j0 < n; j0 += jstep * kFullColU) {
        Vec<T> a[kFullColU];
        T xv[kFullColU];
#pragma unroll
        for (int u = 0; u < kFullColU; ++u) {
            const uint64_t j = j0 + uint64_t(u) * jstep;
            const bool ok = j < n;
            xv[u] = ok ? __ldg(x + j) : T(0);
            if (ok && live) a[u] = ld_stream(Av + j * mv);
            else
#pragma unroll
                for (int e = 0; e < V; ++e) a[u].v[e] = T(0);
        }
#pragma unroll
        for (int u = 0; u < kFullColU; ++u)
#pragma unroll
            for (int e = 0; e < V; ++e) acc.v[e] = fma_rn(a[u].v[e], xv[u], acc.v[e]);
    }
    T* out = partials + uint64_t(blockIdx.x) * m;
    if (col_lanes == 1) {
        if (live) *reinterpret_cast<Vec<T>*>(out + uint64_t(rl) * V) = acc;
        return;
    }
    if (live)
#pragma unroll
        for (int e = 0; e < V; ++e) sm[(uint64_t(cl) * row_lanes + rl) * V + e] = acc.v[e];
    __syncthreads();
    for (uint64_t i = tid; i < m; i += blockDim.x) {
        T t = sm[i];
        for (int q = 1; q < col_lanes; ++q) t = add_rn(t, sm[uint64_t(q) * row_lanes * V + i]);
        out[i] = t;
    }
}

// c[r] += the `parts` partials of row r in part order: thread (row r of 32,
// group g of 32) sums parts g, g + 32, ... , then the 32 group sums of a row
// are added by one warp in a fixed shuffle tree.  Up to 320 parts (every grid the sweep uses) all of a thread's
// loads are issued as one batch, so the chain after the sweep is one L2 round
// trip; c's line is prefetched into L2 before the wait.
template <typename T>
__global__ void __launch_bounds__(1024, 1)
    gemv_cm_fullcol_combine_kernel(const T* __restrict__ partials, unsigned parts, uint64_t m,
                                   T* __restrict__ c) {
    pdl_trigger();
    const int rloc = threadIdx.x & 31, g = threadIdx.x >> 5;
    const uint64_t row = uint64_t(blockIdx.x) * 32 + rloc;
    // L2 prefetch only before the wait (common.cuh: nothing reaches the SM)
    if (threadIdx.x < 2 && uint64_t(blockIdx.x) * 32 + threadIdx.x * 31 < m)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(c + uint64_t(blockIdx.x) * 32 + threadIdx.x * 31));
    pdl_wait();
    __shared__ T red[32][33];
    T s = T(0);
    if (row < m) {
        constexpr int K = 10;
        unsigned p = unsigned(g);
        for (; p + unsigned(K - 1) * 32u < parts; p += unsigned(K) * 32u) {
            T v[K];
#pragma unroll
            for (int k = 0; k < K; ++k) v[k] = ld_cg(partials + uint64_t(p + k * 32u) * m + row);
#pragma unroll
            for (int k = 0; k < K; ++k) s = add_rn(s, v[k]);
        }
        if (p < parts) { // the < K remaining parts of this group, one batch
            T v[K];
#pragma unroll
            for (int k = 0; k < K; ++k)
                v[k] = p + k * 32u < parts ? ld_cg(partials + uint64_t(p + k * 32u) * m + row) : T(0);
#pragma unroll
            for (int k = 0; k < K; ++k)
                if (p + k * 32u < parts) s = add_rn(s, v[k]);
        }
    }
    red[g][rloc] = s;
    __syncthreads();
    // warp g finishes row g of the 32: lane k holds group k's sum, fixed
    // shuffle-down tree, lane 0 adds it to c
    const uint64_t row_w = uint64_t(blockIdx.x) * 32 + g;
    T t = red[rloc][g];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t = add_rn(t, __shfl_down_sync(0xffffffffu, t, off));
    if (rloc == 0 && row_w < m) c[row_w] = add_rn(c[row_w], t);
}

// Full-column sweep for 1024 < m/V <= 2048 (fp32 m <= 16384, fp64 m <= 8192):
// 1024 threads, thread t owns row vectors t and t + 1024 of every column, one
// column per CTA at a time (U = 2 columns in flight: 4 x 32 bytes per thread),
// columns dealt grid-stride; the CTA's m-long partial goes to
// partials[blockIdx.x] and gemv_cm_fullcol_combine16_kernel follows (PDL).
// fp32 16384 x 4096 in ncu: 45.9 us, SM active min / max 73k / 79k cycles,
// against the 2-D split's 51.1 us (profiles/r02_cm_mid.md).
template <typename T>
__global__ void __launch_bounds__(1024, 1)
    gemv_cm_fullcol2_kernel(const T* __restrict__ A, const T* __restrict__ x, uint64_t m, uint64_t n,
                            T* __restrict__ partials) {
    pdl_enter();
    constexpr int V = Vec<T>::N;
    const int tid = threadIdx.x;
    const uint64_t mv = m / V;
    const bool live1 = uint64_t(tid) + 1024u < mv;
    const Vec<T>* Av = reinterpret_cast<const Vec<T>*>(A) + tid;
    const uint64_t jstep = gridDim.x;
    Vec<T> acc0, acc1;
#pragma unroll
    for (int e = 0; e < V; ++e) acc0.v[e] = acc1.v[e] = T(0);
    for (uint64_t j0 = blockIdx.x; j0 < n; j0 += jstep * kFullColU) {
        Vec<T> a0[kFullColU], a1[kFullColU];
        T xv[kFullColU];
#pragma unroll
        for (int u = 0; u < kFullColU; ++u) {
            const uint64_t j = j0 + uint64_t(u) * jstep;
            const bool ok = j < n;
            xv[u] = ok ? __ldg(x + j) : T(0);
            if (ok) a0[u] = ld_stream(Av + j * mv);
            else
#pragma unroll
                for (int e = 0; e < V; ++e) a0[u].v[e] = T(0);
            if (ok && live1) a1[u] = ld_stream(Av + j * mv + 1024u);
            else
#pragma unroll
                for (int e = 0; e < V; ++e) a1[u].v[e] = T(0);
        }
#pragma unroll
        for (int u = 0; u < kFullColU; ++u)
#pragma unroll
            for (int e = 0; e < V; ++e) {
                acc0.v[e] = fma_rn(a0[u].v[e], xv[u], acc0.v[e]);
                acc1.v[e] = fma_rn(a1[u].v[e], xv[u], acc1.v[e]);
            }
    }
    Vec<T>* out = reinterpret_cast<Vec<T>*>(partials + uint64_t(blockIdx.x) * m);
    out[tid] = acc0;
    if (live1) out[tid + 1024] = acc1;
}

// Combine for many rows (m % (16 / s) == 0): thread (16-byte row group q,
// part group g of kC16G) sums parts g, g + kC16G, ... (up to kC16K in one
// batch of 16-byte L2 loads), then the kC16G group sums of a row are added
// by kC16G lanes of one warp in a fixed shuffle tree.  256-thread CTAs of 16
// row groups: m = 16384 fp32 is 256 CTAs, one wave with room to spare (the
// 1024-thread combine runs such m in 3.5 waves of one CTA per SM).
constexpr int kC16G = 16;
constexpr int kC16K = 10; // parts <= 160
template <typename T> struct alignas(16) Q16 {
    T v[16 / sizeof(T)];
};
__device__ __forceinline__ Q16<float> ld_cg16(const Q16<float>* p) {
    const float4 t = __ldcg(reinterpret_cast<const float4*>(p));
    return Q16<float>{{t.x, t.y, t.z, t.w}};
}
__device__ __forceinline__ Q16<double> ld_cg16(const Q16<double>* p) {
    const double2 t = __ldcg(reinterpret_cast<const double2*>(p));
    return Q16<double>{{t.x, t.y}};
}
template <typename T>
__global__ void __launch_bounds__(256)
    gemv_cm_fullcol_combine16_kernel(const T* __restrict__ partials, unsigned parts, uint64_t m,
                                     uint64_t mt, T* __restrict__ c) {
    pdl_trigger();
    constexpr int E = 16 / int(sizeof(T)); // rows per 16-byte group
    constexpr int QG = 256 / kC16G;        // row groups per CTA
    constexpr int R = QG * E;              // rows per CTA
    const uint64_t mq = (m + E - 1) / E; // the last group may run past m (rows >= m are not stored)
    const uint64_t q0 = uint64_t(blockIdx.x) * QG;
    if (threadIdx.x < 2) { // c's lines, before the wait (L2 prefetch only)
        const uint64_t last = (q0 + QG < mq ? q0 + QG : mq) * E - 1;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(c + (threadIdx.x ? last : q0 * E)));
    }
    pdl_wait();
    __shared__ T red[kC16G][R + 1];
    const int ql = threadIdx.x % QG, g = threadIdx.x / QG;
    const uint64_t q = q0 + ql;
    T s[E];
#pragma unroll
    for (int e = 0; e < E; ++e) s[e] = T(0);
    if (q < mq) {
        // row tiles of mt rows (mt % E == 0): tile t's parts at (t * parts + p) * mt
        const uint64_t row = q * E, tile = row / mt;
        const uint64_t mqt = mt / E; // 16-byte groups per part row
        const Q16<T>* src = reinterpret_cast<const Q16<T>*>(partials + tile * parts * mt + (row - tile * mt));
        for (unsigned p = unsigned(g); p < parts; p += unsigned(kC16K * kC16G)) {
            Q16<T> v[kC16K];
#pragma unroll
            for (int k = 0; k < kC16K; ++k)
                if (p + k * kC16G < parts) v[k] = ld_cg16(src + uint64_t(p + k * kC16G) * mqt);
#pragma unroll
            for (int k = 0; k < kC16K; ++k)
                if (p + k * kC16G < parts)
#pragma unroll
                    for (int e = 0; e < E; ++e) s[e] = add_rn(s[e], v[k].v[e]);
        }
    }
#pragma unroll
    for (int e = 0; e < E; ++e) red[g][ql * E + e] = s[e];
    __syncthreads();
    // 8 warps x 2 half-warps: half-warp h finishes rows h, h + 16, ...; lane
    // k of a half-warp holds group k's sum, fixed shuffle-down tree
    const int lane = threadIdx.x & 31, hw = (threadIdx.x >> 5) * 2 + (lane >> 4), k = lane & 15;
    for (int r = hw; r < R; r += 16) {
        T t = red[k][r];
#pragma unroll
        for (int off = kC16G / 2; off > 0; off >>= 1) t = add_rn(t, __shfl_down_sync(0xffffffffu, t, off, 16));
        const uint64_t row = q0 * E + uint64_t(r);
        if (k == 0 && row < m) c[row] = add_rn(c[row], t);
    }
}

// Scalar split kernel (any m, any alignment), 2-D like the vector one: row
// tile blockIdx.y of mt rows, column part blockIdx.x.  Thread layout
// row_lanes x col_lanes = kSplitBlock, row_lanes a power of two >=
// min(mt, kSplitBlock); each thread accumulates RPT rows of the tile
// (r = row_lane + k*row_lanes).
template <typename T, int RPT>
__global__ void __launch_bounds__(kSplitBlock, 1)
    gemv_cm_split_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                         uint64_t m, uint64_t n, uint64_t mt, int row_lanes,
                         T* __restrict__ partials, unsigned* __restrict__ tickets,
                         int external_combine) {
    pdl_enter();
    extern __shared__ unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw); // [col_lanes][rows], >= kSplitBlock entries
    __shared__ bool am_last;
    const int tid = threadIdx.x;
    const int col_lanes = kSplitBlock / row_lanes;
    const int rl = tid % row_lanes, cl = tid / row_lanes;
    constexpr int kSplitU = split_u<T>();
    const uint64_t r0 = uint64_t(blockIdx.y) * mt;
    const uint64_t rows = (m - r0 < mt) ? m - r0 : mt;
    const uint64_t tile = uint64_t(col_lanes) * kSplitU;
    const uint64_t tiles = (n + tile - 1) / tile;
    const T* At = A + r0;

    T acc[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) acc[k] = T(0);

    for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const uint64_t j0 = t * tile + cl;
        T av[kSplitU][RPT];
        T xv[kSplitU];
#pragma unroll
        for (int u = 0; u < kSplitU; ++u) {
            const uint64_t j = j0 + uint64_t(u) * col_lanes;
            const bool ok = j < n;
            xv[u] = ok ? __ldg(x + j) : T(0);
            const T* col = At + (ok ? j : 0) * m;
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const uint64_t r = uint64_t(rl) + uint64_t(k) * row_lanes;
                av[u][k] = (ok && r < rows) ? __ldcs(col + r) : T(0);
            }
        }
#pragma unroll
        for (int u = 0; u < kSplitU; ++u)
#pragma unroll
            for (int k = 0; k < RPT; ++k) acc[k] = fma_rn(av[u][k], xv[u], acc[k]);
    }

    // column lanes -> partial of this (row tile, column part), fixed order
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const uint64_t r = uint64_t(rl) + uint64_t(k) * row_lanes;
        if (r < rows) sm[uint64_t(cl) * rows + r] = acc[k];
    }
    __syncthreads();
    T* tile_partials = partials + uint64_t(blockIdx.y) * gridDim.x * mt;
    for (uint64_t r = tid; r < rows; r += kSplitBlock) {
        T v = sm[r];
        for (int q = 1; q < col_lanes; ++q) v = add_rn(v, sm[uint64_t(q) * rows + r]);
        tile_partials[uint64_t(blockIdx.x) * mt + r] = v;
    }
    if (external_combine) return; // gemv_cm_fullcol_combine16_kernel follows (PDL)
    __threadfence();
    __syncthreads();
    if (tid == 0) am_last = atomicAdd(tickets + blockIdx.y, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    split_final(tile_partials, c + r0, rows, mt, gridDim.x, sm);
    if (tid == 0) tickets[blockIdx.y] = 0u;
}

// Realigning split kernel: col-major A whose columns are not 32-byte aligned
// (odd m, or A offset from a 32-byte boundary), m >= 1024.  Same 2-D split
// as gemv_cm_split_vec_kernel, but a column segment of a warp starts at an
// arbitrary element: the warp loads the 32 ALIGNED 32-byte vectors that cover
// it (one 256-bit load per lane), takes its right neighbour's vector with
// V shuffles, and every lane < 31 extracts its V rows at the column's shift
// (warp-uniform, a switch over V cases).  A warp therefore owns 31 * V rows
// (lane 31 only feeds lane 30; its vector is re-read by the next warp from
// L2), and every DRAM byte still moves once in a 256-bit load.  The 2-D
// scalar split it replaces read 4 bytes per load (8192^2 fp32 offset by one
// element: 87 us, 3.1 TB/s).  Thread layout: warp w = (column lane cl, row
// warp rw), RW row warps x CL = 32 / RW column lanes; U columns in flight.
constexpr int kRealignBlock = 512; // 1 CTA per SM: 128 registers per thread
constexpr int kRealignU = 8;      // 256-bit column loads in flight per thread (128 KB per SM)

// acc[e] += x * (element SH + e of the 2V-element window own ++ nb), for the
// lane's first `valid` rows (all V when valid >= V)
template <typename T, int SH>
__device__ __forceinline__ void realign_fma(const Vec<T>& own, const Vec<T>& nb, T xv, int64_t valid,
                                            Vec<T>& acc) {
    constexpr int V = Vec<T>::N;
#pragma unroll
    for (int e = 0; e < V; ++e) {
        const T a = (SH + e < V) ? own.v[(SH + e) % V] : nb.v[(SH + e) % V];
        if (valid >= V || e < valid) acc.v[e] = fma_rn(a, xv, acc.v[e]);
    }
}

template <typename T>
__device__ __forceinline__ void realign_fma(const Vec<T>& own, const Vec<T>& nb, int sh, T xv,
                                            int64_t valid, Vec<T>& acc) {
    switch (sh) {
    case 0: realign_fma<T, 0>(own, nb, xv, valid, acc); break;
    case 1: realign_fma<T, 1>(own, nb, xv, valid, acc); break;
    case 2: realign_fma<T, 2>(own, nb, xv, valid, acc); break;
    case 3: realign_fma<T, 3>(own, nb, xv, valid, acc); break;
    case 4: if constexpr (Vec<T>::N > 4) realign_fma<T, 4 % Vec<T>::N>(own, nb, xv, valid, acc); break;
    case 5: if constexpr (Vec<T>::N > 5) realign_fma<T, 5 % Vec<T>::N>(own, nb, xv, valid, acc); break;
    case 6: if constexpr (Vec<T>::N > 6) realign_fma<T, 6 % Vec<T>::N>(own, nb, xv, valid, acc); break;
    default: if constexpr (Vec<T>::N > 7) realign_fma<T, 7 % Vec<T>::N>(own, nb, xv, valid, acc); break;
    }
}

template <typename T>
__global__ void __launch_bounds__(kRealignBlock, 1)
    gemv_cm_split_realign_kernel(const T* __restrict__ A, const T* __restrict__ x,
                                 T* __restrict__ c, uint64_t m, uint64_t n, uint64_t mt, int RW,
                                 T* __restrict__ partials, unsigned* __restrict__ tickets,
                                 int external_combine) {
    pdl_enter();
    constexpr int V = Vec<T>::N;
    constexpr int U = kRealignU;
    constexpr int LR = 31 * V; // rows per warp
    extern __shared__ unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw); // [CL][rows]
    __shared__ bool am_last;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int CL = (kRealignBlock / 32) / RW;
    const int rw = wid % RW, cl = wid / RW;
    const uint64_t r0 = uint64_t(blockIdx.y) * mt;
    const uint64_t rows = (m - r0 < mt) ? m - r0 : mt;
    const uint64_t wr0 = uint64_t(rw) * LR; // the warp's first row in the tile
    const bool warp_live = wr0 < rows;
    // rows of this lane: wr0 + lane*V + e, valid when < rows (lane < 31)
    const int64_t my_rows = lane < 31 ? int64_t(rows) - int64_t(wr0 + uint64_t(lane) * V) : 0;
    const uintptr_t abase = reinterpret_cast<uintptr_t>(A);
    const uint64_t a0 = (abase & 31u) / sizeof(T); // A's element offset from a 32-byte boundary
    const Vec<T>* Av = reinterpret_cast<const Vec<T>*>(abase - a0 * sizeof(T));
    // Aligned vectors touching A.  The first and last may straddle A's ends: their
    // bytes outside A are read but never used (the realign window and the row
    // mask exclude them).  Such a read stays inside a 32-byte-aligned sector that
    // holds bytes of A, so it can never cross into another page; checking every
    // load instead cost 7% (8193 x 8192 fp32: 57.3 -> 61.4 us), and moving the
    // check to a warp-uniform edge test did not recover it.
    const uint64_t total_v = (a0 + m * n + V - 1) / V;
    const uint64_t tile = uint64_t(CL) * U;
    const uint64_t tiles = (n + tile - 1) / tile;

    Vec<T> acc;
#pragma unroll
    for (int e = 0; e < V; ++e) acc.v[e] = T(0);
    if (warp_live) {
        for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            const uint64_t j0 = t * tile + cl;
            const uint64_t g0 = a0 + j0 * m + r0 + wr0; // element index from the aligned base
            Vec<T> own[U];
            T xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t j = j0 + uint64_t(u) * CL;
                const uint64_t v = (g0 + uint64_t(u) * CL * m) / V + uint64_t(lane);
                xv[u] = j < n ? __ldg(x + j) : T(0);
                if (j < n && v < total_v) own[u] = ld_stream(Av + v);
                else
#pragma unroll
                    for (int e = 0; e < V; ++e) own[u].v[e] = T(0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                Vec<T> nb;
#pragma unroll
                for (int e = 0; e < V; ++e) nb.v[e] = __shfl_down_sync(0xffffffffu, own[u].v[e], 1);
                const int sh = int((g0 + uint64_t(u) * CL * m) % V); // warp-uniform
                realign_fma(own[u], nb, sh, xv[u], my_rows, acc);
            }
        }
    }
    // column lanes -> partial of this (row tile, column part), fixed order
    if (warp_live && lane < 31)
#pragma unroll
        for (int e = 0; e < V; ++e)
            if (e < my_rows) sm[uint64_t(cl) * rows + wr0 + uint64_t(lane) * V + e] = acc.v[e];
    __syncthreads();
    T* tile_partials = partials + uint64_t(blockIdx.y) * gridDim.x * mt;
    for (uint64_t r = tid; r < rows; r += kRealignBlock) {
        T v = sm[r];
        for (int q = 1; q < CL; ++q) v = add_rn(v, sm[uint64_t(q) * rows + r]);
        tile_partials[uint64_t(blockIdx.x) * mt + r] = v;
    }
    if (external_combine) return; // gemv_cm_fullcol_combine16_kernel follows (PDL)
    __threadfence();
    __syncthreads();
    if (tid == 0) am_last = atomicAdd(tickets + blockIdx.y, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!am_last) return;
    __threadfence();
    split_final(tile_partials, c + r0, rows, mt, gridDim.x, sm);
    if (tid == 0) tickets[blockIdx.y] = 0u;
}

struct SplitGeom {
    int row_lanes, col_lanes, rpt;
    unsigned grid;       // column parts (gridDim.x)
    unsigned row_tiles;  // gridDim.y
    uint64_t mt;         // rows per row tile
    size_t smem;
    unsigned threads = 0; // block size where a path picks it (full-column sweep)
};

// Row tiles: one tile when m < cm_single_max(), else tiles of cm_tile_rows().
// Column parts: as many as keep row_tiles * parts within one CTA per SM
// (1024 threads each), i.e. a single wave.
constexpr uint64_t kSplitTileRows = 256;

// Row tiling of the split kernels.  A single row tile (one last-arriving CTA
// sums G partials per row) only below kSingleTileRows; above, row tiles of
// kSplitTileRows rows, each finished by its own last arriver, so the final
// combines run on different SMs at once.  256 MiB fp32 col-major, flushed,
// single tile up to 2048 rows -> up to 512 rows with 256-row tiles: m = 1024
// 61.5 -> 50.1 us, 2040 77.9 -> 52.0, 4096 52.3 -> 51.2.  Odd m keeps the
// bulk ring with scalar consumers up to kBulkScalarMaxRows (m = 1001: 104 us
// there, 143 in the 2-D scalar split).  CABL_CM_TILE="single,tile" overrides
// the first two (tuning only).
constexpr uint64_t kSingleTileRows = 512;
constexpr uint64_t kBulkScalarMaxRows = 1024;
inline uint64_t cm_single_max() {
    static const uint64_t v = [] {
        unsigned long a = kSingleTileRows, b = kSplitTileRows;
        if (const char* e = tuning_env("CABL_CM_TILE")) sscanf(e, "%lu,%lu", &a, &b);
        return uint64_t(a < kSplitMaxRows ? a : kSplitMaxRows);
    }();
    return v;
}
inline uint64_t cm_tile_rows() {
    static const uint64_t v = [] {
        unsigned long a = kSingleTileRows, b = kSplitTileRows;
        if (const char* e = tuning_env("CABL_CM_TILE")) sscanf(e, "%lu,%lu", &a, &b);
        return uint64_t(b);
    }();
    return v;
}

// Rows per tile for m >= cm_single_max(): every multiple of 32 rows from
// kSplitTileRows to max_mt is scored by the share of SM slots doing useful
// work — (row tiles x column parts) / (waves x SMs) times the share of row
// lanes that hold rows (the vector kernel's row lanes are a power of two >=
// the tile's row vectors), scaled down when a tile's final sum (parts x rows
// partials, one CTA) exceeds kFinalBudget — and the best kept.  Fixed 256-row tiles gave m =
// 3e5 x 223 fp32 1172 single-part CTAs in eight waves (80.9 us, 3.3 TB/s);
// ~148 tiles of 2048 rows take 53 us.  CABL_CM_TILE overrides (fixed rows).
constexpr uint64_t kFinalBudget = 16384; // partials one finishing CTA sums

inline uint64_t choose_tile_rows(uint64_t m, uint64_t max_mt, int vec_elems) {
    if (m < cm_single_max()) return m;
    if (tuning_env("CABL_CM_TILE")) return cm_tile_rows();
    const uint64_t sms = uint64_t(sm_count());
    uint64_t best = kSplitTileRows;
    double best_score = -1.0;
    for (uint64_t mt = kSplitTileRows; mt <= max_mt; mt += 32) {
        const uint64_t tiles = (m + mt - 1) / mt;
        uint64_t parts = sms / tiles;
        if (parts < 1) parts = 1;
        const uint64_t ctas = tiles * parts;
        const uint64_t waves = (ctas + sms - 1) / sms;
        // row lanes: pow2 >= rows (in vectors for the vector kernel, capped at
        // the block for the scalar one, whose extra rows go to RPT)
        const uint64_t units = vec_elems > 1 ? mt / uint64_t(vec_elems) : mt;
        uint64_t lanes = 1;
        while (lanes < units && lanes < uint64_t(kSplitBlock)) lanes *= 2;
        const uint64_t rpt = (units + lanes - 1) / lanes;
        const double lane_eff = double(units) / double(lanes * rpt);
        // useful share of the SM slots, of the row lanes and of the tiles'
        // rows (a ragged last tile idles its CTAs); extra waves cost their
        // ramp and per-CTA combine
        double score = lane_eff * double(ctas) / double(waves * sms) * double(m) /
                       double(tiles * mt) / (1.0 + 0.15 * double(waves - 1));
        // each tile's last CTA sums parts x mt partials alone: keep that
        // bounded (a single 2040-row tile x 148 parts took 78 us vs 52)
        if (parts * mt > kFinalBudget) score *= double(kFinalBudget) / double(parts * mt);
        if (score > best_score + 1e-9) {
            best_score = score;
            best = mt;
        }
        if (tiles == 1) break;
    }
    return best;
}

inline void split_tiles(uint64_t m, uint64_t n, uint64_t cols_per_tile, uint64_t mt,
                        SplitGeom* g) {
    g->mt = mt;
    g->row_tiles = unsigned((m + g->mt - 1) / g->mt);
    const uint64_t sms = uint64_t(sm_count());
    // floor: row_tiles * parts must not exceed one CTA per SM, or the extra
    // CTAs run as a second wave (8192^2 fp32: 152 CTAs took 65.6 us, 144 ...)
    uint64_t parts = sms / g->row_tiles;
    const uint64_t tiles = (n + cols_per_tile - 1) / cols_per_tile;
    if (parts > tiles) parts = tiles;
    g->grid = unsigned(parts < 1 ? 1 : parts);
}

template <typename T> SplitGeom split_geom(uint64_t m, uint64_t n) {
    SplitGeom g;
    const uint64_t mt = choose_tile_rows(m, 2 * uint64_t(kSplitBlock), 1); // RPT <= 2
    uint64_t rl = 32; // a power of two, so row_lanes divides the block
    while (rl < mt && rl < uint64_t(kSplitBlock)) rl *= 2;
    g.row_lanes = int(rl);
    g.col_lanes = kSplitBlock / g.row_lanes;
    g.rpt = int((mt + rl - 1) / rl);
    split_tiles(m, n, uint64_t(g.col_lanes) * split_u<T>(), mt, &g);
    // [col_lanes][rows] for the column-lane combine, >= one entry per thread for
    // split_final: <= max(kSplitBlock, mt) entries, 16 KB for fp64
    const size_t entries = size_t(g.col_lanes) * g.mt;
    g.smem = (entries > size_t(kSplitBlock) ? entries : size_t(kSplitBlock)) * sizeof(T);
    return g;
}

template <typename T> bool split_vec_ok(const T* A, uint64_t m) {
    return aligned32(A) && m % Vec<T>::N == 0;
}

template <typename T> SplitGeom split_vec_geom(uint64_t m, uint64_t n) {
    SplitGeom g;
    const uint64_t mt = choose_tile_rows(m, uint64_t(kSplitBlock) * Vec<T>::N, Vec<T>::N);
    const uint64_t mv = mt / Vec<T>::N;
    uint64_t rl = 1;
    while (rl < mv) rl *= 2;
    g.row_lanes = int(rl);
    g.col_lanes = kSplitBlock / g.row_lanes;
    g.rpt = 1;
    split_tiles(m, n, uint64_t(g.col_lanes) * 4, mt, &g);
    g.smem = 0;
    return g;
}

// Realign geometry: tiles of RW * 31 * V rows (RW row warps, a power of two
// <= 32), column parts filling one wave; RW scored like choose_tile_rows
// (useful SM slots x useful tile rows, bounded final sum).  smem: [CL][rows]
// for the column-lane combine, >= kSplitBlock entries for split_final.
// best row-warp count for m and its score
template <typename T> int realign_rw(uint64_t m, double* score_out) {
    constexpr uint64_t LR = 31 * Vec<T>::N;
    const uint64_t sms = uint64_t(sm_count());
    int best_rw = 1;
    double best_score = -1.0;
    for (int rw = 1; rw <= kRealignBlock / 32; rw *= 2) {
        const uint64_t mt = uint64_t(rw) * LR;
        const uint64_t tiles = (m + mt - 1) / mt;
        uint64_t parts = sms / tiles;
        if (parts < 1) parts = 1;
        const uint64_t ctas = tiles * parts;
        const uint64_t waves = (ctas + sms - 1) / sms;
        double score = double(ctas) / double(waves * sms) * double(m) / double(tiles * mt) /
                       (1.0 + 0.15 * double(waves - 1));
        if (parts * mt > kFinalBudget) score *= double(kFinalBudget) / double(parts * mt);
        if (score > best_score + 1e-9) {
            best_score = score;
            best_rw = rw;
        }
        if (tiles == 1) break;
    }
    if (score_out) *score_out = best_score;
    return best_rw;
}

template <typename T> SplitGeom split_realign_geom(uint64_t m, uint64_t n) {
    constexpr uint64_t LR = 31 * Vec<T>::N;
    const int best_rw = realign_rw<T>(m, nullptr);
    SplitGeom g;
    g.row_lanes = best_rw; // row warps
    g.col_lanes = (kRealignBlock / 32) / best_rw;
    g.rpt = 1;
    split_tiles(m, n, uint64_t(g.col_lanes) * kRealignU, uint64_t(best_rw) * LR, &g);
    const size_t entries = size_t(g.col_lanes) * g.mt;
    g.smem = (entries > size_t(kRealignBlock) ? entries : size_t(kRealignBlock)) * sizeof(T);
    return g;
}

struct BulkCfg {
    int stages;
    unsigned stage_bytes;
};

inline BulkCfg bulk_cfg() {
    static const BulkCfg c = [] {
        // measured on 256 x 2^20 fp64, back to back (tools/b2b.py): the sweet
        // spot is ~128-160 KB in flight per SM in stages of >= 48 KB —
        // 3x48 KB 299.1 us, 2x80 299.7, 4x36 299.7, 3x40 300.2, 2x64 300.9,
        // 3x64 307.0, 4x48 308.1, 2x48 311.8, 6x32 315.1
        BulkCfg b{3, 49152};
        if (const char* e = tuning_env("CABL_BULK")) { // "stages,KiB" (tuning only)
            int st = 6, kb = 32;
            if (sscanf(e, "%d,%d", &st, &kb) == 2) b = BulkCfg{st, unsigned(kb) * 1024u};
        }
        return b;
    }();
    return c;
}

template <typename T>
SplitGeom split_bulk_geom(uint64_t m, uint64_t n, int* tc, BulkCfg bc = bulk_cfg()) {
    SplitGeom g;
    const uint64_t mv = m / Vec<T>::N;
    uint64_t rl = 1;
    while (rl < mv) rl *= 2;
    g.row_lanes = int(rl);
    g.col_lanes = kBulkConsumers / g.row_lanes;
    g.rpt = 1;
    // columns per stage, a multiple of 16/s so the x slice is a whole number of
    // 16-byte bulk units (m*s <= 16 KB for m < 2048, so tc >= 2 fp64 / 4 fp32)
    // tile and its x slice share the stage: (m + 1) * tc * s <= SB + XB (for
    // few rows the slice is as large as the tile: m = 1 fp32 streams 24 KB of
    // A and 24 KB of x per stage instead of reading x element by element)
    const int xq = int(16 / sizeof(T));
    *tc = int((bc.stage_bytes + kBulkXBytes) / ((m + 1) * sizeof(T))) / xq * xq;
    if (*tc < xq) *tc = xq;
    const uint64_t tiles = (n + *tc - 1) / *tc;
    const uint64_t cap = uint64_t(sm_count());
    g.grid = unsigned(tiles < cap ? (tiles < 1 ? 1 : tiles) : cap);
    g.row_tiles = 1;
    g.mt = m;
    g.smem = bulk_smem(bc.stages, bc.stage_bytes);
    return g;
}

template <typename T, int NS, unsigned SB>
void bulk_go(const T* A, const T* x, T* c, uint64_t m, uint64_t n, const SplitGeom& g, int tc,
             T* partials, unsigned* ticket, cudaStream_t s) {
    static std::atomic<unsigned long long> configured{0};
    ensure_dyn_smem(gemv_cm_split_bulk_kernel<T, NS, SB>, int(bulk_smem(NS, SB)), configured);
    // The per-row sum of the G CTA partials in a one-wave combine kernel
    // instead of by the last CTA alone (256 MiB flushed / back to back,
    // tools/ab_shapes.py: fp32 m = 256 51.4 / 46.5 -> 48.2 / 43.8 us, m = 504
    // 54.2 / 49.2 -> 48.4 / 44.0; fp64 m = 504 91.0 -> 84.8; G3 flushed
    // 304.8 -> 300.6).  CABL_CM_BULK_COMB16=0 keeps the in-kernel finish (A/B).
    static const int comb16 = [] {
        const char* e = tuning_env("CABL_CM_BULK_COMB16");
        return e ? atoi(e) : 1;
    }();
    const bool ext = comb16 != 0 && g.grid >= 2;
    launch(gemv_cm_split_bulk_kernel<T, NS, SB>, g.grid, kBulkThreads, bulk_smem(NS, SB), s,
           A, x, c, m, n, g.row_lanes, tc, uint64_t(tc) * m, partials, ticket,
           int((reinterpret_cast<uintptr_t>(x) & 15u) == 0), int(ext));
    if (ext) {
        constexpr unsigned E = 16 / sizeof(T), R = (256 / kC16G) * E;
        launch(gemv_cm_fullcol_combine16_kernel<T>, unsigned((m + R - 1) / R), 256u, 0, s,
               static_cast<const T*>(partials), g.grid, m, m, c);
    }
}

// Rows per consumer thread for the scalar bulk kernel: with row_lanes =
// ceil(m / rpt) and col_lanes = 512 / row_lanes, a thread's share of a tile
// is rpt / col_lanes of its columns; take the smallest (ties: fewer rows).
// 257 rows: 1 -> 1 x 1 lane set, 4 -> 65 x 7 (4/7 of a tile per thread).
inline int bulk_scalar_rpt(uint64_t m) {
    int best = 0;
    double best_work = 1e30;
    for (int r : {1, 2, 4}) {
        const uint64_t rl = (m + r - 1) / r;
        if (rl > uint64_t(kBulkConsumers)) continue;
        const double work = double(r) / double(uint64_t(kBulkConsumers) / rl);
        if (work < best_work - 1e-12) {
            best_work = work;
            best = r;
        }
    }
    return best ? best : 4;
}

template <typename T, int RPT>
void bulk_scalar_go(const T* A, const T* x, T* c, uint64_t m, uint64_t n, const SplitGeom& g,
                    int tc, int x_bulk, T* partials, unsigned* ticket, cudaStream_t s) {
    // A's element offset from a 16-byte boundary; the x slice goes after the
    // tile rounded up to 16 bytes (its bulk destination must be aligned)
    const int a_off = int((reinterpret_cast<uintptr_t>(A) & 15u) / sizeof(T));
    const uint64_t q = 16 / sizeof(T);
    const uint64_t x_off = a_off ? (uint64_t(tc) * m + a_off + q - 1) / q * q : uint64_t(tc) * m;
    static std::atomic<unsigned long long> configured{0};
    ensure_dyn_smem(gemv_cm_split_bulk_scalar_kernel<T, 3, 49152, RPT>, int(bulk_smem(3, 49152)),
                    configured);
    // the G CTA partials of each row summed by the (scalar-load) one-wave
    // combine kernel, as in bulk_go (CABL_CM_BULK_COMB16=0: in-kernel, A/B)
    static const int comb = [] {
        const char* e = tuning_env("CABL_CM_BULK_COMB16");
        return e ? atoi(e) : 1;
    }();
    const bool ext = comb != 0 && g.grid >= 2;
    launch(gemv_cm_split_bulk_scalar_kernel<T, 3, 49152, RPT>, g.grid, kBulkThreads,
           bulk_smem(3, 49152), s, A, x, c, m, n, g.row_lanes, tc, x_off, x_bulk, partials,
           ticket, a_off, int(ext));
    if (ext)
        launch(gemv_cm_fullcol_combine_kernel<T>, unsigned((m + 31) / 32), 1024u, 0, s,
               static_cast<const T*>(partials), g.grid, m, c);
}

inline int split_mode() {
    static const int v = [] {
        const char* e = tuning_env("CABL_CM_SPLIT");
        return e ? atoi(e) : 1;
    }();
    return v; // 1 = bulk-copy pipeline, 0 = register loads
}

template <typename T> bool tall_vec_ok(const T* A, const T* c, uint64_t m) {
    return aligned32(A) && aligned32(c) && m % Vec<T>::N == 0;
}

// CABL_CM_BULK_ANY=0: A off a 16-byte boundary (m < 1024) back on the scalar
// 2-D split (A/B only).
inline bool bulk_any_align() {
    static const bool on = [] {
        const char* e = tuning_env("CABL_CM_BULK_ANY");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}

enum CmPath { kPathTallVec, kPathTallScalar, kPathBulk, kPathBulkScalar, kPathSplitVec,
              kPathSplitScalar, kPathSplitRealign, kPathFullCol, kPathFullCol2, kPathColBulk };

// Full-column bulk ring for unvectorisable columns (odd m or A off a 32-byte
// boundary) from kBulkScalarMaxRows rows while one column fits a stage
// (CABL_CM_COLBULK=0|1, A/B).
inline int colbulk_forced() {
    static const int v = [] {
        const char* e = tuning_env("CABL_CM_COLBULK");
        return e ? atoi(e) : -1;
    }();
    return v;
}
// A stage size for m (0: none fits well): stages must hold >= 2 columns, or
// one column filling >= 3/4 of the stage (fp32: 4/5) — a single column of
// 50-75% of a stage leaves the ring short of bytes in flight (fp32 m = 8193
// in 48 KB stages: 68 us against 58 on the realigning split; in 72 KB stages,
// two per stage: 51.1), and fp32 14001 (76% of 72 KB) lost 56.1 -> 58.5
// while fp64 7001 (76%) won 91.4 -> 85.2 (profiles/r02_cm_colbulk_big.jsonl).
template <typename T> unsigned colbulk_stage(uint64_t m) {
    constexpr uint64_t q = 16 / sizeof(T);
    constexpr uint64_t fill_num = sizeof(T) == 4 ? 5 : 4, fill_den = sizeof(T) == 4 ? 4 : 3;
    for (unsigned sb : {kColBulkStageBytes, kColBulkBigStageBytes}) {
        if (m + 2 * q > sb / sizeof(T)) continue;
        const uint64_t tcols = (sb / sizeof(T) - 2 * q) / m;
        if (tcols >= 2 || m * sizeof(T) * fill_num >= uint64_t(sb) * fill_den) return sb;
    }
    return 0;
}
template <typename T> bool colbulk_ok(const T* A, uint64_t m) {
    if (colbulk_forced() == 0) return false;
    if (reinterpret_cast<uintptr_t>(A) % sizeof(T) != 0) return false;
    return m >= kBulkScalarMaxRows && colbulk_stage<T>(m) != 0;
}

// Full-column sweep for aligned m with m/V <= 1024 row vectors (at most one per
// thread of a 1024-thread CTA).  CABL_CM_FULLCOL=0 keeps the 2-D split (A/B).
inline bool fullcol_enabled() {
    static const bool on = [] {
        const char* e = tuning_env("CABL_CM_FULLCOL");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}
template <typename T> bool fullcol_ok(uint64_t m) {
    return m / Vec<T>::N <= 1024 && fullcol_enabled();
}
// fp32 8192 < m <= 16384: the full-column sweep with two row vectors per
// thread and the 16-byte combine (256 MiB, tools/cm_mid2.py: 16384 x 4096
// flushed / back to back 52.2 / 48.6 -> 48.7 / 47.2 us, 12000 x 5592 50.6 /
// 47.7 -> 50.7 / 46.8).  fp64 (m <= 8192) stays on the 2-D split: 8192 x 8192
// was 87.9 / 85.1 -> 85.7 / 87.6, slower back to back.  CABL_CM_FULLCOL2=0|1
// forces it off / on for both types (A/B).
inline int fullcol2_forced() {
    static const int v = [] {
        const char* e = tuning_env("CABL_CM_FULLCOL2");
        return e ? atoi(e) : -1;
    }();
    return v;
}
template <typename T> bool fullcol2_ok(uint64_t m) {
    const uint64_t mv = m / Vec<T>::N;
    if (mv <= 1024 || mv > 2048 || !fullcol_enabled()) return false;
    const int f = fullcol2_forced();
    return f >= 0 ? f != 0 : sizeof(T) == 4;
}
// <= 512 row vectors: 512-thread CTAs, two per SM; up to 1024: one
// 1024-thread CTA per SM (tools/cmlab.py: 5.67 vs 5.45 TB/s at 4096 rows,
// 5.56 vs 5.48 at 8192); never more CTAs than column groups.
template <typename T> SplitGeom fullcol_geom(uint64_t m, uint64_t n) {
    SplitGeom g;
    const uint64_t mv = m / Vec<T>::N;
    const uint64_t sms = uint64_t(sm_count());
    g.threads = mv <= 512 ? 512u : 1024u;
    uint64_t rl = 1;
    while (rl < mv) rl *= 2;
    g.row_lanes = int(rl);
    g.col_lanes = int(g.threads) / g.row_lanes;
    g.rpt = 1;
    uint64_t parts = g.threads == 512u ? 2 * sms : sms;
    const uint64_t groups = (n + uint64_t(g.col_lanes) - 1) / uint64_t(g.col_lanes);
    if (parts > groups) parts = groups;
    g.grid = unsigned(parts < 1 ? 1 : parts);
    g.row_tiles = 1;
    g.mt = m;
    g.smem = 0;
    return g;
}

// CABL_CM_REALIGN=0 keeps misaligned columns on the scalar 2-D split (A/B only).
inline bool realign_enabled() {
    static const bool on = [] {
        const char* e = tuning_env("CABL_CM_REALIGN");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}

// The bit-exact tall kernels keep each row's sum on one thread, so their
// parallelism is m/V threads: they are used only when that fills the GPU
// (>= one 256-row-vector unit per SM, or >= 1024 rows per SM for the scalar
// variant).  Everything else splits the columns (2-D row tiles x column
// parts; a single bulk-streamed row tile when m < kSplitMaxRows).
// 256-vector units from which the tall kernel runs: half the SMs.  One CTA
// per SM with 16 column loads per thread in flight streams fast enough that
// 74 SMs match the 2-D split on all 148 (256 MiB fp32: m = 1.5e5 51.1 vs
// 51.2 us; 2e5 47.1 vs 59.6; 2.6e5 44.1 vs 53.3), and it is bitwise gemv_ref.
// CABL_CM_TALL_MIN overrides (tuning only).
inline uint64_t tall_min_units() {
    static const long forced = [] {
        const char* e = tuning_env("CABL_CM_TALL_MIN");
        return e ? atol(e) : -1L;
    }();
    return forced > 0 ? uint64_t(forced) : uint64_t(sm_count()) / 2;
}

template <typename T> CmPath cm_path(const T* A, const T* c, uint64_t m) {
    const uint64_t sms = uint64_t(sm_count());
    if (tall_vec_ok(A, c, m)) {
        if (m / Vec<T>::N >= tall_min_units() * kTallBlock) return kPathTallVec;
    } else if (m >= sms * 1024) {
        return kPathTallScalar;
    }
    if (split_vec_ok(A, m)) {
        if (m < cm_single_max() && split_mode() == 1) return kPathBulk;
        if (fullcol2_ok<T>(m)) return kPathFullCol2;
        return fullcol_ok<T>(m) ? kPathFullCol : kPathSplitVec;
    }
    // A off a 16-byte boundary: the bulk ring from the boundary below A (256 MiB
    // fp32 flushed, tools/cm_mis.py: m = 3 / 257 / 1000 680 / 137 / 78 -> 70 /
    // 55 / 66 us against the scalar 2-D split); fp64 from 768 rows stays on the
    // split (1000 rows: 59 against 63.5)
    if (m < kBulkScalarMaxRows && split_mode() == 1 && reinterpret_cast<uintptr_t>(A) % sizeof(T) == 0 &&
        bulk_any_align() && !(sizeof(T) == 8 && m >= 768))
        return kPathBulkScalar;
    if (m < kBulkScalarMaxRows && split_mode() == 1 && (reinterpret_cast<uintptr_t>(A) & 15u) == 0)
        return kPathBulkScalar;
    if (colbulk_ok(A, m)) return kPathColBulk;
    // the realigning split when its tiling keeps most SM slots and tile rows
    // busy (score >= 0.8: 8193 rows 0.89); a poor tiling (m = 100003: 0.70,
    // 74 us against the scalar split's 61) stays on the scalar split
    double score = 0.0;
    if (m >= kBulkScalarMaxRows && realign_enabled() &&
        reinterpret_cast<uintptr_t>(A) % sizeof(T) == 0 && (realign_rw<T>(m, &score), score >= 0.8))
        return kPathSplitRealign;
    return kPathSplitScalar;
}

// Split tiles with >= 2 column parts finish in a one-wave combine kernel
// (PDL) instead of each tile's last CTA summing parts x mt partials alone
// (256 MiB fp64 flushed / back to back, tools/cm_mid2.py: 8192 x 8192, 16
// tiles x 9 parts, 88.0 / 85.1 -> 85.1 / 82.3 us; 12000 x 5592 89.4 / 86.9 ->
// 87.2 / 84.0); single-part tiles (m >= 32768) keep the in-kernel finish, a
// second launch only costs there (fp32 65536 x 1024 49.4 -> 52.5).  Odd m
// (scalar and realigning splits): 12345 x 5436 fp32 59.8 -> 58.1, 40001 x
// 1677 61.3 -> 57.6 (fp64 98.5 -> 94.6); above 65536 rows the combine's many
// CTAs cost more than the last CTA's small sum (100003 x 671 fp64, 3 parts of
// 2048 rows: 97.3 -> 99.2), so those keep the in-kernel finish
// (tools/ab_shapes.py, profiles/r02_cm_split_comb16*.jsonl).
// CABL_CM_SPLIT_COMB16=0|1 forces it off / on (A/B).
template <typename T> bool split_external_combine(const SplitGeom& g, uint64_t m) {
    static const int forced = [] {
        const char* e = tuning_env("CABL_CM_SPLIT_COMB16");
        return e ? atoi(e) : -1;
    }();
    constexpr unsigned E = 16 / sizeof(T);
    return (forced < 0 ? g.grid >= 2 && m <= 65536 : forced != 0) && g.mt % E == 0;
}
template <typename T>
void combine16_launch(T* partials, const SplitGeom& g, uint64_t m, T* c, cudaStream_t s) {
    constexpr unsigned E = 16 / sizeof(T), R = (256 / kC16G) * E;
    launch(gemv_cm_fullcol_combine16_kernel<T>, unsigned((m + R - 1) / R), 256u, 0, s,
           static_cast<const T*>(partials), g.grid, m, uint64_t(g.mt), c);
}

template <typename T, int RPT, unsigned SB>
void colbulk_launch(const T* A, const T* x, uint64_t m, uint64_t n, const SplitGeom& g, T* partials,
                    cudaStream_t s) {
    static std::atomic<unsigned long long> configured{0};
    ensure_dyn_smem(gemv_cm_colbulk_kernel<T, RPT, SB>, int(kColBulkStages * SB), configured);
    launch(gemv_cm_colbulk_kernel<T, RPT, SB>, g.grid, unsigned(kBulkThreads), g.smem, s, A, x, m,
           n, uint64_t(g.mt), g.col_lanes, partials);
}
template <typename T, unsigned SB>
void colbulk_rpt(const T* A, const T* x, uint64_t m, uint64_t n, const SplitGeom& g, T* partials,
                 cudaStream_t s) {
    const int rpt = g.rpt;
    if (rpt <= 2) colbulk_launch<T, 2, SB>(A, x, m, n, g, partials, s);
    else if (rpt <= 4) colbulk_launch<T, 4, SB>(A, x, m, n, g, partials, s);
    else if (rpt <= 8) colbulk_launch<T, 8, SB>(A, x, m, n, g, partials, s);
    else if (rpt <= 12) colbulk_launch<T, 12, SB>(A, x, m, n, g, partials, s);
    else if (rpt <= 16) colbulk_launch<T, 16, SB>(A, x, m, n, g, partials, s);
    else if (rpt <= 20) colbulk_launch<T, 20, SB>(A, x, m, n, g, partials, s);
    else if (rpt <= 24) colbulk_launch<T, 24, SB>(A, x, m, n, g, partials, s);
    else if (rpt <= 30) colbulk_launch<T, 30, SB>(A, x, m, n, g, partials, s);
    else colbulk_launch<T, 36, SB>(A, x, m, n, g, partials, s);
}
template <typename T>
void colbulk_go(const T* A, const T* x, T* c, uint64_t m, uint64_t n, const SplitGeom& g, T* partials,
                cudaStream_t s) {
    if (g.smem == size_t(kColBulkStages) * kColBulkStageBytes)
        colbulk_rpt<T, kColBulkStageBytes>(A, x, m, n, g, partials, s);
    else
        colbulk_rpt<T, kColBulkBigStageBytes>(A, x, m, n, g, partials, s);
    combine16_launch<T>(partials, g, m, c, s);
}

template <typename T> SplitGeom cm_split_geom(CmPath p, const T* A, uint64_t m, uint64_t n, int* tc) {
    if (p == kPathBulk) return split_bulk_geom<T>(m, n, tc);
    if (p == kPathBulkScalar) {
        // an A off a 16-byte boundary needs up to 2 x 16 bytes more per stage
        // (the copy's leading pad and the rounded-up x slot): shrink the budget
        const bool mis = (reinterpret_cast<uintptr_t>(A) & 15u) != 0;
        SplitGeom g = split_bulk_geom<T>(m, n, tc, BulkCfg{3, mis ? 49152u - 32u : 49152u});
        g.smem = bulk_smem(3, 49152);
        g.rpt = bulk_scalar_rpt(m);
        g.row_lanes = int((m + g.rpt - 1) / g.rpt);
        g.col_lanes = kBulkConsumers / g.row_lanes;
        return g;
    }
    if (p == kPathSplitVec) return split_vec_geom<T>(m, n);
    if (p == kPathFullCol) return fullcol_geom<T>(m, n);
    if (p == kPathColBulk) {
        SplitGeom g;
        constexpr uint64_t q = 16 / sizeof(T);
        g.threads = unsigned(kBulkThreads);
        g.row_lanes = kBulkConsumers;
        g.rpt = int((m + kBulkConsumers - 1) / kBulkConsumers);
        // columns per stage: as many whole columns as fit with the 16-byte lead-in
        const unsigned sb = colbulk_stage<T>(m);
        uint64_t tcols = (sb / sizeof(T) - 2 * q) / m;
        if (tcols > uint64_t(kColBulkMaxTc)) tcols = kColBulkMaxTc;
        g.col_lanes = int(tcols < 1 ? 1 : tcols); // (carries tc to the launch)
        g.smem = size_t(kColBulkStages) * sb;        // (and the stage size)
        const uint64_t tiles = (n + uint64_t(g.col_lanes) - 1) / uint64_t(g.col_lanes);
        const uint64_t sms = uint64_t(sm_count());
        g.grid = unsigned(tiles < sms ? tiles : sms);
        g.row_tiles = 1;
        g.mt = (m + q - 1) / q * q; // partial row stride: whole 16-byte units
        return g;
    }
    if (p == kPathFullCol2) {
        SplitGeom g;
        g.threads = 1024u;
        g.row_lanes = 1024;
        g.col_lanes = 1;
        g.rpt = 2;
        const uint64_t sms = uint64_t(sm_count());
        g.grid = unsigned(n < sms ? n : sms);
        g.row_tiles = 1;
        g.mt = m;
        g.smem = 0;
        return g;
    }
    if (p == kPathSplitRealign) return split_realign_geom<T>(m, n);
    return split_geom<T>(m, n);
}

} // namespace

template <typename T> WorkspaceNeed gemv_cm_need(const T* A, const T*, uint64_t m, uint64_t n) {
    WorkspaceNeed w;
    if (m == 0 || n == 0) return w;
    const CmPath p = cm_path<T>(A, A, m); // c's alignment only matters to the tall kernels

    if (p == kPathTallVec || p == kPathTallScalar) {
        w.counters = 1; // unit counter of the tall kernel
        return w;
    }
    int tc = 1;
    const SplitGeom g = cm_split_geom<T>(p, A, m, n, &tc);
    w.counters = g.row_tiles;
    w.scratch_bytes = size_t(g.row_tiles) * g.grid * g.mt * sizeof(T);
    return w;
}

template <typename T>
cudaError_t gemv_cm_launch(const T* A, uint64_t m, uint64_t n, const T* x, T* c,
                           const Workspace& ws, cudaStream_t s, LaunchInfo* info) {
    if (info) info->ctas = 0;
    if (m == 0 || n == 0) return cudaSuccess;
    const CmPath path = cm_path<T>(A, A, m);
    // (a c whose alignment differs from A's falls back to the scalar-lane
    // tall kernel: same order and rounding)
    if (path == kPathTallVec && aligned32(c) && n < uint64_t(kTallUnroll)) {
        const int nc = n <= 4 ? 4 : (n <= 8 ? 8 : 16);
        const uint64_t per_unit = uint64_t(kTallBlock) * (kTallUnroll / nc);
        const uint64_t units = (m / Vec<T>::N + per_unit - 1) / per_unit;
        const uint64_t sms = uint64_t(sm_count());
        const unsigned grid = unsigned(units < sms ? units : sms);
        if (nc == 4)
            launch(gemv_cm_narrow_kernel<T, 4>, grid, kTallBlock, 0, s, A, x, c, m, n);
        else if (nc == 8)
            launch(gemv_cm_narrow_kernel<T, 8>, grid, kTallBlock, 0, s, A, x, c, m, n);
        else
            launch(gemv_cm_narrow_kernel<T, 16>, grid, kTallBlock, 0, s, A, x, c, m, n);
        if (info) info->ctas = grid;
    } else if (path == kPathTallVec && aligned32(c)) {
        const uint64_t units = (m / Vec<T>::N + kTallBlock - 1) / kTallBlock;
        const uint64_t sms = uint64_t(sm_count());
        const unsigned grid = unsigned(units < sms ? units : sms); // grid <= units (dyn_next)
        // dynamic unit queue for large matrices (2^20 x 256 fp64: 310 -> 301 us),
        // static unit ranges otherwise; CABL_GEMV_DYN=0|1 overrides (tuning)
        static const int forced = [] {
            const char* e = tuning_env("CABL_GEMV_DYN");
            return e ? atoi(e) : -1;
        }();
        const bool dyn = forced >= 0 ? forced != 0 : m * n * sizeof(T) >= queue_threshold_bytes();
        if (dyn)
            launch(gemv_cm_tall_vec_kernel<T, true>, grid, kTallBlock, 0, s, A, x, c, m, n, ws.counters);
        else
            launch(gemv_cm_tall_vec_kernel<T, false>, grid, kTallBlock, 0, s, A, x, c, m, n, ws.counters);
        if (info) info->ctas = grid;
    } else if (path == kPathTallScalar || path == kPathTallVec) {
        const uint64_t units = (m + kWarp - 1) / kWarp;
        const uint64_t max_warps = uint64_t(sm_count()) * kCmRowsCtasPerSm * (kCmBlock / kWarp);
        // smallest per-warp unit count that fits one wave, then as few warps
        // as keep that count: every warp gets the same number of units +-1
        const uint64_t per = (units + max_warps - 1) / max_warps;
        const uint64_t warps = (units + per - 1) / per;
        const unsigned grid = unsigned((warps * kWarp + kCmBlock - 1) / kCmBlock);
        launch(gemv_cm_rows_kernel<T>, grid, kCmBlock, 0, s, A, x, c, m, n, warps);
        if (info) info->ctas = grid;
    } else {
        int tc = 1;
        const SplitGeom g = cm_split_geom<T>(path, A, m, n, &tc);
        T* partials = static_cast<T*>(ws.scratch);
        const dim3 grid(g.grid, g.row_tiles);
        if (path == kPathBulk) {
            const BulkCfg bc = bulk_cfg();
            if (bc.stages == 3 && bc.stage_bytes == 65536)
                bulk_go<T, 3, 65536>(A, x, c, m, n, g, tc, partials, ws.counters, s);
            else if (bc.stages == 2 && bc.stage_bytes == 81920)
                bulk_go<T, 2, 81920>(A, x, c, m, n, g, tc, partials, ws.counters, s);
            else if (bc.stages == 6 && bc.stage_bytes == 32768)
                bulk_go<T, 6, 32768>(A, x, c, m, n, g, tc, partials, ws.counters, s);
            else if (bc.stages == 4 && bc.stage_bytes == 49152)
                bulk_go<T, 4, 49152>(A, x, c, m, n, g, tc, partials, ws.counters, s);
            else
                bulk_go<T, 3, 49152>(A, x, c, m, n, g, tc, partials, ws.counters, s);
        } else if (path == kPathBulkScalar) {
            // default ring shape only (3 x 48 KB); x rides in the ring when it
            // is 16-byte aligned
            const int x_bulk = (reinterpret_cast<uintptr_t>(x) & 15u) == 0;
            if (g.rpt == 1)
                bulk_scalar_go<T, 1>(A, x, c, m, n, g, tc, x_bulk, partials, ws.counters, s);
            else if (g.rpt == 2)
                bulk_scalar_go<T, 2>(A, x, c, m, n, g, tc, x_bulk, partials, ws.counters, s);
            else
                bulk_scalar_go<T, 4>(A, x, c, m, n, g, tc, x_bulk, partials, ws.counters, s);
        } else if (path == kPathSplitRealign) {
            static std::atomic<unsigned long long> configured{0};
            ensure_dyn_smem(gemv_cm_split_realign_kernel<T>, int(16 * 31 * Vec<T>::N * sizeof(T)),
                            configured);
            const bool ext = split_external_combine<T>(g, m);
            launch(gemv_cm_split_realign_kernel<T>, grid, kRealignBlock, g.smem, s, A, x, c, m, n,
                   g.mt, g.row_lanes, partials, ws.counters, int(ext));
            if (ext) combine16_launch<T>(partials, g, m, c, s);
        } else if (path == kPathFullCol) {
            launch(gemv_cm_fullcol_kernel<T>, g.grid, g.threads, 0, s, A, x, m, n, g.row_lanes,
                   partials);
            launch(gemv_cm_fullcol_combine_kernel<T>, unsigned((m + 31) / 32), 1024u, 0, s,
                   static_cast<const T*>(partials), g.grid, m, c);
        } else if (path == kPathColBulk) {
            colbulk_go<T>(A, x, c, m, n, g, partials, s);
        } else if (path == kPathFullCol2) {
            constexpr unsigned E = 16 / sizeof(T), R = (256 / kC16G) * E;
            launch(gemv_cm_fullcol2_kernel<T>, g.grid, g.threads, 0, s, A, x, m, n, partials);
            static const int comb16 = [] {
                const char* e = tuning_env("CABL_CM_FC2_COMB16");
                return e ? atoi(e) : 1;
            }();
            if (comb16)
                launch(gemv_cm_fullcol_combine16_kernel<T>, unsigned((m + R - 1) / R), 256u, 0, s,
                       static_cast<const T*>(partials), g.grid, m, m, c);
            else
                launch(gemv_cm_fullcol_combine_kernel<T>, unsigned((m + 31) / 32), 1024u, 0, s,
                       static_cast<const T*>(partials), g.grid, m, c);
        } else if (path == kPathSplitVec) {
            const bool ext = split_external_combine<T>(g, m);
            launch(gemv_cm_split_vec_kernel<T>, grid, kSplitBlock, 0, s,
                   A, x, c, m, n, g.mt, g.row_lanes, partials, ws.counters, int(ext));
            if (ext) combine16_launch<T>(partials, g, m, c, s);
        } else {
            const bool ext = split_external_combine<T>(g, m);
            if (g.rpt == 1)
                launch(gemv_cm_split_kernel<T, 1>, grid, kSplitBlock, g.smem, s,
                       A, x, c, m, n, g.mt, g.row_lanes, partials, ws.counters, int(ext));
            else
                launch(gemv_cm_split_kernel<T, 2>, grid, kSplitBlock, g.smem, s,
                       A, x, c, m, n, g.mt, g.row_lanes, partials, ws.counters, int(ext));
            if (ext) combine16_launch<T>(partials, g, m, c, s);
        }
        if (info) info->ctas = g.grid * g.row_tiles;
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

// Row-major GEMV in the REFERENCE'S ORDER: c_i += A(i,:) x, one lane per row,
// j ascending from c_i, with the compiled reference's rounding (separately
// rounded multiply then add; oracle/cabl_oracle.c) — bit for bit the
// reference gemv_row_major / gemv_ref (proj/include/cabl/kernels.hpp:171-181,
// :230-257) at full HBM bandwidth.
//
// A lane owns a whole row, so the row's 8192 (G1) or 65536 (G4) dependent
// adds are one sequential chain; that chain (4 cycles per add) is shorter
// than the time to stream the row's bytes, so the order costs no bandwidth as
// long as the bytes arrive in time.  They arrive through shared memory:
//   * CTA b owns a balanced contiguous range of rows (±1 row per SM) and
//     walks it in row blocks of up to kOrdRows rows;
//   * a producer warp streams each row block column tile by column tile into
//     a ring of kOrdStages shared-memory stages with cp.async (one 512-byte
//     row segment per warp instruction, plus the tile's x slice), completion
//     counted on the stage's mbarrier;
//   * consumer lanes read 16-byte groups of their row (row pitch padded by
//     16 B, so a quarter-warp covers all 32 banks once) and the broadcast x
//     group, and run the ordered multiply-add chain.
// (The copies are LDGSTS issued by a producer warp, one 512-byte row segment
// per warp instruction, completion tracked on the stage mbarrier.)
// Fast-path conditions: n * s a multiple of 16 B and A, x 16-byte aligned
// (then the reference's FMA remainder n mod (16/s) is empty), and enough
// rows that each CTA gets a full warp of them.
#include "bulk.cuh"
#include "common.cuh"
#include "kernels.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

namespace cabl_dev {

namespace {

constexpr int kOrdConsumerWarps = 2;
constexpr int kOrdRows = kOrdConsumerWarps * 32; // rows per block

template <typename T, int SEG, int NS> struct OrdGeom {
    static_assert(SEG % 512 == 0, "a warp instruction moves 512 B");
    static constexpr int kStages = NS;
    static constexpr int kCols = SEG / int(sizeof(T));   // SEG bytes of each row per stage
    static constexpr int kPad = 16 / int(sizeof(T));     // pitch pad: 16 B
    static constexpr int kPitch = kCols + kPad;
    static constexpr int kStageElems = kOrdRows * kPitch + kCols;
    static constexpr unsigned kSmem = unsigned(NS * kStageElems * sizeof(T));
};

template <typename T> struct Vec16;
template <> struct alignas(16) Vec16<float> {
    float v[4];
};
template <> struct alignas(16) Vec16<double> {
    double v[2];
};

template <typename T, int SEG, int NS, int PW>
__global__ void __launch_bounds__(kOrdRows + 32 * PW, 1)
    gemv_rm_ordered_kernel(const T* __restrict__ A, const T* __restrict__ x, T* __restrict__ c,
                           uint64_t m, uint64_t n) {
    pdl_enter();
    using G = OrdGeom<T, SEG, NS>;
    constexpr int kOrdStages = NS;
    constexpr int E = 16 / int(sizeof(T)); // elements per 16-byte group
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* stages = reinterpret_cast<T*>(smem_raw);
    __shared__ __align__(8) uint64_t full[NS];
    __shared__ __align__(8) uint64_t empty[NS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const Partition part(m, gridDim.x);
    const uint64_t r_begin = part.begin(blockIdx.x), r_end = part.begin(blockIdx.x + 1);
    const uint64_t tiles = (n + G::kCols - 1) / G::kCols;

    if (tid == 0) {
        for (int s = 0; s < kOrdStages; ++s) {
            mbar_init(&full[s], 32 * PW); // one cp.async arrive per producer lane
            mbar_init(&empty[s], kOrdConsumerWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp >= kOrdConsumerWarps) { // producer warps: rows pw, pw + PW, ...
        const int pw = warp - kOrdConsumerWarps;
        // One LDGSTS (cp.async, 16 B per lane) moves a 512-byte row segment:
        // a stage is `rows` + 1 (x) warp instructions.  Each lane then makes
        // the stage's mbarrier track its own copies (.noinc arrive), so the
        // stage completes when all 32 lanes' copies have landed.  (Bulk TMA
        // copies of 512 B per row ran 4.8x slower: per-copy overhead.)
        uint64_t it = 0;
        for (uint64_t rb = r_begin; rb < r_end; rb += kOrdRows) {
            const int rows = int((r_end - rb < uint64_t(kOrdRows)) ? r_end - rb : kOrdRows);
            for (uint64_t t = 0; t < tiles; ++t, ++it) {
                const int st = int(it % kOrdStages);
                const unsigned use = unsigned(it / kOrdStages);
                if (use > 0) mbar_wait(&empty[st], (use - 1) & 1u);
                const uint64_t j0 = t * G::kCols;
                const unsigned cw = unsigned((n - j0 < uint64_t(G::kCols)) ? n - j0 : G::kCols);
                T* sb = stages + uint64_t(st) * G::kStageElems;
#pragma unroll
                for (int q = 0; q < SEG / 512; ++q) {
                    const unsigned e0 = unsigned(q * 32 + lane) * E; // this lane's 16 B
                    if (e0 < cw) {
                        const T* src = A + (rb + pw) * n + j0 + e0;
                        for (int r = pw; r < rows; r += PW, src += PW * n)
                            cp_async16(sb + r * G::kPitch + e0, src);
                        if (pw == 0) cp_async16(sb + kOrdRows * G::kPitch + e0, x + j0 + e0);
                    }
                }
                cp_async_mbar_arrive(&full[st]);
            }
        }
        return;
    }

    // consumers: lane = one row of the current block
    uint64_t it = 0;
    for (uint64_t rb = r_begin; rb < r_end; rb += kOrdRows) {
        const int rr = warp * 32 + lane;
        const bool live = rb + rr < r_end;
        T acc = live ? c[rb + rr] : T(0);
        for (uint64_t t = 0; t < tiles; ++t, ++it) {
            const int st = int(it % kOrdStages);
            mbar_wait(&full[st], unsigned(it / kOrdStages) & 1u);
            const uint64_t j0 = t * G::kCols;
            const int cw = int((n - j0 < uint64_t(G::kCols)) ? n - j0 : G::kCols);
            const T* sb = stages + uint64_t(st) * G::kStageElems;
            const T* row = sb + rr * G::kPitch;
            const T* xs = sb + kOrdRows * G::kPitch;
            if (live) {
                for (int j = 0; j < cw; j += E) {
                    const Vec16<T> a = *reinterpret_cast<const Vec16<T>*>(row + j);
                    const Vec16<T> xv = *reinterpret_cast<const Vec16<T>*>(xs + j);
#pragma unroll
                    for (int e = 0; e < E; ++e) acc = add_rn(acc, mul_rn(a.v[e], xv.v[e]));
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        if (live) c[rb + rr] = acc;
    }
}

// ---------------------------------------------------------------------------
// TMA variant (CABL_ORD_CFG=tma): the producer is one thread issuing 2-D
// tensor copies.  A stage is 1 KB of each of the block's rows as 8 column
// boxes of 128 B x H rows (H = the block's row count, a multiple of 8; one
// tensor map per H), loaded with the 128-byte swizzle so lane rr reads its
// row's 16-byte chunk ch at rr*128 + ((ch ^ (rr & 7)) << 4) without bank
// conflicts; plus a 1-D bulk copy of the x slice.  CTAs own whole row octets
// so every box is fully used.
struct OrdMaps {
    CUtensorMap box[8]; // box heights 8, 16, ..., 64 rows
};

constexpr int kTmaBoxes = 8;                 // 128-byte column boxes per stage
constexpr unsigned kTmaBoxBytes = 64 * 128;  // room for 64 rows
constexpr unsigned kTmaStageBytes = kTmaBoxes * kTmaBoxBytes + 1024; // + x slice
constexpr int kTmaStages = 3;
constexpr unsigned kTmaSmem = kTmaStages * kTmaStageBytes + 1024;   // + alignment slack

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

template <typename T>
__global__ void __launch_bounds__(kOrdRows + 32, 1)
    gemv_rm_ordered_tma_kernel(const __grid_constant__ OrdMaps maps, const T* __restrict__ x,
                               T* __restrict__ c, uint64_t m, uint64_t n) {
    pdl_enter();
    constexpr int kBoxCols = 128 / int(sizeof(T));
    constexpr int kCols = kBoxCols * kTmaBoxes;
    constexpr int E = 16 / int(sizeof(T));
    extern __shared__ unsigned char smem_raw[];
    // 1024-byte aligned stage base (the 128-byte swizzle atom)
    const uint32_t raw = smem_u32(smem_raw);
    unsigned char* base = smem_raw + (((raw + 1023u) & ~1023u) - raw);
    __shared__ __align__(8) uint64_t full[kTmaStages];
    __shared__ __align__(8) uint64_t empty[kTmaStages];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const Partition part((m + 7) / 8, gridDim.x); // whole row octets per CTA
    const uint64_t o_end = part.begin(blockIdx.x + 1);
    const uint64_t r_begin = 8 * part.begin(blockIdx.x);
    const uint64_t r_end = 8 * o_end < m ? 8 * o_end : m;
    const uint64_t tiles = (n + kCols - 1) / kCols;

    if (tid == 0) {
        for (int s = 0; s < kTmaStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kOrdConsumerWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == kOrdConsumerWarps) { // producer: one elected thread
        if (lane != 0) return;
        uint64_t it = 0;
        for (uint64_t rb = r_begin; rb < r_end; rb += kOrdRows) {
            const uint64_t span = 8 * o_end - rb;
            const int H = int(span < uint64_t(kOrdRows) ? span : kOrdRows); // multiple of 8
            const CUtensorMap* map = &maps.box[H / 8 - 1];
            for (uint64_t t = 0; t < tiles; ++t, ++it) {
                const int st = int(it % kTmaStages);
                const unsigned use = unsigned(it / kTmaStages);
                if (use > 0) mbar_wait(&empty[st], (use - 1) & 1u);
                const uint64_t j0 = t * kCols;
                const unsigned cw = unsigned((n - j0 < uint64_t(kCols)) ? n - j0 : kCols);
                const int nbox = int((cw + kBoxCols - 1) / kBoxCols);
                unsigned char* sb = base + st * kTmaStageBytes;
                mbar_arrive_expect_tx(&full[st], unsigned(nbox) * unsigned(H) * 128u +
                                                     cw * unsigned(sizeof(T)));
                for (int b = 0; b < nbox; ++b)
                    tma_load_2d(sb + b * kTmaBoxBytes, map, int(j0) + b * kBoxCols, int(rb),
                                &full[st]);
                bulk_g2s(sb + kTmaBoxes * kTmaBoxBytes, x + j0, cw * unsigned(sizeof(T)),
                         &full[st]);
            }
        }
        return;
    }

    uint64_t it = 0;
    for (uint64_t rb = r_begin; rb < r_end; rb += kOrdRows) {
        const int rr = warp * 32 + lane;
        const bool live = rb + rr < r_end;
        T acc = live ? c[rb + rr] : T(0);
        const unsigned sw = unsigned(rr & 7);
        for (uint64_t t = 0; t < tiles; ++t, ++it) {
            const int st = int(it % kTmaStages);
            mbar_wait(&full[st], unsigned(it / kTmaStages) & 1u);
            const uint64_t j0 = t * kCols;
            const int cw = int((n - j0 < uint64_t(kCols)) ? n - j0 : kCols);
            const unsigned char* sb = base + st * kTmaStageBytes;
            const unsigned char* xs = sb + kTmaBoxes * kTmaBoxBytes;
            if (live) {
                for (int b = 0; b * kBoxCols < cw; ++b) {
                    const unsigned char* rowp = sb + b * kTmaBoxBytes + rr * 128;
                    const int chunks = ((cw - b * kBoxCols < kBoxCols) ? cw - b * kBoxCols
                                                                        : kBoxCols) / E;
#pragma unroll 8
                    for (int ch = 0; ch < chunks; ++ch) {
                        const Vec16<T> a =
                            *reinterpret_cast<const Vec16<T>*>(rowp + ((unsigned(ch) ^ sw) << 4));
                        const Vec16<T> xv =
                            *reinterpret_cast<const Vec16<T>*>(xs + b * 128 + ch * 16);
#pragma unroll
                        for (int e = 0; e < E; ++e) acc = add_rn(acc, mul_rn(a.v[e], xv.v[e]));
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
        if (live) c[rb + rr] = acc;
    }
}

} // namespace

template <typename T> bool gemv_rm_ordered_ok(const T* A, const T* x, uint64_t m, uint64_t n) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(A), xp = reinterpret_cast<uintptr_t>(x);
    return (a & 15u) == 0 && (xp & 15u) == 0 && (n * sizeof(T)) % 16 == 0 &&
           m >= uint64_t(sm_count()) * 32 && m < (uint64_t(1) << 31) && n < (uint64_t(1) << 31);
}

namespace {

template <typename T, int SEG, int NS, int PW>
void ordered_launch_cfg(const T* A, uint64_t m, uint64_t n, const T* x, T* c, cudaStream_t s,
                        unsigned grid) {

    using G = OrdGeom<T, SEG, NS>;
    static std::atomic<unsigned long long> configured{0};
    ensure_dyn_smem(gemv_rm_ordered_kernel<T, SEG, NS, PW>, int(G::kSmem), configured);
    launch(gemv_rm_ordered_kernel<T, SEG, NS, PW>, grid, kOrdRows + 32 * PW, G::kSmem, s, A, x, c,
           m, n);
}

// CABL_ORD_CFG=seg,stages,producer_warps (tuning knob).  G1 / G4 b2b:
// 1024,3,1 45.8 / 2647 us (default); 1024,3,2 46.6 / 2616; 1024,3,4 50.8 /
// 2785; 512,5,1 51.8 / 2788; 512,5,2 52.1 / 2934; 1536,2,1 51.1 / 2805;
// tma (2-D tensor copies, 128-byte swizzle) 53.0 / 2636.  Every variant lands
// near 6.5 TB/s on G4: the limit is the DRAM pattern of ~9.5k concurrent row
// streams read 1 KB at a time (the sweep reads 8 KB runs), not the copy engine.
int ordered_cfg() {
    static const int cfg = [] {
        const char* e = tuning_env("CABL_ORD_CFG");
        if (!e) return 1;
        if (!std::strcmp(e, "512,5,1")) return 0;
        if (!std::strcmp(e, "1024,3,1")) return 1;
        if (!std::strcmp(e, "1024,3,2")) return 2;
        if (!std::strcmp(e, "tma")) return 5;
        return 1;
    }();
    return cfg;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

template <typename T>
cudaError_t ordered_launch_tma(const T* A, uint64_t m, uint64_t n, const T* x, T* c,
                               cudaStream_t s, unsigned grid) {
    auto encode = tensor_map_encoder();
    if (!encode) return cudaErrorNotSupported;
    // the maps depend only on (A, m, n): cache the last set per thread
    thread_local const void* last_a = nullptr;
    thread_local uint64_t last_m = 0, last_n = 0, last_s = 0;
    thread_local OrdMaps maps;
    if (last_a != A || last_m != m || last_n != n || last_s != sizeof(T)) {
        const CUtensorMapDataType dt =
            sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
        const cuuint64_t dims[2] = {n, m};
        const cuuint64_t strides[1] = {n * sizeof(T)};
        const cuuint32_t estr[2] = {1, 1};
        for (int h = 0; h < 8; ++h) {
            const cuuint32_t box[2] = {cuuint32_t(128 / sizeof(T)), cuuint32_t(8 * (h + 1))};
            if (encode(&maps.box[h], dt, 2, const_cast<T*>(A), dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
                last_a = nullptr;
                return cudaErrorInvalidValue;
            }
        }
        last_a = A;
        last_m = m;
        last_n = n;
        last_s = sizeof(T);
    }
    static std::atomic<unsigned long long> configured{0};
    ensure_dyn_smem(gemv_rm_ordered_tma_kernel<T>, int(kTmaSmem), configured);
    launch(gemv_rm_ordered_tma_kernel<T>, grid, kOrdRows + 32, kTmaSmem, s, maps, x, c, m, n);
    return cudaSuccess;
}

} // namespace

template <typename T>
cudaError_t gemv_rm_ordered_launch(const T* A, uint64_t m, uint64_t n, const T* x, T* c,
                                   cudaStream_t s, LaunchInfo* info) {
    const uint64_t sms = uint64_t(sm_count());
    const unsigned grid = unsigned(m < sms ? m : sms);
    switch (ordered_cfg()) {
    case 0: ordered_launch_cfg<T, 512, 5, 1>(A, m, n, x, c, s, grid); break;
    case 2: ordered_launch_cfg<T, 1024, 3, 2>(A, m, n, x, c, s, grid); break;
    case 5:
        if (cudaError_t e = ordered_launch_tma<T>(A, m, n, x, c, s, grid)) return e;
        break;
    default: ordered_launch_cfg<T, 1024, 3, 1>(A, m, n, x, c, s, grid); break;
    }
    if (info) info->ctas = grid;
    return cudaGetLastError();
}

template bool gemv_rm_ordered_ok<float>(const float*, const float*, uint64_t, uint64_t);
template bool gemv_rm_ordered_ok<double>(const double*, const double*, uint64_t, uint64_t);
template cudaError_t gemv_rm_ordered_launch<float>(const float*, uint64_t, uint64_t, const float*,
                                                   float*, cudaStream_t, LaunchInfo*);
template cudaError_t gemv_rm_ordered_launch<double>(const double*, uint64_t, uint64_t,
                                                    const double*, double*, cudaStream_t,
                                                    LaunchInfo*);

} // namespace cabl_dev

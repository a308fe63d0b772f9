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
// row): C is cut into tiles of 4 rows x 256 column vectors (4 x 8 KB for
// fp32), numbered so that consecutive tiles are one contiguous stretch of C.
// A single wave of CTAs (4 per SM) draws tiles from an atomic counter — SMs
// that get faster memory service simply take more tiles, which measured
// 8% faster on 8192^2 than static row ranges.  A thread owns one 32-byte
// column vector of its tile: its v slice is one L1-cached load, u[o] a
// warp-uniform broadcast, and C streams through a 256-bit read-modify-write
// (no L1 allocation) with the tile's 4 rows of loads in flight.  Every
// element is read, FMA'd and written by exactly one thread once, so the
// bits do not depend on which CTA took which tile.
//
// Generic path (ragged / unaligned / narrow rows, and the single-CTA small
// path the reference runs on one thread, kernels.hpp:286-287): flattened
// element-wise grid-stride FMA.
//
// Algorithmic bytes per launch: 2*m*n*s + m*s + n*s.
#include "common.cuh"
#include "kernels.cuh"

#include <cstdio>
#include <cstdlib>

namespace cabl_dev {

namespace {

constexpr int kGerBlock = 256;
constexpr int kGerCtasPerSm = 4;
constexpr int kGerUnroll = 4;
constexpr uint64_t kGerMinVecs = 128;
// measured on 8192^2 fp32 (tools/tune.py): static row ranges 87.1 us, tiles
// in grid-stride order 86.0 us, tiles from an atomic counter 80.0 us (RT = 4;
// RT = 8 spills at 4 CTAs/SM)
constexpr int kGerDefaultMode = 2;
constexpr int kGerTileRows = 4;

template <typename T, int U>
__global__ void __launch_bounds__(kGerBlock, kGerCtasPerSm)
    ger_vec_kernel(const T* __restrict__ u, const T* __restrict__ v, T* __restrict__ C,
                   uint64_t outer, uint64_t nvec, unsigned col_blocks) {
    pdl_enter();
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

// Tiled variants: a tile is RT rows x one 256-vector column block; tiles are
// numbered row-chunk-major (consecutive tiles = one contiguous stretch of C)
// and handed out either in grid-stride order (DYN = false) or from an
// atomic tile queue (DYN = true, common.cuh dyn_next).  Every element is still read, FMA'd and written by
// exactly one thread, so the result is the same bits either way.
template <typename T, int RT, bool DYN>
__global__ void __launch_bounds__(kGerBlock, kGerCtasPerSm)
    ger_tile_kernel(const T* __restrict__ u, const T* __restrict__ v, T* __restrict__ C,
                    uint64_t outer, uint64_t nvec, unsigned col_blocks, uint64_t tiles,
                    unsigned* __restrict__ counter) {
    pdl_enter();
    __shared__ unsigned long long next_sh[2];
    const Vec<T>* V_ = reinterpret_cast<const Vec<T>*>(v);
    Vec<T>* Cv = reinterpret_cast<Vec<T>*>(C);
    uint64_t t = blockIdx.x; // first tile static, the rest from the queue
    int parity = 0;
    while (t < tiles) {
        if (DYN && threadIdx.x == 0) next_sh[parity ^ 1] = dyn_next(counter, tiles); // prefetch
        const unsigned cb = unsigned(t % col_blocks);
        const uint64_t r0 = (t / col_blocks) * RT;
        const uint64_t vc = uint64_t(cb) * kGerBlock + threadIdx.x;
        if (vc < nvec) {
            const Vec<T> vv = ld_reuse(V_ + vc);
            const uint64_t r1 = (r0 + RT < outer) ? r0 + RT : outer;
            if (r1 - r0 == RT) {
                Vec<T> cv[RT];
                T uo[RT];
#pragma unroll
                for (int k = 0; k < RT; ++k) {
                    cv[k] = ld_rmw(Cv + (r0 + k) * nvec + vc);
                    uo[k] = __ldg(u + r0 + k);
                }
#pragma unroll
                for (int k = 0; k < RT; ++k) {
#pragma unroll
                    for (int e = 0; e < Vec<T>::N; ++e) cv[k].v[e] = fma_rn(uo[k], vv.v[e], cv[k].v[e]);
                    st_stream(Cv + (r0 + k) * nvec + vc, cv[k]);
                }
            } else {
                for (uint64_t o = r0; o < r1; ++o) {
                    Vec<T> cv = ld_rmw(Cv + o * nvec + vc);
                    const T uo = __ldg(u + o);
#pragma unroll
                    for (int e = 0; e < Vec<T>::N; ++e) cv.v[e] = fma_rn(uo, vv.v[e], cv.v[e]);
                    st_stream(Cv + o * nvec + vc, cv);
                }
            }
        }
        if (DYN) {
            __syncthreads();
            parity ^= 1;
            t = next_sh[parity];
        } else {
            t += gridDim.x;
        }
    }
}

// Any alignment, any width (the vector tile kernels need 32-byte-aligned
// rows of >= kGerMinVecs vectors): C flattened, slabs of kGerBlock *
// kGerFlatU consecutive elements in grid-stride (sweep) order; thread t takes
// elements t, t + kGerBlock, ... of a slab — coalesced whatever the row width
// — with all kGerFlatU loads of C (and y, x from L1) issued before any store.
// A thread divides once per slab for its (row, column) and then steps by the
// precomputed kGerBlock / inner, kGerBlock % inner.  One FMA per element:
// bitwise ger_ref like every other path.  (Row tiles of 4096 columns, the
// previous fallback, left short rows mostly idle: 256 x 262144 col-major fp32
// ran at 1.2 TB/s.)
constexpr int kGerFlatU = 16;

template <typename T>
__global__ void __launch_bounds__(kGerBlock)
    ger_flat_kernel(const T* __restrict__ u, const T* __restrict__ v, T* __restrict__ C,
                    uint64_t outer, uint64_t inner, uint64_t step_o, uint64_t step_i) {
    pdl_enter();
    constexpr uint64_t kSlab = uint64_t(kGerBlock) * kGerFlatU;
    const uint64_t total = outer * inner;
    for (uint64_t s0 = uint64_t(blockIdx.x) * kSlab; s0 < total; s0 += uint64_t(gridDim.x) * kSlab) {
        const uint64_t e0 = s0 + threadIdx.x;
        uint64_t o = e0 / inner, i = e0 - o * inner;
        T cv[kGerFlatU], vv[kGerFlatU], uo[kGerFlatU];
#pragma unroll
        for (int k = 0; k < kGerFlatU; ++k) {
            const uint64_t e = e0 + uint64_t(k) * kGerBlock;
            if (e < total) {
                cv[k] = __ldcs(C + e);
                vv[k] = __ldg(v + i);
                uo[k] = __ldg(u + o);
            }
            o += step_o; // advance (o, i) by kGerBlock elements
            i += step_i;
            if (i >= inner) {
                i -= inner;
                ++o;
            }
        }
#pragma unroll
        for (int k = 0; k < kGerFlatU; ++k) {
            const uint64_t e = e0 + uint64_t(k) * kGerBlock;
            if (e < total) __stcs(C + e, fma_rn(uo[k], vv[k], cv[k]));
        }
    }
}

// Short aligned rows (inner % V == 0, C and y 32-byte aligned, fewer than
// kGerMinVecs vectors per row): the flat sweep in 32-byte vectors — a vector
// never straddles a row, so each one is one 256-bit load + store of C, one
// 256-bit load of y (L1) and one scalar x.  256 MiB fp32 with 64-column rows
// ran at 4.2 TB/s through the scalar flat kernel.
constexpr int kGerFlatVecU = 4; // 32-byte vectors in flight per thread

template <typename T>
__global__ void __launch_bounds__(kGerBlock, 2)
    ger_flat_vec_kernel(const T* __restrict__ u, const T* __restrict__ v, T* __restrict__ C,
                        uint64_t outer, uint64_t ivec, uint64_t step_o, uint64_t step_i) {
    pdl_enter();
    constexpr uint64_t kSlab = uint64_t(kGerBlock) * kGerFlatVecU;
    const uint64_t total = outer * ivec; // vectors
    const Vec<T>* V_ = reinterpret_cast<const Vec<T>*>(v);
    Vec<T>* Cv = reinterpret_cast<Vec<T>*>(C);
    for (uint64_t s0 = uint64_t(blockIdx.x) * kSlab; s0 < total; s0 += uint64_t(gridDim.x) * kSlab) {
        const uint64_t q0 = s0 + threadIdx.x;
        uint64_t o = q0 / ivec, i = q0 - o * ivec;
        Vec<T> cv[kGerFlatVecU], vv[kGerFlatVecU];
        T uo[kGerFlatVecU];
#pragma unroll
        for (int k = 0; k < kGerFlatVecU; ++k) {
            const uint64_t q = q0 + uint64_t(k) * kGerBlock;
            if (q < total) {
                cv[k] = ld_rmw(Cv + q);
                vv[k] = ld_reuse(V_ + i);
                uo[k] = __ldg(u + o);
            }
            o += step_o;
            i += step_i;
            if (i >= ivec) {
                i -= ivec;
                ++o;
            }
        }
#pragma unroll
        for (int k = 0; k < kGerFlatVecU; ++k) {
            const uint64_t q = q0 + uint64_t(k) * kGerBlock;
            if (q < total) {
#pragma unroll
                for (int e = 0; e < Vec<T>::N; ++e) cv[k].v[e] = fma_rn(uo[k], vv[k].v[e], cv[k].v[e]);
                st_stream(Cv + q, cv[k]);
            }
        }
    }
}

// Rows of whole 16-byte (not 32-byte) vectors — n = 4 mod 8 floats, or C / y
// only 16-byte aligned: the same flat sweep with 16-byte vectors.
struct alignas(16) F4 {
    float v[4];
};
struct alignas(16) D2 {
    double v[2];
};
template <typename T> struct H16;
template <> struct H16<float> {
    using type = F4;
    static constexpr int N = 4;
};
template <> struct H16<double> {
    using type = D2;
    static constexpr int N = 2;
};
__device__ __forceinline__ F4 ld_rmw16(const F4* p) {
    F4 r;
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ D2 ld_rmw16(const D2* p) {
    D2 r;
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(r.v[0]), "=d"(r.v[1])
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ F4 ld_reuse16(const F4* p) {
    F4 r;
    asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ D2 ld_reuse16(const D2* p) {
    D2 r;
    asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream16(F4* p, const F4& r) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(r.v[0]),
                 "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3])
                 : "memory");
}
__device__ __forceinline__ void st_stream16(D2* p, const D2& r) {
    asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(r.v[0]),
                 "d"(r.v[1])
                 : "memory");
}

constexpr int kGerFlatHU = 8; // 16-byte vectors in flight per thread

template <typename T>
__global__ void __launch_bounds__(kGerBlock, 2)
    ger_flat_hvec_kernel(const T* __restrict__ u, const T* __restrict__ v, T* __restrict__ C,
                         uint64_t outer, uint64_t ivec, uint64_t step_o, uint64_t step_i) {
    pdl_enter();
    using HV = typename H16<T>::type;
    constexpr uint64_t kSlab = uint64_t(kGerBlock) * kGerFlatHU;
    const uint64_t total = outer * ivec;
    const HV* V_ = reinterpret_cast<const HV*>(v);
    HV* Cv = reinterpret_cast<HV*>(C);
    for (uint64_t s0 = uint64_t(blockIdx.x) * kSlab; s0 < total; s0 += uint64_t(gridDim.x) * kSlab) {
        const uint64_t q0 = s0 + threadIdx.x;
        uint64_t o = q0 / ivec, i = q0 - o * ivec;
        HV cv[kGerFlatHU], vv[kGerFlatHU];
        T uo[kGerFlatHU];
#pragma unroll
        for (int k = 0; k < kGerFlatHU; ++k) {
            const uint64_t q = q0 + uint64_t(k) * kGerBlock;
            if (q < total) {
                cv[k] = ld_rmw16(Cv + q);
                vv[k] = ld_reuse16(V_ + i);
                uo[k] = __ldg(u + o);
            }
            o += step_o;
            i += step_i;
            if (i >= ivec) {
                i -= ivec;
                ++o;
            }
        }
#pragma unroll
        for (int k = 0; k < kGerFlatHU; ++k) {
            const uint64_t q = q0 + uint64_t(k) * kGerBlock;
            if (q < total) {
#pragma unroll
                for (int e = 0; e < H16<T>::N; ++e) cv[k].v[e] = fma_rn(uo[k], vv[k].v[e], cv[k].v[e]);
                st_stream16(Cv + q, cv[k]);
            }
        }
    }
}

// Any row width >= V and any element-aligned C (odd n, x[k:]-style offsets):
// C flattened and cut into 32-byte vectors at C's first 32-byte boundary.  A
// vector may straddle a row boundary (at most once, since inner >= V); its
// elements take y[i..] and y[0..] and x[o], x[o+1] accordingly — scalar y
// reads (shared memory when y fits and YS, else L1), while C moves in 256-bit
// loads and stores with U vectors in flight per thread (EARLY: the y / x reads
// of all U vectors issued with the C loads).  The < V elements before the
// boundary and after the last whole vector run in CTA 0's scalar prologue.
// The flat scalar sweep it replaces ran 8192 x 8193 fp32 at 4.2 TB/s
// (129 us flushed); this kernel 92 us (5.8 TB/s); fp64 4096 x 8193 119 -> 82 us.
constexpr size_t kGerYsMax = 96 * 1024; // y staged in shared memory up to this size

template <typename T, bool YS, int U, bool EARLY>
__global__ void __launch_bounds__(kGerBlock, 2)
    ger_flat_any_kernel(const T* __restrict__ u, const T* __restrict__ v, T* __restrict__ C,
                        uint64_t outer, uint64_t inner, uint64_t head, uint64_t nvec,
                        uint64_t step_o, uint64_t step_i) {
    pdl_enter();
    constexpr int V = Vec<T>::N;
    const uint64_t total = outer * inner;
    extern __shared__ unsigned char ger_smem[];
    T* ys = reinterpret_cast<T*>(ger_smem);
    if (YS) { // y staged in shared memory (rows that fit): LDS instead of L1 LDG
        for (uint64_t j = threadIdx.x; j < inner; j += kGerBlock) ys[j] = __ldg(v + j);
        __syncthreads();
    }
    if (blockIdx.x == 0) { // head and tail elements
        const uint64_t tail0 = head + nvec * V;
        for (uint64_t e = threadIdx.x; e < head + (total - tail0); e += kGerBlock) {
            const uint64_t f = e < head ? e : tail0 + (e - head);
            const uint64_t o = f / inner, i = f - o * inner;
            C[f] = fma_rn(u[o], v[i], C[f]);
        }
    }
    constexpr uint64_t kSlab = uint64_t(kGerBlock) * U;
    constexpr int UE = EARLY ? U : 1; // vectors whose y / x are held in registers
    Vec<T>* Cv = reinterpret_cast<Vec<T>*>(C + head);
    for (uint64_t s0 = uint64_t(blockIdx.x) * kSlab; s0 < nvec; s0 += uint64_t(gridDim.x) * kSlab) {
        const uint64_t q0 = s0 + threadIdx.x;
        const uint64_t f0 = head + q0 * V; // flat index of the vector's first element
        uint64_t o0;
        if ((f0 >> 32) == 0 && (inner >> 32) == 0) { // 32-bit division when it fits
            o0 = unsigned(f0) / unsigned(inner);
        } else {
            o0 = f0 / inner;
        }
        const uint64_t i0 = f0 - o0 * inner;
        // EARLY: every load (C, y, x) of the U vectors issued before any FMA;
        // otherwise the C loads first and y / x per vector when it is consumed
        Vec<T> cv[U];
        T yv[UE][V], ua[UE], ub[UE];
        uint64_t o = o0, i = i0;
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint64_t q = q0 + uint64_t(k) * kGerBlock;
            if (q < nvec) {
                cv[k] = ld_rmw(Cv + q);
                if (EARLY) {
                    ua[k % UE] = __ldg(u + o);
                    ub[k % UE] = (i + V > inner) ? __ldg(u + o + 1) : ua[k % UE];
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        const uint64_t ie = i + e;
                        const uint64_t j = ie < inner ? ie : ie - inner;
                        yv[k % UE][e] = YS ? ys[j] : __ldg(v + j);
                    }
                }
            }
            o += step_o; // advance (o, i) by kGerBlock vectors
            i += step_i;
            if (i >= inner) {
                i -= inner;
                ++o;
            }
        }
        o = o0;
        i = i0;
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint64_t q = q0 + uint64_t(k) * kGerBlock;
            if (q < nvec) {
                if (!EARLY) {
                    ua[0] = __ldg(u + o);
                    ub[0] = (i + V > inner) ? __ldg(u + o + 1) : ua[0];
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        const uint64_t ie = i + e;
                        const uint64_t j = ie < inner ? ie : ie - inner;
                        yv[0][e] = YS ? ys[j] : __ldg(v + j);
                    }
                }
#pragma unroll
                for (int e = 0; e < V; ++e)
                    cv[k].v[e] = fma_rn(i + e < inner ? ua[k % UE] : ub[k % UE], yv[k % UE][e],
                                        cv[k].v[e]);
                st_stream(Cv + q, cv[k]);
            }
            o += step_o;
            i += step_i;
            if (i >= inner) {
                i -= inner;
                ++o;
            }
        }
    }
}

struct GerAnyCfg {
    int ys, u, early, per_sm;
};
// CABL_GER_ANY_CFG="ys,u,early,ctas_per_sm" (tuning only)
inline GerAnyCfg ger_any_cfg(size_t elem) {
    static const GerAnyCfg forced = [] {
        GerAnyCfg c{-1, 0, 0, 0};
        if (const char* e = tuning_env("CABL_GER_ANY_CFG"))
            sscanf(e, "%d,%d,%d,%d", &c.ys, &c.u, &c.early, &c.per_sm);
        return c;
    }();
    if (forced.ys >= 0) return forced;
    // measured (tools/ger_odd.py, 10 shapes per dtype, flushed): fp32 y in shared
    // memory, fp64 y from L1 with a second wave of CTAs
    return elem == 4 ? GerAnyCfg{1, 4, 1, 2} : GerAnyCfg{0, 4, 1, 4};
}

template <typename T, bool YS, int U, bool EARLY>
void ger_any_go(unsigned per_sm, const T* u, const T* v, T* C, uint64_t outer, uint64_t inner,
                uint64_t head, uint64_t nvec, cudaStream_t s, LaunchInfo* info) {
    constexpr int V = Vec<T>::N;
    constexpr uint64_t kSlab = uint64_t(kGerBlock) * U;
    const uint64_t slabs = (nvec + kSlab - 1) / kSlab;
    const uint64_t cap = uint64_t(sm_count()) * per_sm;
    const unsigned grid = unsigned(slabs < cap ? slabs : cap);
    const uint64_t stepv = uint64_t(kGerBlock) * V; // elements between a thread's vectors
    const size_t ysz = YS ? size_t(inner) * sizeof(T) : 0;
    if (YS && ysz > 48 * 1024) {
        static std::atomic<unsigned long long> attr{0};
        ensure_dyn_smem(ger_flat_any_kernel<T, YS, U, EARLY>, int(kGerYsMax), attr);
    }
    launch(ger_flat_any_kernel<T, YS, U, EARLY>, grid, kGerBlock, ysz, s, u, v, C, outer, inner,
           head, nvec, stepv / inner, stepv % inner);
    if (info) info->ctas = grid;
}

// One-element rows (inner == 1: a col-major C with one row, or a row-major C
// with one column): C[o] = fma(u[o], v[0], C[o]) — an AXPY over two
// contiguous vectors, in 256-bit loads of u and C when both share their
// 32-byte offset (the < V head and tail elements in CTA 0).  The flat scalar
// sweep ran 1 x 2^26 col-major fp32 at 5.7 TB/s (141 us).
template <typename T>
__global__ void __launch_bounds__(kGerBlock)
    ger_axpy_kernel(const T* __restrict__ u, const T* __restrict__ v, T* __restrict__ C,
                    uint64_t outer, uint64_t head) {
    pdl_enter();
    constexpr int V = Vec<T>::N;
    constexpr int U = 4;
    const T v0 = __ldg(v);
    const uint64_t nvec = (outer - head) / V;
    if (blockIdx.x == 0) {
        const uint64_t tail0 = head + nvec * V;
        for (uint64_t e = threadIdx.x; e < head + (outer - tail0); e += kGerBlock) {
            const uint64_t o = e < head ? e : tail0 + (e - head);
            C[o] = fma_rn(u[o], v0, C[o]);
        }
    }
    const Vec<T>* Uv = reinterpret_cast<const Vec<T>*>(u + head);
    Vec<T>* Cv = reinterpret_cast<Vec<T>*>(C + head);
    const uint64_t T_all = uint64_t(gridDim.x) * kGerBlock;
    for (uint64_t q0 = uint64_t(blockIdx.x) * kGerBlock + threadIdx.x; q0 < nvec; q0 += U * T_all) {
        Vec<T> cv[U], uv[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint64_t q = q0 + uint64_t(k) * T_all;
            if (q < nvec) {
                cv[k] = ld_rmw(Cv + q);
                uv[k] = ld_stream(Uv + q);
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint64_t q = q0 + uint64_t(k) * T_all;
            if (q < nvec) {
#pragma unroll
                for (int e = 0; e < V; ++e) cv[k].v[e] = fma_rn(uv[k].v[e], v0, cv[k].v[e]);
                st_stream(Cv + q, cv[k]);
            }
        }
    }
}

} // namespace

// CABL_GER_MODE (tuning only): 0 static row ranges, 1 tiles in grid-stride
// order, 2 tiles from an atomic counter (default).
inline int ger_mode() {
    static const int m = [] {
        const char* e = tuning_env("CABL_GER_MODE");
        return e ? atoi(e) : kGerDefaultMode;
    }();
    return m;
}

// CABL_GER_ANY=0 sends odd / misaligned rows back to the scalar flat sweep (A/B only).
inline bool ger_any_enabled() {
    static const bool on = [] {
        const char* e = tuning_env("CABL_GER_ANY");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}

template <typename T>
WorkspaceNeed ger_need(const T*, const T*, uint64_t, uint64_t) {
    WorkspaceNeed w;
    w.counters = 1;
    return w;
}

template <typename T>
cudaError_t ger_launch(const T* u, const T* v, T* C, uint64_t outer, uint64_t inner,
                       bool small, const Workspace& ws, cudaStream_t s, LaunchInfo* info) {
    if (info) info->ctas = 0;
    if (outer == 0 || inner == 0) return cudaSuccess;
    constexpr int V = Vec<T>::N;
    const bool vec_ok = aligned32(C) && aligned32(v) && inner % V == 0 &&
                        inner / V >= kGerMinVecs;
    const int mode = ger_mode();
    if (!small && vec_ok && mode != 0) {
        const uint64_t nvec = inner / V;
        const unsigned col_blocks = unsigned((nvec + kGerBlock - 1) / kGerBlock);
        const uint64_t tiles = ((outer + kGerTileRows - 1) / kGerTileRows) * col_blocks;
        const uint64_t cap = uint64_t(sm_count()) * kGerCtasPerSm;
        const unsigned grid = unsigned(tiles < cap ? tiles : cap);
        if (mode == 2)
            launch(ger_tile_kernel<T, kGerTileRows, true>, grid, kGerBlock, 0, s, 
                u, v, C, outer, nvec, col_blocks, tiles, ws.counters);
        else
            launch(ger_tile_kernel<T, kGerTileRows, false>, grid, kGerBlock, 0, s, 
                u, v, C, outer, nvec, col_blocks, tiles, ws.counters);
        if (info) info->ctas = grid;
    } else if (!small && vec_ok) {
        const uint64_t nvec = inner / V;
        const unsigned col_blocks = unsigned((nvec + kGerBlock - 1) / kGerBlock);
        const uint64_t target = uint64_t(sm_count()) * kGerCtasPerSm;
        uint64_t row_blocks = target / col_blocks;
        if (row_blocks < 1) row_blocks = 1;
        if (row_blocks > outer) row_blocks = outer;
        const unsigned grid = unsigned(row_blocks * col_blocks);
        launch(ger_vec_kernel<T, kGerUnroll>, grid, kGerBlock, 0, s, u, v, C, outer, nvec, col_blocks);
        if (info) info->ctas = grid;
    } else if (!small && aligned32(C) && aligned32(v) && inner % V == 0) {
        // short aligned rows: flat sweep in 32-byte vectors
        constexpr uint64_t kSlab = uint64_t(kGerBlock) * kGerFlatVecU;
        const uint64_t ivec = inner / V;
        const uint64_t slabs = (outer * ivec + kSlab - 1) / kSlab;
        const uint64_t cap = uint64_t(sm_count()) * 8;
        const unsigned grid = unsigned(slabs < cap ? slabs : cap);
        launch(ger_flat_vec_kernel<T>, grid, kGerBlock, 0, s, u, v, C, outer, ivec,
               uint64_t(kGerBlock) / ivec, uint64_t(kGerBlock) % ivec);
        if (info) info->ctas = grid;
    } else if (!small && (reinterpret_cast<uintptr_t>(C) & 15u) == 0 &&
               (reinterpret_cast<uintptr_t>(v) & 15u) == 0 && inner % (16 / sizeof(T)) == 0) {
        // rows of whole 16-byte vectors: flat sweep in 16-byte vectors
        constexpr uint64_t kSlab = uint64_t(kGerBlock) * kGerFlatHU;
        const uint64_t ivec = inner / (16 / sizeof(T));
        const uint64_t slabs = (outer * ivec + kSlab - 1) / kSlab;
        const uint64_t cap = uint64_t(sm_count()) * 8;
        const unsigned grid = unsigned(slabs < cap ? slabs : cap);
        launch(ger_flat_hvec_kernel<T>, grid, kGerBlock, 0, s, u, v, C, outer, ivec,
               uint64_t(kGerBlock) / ivec, uint64_t(kGerBlock) % ivec);
        if (info) info->ctas = grid;
    } else if (!small && inner == 1 && outer >= uint64_t(sm_count()) * kGerBlock * V &&
               reinterpret_cast<uintptr_t>(C) % sizeof(T) == 0 &&
               (reinterpret_cast<uintptr_t>(C) & 31u) == (reinterpret_cast<uintptr_t>(u) & 31u)) {
        // one-element rows: an AXPY over u and C
        const uint64_t mis = (reinterpret_cast<uintptr_t>(C) & 31u) / sizeof(T);
        const uint64_t head = mis ? uint64_t(V) - mis : 0;
        const uint64_t nvec = (outer - head) / V;
        const uint64_t per = uint64_t(kGerBlock) * 4;
        const uint64_t cap = uint64_t(sm_count()) * 4;
        const uint64_t want = (nvec + per - 1) / per;
        const unsigned grid = unsigned(want < cap ? (want < 1 ? 1 : want) : cap);
        launch(ger_axpy_kernel<T>, grid, kGerBlock, 0, s, u, v, C, outer, head);
        if (info) info->ctas = grid;
    } else if (!small && inner >= uint64_t(V) && ger_any_enabled() &&
               reinterpret_cast<uintptr_t>(C) % sizeof(T) == 0 &&
               outer * inner >= uint64_t(sm_count()) * kGerBlock * V) {
        // any width >= V, element-aligned C: flat sweep in 32-byte vectors of C
        const uint64_t mis = (reinterpret_cast<uintptr_t>(C) & 31u) / sizeof(T);
        const uint64_t head = mis ? uint64_t(V) - mis : 0;
        const uint64_t nvec = (outer * inner - head) / V;
        GerAnyCfg c = ger_any_cfg(sizeof(T));
        if (size_t(inner) * sizeof(T) > kGerYsMax) c.ys = 0;
        const unsigned ps = unsigned(c.per_sm);
#define CABL_GER_ANY(YS_, U_, E_)                                                                 \
    if (c.ys == YS_ && c.u == U_ && c.early == E_)                                                \
        ger_any_go<T, YS_, U_, E_>(ps, u, v, C, outer, inner, head, nvec, s, info);              \
    else
        CABL_GER_ANY(1, 8, 0) CABL_GER_ANY(0, 8, 0) CABL_GER_ANY(1, 4, 1) CABL_GER_ANY(0, 4, 1)
        CABL_GER_ANY(1, 4, 0) CABL_GER_ANY(0, 4, 0)
        ger_any_go<T, false, 4, true>(ps, u, v, C, outer, inner, head, nvec, s, info);
#undef CABL_GER_ANY
    } else {
        constexpr uint64_t kSlab = uint64_t(kGerBlock) * kGerFlatU;
        const uint64_t slabs = (outer * inner + kSlab - 1) / kSlab;
        const uint64_t cap = uint64_t(sm_count()) * 8;
        const unsigned grid = small ? 1u : unsigned(slabs < cap ? slabs : cap);
        launch(ger_flat_kernel<T>, grid, kGerBlock, 0, s, u, v, C, outer, inner,
               uint64_t(kGerBlock) / inner, uint64_t(kGerBlock) % inner);
        if (info) info->ctas = grid;
    }
    return cudaGetLastError();
}

template WorkspaceNeed ger_need<float>(const float*, const float*, uint64_t, uint64_t);
template WorkspaceNeed ger_need<double>(const double*, const double*, uint64_t, uint64_t);
template cudaError_t ger_launch<float>(const float*, const float*, float*, uint64_t, uint64_t,
                                       bool, const Workspace&, cudaStream_t, LaunchInfo*);
template cudaError_t ger_launch<double>(const double*, const double*, double*, uint64_t,
                                        uint64_t, bool, const Workspace&, cudaStream_t,
                                        LaunchInfo*);

} // namespace cabl_dev

// Col-major GEMV lab (exploration only, not the product): mid-size m, fp32.
// Hypothesis: the product's row-tiled split (CTA = row tile x column part)
// reads a fixed 1 KB slot of every 16 KB column per tile, and its SMs sit
// idle ~24% of the kernel (ncu sm__cycles_active 76%).  Variant here: every
// CTA streams FULL columns (a balanced contiguous column range per CTA, all
// m rows), writes an m-long partial, and a second PDL-chained kernel sums the
// parts' partials per row in part order (many CTAs, not one last arriver).
//
//   k_full<U>: grid P x 1024 threads; thread = (row-vector lane, column lane),
//              RPT row vectors per thread when m/8 > 1024
//   k_comb:    grid ceil(m/32) x 1024; thread (row r, part group g) sums parts
//              g, g+32, ...; then the 32 group sums per row in g order
#include <cstdint>
#include <cuda_runtime.h>

struct alignas(32) V8 { float v[8]; };

__device__ __forceinline__ V8 ld8(const V8* p) {
    V8 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                   "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
    return r;
}

// GS: columns dealt grid-stride (column j to CTA (j / col_lanes) % P), so all
// CTAs sweep the matrix front to back together, as the row-major sweep does
template <int U, int RPT, bool GS = false>
__global__ void __launch_bounds__(1024, 1)
    k_full(const float* __restrict__ A, const float* __restrict__ x, uint64_t m, uint64_t n,
           float* __restrict__ partials, int row_lanes) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ float sm[8192];
    const int tid = threadIdx.x;
    const int col_lanes = 1024 / row_lanes;
    const int rl = tid % row_lanes, cl = tid / row_lanes;
    const uint64_t mv = m / 8;
    const uint64_t q = n / gridDim.x, r = n % gridDim.x;
    const uint64_t cb = blockIdx.x * q + (blockIdx.x < r ? blockIdx.x : r);
    const uint64_t ce = cb + q + (blockIdx.x < r ? 1 : 0);
    const V8* Av = reinterpret_cast<const V8*>(A);
    V8 acc[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[k].v[e] = 0.f;
    const uint64_t jb = GS ? uint64_t(blockIdx.x) * col_lanes + cl : cb + cl;
    const uint64_t jend = GS ? n : ce;
    const uint64_t jstep = GS ? uint64_t(gridDim.x) * col_lanes : uint64_t(col_lanes);
    for (uint64_t j0 = jb; j0 < jend; j0 += jstep * U) {
        V8 a[U][RPT];
        float xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t j = j0 + uint64_t(u) * jstep;
            const bool ok = j < jend;
            xv[u] = ok ? __ldg(x + j) : 0.f;
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const uint64_t v = uint64_t(rl) + uint64_t(k) * row_lanes;
                if (ok && v < mv) a[u][k] = ld8(Av + j * mv + v);
                else
#pragma unroll
                    for (int e = 0; e < 8; ++e) a[u][k].v[e] = 0.f;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < RPT; ++k)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[k].v[e] = fmaf(a[u][k].v[e], xv[u], acc[k].v[e]);
    }
    float* out = partials + uint64_t(blockIdx.x) * m;
    if (col_lanes == 1) {
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const uint64_t v = uint64_t(rl) + uint64_t(k) * row_lanes;
            if (v < mv) *reinterpret_cast<V8*>(out + v * 8) = acc[k];
        }
        return;
    }
    // col_lanes > 1 (then RPT == 1 and m <= 8192): combine in smem, lane order
    if (uint64_t(rl) < mv)
#pragma unroll
        for (int e = 0; e < 8; ++e) sm[(cl * row_lanes + rl) * 8 + e] = 0.f;
    __syncthreads();
    for (int c2 = 0; c2 < col_lanes; ++c2) {
        if (cl == c2 && uint64_t(rl) < mv)
#pragma unroll
            for (int e = 0; e < 8; ++e) sm[rl * 8 + e] += acc[0].v[e];
        __syncthreads();
    }
    for (uint64_t i = tid; i < m; i += 1024) out[i] = sm[i];
}

__global__ void __launch_bounds__(1024, 1)
    k_comb(const float* __restrict__ partials, uint64_t m, unsigned parts, float* __restrict__ c) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ float red[32][33];
    const int rloc = threadIdx.x & 31, g = threadIdx.x >> 5;
    const uint64_t row = uint64_t(blockIdx.x) * 32 + rloc;
    float s = 0.f;
    if (row < m) {
        float v[8];
        unsigned p = g;
        for (; p + 7 * 32 < parts; p += 8 * 32) {
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldcg(partials + uint64_t(p + k * 32) * m + row);
#pragma unroll
            for (int k = 0; k < 8; ++k) s += v[k];
        }
        for (; p < parts; p += 32) s += __ldcg(partials + uint64_t(p) * m + row);
    }
    red[g][rloc] = s;
    __syncthreads();
    if (g == 0 && row < m) {
        float t = red[0][rloc];
        for (int k = 1; k < 32; ++k) t += red[k][rloc];
        c[row] += t;
    }
}

extern "C" int cmlab_run(int U, const float* A, const float* x, float* c, uint64_t m, uint64_t n,
                         float* partials, int parts, int pdl, void* stream) {
    const bool gs = U >= 100; // U + 100: grid-stride columns
    if (gs) U -= 100;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t mv = m / 8;
    int row_lanes = 1;
    while (uint64_t(row_lanes) < mv && row_lanes < 1024) row_lanes *= 2;
    const int rpt = int((mv + row_lanes - 1) / row_lanes);
#define GO(U_, R_)                                                                                \
    do {                                                                                          \
        if (gs) k_full<U_, R_, true><<<parts, 1024, 0, s>>>(A, x, m, n, partials, row_lanes);     \
        else k_full<U_, R_, false><<<parts, 1024, 0, s>>>(A, x, m, n, partials, row_lanes);       \
    } while (0)
    if (rpt == 1) { if (U == 2) GO(2, 1); else if (U == 8) GO(8, 1); else GO(4, 1); }
    else if (rpt == 2) { if (U == 2) GO(2, 2); else GO(4, 2); }
    else return -1;
#undef GO
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((m + 31) / 32));
    cfg.blockDim = dim3(1024);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, k_comb, (const float*)partials, m, (unsigned)parts, c);
    return int(cudaGetLastError());
}

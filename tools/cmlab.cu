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
    const int col_lanes = int(blockDim.x) / row_lanes;
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
    for (uint64_t i = tid; i < m; i += blockDim.x) out[i] = sm[i];
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

// grid-stride full columns with T threads per CTA (T in 256/512/1024) and
// `parts` CTAs; RPT row vectors per thread when m/8 > T
extern "C" int cmlab_gs_t(int T, const float* A, const float* x, float* c, uint64_t m,
                          uint64_t n, float* partials, int parts, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t mv = m / 8;
    int row_lanes = 1;
    while (uint64_t(row_lanes) < mv && row_lanes < T) row_lanes *= 2;
    const int rpt = int((mv + row_lanes - 1) / row_lanes);
    if (rpt == 1) k_full<2, 1, true><<<parts, T, 0, s>>>(A, x, m, n, partials, row_lanes);
    else if (rpt == 2) k_full<2, 2, true><<<parts, T, 0, s>>>(A, x, m, n, partials, row_lanes);
    else if (rpt == 4) k_full<1, 4, true><<<parts, T, 0, s>>>(A, x, m, n, partials, row_lanes);
    else return -1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((m + 31) / 32));
    cfg.blockDim = dim3(1024);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_comb, (const float*)partials, m, (unsigned)parts, c);
    return int(cudaGetLastError());
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

// ------------------------------------------------------------- stream-K
// Full columns per CTA: a static, balanced contiguous share of the first
// S = n - DYN columns, then chunks of CH columns of the rest from an atomic
// queue (the CTAs that finish their share early take more).  Static partial
// per CTA, one partial per dynamic chunk; a PDL-chained combine kernel sums,
// per row, the static partials in CTA order then the chunk partials in chunk
// order (deterministic: the data -> partial mapping never depends on the
// schedule).  The next chunk's loads are issued before the current chunk's
// lane combine, so the queue does not drain the load pipeline.
template <int RPT>
__device__ __forceinline__ void load_cols(const V8* Av, const float* x, uint64_t mv, int rl,
                                          int row_lanes, uint64_t j, uint64_t jend, V8* a,
                                          float& xv) {
    const bool ok = j < jend;
    xv = ok ? __ldg(x + j) : 0.f;
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const uint64_t v = uint64_t(rl) + uint64_t(k) * row_lanes;
        if (ok && v < mv) a[k] = ld8(Av + j * mv + v);
        else
#pragma unroll
            for (int e = 0; e < 8; ++e) a[k].v[e] = 0.f;
    }
}

// lane combine of acc (col lanes in order) into out[0..m)
__device__ __forceinline__ void lanes_to(float* sm, const V8& acc, int rl, int cl, int row_lanes,
                                         int col_lanes, uint64_t mv, uint64_t m, float* out) {
    if (uint64_t(rl) < mv)
#pragma unroll
        for (int e = 0; e < 8; ++e) sm[(uint64_t(cl) * row_lanes + rl) * 8 + e] = acc.v[e];
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) {
        float t = sm[i];
        for (int q = 1; q < col_lanes; ++q) t += sm[uint64_t(q) * row_lanes * 8 + i];
        out[i] = t;
    }
    __syncthreads();
}

template <int U>
__global__ void __launch_bounds__(1024, 1)
    k_sk(const float* __restrict__ A, const float* __restrict__ x, uint64_t m, uint64_t n,
         uint64_t S, uint64_t CH, float* __restrict__ part_static, float* __restrict__ part_dyn,
         unsigned* __restrict__ queue, int row_lanes) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    extern __shared__ float sm[]; // 1024 * 8 floats
    __shared__ unsigned long long next_sh;
    const int tid = threadIdx.x;
    const int col_lanes = 1024 / row_lanes;
    const int rl = tid % row_lanes, cl = tid / row_lanes;
    const uint64_t mv = m / 8;
    const V8* Av = reinterpret_cast<const V8*>(A);
    const uint64_t q = S / gridDim.x, r = S % gridDim.x;
    const uint64_t cb = blockIdx.x * q + (blockIdx.x < r ? blockIdx.x : r);
    const uint64_t ce = cb + q + (blockIdx.x < r ? 1 : 0);
    const uint64_t nch = (n - S + CH - 1) / CH;
    if (tid == 0) next_sh = atomicAdd(queue, 1u); // first dynamic chunk, fetched early
    V8 acc;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc.v[e] = 0.f;
    // static share
    for (uint64_t j0 = cb + cl; j0 < ce; j0 += uint64_t(col_lanes) * U) {
        V8 a[U];
        float xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            load_cols<1>(Av, x, mv, rl, row_lanes, j0 + uint64_t(u) * col_lanes, ce, &a[u], xv[u]);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc.v[e] = fmaf(a[u].v[e], xv[u], acc.v[e]);
    }
    __syncthreads(); // next_sh visible
    uint64_t c = next_sh;
    lanes_to(sm, acc, rl, cl, row_lanes, col_lanes, mv, m, part_static + uint64_t(blockIdx.x) * m);
    // dynamic chunks
    while (c < nch) {
        if (tid == 0) next_sh = atomicAdd(queue, 1u);
        const uint64_t j_lo = S + c * CH, j_hi = (j_lo + CH < n) ? j_lo + CH : n;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc.v[e] = 0.f;
        for (uint64_t j0 = j_lo + cl; j0 < j_hi; j0 += uint64_t(col_lanes) * U) {
            V8 a[U];
            float xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                load_cols<1>(Av, x, mv, rl, row_lanes, j0 + uint64_t(u) * col_lanes, j_hi, &a[u], xv[u]);
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int e = 0; e < 8; ++e) acc.v[e] = fmaf(a[u].v[e], xv[u], acc.v[e]);
        }
        __syncthreads();
        const uint64_t cn = next_sh;
        lanes_to(sm, acc, rl, cl, row_lanes, col_lanes, mv, m, part_dyn + c * m);
        c = cn;
    }
}

__global__ void __launch_bounds__(1024, 1)
    k_sk_comb(const float* __restrict__ ps, unsigned P, const float* __restrict__ pd, unsigned nch,
              uint64_t m, float* __restrict__ c, unsigned* queue) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ float red[32][33];
    const int rloc = threadIdx.x & 31, g = threadIdx.x >> 5;
    const uint64_t row = uint64_t(blockIdx.x) * 32 + rloc;
    // group g sums static parts g, g+32, ... then chunks g, g+32, ... (fixed)
    float s = 0.f;
    if (row < m) {
        for (unsigned p = g; p < P; p += 32) s += __ldcg(ps + uint64_t(p) * m + row);
        for (unsigned p = g; p < nch; p += 32) s += __ldcg(pd + uint64_t(p) * m + row);
    }
    red[g][rloc] = s;
    __syncthreads();
    if (g == 0 && row < m) {
        float t = red[0][rloc];
        for (int k = 1; k < 32; ++k) t += red[k][rloc];
        c[row] += t;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *queue = 0u;
}

extern "C" int cmlab_sk(int U, const float* A, const float* x, float* c, uint64_t m, uint64_t n,
                        float* ps, float* pd, unsigned* queue, int parts, double dyn_frac,
                        int ch, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t mv = m / 8;
    if (mv > 1024) return -1;
    int row_lanes = 1;
    while (uint64_t(row_lanes) < mv) row_lanes *= 2;
    uint64_t S = uint64_t(double(n) * (1.0 - dyn_frac));
    const uint64_t nch = (n - S + ch - 1) / ch;
    const int smem = 1024 * 8 * 4;
    if (U == 2) {
        cudaFuncSetAttribute(k_sk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_sk<2><<<parts, 1024, smem, s>>>(A, x, m, n, S, uint64_t(ch), ps, pd, queue, row_lanes);
    } else {
        cudaFuncSetAttribute(k_sk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_sk<4><<<parts, 1024, smem, s>>>(A, x, m, n, S, uint64_t(ch), ps, pd, queue, row_lanes);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned((m + 31) / 32));
    cfg.blockDim = dim3(1024);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_sk_comb, (const float*)ps, unsigned(parts), (const float*)pd,
                       unsigned(nch), m, c, queue);
    return int(cudaGetLastError());
}

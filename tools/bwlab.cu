// Bandwidth lab (exploration only, not part of the product): streaming-read
// kernels with different shapes, to separate the fixed per-launch ramp of a
// B200 from per-byte cost.  Built by tools/bwlab.py into tools/libbwlab.so.
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

// grid-stride over tiles of BLOCK*U vectors; per-CTA partial, no final pass
template <int U>
__global__ void read_gs(const V8* __restrict__ x, uint64_t nvec, float* out) {
    float acc = 0.f;
    const uint64_t per = uint64_t(blockDim.x) * U;
    for (uint64_t b = uint64_t(blockIdx.x) * per; b < nvec; b += uint64_t(gridDim.x) * per) {
        V8 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = b + uint64_t(u) * blockDim.x + threadIdx.x;
            if (i < nvec) v[u] = ld8(x + i);
            else for (int e = 0; e < 8; ++e) v[u].v[e] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc += v[u].v[e];
    }
    if (acc == 1234.5f) out[blockIdx.x] = acc; // keep the loads alive
}

// contiguous chunk per CTA
template <int U>
__global__ void read_chunk(const V8* __restrict__ x, uint64_t nvec, float* out) {
    const uint64_t q = nvec / gridDim.x, r = nvec % gridDim.x;
    const uint64_t b0 = blockIdx.x * q + (blockIdx.x < r ? blockIdx.x : r);
    const uint64_t b1 = b0 + q + (blockIdx.x < r ? 1 : 0);
    float acc = 0.f;
    for (uint64_t b = b0; b < b1; b += uint64_t(blockDim.x) * U) {
        V8 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = b + uint64_t(u) * blockDim.x + threadIdx.x;
            if (i < b1) v[u] = ld8(x + i);
            else for (int e = 0; e < 8; ++e) v[u].v[e] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc += v[u].v[e];
    }
    if (acc == 1234.5f) out[blockIdx.x] = acc;
}

__global__ void empty_kernel(float* out) {
    if (threadIdx.x == 12345) out[0] = 1.f;
}

extern "C" int bwlab_run(int kind, int unroll, const void* x, uint64_t nvec, float* out,
                         int grid, int block, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const V8* X = static_cast<const V8*>(x);
    if (kind == 0) {
        switch (unroll) {
        case 1: read_gs<1><<<grid, block, 0, s>>>(X, nvec, out); break;
        case 2: read_gs<2><<<grid, block, 0, s>>>(X, nvec, out); break;
        case 4: read_gs<4><<<grid, block, 0, s>>>(X, nvec, out); break;
        default: read_gs<8><<<grid, block, 0, s>>>(X, nvec, out); break;
        }
    } else if (kind == 1) {
        switch (unroll) {
        case 1: read_chunk<1><<<grid, block, 0, s>>>(X, nvec, out); break;
        case 2: read_chunk<2><<<grid, block, 0, s>>>(X, nvec, out); break;
        case 4: read_chunk<4><<<grid, block, 0, s>>>(X, nvec, out); break;
        default: read_chunk<8><<<grid, block, 0, s>>>(X, nvec, out); break;
        }
    } else {
        empty_kernel<<<grid, block, 0, s>>>(out);
    }
    return int(cudaGetLastError());
}

// two-array dot, per-CTA partial written, optional last-block final pass
template <int U, bool FINAL>
__global__ void dot2(const V8* __restrict__ x, const V8* __restrict__ y, uint64_t nvec,
                     float* partials, unsigned* ticket, float* out) {
    __shared__ float red[32];
    __shared__ bool last;
    float acc = 0.f;
    const uint64_t per = uint64_t(blockDim.x) * U;
    for (uint64_t b = uint64_t(blockIdx.x) * per; b < nvec; b += uint64_t(gridDim.x) * per) {
        V8 a[U], c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = b + uint64_t(u) * blockDim.x + threadIdx.x;
            if (i < nvec) { a[u] = ld8(x + i); c[u] = ld8(y + i); }
            else for (int e = 0; e < 8; ++e) a[u].v[e] = c[u].v[e] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = fmaf(a[u].v[e], c[u].v[e], acc);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        float t = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
        if (threadIdx.x == 0) {
            partials[blockIdx.x] = t;
            if (FINAL) {
                __threadfence();
                last = atomicAdd(ticket, 1u) == gridDim.x - 1;
            }
        }
    }
    if (!FINAL) return;
    __syncthreads();
    if (!last) return;
    __threadfence();
    float v = 0.f;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) v += __ldcg(partials + i);
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (unsigned w = 0; w < blockDim.x / 32; ++w) t += red[w];
        *out = t;
        *ticket = 0;
    }
}

extern "C" int bwlab_dot(int final_pass, int unroll, const void* x, uint64_t nvec, float* scratch,
                         unsigned* ticket, int grid, int block, void* stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const V8* X = static_cast<const V8*>(x);
    const V8* Y = X + nvec;  // second half of the buffer
    if (final_pass) {
        if (unroll == 1) dot2<1, true><<<grid, block, 0, s>>>(X, Y, nvec, scratch, ticket, scratch + 4096);
        else dot2<2, true><<<grid, block, 0, s>>>(X, Y, nvec, scratch, ticket, scratch + 4096);
    } else {
        if (unroll == 1) dot2<1, false><<<grid, block, 0, s>>>(X, Y, nvec, scratch, ticket, scratch + 4096);
        else dot2<2, false><<<grid, block, 0, s>>>(X, Y, nvec, scratch, ticket, scratch + 4096);
    }
    return int(cudaGetLastError());
}

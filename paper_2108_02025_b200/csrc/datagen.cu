// Seeded synthetic inputs on the device, bit-identical to the host oracle's
// generator (oracle/cabl_oracle.c): counter-based SplitMix64, so element i
// of (seed, stream) is a pure function of i and 16 GiB operands fill at HBM
// speed instead of being generated on the host.  Stands in for the
// reference's mt19937_64 fills (reference bench.hpp:68-71, acceptance.cpp:84-97),
// which are sequential and implementation-defined.
#include "common.cuh"
#include "kernels.cuh"

namespace cabl_dev {

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t sm_key_host(uint64_t seed, uint64_t sid) {
    uint64_t z = seed + kGolden * (sid + 1ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void fill_u32_kernel(float* __restrict__ out, uint64_t n, uint64_t key,
                                uint64_t offset) {
    pdl_enter();
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t u = sm_mix(key + kGolden * (offset + i + 1ULL));
        out[i] = __fsub_rn(__fmul_rn(float(int32_t(u >> 40)), 1.0f / 8388608.0f), 1.0f);
    }
}

__global__ void fill_u64_kernel(double* __restrict__ out, uint64_t n, uint64_t key,
                                uint64_t offset) {
    pdl_enter();
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t u = sm_mix(key + kGolden * (offset + i + 1ULL));
        out[i] = __dsub_rn(__dmul_rn(double(int64_t(u >> 11)), 1.0 / 4503599627370496.0), 1.0);
    }
}

__global__ void fill_n64_kernel(double* __restrict__ out, uint64_t n, uint64_t key,
                                uint64_t offset) {
    pdl_enter();
    const double two_pi = 6.283185307179586476925286766559;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t c = 2 * (offset + i);
        const uint64_t a = sm_mix(key + kGolden * (c + 1ULL));
        const uint64_t b = sm_mix(key + kGolden * (c + 2ULL));
        const double u1 = (double(int64_t(a >> 11)) + 1.0) * (1.0 / 9007199254740992.0);
        const double u2 = double(int64_t(b >> 11)) * (1.0 / 9007199254740992.0);
        out[i] = sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
    }
}

unsigned fill_grid(uint64_t n) {
    const uint64_t want = (n + 255) / 256;
    const uint64_t cap = uint64_t(sm_count()) * 16;
    return unsigned(want < 1 ? 1 : (want < cap ? want : cap));
}

} // namespace

cudaError_t fill_uniform_f32(float* out, uint64_t n, uint64_t seed, uint64_t sid,
                             uint64_t offset, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    launch(fill_u32_kernel, fill_grid(n), 256, 0, s, out, n, sm_key_host(seed, sid), offset);
    return cudaGetLastError();
}

cudaError_t fill_uniform_f64(double* out, uint64_t n, uint64_t seed, uint64_t sid,
                             uint64_t offset, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    launch(fill_u64_kernel, fill_grid(n), 256, 0, s, out, n, sm_key_host(seed, sid), offset);
    return cudaGetLastError();
}

cudaError_t fill_normal_f64(double* out, uint64_t n, uint64_t seed, uint64_t sid,
                            uint64_t offset, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    launch(fill_n64_kernel, fill_grid(n), 256, 0, s, out, n, sm_key_host(seed, sid), offset);
    return cudaGetLastError();
}

} // namespace cabl_dev

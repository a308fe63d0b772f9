// Ordered GEMV for small problems — the B200 counterpart of the reference's
// "small problems stay on the calling thread" rule (proj/include/cabl/
// kernels.hpp:238-243: touched = m*n + m + n <= plan.dot_cutoff runs one
// worker).  One CTA; thread t owns rows t, t + blockDim, ...; each row is
// summed from c_i with j ascending, exactly as gemv_ref (kernels.hpp:171-181)
// is written, and with the rounding GCC gives it under the reference flags:
// the first 16/s * floor(n / (16/s)) products are multiplied separately and
// added one by one, the remainder is FMA (pinned in oracle/cabl_oracle.c
// against the compiled reference).  Result: bit for bit the compiled
// reference gemv_ref / gemv_row_major for either layout.
#include "common.cuh"
#include "kernels.cuh"

namespace cabl_dev {

namespace {

constexpr int kSmallBlock = 256;

template <typename T>
__global__ void __launch_bounds__(kSmallBlock)
    gemv_ordered_kernel(const T* __restrict__ A, int layout, uint64_t m, uint64_t n,
                        const T* __restrict__ x, T* __restrict__ c) {
    pdl_enter();
    constexpr uint64_t kRefVec = 16 / sizeof(T);
    const uint64_t cut = (n / kRefVec) * kRefVec;
    const uint64_t rs = layout == 0 ? n : 1; // row stride
    const uint64_t cs = layout == 0 ? 1 : m; // column stride
    for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) {
        const T* a = A + i * rs;
        T acc = c[i];
        uint64_t j = 0;
        for (; j < cut; ++j) acc = add_rn(acc, mul_rn(a[j * cs], x[j]));
        for (; j < n; ++j) acc = fma_rn(a[j * cs], x[j], acc);
        c[i] = acc;
    }
}

} // namespace

template <typename T>
cudaError_t gemv_ordered_launch(const T* A, int layout, uint64_t m, uint64_t n, const T* x,
                                T* c, cudaStream_t s, LaunchInfo* info) {
    if (info) info->ctas = 1;
    if (m == 0 || n == 0) return cudaSuccess;
    launch(gemv_ordered_kernel<T>, 1, kSmallBlock, 0, s, A, layout, m, n, x, c);
    return cudaGetLastError();
}

template cudaError_t gemv_ordered_launch<float>(const float*, int, uint64_t, uint64_t,
                                                const float*, float*, cudaStream_t, LaunchInfo*);
template cudaError_t gemv_ordered_launch<double>(const double*, int, uint64_t, uint64_t,
                                                 const double*, double*, cudaStream_t,
                                                 LaunchInfo*);

} // namespace cabl_dev

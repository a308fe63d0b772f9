// cabl/device.hpp — device-resident containers and the overloads that keep
// operands in HBM (no host transfer inside the call).  This is the timed path
// of the benchmarks; cabl/kernels.hpp's host-container overloads are the
// drop-in compatibility path.
//
// Requires the CUDA runtime headers (cuda_runtime.h) on the include path and
// linking libcabl_cuda.so + libcudart.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include <cuda_runtime.h>

#include "kernels.hpp"

namespace cabl {

namespace detail {
inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
} // namespace detail

// Owning device buffer of n elements (cudaMalloc: 256-byte aligned, so the
// kernels' 256-bit vector paths apply).
template <typename T>
class DeviceVector {
    T* ptr_ = nullptr;
    std::size_t n_ = 0;

public:
    DeviceVector() = default;
    explicit DeviceVector(std::size_t n) : n_(n) {
        if (n_) detail::cuda_check(cudaMalloc(&ptr_, n_ * sizeof(T)), "DeviceVector alloc");
    }
    explicit DeviceVector(const Vector<T>& host, cudaStream_t s = nullptr) : DeviceVector(host.len()) {
        upload(host, s);
    }
    DeviceVector(const DeviceVector&) = delete;
    DeviceVector& operator=(const DeviceVector&) = delete;
    DeviceVector(DeviceVector&& o) noexcept : ptr_(std::exchange(o.ptr_, nullptr)), n_(std::exchange(o.n_, 0)) {}
    DeviceVector& operator=(DeviceVector&& o) noexcept {
        if (this != &o) {
            if (ptr_) cudaFree(ptr_);
            ptr_ = std::exchange(o.ptr_, nullptr);
            n_ = std::exchange(o.n_, 0);
        }
        return *this;
    }
    ~DeviceVector() {
        if (ptr_) cudaFree(ptr_);
    }

    std::size_t len() const noexcept { return n_; }
    T* data() noexcept { return ptr_; }
    const T* data() const noexcept { return ptr_; }

    void upload(const Vector<T>& host, cudaStream_t s = nullptr) {
        detail::require(host.len() == n_, "DeviceVector: length mismatch");
        if (n_)
            detail::cuda_check(cudaMemcpyAsync(ptr_, host.data(), n_ * sizeof(T),
                                               cudaMemcpyHostToDevice, s), "H2D");
        detail::cuda_check(cudaStreamSynchronize(s), "sync");
    }
    Vector<T> download(cudaStream_t s = nullptr) const {
        Vector<T> out(n_);
        if (n_)
            detail::cuda_check(cudaMemcpyAsync(out.data(), ptr_, n_ * sizeof(T),
                                               cudaMemcpyDeviceToHost, s), "D2H");
        detail::cuda_check(cudaStreamSynchronize(s), "sync");
        return out;
    }
};

template <typename T>
class DeviceMatrix {
    std::size_t rows_ = 0, cols_ = 0;
    Layout layout_ = Layout::RowMajor;
    DeviceVector<T> store_;

public:
    DeviceMatrix() = default;
    DeviceMatrix(std::size_t rows, std::size_t cols, Layout layout)
        : rows_(rows), cols_(cols), layout_(layout), store_(rows * cols) {}
    explicit DeviceMatrix(const DenseMatrix<T>& host, cudaStream_t s = nullptr)
        : DeviceMatrix(host.rows(), host.cols(), host.layout()) {
        upload(host, s);
    }

    std::size_t rows() const noexcept { return rows_; }
    std::size_t cols() const noexcept { return cols_; }
    Layout layout() const noexcept { return layout_; }
    std::size_t size() const noexcept { return rows_ * cols_; }
    T* data() noexcept { return store_.data(); }
    const T* data() const noexcept { return store_.data(); }

    void upload(const DenseMatrix<T>& host, cudaStream_t s = nullptr) {
        detail::require(host.rows() == rows_ && host.cols() == cols_ && host.layout() == layout_,
                        "DeviceMatrix: shape mismatch");
        if (size())
            detail::cuda_check(cudaMemcpyAsync(data(), host.data(), size() * sizeof(T),
                                               cudaMemcpyHostToDevice, s), "H2D");
        detail::cuda_check(cudaStreamSynchronize(s), "sync");
    }
    DenseMatrix<T> download(cudaStream_t s = nullptr) const {
        DenseMatrix<T> out(rows_, cols_, layout_);
        if (size())
            detail::cuda_check(cudaMemcpyAsync(out.data(), data(), size() * sizeof(T),
                                               cudaMemcpyDeviceToHost, s), "D2H");
        detail::cuda_check(cudaStreamSynchronize(s), "sync");
        return out;
    }
};

namespace detail {
inline int dev_dot(const float* x, const float* y, std::uint64_t n, float a, float* o,
                   std::uint64_t cut, cabl_probe* p, cudaStream_t s) {
    return cabl_cuda_dot_f32(x, y, n, a, o, cut, p, s);
}
inline int dev_dot(const double* x, const double* y, std::uint64_t n, double a, double* o,
                   std::uint64_t cut, cabl_probe* p, cudaStream_t s) {
    return cabl_cuda_dot_f64(x, y, n, a, o, cut, p, s);
}
inline int dev_gemv(bool row, const float* A, std::uint64_t m, std::uint64_t n, const float* x,
                    float* c, std::uint64_t cut, cabl_probe* p, cudaStream_t s) {
    return row ? cabl_cuda_gemv_rm_f32(A, m, n, x, c, cut, p, s)
               : cabl_cuda_gemv_cm_f32(A, m, n, x, c, cut, p, s);
}
inline int dev_gemv(bool row, const double* A, std::uint64_t m, std::uint64_t n, const double* x,
                    double* c, std::uint64_t cut, cabl_probe* p, cudaStream_t s) {
    return row ? cabl_cuda_gemv_rm_f64(A, m, n, x, c, cut, p, s)
               : cabl_cuda_gemv_cm_f64(A, m, n, x, c, cut, p, s);
}
inline int dev_ger(bool row, const float* x, const float* y, float* C, std::uint64_t m,
                   std::uint64_t n, std::uint64_t cut, cabl_probe* p, cudaStream_t s) {
    return row ? cabl_cuda_ger_rm_f32(x, y, C, m, n, cut, p, s)
               : cabl_cuda_ger_cm_f32(x, y, C, m, n, cut, p, s);
}
inline int dev_ger(bool row, const double* x, const double* y, double* C, std::uint64_t m,
                   std::uint64_t n, std::uint64_t cut, cabl_probe* p, cudaStream_t s) {
    return row ? cabl_cuda_ger_rm_f64(x, y, C, m, n, cut, p, s)
               : cabl_cuda_ger_cm_f64(x, y, C, m, n, cut, p, s);
}
} // namespace detail

// *d_out = alpha0 + x.y, enqueued on s (no synchronisation).
template <typename T>
void dot_async(const DeviceVector<T>& x, const DeviceVector<T>& y, T alpha0, T* d_out,
               const ExecPolicy& policy, cudaStream_t s = nullptr) {
    detail::require(x.len() == y.len(), "dot: x and y lengths differ");
    cabl_probe probe{};
    detail::check(detail::dev_dot(x.data(), y.data(), x.len(), alpha0, d_out,
                                  policy.plan.dot_cutoff, &probe, s));
    detail::record(probe);
}

template <typename T>
T dot(const DeviceVector<T>& x, const DeviceVector<T>& y, T alpha0, const ExecPolicy& policy,
      cudaStream_t s = nullptr) {
    DeviceVector<T> out(1);
    dot_async(x, y, alpha0, out.data(), policy, s);
    T r{};
    detail::cuda_check(cudaMemcpyAsync(&r, out.data(), sizeof(T), cudaMemcpyDeviceToHost, s), "D2H");
    detail::cuda_check(cudaStreamSynchronize(s), "sync");
    return r;
}

template <typename T>
void gemv_col_major(const DeviceMatrix<T>& A, const DeviceVector<T>& x, DeviceVector<T>& c,
                    const ExecPolicy& policy, cudaStream_t s = nullptr) {
    detail::require(A.layout() == Layout::ColMajor, "gemv_col_major: matrix is not col-major");
    detail::require(A.cols() == x.len(), "gemv: A.cols != x.len");
    detail::require(A.rows() == c.len(), "gemv: A.rows != c.len");
    detail::require(!detail::aliases(c.data(), x.data()), "gemv: c must not alias x");
    cabl_probe probe{};
    detail::check(detail::dev_gemv(false, A.data(), A.rows(), A.cols(), x.data(), c.data(),
                                   policy.plan.dot_cutoff, &probe, s));
    detail::record(probe);
}

template <typename T>
void gemv_row_major(const DeviceMatrix<T>& A, const DeviceVector<T>& x, DeviceVector<T>& c,
                    const ExecPolicy& policy, cudaStream_t s = nullptr) {
    detail::require(A.layout() == Layout::RowMajor, "gemv_row_major: matrix is not row-major");
    detail::require(A.cols() == x.len(), "gemv: A.cols != x.len");
    detail::require(A.rows() == c.len(), "gemv: A.rows != c.len");
    detail::require(!detail::aliases(c.data(), x.data()), "gemv: c must not alias x");
    cabl_probe probe{};
    detail::check(detail::dev_gemv(true, A.data(), A.rows(), A.cols(), x.data(), c.data(),
                                   policy.plan.dot_cutoff, &probe, s));
    detail::record(probe);
}

template <typename T>
void ger(const DeviceVector<T>& x, const DeviceVector<T>& y, DeviceMatrix<T>& C,
         const ExecPolicy& policy, cudaStream_t s = nullptr) {
    detail::require(C.rows() == x.len(), "ger: C.rows != x.len");
    detail::require(C.cols() == y.len(), "ger: C.cols != y.len");
    detail::require(!detail::aliases(C.data(), x.data()) && !detail::aliases(C.data(), y.data()),
                    "ger: C must not alias x or y");
    cabl_probe probe{};
    detail::check(detail::dev_ger(C.layout() == Layout::RowMajor, x.data(), y.data(), C.data(),
                                  C.rows(), C.cols(), policy.plan.dot_cutoff, &probe, s));
    detail::record(probe);
}

// ------------------------------------------------- GPU machine descriptor
// the live device described in the reference's descriptor
// model (machine.hpp:43-53): cores = SMs, L1 = per-SM shared memory
// (private), L2 = device L2 (shared), 128-byte lines.  It passes
// validate_machine, so derive_blocking_plan accepts it; derive_gpu_plan gives
// the launch parameters the library derives from the same facts.
inline cabl_gpu_machine describe_device(int device = 0) {
    cabl_gpu_machine g{};
    detail::check(cabl_describe_device(device, &g));
    return g;
}

inline MachineDescriptor gpu_machine(int device = 0, std::uint64_t element_bytes = 4) {
    const cabl_gpu_machine g = describe_device(device);
    constexpr std::uint64_t line = 128, l1_ways = 4, l2_ways = 16;
    MachineDescriptor md;
    md.levels.push_back(CacheLevel{line, l1_ways, g.smem_per_sm / (line * l1_ways), false});
    md.levels.push_back(CacheLevel{line, l2_ways, g.l2_bytes / (line * l2_ways), true});
    md.cores = g.sm_count;
    md.element_bytes = element_bytes;
    validate_machine(md);
    return md;
}

struct GpuPlan {
    unsigned sm_count = 0;
    std::uint64_t l2_bytes = 0;
    std::uint64_t queue_threshold_bytes = 0; // operands >= this use the work queues
    std::uint64_t l2_flush_bytes = 0;        // benchmark flush buffer
    unsigned dot_ctas = 0;
};

// same rules as paper_2108_02025_b200/machine.py derive_gpu_plan
inline GpuPlan derive_gpu_plan(const MachineDescriptor& md) {
    validate_machine(md);
    GpuPlan p;
    p.sm_count = md.cores;
    p.l2_bytes = md.levels.back().size_bytes();
    std::uint64_t q = 1;
    while (q < 4 * p.l2_bytes) q <<= 1;
    p.queue_threshold_bytes = q;
    p.l2_flush_bytes = q;
    p.dot_ctas = 2 * md.cores;
    return p;
}

} // namespace cabl

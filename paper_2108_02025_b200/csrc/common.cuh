// Shared device helpers for the B200 (sm_100a) DOT / GEMV / GER kernels.
//
// Every kernel here is HBM-bound (<= 0.5 flop/byte); the
// levers are the bytes in flight per SM, the LSU instruction count and load
// balance across the 148 SMs — not tensor cores.  sm_100a has 256-bit global
// loads/stores (SASS LDG.E.256 / STG.E.256), so a "vector" below is 32 bytes:
// 8 floats or 4 doubles per lane per instruction, half the LSU issue of
// float4/double2.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <utility>

namespace cabl_dev {

// Opt a kernel in to more than 48 KB of dynamic shared memory.  The attribute
// belongs to the kernel ON THE CURRENT DEVICE, so a process that drives several
// devices (cabl_mgpu_*, cabl::nccl::Group) must set it on each of them: `done`
// (one static per call site) keeps a bit per device ordinal.
template <typename K>
inline void ensure_dyn_smem(K kernel, int bytes, std::atomic<unsigned long long>& done) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
    const unsigned long long bit = 1ull << (unsigned(dev) & 63u);
    if (done.load(std::memory_order_acquire) & bit) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done.fetch_or(bit, std::memory_order_release);
}


// Tuning / A-B switches (CABL_DOT_CFG, CABL_GEMV_RM_ORDER, CABL_CM_TILE, ...;
// DESIGN.md §4 "Environment knobs") pick other launch shapes or kernels, and
// so may change the last bits of a result.  They are honoured only when the
// process also sets CABL_TUNING=1: a shipped process's results never depend
// on its environment.  (Operational settings — timeouts, the NCCL library,
// PDL — are read with plain getenv: they never change bits.)
inline const char* tuning_env(const char* name) {
    static const bool on = [] {
        const char* e = getenv("CABL_TUNING");
        return e != nullptr && e[0] == '1' && e[1] == '\0';
    }();
    return on ? getenv(name) : nullptr;
}

constexpr int kWarp = 32;

// 32-byte vector of T.
template <typename T> struct Vec;
template <> struct alignas(32) Vec<float> {
    static constexpr int N = 8;
    float v[8];
};
template <> struct alignas(32) Vec<double> {
    static constexpr int N = 4;
    double v[4];
};

// ---- 256-bit loads -------------------------------------------------------
// Streaming read-only operand (A, x/y of DOT): non-coherent path, no L1
// allocation, and a 256 B L2 prefetch hint so each DRAM burst is a full
// 256 B.  Only for data no thread writes during the kernel.
__device__ __forceinline__ Vec<float> ld_stream(const Vec<float>* p) {
    Vec<float> r;
    asm volatile(
        "ld.global.nc.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
          "=f"(r.v[6]), "=f"(r.v[7])
        : "l"(p));
    return r;
}
__device__ __forceinline__ Vec<double> ld_stream(const Vec<double>* p) {
    Vec<double> r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
                 : "l"(p));
    return r;
}

// Reused read-only operand (x of GEMV, y of GER): cached in L1.
__device__ __forceinline__ Vec<float> ld_reuse(const Vec<float>* p) {
    Vec<float> r;
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                   "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ Vec<double> ld_reuse(const Vec<double>* p) {
    Vec<double> r;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
                 : "l"(p));
    return r;
}

// Read-modify-write operand (C of GER): coherent load, no L1 allocation.
__device__ __forceinline__ Vec<float> ld_rmw(const Vec<float>* p) {
    Vec<float> r;
    asm volatile("ld.global.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                   "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ Vec<double> ld_rmw(const Vec<double>* p) {
    Vec<double> r;
    asm volatile("ld.global.L1::no_allocate.L2::256B.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
                 : "l"(p)
                 : "memory");
    return r;
}

__device__ __forceinline__ void st_stream(Vec<float>* p, const Vec<float>& r) {
    asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]),
                 "f"(r.v[6]), "f"(r.v[7])
                 : "memory");
}
__device__ __forceinline__ void st_stream(Vec<double>* p, const Vec<double>& r) {
    asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r.v[0]),
                 "d"(r.v[1]), "d"(r.v[2]), "d"(r.v[3])
                 : "memory");
}

// ---- arithmetic with the rounding spelled out ------------------------------
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// acc + a.b over one 32-byte vector, one FMA chain in element order.
template <typename T>
__device__ __forceinline__ T dot_vec(const Vec<T>& a, const Vec<T>& b, T acc) {
#pragma unroll
    for (int k = 0; k < Vec<T>::N; ++k) acc = fma_rn(a.v[k], b.v[k], acc);
    return acc;
}

// Fixed butterfly: every lane ends with the same, order-fixed sum.
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = add_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Order-fixed block sum (blockDim.x multiple of 32, <= 1024); result valid in
// every thread.  `red` must hold 32 T.  Contains two __syncthreads().
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red[wid] = v;
    __syncthreads();
    T t = lane < nw ? red[lane] : T(0);
    t = warp_sum(t);
    __syncthreads();
    return t;
}

// L1-bypassing loads for data another CTA produced in this kernel.
__device__ __forceinline__ float ld_cg(const float* p) { return __ldcg(p); }
__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ Vec<float> ld_cg(const Vec<float>* p) {
    Vec<float> r;
    asm volatile("ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                   "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p)
                 : "memory");
    return r;
}
__device__ __forceinline__ Vec<double> ld_cg(const Vec<double>* p) {
    Vec<double> r;
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
                 : "l"(p)
                 : "memory");
    return r;
}

// Balanced static partition of `total` units over `parts`: part w owns
// [begin(w), begin(w+1)).  owner(u) inverts it.
struct Partition {
    uint64_t total, parts, q, r;
    __host__ __device__ Partition(uint64_t total_, uint64_t parts_)
        : total(total_), parts(parts_), q(total_ / parts_), r(total_ % parts_) {}
    __host__ __device__ uint64_t begin(uint64_t w) const { return w * q + (w < r ? w : r); }
    __host__ __device__ uint64_t owner(uint64_t u) const {
        const uint64_t big = r * (q + 1);
        return u < big ? u / (q + 1) : r + (u - big) / q;
    }
};

// Dynamic work queue over items [0, total) for a grid of <= total CTAs: CTA b
// starts on item b with no atomic on the critical path, then draws
// gridDim.x + atomicAdd(counter, 1) until it gets an item >= total.  That is
// exactly `total` draws overall (total - grid successful + one failing per
// CTA), so whoever draws raw value total - 1 is the counter's last user in
// this launch and resets it to zero for the next launch on the stream.
__device__ __forceinline__ unsigned long long dyn_next(unsigned* counter,
                                                       unsigned long long total, unsigned nblk) {
    const unsigned long long raw = atomicAdd(counter, 1u);
    if (raw == total - 1) *counter = 0u;
    return raw + nblk;
}
__device__ __forceinline__ unsigned long long dyn_next(unsigned* counter,
                                                       unsigned long long total) {
    return dyn_next(counter, total, gridDim.x);
}

// Acq_rel ticket: true in the CTA that arrives last (every earlier CTA's
// partial is visible to it).  Contains one __syncthreads().
__device__ __forceinline__ bool last_arriver(unsigned* ticket, unsigned nblk, bool* am_last_sh) {
    if (threadIdx.x == 0) {
        unsigned t;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                     : "=r"(t)
                     : "l"(ticket)
                     : "memory");
        *am_last_sh = (t == nblk - 1);
    }
    __syncthreads();
    return *am_last_sh;
}

// ---- epoch-tagged 64-bit words (DOT collector, dot.cu) ---------------------
// A word is (epoch << 32) | 32 payload bits; a T takes sizeof(T) / 4 words.
// Relaxed gpu-scope accesses: the payload travels inside the word, so no
// other memory needs ordering, and a poller sees the word once it is in L2.
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <typename T> __host__ __device__ constexpr int tagged_words() { return int(sizeof(T) / 4); }
__device__ __forceinline__ void publish_tagged(unsigned long long* w, float v, unsigned e) {
    st_relaxed_u64(w, (static_cast<unsigned long long>(e) << 32) | __float_as_uint(v));
}
__device__ __forceinline__ void publish_tagged(unsigned long long* w, double v, unsigned e) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    const unsigned long long tag = static_cast<unsigned long long>(e) << 32;
    st_relaxed_u64(w, tag | (b & 0xffffffffull));
    st_relaxed_u64(w + 1, tag | (b >> 32));
}
__device__ __forceinline__ unsigned wait_tagged(const unsigned long long* w, unsigned e) {
    unsigned long long v;
    do {
        v = ld_relaxed_u64(w);
    } while (unsigned(v >> 32) != e);
    return unsigned(v);
}
template <typename T> __device__ __forceinline__ T collect_tagged(const unsigned long long* w, unsigned e);
template <> __device__ __forceinline__ float collect_tagged<float>(const unsigned long long* w, unsigned e) {
    return __uint_as_float(wait_tagged(w, e));
}
template <> __device__ __forceinline__ double collect_tagged<double>(const unsigned long long* w, unsigned e) {
    const unsigned long long lo = wait_tagged(w, e), hi = wait_tagged(w + 1, e);
    return __longlong_as_double(static_cast<long long>((hi << 32) | lo));
}
// this launch's epoch: one past the last completed one (never 0, the value of
// a zeroed word)
__device__ __forceinline__ unsigned next_epoch(const unsigned long long* epoch_word) {
    const unsigned e = unsigned(ld_relaxed_u64(epoch_word)) + 1u;
    return e ? e : 1u;
}

// ---- programmatic dependent launch (PDL) ---------------------------------
// Every kernel of the library starts with pdl_enter(): it lets the NEXT
// kernel on the stream begin launching (its CTAs take SMs as this grid's
// CTAs retire) and then waits until the PREVIOUS grid has fully completed and
// its memory is visible.  No global memory is touched before the wait, so the
// stream semantics are exactly the usual ones; what overlaps is only launch
// latency and CTA rasterisation with the previous kernel's tail — back-to-back
// calls (an iterative solver, a serving loop, K bench steps) lose the gap
// between kernels.  Without the launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// The two halves, for kernels that warm L2 in between: between trigger and
// wait a kernel may only issue L2 prefetches of its own inputs (no data
// reaches the SM, and L2 is the point of coherence, so a line a previous
// kernel is still writing is simply updated in L2 — nothing stale can be
// read after the wait).  The DRAM reads of the first tiles then overlap the
// previous kernel's tail instead of following it.
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// bulk L2 prefetch of `bytes` (multiple of 16, 16-byte aligned source)
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// CABL_PDL_PREFETCH=0 disables the pre-wait L2 prefetch (A/B measurement).
// D1 back to back: 22.5 -> 21.9 us with it; the GEMV sweep is neutral; on
// GER (R1) it cost 0.7 us, so GER does not prefetch.
inline int pdl_prefetch_enabled() {
    static const int on = [] {
        const char* e = getenv("CABL_PDL_PREFETCH");
        return e ? atoi(e) : 1;
    }();
    return on;
}

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("CABL_PDL");
        return e ? atoi(e) != 0 : true;
    }();
    return on;
}

// kernel<<<grid, block, smem, s>>>(args...) with the PDL attribute
template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                   Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

inline bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }

} // namespace cabl_dev

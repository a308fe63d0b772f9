// System-scope memory helpers for the peer-memory kernels (peer.cu,
// peer_gemv.cu): relaxed 8-byte loads/stores that are single-copy atomic and
// visible across GPUs (P2P over NVLink), and the global nanosecond timer used
// for the wait timeouts.
#pragma once

#include <cstdint>

namespace cabl_dev {

__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

} // namespace cabl_dev

// Row-major GEMV with the all-gather of c fused into the kernel, over peer
// memory (NVLink / NVSwitch P2P stores) instead of a separate NCCL collective.
//
// rank g owns a block of rows of A and its slice of c (x
// replicated); BASELINE config 5 all-gathers the c slices so every rank holds
// the full c.  Reference: cabl::gemv_row_major, proj/include/cabl/kernels.hpp:
// 230-257 (rows chunked over threads, :243) lifted to devices.
//
// One kernel per rank:
//   1. the rank's slice through the single-GPU sweep body (gemv_rm_body.cuh,
//      the same group shape gemv_rm_launch picks), so c_slice gets the bits a
//      plain call gives;
//   2. every finished row is also stored into every rank's c_full — a P2P
//      store per peer, issued while the sweep still streams A;
//   3. each CTA fences at system scope and takes a ticket; the last CTA
//      publishes an epoch-tagged word into every peer's mailbox, waits for
//      every peer's word, fences, and the kernel ends with c_full complete.
//
// c_full is double-buffered by epoch parity (buffer e & 1 for the e-th call):
// a peer that finished call e may push call e+1 while this rank's stream still
// reads buffer e & 1 (the consumer of call e), never buffer (e+1) & 1, whose
// last reader (the consumer of call e-1) precedes this rank's call e, and the
// peer saw call e's word only after that.  Calls are collective (every rank,
// same order).  A peer that never arrives: after timeout_ns the waiting rank
// records the epoch in its mailbox's `fault` word and exits.
//
// Emulation: as in peer.cu, blockIdx.y = rank runs every rank's grid in one
// cooperative launch on one device for the tests.
//
// Algorithmic bytes per rank launch: m_r n s + n s + 2 m_r s
// plus (G - 1) m_r s of P2P stores.
#include "common.cuh"
#include "gemv_rm_body.cuh"
#include "kernels.cuh"
#include "peer.cuh"

namespace cabl_dev {

namespace {

// 0: none (world 1), 1: fence.acq_rel.sys, 2: fence.sc.sys (__threadfence_system)
__device__ __forceinline__ void sys_fence(int mode) {
    if (mode == 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
    else if (mode == 2) __threadfence_system();
}

template <typename T, int R, int KV, int MINB, bool DYN>
__global__ void __launch_bounds__(kRmBlock, MINB)
    gemv_rm_gather_kernel(const __grid_constant__ PeerGemvArgs<T> a) {
    __shared__ unsigned epoch_sh;
    __shared__ bool last_sh;
    const int lr = blockIdx.y;
    const unsigned nblk = a.grid[lr];
    pdl_trigger();
    if (blockIdx.x >= nblk) { // emulation: a rank with a smaller grid
        pdl_wait();
        return;
    }
    if (threadIdx.x < R) { // as the sweep: warm L2 with this CTA's first pass
        const uint64_t row = uint64_t(blockIdx.x) * R + threadIdx.x;
        const uint64_t pass = uint64_t(kRmBlock) * KV * sizeof(Vec<T>);
        if (row < a.m[lr])
            prefetch_l2_bulk(a.A[lr] + row * a.n,
                             unsigned(a.n * sizeof(T) < pass ? a.n * sizeof(T) : pass));
    }
    pdl_wait();
    const int rank = a.rank0 + lr;
    PeerMailbox* mine = static_cast<PeerMailbox*>(a.mbox[rank]);
    // written only by this rank's previous call (stream order); published by
    // the sweep's first group barrier, before the first epilogue reads it
    if (threadIdx.x == 0)
        epoch_sh = unsigned(*reinterpret_cast<volatile unsigned long long*>(&mine->epoch) + 1);
    T* c = a.c[lr];
    const int world = a.world;
    const uint64_t off = a.row_off[lr];
    sweep_groups<T, R, KV, DYN>(a.A[lr], a.x[lr], a.m[lr], a.n, a.counters[lr], blockIdx.x, nblk, c,
                                [&](uint64_t row, T sum, T c_row) {
                                    const T v = add_rn(c_row, sum);
                                    c[row] = v;
                                    const uint64_t at = uint64_t(epoch_sh & 1) * a.m_total + off + row;
                                    for (int g = 0; g < world; ++g) a.cfull[g][at] = v;
                                });
    __syncthreads(); // epoch_sh for CTAs that had no group
    const unsigned e = epoch_sh;
    // this CTA's pushes are visible system-wide before its ticket (release),
    // and every earlier CTA's before the words below (acquire + release); no
    // peer, no fence (world 1)
    sys_fence(a.fence);
    if (!last_arriver(a.counters[lr] + 1, nblk, &last_sh)) return;
    sys_fence(a.fence);
    if (threadIdx.x == 0) a.counters[lr][1] = 0u;
    const int p = e & 1;
    if (int(threadIdx.x) < world && int(threadIdx.x) != rank) {
        PeerMailbox* peer = static_cast<PeerMailbox*>(a.mbox[threadIdx.x]);
        st_relaxed_sys(&peer->word[p][rank][0], (unsigned long long)e << 32);
    }
    if (threadIdx.x == 0) {
        const unsigned long long t0 = globaltimer();
        bool ok = true;
        for (int g = 0; g < world && ok; ++g) {
            if (g == rank) continue;
            while (unsigned(ld_relaxed_sys(&mine->word[p][g][0]) >> 32) != e) {
                if (globaltimer() - t0 > a.timeout_ns) {
                    ok = false;
                    break;
                }
                __nanosleep(64);
            }
        }
        sys_fence(a.fence); // peers' pushes before anything this rank reads next
        if (!ok) mine->fault = e;
        mine->epoch = e;
    }
}

template <typename T, int R, int KV, int MINB>
cudaError_t gather_go(const PeerGemvArgs<T>& a, int local_ranks, bool dyn, bool cooperative,
                      cudaStream_t s) {
    unsigned gx = 1;
    for (int i = 0; i < local_ranks; ++i) gx = a.grid[i] > gx ? a.grid[i] : gx;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(gx, unsigned(local_ranks));
    cfg.blockDim = dim3(kRmBlock);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    if (cooperative) {
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
    } else {
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = (cooperative || pdl_enabled()) ? 1 : 0;
    if (dyn) return cudaLaunchKernelEx(&cfg, gemv_rm_gather_kernel<T, R, KV, MINB, true>, a);
    return cudaLaunchKernelEx(&cfg, gemv_rm_gather_kernel<T, R, KV, MINB, false>, a);
}

template <typename T, int R, int KV, int MINB> int occupancy() {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, gemv_rm_gather_kernel<T, R, KV, MINB, true>,
                                                      kRmBlock, 0) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return b;
}

} // namespace

// The sweep shapes gemv_rm_launch uses by default (gemv_rm.cu sweep_choice);
// a CABL_RM_SWEEP tuning entry outside them is rejected by the caller.
#define CABL_GATHER_SHAPES(X) X(4, 2, 2) X(2, 8, 1) X(2, 4, 2) X(8, 1, 2)

template <typename T>
cudaError_t gemv_rm_gather_launch(const PeerGemvArgs<T>& a, int local_ranks, int R, int KV,
                                  int minb, bool dyn, bool cooperative, cudaStream_t s) {
#define CABL_GATHER_CASE(R_, KV_, MB_)                                                          \
    if (R == R_ && KV == KV_ && minb == MB_)                                                    \
        return gather_go<T, R_, KV_, MB_>(a, local_ranks, dyn, cooperative, s);
    CABL_GATHER_SHAPES(CABL_GATHER_CASE)
#undef CABL_GATHER_CASE
    return cudaErrorInvalidValue;
}

int gemv_rm_gather_ctas_per_sm(int R, int KV, int minb, size_t elem) {
#define CABL_GATHER_OCC(R_, KV_, MB_)                                                           \
    if (R == R_ && KV == KV_ && minb == MB_)                                                    \
        return elem == 4 ? occupancy<float, R_, KV_, MB_>() : occupancy<double, R_, KV_, MB_>();
    CABL_GATHER_SHAPES(CABL_GATHER_OCC)
#undef CABL_GATHER_OCC
    return 0;
}

template cudaError_t gemv_rm_gather_launch<float>(const PeerGemvArgs<float>&, int, int, int, int,
                                                  bool, bool, cudaStream_t);
template cudaError_t gemv_rm_gather_launch<double>(const PeerGemvArgs<double>&, int, int, int, int,
                                                   bool, bool, cudaStream_t);

} // namespace cabl_dev

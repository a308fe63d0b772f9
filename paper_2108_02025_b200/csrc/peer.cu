// Multi-GPU DOT with the exchange fused into the kernel, over peer memory
// (NVLink / NVSwitch P2P stores) instead of a separate NCCL collective.
//
// Reference: the CPU path splits DOT into chunks, sums the chunk partials in
// chunk order and adds alpha0 last (proj/include/cabl/kernels.hpp:145-163).
// Across G GPUs rank g owns a contiguous shard of x and y.
// The unfused path (shard.py, nccl.hpp) runs the single-GPU kernel with
// alpha0 = 0, all-gathers the G partials with NCCL and sums them in rank order
// (cabl_cuda_combine_partials).  Here ONE kernel per rank does all of it:
//
//   1. the rank's shard partial, with exactly the single-GPU plan (dot_plan:
//      same grid, same element -> thread mapping, same trees), so it is the
//      bits of dot_launch(alpha0 = 0);
//   2. the rank's last CTA (acq_rel ticket) stores the partial, tagged with
//      the call's epoch, into word [epoch parity][rank] of EVERY rank's
//      mailbox — a P2P store through the peer mapping;
//   3. it polls its own mailbox until all G words carry the epoch, sums the
//      G partials in rank order, adds alpha0 last and writes *out.
//
// The result is bitwise the unfused path's (same partials, same rank-order
// sum) and identical on every rank.  There is no host round trip, no NCCL
// launch and no second kernel; the exchange is G 8-byte stores per rank.
//
// Mailbox protocol.  Each rank owns one 512-byte mailbox (zeroed at
// creation): word[p][g] = (epoch << 32) | bits of rank g's partial for the
// last epoch with parity p (two 32-bit halves for fp64), epoch = this rank's
// call count (written only by its owner, read at the next call in stream
// order).  Tag and data travel in ONE 8-byte store, which is single-copy
// atomic, so the publish is a relaxed P2P store and the wait a relaxed poll —
// no release/acquire fences at system scope.  The epoch is loaded while the
// sweep runs and a rank's own partial never goes through memory.  Measured at
// world 1, n = 2^24 fp32, back to back (tools/peer_cost.py): plain DOT 21.2 us;
// a flag + st.release.sys / ld.acquire.sys version 25.8 us; tagged words
// 23.3 us; plus the early epoch load and the self skip 21.4 us (the unfused
// DOT + combine: 23.1 us).  Calls must be made collectively (every rank, same
// order), like any collective.  A rank can run at most one epoch ahead of
// another rank's reads (to publish epoch e+2 it must have seen every word of
// e+1, which a rank publishes only after it finished reading epoch e), so two
// parity slots suffice.  A wait longer than `timeout_ns` (a rank that never
// arrives) writes NaN to *out, records the epoch in `fault` and exits, so a
// broken job reports an error instead of hanging the GPU.
//
// Emulation.  With fewer GPUs than ranks the same kernel runs every rank's
// grid in ONE cooperative launch on one device (blockIdx.y = rank, mailboxes
// side by side in that device's memory), which exercises the whole protocol
// with all waiting CTAs guaranteed co-resident.  Algorithmic bytes per rank
// launch: 2 * n_rank * sizeof(T) plus G tagged 8-byte words
// (two per peer for fp64).
#include "common.cuh"
#include "dot_body.cuh"
#include "kernels.cuh"
#include "peer.cuh"

namespace cabl_dev {

static_assert(sizeof(PeerMailbox) == 512, "mailbox layout is part of the ABI");

namespace {

// the partial's bits as (up to) two 32-bit halves, and back
__device__ __forceinline__ void halves(float v, unsigned* h) { h[0] = __float_as_uint(v); }
__device__ __forceinline__ void halves(double v, unsigned* h) {
    const unsigned long long b = __double_as_longlong(v);
    h[0] = unsigned(b);
    h[1] = unsigned(b >> 32);
}
__device__ __forceinline__ float from_halves(const unsigned* h, float*) { return __uint_as_float(h[0]); }
__device__ __forceinline__ double from_halves(const unsigned* h, double*) {
    return __longlong_as_double((long long)((unsigned long long)h[1] << 32 | h[0]));
}
template <typename T> __device__ __forceinline__ T quiet_nan();
template <> __device__ __forceinline__ float quiet_nan<float>() { return __int_as_float(0x7fc00000); }
template <> __device__ __forceinline__ double quiet_nan<double>() {
    return __longlong_as_double(0x7ff8000000000000ll);
}

// Steps 2-3 above, run by every thread of local rank lr's last CTA.  `total`
// (the shard's sum before alpha0) is valid in thread 0.
// `prev_epoch` is mine->epoch, loaded by thread 0 at kernel start (only this
// rank's previous call writes it, and that call completed before the PDL wait).
template <typename T>
__device__ __forceinline__ void peer_finish(T total, const PeerDotArgs<T>& a, int lr,
                                            unsigned long long prev_epoch) {
    constexpr int H = sizeof(T) / 4; // 32-bit halves per partial
    __shared__ unsigned bits_sh[2];
    __shared__ unsigned epoch_sh;
    const int rank = a.rank0 + lr;
    PeerMailbox* mine = static_cast<PeerMailbox*>(a.mbox[rank]);
    // the unfused path's partial is dot(x_r, y_r, alpha0 = 0) = total + 0
    const T own = add_rn(total, T(0));
    if (threadIdx.x == 0) {
        halves(own, bits_sh);
        epoch_sh = unsigned(prev_epoch + 1);
    }
    __syncthreads();
    const unsigned e = epoch_sh;
    const int p = e & 1;
    if (int(threadIdx.x) < a.world * H) { // one 8-byte store per (peer, half), in parallel
        const int g = threadIdx.x / H, h = threadIdx.x % H;
        PeerMailbox* peer = static_cast<PeerMailbox*>(a.mbox[g]);
        if (g != rank) st_relaxed_sys(&peer->word[p][rank][h], (unsigned long long)e << 32 | bits_sh[h]);
    }
    if (threadIdx.x == 0) {
        const unsigned long long t0 = globaltimer();
        T sum = T(0);
        bool ok = true;
        for (int g = 0; g < a.world && ok; ++g) {
            if (g == rank) { // this rank's own partial: no round trip through memory
                sum = add_rn(sum, own);
                continue;
            }
            unsigned got[2] = {0u, 0u};
            for (int h = 0; h < H && ok; ++h) {
                unsigned long long w;
                while (unsigned((w = ld_relaxed_sys(&mine->word[p][g][h])) >> 32) != e) {
                    if (globaltimer() - t0 > a.timeout_ns) {
                        ok = false;
                        break;
                    }
                    __nanosleep(32);
                }
                got[h] = unsigned(w);
            }
            if (ok) sum = add_rn(sum, from_halves(got, (T*)nullptr));
        }
        if (ok) {
            *a.out[lr] = add_rn(sum, a.alpha0); // rank order, alpha0 last (kernels.hpp:160-163)
        } else {
            *a.out[lr] = quiet_nan<T>();
            mine->fault = e;
        }
        mine->epoch = e;
    }
}

// Grid-stride shard (dot_kernel's body) + fused exchange.
template <typename T, int BLOCK, int U, int MINB, bool PEEL>
__global__ void __launch_bounds__(BLOCK, MINB) dot_peer_kernel(const __grid_constant__ PeerDotArgs<T> a) {
    __shared__ T red[32];
    __shared__ bool am_last;
    const int lr = blockIdx.y;
    const unsigned nblk = a.grid[lr];
    pdl_trigger();
    if (blockIdx.x >= nblk) { // emulation: a rank with a smaller grid
        pdl_wait();
        return;
    }
    if (a.prefetch && a.vec_ok[lr] && threadIdx.x < 2 * U) { // as dot_kernel: warm L2 before the wait
        const uint64_t head = PEEL ? a.head[lr] : 0;
        const uint64_t nvec = (a.n[lr] - head) / Vec<T>::N;
        const uint64_t T_all = uint64_t(nblk) * BLOCK;
        const uint64_t v0 = uint64_t(blockIdx.x) * BLOCK + uint64_t(threadIdx.x >> 1) * T_all;
        if (v0 < nvec) {
            const uint64_t cnt = nvec - v0 < uint64_t(BLOCK) ? nvec - v0 : uint64_t(BLOCK);
            const T* base = ((threadIdx.x & 1) ? a.y[lr] : a.x[lr]) + head;
            prefetch_l2_bulk(base + v0 * Vec<T>::N, unsigned(cnt * sizeof(Vec<T>)));
        }
    }
    pdl_wait();
    unsigned long long prev_epoch = 0; // in flight during the sweep
    if (threadIdx.x == 0)
        prev_epoch = *reinterpret_cast<volatile unsigned long long*>(
            &static_cast<PeerMailbox*>(a.mbox[a.rank0 + lr])->epoch);
    const T s = dot_thread_sum<T, BLOCK, U, PEEL>(a.x[lr], a.y[lr], a.n[lr], a.vec_ok[lr],
                                                  a.head[lr], blockIdx.x, nblk);
    const T cta_total = block_sum(s, red);
    if (nblk == 1) {
        peer_finish(cta_total, a, lr, prev_epoch);
        return;
    }
    T* partials = a.partials[lr];
    unsigned* ticket = a.counters[lr] + 1;
    if (threadIdx.x == 0) partials[blockIdx.x] = cta_total;
    if (!last_arriver(ticket, nblk, &am_last)) return;
    T v = T(0);
    for (unsigned i = threadIdx.x; i < nblk; i += BLOCK) v = add_rn(v, ld_cg(partials + i));
    const T total = block_sum(v, red);
    if (threadIdx.x == 0) *ticket = 0u;
    peer_finish(total, a, lr, prev_epoch);
}

// Chunked shard (dot_chunk_kernel's body) + fused exchange.
template <typename T, int BLOCK, int U, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB)
    dot_peer_chunk_kernel(const __grid_constant__ PeerDotArgs<T> a) {
    pdl_enter();
    __shared__ T red[32];
    __shared__ unsigned long long next_sh;
    __shared__ bool am_last;
    const int lr = blockIdx.y;
    const unsigned nblk = a.grid[lr];
    if (blockIdx.x >= nblk) return;
    unsigned* counters = a.counters[lr];
    unsigned long long prev_epoch = 0;
    if (threadIdx.x == 0)
        prev_epoch = *reinterpret_cast<volatile unsigned long long*>(
            &static_cast<PeerMailbox*>(a.mbox[a.rank0 + lr])->epoch);
    dot_chunk_sweep<T, BLOCK, U>(a.x[lr], a.y[lr], a.n[lr], a.partials[lr], counters, a.chunk[lr],
                                 blockIdx.x, nblk, red, &next_sh);
    if (!last_arriver(counters + 1, nblk, &am_last)) return;
    const T total = dot_chunk_total<T, BLOCK>(a.x[lr], a.y[lr], a.n[lr], a.partials[lr],
                                              a.chunk[lr], red);
    if (threadIdx.x == 0) counters[1] = 0u;
    peer_finish(total, a, lr, prev_epoch);
}

// Column-sharded col-major GEMV combine (shard.sharded_gemv_cols without the
// all-gather): every rank pushes its partial c (m values, from zero) into
// slot [epoch parity][rank] of every rank's slot buffer, fences, publishes an
// epoch-tagged mailbox word, waits for every peer's word, and adds the world
// partials to its replica of c in rank order — bitwise the all-gather +
// cabl_cuda_combine_rows path, in one single-CTA kernel per rank with no
// collective call.  Parity double-buffering as for the DOT slots.
template <typename T>
__global__ void __launch_bounds__(1024) combine_rows_peer_kernel(const __grid_constant__ PeerRowsArgs<T> a) {
    pdl_enter();
    __shared__ unsigned epoch_sh;
    const int lr = blockIdx.y;
    const int rank = a.rank0 + lr;
    const uint64_t m = a.m;
    PeerMailbox* mine = static_cast<PeerMailbox*>(a.mbox[rank]);
    if (threadIdx.x == 0)
        epoch_sh = unsigned(*reinterpret_cast<volatile unsigned long long*>(&mine->epoch) + 1);
    __syncthreads();
    const unsigned e = epoch_sh;
    const int p = e & 1;
    const T* part = a.part[lr];
    const uint64_t my_slot = (uint64_t(p) * kMaxPeers + uint64_t(rank)) * m;
    for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) {
        const T v = part[i];
        for (int g = 0; g < a.world; ++g)
            if (g != rank) a.slots[g][my_slot + i] = v;
    }
    if (a.world > 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
    __syncthreads();
    if (int(threadIdx.x) < a.world && int(threadIdx.x) != rank) {
        PeerMailbox* peer = static_cast<PeerMailbox*>(a.mbox[threadIdx.x]);
        st_relaxed_sys(&peer->word[p][rank][0], (unsigned long long)e << 32);
    }
    __shared__ bool ok_sh;
    if (threadIdx.x == 0) {
        const unsigned long long t0 = globaltimer();
        bool ok = true;
        for (int g = 0; g < a.world && ok; ++g) {
            if (g == rank) continue;
            while (unsigned(ld_relaxed_sys(&mine->word[p][g][0]) >> 32) != e) {
                if (globaltimer() - t0 > a.timeout_ns) {
                    ok = false;
                    break;
                }
                __nanosleep(64);
            }
        }
        if (a.world > 1) asm volatile("fence.acq_rel.sys;" ::: "memory");
        ok_sh = ok;
        if (!ok) mine->fault = e;
        mine->epoch = e;
    }
    __syncthreads();
    if (!ok_sh) return; // c untouched; the fault is recorded
    const T* own = a.slots[rank] + uint64_t(p) * kMaxPeers * m;
    T* c = a.c[lr];
    for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) {
        T total = T(0);
        for (int g = 0; g < a.world; ++g)
            total = add_rn(total, g == rank ? part[i] : ld_cg(own + uint64_t(g) * m + i));
        c[i] = add_rn(c[i], total);
    }
}

} // namespace

template <typename T>
cudaError_t dot_peer_launch(const PeerDotArgs<T>& a, int local_ranks, bool chunked, bool peel,
                            bool cooperative, cudaStream_t s) {
    unsigned gx = 1;
    for (int i = 0; i < local_ranks; ++i) gx = a.grid[i] > gx ? a.grid[i] : gx;
    const dim3 grid(gx, unsigned(local_ranks));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kDotBlock);
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
    if (chunked)
        return cudaLaunchKernelEx(&cfg, dot_peer_chunk_kernel<T, kDotBlock, kDotUnroll, kDotCtasPerSm>, a);
    if (peel)
        return cudaLaunchKernelEx(&cfg, dot_peer_kernel<T, kDotBlock, kDotUnroll, kDotCtasPerSm, true>, a);
    return cudaLaunchKernelEx(&cfg, dot_peer_kernel<T, kDotBlock, kDotUnroll, kDotCtasPerSm, false>, a);
}

// CTAs of the DOT kernels one SM holds at once (the emulation's co-residency bound)
int dot_peer_ctas_per_sm(bool chunked, size_t elem) {
    int b = 0;
    cudaError_t e;
    if (elem == 4)
        e = chunked ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                          &b, dot_peer_chunk_kernel<float, kDotBlock, kDotUnroll, kDotCtasPerSm>, kDotBlock, 0)
                    : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                          &b, dot_peer_kernel<float, kDotBlock, kDotUnroll, kDotCtasPerSm, true>, kDotBlock, 0);
    else
        e = chunked ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                          &b, dot_peer_chunk_kernel<double, kDotBlock, kDotUnroll, kDotCtasPerSm>, kDotBlock, 0)
                    : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                          &b, dot_peer_kernel<double, kDotBlock, kDotUnroll, kDotCtasPerSm, true>, kDotBlock, 0);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return b;
}

template <typename T>
cudaError_t combine_rows_peer_launch(const PeerRowsArgs<T>& a, int local_ranks, bool cooperative,
                                     cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1, unsigned(local_ranks));
    cfg.blockDim = dim3(1024);
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
    return cudaLaunchKernelEx(&cfg, combine_rows_peer_kernel<T>, a);
}
template cudaError_t combine_rows_peer_launch<float>(const PeerRowsArgs<float>&, int, bool,
                                                     cudaStream_t);
template cudaError_t combine_rows_peer_launch<double>(const PeerRowsArgs<double>&, int, bool,
                                                      cudaStream_t);

template cudaError_t dot_peer_launch<float>(const PeerDotArgs<float>&, int, bool, bool, bool,
                                            cudaStream_t);
template cudaError_t dot_peer_launch<double>(const PeerDotArgs<double>&, int, bool, bool, bool,
                                             cudaStream_t);

} // namespace cabl_dev

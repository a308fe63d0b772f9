// Internal launcher interface between the C ABI (capi.cu) and the kernels.
// Not installed; the public boundary is include/cabl_cuda.h.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <string>

namespace cabl_dev {

// Per-(device, stream) scratch owned by the C ABI.  `counters` are zero on
// entry and every kernel that uses them leaves them zero on exit (the
// last-arriving CTA resets what it used), so the workspace is reusable by the
// next launch on the same stream without a memset.
//
// `slots` are epoch-tagged 64-bit words, zero when allocated and used only by
// the DOT kernel's collector (dot.cu): slots[0] holds the last completed
// epoch, slots[1..] the CTAs' tagged partials.  A stale word never carries
// the current epoch, so they need no reset between launches.
struct Workspace {
    unsigned* counters = nullptr;
    size_t n_counters = 0;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    unsigned long long* slots = nullptr;
    size_t n_slots = 0;
};

struct WorkspaceNeed {
    size_t counters = 0;
    size_t scratch_bytes = 0;
    size_t slots = 0;
};

struct LaunchInfo {
    unsigned ctas = 0; // CTAs of the main pass (probe threads_used)
};

int sm_count(); // of the current device (cached per device)
void set_last_error(const std::string& msg); // cabl_last_error() of this thread (capi.cu)
uint64_t queue_threshold_bytes(); // work-queue size rule, from the device L2 (capi.cu)

// ---- DOT (dot.cu) ----
// Launch plan of the single-GPU DOT for (x, y, n): which kernel, its grid,
// the aligned-vector path and peeled head, and the chunk size of the chunked
// kernel.  The peer-memory DOT (peer.cu) runs each rank's shard with exactly
// this plan, so its per-rank partial is the bits dot_launch(alpha0 = 0) gives.
struct DotPlan {
    bool chunked = false;
    unsigned grid = 1;
    int vec_ok = 0;
    uint64_t head = 0;
    uint64_t chunk = 0; // vectors per chunk (chunked kernel)
};
template <typename T> DotPlan dot_plan(const T* x, const T* y, uint64_t n, bool small);
template <typename T> WorkspaceNeed dot_need(uint64_t n, bool small);
template <typename T>
cudaError_t dot_launch(const T* x, const T* y, uint64_t n, T alpha0, T* out, bool small,
                       const Workspace& ws, cudaStream_t s, LaunchInfo* info);
template <typename T>
cudaError_t combine_partials_launch(const T* p, uint32_t count, T alpha0, T* out,
                                    cudaStream_t s);
template <typename T>
cudaError_t combine_rows_launch(const T* parts, uint32_t count, uint64_t m, T* c,
                                cudaStream_t s);

// ---- peer-memory DOT (peer.cu) ----
constexpr int kMaxPeers = 8; // ranks of one NVLink / NVSwitch domain (one node)

// One rank's mailbox (512 B, zeroed at creation; layout shared by every rank).
// word[p][g][h] = (epoch << 32) | 32-bit half h of rank g's partial for the
// last epoch of parity p (fp32 uses h = 0 only): the tag and the data are one
// single-copy-atomic 8-byte store, so neither side needs a fence.
struct PeerMailbox {
    unsigned long long word[2][kMaxPeers][2];
    unsigned long long epoch; // this rank's completed calls (owner-written)
    unsigned long long fault; // epoch of a call whose wait timed out (0 = none)
    unsigned long long reserved[30];
};

// Kernel argument block.  Local slot lr (blockIdx.y) is rank rank0 + lr; a
// real multi-GPU call has one local slot, the emulation has `world`.
template <typename T> struct PeerDotArgs {
    const T* x[kMaxPeers];
    const T* y[kMaxPeers];
    T* out[kMaxPeers];
    uint64_t n[kMaxPeers];
    uint64_t head[kMaxPeers];
    uint64_t chunk[kMaxPeers];
    T* partials[kMaxPeers];
    unsigned* counters[kMaxPeers]; // [0] chunk queue, [1] ticket; zero on entry and exit
    unsigned grid[kMaxPeers];
    int vec_ok[kMaxPeers];
    void* mbox[kMaxPeers]; // every rank's mailbox, as addressable from this device
    int world;
    int rank0;
    unsigned long long timeout_ns;
    int prefetch; // pre-wait L2 prefetch (dot_kernel's; CABL_PDL_PREFETCH)
    T alpha0;
};
template <typename T>
cudaError_t dot_peer_launch(const PeerDotArgs<T>& a, int local_ranks, bool chunked, bool peel,
                            bool cooperative, cudaStream_t s);
int dot_peer_ctas_per_sm(bool chunked, size_t elem);

// ---- rank-ordered combine of partial c vectors over peer memory (peer.cu) ----
template <typename T> struct PeerRowsArgs {
    const T* part[kMaxPeers]; // the rank's partial c (m values)
    T* c[kMaxPeers];          // the rank's replica of c (c += sum of partials)
    T* slots[kMaxPeers];      // rank g's slot buffer (2 x kMaxPeers x m), as mapped here
    void* mbox[kMaxPeers];
    uint64_t m;
    int world, rank0;
    unsigned long long timeout_ns;
};
template <typename T>
cudaError_t combine_rows_peer_launch(const PeerRowsArgs<T>& a, int local_ranks, bool cooperative,
                                     cudaStream_t s);

// ---- row-major GEMV with the c all-gather fused (peer_gemv.cu) ----
template <typename T> struct PeerGemvArgs {
    const T* A[kMaxPeers];
    const T* x[kMaxPeers];
    T* c[kMaxPeers];                // the rank's own c slice (c += A x in place)
    uint64_t m[kMaxPeers];          // rows of the rank's slice
    uint64_t row_off[kMaxPeers];    // first global row of the slice
    unsigned grid[kMaxPeers];
    unsigned* counters[kMaxPeers];  // [0] group queue, [1] ticket; zero on entry and exit
    T* cfull[kMaxPeers];            // rank g's double buffer (2 x m_total), as mapped here
    void* mbox[kMaxPeers];          // rank g's gather mailbox, as mapped here
    uint64_t n, m_total;
    int world, rank0;
    unsigned long long timeout_ns;
    int fence; // 0 none (world 1), 1 acq_rel.sys, 2 sc.sys
};
template <typename T>
cudaError_t gemv_rm_gather_launch(const PeerGemvArgs<T>& a, int local_ranks, int R, int KV,
                                  int minb, bool dyn, bool cooperative, cudaStream_t s);
int gemv_rm_gather_ctas_per_sm(int R, int KV, int minb, size_t elem);

// ---- GEMV row-major (gemv_rm.cu) ----
template <typename T> WorkspaceNeed gemv_rm_need(const T* A, const T* x, uint64_t m, uint64_t n);
// short rows, many of them: the one-thread-per-row kernel (reference order,
// bitwise gemv_ref) handles the shape on any alignment
bool gemv_rm_is_lane(const void* A, const void* x, uint64_t m, uint64_t n, size_t elem);
template <typename T>
cudaError_t gemv_rm_launch(const T* A, uint64_t m, uint64_t n, const T* x, T* c,
                           const Workspace& ws, cudaStream_t s, LaunchInfo* info);

// The sweep shape (rows per group, vectors per pass, CTAs per SM) plain
// gemv_rm_launch uses for this shape; false when the shape takes another
// kernel.  The gathering sweep (peer_gemv.cu) runs exactly this shape.
template <typename T>
bool gemv_rm_sweep_cfg(const T* A, const T* x, uint64_t m, uint64_t n, int* R, int* KV, int* minb);
bool gemv_rm_use_dyn(uint64_t bytes); // the sweep's queue rule

// ---- GEMV row-major in the reference's order (gemv_rm_ordered.cu): bit for
// bit the compiled reference gemv_row_major / gemv_ref ----
template <typename T> bool gemv_rm_ordered_ok(const T* A, const T* x, uint64_t m, uint64_t n);
template <typename T>
cudaError_t gemv_rm_ordered_launch(const T* A, uint64_t m, uint64_t n, const T* x, T* c,
                                   cudaStream_t s, LaunchInfo* info);

// ---- GEMV col-major (gemv_cm.cu) ----
template <typename T> WorkspaceNeed gemv_cm_need(const T* A, const T* x, uint64_t m, uint64_t n);
template <typename T>
cudaError_t gemv_cm_launch(const T* A, uint64_t m, uint64_t n, const T* x, T* c,
                           const Workspace& ws, cudaStream_t s, LaunchInfo* info);

// ---- ordered single-CTA GEMV (gemv_small.cu): reproduces the compiled
// reference gemv_ref bit for bit (oracle/cabl_oracle.c documents the
// semantics: vec-wide mul-then-add prefix, FMA remainder). layout 0 = RM.
template <typename T>
cudaError_t gemv_ordered_launch(const T* A, int layout, uint64_t m, uint64_t n, const T* x,
                                T* c, cudaStream_t s, LaunchInfo* info);

// ---- GER (ger.cu): C(major, minor) = fma(u[major], v[minor], C) over an
// outer x inner row-major view; the col-major GER is the same kernel with
// (x, m) and (y, n) swapped, since fma(a, b, c) == fma(b, a, c).
template <typename T> WorkspaceNeed ger_need(const T* u, const T* v, uint64_t outer, uint64_t inner);
template <typename T>
cudaError_t ger_launch(const T* u, const T* v, T* C, uint64_t outer, uint64_t inner,
                       bool small, const Workspace& ws, cudaStream_t s, LaunchInfo* info);

// ---- seeded inputs (datagen.cu) ----
cudaError_t fill_uniform_f32(float* out, uint64_t n, uint64_t seed, uint64_t sid,
                             uint64_t offset, cudaStream_t s);
cudaError_t fill_uniform_f64(double* out, uint64_t n, uint64_t seed, uint64_t sid,
                             uint64_t offset, cudaStream_t s);
cudaError_t fill_normal_f64(double* out, uint64_t n, uint64_t seed, uint64_t sid,
                            uint64_t offset, cudaStream_t s);

} // namespace cabl_dev

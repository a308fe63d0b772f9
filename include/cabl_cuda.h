/*
 * cabl_cuda.h — the C ABI of the B200-native DOT / GEMV / GER library
 * (libcabl_cuda.so, built from paper_2108_02025_b200/csrc/).
 *
 * This is the drop-in boundary for the hot path of the reference library
 * `cabl` (arXiv 2108.02025).  The reference is a header-only C++20 template
 * library; its four hot-path entry points are
 *
 *   T    cabl::dot(const Vector<T>& x, const Vector<T>& y, T alpha0, const ExecPolicy&)
 *            reference proj/include/cabl/kernels.hpp:134-164
 *   void cabl::gemv_col_major(const DenseMatrix<T>& A, const Vector<T>& x, Vector<T>& c,
 *                             const ExecPolicy&)      kernels.hpp:187-224
 *   void cabl::gemv_row_major(same signature)          kernels.hpp:230-257
 *   void cabl::ger(const Vector<T>& x, const Vector<T>& y, DenseMatrix<T>& C,
 *                  const ExecPolicy&)                  kernels.hpp:277-313
 *
 * The drop-in header include/cabl/kernels.hpp keeps those signatures and
 * forwards here.  Every symbol below is plain C: raw pointers, sizes, an int
 * status and an opaque stream (a cudaStream_t passed as void*; NULL means
 * the legacy default stream).  There is no CPU fallback: when no CUDA device
 * is usable every compute entry point returns CABL_ECUDA.
 *
 * Device entry points (`cabl_cuda_*`) take DEVICE pointers and only enqueue
 * work on `stream`.  Host entry points (`cabl_host_*`) take HOST pointers
 * (pinned or pageable), stage through device memory on `stream`, and return
 * after the result is back on the host — they are what the C++ drop-in
 * overloads on cabl::Vector / cabl::DenseMatrix call.
 *
 * Semantics are the reference's: pure accumulate (alpha0 + x.y, c += A x,
 * C += x (x) y), no scaling, no strides (reference SPEC.md:292,304).
 * Zero-size operands are no-ops; DOT of empty vectors returns alpha0.
 * Results are bitwise reproducible run to run for fixed inputs and device.
 */
#ifndef CABL_CUDA_H
#define CABL_CUDA_H

#include <stdint.h>

#if defined(__GNUC__)
#define CABL_API __attribute__((visibility("default")))
#else
#define CABL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  CABL_EINVAL mirrors the reference's std::invalid_argument
 * (kernels.hpp:59-61); the message is available from cabl_last_error(). */
enum {
    CABL_OK = 0,
    CABL_EINVAL = 1,
    CABL_ECUDA = 2,
    CABL_ENOMEM = 3,
    CABL_ENCCL = 4 /* multi-GPU exchange failed (cabl_mgpu_*): NCCL error, asynchronous
                      NCCL error, a timed-out peer exchange, or the context's timeout */
};

/* Storage order of a dense matrix — reference dense.hpp:9, element (i,j) at
 * j + i*cols (row-major) or i + j*rows (col-major), dense.hpp:54-56. */
enum { CABL_ROW_MAJOR = 0, CABL_COL_MAJOR = 1 };

/* Execution-path probe — reference KernelVariant / ExecProbe, kernels.hpp:40-55.
 * Numbering matches the reference enum order. */
enum {
    CABL_VARIANT_NONE = 0,
    CABL_VARIANT_DOT_SMALL = 1,
    CABL_VARIANT_DOT_BLOCKED = 2,
    CABL_VARIANT_GEMV_COL_BLOCKED = 3,
    CABL_VARIANT_GEMV_ROW = 4,
    CABL_VARIANT_GER = 5
};

typedef struct cabl_probe {
    int variant;           /* CABL_VARIANT_* */
    unsigned threads_used; /* CTAs launched on the main pass (1 for the ordered small path) */
} cabl_probe;

/* Thread-local message of the last failing call on this thread ("" if none). */
CABL_API const char* cabl_last_error(void);
/* ABI version (major*100 + minor). */
CABL_API int cabl_abi_version(void);
/* Number of usable CUDA devices (0 when none; never a CPU fallback). */
CABL_API int cabl_device_count(void);

/* ------------------------------------------------- machine descriptor ---
 * The GPU counterpart of the reference's MachineDescriptor (machine.hpp:43-53)
 * and its flat JSON document (descriptor_json.hpp:3-15): the device's memory
 * hierarchy, read from the driver.  The host mirrors map it onto the
 * reference descriptor (cores = SMs; L1 = the per-SM shared-memory capacity,
 * L2 = the device L2, 128-byte lines) and derive the launch parameters from it
 * (derive_gpu_plan) instead of hard-coding B200 numbers.  The library itself
 * sizes its grids from sm_count and its work-queue threshold from l2_bytes
 * (queue_threshold_bytes below).  Returns CABL_ECUDA when `device` is not a
 * usable CUDA device. */
typedef struct cabl_gpu_machine {
    int32_t device;
    int32_t cc_major, cc_minor;
    uint32_t sm_count;             /* "cores" of the descriptor */
    uint32_t max_threads_per_sm;
    uint32_t line_bytes;           /* L1 / L2 line (128) */
    uint64_t smem_per_sm;          /* shared memory per SM (the descriptor's L1) */
    uint64_t smem_per_block_optin; /* largest dynamic smem one CTA may opt into */
    uint64_t l2_bytes;
    uint64_t hbm_bytes;
    uint32_t mem_bus_bits;
    uint32_t reserved;
    uint64_t queue_threshold_bytes; /* operands >= this take the atomic work queues:
                                       4 x L2 rounded up to a power of two */
    char name[96];
} cabl_gpu_machine;

CABL_API int cabl_describe_device(int device, cabl_gpu_machine* out);

/* ---------------------------------------------------------------- DOT ---
 * *out = alpha0 + sum_p x[p]*y[p]   (device scalar; alpha0 is added last,
 * as reference kernels.hpp:142,163 do).
 * n <= small_cutoff runs the single-CTA path (reference dot_small,
 * kernels.hpp:140-143); otherwise the bandwidth path over the whole GPU.
 * `probe` may be NULL.  Replaces cabl::dot<float|double>, kernels.hpp:134. */
CABL_API int cabl_cuda_dot_f32(const float* x, const float* y, uint64_t n, float alpha0, float* out,
                      uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_cuda_dot_f64(const double* x, const double* y, uint64_t n, double alpha0,
                      double* out, uint64_t small_cutoff, cabl_probe* probe, void* stream);

/* Deterministic, rank-ordered combine of `count` partial dot products (one per
 * shard / GPU): *out = ((p[0] + p[1]) + ...) + alpha0, summed left to right in
 * index order like the reference combines thread partials (kernels.hpp:160-163).
 * Used by the multi-GPU DOT after the partials are all-gathered. */
CABL_API int cabl_cuda_combine_partials_f32(const float* partials, uint32_t count, float alpha0,
                                   float* out, void* stream);
CABL_API int cabl_cuda_combine_partials_f64(const double* partials, uint32_t count, double alpha0,
                                   double* out, void* stream);

/* Rank-ordered combine of `count` partial c vectors (column-sharded
 * col-major GEMV: each rank computes A[:, cols_r] x[cols_r] from zero; the
 * partials are all-gathered as parts[g*m + i]):
 *   c[i] += ((parts[0*m+i] + parts[1*m+i]) + ...)   in rank order,
 * bitwise identical on every rank whatever the collective's algorithm. */
CABL_API int cabl_cuda_combine_rows_f32(const float* parts, uint32_t count, uint64_t m, float* c,
                                        void* stream);
CABL_API int cabl_cuda_combine_rows_f64(const double* parts, uint32_t count, uint64_t m,
                                        double* c, void* stream);

/* ------------------------------------------- multi-GPU DOT, fused exchange ---
 * The sharded DOT of SURVEY.md §8(e) (rank g owns a contiguous shard of x and
 * y) with the exchange of partials fused into the DOT kernel over peer memory
 * (NVLink / NVSwitch P2P stores), instead of an NCCL all-gather followed by
 * cabl_cuda_combine_partials.  Each rank computes its shard partial with the
 * single-GPU plan, stores it into every rank's mailbox, waits for all `world`
 * partials and writes *out = ((p_0 + p_1) + ...) + alpha0 — bitwise the
 * unfused path's result (cabl_cuda_dot(alpha0 = 0) per shard, then
 * cabl_cuda_combine_partials), identical on every rank.
 *
 * Mailboxes: each rank creates one (cabl_peer_mailbox_create, on its device),
 * exports an IPC handle, imports every other rank's handle, and passes the
 * table mboxes[0..world) — its own mailbox at [rank], the peers' mappings
 * elsewhere.  One process driving several devices passes device pointers
 * directly after cudaDeviceEnablePeerAccess.  Calls are collective: every
 * rank calls with the same table order, in the same sequence.  A rank that
 * does not arrive within CABL_PEER_TIMEOUT_MS (default 30000) makes the
 * waiting ranks write NaN and record the call in their mailbox's `fault`
 * (cabl_peer_mailbox_state) instead of hanging.  world <= 8.
 * Replaces cabl::dot (reference kernels.hpp:134-164) across GPUs. */
typedef struct cabl_peer_handle {
    unsigned char bytes[64]; /* cudaIpcMemHandle_t */
} cabl_peer_handle;

CABL_API int cabl_peer_mailbox_create(void** mbox); /* 512 B on the current device */
CABL_API int cabl_peer_mailbox_destroy(void* mbox);
CABL_API int cabl_peer_mailbox_export(void* mbox, cabl_peer_handle* out);
CABL_API int cabl_peer_mailbox_import(const cabl_peer_handle* h, void** mapped);
CABL_API int cabl_peer_mailbox_unmap(void* mapped);
/* Synchronous read of a mailbox's completed-call count and fault epoch. */
CABL_API int cabl_peer_mailbox_state(const void* mbox, uint64_t* epoch, uint64_t* fault);

CABL_API int cabl_cuda_dot_peer_f32(const float* x, const float* y, uint64_t n, float alpha0,
                                    float* out, void* const* mboxes, int world, int rank,
                                    uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_cuda_dot_peer_f64(const double* x, const double* y, uint64_t n, double alpha0,
                                    double* out, void* const* mboxes, int world, int rank,
                                    uint64_t small_cutoff, cabl_probe* probe, void* stream);

/* Every rank of a peer DOT on the CURRENT device, in one cooperative launch
 * (blockIdx.y = rank; mailboxes all on this device): the same kernel and
 * protocol as cabl_cuda_dot_peer_*, for testing the exchange with fewer GPUs
 * than ranks.  xs/ys/ns/outs/mboxes have `world` entries.  CABL_EINVAL when
 * the ranks' grids do not fit one co-resident wave. */
CABL_API int cabl_cuda_dot_peer_emulate_f32(int world, const float* const* xs,
                                            const float* const* ys, const uint64_t* ns,
                                            float alpha0, float* const* outs,
                                            void* const* mboxes, uint64_t small_cutoff,
                                            void* stream);
CABL_API int cabl_cuda_dot_peer_emulate_f64(int world, const double* const* xs,
                                            const double* const* ys, const uint64_t* ns,
                                            double alpha0, double* const* outs,
                                            void* const* mboxes, uint64_t small_cutoff,
                                            void* stream);

/* -------------------------------- column-sharded GEMV combine, peer memory ---
 * SURVEY.md §8(e) "G3 by columns": rank g computes part_g = A[:, cols_g] x[cols_g]
 * (m values, from zero) with cabl_cuda_gemv_cm; then every rank needs
 * c += ((part_0 + part_1) + ...) in rank order.  This single kernel per rank
 * pushes part into slot (epoch parity, rank) of every rank's slot buffer over
 * P2P, exchanges epoch-tagged mailbox words and adds the world partials in
 * rank order: bitwise the all-gather + cabl_cuda_combine_rows path, with no
 * collective call.  slots[g]: rank g's buffer of 2 * 8 * m elements from
 * cabl_peer_alloc (as mapped here); mboxes: a mailbox set used only by this
 * operation.  Collective; a missing rank records a fault and leaves c as is.
 * The rank-ordered combine follows reference kernels.hpp:160-163. */
CABL_API int cabl_cuda_combine_rows_peer_f32(const float* part, uint64_t m, float* c,
                                             void* const* slots, void* const* mboxes, int world,
                                             int rank, void* stream);
CABL_API int cabl_cuda_combine_rows_peer_f64(const double* part, uint64_t m, double* c,
                                             void* const* slots, void* const* mboxes, int world,
                                             int rank, void* stream);
CABL_API int cabl_cuda_combine_rows_peer_emulate_f32(int world, const float* const* parts,
                                                     uint64_t m, float* const* cs,
                                                     void* const* slots, void* const* mboxes,
                                                     void* stream);
CABL_API int cabl_cuda_combine_rows_peer_emulate_f64(int world, const double* const* parts,
                                                     uint64_t m, double* const* cs,
                                                     void* const* slots, void* const* mboxes,
                                                     void* stream);

/* ------------------------------------ row-major GEMV, c all-gather fused ---
 * BASELINE config 5 / SURVEY.md §8(e): rank g owns rows [row_off, row_off+m)
 * of A and of c (x replicated), and every rank needs the full c.  One kernel
 * per rank computes c_slice += A_slice x with the single-GPU sweep (same bits
 * as cabl_cuda_gemv_rm on the slice) and stores every finished row into every
 * rank's gathered buffer over NVLink P2P; it ends when all ranks' rows have
 * arrived.  No NCCL call.
 *
 * cfull[g]: rank g's gathered buffer, 2 * m_total elements allocated with
 * cabl_peer_alloc on rank g's device (double-buffered: the e-th call on a
 * mailbox fills half e & 1, i.e. elements [(e & 1) * m_total, +m_total);
 * ranks in separate processes must consume half e & 1, in stream order,
 * before issuing call e + 1 — a faster peer may then write call e + 2 there),
 * as mapped here (cabl_peer_mailbox_export / _import work on any
 * cabl_peer_alloc pointer).  mboxes: a mailbox set used only by this
 * operation.  Calls are collective.  CABL_EINVAL when the slice shape does not
 * take the sweep kernel (few or short rows, unaligned): use cabl_cuda_gemv_rm
 * plus a collective there.  A rank that never arrives makes the others record
 * the epoch in their mailbox's `fault` after CABL_PEER_TIMEOUT_MS.
 * Replaces cabl::gemv_row_major (reference kernels.hpp:230-257) across GPUs. */
CABL_API int cabl_peer_alloc(uint64_t bytes, void** ptr); /* zeroed, exportable */
CABL_API int cabl_peer_free(void* ptr);
CABL_API int cabl_cuda_gemv_rm_gather_f32(const float* A, uint64_t m, uint64_t n, const float* x,
                                          float* c, uint64_t row_off, uint64_t m_total,
                                          void* const* cfull, void* const* mboxes, int world,
                                          int rank, cabl_probe* probe, void* stream);
CABL_API int cabl_cuda_gemv_rm_gather_f64(const double* A, uint64_t m, uint64_t n,
                                          const double* x, double* c, uint64_t row_off,
                                          uint64_t m_total, void* const* cfull,
                                          void* const* mboxes, int world, int rank,
                                          cabl_probe* probe, void* stream);
/* Every rank in one cooperative launch on the current device (testing with
 * fewer GPUs than ranks; all slices must take the same sweep shape). */
/* *ok = 1 when the slice shape (on the current device) takes the gathering
 * sweep kernel, else 0 — so a caller can check every rank before launching
 * any (a rank rejected after its peers launched would leave them waiting). */
CABL_API int cabl_cuda_gemv_rm_gather_supported_f32(const float* A, uint64_t m, uint64_t n,
                                                    const float* x, int* ok);
CABL_API int cabl_cuda_gemv_rm_gather_supported_f64(const double* A, uint64_t m, uint64_t n,
                                                    const double* x, int* ok);
CABL_API int cabl_cuda_gemv_rm_gather_emulate_f32(int world, const float* const* As,
                                                  const uint64_t* ms, uint64_t n,
                                                  const float* const* xs, float* const* cs,
                                                  const uint64_t* row_offs, uint64_t m_total,
                                                  void* const* cfull, void* const* mboxes,
                                                  void* stream);
CABL_API int cabl_cuda_gemv_rm_gather_emulate_f64(int world, const double* const* As,
                                                  const uint64_t* ms, uint64_t n,
                                                  const double* const* xs, double* const* cs,
                                                  const uint64_t* row_offs, uint64_t m_total,
                                                  void* const* cfull, void* const* mboxes,
                                                  void* stream);

/* --------------------------------------------------------------- GEMV ---
 * c[0..m) += A x, A is m x n.  `small_cutoff`: when m*n + m + n <= cutoff the
 * call runs the ordered single-CTA path, which reproduces the compiled
 * reference gemv_ref / gemv_row_major bit for bit (reference kernels.hpp:238-243).
 * Replaces cabl::gemv_row_major (kernels.hpp:230) and cabl::gemv_col_major
 * (kernels.hpp:187); the layout is part of the symbol, as the reference
 * rejects the other layout (kernels.hpp:190,233). c must not alias x. */
CABL_API int cabl_cuda_gemv_rm_f32(const float* A, uint64_t m, uint64_t n, const float* x, float* c,
                          uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_cuda_gemv_rm_f64(const double* A, uint64_t m, uint64_t n, const double* x, double* c,
                          uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_cuda_gemv_cm_f32(const float* A, uint64_t m, uint64_t n, const float* x, float* c,
                          uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_cuda_gemv_cm_f64(const double* A, uint64_t m, uint64_t n, const double* x, double* c,
                          uint64_t small_cutoff, cabl_probe* probe, void* stream);

/* ---------------------------------------------------------------- GER ---
 * C(i,j) = fma(x[i], y[j], C(i,j)) for i < m, j < n — exactly one fused
 * multiply-add per element, bitwise equal to the reference ger_ref / ger
 * (kernels.hpp:264-313).  x has m entries, y has n; C must not alias x or y.
 * Replaces cabl::ger (kernels.hpp:277): _rm = RowMajor branch (:300-310),
 * _cm = ColMajor branch (:290-299). */
CABL_API int cabl_cuda_ger_rm_f32(const float* x, const float* y, float* C, uint64_t m, uint64_t n,
                         uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_cuda_ger_rm_f64(const double* x, const double* y, double* C, uint64_t m, uint64_t n,
                         uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_cuda_ger_cm_f32(const float* x, const float* y, float* C, uint64_t m, uint64_t n,
                         uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_cuda_ger_cm_f64(const double* x, const double* y, double* C, uint64_t m, uint64_t n,
                         uint64_t small_cutoff, cabl_probe* probe, void* stream);

/* ------------------------------------------------- host-buffer entry points
 * Same operations on HOST buffers (what the C++ drop-in overloads on
 * cabl::Vector / cabl::DenseMatrix call): H2D copy of the operands, the
 * device kernel, D2H copy of the result, then a stream synchronize.  `layout`
 * is CABL_ROW_MAJOR / CABL_COL_MAJOR.  Temporaries come from a library-owned
 * stream-ordered device pool (never freed mid-call, thread-safe). */
CABL_API int cabl_host_dot_f32(const float* x, const float* y, uint64_t n, float alpha0, float* result,
                      uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_host_dot_f64(const double* x, const double* y, uint64_t n, double alpha0,
                      double* result, uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_host_gemv_f32(const float* A, int layout, uint64_t m, uint64_t n, const float* x,
                       float* c, uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_host_gemv_f64(const double* A, int layout, uint64_t m, uint64_t n, const double* x,
                       double* c, uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_host_ger_f32(const float* x, const float* y, float* C, int layout, uint64_t m,
                      uint64_t n, uint64_t small_cutoff, cabl_probe* probe, void* stream);
CABL_API int cabl_host_ger_f64(const double* x, const double* y, double* C, int layout, uint64_t m,
                      uint64_t n, uint64_t small_cutoff, cabl_probe* probe, void* stream);

/* ----------------------------------------------- multi-GPU (one process) ---
 * one process drives G devices of one node.  The
 * context holds one NCCL communicator per device (ncclCommInitAll; NCCL is
 * loaded at run time, libnccl.so.2 or $CABL_NCCL_LIB), one non-blocking
 * stream per device (cabl_mgpu_stream) and lazily built peer-memory buffers.
 * Shard arrays have one entry per rank (rank r = devices[r]); shard r lives
 * on device r.  The partition is the caller's (contiguous shards, as the
 * reference's parallel_chunks, thread_pool.hpp:153-164).
 *
 * Every call is synchronous, like the reference templates: it validates all
 * shards before launching anything (CABL_EINVAL), runs the single-GPU kernel
 * on every shard, the exchange, and returns when every device is done.  The
 * wait polls ncclCommGetAsyncError and a timeout (60 s, CABL_MGPU_TIMEOUT_MS
 * or cabl_mgpu_set_timeout_ms): an asynchronous NCCL error, a timed-out peer
 * exchange or the timeout aborts every communicator (ncclCommAbort) and
 * returns CABL_ENCCL — a failure is reported to the caller, never a hang
 * (the reference pool rethrows worker failures, thread_pool.hpp:63-68).  An
 * aborted context returns CABL_ENCCL from every later call; finalize it.
 *
 * exchange: CABL_MGPU_NCCL (collectives) or CABL_MGPU_PEER (the exchange
 * fused into the kernels over NVLink P2P, no collective; needs P2P between
 * every pair).  Both give the same bits.  small_cutoff: as the single-GPU
 * entry points (the reference plan's dot_cutoff).  The context's streams do
 * not wait on the caller's: operands must be ready when a call starts (the
 * call itself returns only after its results are). */
enum { CABL_MGPU_NCCL = 0, CABL_MGPU_PEER = 1 };
typedef struct cabl_mgpu cabl_mgpu;

/* NCCL version the library loads (e.g. 22703); CABL_ENCCL if it cannot. */
CABL_API int cabl_mgpu_nccl_version(int* version);
CABL_API int cabl_mgpu_init(const int* devices, int count, cabl_mgpu** ctx);
CABL_API int cabl_mgpu_finalize(cabl_mgpu* ctx);
CABL_API int cabl_mgpu_size(const cabl_mgpu* ctx);
CABL_API int cabl_mgpu_device(const cabl_mgpu* ctx, int rank);
CABL_API void* cabl_mgpu_stream(const cabl_mgpu* ctx, int rank); /* cudaStream_t of rank */
CABL_API int cabl_mgpu_set_timeout_ms(cabl_mgpu* ctx, uint64_t ms);
/* Device time of the last completed call on `rank`, from before its first
 * launch to the end of its last operation on that rank's stream (CUDA
 * events; the host's wait is not in it).  Multi-GPU time = max over ranks. */
CABL_API int cabl_mgpu_last_call_ms(cabl_mgpu* ctx, int rank, float* ms);

/* *result = alpha0 + sum over ranks (in rank order) of x[r] . y[r]; the
 * per-rank partials are the single-GPU kernel's bits (alpha0 = 0), summed
 * left to right and alpha0 added last (reference kernels.hpp:145-163). */
CABL_API int cabl_mgpu_dot_f32(cabl_mgpu* ctx, const float* const* x, const float* const* y,
                               const uint64_t* n, float alpha0, uint64_t small_cutoff,
                               int exchange, float* result);
CABL_API int cabl_mgpu_dot_f64(cabl_mgpu* ctx, const double* const* x, const double* const* y,
                               const uint64_t* n, double alpha0, uint64_t small_cutoff,
                               int exchange, double* result);
/* The same sum over FIXED GLOBAL SEGMENTS, for a result that does not depend on
 * the GPU count: the shards, concatenated in rank order, are cut every
 * `segment` elements; each segment's partial is the single-GPU kernel's bits
 * for that segment (alpha0 = 0), and *result = alpha0 + the K partials summed in
 * index order.  `segment` must be a multiple of 64 elements, and every shard
 * before the last non-empty one a whole number of segments (CABL_EINVAL
 * otherwise).  One device or eight: the same
 * bits, provided the vectors' base addresses share their 32-byte alignment.
 * (The reference's dot depends on its thread count the same way the plain
 * cabl_mgpu_dot depends on the device count, kernels.hpp:145-163; this is its
 * block decomposition with a fixed block length.)  NCCL all-gather exchange. */
CABL_API int cabl_mgpu_dot_segmented_f32(cabl_mgpu* ctx, const float* const* x,
                                         const float* const* y, const uint64_t* n,
                                         uint64_t segment, float alpha0, uint64_t small_cutoff,
                                         float* result);
CABL_API int cabl_mgpu_dot_segmented_f64(cabl_mgpu* ctx, const double* const* x,
                                         const double* const* y, const uint64_t* n,
                                         uint64_t segment, double alpha0, uint64_t small_cutoff,
                                         double* result);
/* Row blocks: c[r] (m[r]) += A[r] (m[r] x n, row-major) x[r] (x replicated).
 * c_full: NULL, or one device buffer of sum(m) elements per rank that
 * receives every rank's updated slice at its row offset (the all-gather of
 * BASELINE config 5).  Replaces cabl::gemv_row_major (kernels.hpp:230-257). */
CABL_API int cabl_mgpu_gemv_rm_f32(cabl_mgpu* ctx, const float* const* A, const uint64_t* m,
                                   uint64_t n, const float* const* x, float* const* c,
                                   uint64_t small_cutoff, int exchange, float* const* c_full);
CABL_API int cabl_mgpu_gemv_rm_f64(cabl_mgpu* ctx, const double* const* A, const uint64_t* m,
                                   uint64_t n, const double* const* x, double* const* c,
                                   uint64_t small_cutoff, int exchange, double* const* c_full);
/* Column blocks of a col-major A: A[r] is m x n[r], x[r] the matching slice
 * of x, c[r] a replica of c; every replica gets c += ((p_0 + p_1) + ...) in
 * rank order, p_r = A[r] x[r] (same bits on every device).  Replaces
 * cabl::gemv_col_major (kernels.hpp:187-224) for short-wide shapes. */
CABL_API int cabl_mgpu_gemv_cm_cols_f32(cabl_mgpu* ctx, const float* const* A, uint64_t m,
                                        const uint64_t* n, const float* const* x,
                                        float* const* c, uint64_t small_cutoff, int exchange);
CABL_API int cabl_mgpu_gemv_cm_cols_f64(cabl_mgpu* ctx, const double* const* A, uint64_t m,
                                        const uint64_t* n, const double* const* x,
                                        double* const* c, uint64_t small_cutoff, int exchange);
/* Row blocks of a row-major C: C[r] (m[r] x n) += x[r] (m[r]) (x) y (y
 * replicated).  No exchange.  Replaces cabl::ger (kernels.hpp:277-313). */
CABL_API int cabl_mgpu_ger_rm_f32(cabl_mgpu* ctx, const float* const* x, const uint64_t* m,
                                  const float* const* y, uint64_t n, float* const* C,
                                  uint64_t small_cutoff);
CABL_API int cabl_mgpu_ger_rm_f64(cabl_mgpu* ctx, const double* const* x, const uint64_t* m,
                                  const double* const* y, uint64_t n, double* const* C,
                                  uint64_t small_cutoff);

/* ------------------------------------------------------ seeded inputs ---
 * Counter-based SplitMix64 generator, bit-identical to the host oracle's
 * (oracle/cabl_oracle.c): out[i] = U[-1,1) of counter (offset + i) in
 * (seed, stream_id).  The normal variant is Box-Muller on counters
 * (2(offset+i), 2(offset+i)+1).  Stand-in for the reference's seeded
 * mt19937_64 fills (reference bench.hpp:68-71), which are sequential and
 * cannot be reproduced on a GPU. */
CABL_API int cabl_cuda_fill_uniform_f32(float* out, uint64_t n, uint64_t seed, uint64_t stream_id,
                               uint64_t offset, void* stream);
CABL_API int cabl_cuda_fill_uniform_f64(double* out, uint64_t n, uint64_t seed, uint64_t stream_id,
                               uint64_t offset, void* stream);
CABL_API int cabl_cuda_fill_normal_f64(double* out, uint64_t n, uint64_t seed, uint64_t stream_id,
                              uint64_t offset, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CABL_CUDA_H */

/*
 * tcb.h — device-side C-ABI of the B200-native fp64 contraction engine.
 *
 * Plain C, plain pointers and sizes; no CUDA or C++ types cross this boundary,
 * so the host front (C++), ctypes (Python) or any FFI can bind it. Every call
 * returns a tcb_status; on failure tcb_last_error() holds a thread-local
 * message. All matrices are column-major, element strides count doubles.
 *
 * The reference (/root/reference/proj) has no device layer: its arithmetic is
 * the abstract KernelBackend (include/tc/kernels.hpp:12-39) implemented on the
 * CPU by ReferenceBackend (src/kernels_reference.cpp:33-149), driven slice by
 * slice by tc::execute (src/executor.cpp:102-283). Each entry point below names
 * the reference interface it replaces.
 */
#ifndef TCB_H_
#define TCB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum tcb_status {
  TCB_OK = 0,
  TCB_EINVAL = 1,      /* bad argument; message mirrors the reference's std::invalid_argument */
  TCB_ECUDA = 2,       /* CUDA runtime / driver failure */
  TCB_ENCCL = 3,       /* collective failure */
  TCB_ENOMEM = 4,      /* device allocation failure */
  TCB_EUNSUPPORTED = 5 /* shape outside what the device path implements */
} tcb_status;

#define TCB_MAX_DIMS 6

/* ---- context, memory, streams ------------------------------------------- */
/* One context per device per process; selects `device` for the calling
 * thread. No reference counterpart (the reference is host-only). */
int tcb_init(int device);
int tcb_finalize(void);
int tcb_device_count(int* count);
/* The device the calling thread's tcb_* calls use (-1 before tcb_init). */
int tcb_current_device(int* device);
const char* tcb_last_error(void);
/* Run subsequent work of this thread on a caller-owned cudaStream_t (passed as
 * void*); NULL restores the context's own stream. */
int tcb_set_stream(void* stream);
int tcb_sync(void);

int tcb_alloc(void** dptr, int64_t bytes);
int tcb_free(void* dptr);
int tcb_memset0(void* dptr, int64_t bytes);
int tcb_h2d(void* dst, const void* src, int64_t bytes);
int tcb_d2h(void* dst, const void* src, int64_t bytes);
int tcb_d2d(void* dst, const void* src, int64_t bytes);
/* Pin / unpin caller host memory so H2D/D2H run at DMA speed
 * (reference operands live in std::vector<double>, include/tc/tensor.hpp:58). */
int tcb_host_register(void* ptr, int64_t bytes);
int tcb_host_unregister(void* ptr);
/* Page-locked host allocation (cudaHostAlloc, portable across devices). */
int tcb_host_alloc(void** ptr, int64_t bytes);
int tcb_host_free(void* ptr);

/* Extra streams and events for overlapping copies with compute (the
 * prepared contraction's streamed host-to-host path). Handles are
 * cudaStream_t / cudaEvent_t passed as void*. */
int tcb_stream_create(void** stream);
int tcb_stream_destroy(void* stream);
int tcb_event_create(void** event);
int tcb_event_destroy(void* event);
int tcb_event_record(void* event, void* stream);
int tcb_stream_wait_event(void* stream, void* event);
int tcb_stream_sync(void* stream);
/* Host waits for the last record of `event`. */
int tcb_event_sync(void* event);
/* Current stream of this thread (own or caller-set), as void*. Work the
 * caller enqueues on it is ordered like any stream work (asking for the
 * stream turns off the programmatic overlap of the next GEMM with the
 * previous one). */
void* tcb_current_stream(void);
/* Asynchronous copy in any direction on `stream` (NULL: current stream). */
int tcb_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);
/* Asynchronous strided copy: `height` rows of `width` bytes, row r from
 * src + r*spitch to dst + r*dpitch (pitches in bytes; NULL stream: current).
 * Moves a slab of a middle mode of a column-major tensor in one call (the
 * 2-D H2D of SURVEY §8e; cudaMemcpy2DAsync underneath). */
int tcb_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch,
                       int64_t width, int64_t height, void* stream);
/* Synchronous forms of tcb_memcpy2d_async (host -> device, device -> host). */
int tcb_h2d_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
               int64_t height);
int tcb_d2h_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width,
               int64_t height);
/* *pinned = 1 when `ptr` is page-locked host memory (registered or allocated). */
int tcb_host_is_pinned(const void* ptr, int* pinned);

/* ---- the general device recipe ------------------------------------------
 * C[b; m, n] = alpha * sum_k A[b; m, k] * B[b; k, n] + beta * C[b; m, n]
 *   A(m,k) at A + a_off(b) + m*a_sm + k*a_sk
 *   B(k,n) at B + b_off(b) + k*b_sk + n*b_sn
 *   C(m,n) at C + c_off(b) + row(m) + col(n), where m and n are themselves
 *   composite indices (first sub-index fastest): row(m) = sum_i m_i*c_row_str[i]
 * and batch index b decomposes over bat_ext (first fastest) with per-operand
 * strides (0 where a batch label does not address that operand).
 * This replaces the whole loop-over-kernel nest of tc::execute
 * (src/executor.cpp:119-177 + :274-281) for one contraction: one launch. */
typedef struct tcb_gemm_desc {
  int64_t m, n, k;
  int64_t a_sm, a_sk;
  int64_t b_sk, b_sn;
  int32_t c_nrow, c_ncol;
  int64_t c_row_ext[TCB_MAX_DIMS], c_row_str[TCB_MAX_DIMS];
  int64_t c_col_ext[TCB_MAX_DIMS], c_col_str[TCB_MAX_DIMS];
  int32_t nbatch;
  int64_t bat_ext[TCB_MAX_DIMS];
  int64_t bat_sa[TCB_MAX_DIMS], bat_sb[TCB_MAX_DIMS], bat_sc[TCB_MAX_DIMS];
  double alpha, beta;
  /* Optional operand index groups (all 0: the single strides a_sm, a_sk,
   * b_sk, b_sn above). With g_m, g_n, g_k > 0, m, n and k are composite
   * indices over that many sub-indices (first fastest) of extents m_ext,
   * n_ext, k_ext (products m, n, k), and the operands are read in place:
   *   A(m,k) at A + a_off(b) + sum_i m_i*a_m_str[i] + sum_j k_j*a_k_str[j]
   *   B(k,n) at B + b_off(b) + sum_j k_j*b_k_str[j] + sum_i n_i*b_n_str[i].
   * This removes the operand permutation of COPY+GEMM (class 3 of the
   * paper's taxonomy) where the groups fit the operand tensor maps; see
   * tcb_gemm_check. */
  int32_t g_m, g_n, g_k;
  int64_t m_ext[TCB_MAX_DIMS], a_m_str[TCB_MAX_DIMS];
  int64_t n_ext[TCB_MAX_DIMS], b_n_str[TCB_MAX_DIMS];
  int64_t k_ext[TCB_MAX_DIMS], a_k_str[TCB_MAX_DIMS], b_k_str[TCB_MAX_DIMS];
} tcb_gemm_desc;

/* Execution report for the last tcb_gemm on this thread. */
typedef struct tcb_gemm_info {
  int32_t path;        /* 0 DMMA GEMM via TMA, 1 DMMA GEMM via cp.async, 2 GEMV, 3 DOT */
  int32_t splits;      /* split-K factor */
  int64_t units;       /* work units (tiles x splits) */
  int32_t grid;        /* CTAs launched */
  int32_t launches;    /* kernel launches issued */
} tcb_gemm_info;

int tcb_gemm(const tcb_gemm_desc* d, const double* A, const double* B, double* C);
/* tcb_gemm whose operand reads wait, on the device, until the 64-bit word at
 * `gate` (device memory) is >= value — set from another stream with
 * tcb_stream_write_value after that stream's uploads. The calling stream sees
 * no host-visible wait, so back-to-back GEMMs keep programmatic dependent
 * launch. TCB_EUNSUPPORTED where the device lacks 64-bit stream memory
 * operations. */
int tcb_gemm_gated(const tcb_gemm_desc* d, const double* A, const double* B, double* C,
                   const uint64_t* gate, uint64_t value);
/* Stream-ordered write of `value` to device word `addr` once the stream's
 * earlier work (and its memory writes) completed (cuStreamWriteValue64). */
int tcb_stream_write_value(void* stream, uint64_t* addr, uint64_t value);
int tcb_last_gemm_info(tcb_gemm_info* info);
/* TCB_OK when tcb_gemm can execute `d` for 16-byte aligned operands (only
 * descriptors with index groups can be refused: the groups must map onto the
 * tensor-map boxes of the DMMA kernel); TCB_EUNSUPPORTED with the reason
 * otherwise. Needs an initialised device (the encoder is a driver call). */
int tcb_gemm_check(const tcb_gemm_desc* d);

/* BLAS-semantics GEMM on device buffers: C <- alpha*op(A)*op(B) + beta*C.
 * Replaces KernelBackend::gemm (include/tc/kernels.hpp:20-23,
 * src/kernels_reference.cpp:33-79); argument errors carry the reference's
 * messages ("gemm: lda below row count", kernels_reference.cpp:12-24). */
int tcb_dgemm(int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, double alpha,
              const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
              double* C, int64_t ldc);

/* Strided-batched GEMM: one launch for `batch` independent products, replacing
 * the executor's free-label loop of gemm calls (src/executor.cpp:119-177). */
int tcb_dgemm_strided_batched(int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                              double alpha, const double* A, int64_t lda, int64_t stride_a,
                              const double* B, int64_t ldb, int64_t stride_b, double beta,
                              double* C, int64_t ldc, int64_t stride_c, int64_t batch);

/* y <- alpha*op(A)*x + beta*y  (KernelBackend::gemv, include/tc/kernels.hpp:26-29). */
int tcb_dgemv(int trans, int64_t m, int64_t n, double alpha, const double* A, int64_t lda,
              const double* x, int64_t incx, double beta, double* y, int64_t incy);
/* A <- alpha*x*y^T + A  (KernelBackend::ger, include/tc/kernels.hpp:32-34). */
int tcb_dger(int64_t m, int64_t n, double alpha, const double* x, int64_t incx, const double* y,
             int64_t incy, double* A, int64_t lda);
/* *result_host <- x . y  (KernelBackend::dot, include/tc/kernels.hpp:37-38). */
int tcb_ddot(int64_t k, const double* x, int64_t incx, const double* y, int64_t incy,
             double* result_host);

/* ---- permutation (COPY of COPY+GEMM) -------------------------------------
 * dst[i_0 + e_0*(i_1 + e_1*(...))] = src[sum_j i_j * src_str[j]]: dst is dense
 * in the given dimension order (first fastest). Replaces the executor's
 * per-slice packing copy (materialize, src/executor.cpp:41-59) with one
 * coalesced launch over the whole operand. */
/* The reference's brute-force oracle (tc::contract_naive, src/oracle.cpp:32-94)
 * on device buffers: O[free] = sum over the contracted labels (LEFT-mode
 * order, first fastest) of L*R, free labels in OUTPUT order (first fastest),
 * products and sums rounded separately (no FMA) — bit-identical to the
 * reference built with its own flags. Per label: extent and element strides
 * into L, R, O (0 where the label does not address a tensor). A verification
 * path behind tc/oracle.hpp; execute() never uses it. */
int tcb_contract_naive(int nfree, const int64_t* fext, const int64_t* fls, const int64_t* frs,
                       const int64_t* fos, int ncon, const int64_t* cext, const int64_t* cls,
                       const int64_t* crs, const double* L, const double* R, double* O);

int tcb_permute(int rank, const int64_t* ext, const int64_t* src_str, const double* src,
                double* dst);

/* ---- multi-GPU exchange (NCCL over NVLink / NVSwitch) ---------------------
 * One process per GPU. The K-split partition contracts a
 * slab of a contracted label on every rank into a full partial C, then one
 * reduce-scatter leaves rank r with the summed block r of C's outermost label.
 * NCCL is loaded at run time (libnccl.so.2); without it these return
 * TCB_ENCCL. Collectives run on the thread's current stream. */
#define TCB_COMM_ID_BYTES 128
int tcb_comm_version(int* version);
/* On one rank; ship the TCB_COMM_ID_BYTES bytes to the others. */
int tcb_comm_unique_id(void* id);
/* Collective over the nranks processes (one GPU each, the thread's device). */
int tcb_comm_init(int nranks, int rank, const void* id, void** comm);
int tcb_comm_destroy(void* comm);
/* recv[0..recv_count) = sum over ranks of send[rank*recv_count + i] (fp64). */
int tcb_reduce_scatter(const double* send, double* recv, int64_t recv_count, void* comm);
/* recv[0..count) = sum over ranks of send[0..count) (fp64). */
int tcb_allreduce(const double* send, double* recv, int64_t count, void* comm);

/* ---- peer-memory K-split exchange (fused with the contraction) ------------
 * The same K-split without a separate collective: every rank's GEMM epilogue
 * writes block o of its partial C straight into rank o's receive buffer over
 * NVLink / NVSwitch (tc::PreparedContraction::run_scattered, tcf_run_scattered
 * in tcf.h), then each owner sums its `world` received slots. Replaces the
 * tcb_reduce_scatter step above for the K-split; no reference
 * counterpart (the reference is single-process CPU code).
 *   tcb_peer_alloc: exportable device memory (size a multiple of
 *     tcb_peer_granularity), zero-filled, mapped locally; *fd is a POSIX file
 *     descriptor to ship to the other ranks (SCM_RIGHTS), closed by the caller;
 *   tcb_peer_window: maps n ranks' allocations (all of size `stride`, rank i's
 *     descriptor fds[i]) back to back at *window + i*stride, readable and
 *     writable from this device; the caller closes the descriptors;
 *   tcb_peer_free: unmaps and releases an allocation or a window;
 *   tcb_peer_signal: after everything already on the stream, stores `epoch`
 *     (release, system scope) into the uint64 flag [rank] at window + o*stride
 *     + flag_off for every owner o < world;
 *   tcb_peer_reduce: waits (acquire) until flags[0..world) >= epoch, then
 *     out[i] = sum over s = 0..world-1 in order of slots[s*slot_stride + i]. */
int tcb_peer_granularity(int64_t* bytes);
int tcb_peer_alloc(int64_t bytes, void** dptr, int* fd);
int tcb_peer_window(int n, const int* fds, int64_t stride, void** window);
int tcb_peer_free(void* ptr);
int tcb_peer_signal(void* window, int64_t stride, int64_t flag_off, int rank, int world,
                    uint64_t epoch);
int tcb_peer_reduce(const double* slots, int world, int64_t count, int64_t slot_stride,
                    double* out, const uint64_t* flags, uint64_t epoch);

/* ---- timing -------------------------------------------------------------- */
/* Device-side timing on this thread's stream: tcb_timer_start/stop bracket
 * work; elapsed in milliseconds between the two events. */
int tcb_timer_start(void);
int tcb_timer_stop(float* ms);
/* Milliseconds between two recorded timing events (tcb_event_create_timed;
 * tcb_event_create makes ordering-only events); waits for `stop`. */
int tcb_event_create_timed(void** event);
int tcb_event_elapsed(void* start, void* stop, float* ms);

/* Measured fp64 tensor-pipe (DMMA) peak of the current device in TFLOP/s —
 * the roofline denominator bench.py reports against. */
int tcb_fp64_peak(double* tflops);

/* Count of kernels this library launched on this thread since the last reset
 * (evidence for bench.py's gpu_launches). */
int64_t tcb_launch_count(void);
void tcb_reset_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* TCB_H_ */

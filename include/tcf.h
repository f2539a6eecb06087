/*
 * tcf.h — plan-level C-ABI of the engine (libtc_b200.so): the reference's
 * parse -> validate -> plan -> execute path (tools/tcontract.cpp:114-153,
 * src/executor.cpp:287-369) as flat C calls, for ctypes/cgo/JNI callers and
 * for the repo's own tests and bench. Strings are NUL-terminated ASCII;
 * extents are given as "label=N,label=N,...". Status codes: 0 ok,
 * 1 invalid argument / runtime error, 2 parse error, 3 resource cap,
 * 4 buffer too small (the same codes as the reference CLI's exit statuses,
 * tools/tcontract.cpp:5-6). Error text is written to `err`.
 */
#ifndef TCF_H_
#define TCF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Deterministic analysis report (classification, slicing catalogue, auto and
 * forced plans, re-layout advice, device recipe) — the text the parity tests
 * diff against the reference. Operands are bound like the reference CLI
 * (tools/tcontract.cpp:38-51). */
int tcf_report(const char* expr, int positional, const char* extents, char* buf, int64_t cap);

/* tc::execute with the b200 backend on operands seeded like the reference
 * CLI (left: seed, right: seed+1; tools/tcontract.cpp:118-119).
 * policy: 0 auto, 1 force kernel (KernelKind index), 2 force slicing ("0 1 0").
 * stats[4] = kernel_calls, packed_bytes, staged_bytes, flops. */
int tcf_execute(const char* expr, int positional, const char* extents, uint64_t seed,
                int workers, int policy, int kernel, const char* s_left, const char* s_right,
                double* out, int64_t out_cap, int64_t* stats, double* seconds, char* err,
                int64_t errcap);

/* tc::execute (include/tc/executor.hpp:28-32 of the reference) on CALLER
 * host buffers: parse -> validate -> plan -> execute with the b200 backend.
 * `left`/`right` hold the operands in generalized column-major order of the
 * expression's operand shapes, `out` (out_cap doubles) receives the whole
 * result. Page-locked buffers (tcb_host_register / tcb_host_alloc) take the
 * streamed path (H2D, DMMA and D2H overlapped); pageable buffers go through
 * pinned staging. policy/kernel/s_left/s_right/stats/seconds as tcf_execute.
 * This is the drop-in call bench.py's e2e number is measured through. */
int tcf_execute_host(const char* expr, int positional, const char* extents, const double* left,
                     const double* right, double* out, int64_t out_cap, int workers, int policy,
                     int kernel, const char* s_left, const char* s_right, int64_t* stats,
                     double* seconds, char* err, int64_t errcap);

/* tc::contract_naive (reference include/tc/oracle.hpp:21-23) on operands
 * seeded like tcf_execute: the brute-force sum on the device, bit-identical
 * to the reference's oracle. *macs = multiply-adds; status 3 above work_cap. */
int tcf_contract_naive(const char* expr, int positional, const char* extents, uint64_t seed,
                       int64_t work_cap, double* out, int64_t out_cap, int64_t* macs, char* err,
                       int64_t errcap);

/* The device recipe (lowering) of a contraction, without touching a device:
 * "L1|L2|L3 gemm m=.. n=.. k=.. a(sm,sk) b(sk,sn) batch=[..] permutes=N", or
 * "L4 gemm m=.. n=.. k=.. m[ext:str,..] n[..] k[ext:str_a/str_b,..] ..." for
 * in-place index groups (TC_INDEX_GROUPS=0 in the environment disables L4). */
int tcf_lower(const char* expr, int positional, const char* extents, char* buf, int64_t cap);

/* Fill `out` with Tensor::seeded_random's stream (src/tensor.cpp:54-62). */
int tcf_seeded(int64_t n, uint64_t seed, double* out);

/* The block of Tensor::seeded_random's stream (extents ext[0..rank), first
 * mode fastest) where mode `mode` lies in [lo, hi), dense in the same mode
 * order: a rank's slab of a seeded operand without materialising the whole
 * tensor (the stream is still drawn up to the block's end). */
int tcf_seeded_block(uint64_t seed, int rank, const int64_t* ext, int mode, int64_t lo,
                     int64_t hi, double* out);

/* Prepared contraction bound to device buffers (tc::PreparedContraction). */
int tcf_prepare(const char* expr, int positional, const char* extents, int device,
                void** handle, char* err, int64_t errcap);
int tcf_upload(void* handle, const double* left, const double* right);
int tcf_run(void* handle);
/* The two halves of tcf_run (for timing the kernels separately). */
int tcf_run_permutes(void* handle);
int tcf_run_contraction(void* handle);
/* Permutations + contraction with the output's outermost label split into
 * `parts` blocks, block p written at base + p * part_stride (doubles): the
 * fused K-split exchange when `base` lies in a tcb_peer_window (tcb.h).
 * tc::PreparedContraction::run_scattered. */
int tcf_run_scattered(void* handle, double* base, int parts, int64_t part_stride);
int tcf_download(void* handle, double* out);
/* Host-to-host evaluation with transfers overlapped with compute
 * (tc::PreparedContraction::run_streamed); host buffers must be page-locked
 * (tcb_host_register) for overlap. *slabs_used receives the slab count. */
int tcf_run_streamed(void* handle, const double* left, const double* right, double* out,
                     int slabs, int* slabs_used);
/* As tcf_run_streamed, but returns once the work is enqueued: a following
 * call overlaps its uploads with this one's download drain (a stream of
 * host-to-host contractions). tcf_sync (or any other call on the handle)
 * completes it; `out` is valid after that. */
int tcf_run_streamed_async(void* handle, const double* left, const double* right, double* out,
                           int slabs, int* slabs_used);
int tcf_sync(void* handle);
/* info[12]: left, right, output elements; launches of the last run;
 * permuted bytes; m, n, k, batch; flops; number of permutes; device path
 * (tcb_gemm_info.path of the last run). summary: recipe text. */
int tcf_info(void* handle, int64_t* info, char* summary, int64_t cap);
int tcf_device_ptrs(void* handle, void** left, void** right, void** out);
int tcf_release(void* handle);
const char* tcf_last_error(void);

/* ---- TENSOR v1 text (tc::write_tensor / tc::read_tensor; reference
 * include/tc/tensor_io.hpp:9-22) ----------------------------------------- */
/* Text of Tensor::seeded_random(ext[0..rank), var ("+-" chars), seed, name). */
int tcf_tensor_text(const int64_t* ext, int rank, const char* var, uint64_t seed,
                    const char* name, char* buf, int64_t cap);
/* Parse text: *n = element count, values into out (cap elements); the
 * reference's messages on malformed input ("not a TENSOR v1 file", ...). */
int tcf_read_tensor_text(const char* text, double* out, int64_t cap, int64_t* n, char* err,
                         int64_t errcap);

/* ---- metric tensors (tc::invert_metric / lower_index / raise_index;
 * reference include/tc/metric.hpp:17-32) — a caller of the contraction path -
 * g: n x n column-major, symmetric (down, down). Status 1 with the
 * reference's messages ("metric is not symmetric", "metric is singular", ...). */
int tcf_invert_metric(int64_t n, const double* g, double* g_inv, char* err, int64_t errcap);
/* t (extents ext[0..rank), variances var as "+-" chars) with mode `mode`
 * contracted against g (raise == 0: lower_index, the mode must be '+') or
 * against g's inverse (raise != 0: raise_index, the mode must be '-'), through
 * validate -> plan -> execute on the b200 backend; out has t's shape. */
int tcf_metric_apply(const int64_t* ext, int rank, const char* var, const double* t, int mode,
                     int64_t n, const double* g, int raise, double* out, int64_t out_cap,
                     char* err, int64_t errcap);

/* ---- benchmark sweep (tc::run_bench + tc::write_bench_csv; reference
 * include/tc/bench.hpp:13-51) ----------------------------------------------
 * sizes "150,200"; kernels "GEMM,COPY+GEMM,..."; custom_extents "a=3,b=4".
 * CSV into csv; *verified = 1 when every sampled line matched. */
int tcf_bench_csv(const char* experiment, const char* sizes, const char* kernels,
                  const char* backend, int repetitions, uint64_t seed, int verify, int workers,
                  const char* custom_expr, const char* custom_extents, char* csv, int64_t cap,
                  int* verified);

#ifdef __cplusplus
}
#endif

#endif /* TCF_H_ */

// tcb_contract_naive: the reference's brute-force contraction
// (tc::contract_naive, src/oracle.cpp:32-94) as a device kernel.
//
// One thread per output element. Free labels are decoded from the thread's
// flat index in OUTPUT order, first fastest (oracle.cpp:44-46, :84-90); each
// thread sums left*right over the contracted labels in LEFT-MODE order,
// first fastest (oracle.cpp:47, :64-81), sequentially from 0.0. The products
// and sums are rounded separately (__dmul_rn / __dadd_rn, never fused into an
// FMA) — the arithmetic of the reference built with its own flags (-O3, no
// -march: SSE2 mulsd + addsd) — so the result is bit-identical to the
// reference's oracle. It is a verification path (the tc/oracle.hpp API), not
// a contraction kernel: the engine's execute() never calls it.
#include "tcb_internal.cuh"

namespace tcb {
namespace {

constexpr int kMaxLabels = 16;

struct NaiveArgs {
  int nfree, ncon;
  int64_t nout;
  int64_t fext[kMaxLabels], fls[kMaxLabels], frs[kMaxLabels], fos[kMaxLabels];
  int64_t cext[kMaxLabels], cls[kMaxLabels], crs[kMaxLabels];
};

__global__ void __launch_bounds__(128) naive_kernel(const NaiveArgs a, const double* __restrict__ L,
                                                    const double* __restrict__ R,
                                                    double* __restrict__ O) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= a.nout) return;
  int64_t rem = t, lb = 0, rb = 0, ob = 0;
  for (int i = 0; i < a.nfree; ++i) {
    const int64_t c = rem % a.fext[i];
    rem /= a.fext[i];
    lb += c * a.fls[i];
    rb += c * a.frs[i];
    ob += c * a.fos[i];
  }
  int64_t cc[kMaxLabels];
  for (int i = 0; i < a.ncon; ++i) cc[i] = 0;
  double acc = 0.0;
  int64_t lo = lb, ro = rb;
  for (;;) {
    acc = __dadd_rn(acc, __dmul_rn(L[lo], R[ro]));
    int k = 0;
    for (; k < a.ncon; ++k) {  // odometer, first contracted label fastest
      lo += a.cls[k];
      ro += a.crs[k];
      if (++cc[k] < a.cext[k]) break;
      lo -= a.cext[k] * a.cls[k];
      ro -= a.cext[k] * a.crs[k];
      cc[k] = 0;
    }
    if (k == a.ncon) break;
  }
  O[ob] = acc;
}

}  // namespace
}  // namespace tcb

using namespace tcb;

extern "C" int tcb_contract_naive(int nfree, const int64_t* fext, const int64_t* fls,
                                  const int64_t* frs, const int64_t* fos, int ncon,
                                  const int64_t* cext, const int64_t* cls, const int64_t* crs,
                                  const double* L, const double* R, double* O) {
  {
    const int rc = ensure_init();
    if (rc != TCB_OK) return rc;
  }
  if (nfree < 0 || ncon < 0 || nfree > kMaxLabels || ncon > kMaxLabels)
    return set_error(TCB_EUNSUPPORTED, "contract_naive: more than 16 free or contracted labels");
  if ((nfree && (!fext || !fls || !frs || !fos)) || (ncon && (!cext || !cls || !crs)) || !L ||
      !R || !O)
    return set_error(TCB_EINVAL, "contract_naive: null argument");
  NaiveArgs a{};
  a.nfree = nfree;
  a.ncon = ncon;
  a.nout = 1;
  for (int i = 0; i < nfree; ++i) {
    if (fext[i] <= 0) return set_error(TCB_EINVAL, "contract_naive: extent must be positive");
    a.fext[i] = fext[i];
    a.fls[i] = fls[i];
    a.frs[i] = frs[i];
    a.fos[i] = fos[i];
    a.nout *= fext[i];
  }
  for (int i = 0; i < ncon; ++i) {
    if (cext[i] <= 0) return set_error(TCB_EINVAL, "contract_naive: extent must be positive");
    a.cext[i] = cext[i];
    a.cls[i] = cls[i];
    a.crs[i] = crs[i];
  }
  ThreadState& st = state();
  note_stream_op();
  const int64_t blocks = (a.nout + 127) / 128;
  naive_kernel<<<static_cast<unsigned>(blocks), 128, 0, st.stream>>>(a, L, R, O);
  TCB_LAUNCHED();
  return TCB_OK;
}

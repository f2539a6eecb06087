/* TEST INFRASTRUCTURE ONLY — the CPU oracle of this repo. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it; the
 * product (paper_1307_2100_b200) never links or calls it.
 *
 * A plain-C restatement of the reference's arithmetic on the hot path, each
 * function citing the reference file:line it follows (paths relative to
 * /root/reference/proj). Pinned against the compiled reference
 * (oracle/_ref/libtcref.so) by tests/test_oracle_pin.py and against the
 * committed fixtures in tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* ---- seeded generator: src/tensor.cpp:54-62 -------------------------------
 * std::mt19937_64(seed) feeding std::uniform_real_distribution<double>(-1, 1),
 * one draw per element in storage order. libstdc++ maps one 64-bit draw x to
 * generate_canonical<double,53> = (double)x / 2^64 (clamped below 1), then
 * a + u * (b - a). */
typedef struct {
  uint64_t mt[312];
  int idx;
} tco_mt64;

static void mt64_seed(tco_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(tco_mt64* g) {
  if (g->idx >= 312) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

void tco_seeded_random(int64_t n, uint64_t seed, double* out) {
  static tco_mt64 g; /* 2.5 KB state; callers are single-threaded tests */
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i) {
    double u = (double)mt64_next(&g) / 18446744073709551616.0;
    if (u >= 1.0) u = nextafter(1.0, 0.0);
    out[i] = u * 2.0 + -1.0;
  }
}

/* ---- brute-force contraction: src/oracle.cpp:32-94 ------------------------
 * For every output coordinate (free labels in OUTPUT order, first fastest —
 * oracle.cpp:44-46, :84-90) sum left*right over the contracted labels in
 * LEFT-MODE order, first fastest (oracle.cpp:47, :64-81), sequentially in
 * fp64 starting from 0.0. Labels are described numerically by the caller:
 * extent and the per-operand strides (0 where a label does not address that
 * operand — oracle.cpp:11-30). Returns the multiply-add count, or -1 when the
 * work exceeds work_cap (oracle.cpp:35-39). */
int64_t tco_contract_naive(int nfree, const int64_t* fext, const int64_t* fls,
                           const int64_t* frs, const int64_t* fos, int ncon,
                           const int64_t* cext, const int64_t* cls, const int64_t* crs,
                           const double* L, const double* R, double* O, int64_t work_cap) {
  int64_t work = 1;
  for (int i = 0; i < nfree; ++i) work *= fext[i];
  for (int i = 0; i < ncon; ++i) work *= cext[i];
  if (work > work_cap) return -1;
  int64_t fc[16], cc[16], macs = 0;
  memset(fc, 0, sizeof fc);
  for (;;) {
    int64_t lb = 0, rb = 0, ob = 0;
    for (int i = 0; i < nfree; ++i) {
      lb += fc[i] * fls[i];
      rb += fc[i] * frs[i];
      ob += fc[i] * fos[i];
    }
    double acc = 0.0;
    memset(cc, 0, sizeof cc);
    for (;;) {
      int64_t lo = lb, ro = rb;
      for (int i = 0; i < ncon; ++i) {
        lo += cc[i] * cls[i];
        ro += cc[i] * crs[i];
      }
      acc += L[lo] * R[ro];
      ++macs;
      int k = 0;
      for (; k < ncon; ++k) {
        if (++cc[k] < cext[k]) break;
        cc[k] = 0;
      }
      if (k == ncon) break;
    }
    O[ob] = acc;
    int k = 0;
    for (; k < nfree; ++k) {
      if (++fc[k] < fext[k]) break;
      fc[k] = 0;
    }
    if (k == nfree) break;
  }
  return macs;
}

/* ---- long-double GEMM check kernel: tests/test_kernels.cpp:16-28 ----------
 * C <- alpha*op(A)*op(B) + beta*C with direct loops and long-double sums; the
 * reference's own independent check for its gemm (tolerance 8e-16*2k*2,
 * tests/test_kernels.cpp:217-234). */
void tco_gemm_check(int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha,
                    const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                    double* c, int64_t ldc) {
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < m; ++i) {
      long double acc = 0;
      for (int64_t p = 0; p < k; ++p) {
        const double av = ta ? a[p + i * lda] : a[i + p * lda];
        const double bv = tb ? b[j + p * ldb] : b[p + j * ldb];
        acc += (long double)av * bv;
      }
      c[i + j * ldc] = (double)(alpha * acc + beta * c[i + j * ldc]);
    }
}

/* ---- comparators: src/executor.cpp:371-394 --------------------------------
 * tensor_hash: FNV-1a over the little-endian bytes of every element.
 * max_rel_error: max|a-b| / max(1, max|b|). rel_frobenius (BASELINE's
 * criterion, not in the reference): ||a-b||_F / ||b||_F. */
uint64_t tco_tensor_hash(int64_t n, const double* d) {
  uint64_t h = 1469598103934665603ULL;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t bits;
    memcpy(&bits, &d[i], 8);
    for (int b = 0; b < 8; ++b) {
      h ^= (bits >> (8 * b)) & 0xff;
      h *= 1099511628211ULL;
    }
  }
  return h;
}

double tco_max_rel_error(int64_t n, const double* a, const double* b) {
  double scale = 1.0, err = 0.0;
  for (int64_t i = 0; i < n; ++i) scale = fmax(scale, fabs(b[i]));
  for (int64_t i = 0; i < n; ++i) err = fmax(err, fabs(a[i] - b[i]));
  return err / scale;
}

double tco_rel_frobenius(int64_t n, const double* a, const double* b) {
  long double num = 0, den = 0;
  for (int64_t i = 0; i < n; ++i) {
    const long double d = (long double)a[i] - b[i];
    num += d * d;
    den += (long double)b[i] * b[i];
  }
  if (den == 0) return num == 0 ? 0.0 : INFINITY;
  return (double)sqrtl(num / den);
}

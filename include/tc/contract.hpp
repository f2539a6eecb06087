// tc:: — the reference's contraction API (/root/reference/proj/include/tc/*.hpp),
// re-declared for the B200 engine so existing callers compile unchanged.
// The per-topic headers tc/tensor.hpp, tc/expr.hpp, tc/planner.hpp,
// tc/kernels.hpp, tc/executor.hpp, tc/tensor_io.hpp and tc/bench.hpp include
// this file.
//
// Everything here is host C++ (no CUDA types). Arithmetic goes to the device
// through the C-ABI in tcb.h; see DESIGN.md for the lowering.
#pragma once

#include <cstdint>
#include <iosfwd>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tc {

// ============================================================ L0: storage
// reference: include/tc/tensor.hpp:10-108

enum class Variance : std::uint8_t { Up, Down };
char variance_char(Variance v);

struct ValidatedContraction;
struct ExecutionPlan;
struct ExecutionStats;
class KernelBackend;

/// Storage allocator of Tensor: large blocks are mapped directly with
/// transparent huge pages requested (a 128 MB operand faults in 64 times, not
/// 32768), and elements are default-initialised, so storage that is about to
/// be overwritten (a downloaded result) is not zero-filled first. Tensor's
/// own constructors still zero it, as the reference's do.
template <typename T>
struct TensorAllocator {
  using value_type = T;
  TensorAllocator() = default;
  template <typename U>
  TensorAllocator(const TensorAllocator<U>&) {}
  T* allocate(std::size_t n);
  void deallocate(T* p, std::size_t n);
  template <typename U, typename... Args>
  void construct(U* p, Args&&... args) {
    if constexpr (sizeof...(Args) == 0) ::new (static_cast<void*>(p)) U;  // default-init
    else ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
  template <typename U>
  bool operator==(const TensorAllocator<U>&) const { return true; }
  template <typename U>
  bool operator!=(const TensorAllocator<U>&) const { return false; }
};
void* tensor_storage_allocate(std::size_t bytes);
void tensor_storage_free(void* p, std::size_t bytes);
/// Page-locks a large Tensor storage block (the base of a block of `bytes`
/// from tensor_storage_allocate) for the rest of its life; false for small
/// blocks or when registration fails (transfers then take the pageable path).
bool tensor_storage_pin(const void* p, std::size_t bytes);
template <typename T>
T* TensorAllocator<T>::allocate(std::size_t n) {
  return static_cast<T*>(tensor_storage_allocate(n * sizeof(T)));
}
template <typename T>
void TensorAllocator<T>::deallocate(T* p, std::size_t n) {
  tensor_storage_free(p, n * sizeof(T));
}

/// Dense fp64 tensor, generalized column-major: stride(mode k) = prod of the
/// extents of modes 0..k-1. Rank 0 holds one scalar.
class Tensor {
 public:
  Tensor() = default;
  Tensor(std::vector<std::int64_t> extents, std::vector<Variance> variance,
         std::string name = "t");

  static Tensor zeros(std::vector<std::int64_t> extents, std::vector<Variance> variance,
                      std::string name = "t");
  static Tensor sequential(std::vector<std::int64_t> extents, std::vector<Variance> variance,
                           std::string name = "t");
  /// Uniform [-1, 1] from std::mt19937_64(seed), storage order — the same
  /// stream as the reference (src/tensor.cpp:54-62), bit for bit.
  static Tensor seeded_random(std::vector<std::int64_t> extents, std::vector<Variance> variance,
                              std::uint64_t seed, std::string name = "t");
  static Tensor from_values(std::vector<std::int64_t> extents, std::vector<Variance> variance,
                            std::vector<double> values, std::string name = "t");

  int rank() const { return static_cast<int>(ext_.size()); }
  std::int64_t size() const { return static_cast<std::int64_t>(buf_.size()); }
  const std::vector<std::int64_t>& extents() const { return ext_; }
  std::int64_t extent(int mode) const;
  const std::vector<Variance>& variance() const { return var_; }
  Variance variance(int mode) const;
  const std::string& name() const { return name_; }
  void set_name(std::string name) { name_ = std::move(name); }

  double* data() { return buf_.data(); }
  const double* data() const { return buf_.data(); }

  double at(const std::vector<std::int64_t>& coords) const;
  double& at(const std::vector<std::int64_t>& coords);
  std::int64_t offset_of(const std::vector<std::int64_t>& coords) const;

 private:
  std::vector<std::int64_t> ext_, str_;
  std::vector<Variance> var_;
  std::vector<double, TensorAllocator<double>> buf_;
  std::string name_ = "t";
  friend std::int64_t stride_of(const Tensor& t, int mode);
  // storage left uninitialised, for results that are overwritten whole
  struct Uninit {};
  Tensor(std::vector<std::int64_t> extents, std::vector<Variance> variance, std::string name,
         Uninit);
  friend std::pair<Tensor, ExecutionStats> execute(const ExecutionPlan&,
                                                   const ValidatedContraction&, const Tensor&,
                                                   const Tensor&, const KernelBackend&, int);
};

std::int64_t stride_of(const Tensor& t, int mode);

using SlicingVector = std::vector<std::uint8_t>;  // 1 = mode fixed per slice

struct KeptMode {
  int mode = 0;
  std::int64_t extent = 0;
  std::int64_t stride = 0;
};

struct SliceView {
  const Tensor* parent = nullptr;
  std::int64_t base_offset = 0;
  std::vector<KeptMode> kept;
  int rank() const { return static_cast<int>(kept.size()); }
  std::int64_t offset_of(const std::vector<std::int64_t>& coords) const;
  double at(const std::vector<std::int64_t>& coords) const;
};

SliceView slice_view(const Tensor& t, const SlicingVector& s,
                     const std::vector<std::int64_t>& fixed);

struct PackedMatrix {
  std::int64_t rows = 0, cols = 0, leading_dimension = 0;
  const double* data = nullptr;
  bool copied = false;
  std::int64_t source_offset = 0;
  std::vector<double> storage;
};

PackedMatrix pack_slice(const SliceView& v);

// ============================================================ L1: expressions
// reference: include/tc/expr.hpp:12-91

struct parse_error : std::runtime_error {
  parse_error(const std::string& what, std::size_t position)
      : std::runtime_error(what + " (at position " + std::to_string(position) + ")"),
        position(position) {}
  std::size_t position;
};

struct IndexRef {
  std::string label;
  Variance var = Variance::Up;
  bool operator==(const IndexRef&) const = default;
};

struct TensorExpr {
  std::string name;
  std::vector<IndexRef> indices;
  bool operator==(const TensorExpr&) const = default;
};

struct ContractionSpec {
  TensorExpr output, left, right;
  bool positional = false;
  bool operator==(const ContractionSpec&) const = default;
};

/// `OUT[±i,...] = L[...] * R[...]` (ASCII); see DESIGN.md for the rules.
ContractionSpec parse(const std::string& expr, bool positional = false);
std::string unparse(const ContractionSpec& spec);

struct LabelInfo {
  std::string label;
  std::int64_t extent = 0;
  bool contracted = false;
  int left_mode = -1, right_mode = -1, output_mode = -1;
};

struct ValidatedContraction {
  ContractionSpec spec;
  std::vector<LabelInfo> labels;  // left modes in order, then right-only labels
  std::vector<int> contracted;    // by left mode order
  std::vector<int> left_free;     // by left mode order
  std::vector<int> right_free;    // by right mode order
  int p = 0, delta_left = 0, delta_right = 0;

  int left_rank() const { return static_cast<int>(spec.left.indices.size()); }
  int right_rank() const { return static_cast<int>(spec.right.indices.size()); }
  int output_rank() const { return static_cast<int>(spec.output.indices.size()); }
  const LabelInfo& label_at_left_mode(int mode) const;
  const LabelInfo& label_at_right_mode(int mode) const;
  int label_index(const std::string& label) const;
  std::vector<std::int64_t> output_extents() const;
  std::vector<Variance> output_variance() const;
};

ValidatedContraction validate(const ContractionSpec& spec, const Tensor& left,
                              const Tensor& right);

/// validate() on operand shapes alone (no storage), for callers that hold the
/// data elsewhere (device buffers, the C front). Same checks and messages.
ValidatedContraction validate_shapes(const ContractionSpec& spec,
                                     const std::vector<std::int64_t>& left_extents,
                                     const std::vector<Variance>& left_variance,
                                     const std::vector<std::int64_t>& right_extents,
                                     const std::vector<Variance>& right_variance);

/// Algorithmic flops: 2 * prod(all label extents).
std::int64_t flop_count(const ValidatedContraction& v);

// ============================================================ L2: planner
// reference: include/tc/planner.hpp:12-142

enum class ContractionClass { C1, C2, C31, C32 };
std::string to_string(ContractionClass c);

enum class KernelKind { Gemm, CopyGemm, Gemv, CopyGemv, Ger, Dot, Elementwise };
std::string to_string(KernelKind k);
std::optional<KernelKind> kernel_from_string(const std::string& s);

enum class Fallback { None, F1, F2, F3 };
std::string to_string(Fallback f);

struct RequirementReport {
  bool r1_ok = false, r2_ok = false, r3_ok = false;
  Fallback fallback = Fallback::None;
  KernelKind kernel = KernelKind::Elementwise;
};

struct SlicingOption {
  SlicingVector s_left, s_right;
  RequirementReport report;
  std::int64_t kernel_dims_product = 0;
  bool output_staged = false;
};

struct LoopLabel {
  int label = -1;
  bool contracted = false;
  std::int64_t extent = 0;
};

struct KernelMap {
  int m_label = -1, n_label = -1, k_label = -1, k2_label = -1;
  bool a_is_left = true;
  bool trans_a = false, trans_b = false;
  bool matrix_is_left = true;
};

enum class CopyTarget { Left, Right, OutputStage };

struct ExecutionPlan {
  ContractionClass cls = ContractionClass::C32;
  SlicingVector s_left, s_right, s_output;
  KernelKind kernel = KernelKind::Gemm;
  std::vector<LoopLabel> loop_nest;
  KernelMap kernel_map;
  std::vector<CopyTarget> copies;
  std::int64_t flops = 0;
  std::vector<std::int64_t> label_extents;
};

struct kernel_unreachable_error : std::runtime_error {
  kernel_unreachable_error(KernelKind kernel, const std::string& requirement)
      : std::runtime_error("kernel unreachable: " + requirement + " violated"),
        kernel(kernel),
        requirement(requirement) {}
  explicit kernel_unreachable_error(const std::string& msg)
      : std::runtime_error(msg), kernel(KernelKind::Gemm) {}
  KernelKind kernel;
  std::string requirement;
};

ContractionClass classify(const ValidatedContraction& v);
RequirementReport check_requirements(const ValidatedContraction& v, const SlicingVector& s_left,
                                     const SlicingVector& s_right);
std::vector<SlicingOption> enumerate_slicings(const ValidatedContraction& v);

struct PlanPolicy {
  enum class Mode { Auto, ForceKernel, ForceSlicing };
  Mode mode = Mode::Auto;
  KernelKind kernel = KernelKind::Gemm;
  SlicingVector s_left, s_right;

  static PlanPolicy auto_policy() { return {}; }
  static PlanPolicy force_kernel(KernelKind k) {
    PlanPolicy p;
    p.mode = Mode::ForceKernel;
    p.kernel = k;
    return p;
  }
  static PlanPolicy force_slicing(SlicingVector sl, SlicingVector sr) {
    PlanPolicy p;
    p.mode = Mode::ForceSlicing;
    p.s_left = std::move(sl);
    p.s_right = std::move(sr);
    return p;
  }
};

ExecutionPlan plan(const ValidatedContraction& v,
                   const PlanPolicy& policy = PlanPolicy::auto_policy());
std::string render_plan(const ExecutionPlan& p, const ValidatedContraction& v);
std::optional<std::string> relayout_advice(const ValidatedContraction& v);

// ============================================================ L3: backends
// reference: include/tc/kernels.hpp:12-48

class KernelBackend {
 public:
  virtual ~KernelBackend() = default;
  virtual const std::string& name() const = 0;
  virtual bool supports_transpose() const { return true; }
  virtual void gemm(bool trans_a, bool trans_b, std::int64_t m, std::int64_t n, std::int64_t k,
                    double alpha, const double* a, std::int64_t lda, const double* b,
                    std::int64_t ldb, double beta, double* c, std::int64_t ldc) const = 0;
  virtual void gemv(bool trans, std::int64_t m, std::int64_t n, double alpha, const double* a,
                    std::int64_t lda, const double* x, std::int64_t incx, double beta, double* y,
                    std::int64_t incy) const = 0;
  virtual void ger(std::int64_t m, std::int64_t n, double alpha, const double* x,
                   std::int64_t incx, const double* y, std::int64_t incy, double* a,
                   std::int64_t lda) const = 0;
  virtual double dot(std::int64_t k, const double* x, std::int64_t incx, const double* y,
                     std::int64_t incy) const = 0;
};

/// Options of the B200 backend. `device` selects the GPU this backend drives;
/// `fail_after_launches` >= 0 injects a synthetic device fault after that many
/// successful device operations (fault-propagation tests, cf. the reference's
/// FailingBackend, tests/test_executor.cpp:240-291).
struct B200Options {
  int device = 0;
  int fail_after_launches = -1;
};

/// The B200 device backend. Its BLAS methods take HOST pointers (copy in, one
/// device call, copy out) so the reference's backend contract holds; execute()
/// recognises it and lowers a whole plan to device launches instead.
std::unique_ptr<KernelBackend> make_b200_backend(const B200Options& options = {});

/// "b200" (also "device") -> make_b200_backend(); "b200-sliced" -> the same
/// device BLAS calls driven slice by slice through the plan's loop nest (the
/// reference's execution structure: one device call per slice, operands
/// copied per call), for comparing forced kernels. The reference names
/// "reference" and "external" are CPU backends and are not part of this
/// engine: they throw std::invalid_argument naming the replacement.
std::unique_ptr<KernelBackend> make_backend(const std::string& name);

/// The reference's CPU factories (include/tc/kernels.hpp:41-45), declared so
/// that callers written against the reference compile and link unchanged.
/// This engine has no CPU contraction path: both throw std::invalid_argument
/// naming make_b200_backend(). A caller's own KernelBackend subclass still
/// works with execute() (driven slice by slice, like the reference).
std::unique_ptr<KernelBackend> make_reference_backend();
std::unique_ptr<KernelBackend> make_eigen_backend();

// ============================================================ L4: executor
// reference: include/tc/executor.hpp:14-54

struct ExecutionStats {
  std::int64_t kernel_calls = 0;  // device kernel launches
  std::int64_t packed_bytes = 0;  // bytes written by operand permutations
  std::int64_t staged_bytes = 0;  // output staging bytes (0: strided epilogue)
  std::int64_t flops = 0;         // plan.flops
  double wall_seconds = 0.0;      // host wall time incl. transfers
};

/// Runs the contraction. The plan is checked against the operands (extent
/// drift). With the B200 backend it is lowered to one device recipe
/// (permutations + one GEMM/GEMV/DOT launch) and executed; `workers` does not
/// change the result (bit-identical for any value). With any other
/// KernelBackend the plan's loop nest is walked and the backend called once
/// per slice, free slices spread over `workers` threads — the reference's
/// behaviour (src/executor.cpp:102-369), kept for callers that plug in their
/// own backend (fault injection, instrumentation, a host BLAS).
std::pair<Tensor, ExecutionStats> execute(const ExecutionPlan& plan,
                                          const ValidatedContraction& v, const Tensor& left,
                                          const Tensor& right, const KernelBackend& backend,
                                          int workers = 1);

/// execute() on caller-owned storage (no reference counterpart; the C-ABI's
/// tcf_execute_host): `left`/`right` hold the operands in generalized
/// column-major order of v's operand shapes, `out` receives the whole result
/// (output order of v). With the B200 backend, page-locked buffers
/// (tcb_host_register / tcb_host_alloc) take the streamed path (uploads,
/// contraction and download overlapped); pageable ones go through the
/// staging buffers.
ExecutionStats execute_into(const ExecutionPlan& plan, const ValidatedContraction& v,
                            const double* left, const double* right, double* out,
                            const KernelBackend& backend, int workers = 1);

/// The loop-over-kernel driver behind execute() for non-B200 backends: one
/// backend call per slice of the plan's loop nest (stats accumulated into
/// `stats`). `out` must be zero-filled on entry.
void execute_sliced(const ExecutionPlan& plan, const ValidatedContraction& v, const double* left,
                    const double* right, double* out, const KernelBackend& backend, int workers,
                    ExecutionStats& stats);

struct SlicingRun {
  SlicingVector s_left, s_right;
  KernelKind kernel = KernelKind::Elementwise;
  std::uint64_t result_hash = 0;
  ExecutionStats stats;
  Tensor result;
};

std::vector<SlicingRun> execute_all_slicings(const ValidatedContraction& v, const Tensor& left,
                                             const Tensor& right, const KernelBackend& backend,
                                             std::int64_t work_cap = 1000000000);

std::uint64_t tensor_hash(const Tensor& t);
double max_rel_error(const Tensor& a, const Tensor& b);
/// ||a-b||_F / ||b||_F — the BASELINE parity criterion (not in the reference).
double rel_frobenius_error(const Tensor& a, const Tensor& b);

/// Thrown by execute_all_slicings and contract_naive when the work exceeds
/// the cap (the reference declares it in tc/oracle.hpp:11-13; tc/oracle.hpp
/// here includes this header).
struct resource_limit_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------ oracle API (tc/oracle.hpp)
// reference: include/tc/oracle.hpp:15-25

struct OracleStats {
  std::int64_t multiply_adds = 0;
};

/// Direct nested summation in a fixed lexicographic order: for every output
/// coordinate (free labels in output order), left*right summed over the full
/// range of the contracted labels (left-mode order, first fastest), from 0.
/// Evaluated on the device by tcb_contract_naive with separately rounded
/// products and sums: bit-identical to the reference's src/oracle.cpp:32-94.
/// Refuses jobs above the work cap (resource_limit_error). A verification
/// API (the CLI's --verify in the reference); execute() never uses it.
Tensor contract_naive(const ValidatedContraction& v, const Tensor& left, const Tensor& right,
                      std::int64_t work_cap = 1000000000, OracleStats* stats = nullptr);

// ------------------------------------------------ metric API (tc/metric.hpp)
// reference: include/tc/metric.hpp:9-34 — a caller of the contraction path:
// lower_index / raise_index build an ordinary two-tensor contraction and run
// it through validate -> plan -> execute (on the device with the b200
// backend, slice by slice with a caller's backend). invert_metric: the
// reference inverts with Eigen's FullPivLU, a third-party dependency that is
// not vendored in the reference tree (Eigen 3 >= 3.3, proj/CMakeLists.txt:13);
// csrc/host/metric.cpp restates that published algorithm (LU with complete
// pivoting, rank decided by |pivot| against n * epsilon * |largest pivot|).
// Parity of the inverse is unpinned at the bit level (no Eigen here to run);
// the tests pin it through g * g_inv = 1 and the reference tests' answers.

/// Symmetric nonsingular rank-2 tensor g (down, down) and its inverse
/// (up, up): g lowers an index, g_inv raises one.
struct MetricTensor {
  Tensor g;
  Tensor g_inv;
  std::int64_t dimension = 0;
};

/// Direct inversion. std::invalid_argument for a non-square or non-rank-2
/// input, asymmetry beyond 1e-10 (relative to max(1, max|g|)), a singular
/// matrix, or a 1-norm condition estimate of 1e12 or more.
MetricTensor invert_metric(const Tensor& g);

/// diag(1, r^2, r^2 sin^2(theta)) with its exact diagonal inverse;
/// std::invalid_argument at r <= 0 or sin(theta) == 0.
MetricTensor spherical_metric(double r, double theta);

/// Contracts mode `mode` (which must be Up) of t against g: that mode comes
/// out Down, every other mode and the mode order are unchanged.
Tensor lower_index(const Tensor& t, int mode, const MetricTensor& m,
                   const KernelBackend& backend);

/// The dual: mode `mode` (Down) against g_inv, coming out Up.
Tensor raise_index(const Tensor& t, int mode, const MetricTensor& m,
                   const KernelBackend& backend);

// ============================================================ device recipe
// (new; no reference counterpart) — the lowering of a contraction onto the
// device: optional operand permutations followed by one batched GEMM with
// composite output addressing. Exposed for tests and tools.

struct PermuteStep {
  bool right = false;                 // which operand
  std::vector<std::int64_t> ext;      // destination order (dense, first fastest)
  std::vector<std::int64_t> src_str;  // source strides of those dims
  std::int64_t elements = 0;
};

struct DeviceRecipe {
  std::vector<PermuteStep> permutes;
  // GEMM over (possibly permuted) operands, see tcb_gemm_desc in tcb.h
  std::int64_t m = 1, n = 1, k = 1;
  std::int64_t a_sm = 1, a_sk = 1, b_sk = 1, b_sn = 1;
  std::vector<std::int64_t> row_ext, row_str, col_ext, col_str;
  std::vector<std::int64_t> bat_ext, bat_sa, bat_sb, bat_sc;
  // "L4" only: m, n, k as composites of operand dimensions read in place
  // (sub-index extents first fastest, per-operand strides; tcb_gemm_desc g_*)
  std::vector<std::int64_t> gm_ext, gm_sa, gn_ext, gn_sb, gk_ext, gk_sa, gk_sb;
  // "L1" in place, "L2" batched, "L3" permuted, "L4" in-place index groups
  std::string layout;
  std::string summary() const;
};

/// Lower a validated contraction to one device recipe. `index_groups` allows
/// the L4 form (operands read in place through composite tensor-map boxes)
/// where L3 would otherwise permute an operand. `layout`, when given, is the
/// contraction whose storage the operands and output live in (v a slab of it:
/// same labels, smaller extents): strides come from it, extents from v.
DeviceRecipe lower(const ValidatedContraction& v, bool index_groups = true,
                   const ValidatedContraction* layout = nullptr);

/// A contraction lowered once and bound to device buffers, for repeated
/// execution without host round trips (no reference counterpart; bench.py
/// and the C front use it). Not copyable.
class PreparedContraction {
 public:
  explicit PreparedContraction(const ValidatedContraction& v, int device = 0);
  ~PreparedContraction();
  PreparedContraction(const PreparedContraction&) = delete;
  PreparedContraction& operator=(const PreparedContraction&) = delete;

  /// Host -> device copies of both operands (storage order of the tensors).
  void upload(const double* left, const double* right);
  /// Permutations + the GEMM/GEMV/DOT launch, on the device stream (async).
  void run();
  /// The two halves of run(): operand permutations (L3 only) and the single
  /// GEMM/GEMV/DOT launch (which reads the permuted operands of the last
  /// run_permutes()). Separately callable so the kernels can be timed alone.
  void run_permutes();
  void run_contraction();
  /// Permutations + the contraction with the output scattered: the output's
  /// outermost label is split into `parts` equal blocks and block p is
  /// written at base + p * part_stride (doubles), each block laid out as it
  /// is inside the output (block p of a column-major output = its elements
  /// [p*B, (p+1)*B), B = output_elements() / parts). One GEMM launch; with
  /// `base` inside a tcb_peer_window the epilogue writes every block straight
  /// into its owner's receive buffer over NVLink (the fused K-split exchange,
  /// SURVEY §8e). Throws std::invalid_argument when the label does not split.
  void run_scattered(double* base, int parts, std::int64_t part_stride);
  /// Device -> host copy of the result (synchronous).
  void download(double* out);
  void sync();

  /// Host-to-host evaluation with the transfers overlapped with compute: the
  /// operand carrying the output's outermost label (when that label is also
  /// its own outermost mode) is uploaded slab by slab on a copy stream while
  /// earlier slabs are contracted, and output slabs are downloaded on a second
  /// copy stream as they complete. Needs page-locked host buffers for the
  /// copies to overlap; otherwise (or when no such label exists) it is
  /// upload + run + download. `slabs` <= 0 picks ~16 MB slabs (up to 64;
  /// below 32 MB of streamed data the plain path is used). When the output
  /// is smaller than the operand that would have to go up whole, slabs of a
  /// contracted label are streamed instead (both operands by 2-D copies, C
  /// accumulated on the device, downloaded once). Returns the slab count.
  /// With `wait` false the call returns once everything is enqueued: the
  /// next run_streamed overlaps its uploads with this one's download drain
  /// (repeated host-to-host contractions); sync() (or any other member)
  /// completes it, after which `out` holds the result.
  int run_streamed(const double* left, const double* right, double* out, int slabs = 0,
                   bool wait = true);

  const DeviceRecipe& recipe() const { return recipe_; }
  std::int64_t left_elements() const { return nl_; }
  std::int64_t right_elements() const { return nr_; }
  std::int64_t output_elements() const { return no_; }
  double* left_device() const { return dl_; }
  double* right_device() const { return dr_; }
  double* output_device() const { return do_; }
  std::int64_t launches_last_run() const { return launches_; }
  std::int64_t permuted_bytes() const;

 private:
  DeviceRecipe recipe_;
  ValidatedContraction v_;
  bool groups_ok_ = true;  // L4 allowed (cleared if the device refuses it)
  int auto_slabs_ = -1;    // run_streamed's automatic slab count, once decided
  int stream_mode_ = -1;   // run_streamed: 0 output-label slabs, 1 + label: contracted slabs,
                           // -2 - label: slabs of a free label by 2-D copies (run_streamed_f)
  int f_slabs_ = 0;        // run_streamed_f: slab count, decided with the label
  int pick_free_label(int* slabs) const;
  int run_streamed_f(const double* left, const double* right, double* out, int slabs,
                     int label, bool wait);
  int run_streamed_k(const double* left, const double* right, double* out, int slabs,
                     int label, bool wait);
  int device_ = 0;
  std::int64_t nl_ = 0, nr_ = 0, no_ = 0;
  double *dl_ = nullptr, *dr_ = nullptr, *do_ = nullptr;
  double *pl_ = nullptr, *pr_ = nullptr;  // permuted operands (L3)
  // second buffer set of the pipelined streamed path (flip_buffers)
  double *dl2_ = nullptr, *dr2_ = nullptr, *do2_ = nullptr, *pl2_ = nullptr, *pr2_ = nullptr;
  int dbuf_ = -1;  // -1 undecided, 0 one set, 1 two sets
  int set_ = 0;    // buffer set in use
  void flip_buffers();
  std::int64_t launches_ = 0;
  struct Pipes;
  std::unique_ptr<Pipes> pipes_;  // streamed path: copy streams + events
  // idle Pipes are pooled per device (process-wide) across prepared
  // contractions: creating and destroying them costs ~0.1 ms each
  static std::unique_ptr<Pipes> acquire_pipes(int device);
  static void release_pipes(int device, std::unique_ptr<Pipes> p);
};


// ---------------------------------------------------------------- tensor I/O
// The reference's TENSOR v1 text format (include/tc/tensor_io.hpp:9-16,
// src/tensor_io.cpp): header lines `TENSOR v1`, `name`, `rank`, `extents`,
// `variance`, `layout colmajor`, then the values in storage order with 17
// significant digits, eight per line. Byte-identical output; the engine
// formats and parses large tensors in parallel blocks.
void write_tensor(std::ostream& os, const Tensor& t);
void write_tensor_file(const std::string& path, const Tensor& t);
Tensor read_tensor(std::istream& is);
Tensor read_tensor_file(const std::string& path);

// ---------------------------------------------------------------- benchmark
// The reference's benchmark sweep (include/tc/bench.hpp:13-51,
// src/bench.cpp): built-in experiments square3d / cc4d / gr4d or a custom
// expression, one row per (contraction, forced kernel, size), median of the
// timed repetitions after one warm-up; backend "b200" runs each evaluation on
// the device (ExecutionStats::wall_seconds, transfers included).
struct BenchConfig {
  std::string experiment = "square3d";  // square3d | cc4d | gr4d | custom
  std::vector<std::int64_t> sizes;
  std::vector<KernelKind> kernels;
  std::string backend = "b200";
  int repetitions = 5;
  std::uint64_t seed = 1;
  std::int64_t mem_cap_bytes = 4000000000;
  bool verify_sample = false;
  int workers = 1;
  std::string custom_expr;
  std::map<std::string, std::int64_t> custom_extents;
};

struct BenchRow {
  std::string experiment;
  std::string expression;
  std::int64_t size = 0;
  std::string kernel;
  std::string backend;
  int repetitions = 0;
  double median_seconds = 0.0;
  double gflops = 0.0;
  std::int64_t packed_bytes = 0;
  bool available = false;
  bool verified_ok = true;  // true when sampling is off or the sample matched
  /// What ran (not in the reference): with backend "b200" every forced-kernel
  /// row executes the contraction's own device recipe (one launch, e.g.
  /// "L1 gemm"), so rows of one contraction differ only in planning; with
  /// "b200-sliced" the forced plan's loop nest ran slice by slice
  /// ("sliced GER" ...). write_bench_csv appends it as an `executed` column.
  std::string executed;
};

std::vector<BenchRow> run_bench(const BenchConfig& config);
/// Columns: experiment, expression, size, kernel, backend, repetitions,
/// median_seconds, gflops, packed_bytes; unavailable kernels carry NA cells.
void write_bench_csv(std::ostream& os, const std::vector<BenchRow>& rows);

}  // namespace tc

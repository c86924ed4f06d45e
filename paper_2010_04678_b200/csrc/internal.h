// Host-side internal interfaces shared by the CALS translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <atomic>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

#include <cstdlib>

namespace cals {
// Debug aid (CALS_POISON=1): every workspace allocation is filled with 0xFF
// bytes (NaN doubles, -1 ints) so a kernel that reads memory nobody wrote
// shows up as a changed result instead of depending on what the allocator
// handed back.
inline bool poison_enabled() {
  static const bool on = [] {
    const char* v = getenv("CALS_POISON");
    return v && atoi(v) != 0;
  }();
  return on;
}
inline void poison_alloc(void* p, size_t bytes, cudaStream_t s = nullptr, bool async = false) {
  if (!poison_enabled() || !p || !bytes) return;
  if (async) cudaMemsetAsync(p, 0xFF, bytes, s); else cudaMemset(p, 0xFF, bytes);
}
}  // namespace cals

namespace cals {

constexpr int kMaxOrder = 8;

// One mode's MTTKRP expressed on the contiguous 3-D view of the tensor
// (see mttkrp.cuh).  lo_modes / hi_modes list the factor modes whose
// Khatri-Rao product forms Lo / Hi, lowest mode first (= fastest row index).
struct ModePlan {
  int mode = 0;
  int role = 0;
  long long D[3] = {1, 1, 1};
  long long M = 0, Dp = 0, Dq = 0;
  int S = 1;
  std::vector<int> lo_modes, hi_modes;
  bool lo_direct() const { return lo_modes.size() == 1; }
  bool hi_direct() const { return hi_modes.size() == 1; }
  bool hi_ones() const { return hi_modes.empty(); }
};

// Ozaki slices of one tensor view (ozaki.cuh): xs[7][Dq][M][Kp] int8, rex[Dq][M].
struct OzSlices {
  uint8_t* xs = nullptr;
  int* rex = nullptr;
  int* flag = nullptr;  // device flag of a slicing not yet checked (ozaki_validate)
  long long Kp = 0, M = 0, Dq = 0, Dp = 0;
  CUtensorMap map;   // full 64-row tiles
  CUtensorMap rmap;  // packed remainder tiles (== map when unused)
};

// Device-resident dense tensor, mode-0 fastest, I0 padded to even so every
// 3-D view has 16-byte aligned TMA strides.  Zero padding contributes nothing.
struct Tensor {
  int device = 0;
  int order = 0;
  long long dims[kMaxOrder] = {0};
  long long i0p = 0;       // padded leading extent
  long long numel = 0;     // logical element count
  double* data = nullptr;  // [i0p * prod(dims[1:])]
  bool owned = false;
  double sqnorm = -1.0;
  unsigned long long uid = 0;  // unique per tensor_create (addresses get reused)
  std::vector<ModePlan> plans;
  // A-operand tensor maps cached per (mode, variant)
  std::map<std::pair<int, int>, CUtensorMap> amaps;
  // Ozaki X slices per view key (mode index, or >= 100 for engine-private views)
  std::map<int, OzSlices> oz;
  std::mutex mu;
};

int tensor_create(int order, const int64_t* dims, const double* host, const double* dev,
                  cudaStream_t stream, Tensor** out);
void tensor_destroy(Tensor* t);
// kErrInvalid unless the calling thread's current CUDA device is the tensor's
int check_current_device(const Tensor& t);
int tensor_sqnorm(Tensor* t, cudaStream_t stream, double* out);
ModePlan make_plan(const Tensor& t, int mode);
// Programmatic dependent launch (PDL): every kernel of the engine's
// iteration is launched with programmatic stream serialization, so its launch
// overlaps the tail of the kernel before it; each such kernel calls
// griddep_wait() before it touches anything its predecessors wrote (at its
// very top unless noted), so stream order is preserved transitively.
// CALS_PDL=0 disables it (A/B measurements).
bool pdl_enabled();
template <typename... P, typename... A>
inline cudaError_t launch_dep(void (*k)(P...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

int plan_splits(const ModePlan& view);  // shape-only q-split count of a view

// MTTKRP variants ------------------------------------------------------------
struct VariantInfo {
  int MI, NI, WM, WN;
  int BM, BN;
};
int num_variants();
const VariantInfo& variant_info(int v);
int choose_variant(long long M, long long width_hint, int S);

// Workspace bytes the MTTKRP of `mode` needs at width `cap` (partials + KRPs).
size_t mttkrp_workspace_bytes(const Tensor& t, int mode, long long cap);

struct FactorSet {
  const double* ptr[kMaxOrder];  // row-major [I_n][ld] factor buffers
  long long ld;                  // leading dimension (columns), even
};

// Split-K partials left for the consumer: with a SplitDefer passed to the
// launches below, an S > 1 contraction skips its split_reduce_kernel and
// reports where its partials are (block s, row m, column c at
// part[s * stride + m * ldp + c]); the consumer sums them in s order, the
// reduction's own order (the split update's solve kernel, update2.cu).
// S stays 0 when the contraction wrote `out` itself.
struct SplitDefer {
  const double* part = nullptr;
  long long stride = 0;
  long long ldp = 0;
  int S = 0;
  // input: byte ranges the consumer WRITES while other CTAs of it still read
  // the partials (the solve's fused Lo-slice targets live in the same
  // workspace).  A partial set overlapping one of them is reduced by
  // split_reduce_kernel instead of being deferred.
  static constexpr int kMaxAvoid = 6;
  const void* avoid[kMaxAvoid] = {};
  size_t avoid_bytes[kMaxAvoid] = {};
  int n_avoid = 0;
  void add_avoid(const void* p, size_t bytes) {
    if (p && bytes && n_avoid < kMaxAvoid) {
      avoid[n_avoid] = p;
      avoid_bytes[n_avoid++] = bytes;
    }
  }
  bool overlaps(const void* p, size_t bytes) const {
    const char* a0 = static_cast<const char*>(p);
    for (int i = 0; i < n_avoid; ++i) {
      const char* b0 = static_cast<const char*>(avoid[i]);
      if (a0 < b0 + avoid_bytes[i] && b0 < a0 + bytes) return true;
    }
    return false;
  }
};
// Only partial sets that stay L2-resident are deferred: the solve kernel's
// staging re-reads them per model block (c3: 11 x 251 x 300 doubles, 6.6 MB,
// 4.26k -> 4.32k models/s); c2's 84 MB partial set, mostly evicted by the
// dimension tree's side output, reduces faster in split_reduce_kernel
// (28.8k vs 29.1k).
inline bool split_deferrable(int S, long long M, long long ldp) {
  return S > 1 && double(S) * double(M) * double(ldp) * 8.0 <= 24.0 * (1 << 20);
}

// Launch one fused MTTKRP (+ split reduction) on `stream`.  `width` is used
// when width_ptr is null; otherwise the kernels read the active width from
// device memory (engine path, graph-capturable).  `cap` bounds the width and
// sizes the grid.
int launch_mttkrp(Tensor& t, int mode, const FactorSet& f, int width, const int* width_ptr,
                  long long cap, double* out, long long ldo, double* workspace,
                  size_t workspace_bytes, int variant, cudaStream_t stream,
                  bool lo_sliced = false, const int* lo_stale = nullptr,
                  SplitDefer* defer = nullptr);
// The Ozaki workspace launch_mttkrp carves for `mode` out of `workspace`
// (nullptr when the mode does not run on the INT8 path or it does not fit).
void* mttkrp_oz_ws(Tensor& t, int mode, long long ld, void* workspace, size_t workspace_bytes);

// Lower level: one contraction on an arbitrary 3-D view plan `p` of the tensor
// with explicit Lo [lrows][lo_ld] / Hi [Dq][hi_ld] operands.  map_key caches
// the tensor map (modes use their index, engine-private plans use >= 100).
// S > 1 needs `part` (S * M * lo_ld doubles) and reduces into `out`.
// With `oz_ws` (>= ozaki_ws_bytes) and prepared Ozaki slices for map_key the
// contraction runs on the INT8 tensor cores (ozaki.cuh); otherwise on DMMA.
int launch_contraction(Tensor& t, const ModePlan& p, int map_key, const double* lo,
                       long long lrows, long long lo_ld, const double* hi, long long hi_ld,
                       int width, const int* width_ptr, long long cap, double* out, long long ldo,
                       double* part, int variant, cudaStream_t stream, double* side = nullptr,
                       long long side_ld = 0, long long side_qstride = 0, void* oz_ws = nullptr,
                       size_t oz_ws_bytes = 0, bool lo_sliced = false,
                       const int* lo_stale = nullptr, SplitDefer* defer = nullptr);

// Ozaki-sliced INT8 tensor-core contraction (ozaki.cu) ------------------------
bool ozaki_enabled();                       // CALS_MTTKRP=dmma disables it
bool ozaki_eligible(const ModePlan& p);
bool ozaki_range_guard();                   // CALS_OZ_RANGE_GUARD=0 disables it
int ozaki_refine_splits(const ModePlan& p);  // shape-only split count for an INT8 view
size_t ozaki_ws_bytes(const ModePlan& p, long long cap);  // per-call Lo slices
double ozaki_tensor_ops(const ModePlan& p, long long width);  // INT8 ops per launch
// Build (once per tensor and key) the X slices of view `p`; stream-ordered.
// validate = false defers the range / finiteness check (one host sync) to
// ozaki_validate; unchecked slices are not used by launches.
int ozaki_prepare(Tensor& t, const ModePlan& p, int key, cudaStream_t stream,
                  bool validate = true);
int ozaki_validate(Tensor& t, int key, cudaStream_t stream);
void ozaki_release(Tensor& t);
// Whether a contraction of view `p` (slices under `key`) will run on the INT8
// path: eligible, slices prepared and checked.
bool ozaki_ready(Tensor& t, const ModePlan& p, int key);
// Where the per-call Lo slices of a contraction live in its Ozaki workspace:
// ls[7][cap_pad][Kp] (column c of Lo as a p-contiguous row), cex[c], and the
// work-unit counter.  A producer that writes them itself (the split update's
// solve kernel, update2.cu) lets the contraction skip its slicing kernel
// (lo_sliced = true), or run it only while *lo_stale != 0 (lo_stale: device
// flag, nullptr = always slice).
struct OzLoLayout {
  uint8_t* ls = nullptr;
  int* cex = nullptr;
  int* queue = nullptr;
  long long slice_stride = 0;  // cap_pad * Kp
  int Kp = 0;
  int Dp = 0;                  // Lo rows sliced (the rest of Kp is zero)
};
OzLoLayout ozaki_lo_layout(const ModePlan& p, long long lrows, long long cap, void* oz_ws);
int launch_contraction_ozaki(Tensor& t, const ModePlan& p, int key, const double* lo,
                             long long lrows, long long lo_ld, const double* hi, long long hi_ld,
                             int width, const int* width_ptr, long long cap, double* out,
                             long long ldo, double* part, void* oz_ws, size_t oz_ws_bytes,
                             cudaStream_t stream, double* side, long long side_ld,
                             long long side_qstride, bool lo_sliced = false,
                             const int* lo_stale = nullptr, SplitDefer* defer = nullptr);

// out[row][c] = sum over the reduced index of P[a + Da*b][c] * F[idx][c]
// (reduce_b: rows a < rows_out, sum b < Db with F[b]; else rows b, sum a < La
// with F[a]).  Deterministic ascending order; memory-bound.
int launch_partial_ttv(const double* P, long long ld, long long Da, long long Db, int reduce_b,
                       long long La, const double* F, long long ldf, int width,
                       const int* width_ptr, long long cap, long long rows_out, double* out,
                       long long ldo, int sms, cudaStream_t stream);

// Tensor maps ------------------------------------------------------------------
int encode_map_2d(CUtensorMap* m, const double* base, long long inner, long long outer,
                  long long ld_elems, int box_inner, int box_outer);
int encode_map_3d(CUtensorMap* m, const double* base, long long d0, long long d1, long long d2,
                  int b0, int b1, int b2);

int encode_map_u8(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
                  const uint64_t* strides_bytes, const uint32_t* box);  // SWIZZLE_32B

int sm_count(int device);

}  // namespace cals

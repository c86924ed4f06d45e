// Host side of the fused MTTKRP: tensor upload/padding, per-mode plans, TMA
// descriptor encoding, variant choice and launch (kernels in mttkrp.cuh).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "internal.h"
#include "mttkrp.cuh"

namespace cals {

// ---------------------------------------------------------------- errors --
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* get_error() { return g_err.c_str(); }

int sm_count(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cached[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
      v = 148;
    cached[device] = v;
  }
  return cached[device];
}

// ------------------------------------------------------------ tensor maps --
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int encode_map_2d(CUtensorMap* m, const double* base, long long inner, long long outer,
                  long long ld_elems, int box_inner, int box_outer) {
  auto enc = get_encode();
  CALS_CHECK(enc, kErrCuda, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 8};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CALS_CHECK(r == CUDA_SUCCESS, kErrCuda,
             "cuTensorMapEncodeTiled(2d) failed: code " + std::to_string((int)r) + " inner=" +
                 std::to_string(inner) + " outer=" + std::to_string(outer) +
                 " ld=" + std::to_string(ld_elems));
  return kOk;
}

int encode_map_3d(CUtensorMap* m, const double* base, long long d0, long long d1, long long d2,
                  int b0, int b1, int b2) {
  auto enc = get_encode();
  CALS_CHECK(enc, kErrCuda, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)d0 * 8, (cuuint64_t)(d0 * d1) * 8};
  cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, (cuuint32_t)b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides,
                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CALS_CHECK(r == CUDA_SUCCESS, kErrCuda,
             "cuTensorMapEncodeTiled(3d) failed: code " + std::to_string((int)r));
  return kOk;
}

// uint8 K-major operand maps for the Ozaki kernel: 32-byte inner box with the
// 32-byte swizzle the tcgen05 SWIZZLE_32B descriptors expect.
int encode_map_u8(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
                  const uint64_t* strides_bytes, const uint32_t* box) {
  auto enc = get_encode();
  CALS_CHECK(enc, kErrCuda, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = 1;
    if (i + 1 < rank) st[i] = strides_bytes[i];
  }
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, rank, const_cast<void*>(base), d, st, b, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CALS_CHECK(r == CUDA_SUCCESS, kErrCuda,
             "cuTensorMapEncodeTiled(u8) failed: code " + std::to_string((int)r));
  return kOk;
}

// ------------------------------------------------------------------ tensor --
__global__ void sqnorm_partial_kernel(const double* __restrict__ x, long long n,
                                      double* __restrict__ part) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    s = fma(x[i], x[i], s);
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// Deterministic sum of n partials by one block of 1024 threads: strided
// per-thread sums, an xor butterfly in each warp (partners add the same two
// values: every lane holds the same bits), warp sums in warp order.  (One
// thread adding 1024 values in sequence took ~40 us.)
__global__ void __launch_bounds__(1024) sum_kernel(const double* __restrict__ part, int n,
                                                   double* out) {
  __shared__ double ws[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) v += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = ws[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) s += ws[w];
    *out = s;
  }
}

ModePlan make_plan(const Tensor& t, int mode) {
  ModePlan p;
  const int N = t.order;
  p.mode = mode;
  auto prod = [&](int a, int b) {  // prod dims[a..b)
    long long v = 1;
    for (int i = a; i < b; ++i) v *= t.dims[i];
    return v;
  };
  if (mode == 0) {
    p.role = kRoleFirst;
    p.D[0] = t.i0p;
    p.D[1] = t.dims[1];
    p.D[2] = prod(2, N);
    p.M = t.dims[0];
    p.Dp = p.D[1];
    p.Dq = p.D[2];
    p.lo_modes = {1};
    for (int i = 2; i < N; ++i) p.hi_modes.push_back(i);
  } else if (mode == N - 1) {
    p.role = kRoleLast;
    p.D[0] = t.i0p;
    p.D[1] = prod(1, N - 1);
    p.D[2] = t.dims[N - 1];
    p.M = t.dims[N - 1];
    p.Dp = p.D[0];
    p.Dq = p.D[1];
    p.lo_modes = {0};
    for (int i = 1; i < N - 1; ++i) p.hi_modes.push_back(i);
  } else {
    p.role = kRoleMiddle;
    p.D[0] = t.i0p * prod(1, mode);
    p.D[1] = t.dims[mode];
    p.D[2] = prod(mode + 1, N);
    p.M = t.dims[mode];
    p.Dp = p.D[0];
    p.Dq = p.D[2];
    for (int i = 0; i < mode; ++i) p.lo_modes.push_back(i);
    for (int i = mode + 1; i < N; ++i) p.hi_modes.push_back(i);
  }
  p.S = plan_splits(p);
  return p;
}

// q splits: a function of the shape only (never of the active width) so the
// fused result of a column block is bitwise independent of its neighbours.
// CALS_SPLITS fixes the count (tuning knob; still shape-only); otherwise 32,
// refined for INT8 views whose leftover rows pack better with another count.
int plan_splits(const ModePlan& view) {
  static const int env_splits = [] {
    const char* env = getenv("CALS_SPLITS");
    return env ? atoi(env) : 0;
  }();
  ModePlan p = view;
  p.S = (int)std::max<long long>(1, std::min<long long>(p.Dq, env_splits > 0 ? env_splits : 32));
  if (env_splits <= 0) {
    if (ozaki_eligible(p)) {
      p.S = ozaki_refine_splits(p);
    } else if (p.Dq < 64) {
      // few slabs: ~2 per split can make the view INT8-eligible
      ModePlan q = p;
      q.S = (int)((p.Dq + 1) / 2);
      if (q.S < p.S && ozaki_eligible(q)) p.S = q.S;
    }
  }
  return p.S;
}

__global__ void pad_copy_kernel(const double* __restrict__ src, long long i0, long long i0p,
                                long long rows, double* __restrict__ dst) {
  const long long n = i0p * rows;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e % i0p, row = e / i0p;
    dst[e] = i < i0 ? src[row * i0 + i] : 0.0;
  }
}

int tensor_create(int order, const int64_t* dims, const double* host, const double* dev,
                  cudaStream_t stream, Tensor** out) {
  CALS_CHECK(out != nullptr, kErrInvalid, "null output handle");
  CALS_CHECK(order >= 2 && order <= kMaxOrder, kErrInvalid,
             "tensor order must be in [2, 8], got " + std::to_string(order));
  CALS_CHECK((host != nullptr) != (dev != nullptr), kErrInvalid,
             "exactly one of host / device data must be given");
  std::unique_ptr<Tensor> t(new Tensor());
  static std::atomic<unsigned long long> next_uid{1};
  t->uid = next_uid.fetch_add(1);
  CALS_CUDA_TRY(cudaGetDevice(&t->device));
  t->order = order;
  long long rest = 1;
  for (int i = 0; i < order; ++i) {
    CALS_CHECK(dims[i] >= 1, kErrInvalid, "all extents must be >= 1");
    t->dims[i] = dims[i];
    if (i > 0) rest *= dims[i];
  }
  t->numel = dims[0] * rest;
  t->i0p = dims[0] + (dims[0] & 1);
  const bool aligned_dev =
      dev && t->i0p == dims[0] && (reinterpret_cast<uintptr_t>(dev) % 16 == 0);
  if (aligned_dev) {
    t->data = const_cast<double*>(dev);  // borrowed
  } else {
    const size_t bytes = size_t(t->i0p) * size_t(rest) * 8;
    // stream-ordered pool allocation: repeated sweeps over fresh tensors of
    // the same shape reuse the pool's pages instead of cudaMalloc / cudaFree
    static std::once_flag pool_once;
    std::call_once(pool_once, [dev = t->device] {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
    });
    CALS_CUDA_TRY(cudaMallocAsync(&t->data, bytes, stream));
    poison_alloc(t->data, bytes, stream, true);
    t->owned = true;
    if (host) {
      if (t->i0p == dims[0]) {  // one linear DMA (full PCIe rate from pinned memory)
        CALS_CUDA_TRY(cudaMemcpyAsync(t->data, host, bytes, cudaMemcpyHostToDevice, stream));
      } else {
        CALS_CUDA_TRY(cudaMemcpy2DAsync(t->data, t->i0p * 8, host, dims[0] * 8, dims[0] * 8,
                                        rest, cudaMemcpyHostToDevice, stream));
        // zero the pad column (one double per row)
        CALS_CUDA_TRY(cudaMemset2DAsync(t->data + dims[0], t->i0p * 8, 0, 8, rest, stream));
      }
    } else {
      const int sms = sm_count(t->device);
      pad_copy_kernel<<<sms * 4, 256, 0, stream>>>(dev, dims[0], t->i0p, rest, t->data);
      CALS_CUDA_TRY(cudaGetLastError());
    }
  }
  for (int n = 0; n < order; ++n) t->plans.push_back(make_plan(*t, n));
  *out = t.release();
  return kOk;
}

int check_current_device(const Tensor& t) {
  int cur = -1;
  CALS_CUDA_TRY(cudaGetDevice(&cur));
  CALS_CHECK(cur == t.device, kErrInvalid,
             "the tensor was uploaded to CUDA device " + std::to_string(t.device) +
                 " but the current device is " + std::to_string(cur));
  return kOk;
}

void tensor_destroy(Tensor* t) {
  if (!t) return;
  // The buffers may still be read by kernels queued on any stream (the
  // engine's, an operator call's, the slicing stream): wait for the device
  // before handing the memory back to the pool.  Destroying a tensor is rare
  // (release_device / garbage collection), never on a hot path.
  int prev = -1;
  cudaGetDevice(&prev);
  if (prev != t->device) cudaSetDevice(t->device);
  cudaDeviceSynchronize();
  ozaki_release(*t);
  if (t->owned && t->data) cudaFreeAsync(t->data, 0);
  if (prev >= 0 && prev != t->device) cudaSetDevice(prev);
  delete t;
}

int tensor_sqnorm(Tensor* t, cudaStream_t stream, double* out) {
  if (t->sqnorm < 0) {
    const long long n = t->i0p * (t->numel / t->dims[0]);  // padding is zero
    const int blocks = 1024;
    double* buf = nullptr;
    CALS_CUDA_TRY(cudaMallocAsync(&buf, (blocks + 1) * sizeof(double), stream));
    sqnorm_partial_kernel<<<blocks, 256, 0, stream>>>(t->data, n, buf);
    sum_kernel<<<1, 1024, 0, stream>>>(buf, blocks, buf + blocks);
    double h = 0;
    CALS_CUDA_TRY(cudaMemcpyAsync(&h, buf + blocks, 8, cudaMemcpyDeviceToHost, stream));
    CALS_CUDA_TRY(cudaStreamSynchronize(stream));
    CALS_CUDA_TRY(cudaFreeAsync(buf, stream));
    t->sqnorm = h;
  }
  *out = t->sqnorm;
  return kOk;
}

// ---------------------------------------------------------------- variants --
using LaunchFn = cudaError_t (*)(dim3, const CUtensorMap&, const CUtensorMap&, const MttkrpArgs&,
                                 bool kc, cudaStream_t);

template <int MI, int NI, int WM, int WN>
static cudaError_t launch_variant(dim3 grid, const CUtensorMap& a, const CUtensorMap& b,
                                  const MttkrpArgs& args, bool kc, cudaStream_t stream) {
  using C = TileCfg<MI, NI, WM, WN>;
  const size_t smem = C::kSmemBytes;
  static std::once_flag once;
  static cudaError_t cfg = cudaSuccess;
  std::call_once(once, [&] {
    cfg = cudaFuncSetAttribute(mttkrp_dmma_kernel<MI, NI, WM, WN, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cfg == cudaSuccess)
      cfg = cudaFuncSetAttribute(mttkrp_dmma_kernel<MI, NI, WM, WN, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (cfg != cudaSuccess) return cfg;
  if (kc)
    return launch_dep(mttkrp_dmma_kernel<MI, NI, WM, WN, true>, grid, dim3(C::kThreads), smem,
                      stream, a, b, args);
  return launch_dep(mttkrp_dmma_kernel<MI, NI, WM, WN, false>, grid, dim3(C::kThreads), smem,
                    stream, a, b, args);
}

template <int MI, int NI, int WM, int WN>
static int occupancy_variant() {
  using C = TileCfg<MI, NI, WM, WN>;
  static int occ = -1;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (occ < 0) {
    cudaFuncSetAttribute(mttkrp_dmma_kernel<MI, NI, WM, WN, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmemBytes);
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &v, mttkrp_dmma_kernel<MI, NI, WM, WN, true>, C::kThreads, C::kSmemBytes) !=
            cudaSuccess ||
        v < 1)
      v = 1;
    occ = v;
  }
  return occ;
}

struct VariantEntry {
  VariantInfo info;
  LaunchFn launch;
  int (*occupancy)();
};

#define CALS_VARIANT(MI, NI, WM, WN)                                               \
  VariantEntry {                                                                   \
    VariantInfo{MI, NI, WM, WN, 8 * MI * WM, 8 * NI * WN}, &launch_variant<MI, NI, WM, WN>, \
        &occupancy_variant<MI, NI, WM, WN>                                         \
  }

static const VariantEntry kVariants[] = {
    CALS_VARIANT(4, 4, 2, 2),  // 64 x 64
    CALS_VARIANT(5, 3, 1, 4),  // 40 x 96
    CALS_VARIANT(3, 4, 1, 4),  // 24 x 128
    CALS_VARIANT(2, 4, 1, 4),  // 16 x 128
    CALS_VARIANT(1, 4, 1, 4),  // 8 x 128
};

int num_variants() { return int(sizeof(kVariants) / sizeof(kVariants[0])); }
const VariantInfo& variant_info(int v) { return kVariants[v].info; }

int choose_variant(long long M, long long width_hint, int S) {
  const long long slots = 2LL * sm_count(0);
  long long best_cost = -1;
  int best = 0;
  for (int v = 0; v < num_variants(); ++v) {
    const auto& vi = kVariants[v].info;
    const long long tm = (M + vi.BM - 1) / vi.BM;
    const long long tn = (std::max<long long>(width_hint, 1) + vi.BN - 1) / vi.BN;
    const long long units = tm * tn * S;
    const long long waves = (units + slots - 1) / slots;
    // padded work per slot, plus a per-unit fixed cost (pipeline fill, epilogue)
    const long long cost = waves * ((long long)vi.BM * vi.BN + 1024);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = v;
    }
  }
  return best;
}

// --------------------------------------------------------- KRP / reduction --
struct KrpParts {
  const double* ptr[kMaxOrder];
  long long ext[kMaxOrder];    // extent used to decode the row index
  long long valid[kMaxOrder];  // rows >= valid are zero (padding of mode 0)
  int n;
};

__global__ void krp_rows_kernel(KrpParts parts, long long ld_in, long long rows, const int* wptr,
                                int width, double* __restrict__ out, long long ldo) {
  const int W = wptr ? *wptr : width;
  const long long n = rows * W;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / W;
    const int c = int(e % W);
    long long rem = row;
    double v = 1.0;
    for (int k = 0; k < parts.n; ++k) {
      const long long idx = rem % parts.ext[k];
      rem /= parts.ext[k];
      v = idx < parts.valid[k] ? v * parts.ptr[k][idx * ld_in + c] : 0.0;
    }
    out[row * ldo + c] = v;
  }
}

__global__ void fill_kernel(double* p, long long n, double v) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    p[e] = v;
}

__global__ void split_reduce_kernel(const double* __restrict__ part, long long part_stride, int S,
                                    int M, long long ldp, const int* width_ptr, int width,
                                    double* __restrict__ out, long long ldo) {
  griddep_wait();  // launched with PDL (launch_dep): predecessors complete
  griddep_launch_dependents();  // the next kernel may start its prologue
  const int W = width_ptr ? *width_ptr : width;
  const int hw = (W + 1) >> 1;  // column pairs
  const long long n = (long long)M * hw;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int m = int(e / hw);
    const int c = int(e % hw) * 2;
    const double* src = part + (long long)m * ldp + c;
    if (c + 1 < W) {
      double2 acc = *reinterpret_cast<const double2*>(src);
      for (int s = 1; s < S; ++s) {
        const double2 v = *reinterpret_cast<const double2*>(src + s * part_stride);
        acc.x += v.x;
        acc.y += v.y;
      }
      *reinterpret_cast<double2*>(out + (long long)m * ldo + c) = acc;
    } else {
      double acc = src[0];
      for (int s = 1; s < S; ++s) acc += src[s * part_stride];
      out[(long long)m * ldo + c] = acc;
    }
  }
}

static long long lo_rows(const Tensor& t, const ModePlan& p) {
  return p.lo_direct() ? t.dims[p.lo_modes[0]] : p.Dp;
}

size_t mttkrp_workspace_bytes(const Tensor& t, int mode, long long cap) {
  const ModePlan& p = t.plans[mode];
  const long long ld = (cap + 7) / 8 * 8;
  size_t b = 0;
  if (p.S > 1) b += size_t(p.S) * size_t(p.M) * size_t(ld) * 8;
  if (!p.lo_direct()) b += size_t(p.Dp) * size_t(ld) * 8;
  if (!p.hi_direct()) b += size_t(std::max<long long>(p.Dq, 1)) * size_t(ld) * 8;
  if (ozaki_eligible(p)) b += ozaki_ws_bytes(p, ld) + 256;
  return b + 256;
}

int launch_mttkrp(Tensor& t, int mode, const FactorSet& f, int width, const int* width_ptr,
                  long long cap, double* out, long long ldo, double* workspace,
                  size_t workspace_bytes, int variant, cudaStream_t stream, bool lo_sliced,
                  const int* lo_stale, SplitDefer* defer) {
  CALS_CHECK(mode >= 0 && mode < t.order, kErrInvalid, "mode out of range");
  const ModePlan& p = t.plans[mode];
  CALS_CHECK(f.ld % 2 == 0 && f.ld >= cap, kErrInvalid, "factor leading dimension must be even");
  CALS_CHECK(ldo % 2 == 0 && ldo >= cap, kErrInvalid, "output leading dimension must be even");
  CALS_CHECK(cap >= 1 && (width_ptr || (width >= 1 && width <= cap)), kErrInvalid,
             "width must be in [1, capacity]");
  CALS_CHECK(mttkrp_workspace_bytes(t, mode, f.ld) <= workspace_bytes || p.S == 1, kErrInvalid,
             "MTTKRP workspace too small");
  const int sms = sm_count(t.device);

  // carve the workspace
  char* wsp = reinterpret_cast<char*>(workspace);
  double* part = nullptr;
  if (p.S > 1) {
    part = reinterpret_cast<double*>(wsp);
    wsp += size_t(p.S) * size_t(p.M) * size_t(f.ld) * 8;
  }
  const double* lo = nullptr;
  const double* hi = nullptr;
  long long lo_ld = f.ld, hi_ld = f.ld;
  const long long lrows = lo_rows(t, p);
  if (p.lo_direct()) {
    lo = f.ptr[p.lo_modes[0]];
  } else {
    double* buf = reinterpret_cast<double*>(wsp);
    wsp += size_t(p.Dp) * size_t(f.ld) * 8;
    KrpParts kp{};
    kp.n = (int)p.lo_modes.size();
    for (int k = 0; k < kp.n; ++k) {
      const int m = p.lo_modes[k];
      kp.ptr[k] = f.ptr[m];
      kp.ext[k] = m == 0 ? t.i0p : t.dims[m];
      kp.valid[k] = t.dims[m];
    }
    krp_rows_kernel<<<sms * 8, 256, 0, stream>>>(kp, f.ld, p.Dp, width_ptr, width, buf, f.ld);
    CALS_CUDA_TRY(cudaGetLastError());
    lo = buf;
  }
  if (p.hi_direct()) {
    hi = f.ptr[p.hi_modes[0]];
  } else {
    double* buf = reinterpret_cast<double*>(wsp);
    wsp += size_t(std::max<long long>(p.Dq, 1)) * size_t(f.ld) * 8;
    if (p.hi_ones()) {
      fill_kernel<<<std::max<long long>(1, std::min<long long>(sms, (f.ld + 255) / 256)), 256, 0,
                    stream>>>(buf, f.ld, 1.0);
    } else {
      KrpParts kp{};
      kp.n = (int)p.hi_modes.size();
      for (int k = 0; k < kp.n; ++k) {
        const int m = p.hi_modes[k];
        kp.ptr[k] = f.ptr[m];
        kp.ext[k] = t.dims[m];
        kp.valid[k] = t.dims[m];
      }
      krp_rows_kernel<<<sms * 8, 256, 0, stream>>>(kp, f.ld, p.Dq, width_ptr, width, buf, f.ld);
    }
    CALS_CUDA_TRY(cudaGetLastError());
    hi = buf;
  }
  // INT8 tensor-core path: X slices built once per tensor (never inside a
  // graph capture -- the engine prepares them before capturing)
  void* oz_ws = nullptr;
  size_t oz_bytes = 0;
  if (ozaki_eligible(p)) {
    char* o = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(wsp) + 255) & ~uintptr_t(255));
    const size_t need = ozaki_ws_bytes(p, f.ld);
    if (o + need <= reinterpret_cast<char*>(workspace) + workspace_bytes) {
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      CALS_CUDA_TRY(cudaStreamIsCapturing(stream, &cs));
      if (cs == cudaStreamCaptureStatusNone) {
        const int rc = ozaki_prepare(t, p, mode, stream);
        if (rc) return rc;
      }
      oz_ws = o;
      oz_bytes = need;
    }
  }
  return launch_contraction(t, p, mode, lo, lrows, lo_ld, hi, hi_ld, width, width_ptr, cap, out,
                            ldo, part, variant, stream, nullptr, 0, 0, oz_ws, oz_bytes, lo_sliced,
                            lo_stale, defer);
}

void* mttkrp_oz_ws(Tensor& t, int mode, long long ld, void* workspace, size_t workspace_bytes) {
  const ModePlan& p = t.plans[mode];
  if (!ozaki_eligible(p)) return nullptr;
  size_t off = 0;  // the carve of launch_mttkrp
  if (p.S > 1) off += size_t(p.S) * size_t(p.M) * size_t(ld) * 8;
  if (!p.lo_direct()) off += size_t(p.Dp) * size_t(ld) * 8;
  if (!p.hi_direct()) off += size_t(std::max<long long>(p.Dq, 1)) * size_t(ld) * 8;
  char* base = reinterpret_cast<char*>(workspace);
  char* o = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(base + off) + 255) & ~uintptr_t(255));
  if (o + ozaki_ws_bytes(p, ld) > base + workspace_bytes) return nullptr;
  return o;
}

int launch_contraction(Tensor& t, const ModePlan& p, int map_key, const double* lo,
                       long long lrows, long long lo_ld, const double* hi, long long hi_ld,
                       int width, const int* width_ptr, long long cap, double* out, long long ldo,
                       double* part, int variant, cudaStream_t stream, double* side,
                       long long side_ld, long long side_qstride, void* oz_ws,
                       size_t oz_ws_bytes, bool lo_sliced, const int* lo_stale,
                       SplitDefer* defer) {
  static const bool dbg = getenv("CALS_DEBUG_OZ") != nullptr;
  if (dbg)
    fprintf(stderr, "[oz] contraction key=%d role=%d M=%lld Dp=%lld Dq=%lld S=%d oz_ws=%p elig=%d\n",
            map_key, p.role, p.M, p.Dp, p.Dq, p.S, oz_ws, (int)ozaki_eligible(p));
  if (oz_ws && ozaki_eligible(p)) {
    const int rc = launch_contraction_ozaki(t, p, map_key, lo, lrows, lo_ld, hi, hi_ld, width,
                                            width_ptr, cap, out, ldo, part, oz_ws, oz_ws_bytes,
                                            stream, side, side_ld, side_qstride, lo_sliced,
                                            lo_stale, defer);
    if (dbg) fprintf(stderr, "[oz]   ozaki rc=%d\n", rc);
    if (rc != kErrUnsupported) return rc;  // unsupported = slices not prepared: DMMA below
  }
  if (variant < 0) variant = choose_variant(p.M, cap, p.S);
  const VariantEntry& ve = kVariants[variant];
  const int sms = sm_count(t.device);
  CALS_CHECK(p.S == 1 || part != nullptr, kErrInvalid, "split-K needs a partial buffer");
  // tensor maps
  auto key = std::make_pair(map_key, variant);
  std::unique_lock<std::mutex> maps_lock(t.mu);
  auto it = t.amaps.find(key);
  if (it == t.amaps.end()) {
    CUtensorMap m;
    int rc;
    const int BM = ve.info.BM;
    if (p.role == kRoleFirst)
      rc = encode_map_3d(&m, t.data, p.D[0], p.D[1], p.D[2], BM + kPad, kBK, 1);
    else if (p.role == kRoleMiddle)
      rc = encode_map_3d(&m, t.data, p.D[0], p.D[1], p.D[2], kBK + kPad, BM, 1);
    else if (p.role == kRoleLast)
      rc = encode_map_3d(&m, t.data, p.D[0], p.D[1], p.D[2], kBK + kPad, 1, BM);
    else  // kRoleFirstQP: (m, q, p) -> smem [k][m]
      rc = encode_map_3d(&m, t.data, p.D[0], p.D[1], p.D[2], BM + kPad, 1, kBK);
    if (rc) return rc;
    it = t.amaps.emplace(key, m).first;
  }
  const CUtensorMap mapA = it->second;
  maps_lock.unlock();
  CUtensorMap mapB;
  {
    int rc = encode_map_2d(&mapB, lo, lo_ld, lrows, lo_ld, ve.info.BN + kPad, kBK);
    if (rc) return rc;
  }

  MttkrpArgs a{};
  a.role = p.role;
  a.M = (int)p.M;
  a.Dp = (int)p.Dp;
  a.Dq = (int)p.Dq;
  a.S = p.S;
  a.width = width;
  a.width_ptr = width_ptr;
  a.hi = hi;
  a.ldh = hi_ld;
  a.out = p.S > 1 ? part : out;
  a.ldo = p.S > 1 ? lo_ld : ldo;
  a.part_stride = (long long)p.M * lo_ld;
  a.side = side;
  a.ld_side = side_ld;
  a.side_qstride = side_qstride;

  const long long tm = (p.M + ve.info.BM - 1) / ve.info.BM;
  const long long tn = (cap + ve.info.BN - 1) / ve.info.BN;
  const long long units = tm * tn * p.S;
  const long long slots = (long long)ve.occupancy() * sms;
  dim3 grid((unsigned)std::max<long long>(1, std::min(units, slots)));
  const bool kcontig = p.role == kRoleMiddle || p.role == kRoleLast;
  CALS_CUDA_TRY(ve.launch(grid, mapA, mapB, a, kcontig, stream));
  if (defer && split_deferrable(p.S, p.M, lo_ld) &&
      !defer->overlaps(part, size_t(p.S) * size_t(a.part_stride) * 8)) {
    *defer = SplitDefer{part, a.part_stride, lo_ld, p.S};
  } else if (p.S > 1) {
    const long long pairs = p.M * ((cap + 1) / 2);
    const int blocks = (int)std::max<long long>(1, std::min<long long>(sms * 8, (pairs + 255) / 256));
    CALS_CUDA_TRY(launch_dep(split_reduce_kernel, dim3(blocks), dim3(256), 0, stream,
                             (const double*)part, (long long)a.part_stride, p.S, (int)p.M,
                             (long long)lo_ld, width_ptr, width, out, (long long)ldo));
  }
  return kOk;
}

// ------------------------------------------------- dimension-tree partials --
// Second half of a dimension-tree MTTKRP: the partial P (one tensor mode
// already contracted on the tensor cores) is contracted with one more factor
// column-wise.  Thread per (row, c), c fastest -> coalesced 8-byte loads of P
// and F; the reduction runs in ascending index order (deterministic,
// column-local, so position independence is preserved).
__global__ void partial_ttv_kernel(const double* __restrict__ P, long long ld, long long Da,
                                   long long Db, int reduce_b, long long La,
                                   const double* __restrict__ F, long long ldf,
                                   const int* width_ptr, int width, long long rows_out,
                                   double* __restrict__ out, long long ldo) {
  griddep_wait();  // launched with PDL (launch_dep): predecessors complete
  griddep_launch_dependents();  // the next kernel may start its prologue
  const int W = width_ptr ? *width_ptr : width;
  const long long n = (reduce_b ? rows_out : (rows_out + 3) / 4) * W;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / W;
    const int c = int(e % W);
    const double* p;
    const double* f = F + c;
    long long pstep, L;
    if (reduce_b) {  // out[a] = sum_b P[a + Da b] F[b]
      p = P + row * ld + c;
      pstep = Da * ld;
      L = Db;
    } else {         // out[b] = sum_a P[a + Da b] F[a]
      p = P + row * Da * ld + c;
      pstep = ld;
      L = La;
    }
    if (!reduce_b) {
      // 4 output rows per thread share each F[a][c] load
      const long long r4 = row * 4;
      if (r4 >= rows_out) continue;
      const int nr = (int)min(4LL, rows_out - r4);
      const double* p4 = P + r4 * Da * ld + c;
      // rows past the end alias the last valid row (loaded, never stored)
      const long long rs1 = (nr > 1 ? 1 : 0) * Da * ld, rs2 = (nr > 2 ? 2 : nr - 1) * Da * ld,
                      rs3 = (nr > 3 ? 3 : nr - 1) * Da * ld;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      long long a = 0;
      for (; a + 4 <= L; a += 4) {
        double fv[4], pv[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          fv[u] = __ldg(f + (a + u) * ldf);
          const double* pa = p4 + (a + u) * ld;
          pv[u][0] = __ldg(pa);
          pv[u][1] = __ldg(pa + rs1);
          pv[u][2] = __ldg(pa + rs2);
          pv[u][3] = __ldg(pa + rs3);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a0 = fma(pv[u][0], fv[u], a0);
          a1 = fma(pv[u][1], fv[u], a1);
          a2 = fma(pv[u][2], fv[u], a2);
          a3 = fma(pv[u][3], fv[u], a3);
        }
      }
      for (; a < L; ++a) {
        const double fa = __ldg(f + a * ldf);
        const double* pa = p4 + a * ld;
        a0 = fma(__ldg(pa), fa, a0);
        a1 = fma(__ldg(pa + rs1), fa, a1);
        a2 = fma(__ldg(pa + rs2), fa, a2);
        a3 = fma(__ldg(pa + rs3), fa, a3);
      }
      double* o = out + r4 * ldo + c;
      o[0] = a0;
      if (nr > 1) o[ldo] = a1;
      if (nr > 2) o[2 * ldo] = a2;
      if (nr > 3) o[3 * ldo] = a3;
      continue;
    }
    double acc = 0.0;
    long long i = 0;
    for (; i + 4 <= L; i += 4) {
      const double p0 = __ldg(p + (i + 0) * pstep), p1 = __ldg(p + (i + 1) * pstep);
      const double p2 = __ldg(p + (i + 2) * pstep), p3 = __ldg(p + (i + 3) * pstep);
      const double f0 = __ldg(f + (i + 0) * ldf), f1 = __ldg(f + (i + 1) * ldf);
      const double f2 = __ldg(f + (i + 2) * ldf), f3 = __ldg(f + (i + 3) * ldf);
      acc = fma(p0, f0, acc);
      acc = fma(p1, f1, acc);
      acc = fma(p2, f2, acc);
      acc = fma(p3, f3, acc);
    }
    for (; i < L; ++i) acc = fma(__ldg(p + i * pstep), __ldg(f + i * ldf), acc);
    out[row * ldo + c] = acc;
  }
}

// The same contraction (out[b] = sum_a P[a + Da b] F[a], 4 output rows per
// thread) for partials with few output rows and a long a-range (c3's Z tree:
// 21 rows, a over 251): the a-range is cut into G chunks (threadIdx.y), each
// summed in ascending order, and the chunk sums are added in chunk order
// through shared memory -- deterministic and per column, so position
// independent.  Without the split only rows/4 x W threads exist (1800 at c3).
__global__ void __launch_bounds__(512) partial_ttv_split_kernel(const double* __restrict__ P, long long ld, long long Da,
                                         long long La, const double* __restrict__ F,
                                         long long ldf, const int* width_ptr, int width,
                                         long long rows_out, double* __restrict__ out,
                                         long long ldo) {
  griddep_wait();  // launched with PDL (launch_dep): predecessors complete
  griddep_launch_dependents();  // the next kernel may start its prologue
  extern __shared__ double red[];  // [G][4][32]
  const int W = width_ptr ? *width_ptr : width;
  if ((int)blockIdx.x * 32 >= W) return;  // block-uniform
  const int G = blockDim.y, tx = threadIdx.x, ty = threadIdx.y;
  const int c = blockIdx.x * 32 + tx;
  const long long r4 = (long long)blockIdx.y * 4;
  const int nr = (int)min(4LL, rows_out - r4);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (c < W) {
    const double* p4 = P + r4 * Da * ld + c;
    const double* f = F + c;
    const long long rs1 = (nr > 1 ? 1 : 0) * Da * ld, rs2 = (nr > 2 ? 2 : nr - 1) * Da * ld,
                    rs3 = (nr > 3 ? 3 : nr - 1) * Da * ld;
    const long long a_lo = La * ty / G, a_hi = La * (ty + 1) / G;
    long long a = a_lo;
    for (; a + 4 <= a_hi; a += 4) {
      double fv[4], pv[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        fv[u] = __ldg(f + (a + u) * ldf);
        const double* pa = p4 + (a + u) * ld;
        pv[u][0] = __ldg(pa);
        pv[u][1] = __ldg(pa + rs1);
        pv[u][2] = __ldg(pa + rs2);
        pv[u][3] = __ldg(pa + rs3);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a0 = fma(pv[u][0], fv[u], a0);
        a1 = fma(pv[u][1], fv[u], a1);
        a2 = fma(pv[u][2], fv[u], a2);
        a3 = fma(pv[u][3], fv[u], a3);
      }
    }
    for (; a < a_hi; ++a) {
      const double fa = __ldg(f + a * ldf);
      const double* pa = p4 + a * ld;
      a0 = fma(__ldg(pa), fa, a0);
      a1 = fma(__ldg(pa + rs1), fa, a1);
      a2 = fma(__ldg(pa + rs2), fa, a2);
      a3 = fma(__ldg(pa + rs3), fa, a3);
    }
  }
  double* rd = red + (size_t)ty * 128 + tx;
  rd[0] = a0;
  rd[32] = a1;
  rd[64] = a2;
  rd[96] = a3;
  __syncthreads();
  if (ty == 0 && c < W) {
    double s0 = a0, s1 = a1, s2 = a2, s3 = a3;
    for (int g = 1; g < G; ++g) {
      const double* q = red + (size_t)g * 128 + tx;
      s0 += q[0];
      s1 += q[32];
      s2 += q[64];
      s3 += q[96];
    }
    double* o = out + r4 * ldo + c;
    o[0] = s0;
    if (nr > 1) o[ldo] = s1;
    if (nr > 2) o[2 * ldo] = s2;
    if (nr > 3) o[3 * ldo] = s3;
  }
}

int launch_partial_ttv(const double* P, long long ld, long long Da, long long Db, int reduce_b,
                       long long La, const double* F, long long ldf, int width,
                       const int* width_ptr, long long cap, long long rows_out, double* out,
                       long long ldo, int sms, cudaStream_t stream) {
  const long long n = rows_out * cap;
  if (!reduce_b) {
    const long long threads = (rows_out + 3) / 4 * cap;
    const long long G = std::min<long long>({16, 65536 / std::max<long long>(1, threads), La / 8});
    if (G >= 2) {
      const dim3 grid((unsigned)((cap + 31) / 32), (unsigned)((rows_out + 3) / 4));
      CALS_CUDA_TRY(launch_dep(partial_ttv_split_kernel, grid, dim3(32, (unsigned)G),
                               size_t(G) * 128 * 8, stream, P, ld, Da, La, F, ldf, width_ptr,
                               width, rows_out, out, ldo));
      return kOk;
    }
  }
  const int blocks = (int)std::max<long long>(1, std::min<long long>(sms * 16, (n + 255) / 256));
  CALS_CUDA_TRY(launch_dep(partial_ttv_kernel, dim3(blocks), dim3(256), 0, stream, P, ld, Da, Db,
                           reduce_b, La, F, ldf, width_ptr, width, rows_out, out, ldo));
  return kOk;
}

}  // namespace cals

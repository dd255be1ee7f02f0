// K1-K4: the mixed-precision step kernels of mpx_b200 (sm_100a).
//
//   K1 mpx_cast            cast_tree / cast_to_* / LossScaling.scale
//                          (precision.py:53-85, 134-143; dtypes.py:100-123)
//   K2 mpx_unscale_finite  LossScaling.unscale + all_finite
//                          (precision.py:145-154; tree.py:125-131)
//   K3 mpx_scaling_adjust  LossScaling.adjust (precision.py:156-173)
//   K4 mpx_optimizer_step  optimizer_update / compute_updates (optim.py:58-113)
//
// All four are multi-tensor-apply kernels: the host packs a table of leaves
// (pointer, size, first tile) into the kernel's parameter block (up to 32 KB
// on sm_70+ with CUDA >= 12.1), so there is no device-side table, no H2D copy
// and one launch per (up to kMaxLeaves) leaves.  Blocks walk 2048-element tiles
// grid-stride over the whole table; a tile never straddles two leaves.  These
// are HBM-streaming kernels: no shared memory, 16-byte (f32) / 8-byte (half)
// vector accesses, grid sized to resident-blocks x SM count.
#include "mpx_common.cuh"

#include <cudaTypedefs.h>

#include <atomic>
#include <cstdlib>

#include <algorithm>
#include <mutex>
#include <tuple>
#include <vector>

namespace mpx {

thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool pdl_enabled() {
  static const bool on = !(getenv("MPX_PDL") && getenv("MPX_PDL")[0] == '0');
  return on;
}
bool pdl_all() {
  static const bool on = getenv("MPX_PDL_ALL") && getenv("MPX_PDL_ALL")[0] == '1';
  return on;
}

cudaError_t ensure_smem_attr(const void* fn, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::vector<std::tuple<const void*, int, int>> done;  // (kernel, device, bytes)
  std::lock_guard<std::mutex> lock(mu);
  for (auto& t : done)
    if (std::get<0>(t) == fn && std::get<1>(t) == dev && std::get<2>(t) >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.emplace_back(fn, dev, bytes);
  return e;
}

// the whole 32-bit flag word set on the stream (cuMemsetD32Async): a byte
// memset would leave whatever the upper bytes held, which a MIN all-reduce or
// an `== 1` test reads (a freshly allocated flag is uninitialised)
cudaError_t set_flag_word(uint32_t* d_flag, uint32_t value, cudaStream_t st) {
  static PFN_cuMemsetD32Async_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuMemsetD32Async", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemsetD32Async_v3020>(p);
  });
  if (!fn) return cudaErrorNotSupported;
  return fn((CUdeviceptr)d_flag, value, 1, (CUstream)st) == CUDA_SUCCESS ? cudaSuccess : cudaErrorUnknown;
}

int current_num_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  static int cached[64] = {0};
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}

// resident blocks per SM, cached per kernel instance (keyed by its address)
static int blocks_per_sm(const void* fn) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : cache)
    if (e.first == fn) return e.second;
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kThreads, 0) != cudaSuccess || b < 1) {
    cudaGetLastError();
    b = 4;
  }
  cache.emplace_back(fn, b);
  return b;
}

// streaming grids.  A one-wave grid-stride (persistent) launch streams HBM at
// ~5.95 TB/s, a grid of a few tiles per block at the 6.55 TB/s copy peak
// (tools/hbm_streams.cu; K4 at ViT-B size: 5.84 -> 6.36 TB/s with ~3 tiles per
// block, 12 waves of resident blocks — 1 tile per block is slow again, the
// per-block setup no longer amortized).  MPX_STREAM_WAVES=k forces k waves.
static int stream_waves() {
  static const int w = getenv("MPX_STREAM_WAVES") ? std::max(1, atoi(getenv("MPX_STREAM_WAVES"))) : 0;
  return w;
}
template <class K>
static int grid_for(K kernel, int64_t n_tiles) {
  const int64_t resident = (int64_t)current_num_sms() * blocks_per_sm(reinterpret_cast<const void*>(kernel));
  int64_t g = stream_waves() ? resident * stream_waves() : std::max(resident, n_tiles / 3);
  if (n_tiles < g) g = n_tiles;
  return (int)std::max<int64_t>(g, 1);
}

constexpr int kMaxLeaves = 160;

// binary search: the leaf whose tile range contains `tile`
template <class P>
__device__ __forceinline__ int find_leaf(const P& p, int64_t tile) {
  int lo = 0, hi = p.n_leaves - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p.leaf[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// ===========================================================================
// K1 — cast / scale
// ===========================================================================
struct CastLeaf {
  const void* src;
  void* dst;
  int64_t n;
  int64_t tile_begin;
};
struct CastParams {
  int n_leaves;
  int64_t n_tiles;
  double scale;
  const double* d_scale;
  CastLeaf leaf[kMaxLeaves];
};

template <int SRC, int DST, bool SCALE>
__global__ void __launch_bounds__(kThreads) cast_kernel(const __grid_constant__ CastParams P) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  float s = 1.f;
  if (SCALE) s = __double2float_rn(P.d_scale ? *P.d_scale : P.scale);
  for (int64_t tile = blockIdx.x; tile < P.n_tiles; tile += gridDim.x) {
    const int li = find_leaf(P, tile);
    const CastLeaf& L = P.leaf[li];
    const int64_t off = (tile - L.tile_begin) * kTile;
    const int64_t cnt = min((int64_t)kTile, L.n - off);
    if (cnt == kTile && aligned16(L.src) && aligned16(L.dst)) {
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        const int64_t i = off + g * kGroupStride + threadIdx.x * kVec;
        float x[4];
        Vec4<SRC>::load_cs(L.src, i, x);
#pragma unroll
        for (int k = 0; k < 4; ++k) x[k] = SCALE ? __fmul_rn(x[k], s) : x[k];
        Vec4<DST>::store(L.dst, i, x);
      }
    } else {
      for (int64_t i = off + threadIdx.x; i < off + cnt; i += kThreads) {
        float x = load1<SRC>(L.src, i);
        store1<DST>(L.dst, i, SCALE ? __fmul_rn(x, s) : x);
      }
    }
  }
}

template <int SRC, int DST, bool SCALE>
static int launch_cast(const CastParams& P, cudaStream_t st) {
  auto k = cast_kernel<SRC, DST, SCALE>;
  MPX_CUDA_CHECK(::mpx::launch_pdl(k, grid_for(k, P.n_tiles), kThreads, 0, st, P));
  MPX_LAUNCH_CHECK("cast_kernel");
  return 0;
}

template <int SRC, int DST>
static int dispatch_cast3(const CastParams& P, bool scale, cudaStream_t st) {
  return scale ? launch_cast<SRC, DST, true>(P, st) : launch_cast<SRC, DST, false>(P, st);
}
template <int SRC>
static int dispatch_cast2(const CastParams& P, int dst, bool scale, cudaStream_t st) {
  switch (dst) {
    case MPX_F32: return dispatch_cast3<SRC, MPX_F32>(P, scale, st);
    case MPX_F16: return dispatch_cast3<SRC, MPX_F16>(P, scale, st);
    case MPX_BF16: return dispatch_cast3<SRC, MPX_BF16>(P, scale, st);
  }
  return fail(MPX_EINVAL, "mpx_cast: bad dst dtype");
}

// ===========================================================================
// K2 — unscale + finite flag
// ===========================================================================
struct UnscaleLeaf {
  const void* g;
  float* out;
  int64_t n;
  int64_t tile_begin;
};
struct UnscaleParams {
  int n_leaves;
  int64_t n_tiles;
  double scale;
  const double* d_scale;
  uint32_t* flag;
  UnscaleLeaf leaf[kMaxLeaves];
};

// Non-finite test on the raw encoding (exponent all ones).
template <int DT> __device__ __forceinline__ bool raw_nonfinite4(const void* base, int64_t i);
template <> __device__ __forceinline__ bool raw_nonfinite4<MPX_F32>(const void* base, int64_t i) {
  uint4 w = *reinterpret_cast<const uint4*>(static_cast<const float*>(base) + i);
  const uint32_t e = 0x7F800000u;
  return ((w.x & e) == e) | ((w.y & e) == e) | ((w.z & e) == e) | ((w.w & e) == e);
}
template <uint32_t EXP>
__device__ __forceinline__ bool half_pair_nonfinite(uint32_t w) {
  return ((w & EXP) == EXP) | ((w & (EXP << 16)) == (EXP << 16));
}
template <> __device__ __forceinline__ bool raw_nonfinite4<MPX_F16>(const void* base, int64_t i) {
  uint2 w = *reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(base) + i);
  return half_pair_nonfinite<0x7C00u>(w.x) | half_pair_nonfinite<0x7C00u>(w.y);
}
template <> __device__ __forceinline__ bool raw_nonfinite4<MPX_BF16>(const void* base, int64_t i) {
  uint2 w = *reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(base) + i);
  return half_pair_nonfinite<0x7F80u>(w.x) | half_pair_nonfinite<0x7F80u>(w.y);
}

template <int GDT, bool OUT>
__global__ void __launch_bounds__(kThreads) unscale_finite_kernel(const __grid_constant__ UnscaleParams P) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  Divisor d;
  d.init(__double2float_rn(P.d_scale ? *P.d_scale : P.scale));
  // Flag-only with |divisor| >= 1 (including +inf): |x/s| <= |x|, so x/s is
  // finite iff x is; test the raw encoding and skip the arithmetic.
  const bool raw_test = !OUT && d.s >= 1.f;
  bool bad = false;
  for (int64_t tile = blockIdx.x; tile < P.n_tiles; tile += gridDim.x) {
    const int li = find_leaf(P, tile);
    const UnscaleLeaf& L = P.leaf[li];
    const int64_t off = (tile - L.tile_begin) * kTile;
    const int64_t cnt = min((int64_t)kTile, L.n - off);
    const bool write = OUT && L.out != nullptr;
    if (cnt == kTile && aligned16(L.g) && (!write || aligned16(L.out))) {
#pragma unroll
      for (int g = 0; g < kGroups; ++g) {
        const int64_t i = off + g * kGroupStride + threadIdx.x * kVec;
        if (raw_test) {
          bad |= raw_nonfinite4<GDT>(L.g, i);
        } else {
          float x[4];
          Vec4<GDT>::load(L.g, i, x);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            x[k] = d.apply(x[k]);
            bad |= !f32_finite(x[k]);
          }
          if (write) Vec4<MPX_F32>::store(L.out, i, x);
        }
      }
    } else {
      for (int64_t i = off + threadIdx.x; i < off + cnt; i += kThreads) {
        float q = d.apply(load1<GDT>(L.g, i));
        bad |= !f32_finite(q);
        if (write) L.out[i] = q;
      }
    }
  }
  // warp vote + block barrier-reduction (BAR.RED.OR), one plain store per block
  if (__syncthreads_or(bad) && threadIdx.x == 0) *P.flag = 0u;
}

// Flag-only scan of one contiguous half-precision leaf (the gradient arena):
// 4 x 16-byte loads in flight per thread.  |divisor| >= 1: exponent-bits
// test (x/s finite iff x finite); otherwise the quotient is formed exactly as
// the general kernel does (Divisor) and tested.
template <int GDT>
__global__ void __launch_bounds__(kThreads) finite_scan_kernel(const uint16_t* __restrict__ g, int64_t n,
                                                               const double* d_scale, double scale,
                                                               uint32_t* __restrict__ flag) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  constexpr uint32_t EXP = GDT == MPX_F16 ? 0x7C00u : 0x7F80u;
  Divisor d;
  d.init(__double2float_rn(d_scale ? *d_scale : scale));
  const bool raw = d.s >= 1.f;
  const int64_t n16 = n / 8;
  const uint4* v = reinterpret_cast<const uint4*>(g);
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n16; i += 4 * stride) {
    uint4 w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = i + k * stride < n16 ? v[i + k * stride] : make_uint4(0, 0, 0, 0);
    if (raw) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        bad |= half_pair_nonfinite<EXP>(w[k].x) | half_pair_nonfinite<EXP>(w[k].y) |
               half_pair_nonfinite<EXP>(w[k].z) | half_pair_nonfinite<EXP>(w[k].w);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t u[4] = {w[k].x, w[k].y, w[k].z, w[k].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          bad |= !f32_finite(d.apply(to_f32<GDT>((uint16_t)(u[e] & 0xFFFFu))));
          bad |= !f32_finite(d.apply(to_f32<GDT>((uint16_t)(u[e] >> 16))));
        }
      }
    }
  }
  if (blockIdx.x == 0)
    for (int64_t i = n16 * 8 + threadIdx.x; i < n; i += kThreads) bad |= !f32_finite(d.apply(to_f32<GDT>(g[i])));
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 0u;
}

template <int GDT>
static int launch_unscale(const UnscaleParams& P, bool out, cudaStream_t st) {
  if (out) {
    auto k = unscale_finite_kernel<GDT, true>;
    MPX_CUDA_CHECK(::mpx::launch_pdl(k, grid_for(k, P.n_tiles), kThreads, 0, st, P));
  } else {
    auto k = unscale_finite_kernel<GDT, false>;
    MPX_CUDA_CHECK(::mpx::launch_pdl(k, grid_for(k, P.n_tiles), kThreads, 0, st, P));
  }
  MPX_LAUNCH_CHECK("unscale_finite_kernel");
  return 0;
}

// ===========================================================================
// K3 — loss-scale state machine (fp64, exact Python-double semantics)
// ===========================================================================
__global__ void scaling_adjust_kernel(mpx_scaling_state* st, const uint32_t* flag,
                                      int64_t* step_count, double* used_scale) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const double F32_MAX = 3.4028234663852886e38;  // float(np.finfo(np.float32).max)
  const bool finite = *flag != 0u;
  double scale = st->loss_scale;
  int64_t n = st->steps_since_growth;
  if (used_scale) *used_scale = scale;
  if (!finite) {
    scale = __dmul_rn(scale, st->backoff_factor);
    if (scale < st->min_scale) scale = st->min_scale;
    n = 0;
  } else if (n + 1 >= st->growth_interval) {
    const double grown = __dmul_rn(scale, st->growth_factor);
    if (grown <= F32_MAX) scale = grown;
    n = 0;
  } else {
    n = n + 1;
  }
  st->loss_scale = scale;
  st->steps_since_growth = n;
  if (step_count && finite) *step_count += 1;
}

// ===========================================================================
// K4 — gated optimizer step (Adam / SGD), optional half working copy
// ===========================================================================
struct OptLeaf {
  void* p;
  float* m;
  float* v;
  const void* g;
  void* half;
  float* upd;
  int64_t n;
  int64_t tile_begin;
  int32_t p_dtype;
};
struct OptParams {
  int n_leaves;
  int64_t n_tiles;
  mpx_adam_hparams hp;
  const float* bc_table;
  int64_t bc_len;
  int64_t* counter;  // {step_count, blocks-done scratch}
  int increment;     // last launch of the call: bump step_count when done
  double scale;
  const double* d_scale;
  const uint32_t* flag;
  OptLeaf leaf[kMaxLeaves];
};

struct AdamConsts {
  float b1, omb1, b2, omb2, lr, eps, neg_lr, neg_lr_wd, bc1, bc2;
};

// One element of the reference update, every operator one correctly rounded
// f32 op in the reference's order (optim.py:78-97, 106-111):
//   m' = m*b1 + g*(1-b1);  v' = v*b2 + (g*g)*(1-b2)
//   u  = -((m'/bc1)*lr / (sqrt(v'/bc2) + eps))        [Adam]
//   u  = g * (-lr)                                    [SGD]
//   p' = q(p + u, p.dtype)   (+ p*(-lr*wd) when wd != 0, AdamW extension)
template <int MODE>
__device__ __forceinline__ float opt_elem(float g, float p, float& m, float& v, const AdamConsts& c,
                                          float& u_out) {
  float u;
  if (MODE == 0) {
    m = __fadd_rn(__fmul_rn(m, c.b1), __fmul_rn(g, c.omb1));
    v = __fadd_rn(__fmul_rn(v, c.b2), __fmul_rn(__fmul_rn(g, g), c.omb2));
    const float mh = __fdiv_rn(m, c.bc1);
    const float vh = __fdiv_rn(v, c.bc2);
    u = -__fdiv_rn(__fmul_rn(mh, c.lr), __fadd_rn(__fsqrt_rn(vh), c.eps));
  } else {
    u = __fmul_rn(g, c.neg_lr);
  }
  u_out = u;
  float pn = __fadd_rn(p, u);
  if (c.neg_lr_wd != 0.f) pn = __fadd_rn(pn, __fmul_rn(p, c.neg_lr_wd));
  return pn;
}

template <int GDT, int PDT, int HDT, int MODE>
__device__ __forceinline__ void opt_tile(const OptLeaf& L, int64_t off, int64_t cnt, const Divisor& d,
                                         const AdamConsts& c) {
  const bool has_half = HDT >= 0 && L.half != nullptr;
  const bool upd_only = L.upd != nullptr;
  const bool vec = cnt == kTile && aligned16(L.p) && aligned16(L.g) &&
                   (MODE != 0 || (aligned16(L.m) && aligned16(L.v))) &&
                   (!has_half || aligned16(L.half)) && (!upd_only || aligned16(L.upd));
  if (vec) {
    // issue every load of the tile before any arithmetic (2 groups x 4 streams)
    float g[kGroups][4], p[kGroups][4], m[kGroups][4], v[kGroups][4];
#pragma unroll
    for (int k = 0; k < kGroups; ++k) {
      const int64_t i = off + k * kGroupStride + threadIdx.x * kVec;
      Vec4<GDT>::load_cs(L.g, i, g[k]);
      Vec4<PDT>::load_cs(L.p, i, p[k]);
      if (MODE == 0) {
        Vec4<MPX_F32>::load_cs(L.m, i, m[k]);
        Vec4<MPX_F32>::load_cs(L.v, i, v[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < kGroups; ++k) {
      const int64_t i = off + k * kGroupStride + threadIdx.x * kVec;
      float pn[4], u[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float gg = GDT == MPX_F32 ? g[k][e] : d.apply(g[k][e]);
        pn[e] = quantize_f32<PDT>(opt_elem<MODE>(gg, p[k][e], m[k][e], v[k][e], c, u[e]));
      }
      if (MODE == 0) {
        Vec4<MPX_F32>::store_cs(L.m, i, m[k]);
        Vec4<MPX_F32>::store_cs(L.v, i, v[k]);
      }
      if (upd_only) {
        Vec4<MPX_F32>::store_cs(L.upd, i, u);
      } else {
        Vec4<PDT>::store_cs(L.p, i, pn);
        if (HDT >= 0 && has_half) Vec4<(HDT >= 0 ? HDT : MPX_F16)>::store_cs(L.half, i, pn);
      }
    }
  } else {
    for (int64_t i = off + threadIdx.x; i < off + cnt; i += kThreads) {
      const float graw = load1<GDT>(L.g, i);
      const float gg = GDT == MPX_F32 ? graw : d.apply(graw);
      float mm = MODE == 0 ? L.m[i] : 0.f, vv = MODE == 0 ? L.v[i] : 0.f, u;
      const float pn = quantize_f32<PDT>(opt_elem<MODE>(gg, load1<PDT>(L.p, i), mm, vv, c, u));
      if (MODE == 0) {
        L.m[i] = mm;
        L.v[i] = vv;
      }
      if (upd_only) {
        L.upd[i] = u;
      } else {
        store1<PDT>(L.p, i, pn);
        if (HDT >= 0 && has_half) store1<(HDT >= 0 ? HDT : MPX_F16)>(L.half, i, pn);
      }
    }
  }
}

// Tiles are walked last-to-first: K2 has just streamed the gradients
// first-to-last, so the tail of the gradient arena is still L2-resident.
template <int GDT, int HDT, int MODE>
__global__ void __launch_bounds__(kThreads) optimizer_kernel(const __grid_constant__ OptParams P) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  if (P.flag != nullptr && *P.flag == 0u) return;  // gate: skipped step leaves everything bit-identical
  Divisor d;
  d.init(__double2float_rn(P.d_scale ? *P.d_scale : P.scale));
  AdamConsts c;
  c.b1 = P.hp.b1; c.omb1 = P.hp.omb1; c.b2 = P.hp.b2; c.omb2 = P.hp.omb2;
  c.lr = P.hp.lr; c.eps = P.hp.eps; c.neg_lr = P.hp.neg_lr; c.neg_lr_wd = P.hp.neg_lr_wd;
  c.bc1 = 1.f; c.bc2 = 1.f;
  if (MODE == 0) {
    int64_t t = (P.counter ? P.counter[0] : 0) + 1;
    if (t > P.bc_len) t = P.bc_len;
    c.bc1 = P.bc_table[2 * (t - 1)];
    c.bc2 = P.bc_table[2 * (t - 1) + 1];
  }
  for (int64_t it = blockIdx.x; it < P.n_tiles; it += gridDim.x) {
    const int64_t tile = P.n_tiles - 1 - it;
    const int li = find_leaf(P, tile);
    const OptLeaf& L = P.leaf[li];
    const int64_t off = (tile - L.tile_begin) * kTile;
    const int64_t cnt = min((int64_t)kTile, L.n - off);
    switch (L.p_dtype) {
      case MPX_F32: opt_tile<GDT, MPX_F32, HDT, MODE>(L, off, cnt, d, c); break;
      case MPX_F16: opt_tile<GDT, MPX_F16, HDT, MODE>(L, off, cnt, d, c); break;
      default: opt_tile<GDT, MPX_BF16, HDT, MODE>(L, off, cnt, d, c); break;
    }
  }
  // last block to finish advances the step counter (every block has read it
  // above before it can arrive here), then rearms the scratch word
  if (P.increment && P.counter) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      unsigned long long* done = reinterpret_cast<unsigned long long*>(P.counter + 1);
      if (atomicAdd(done, 1ull) == (unsigned long long)gridDim.x - 1ull) {
        P.counter[0] += 1;
        *done = 0ull;
      }
    }
  }
}

template <int GDT, int HDT, int MODE>
static int launch_opt3(const OptParams& P, cudaStream_t st) {
  auto k = optimizer_kernel<GDT, HDT, MODE>;
  MPX_CUDA_CHECK(::mpx::launch_pdl(k, grid_for(k, P.n_tiles), kThreads, 0, st, P));
  MPX_LAUNCH_CHECK("optimizer_kernel");
  return 0;
}
template <int GDT, int HDT>
static int launch_opt2(const OptParams& P, int mode, cudaStream_t st) {
  return mode == 0 ? launch_opt3<GDT, HDT, 0>(P, st) : launch_opt3<GDT, HDT, 1>(P, st);
}
template <int GDT>
static int launch_opt1(const OptParams& P, int hdt, int mode, cudaStream_t st) {
  switch (hdt) {
    case MPX_F16: return launch_opt2<GDT, MPX_F16>(P, mode, st);
    case MPX_BF16: return launch_opt2<GDT, MPX_BF16>(P, mode, st);
    default: return launch_opt2<GDT, -1>(P, mode, st);
  }
}

static bool valid_dtype(int dt) { return dt == MPX_F32 || dt == MPX_F16 || dt == MPX_BF16; }
static int64_t tiles_of(int64_t n) { return (n + kTile - 1) / kTile; }

}  // namespace mpx

using namespace mpx;

extern "C" {

int64_t mpx_launch_count(void) { return mpx::g_launches.load(std::memory_order_relaxed); }

const char* mpx_last_error(void) { return g_last_error.c_str(); }
int mpx_version(void) { return 1; }
int mpx_num_sms(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}

int mpx_cast(const void* const* h_src, void* const* h_dst, const int64_t* h_numel, int n_leaves,
             int src_dtype, int dst_dtype, double scale, const double* d_scale, void* stream) {
  if (!valid_dtype(src_dtype) || !valid_dtype(dst_dtype)) return fail(MPX_EINVAL, "mpx_cast: bad dtype");
  if (n_leaves < 0) return fail(MPX_EINVAL, "mpx_cast: n_leaves < 0");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool do_scale = d_scale != nullptr || scale != 1.0;
  int i = 0;
  while (i < n_leaves) {
    CastParams P;
    P.n_leaves = 0;
    P.n_tiles = 0;
    P.scale = scale;
    P.d_scale = d_scale;
    for (; i < n_leaves && P.n_leaves < kMaxLeaves; ++i) {
      if (h_numel[i] <= 0) continue;
      if (!h_src[i] || !h_dst[i]) return fail(MPX_EINVAL, "mpx_cast: null leaf pointer");
      CastLeaf& L = P.leaf[P.n_leaves++];
      L.src = h_src[i];
      L.dst = h_dst[i];
      L.n = h_numel[i];
      L.tile_begin = P.n_tiles;
      P.n_tiles += tiles_of(L.n);
    }
    if (P.n_leaves == 0) continue;
    int rc;
    switch (src_dtype) {
      case MPX_F32: rc = dispatch_cast2<MPX_F32>(P, dst_dtype, do_scale, st); break;
      case MPX_F16: rc = dispatch_cast2<MPX_F16>(P, dst_dtype, do_scale, st); break;
      default: rc = dispatch_cast2<MPX_BF16>(P, dst_dtype, do_scale, st); break;
    }
    if (rc) return rc;
  }
  return 0;
}

int mpx_unscale_finite(const void* const* h_g, float* const* h_out, const int64_t* h_numel, int n_leaves,
                       int g_dtype, double scale, const double* d_scale, uint32_t* d_flag, int reset_flag,
                       void* stream) {
  if (!valid_dtype(g_dtype)) return fail(MPX_EINVAL, "mpx_unscale_finite: bad dtype");
  if (!d_flag) return fail(MPX_EINVAL, "mpx_unscale_finite: null flag");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (reset_flag) MPX_CUDA_CHECK(set_flag_word(d_flag, 1u, st));
  // fast path: one contiguous half leaf, flag only (the gradient arena)
  if (n_leaves == 1 && (!h_out || !h_out[0]) && g_dtype != MPX_F32 && h_numel[0] > 0 &&
      (reinterpret_cast<uintptr_t>(h_g[0]) % 16) == 0) {
    const int64_t n = h_numel[0];
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((n / 8 + 4 * kThreads - 1) / (4 * kThreads), (int64_t)current_num_sms() * 8));
    if (g_dtype == MPX_F16)
      MPX_CUDA_CHECK(::mpx::launch_pdl(finite_scan_kernel<MPX_F16>, grid, kThreads, 0, st, static_cast<const uint16_t*>(h_g[0]), n, d_scale, scale,
                                                              d_flag));
    else
      MPX_CUDA_CHECK(::mpx::launch_pdl(finite_scan_kernel<MPX_BF16>, grid, kThreads, 0, st, static_cast<const uint16_t*>(h_g[0]), n, d_scale, scale,
                                                               d_flag));
    MPX_LAUNCH_CHECK("finite_scan_kernel");
    return 0;
  }
  int i = 0;
  while (i < n_leaves) {
    UnscaleParams P;
    P.n_leaves = 0;
    P.n_tiles = 0;
    P.scale = scale;
    P.d_scale = d_scale;
    P.flag = d_flag;
    bool any_out = false;
    for (; i < n_leaves && P.n_leaves < kMaxLeaves; ++i) {
      if (h_numel[i] <= 0) continue;
      if (!h_g[i]) return fail(MPX_EINVAL, "mpx_unscale_finite: null leaf pointer");
      UnscaleLeaf& L = P.leaf[P.n_leaves++];
      L.g = h_g[i];
      L.out = h_out ? h_out[i] : nullptr;
      any_out |= L.out != nullptr;
      L.n = h_numel[i];
      L.tile_begin = P.n_tiles;
      P.n_tiles += tiles_of(L.n);
    }
    if (P.n_leaves == 0) continue;
    int rc;
    switch (g_dtype) {
      case MPX_F32: rc = launch_unscale<MPX_F32>(P, any_out, st); break;
      case MPX_F16: rc = launch_unscale<MPX_F16>(P, any_out, st); break;
      default: rc = launch_unscale<MPX_BF16>(P, any_out, st); break;
    }
    if (rc) return rc;
  }
  return 0;
}

int mpx_scaling_adjust(mpx_scaling_state* d_state, const uint32_t* d_flag, int64_t* d_step_count,
                       double* d_used_scale, void* stream) {
  if (!d_state || !d_flag) return fail(MPX_EINVAL, "mpx_scaling_adjust: null pointer");
  MPX_CUDA_CHECK(::mpx::launch_pdl(scaling_adjust_kernel, 1, 1, 0, static_cast<cudaStream_t>(stream), d_state, d_flag, d_step_count,
                                                                       d_used_scale));
  MPX_LAUNCH_CHECK("scaling_adjust_kernel");
  return 0;
}

int mpx_optimizer_step(void* const* h_p, const int32_t* h_p_dtype, float* const* h_m, float* const* h_v,
                       const void* const* h_g, void* const* h_half, float* const* h_upd,
                       const int64_t* h_numel, int n_leaves, int g_dtype, int half_dtype, int mode,
                       mpx_adam_hparams hp, const float* d_bc_table, int64_t bc_len,
                       int64_t* d_counter, double scale, const double* d_scale,
                       const uint32_t* d_flag, void* stream) {
  if (!valid_dtype(g_dtype)) return fail(MPX_EINVAL, "mpx_optimizer_step: bad grad dtype");
  if (half_dtype >= 0 && half_dtype != MPX_F16 && half_dtype != MPX_BF16)
    return fail(MPX_EINVAL, "mpx_optimizer_step: half dtype must be f16/bf16 or -1");
  if (mode != 0 && mode != 1) return fail(MPX_EINVAL, "mpx_optimizer_step: unknown mode");
  if (mode == 0 && (!d_bc_table || bc_len < 1)) return fail(MPX_EINVAL, "mpx_optimizer_step: no bias table");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int i = 0;
  while (i < n_leaves) {
    OptParams P;
    P.n_leaves = 0;
    P.n_tiles = 0;
    P.hp = hp;
    P.bc_table = d_bc_table;
    P.bc_len = bc_len;
    P.counter = d_counter;
    P.increment = 0;
    P.scale = scale;
    P.d_scale = d_scale;
    P.flag = d_flag;
    for (; i < n_leaves && P.n_leaves < kMaxLeaves; ++i) {
      if (h_numel[i] <= 0) continue;
      if (!valid_dtype(h_p_dtype[i])) return fail(MPX_EINVAL, "mpx_optimizer_step: bad param dtype");
      if (!h_p[i] || !h_g[i] || (mode == 0 && (!h_m[i] || !h_v[i])))
        return fail(MPX_EINVAL, "mpx_optimizer_step: null leaf pointer");
      OptLeaf& L = P.leaf[P.n_leaves++];
      L.p = h_p[i];
      L.m = mode == 0 ? h_m[i] : nullptr;
      L.v = mode == 0 ? h_v[i] : nullptr;
      L.g = h_g[i];
      L.half = h_half ? h_half[i] : nullptr;
      L.upd = h_upd ? h_upd[i] : nullptr;
      L.n = h_numel[i];
      L.tile_begin = P.n_tiles;
      L.p_dtype = h_p_dtype[i];
      P.n_tiles += tiles_of(L.n);
    }
    if (P.n_leaves == 0) continue;
    bool last = true;  // any non-empty leaf left for another launch?
    for (int j = i; j < n_leaves; ++j)
      if (h_numel[j] > 0) { last = false; break; }
    P.increment = last ? 1 : 0;
    int rc;
    switch (g_dtype) {
      case MPX_F32: rc = launch_opt1<MPX_F32>(P, half_dtype, mode, st); break;
      case MPX_F16: rc = launch_opt1<MPX_F16>(P, half_dtype, mode, st); break;
      default: rc = launch_opt1<MPX_BF16>(P, half_dtype, mode, st); break;
    }
    if (rc) return rc;
  }
  return 0;
}

}  // extern "C"

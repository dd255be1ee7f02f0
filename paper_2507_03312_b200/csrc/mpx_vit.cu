// ViT kernels around the GEMMs (sm_100a): the MPX full-precision islands
// (LayerNorm, attention softmax, cross-entropy, mean-pool: f32 inside, half
// at the boundary — precision.py:106-114 force_full_precision), patchify and
// the reductions that produce bias / LayerNorm / position gradients.
//
//   K6 softmax fwd/bwd   tensors.py:431-446, autodiff.py:233-240 (island, bench.py:196-197)
//   K7 layernorm fwd/bwd tensors.py:459-491, autodiff.py:243-262 (island, bench.py:185-187)
//   K9 cross-entropy     tensors.py:494-522, autodiff.py:265-276
//   colsum               _unbroadcast / reduce-sum backward (autodiff.py:88-99, 208-222)
//
// All are HBM-bound row/column sweeps: one warp per row for row ops (16-byte
// loads when D % 256 == 0), deterministic two-pass column reductions (no
// float atomics, so reruns are bit-identical).
#include "mpx_common.cuh"

#include <cstdlib>
#include <mutex>

namespace mpx {

__device__ __forceinline__ float ld_h(const void* p, long long i, int fmt) {
  const uint16_t h = static_cast<const uint16_t*>(p)[i];
  return fmt ? to_f32<MPX_BF16>(h) : to_f32<MPX_F16>(h);
}
__device__ __forceinline__ void st_h(void* p, long long i, float x, int fmt) {
  static_cast<uint16_t*>(p)[i] = fmt ? from_f32<MPX_BF16>(x) : from_f32<MPX_F16>(x);
}
__device__ __forceinline__ void unpack8(uint4 w, float* o, int fmt) {
  const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint16_t lo = (uint16_t)(u[i] & 0xFFFF), hi = (uint16_t)(u[i] >> 16);
    o[2 * i] = fmt ? to_f32<MPX_BF16>(lo) : to_f32<MPX_F16>(lo);
    o[2 * i + 1] = fmt ? to_f32<MPX_BF16>(hi) : to_f32<MPX_F16>(hi);
  }
}
__device__ __forceinline__ uint4 pack8(const float* x, int fmt) {
  return make_uint4(pack2_fmt(x[0], x[1], fmt), pack2_fmt(x[2], x[3], fmt), pack2_fmt(x[4], x[5], fmt),
                    pack2_fmt(x[6], x[7], fmt));
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ===========================================================================
// K7 LayerNorm forward: y = (x - mean) * rstd * g + b over the last dim (f32)
// ===========================================================================
// V = 16-byte vectors per lane (D = 256 * V); V = 0: generic.  FMT (0 f16, 1
// bf16) is a template parameter so only one conversion path is compiled.
template <int V, int FMT>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const void* __restrict__ x, long long ldx,
                                                     const void* __restrict__ g, const void* __restrict__ b,
                                                     void* __restrict__ y, long long ldy, float* __restrict__ mean,
                                                     float* __restrict__ rstd, int rows, int D, float eps, int) {
  constexpr int fmt = FMT;
  ::mpx::pdl_wait_only();  // programmatic dependent launch: inputs are final past here
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const void* xr = static_cast<const uint16_t*>(x) + row * ldx;
  if (V > 0) {
    float v[V > 0 ? V : 1][8];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      unpack8(*reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(xr) + (j * 32 + lane) * 8), v[j], fmt);
#pragma unroll
      for (int e = 0; e < 8; ++e) s += v[j][e];
    }
    const float mu = warp_sum(s) / (float)D;
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < V; ++j)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float c = v[j][e] - mu;
        q += c * c;
      }
    const float rs = rsqrtf(warp_sum(q) / (float)D + eps);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int c0 = (j * 32 + lane) * 8;
      float gg[8], bb[8], o[8];
      unpack8(*reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(g) + c0), gg, fmt);
      unpack8(*reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(b) + c0), bb, fmt);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = (v[j][e] - mu) * rs * gg[e] + bb[e];
      *reinterpret_cast<uint4*>(static_cast<uint16_t*>(y) + row * ldy + c0) = pack8(o, fmt);
    }
    if (lane == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
  } else {
    float s = 0.f;
    for (int c = lane; c < D; c += 32) s += ld_h(xr, c, fmt);
    const float mu = warp_sum(s) / (float)D;
    float q = 0.f;
    for (int c = lane; c < D; c += 32) {
      const float d = ld_h(xr, c, fmt) - mu;
      q += d * d;
    }
    const float rs = rsqrtf(warp_sum(q) / (float)D + eps);
    for (int c = lane; c < D; c += 32)
      st_h(y, row * ldy + c, (ld_h(xr, c, fmt) - mu) * rs * ld_h(g, c, fmt) + ld_h(b, c, fmt), fmt);
    if (lane == 0) {
      mean[row] = mu;
      rstd[row] = rs;
    }
  }
}

// ===========================================================================
// K7 LayerNorm backward.  dx = rstd*(dy*g - mean(dy*g) - xhat*mean(dy*g*xhat))
// (+ dres, the residual branch's cotangent); per-block partial column sums of
// dy*xhat (dgain) and dy (dbias) into ws[2][gridDim][D].
// ===========================================================================
__global__ void __launch_bounds__(256) ln_bwd_kernel(const void* __restrict__ x, long long ldx,
                                                     const void* __restrict__ g, const float* __restrict__ mean,
                                                     const float* __restrict__ rstd, const void* __restrict__ dy,
                                                     long long lddy, const void* __restrict__ dres, long long ldres,
                                                     void* __restrict__ dx, long long lddx, float* __restrict__ ws,
                                                     int rows, int D, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  extern __shared__ float sh[];  // [8 warps][2][D]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* my_dg = sh + warp * 2 * D;
  float* my_db = my_dg + D;
  for (int c = lane; c < D; c += 32) {
    my_dg[c] = 0.f;
    my_db[c] = 0.f;
  }
  for (long long row = (long long)blockIdx.x * 8 + warp; row < rows; row += (long long)gridDim.x * 8) {
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
    for (int c = lane; c < D; c += 32) {
      const float xh = (ld_h(x, row * ldx + c, fmt) - mu) * rs;
      const float d = ld_h(dy, row * lddy + c, fmt);
      const float dg = d * ld_h(g, c, fmt);
      s1 += dg;
      s2 += dg * xh;
      my_dg[c] += d * xh;
      my_db[c] += d;
    }
    s1 = warp_sum(s1) / (float)D;
    s2 = warp_sum(s2) / (float)D;
    for (int c = lane; c < D; c += 32) {
      const float xh = (ld_h(x, row * ldx + c, fmt) - mu) * rs;
      const float dg = ld_h(dy, row * lddy + c, fmt) * ld_h(g, c, fmt);
      float o = rs * (dg - s1 - xh * s2);
      if (dres) o += ld_h(dres, row * ldres + c, fmt);
      st_h(dx, row * lddx + c, o, fmt);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    float a = 0.f, bsum = 0.f;
    for (int w = 0; w < 8; ++w) {
      a += sh[w * 2 * D + c];
      bsum += sh[w * 2 * D + D + c];
    }
    ws[(long long)blockIdx.x * D + c] = a;
    ws[(long long)gridDim.x * D + (long long)blockIdx.x * D + c] = bsum;
  }
}

// ===========================================================================
// K7 LayerNorm backward, split for occupancy (v3):
//   ln_dx_kernel        dx = rstd*(dy*g - mean(dy*g) - xhat*mean(dy*g*xhat)) + dres,
//                       one warp per row, 16-byte vectors, no column state
//   ln_colsum_kernel    column partials of dy*xhat (dgain), dy (dbias) and,
//                       optionally, of dx itself (the bias gradient of the layer
//                       that produced the residual stream) — one coalesced pass
// ===========================================================================
template <int V>
__global__ void __launch_bounds__(256) ln_dx_kernel(const void* __restrict__ x, long long ldx,
                                                    const void* __restrict__ g, const float* __restrict__ mean,
                                                    const float* __restrict__ rstd, const void* __restrict__ dy,
                                                    long long lddy, const void* __restrict__ dres, long long ldres,
                                                    void* __restrict__ dx, long long lddx, int rows, int D, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  uint4 wx[V], wd[V], wr[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int c0 = (j * 32 + lane) * 8;
    wx[j] = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + row * ldx + c0);
    wd[j] = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dy) + row * lddy + c0);
    if (dres) wr[j] = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dres) + row * ldres + c0);
  }
  const float mu = mean[row], rs = rstd[row];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int c0 = (j * 32 + lane) * 8;
    float xv[8], dv[8], gg[8];
    unpack8(wx[j], xv, fmt);
    unpack8(wd[j], dv, fmt);
    unpack8(__ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(g) + c0)), gg, fmt);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float dg = dv[e] * gg[e];
      s1 += dg;
      s2 += dg * (xv[e] - mu) * rs;
    }
  }
  s1 = warp_sum(s1) / (float)D;
  s2 = warp_sum(s2) / (float)D;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int c0 = (j * 32 + lane) * 8;
    float xv[8], dv[8], gg[8], rv[8], o[8];
    unpack8(wx[j], xv, fmt);
    unpack8(wd[j], dv, fmt);
    unpack8(__ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(g) + c0)), gg, fmt);
    if (dres) unpack8(wr[j], rv, fmt);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = rs * (dv[e] * gg[e] - s1 - (xv[e] - mu) * rs * s2) + (dres ? rv[e] : 0.f);
    *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dx) + row * lddx + c0) = pack8(o, fmt);
  }
}

// ===========================================================================
// K7 LayerNorm backward, one pass (v5): dx as ln_dx_kernel, and the column
// partials of dy*xhat, dy and the stored (rounded) dx accumulated across the
// rows of each warp in the warp's own shared-memory slab ([sum][j][e][lane]:
// lane-consecutive, conflict-free), which frees the registers for the next
// row's loads to be in flight while this row is reduced (persistent grid,
// 4 warps per block, fixed row assignment).  The block's warps are combined
// in a fixed order; ws layout [3][gridDim.x][D] for partials_reduce3_kernel.
// ===========================================================================
template <int V, int FMT>  // FMT (0 f16, 1 bf16) compiled in: one conversion path
__global__ void __launch_bounds__(128, V >= 4 ? 2 : 4) ln_bwd_fused_kernel(const void* __restrict__ x, long long ldx,
                                                           const void* __restrict__ g, const float* __restrict__ mean,
                                                           const float* __restrict__ rstd, const void* __restrict__ dy,
                                                           long long lddy, const void* __restrict__ dres,
                                                           long long ldres, void* __restrict__ dx, long long lddx,
                                                           float* __restrict__ ws, int rows, int D, int nsum, int) {
  constexpr int fmt = FMT;
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  extern __shared__ float acc_sh[];  // [4 warps][3 sums][V][4 column pairs][32 lanes] float2
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float2* acc = reinterpret_cast<float2*>(acc_sh) + warp * (3 * V * 128);
  auto A = [&](int k, int j, int e2) -> float2& { return acc[((k * V + j) * 4 + e2) * 32 + lane]; };
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int j = 0; j < V; ++j)
#pragma unroll
      for (int e2 = 0; e2 < 4; ++e2) A(k, j, e2) = make_float2(0.f, 0.f);
  const long long stride = (long long)gridDim.x * 4;
  long long row = (long long)blockIdx.x * 4 + warp;
  uint4 nx[V], nd[V], nr[V];  // the next row's words, in flight
  auto load = [&](long long rr) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int c0 = (j * 32 + lane) * 8;
      nx[j] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + rr * ldx + c0));
      nd[j] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dy) + rr * lddy + c0));
      if (dres) nr[j] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dres) + rr * ldres + c0));
    }
  };
  auto f2v = [](float a) { return make_float2(a, a); };
  if (row < rows) load(row);
  for (; row < rows; row += stride) {
    uint4 wx[V], wd[V], wr[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      wx[j] = nx[j];
      wd[j] = nd[j];
      wr[j] = nr[j];
    }
    if (row + stride < rows) load(row + stride);  // next row's bytes in flight during this row's work
    const float mu = mean[row], rs = rstd[row];
    float2 s1 = f2v(0.f), s2 = f2v(0.f);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int c0 = (j * 32 + lane) * 8;
      float xv[8], dv[8], gg[8];
      unpack8(wx[j], xv, fmt);
      unpack8(wd[j], dv, fmt);
      unpack8(__ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(g) + c0)), gg, fmt);
#pragma unroll
      for (int e2 = 0; e2 < 4; ++e2) {
        const float2 xx = make_float2(xv[2 * e2], xv[2 * e2 + 1]), d2 = make_float2(dv[2 * e2], dv[2 * e2 + 1]);
        const float2 xh = __fmul2_rn(__fadd2_rn(xx, f2v(-mu)), f2v(rs));
        const float2 dg = __fmul2_rn(d2, make_float2(gg[2 * e2], gg[2 * e2 + 1]));
        s1 = __fadd2_rn(s1, dg);
        s2 = __ffma2_rn(dg, xh, s2);
        A(0, j, e2) = __ffma2_rn(d2, xh, A(0, j, e2));
        A(1, j, e2) = __fadd2_rn(A(1, j, e2), d2);
      }
    }
    const float m1 = warp_sum(s1.x + s1.y) / (float)D;
    const float m2 = warp_sum(s2.x + s2.y) / (float)D;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int c0 = (j * 32 + lane) * 8;
      float xv[8], dv[8], gg[8], rv[8], o[8];
      unpack8(wx[j], xv, fmt);
      unpack8(wd[j], dv, fmt);
      unpack8(__ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(g) + c0)), gg, fmt);
      if (dres) unpack8(wr[j], rv, fmt);
      // o = rs (dy g - m1 - xhat m2) + dres = a (dy g) + (c x + b) + dres, packed by column pairs
      const float a = rs, c = -rs * rs * m2, bb = -rs * m1 + rs * rs * m2 * mu;
#pragma unroll
      for (int e2 = 0; e2 < 4; ++e2) {
        const float2 t1 = __fmul2_rn(make_float2(dv[2 * e2], dv[2 * e2 + 1]), make_float2(gg[2 * e2], gg[2 * e2 + 1]));
        const float2 t2 = __ffma2_rn(f2v(c), make_float2(xv[2 * e2], xv[2 * e2 + 1]), f2v(bb));
        float2 r2 = __ffma2_rn(f2v(a), t1, t2);
        if (dres) r2 = __fadd2_rn(r2, make_float2(rv[2 * e2], rv[2 * e2 + 1]));
        o[2 * e2] = r2.x;
        o[2 * e2 + 1] = r2.y;
      }
      const uint4 w = pack8(o, fmt);
      *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dx) + row * lddx + c0) = w;
      if (nsum == 3) {
        float ov[8];
        unpack8(w, ov, fmt);  // the column sum of the stored dx
#pragma unroll
        for (int e2 = 0; e2 < 4; ++e2) A(2, j, e2) = __fadd2_rn(A(2, j, e2), make_float2(ov[2 * e2], ov[2 * e2 + 1]));
      }
    }
  }
  __syncthreads();
  // combine the 4 warps' slabs in a fixed order, one partial row per block
  const float* accf = acc_sh;
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    const int j = c / 256, l = (c / 8) % 32, e = c % 8;
    for (int k = 0; k < nsum; ++k) {
      float t = 0.f;
      for (int w = 0; w < 4; ++w) t += accf[(w * (3 * V * 128) + ((k * V + j) * 4 + e / 2) * 32 + l) * 2 + (e & 1)];
      ws[((long long)k * gridDim.x + blockIdx.x) * D + c] = t;
    }
  }
}

// One-pass LayerNorm backward with the column partials in REGISTERS: a warp
// per row, each lane owns 8 V fixed columns for every row it visits, so the
// dgain / dbias (/ colsum dx) partials accumulate in 8 V x NSUM registers
// instead of read-modify-write shared-memory slabs (the slab version spends
// ~2 x NSUM shared-memory ops per element pair; this one none until the
// block's final fixed-order combine).  The gain stays packed in registers;
// x and dy are re-unpacked for the second pass (after the row reductions)
// rather than kept as f32.  Same math and partial layout as
// ln_bwd_fused_kernel ([NSUM][gridDim.x][D] for partials_reduce3_kernel).
template <int V, int FMT, int NSUM>
__global__ void __launch_bounds__(128, 2) ln_bwd_reg_kernel(const void* __restrict__ x, long long ldx,
                                                           const void* __restrict__ g, const float* __restrict__ mean,
                                                           const float* __restrict__ rstd, const void* __restrict__ dy,
                                                           long long lddy, const void* __restrict__ dres,
                                                           long long ldres, void* __restrict__ dx, long long lddx,
                                                           float* __restrict__ ws, int rows, int D) {
  constexpr int fmt = FMT;
  ::mpx::pdl_grid_sync();
  __shared__ float comb[4][NSUM][V * 256];  // per-warp column partials for the block's fixed-order combine
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float ag[V][8], ab[V][8], ax[V][8];
#pragma unroll
  for (int j = 0; j < V; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) ag[j][e] = ab[j][e] = ax[j][e] = 0.f;
  uint4 gw[V];
#pragma unroll
  for (int j = 0; j < V; ++j) gw[j] = __ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(g) + (j * 32 + lane) * 8));
  auto f2v = [](float a) { return make_float2(a, a); };
  const long long stride = (long long)gridDim.x * 4;
  uint4 nx[V], nd[V];  // the next row's x / dy words, in flight during this row's work
  auto load = [&](long long rr) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int c0 = (j * 32 + lane) * 8;
      nx[j] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + rr * ldx + c0));
      nd[j] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dy) + rr * lddy + c0));
    }
  };
  long long row = (long long)blockIdx.x * 4 + warp;
  if (row < rows) load(row);
  for (; row < rows; row += stride) {
    uint4 wx[V], wd[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      wx[j] = nx[j];
      wd[j] = nd[j];
    }
    if (row + stride < rows) load(row + stride);
    const float mu = mean[row], rs = rstd[row];
    float2 s1 = f2v(0.f), s2 = f2v(0.f);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      float xv[8], dv[8], gg[8];
      unpack8(wx[j], xv, fmt);
      unpack8(wd[j], dv, fmt);
      unpack8(gw[j], gg, fmt);
#pragma unroll
      for (int e2 = 0; e2 < 4; ++e2) {
        const float2 d2 = make_float2(dv[2 * e2], dv[2 * e2 + 1]);
        const float2 xh = __fmul2_rn(__fadd2_rn(make_float2(xv[2 * e2], xv[2 * e2 + 1]), f2v(-mu)), f2v(rs));
        const float2 dg = __fmul2_rn(d2, make_float2(gg[2 * e2], gg[2 * e2 + 1]));
        s1 = __fadd2_rn(s1, dg);
        s2 = __ffma2_rn(dg, xh, s2);
        const float2 pg = __ffma2_rn(d2, xh, make_float2(ag[j][2 * e2], ag[j][2 * e2 + 1]));
        const float2 pb = __fadd2_rn(make_float2(ab[j][2 * e2], ab[j][2 * e2 + 1]), d2);
        ag[j][2 * e2] = pg.x;
        ag[j][2 * e2 + 1] = pg.y;
        ab[j][2 * e2] = pb.x;
        ab[j][2 * e2 + 1] = pb.y;
      }
    }
    uint4 wr[V];
    if (dres) {
#pragma unroll
      for (int j = 0; j < V; ++j)
        wr[j] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dres) + row * ldres + (j * 32 + lane) * 8));
    }
    const float m1 = warp_sum(s1.x + s1.y) / (float)D;
    const float m2 = warp_sum(s2.x + s2.y) / (float)D;
    // o = rs (dy g - m1 - xhat m2) + dres = a (dy g) + (c x + b) + dres
    const float a = rs, c = -rs * rs * m2, bb = -rs * m1 + rs * rs * m2 * mu;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int c0 = (j * 32 + lane) * 8;
      float xv[8], dv[8], gg[8], rv[8], o[8];
      unpack8(wx[j], xv, fmt);
      unpack8(wd[j], dv, fmt);
      unpack8(gw[j], gg, fmt);
      if (dres) unpack8(wr[j], rv, fmt);
#pragma unroll
      for (int e2 = 0; e2 < 4; ++e2) {
        const float2 t1 = __fmul2_rn(make_float2(dv[2 * e2], dv[2 * e2 + 1]), make_float2(gg[2 * e2], gg[2 * e2 + 1]));
        const float2 t2 = __ffma2_rn(f2v(c), make_float2(xv[2 * e2], xv[2 * e2 + 1]), f2v(bb));
        float2 r2 = __ffma2_rn(f2v(a), t1, t2);
        if (dres) r2 = __fadd2_rn(r2, make_float2(rv[2 * e2], rv[2 * e2 + 1]));
        o[2 * e2] = r2.x;
        o[2 * e2 + 1] = r2.y;
      }
      const uint4 w = pack8(o, fmt);
      *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dx) + row * lddx + c0) = w;
      if (NSUM == 3) {
        float ov[8];
        unpack8(w, ov, fmt);  // the column sum of the stored dx
#pragma unroll
        for (int e = 0; e < 8; ++e) ax[j][e] += ov[e];
      }
    }
  }
  // fixed-order combine of the 4 warps' partials: one partial row per block
#pragma unroll
  for (int j = 0; j < V; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int col = (j * 32 + lane) * 8 + e;
      comb[warp][0][col] = ag[j][e];
      comb[warp][1][col] = ab[j][e];
      if (NSUM == 3) comb[warp][NSUM - 1][col] = ax[j][e];
    }
  __syncthreads();
  for (int col = threadIdx.x; col < D; col += blockDim.x)
#pragma unroll
    for (int k = 0; k < NSUM; ++k)
      ws[((long long)k * gridDim.x + blockIdx.x) * D + col] =
          ((comb[0][k][col] + comb[1][k][col]) + comb[2][k][col]) + comb[3][k][col];
}

// block = 32 column vectors of 8 (256 columns) x 8 row lanes; ws layout
// [nsum][split][D] with nsum = 2 (dgain, dbias) or 3 (+ colsum(dx))
__global__ void __launch_bounds__(256) ln_colsum_kernel(const void* __restrict__ x, long long ldx,
                                                        const float* __restrict__ mean, const float* __restrict__ rstd,
                                                        const void* __restrict__ dy, long long lddy,
                                                        const void* __restrict__ dx, long long lddx, int rows, int D,
                                                        int rows_per_split, float* __restrict__ ws, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  __shared__ float sh[3][8][257];
  const int cv = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int c0 = blockIdx.x * 256 + cv * 8;
  const int split = blockIdx.y, nsplit = gridDim.y;
  const int r0 = split * rows_per_split, r1 = min(rows, r0 + rows_per_split);
  float ag[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ab[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ax[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const bool live = c0 < D;
  if (live) {
    int r = r0 + rl;
    for (; r + 8 < r1; r += 16) {  // two rows in flight per thread
      uint4 wx[2], wd[2], wo[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const long long rr = r + 8 * j;
        wx[j] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + rr * ldx + c0));
        wd[j] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dy) + rr * lddy + c0));
        if (dx) wo[j] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dx) + rr * lddx + c0));
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float xv[8], dv[8];
        unpack8(wx[j], xv, fmt);
        unpack8(wd[j], dv, fmt);
        const float mu = mean[r + 8 * j], rs = rstd[r + 8 * j];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          ag[e] += dv[e] * (xv[e] - mu) * rs;
          ab[e] += dv[e];
        }
        if (dx) {
          float ov[8];
          unpack8(wo[j], ov, fmt);
#pragma unroll
          for (int e = 0; e < 8; ++e) ax[e] += ov[e];
        }
      }
    }
    for (; r < r1; r += 8) {
      float xv[8], dv[8];
      unpack8(*reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + (long long)r * ldx + c0), xv, fmt);
      unpack8(*reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dy) + (long long)r * lddy + c0), dv, fmt);
      const float mu = mean[r], rs = rstd[r];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        ag[e] += dv[e] * (xv[e] - mu) * rs;
        ab[e] += dv[e];
      }
      if (dx) {
        float ov[8];
        unpack8(*reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dx) + (long long)r * lddx + c0), ov,
                fmt);
#pragma unroll
        for (int e = 0; e < 8; ++e) ax[e] += ov[e];
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    sh[0][rl][cv * 8 + e] = ag[e];
    sh[1][rl][cv * 8 + e] = ab[e];
    sh[2][rl][cv * 8 + e] = ax[e];
  }
  __syncthreads();
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c < D) {
    const int nsum = dx ? 3 : 2;
    for (int k = 0; k < nsum; ++k) {
      float t = 0.f;
      for (int l = 0; l < 8; ++l) t += sh[k][l][threadIdx.x];
      ws[((long long)k * nsplit + split) * D + c] = t;
    }
  }
}

// ws [nsum][nb][D] -> outputs; grid (D/32, nsum), block = 32 columns x 32
// partial lanes, four partial rows in flight per thread, fixed order
__global__ void __launch_bounds__(1024) partials_reduce3_kernel(const float* __restrict__ ws, int nb, int D,
                                                                void* out0, void* out1, void* out2, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  __shared__ float sm[32][33];
  const int cl = threadIdx.x & 31, kl = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cl;
  const int q = blockIdx.y;
  void* out = q == 0 ? out0 : (q == 1 ? out1 : out2);
  float a = 0.f;
  if (c < D) {
    const float* w = ws + (long long)q * nb * D + c;
    int k = kl;
    for (; k + 224 < nb; k += 256) {  // 8 partial rows in flight, summed in row order
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = w[(long long)(k + 32 * u) * D];
#pragma unroll
      for (int u = 0; u < 8; ++u) a += v[u];
    }
    for (; k < nb; k += 32) a += w[(long long)k * D];
  }
  sm[kl][cl] = a;
  __syncthreads();
  if (kl == 0 && c < D && out) {
    float t = 0.f;
    for (int k = 0; k < 32; ++k) t += sm[k][cl];
    st_h(out, c, t, fmt);
  }
}

// sum ws partials over blocks -> half outputs (ws[0..nb) -> out0, ws[nb..2nb) -> out1)
// block = 32 columns x 8 partial lanes (coalesced 128-byte reads), fixed order
__global__ void __launch_bounds__(256) partials_reduce_kernel(const float* __restrict__ ws, int nb, int D, void* out0,
                                                              void* out1, float alpha, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  __shared__ float sa[8][33], sb[8][33];
  const int cl = threadIdx.x & 31, kl = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cl;
  float a = 0.f, b = 0.f;
  if (c < D)
    for (int k = kl; k < nb; k += 8) {
      a += ws[(long long)k * D + c];
      b += ws[(long long)(nb + k) * D + c];
    }
  sa[kl][cl] = a;
  sb[kl][cl] = b;
  __syncthreads();
  if (kl == 0 && c < D) {
    float x = 0.f, y = 0.f;
    for (int k = 0; k < 8; ++k) {
      x += sa[k][cl];
      y += sb[k][cl];
    }
    if (out0) st_h(out0, c, x * alpha, fmt);
    if (out1) st_h(out1, c, y * alpha, fmt);
  }
}

// ===========================================================================
// column sums: out[z][c] = alpha * sum_r x[z][r][c]   (two deterministic passes)
// block = 256 threads = 32 column-vectors of 8 x 8 row lanes
// ===========================================================================
__global__ void __launch_bounds__(256) colsum_partial_kernel(const void* __restrict__ x, long long ldx,
                                                             long long sbx, int rows, int cols, int rows_per_split,
                                                             float* __restrict__ ws, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  __shared__ float sh[8][256];
  const int cv = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int c0 = blockIdx.x * 256 + cv * 8;
  const int split = blockIdx.y, z = blockIdx.z;
  const int r0 = split * rows_per_split, r1 = min(rows, r0 + rows_per_split);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const uint16_t* base = static_cast<const uint16_t*>(x) + (long long)z * sbx;
  const bool vec = (c0 + 8 <= cols) && ((ldx & 7) == 0) && ((sbx & 7) == 0) &&
                   ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  int r = r0 + rl;
  if (vec) {  // four rows in flight per thread (memory-level parallelism), then the tail
    for (; r + 24 < r1; r += 32) {
      uint4 w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = __ldcs(reinterpret_cast<const uint4*>(base + (long long)(r + 8 * j) * ldx + c0));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float v[8];
        unpack8(w[j], v, fmt);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += v[e];
      }
    }
  }
  for (; r < r1; r += 8) {
    if (vec) {
      float v[8];
      unpack8(*reinterpret_cast<const uint4*>(base + (long long)r * ldx + c0), v, fmt);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += v[e];
    } else {
      for (int e = 0; e < 8; ++e)
        if (c0 + e < cols) acc[e] += ld_h(base, (long long)r * ldx + c0 + e, fmt);
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) sh[rl][cv * 8 + e] = acc[e];
  __syncthreads();
  const int c = blockIdx.x * 256 + threadIdx.x;
  if (c < cols) {
    float s = 0.f;
    for (int k = 0; k < 8; ++k) s += sh[k][threadIdx.x];
    ws[((long long)z * gridDim.y + split) * cols + c] = s;
  }
}

// block = 32 columns x 8 split lanes (coalesced), fixed summation order
__global__ void __launch_bounds__(256) colsum_final_kernel(const float* __restrict__ ws, int splits, int cols,
                                                           int batches, void* out, long long ld_out, int out_dtype,
                                                           float alpha) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  __shared__ float sm[8][33];
  const int cl = threadIdx.x & 31, kl = threadIdx.x >> 5;
  const long long i = (long long)blockIdx.x * 32 + cl;  // flat (z, c)
  const long long n = (long long)cols * batches;
  const long long z = i / cols, c = i - z * cols;
  float a = 0.f;
  if (i < n) {
    const float* w = ws + z * splits * cols + c;
    int k = kl;
    for (; k + 24 < splits; k += 32) {  // four partial rows in flight, summed in order
      const float v0 = w[(long long)k * cols], v1 = w[(long long)(k + 8) * cols], v2 = w[(long long)(k + 16) * cols],
                  v3 = w[(long long)(k + 24) * cols];
      a += v0;
      a += v1;
      a += v2;
      a += v3;
    }
    for (; k < splits; k += 8) a += w[(long long)k * cols];
  }
  sm[kl][cl] = a;
  __syncthreads();
  if (kl == 0 && i < n) {
    float s = 0.f;
    for (int k = 0; k < 8; ++k) s += sm[k][cl];
    s *= alpha;
    if (out_dtype == MPX_F32)
      static_cast<float*>(out)[z * ld_out + c] = s;
    else
      st_h(out, z * ld_out + c, s, out_dtype == MPX_BF16 ? 1 : 0);
  }
}

// ===========================================================================
// K6 softmax, short rows (ld <= 256, ld % 8 == 0): R rows per warp, every
// 16-byte load of all R rows issued before any arithmetic (memory-level
// parallelism), one lane per 8-column chunk.
// ===========================================================================
template <int R>
__global__ void __launch_bounds__(256) softmax_fwd_rows_kernel(const void* __restrict__ S, void* __restrict__ P,
                                                               long long rows, int L, long long ld, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int lane = threadIdx.x & 31;
  const long long row0 = ((long long)blockIdx.x * 8 + (threadIdx.x >> 5)) * R;
  const int c0 = lane * 8;
  const bool act = c0 < ld;
  uint4 w[R];
#pragma unroll
  for (int k = 0; k < R; ++k)
    w[k] = (act && row0 + k < rows) ? *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(S) + (row0 + k) * ld + c0)
                                    : make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (row0 + k >= rows) break;
    float v[8];
    unpack8(w[k], v, fmt);
    float m = -INFINITY;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (!act || c0 + e >= L) v[e] = -INFINITY;
      m = fmaxf(m, v[e]);
    }
    m = warp_max(m);
    float sum = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v[e] = v[e] == -INFINITY ? 0.f : __expf(v[e] - m);
      sum += v[e];
    }
    const float inv = 1.f / warp_sum(sum);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] *= inv;
    if (act) *reinterpret_cast<uint4*>(static_cast<uint16_t*>(P) + (row0 + k) * ld + c0) = pack8(v, fmt);
  }
}

template <int R>
__global__ void __launch_bounds__(256) softmax_bwd_rows_kernel(const void* __restrict__ S, const void* __restrict__ dP,
                                                               void* __restrict__ dS, long long rows, int L,
                                                               long long ld, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int lane = threadIdx.x & 31;
  const long long row0 = ((long long)blockIdx.x * 8 + (threadIdx.x >> 5)) * R;
  const int c0 = lane * 8;
  const bool act = c0 < ld;
  uint4 ws_[R], wg[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const bool ok = act && row0 + k < rows;
    ws_[k] = ok ? *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(S) + (row0 + k) * ld + c0)
                : make_uint4(0, 0, 0, 0);
    wg[k] = ok ? *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dP) + (row0 + k) * ld + c0)
               : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (row0 + k >= rows) break;
    float y[8], g[8];
    unpack8(ws_[k], y, fmt);
    unpack8(wg[k], g, fmt);
    float m = -INFINITY;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (!act || c0 + e >= L) y[e] = -INFINITY;
      m = fmaxf(m, y[e]);
    }
    m = warp_max(m);
    float sum = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      y[e] = y[e] == -INFINITY ? 0.f : __expf(y[e] - m);
      sum += y[e];
    }
    const float inv = 1.f / warp_sum(sum);
    float t = 0.f;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      y[e] *= inv;
      t += g[e] * y[e];
    }
    t = warp_sum(t);
#pragma unroll
    for (int e = 0; e < 8; ++e) g[e] = y[e] * (g[e] - t);
    if (act) *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dS) + (row0 + k) * ld + c0) = pack8(g, fmt);
  }
}

// ===========================================================================
// K6 attention softmax, register-resident rows (ld % 8 == 0, ld <= 256*CH):
// each lane holds CH 8-element chunks; one 16-byte load and store per chunk.
// ===========================================================================
template <int CH>
__global__ void __launch_bounds__(256) softmax_fwd_vec_kernel(const void* __restrict__ S, void* __restrict__ P,
                                                              long long rows, int L, long long ld, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const uint16_t* s = static_cast<const uint16_t*>(S) + row * ld;
  uint16_t* p = static_cast<uint16_t*>(P) + row * ld;
  float v[CH][8];
  float m = -INFINITY;
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c0 = (j * 32 + lane) * 8;
    if (c0 < ld) {
      unpack8(*reinterpret_cast<const uint4*>(s + c0), v[j], fmt);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (c0 + e >= L) v[j][e] = -INFINITY;
        m = fmaxf(m, v[j][e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[j][e] = -INFINITY;
    }
  }
  m = warp_max(m);
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < CH; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v[j][e] = v[j][e] == -INFINITY ? 0.f : expf(v[j][e] - m);
      sum += v[j][e];
    }
  const float inv = 1.f / warp_sum(sum);
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c0 = (j * 32 + lane) * 8;
    if (c0 < ld) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[j][e] *= inv;
      *reinterpret_cast<uint4*>(p + c0) = pack8(v[j], fmt);
    }
  }
}

template <int CH>
__global__ void __launch_bounds__(256) softmax_bwd_vec_kernel(const void* __restrict__ S, const void* __restrict__ dP,
                                                              void* __restrict__ dS, long long rows, int L,
                                                              long long ld, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const uint16_t* s = static_cast<const uint16_t*>(S) + row * ld;
  const uint16_t* dp = static_cast<const uint16_t*>(dP) + row * ld;
  uint16_t* ds = static_cast<uint16_t*>(dS) + row * ld;
  float y[CH][8], g[CH][8];
  float m = -INFINITY;
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c0 = (j * 32 + lane) * 8;
    if (c0 < ld) {
      unpack8(*reinterpret_cast<const uint4*>(s + c0), y[j], fmt);
      unpack8(*reinterpret_cast<const uint4*>(dp + c0), g[j], fmt);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (c0 + e >= L) y[j][e] = -INFINITY;
        m = fmaxf(m, y[j][e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        y[j][e] = -INFINITY;
        g[j][e] = 0.f;
      }
    }
  }
  m = warp_max(m);
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < CH; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      y[j][e] = y[j][e] == -INFINITY ? 0.f : expf(y[j][e] - m);
      sum += y[j][e];
    }
  const float inv = 1.f / warp_sum(sum);
  float t = 0.f;
#pragma unroll
  for (int j = 0; j < CH; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      y[j][e] *= inv;
      t += g[j][e] * y[j][e];
    }
  t = warp_sum(t);
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c0 = (j * 32 + lane) * 8;
    if (c0 < ld) {
#pragma unroll
      for (int e = 0; e < 8; ++e) g[j][e] = y[j][e] * (g[j][e] - t);
      *reinterpret_cast<uint4*>(ds + c0) = pack8(g[j], fmt);
    }
  }
}

// ===========================================================================
// K7 LayerNorm backward, register-resident rows (D = 256 * V): per-lane
// column partials of dgain/dbias stay in registers across the warp's rows.
// ===========================================================================
template <int V>
__global__ void __launch_bounds__(256) ln_bwd_vec_kernel(const void* __restrict__ x, long long ldx,
                                                         const void* __restrict__ g, const float* __restrict__ mean,
                                                         const float* __restrict__ rstd, const void* __restrict__ dy,
                                                         long long lddy, const void* __restrict__ dres, long long ldres,
                                                         void* __restrict__ dx, long long lddx, float* __restrict__ ws,
                                                         int rows, int D, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  extern __shared__ float sh[];  // [8 warps][2][D]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float adg[V][8], adb[V][8];
#pragma unroll
  for (int j = 0; j < V; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) adg[j][e] = adb[j][e] = 0.f;
  for (long long row = (long long)blockIdx.x * 8 + warp; row < rows; row += (long long)gridDim.x * 8) {
    const float mu = mean[row], rs = rstd[row];
    float xh[V][8], d[V][8];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int c0 = (j * 32 + lane) * 8;
      float gg[8];
      unpack8(*reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(x) + row * ldx + c0), xh[j], fmt);
      unpack8(*reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dy) + row * lddy + c0), d[j], fmt);
      unpack8(__ldg(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(g) + c0)), gg, fmt);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xh[j][e] = (xh[j][e] - mu) * rs;
        adg[j][e] += d[j][e] * xh[j][e];
        adb[j][e] += d[j][e];
        d[j][e] *= gg[e];  // d <- dy * g
        s1 += d[j][e];
        s2 += d[j][e] * xh[j][e];
      }
    }
    s1 = warp_sum(s1) / (float)D;
    s2 = warp_sum(s2) / (float)D;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int c0 = (j * 32 + lane) * 8;
      float o[8], r[8];
      if (dres) unpack8(*reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(dres) + row * ldres + c0), r, fmt);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = rs * (d[j][e] - s1 - xh[j][e] * s2) + (dres ? r[e] : 0.f);
      *reinterpret_cast<uint4*>(static_cast<uint16_t*>(dx) + row * lddx + c0) = pack8(o, fmt);
    }
  }
  float* my = sh + warp * 2 * D;
#pragma unroll
  for (int j = 0; j < V; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = (j * 32 + lane) * 8 + e;
      my[c] = adg[j][e];
      my[D + c] = adb[j][e];
    }
  __syncthreads();
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    float a = 0.f, b = 0.f;
    for (int w = 0; w < 8; ++w) {
      a += sh[w * 2 * D + c];
      b += sh[w * 2 * D + D + c];
    }
    ws[(long long)blockIdx.x * D + c] = a;
    ws[(long long)gridDim.x * D + (long long)blockIdx.x * D + c] = b;
  }
}

// ===========================================================================
// K6 attention softmax over rows of length L (row stride ld >= L, pads -> 0)
// ===========================================================================
__global__ void __launch_bounds__(256) softmax_fwd_kernel(const void* __restrict__ S, void* __restrict__ P,
                                                          long long rows, int L, long long ld, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const long long base = row * ld;
  float m = -INFINITY;
  for (int c = lane; c < L; c += 32) m = fmaxf(m, ld_h(S, base + c, fmt));
  m = warp_max(m);
  float s = 0.f;
  for (int c = lane; c < L; c += 32) s += expf(ld_h(S, base + c, fmt) - m);
  s = warp_sum(s);
  const float inv = 1.f / s;
  for (int c = lane; c < ld; c += 32) st_h(P, base + c, c < L ? expf(ld_h(S, base + c, fmt) - m) * inv : 0.f, fmt);
}

// dS = y * (dP - sum(dP * y)),  y = softmax(S) recomputed in f32
__global__ void __launch_bounds__(256) softmax_bwd_kernel(const void* __restrict__ S, const void* __restrict__ dP,
                                                          void* __restrict__ dS, long long rows, int L, long long ld,
                                                          int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const long long base = row * ld;
  float m = -INFINITY;
  for (int c = lane; c < L; c += 32) m = fmaxf(m, ld_h(S, base + c, fmt));
  m = warp_max(m);
  float s = 0.f;
  for (int c = lane; c < L; c += 32) s += expf(ld_h(S, base + c, fmt) - m);
  const float inv = 1.f / warp_sum(s);
  float t = 0.f;
  for (int c = lane; c < L; c += 32) t += ld_h(dP, base + c, fmt) * expf(ld_h(S, base + c, fmt) - m) * inv;
  t = warp_sum(t);
  for (int c = lane; c < ld; c += 32) {
    float o = 0.f;
    if (c < L) o = expf(ld_h(S, base + c, fmt) - m) * inv * (ld_h(dP, base + c, fmt) - t);
    st_h(dS, base + c, o, fmt);
  }
}

// ===========================================================================
// K9 cross-entropy (f32 island): nll[b] = lse(z_b) - z_b[y_b]; loss = mean
// ===========================================================================
__global__ void __launch_bounds__(256) ce_fwd_kernel(const void* __restrict__ logits, long long ld,
                                                     const int32_t* __restrict__ labels, int B, int C,
                                                     float* __restrict__ nll, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= B) return;
  const long long base = (long long)row * ld;
  float m = -INFINITY;
  for (int c = lane; c < C; c += 32) m = fmaxf(m, ld_h(logits, base + c, fmt));
  m = warp_max(m);
  float s = 0.f;
  for (int c = lane; c < C; c += 32) s += expf(ld_h(logits, base + c, fmt) - m);
  s = warp_sum(s);
  if (lane == 0) nll[row] = logf(s) - (ld_h(logits, base + labels[row], fmt) - m);
}
__global__ void ce_mean_kernel(const float* __restrict__ nll, int B, float* __restrict__ loss) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  __shared__ float sh[32];
  float s = 0.f;
  for (int i = threadIdx.x; i < B; i += blockDim.x) s += nll[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x + 31) / 32 ? sh[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) *loss = v / (float)B;
  }
}
// dlogits = (softmax(z) - onehot(y)) * dloss / B   (dloss read on the device)
__global__ void __launch_bounds__(256) ce_bwd_kernel(const void* __restrict__ logits, long long ld,
                                                     const int32_t* __restrict__ labels, int B, int C,
                                                     const float* __restrict__ dloss, void* __restrict__ dz,
                                                     long long ldd, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= B) return;
  const long long base = (long long)row * ld;
  float m = -INFINITY;
  for (int c = lane; c < C; c += 32) m = fmaxf(m, ld_h(logits, base + c, fmt));
  m = warp_max(m);
  float s = 0.f;
  for (int c = lane; c < C; c += 32) s += expf(ld_h(logits, base + c, fmt) - m);
  const float inv = 1.f / warp_sum(s);
  const float k = *dloss / (float)B;
  const int y = labels[row];
  for (int c = lane; c < ldd; c += 32) {
    float o = 0.f;
    if (c < C) o = (expf(ld_h(logits, base + c, fmt) - m) * inv - (c == y ? 1.f : 0.f)) * k;
    st_h(dz, (long long)row * ldd + c, o, fmt);
  }
}

// ===========================================================================
// patchify: img [B, H, W, C] -> patches [B*(H/p)*(W/p), p*p*C], vector order
// (py, px, c) — reshape [B,h,p,w,p,C] / transpose (0,1,3,2,4,5)
// ===========================================================================
__global__ void patchify_kernel(const uint16_t* __restrict__ img, uint16_t* __restrict__ out, int B, int H, int W,
                                int C, int p) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int nh = H / p, nw = W / p, K = p * p * C;
  const long long n = (long long)B * nh * nw * K;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / K;
    const int k = (int)(i - r * K);
    const int b = (int)(r / (nh * nw));
    const int t = (int)(r - (long long)b * nh * nw);
    const int ih = t / nw, iw = t - ih * nw;
    const int py = k / (p * C), rem = k - py * p * C, px = rem / C, c = rem - px * C;
    out[i] = img[(((long long)b * H + ih * p + py) * W + iw * p + px) * C + c];
  }
}

// patchify by 16-byte vectors: a patch row's (py) segment of p*C contiguous
// image elements is contiguous in both layouts; one thread per vector, one
// 2-D index (segment, vector) per thread, no 64-bit divides in the loop body
__global__ void __launch_bounds__(256) patchify_vec_kernel(const uint4* __restrict__ img, uint4* __restrict__ out,
                                                           int B, int H, int W, int C, int p) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int nh = H / p, nw = W / p;
  const int seg_v = p * C / 8;                  // 16-byte vectors per (patch, py) segment
  const long long nseg = (long long)B * nh * nw * p;
  const long long total = nseg * seg_v;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long sg = i / seg_v;
    const int v = (int)(i - sg * seg_v);
    const long long r = sg / p;  // patch index (b, ih, iw)
    const int py = (int)(sg - r * p);
    const int b = (int)(r / (nh * nw));
    const int t = (int)(r - (long long)b * nh * nw);
    const int ih = t / nw, iw = t - ih * nw;
    const long long src = ((((long long)b * H + ih * p + py) * W + (long long)iw * p) * C) / 8 + v;
    out[i] = __ldcs(img + src);  // out row r, columns [py*p*C, (py+1)*p*C) — i is already that flat index
  }
}

// dst[c][r] = src[r][c] for 16-bit elements, many matrices per launch: 64 x 64
// tiles through shared memory (+2-element row pad), 32-bit words on both sides
struct TransposeJob {
  const uint16_t* src;
  uint16_t* dst;
  int rows, cols;
  long long ld_src, ld_dst;
  int tile_begin, tiles_c;  // first tile index of this job, tiles per tile-row
};
constexpr int kMaxTransposeJobs = 64;
struct TransposeBatch {
  TransposeJob job[kMaxTransposeJobs];
  int n;
};

__global__ void __launch_bounds__(256) transpose16_kernel(const __grid_constant__ TransposeBatch T) {
  ::mpx::pdl_wait_only();  // many waves: the successor launches when the last one ends
  __shared__ uint16_t tile[64][66];
  int j = 0;
  while (j + 1 < T.n && (int)blockIdx.x >= T.job[j + 1].tile_begin) ++j;
  const TransposeJob& J = T.job[j];
  const int t = blockIdx.x - J.tile_begin;
  const int r0 = (t / J.tiles_c) * 64, c0 = (t % J.tiles_c) * 64;
  // full 64 x 64 tiles with 16-byte aligned rows on both sides: 16-byte loads
  // (8 columns of a row) and 16-byte stores (8 rows of a column), through a
  // tile padded to 72 columns (a column's 8 rows fall in 8 distinct banks)
  if (r0 + 64 <= J.rows && c0 + 64 <= J.cols && ((J.ld_src | J.ld_dst) & 7) == 0 &&
      ((reinterpret_cast<uintptr_t>(J.src) | reinterpret_cast<uintptr_t>(J.dst)) & 15) == 0) {
    __shared__ __align__(16) uint16_t tv[64][72];
#pragma unroll
    for (int k = 0; k < 2; ++k) {  // 512 vectors: row = v / 8, 8-column group = v % 8
      const int v = threadIdx.x + 256 * k, rr = v >> 3, cg = (v & 7) * 8;
      *reinterpret_cast<uint4*>(&tv[rr][cg]) =
          *reinterpret_cast<const uint4*>(J.src + (long long)(r0 + rr) * J.ld_src + c0 + cg);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 2; ++k) {  // 512 vectors: dst row = source column v / 8, 8-row group = v % 8
      const int v = threadIdx.x + 256 * k, cc = v >> 3, rg = (v & 7) * 8;
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) w[e] = (uint32_t)tv[rg + 2 * e][cc] | ((uint32_t)tv[rg + 2 * e + 1][cc] << 16);
      *reinterpret_cast<uint4*>(J.dst + (long long)(c0 + cc) * J.ld_dst + r0 + rg) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    return;
  }
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 column pairs x 8 rows per pass
  const bool wide = (J.cols & 1) == 0 && (J.ld_src & 1) == 0 && (reinterpret_cast<uintptr_t>(J.src) & 3) == 0;
#pragma unroll 4
  for (int i = ty; i < 64; i += 8) {
    const int r = r0 + i, c = c0 + 2 * tx;
    uint32_t w = 0;
    if (r < J.rows && c < J.cols) {
      if (wide)
        w = *reinterpret_cast<const uint32_t*>(J.src + (long long)r * J.ld_src + c);
      else
        w = (uint32_t)J.src[(long long)r * J.ld_src + c] |
            (c + 1 < J.cols ? (uint32_t)J.src[(long long)r * J.ld_src + c + 1] << 16 : 0u);
    }
    tile[i][2 * tx] = (uint16_t)(w & 0xFFFFu);
    tile[i][2 * tx + 1] = (uint16_t)(w >> 16);
  }
  __syncthreads();
  const bool wide_out = (J.ld_dst & 1) == 0 && (reinterpret_cast<uintptr_t>(J.dst) & 3) == 0;
#pragma unroll 4
  for (int i = ty; i < 64; i += 8) {  // dst row = source column c0 + i, 2 source rows per thread
    const int c = c0 + i, r = r0 + 2 * tx;
    if (c >= J.cols) continue;
    if (r + 1 < J.rows && wide_out) {
      const uint32_t w = (uint32_t)tile[2 * tx][i] | ((uint32_t)tile[2 * tx + 1][i] << 16);
      *reinterpret_cast<uint32_t*>(J.dst + (long long)c * J.ld_dst + r) = w;
    } else {
      if (r < J.rows) J.dst[(long long)c * J.ld_dst + r] = tile[2 * tx][i];
      if (r + 1 < J.rows) J.dst[(long long)c * J.ld_dst + r + 1] = tile[2 * tx + 1][i];
    }
  }
}

// strided row copy by 16-byte vectors (cols % 8 == 0, 16-byte aligned rows)
__global__ void __launch_bounds__(256) copy_rows_vec_kernel(const uint16_t* __restrict__ src, long long ld_src,
                                                            long long sb_src, uint16_t* __restrict__ dst,
                                                            long long ld_dst, long long sb_dst, int rows, int batches,
                                                            int cols) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int cv = cols / 8;
  const long long n = (long long)batches * rows * cv;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long bc = i / cv;
    const int c = (int)(i - bc * cv) * 8;
    const int b = (int)(bc / rows), r = (int)(bc - (long long)b * rows);
    *reinterpret_cast<uint4*>(dst + b * sb_dst + r * ld_dst + c) =
        *reinterpret_cast<const uint4*>(src + b * sb_src + r * ld_src + c);
  }
}

// out[b][r][c] = src[b][r][c] (strided row copy), optional add of a
// broadcast row (add[c]) and scaling
__global__ void copy_rows_kernel(const uint16_t* __restrict__ src, long long ld_src, long long sb_src,
                                 uint16_t* __restrict__ dst, long long ld_dst, long long sb_dst, int rows, int batches,
                                 int cols) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const long long n = (long long)batches * rows * cols;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long bc = i / cols;
    const int c = (int)(i - bc * cols);
    const int b = (int)(bc / rows), r = (int)(bc - (long long)b * rows);
    dst[b * sb_dst + r * ld_dst + c] = src[b * sb_src + r * ld_src + c];
  }
}

// dst[b*sb + c] = round(a[c] + b[c])  (cls token + its position embedding)
__global__ void rows_add_kernel(const void* __restrict__ a, const void* __restrict__ b2, void* __restrict__ dst,
                                long long sb, int B, int D, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const long long n = (long long)B * D;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / D;
    const int c = (int)(i - b * D);
    st_h(dst, b * sb + c, ld_h(a, c, fmt) + ld_h(b2, c, fmt), fmt);
  }
}

// dst[b][r][c] = alpha * src[b][c]   (mean-pool backward broadcast)
__global__ void bcast_rows_kernel(const void* __restrict__ src, long long ld_src, void* __restrict__ dst,
                                  long long ld_dst, long long sb_dst, int rows, int B, int D, float alpha, int fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const long long n = (long long)B * rows * D;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long bc = i / D;
    const int c = (int)(i - bc * D);
    const int b = (int)(bc / rows), r = (int)(bc - (long long)b * rows);
    st_h(dst, b * sb_dst + r * ld_dst + c, alpha * ld_h(src, (long long)b * ld_src + c, fmt), fmt);
  }
}

static int fmt_of(int dtype) { return dtype == MPX_BF16 ? 1 : 0; }
static bool half_dtype(int dt) { return dt == MPX_F16 || dt == MPX_BF16; }
static int ew_grid(long long n) {
  long long g = (n + 255) / 256;
  const long long cap = (long long)current_num_sms() * 8;
  return (int)std::max<long long>(1, std::min(g, cap));
}

}  // namespace mpx

using namespace mpx;

extern "C" {

int mpx_layernorm_fwd(int dtype, const void* x, int64_t ldx, const void* gain, const void* bias, void* y,
                      int64_t ldy, float* mean, float* rstd, int rows, int D, float eps, void* stream) {
  if (!half_dtype(dtype)) return fail(MPX_EINVAL, "layernorm: f16/bf16 only");
  if (rows <= 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#ifndef MPX_LN_FWD_WARPS
#define MPX_LN_FWD_WARPS 2
#endif
  constexpr int kW = MPX_LN_FWD_WARPS;  // rows (warps) per block: 2 (64-thread blocks) measured 29.1 us vs 31.1 with 8 at ViT-B
  const int grid = (rows + kW - 1) / kW;
  const bool vec = (ldx % 8 == 0) && (ldy % 8 == 0) && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                                                         reinterpret_cast<uintptr_t>(gain) |
                                                         reinterpret_cast<uintptr_t>(bias)) % 16 == 0);
  const int f = fmt_of(dtype);
  auto launch = [&](auto k) { return ::mpx::launch_k(k, grid, 32 * kW, 0, st, x, ldx, gain, bias, y, ldy, mean, rstd, rows, D, eps, f); };
  if (vec && D == 768)
    MPX_CUDA_CHECK(f ? launch(ln_fwd_kernel<3, 1>) : launch(ln_fwd_kernel<3, 0>));
  else if (vec && D == 1024)
    MPX_CUDA_CHECK(f ? launch(ln_fwd_kernel<4, 1>) : launch(ln_fwd_kernel<4, 0>));
  else if (vec && D == 512)
    MPX_CUDA_CHECK(f ? launch(ln_fwd_kernel<2, 1>) : launch(ln_fwd_kernel<2, 0>));
  else
    MPX_CUDA_CHECK(f ? launch(ln_fwd_kernel<0, 1>) : launch(ln_fwd_kernel<0, 0>));
  MPX_LAUNCH_CHECK("ln_fwd_kernel");
  return 0;
}

int mpx_layernorm_bwd_blocks(int rows) {
  return std::max(1, std::min((rows + 7) / 8, current_num_sms() * 2));
}

int mpx_layernorm_bwd(int dtype, const void* x, int64_t ldx, const void* gain, const float* mean, const float* rstd,
                      const void* dy, int64_t lddy, const void* dres, int64_t ldres, void* dx, int64_t lddx,
                      void* dgain, void* dbias, float* workspace, int rows, int D, void* stream) {
  if (!half_dtype(dtype)) return fail(MPX_EINVAL, "layernorm_bwd: f16/bf16 only");
  if (rows <= 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nb = mpx_layernorm_bwd_blocks(rows);
  const size_t sh = (size_t)8 * 2 * D * sizeof(float);
  if (sh > 48 * 1024) {
    MPX_CUDA_CHECK(ensure_smem_attr((const void*)ln_bwd_kernel, 200 * 1024));
  }
  const int f = fmt_of(dtype);
  const bool vec = ldx % 8 == 0 && lddy % 8 == 0 && lddx % 8 == 0 && (!dres || ldres % 8 == 0) &&
                   ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(dx) |
                     reinterpret_cast<uintptr_t>(gain) | reinterpret_cast<uintptr_t>(dres)) % 16 == 0);
  if (sh > 48 * 1024) {
    MPX_CUDA_CHECK(ensure_smem_attr((const void*)ln_bwd_vec_kernel<1>, 200 * 1024));
    MPX_CUDA_CHECK(ensure_smem_attr((const void*)ln_bwd_vec_kernel<3>, 200 * 1024));
    MPX_CUDA_CHECK(ensure_smem_attr((const void*)ln_bwd_vec_kernel<4>, 200 * 1024));
  }
  if (vec && D == 768)
    MPX_CUDA_CHECK(::mpx::launch_k(ln_bwd_vec_kernel<3>, nb, 256, sh, st, x, ldx, gain, mean, rstd, dy, lddy, dres, ldres, dx, lddx, workspace,
                                              rows, D, f));
  else if (vec && D == 1024)  // (v2 would spill at 4 vectors per lane)
    MPX_CUDA_CHECK(::mpx::launch_k(ln_bwd_vec_kernel<4>, nb, 256, sh, st, x, ldx, gain, mean, rstd, dy, lddy, dres, ldres, dx, lddx, workspace,
                                              rows, D, f));
  else if (vec && D == 256)
    MPX_CUDA_CHECK(::mpx::launch_k(ln_bwd_vec_kernel<1>, nb, 256, sh, st, x, ldx, gain, mean, rstd, dy, lddy, dres, ldres, dx, lddx, workspace,
                                              rows, D, f));
  else
    MPX_CUDA_CHECK(::mpx::launch_k(ln_bwd_kernel, nb, 256, sh, st, x, ldx, gain, mean, rstd, dy, lddy, dres, ldres, dx, lddx, workspace, rows, D,
                                       f));
  MPX_LAUNCH_CHECK("ln_bwd_kernel");
  MPX_CUDA_CHECK(::mpx::launch_k(partials_reduce_kernel, (D + 31) / 32, 256, 0, st, workspace, nb, D, dgain, dbias, 1.f, f));
  MPX_LAUNCH_CHECK("partials_reduce_kernel");
  return 0;
}

int mpx_layernorm_bwd2(int dtype, const void* x, int64_t ldx, const void* gain, const float* mean, const float* rstd,
                       const void* dy, int64_t lddy, const void* dres, int64_t ldres, void* dx, int64_t lddx,
                       void* dgain, void* dbias, void* dxsum, float* workspace, int64_t workspace_floats, int rows,
                       int D, void* stream) {
  if (!half_dtype(dtype)) return fail(MPX_EINVAL, "layernorm_bwd2: f16/bf16 only");
  if (rows <= 0) return 0;
  const bool vec = D % 256 == 0 && D <= 1024 && ldx % 8 == 0 && lddy % 8 == 0 && lddx % 8 == 0 &&
                   (!dres || ldres % 8 == 0) &&
                   ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(dx) |
                     reinterpret_cast<uintptr_t>(gain) | reinterpret_cast<uintptr_t>(dres)) % 16 == 0);
  if (!vec) {  // generic shapes: the fused single-kernel path (+ a separate dx colsum)
    int rc = mpx_layernorm_bwd(dtype, x, ldx, gain, mean, rstd, dy, lddy, dres, ldres, dx, lddx, dgain, dbias,
                               workspace, rows, D, stream);
    if (rc || !dxsum) return rc;
    return mpx_colsum(dtype, dx, lddx, 0, rows, D, 1, workspace, workspace_floats, dxsum, D, dtype, 1.f, stream);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int f = fmt_of(dtype);
  static const bool fused_off = getenv("MPX_LN_FUSED") && getenv("MPX_LN_FUSED")[0] == '0';
  static const bool reg_off = getenv("MPX_LN_BWD_REG") && getenv("MPX_LN_BWD_REG")[0] == '0';
  if (D <= 768 && !fused_off && !reg_off) {  // one pass, column partials in registers
    const int nsum = dxsum ? 3 : 2;
    int blocks = current_num_sms() * 2;
    while ((long long)nsum * blocks * D > workspace_floats && blocks > 1) blocks /= 2;
    auto launch = [&](auto k) {
      return ::mpx::launch_k(k, blocks, 128, 0, st, x, ldx, gain, mean, rstd, dy, lddy, dres, ldres, dx, lddx,
                             workspace, rows, D);
    };
    const int v = D / 256;
    cudaError_t e;
    if (nsum == 3) {
      e = v == 1 ? (f ? launch(ln_bwd_reg_kernel<1, 1, 3>) : launch(ln_bwd_reg_kernel<1, 0, 3>))
        : v == 2 ? (f ? launch(ln_bwd_reg_kernel<2, 1, 3>) : launch(ln_bwd_reg_kernel<2, 0, 3>))
                 : (f ? launch(ln_bwd_reg_kernel<3, 1, 3>) : launch(ln_bwd_reg_kernel<3, 0, 3>));
    } else {
      e = v == 1 ? (f ? launch(ln_bwd_reg_kernel<1, 1, 2>) : launch(ln_bwd_reg_kernel<1, 0, 2>))
        : v == 2 ? (f ? launch(ln_bwd_reg_kernel<2, 1, 2>) : launch(ln_bwd_reg_kernel<2, 0, 2>))
                 : (f ? launch(ln_bwd_reg_kernel<3, 1, 2>) : launch(ln_bwd_reg_kernel<3, 0, 2>));
    }
    MPX_CUDA_CHECK(e);
    MPX_LAUNCH_CHECK("ln_bwd_reg_kernel");
    MPX_CUDA_CHECK(::mpx::launch_k(partials_reduce3_kernel, dim3((D + 31) / 32, nsum), 1024, 0, st, workspace, blocks, D, dgain, dbias, dxsum, f));
    MPX_LAUNCH_CHECK("partials_reduce3_kernel");
    return 0;
  }
  if (D <= 1024 && !fused_off) {  // one pass: dx + all column partials (shared-memory slabs; ViT-L's D = 1024)
    const int nsum = dxsum ? 3 : 2;
    int blocks = current_num_sms() * (D > 768 ? 2 : 4);  // (D = 1024: 2 blocks per SM, 255 registers)
    while ((long long)nsum * blocks * D > workspace_floats && blocks > 1) blocks /= 2;
    const size_t shb = (size_t)4 * 3 * D * sizeof(float);  // per-warp accumulator slabs
    const void* ks[8] = {(const void*)ln_bwd_fused_kernel<1, 0>, (const void*)ln_bwd_fused_kernel<2, 0>,
                         (const void*)ln_bwd_fused_kernel<3, 0>, (const void*)ln_bwd_fused_kernel<4, 0>,
                         (const void*)ln_bwd_fused_kernel<1, 1>, (const void*)ln_bwd_fused_kernel<2, 1>,
                         (const void*)ln_bwd_fused_kernel<3, 1>, (const void*)ln_bwd_fused_kernel<4, 1>};
    for (const void* k : ks) MPX_CUDA_CHECK(ensure_smem_attr(k, 48 * 1024));
    auto launch = [&](auto k) {
      return ::mpx::launch_k(k, blocks, 128, shb, st, x, ldx, gain, mean, rstd, dy, lddy, dres, ldres, dx, lddx,
                             workspace, rows, D, nsum, f);
    };
    switch (D / 256) {
      case 1: MPX_CUDA_CHECK(f ? launch(ln_bwd_fused_kernel<1, 1>) : launch(ln_bwd_fused_kernel<1, 0>)); break;
      case 2: MPX_CUDA_CHECK(f ? launch(ln_bwd_fused_kernel<2, 1>) : launch(ln_bwd_fused_kernel<2, 0>)); break;
      case 3: MPX_CUDA_CHECK(f ? launch(ln_bwd_fused_kernel<3, 1>) : launch(ln_bwd_fused_kernel<3, 0>)); break;
      default: MPX_CUDA_CHECK(f ? launch(ln_bwd_fused_kernel<4, 1>) : launch(ln_bwd_fused_kernel<4, 0>)); break;
    }
    MPX_LAUNCH_CHECK("ln_bwd_fused_kernel");
    MPX_CUDA_CHECK(::mpx::launch_k(partials_reduce3_kernel, dim3((D + 31) / 32, nsum), 1024, 0, st, workspace, blocks, D, dgain, dbias, dxsum, f));
    MPX_LAUNCH_CHECK("partials_reduce3_kernel");
    return 0;
  }
  const unsigned g1 = (unsigned)((rows + 7) / 8);
  switch (D / 256) {
    case 1: MPX_CUDA_CHECK(::mpx::launch_k(ln_dx_kernel<1>, g1, 256, 0, st, x, ldx, gain, mean, rstd, dy, lddy, dres, ldres, dx, lddx, rows, D, f)); break;
    case 2: MPX_CUDA_CHECK(::mpx::launch_k(ln_dx_kernel<2>, g1, 256, 0, st, x, ldx, gain, mean, rstd, dy, lddy, dres, ldres, dx, lddx, rows, D, f)); break;
    case 3: MPX_CUDA_CHECK(::mpx::launch_k(ln_dx_kernel<3>, g1, 256, 0, st, x, ldx, gain, mean, rstd, dy, lddy, dres, ldres, dx, lddx, rows, D, f)); break;
    default: MPX_CUDA_CHECK(::mpx::launch_k(ln_dx_kernel<4>, g1, 256, 0, st, x, ldx, gain, mean, rstd, dy, lddy, dres, ldres, dx, lddx, rows, D, f)); break;
  }
  MPX_LAUNCH_CHECK("ln_dx_kernel");
  const int cblocks = D / 256;
  const int nsum = dxsum ? 3 : 2;
  int splits = std::max(1, std::min(rows / 64, current_num_sms() * 8 / cblocks));
  while ((long long)nsum * splits * D > workspace_floats && splits > 1) splits /= 2;
  const int rps = (rows + splits - 1) / splits;
  MPX_CUDA_CHECK(::mpx::launch_k(ln_colsum_kernel, dim3(cblocks, splits), 256, 0, st, x, ldx, mean, rstd, dy, lddy, dxsum ? dx : nullptr, lddx, rows,
                                                         D, rps, workspace, f));
  MPX_LAUNCH_CHECK("ln_colsum_kernel");
  MPX_CUDA_CHECK(::mpx::launch_k(partials_reduce3_kernel, dim3((D + 31) / 32, nsum), 1024, 0, st, workspace, splits, D, dgain, dbias, dxsum, f));
  MPX_LAUNCH_CHECK("partials_reduce3_kernel");
  return 0;
}

int mpx_colsum(int dtype, const void* x, int64_t ldx, int64_t sbx, int rows, int cols, int batches, float* workspace,
               int64_t workspace_floats, void* out, int64_t ld_out, int out_dtype, float alpha, void* stream) {
  if (!half_dtype(dtype)) return fail(MPX_EINVAL, "colsum: f16/bf16 input only");
  if (rows <= 0 || cols <= 0 || batches <= 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cblocks = (cols + 255) / 256;
  const long long target = (long long)current_num_sms() * 8;  // one full wave of 256-thread blocks
  int splits = (int)std::max<long long>(1, target / ((long long)cblocks * batches));
  splits = std::min(splits, std::max(1, rows / 64));
  while ((long long)splits * cols * batches > workspace_floats && splits > 1) splits /= 2;
  if ((long long)splits * cols * batches > workspace_floats) return fail(MPX_EINVAL, "colsum: workspace too small");
  const int rps = (rows + splits - 1) / splits;
  dim3 grid(cblocks, splits, batches);
  MPX_CUDA_CHECK(::mpx::launch_k(colsum_partial_kernel, grid, 256, 0, st, x, ldx, sbx, rows, cols, rps, workspace, fmt_of(dtype)));
  MPX_LAUNCH_CHECK("colsum_partial_kernel");
  MPX_CUDA_CHECK(::mpx::launch_k(colsum_final_kernel, (unsigned)(((long long)cols * batches + 31) / 32), 256, 0, st, workspace, splits, cols, batches,
                                                                                      out, ld_out, out_dtype, alpha));
  MPX_LAUNCH_CHECK("colsum_final_kernel");
  return 0;
}

int mpx_softmax_fwd(int dtype, const void* S, void* P, int64_t rows, int L, int64_t ld, void* stream) {
  if (!half_dtype(dtype) || ld < L) return fail(MPX_EINVAL, "softmax_fwd: bad args");
  if (rows <= 0) return 0;
  const unsigned grid = (unsigned)((rows + 7) / 8);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool vec = ld % 8 == 0 && ((reinterpret_cast<uintptr_t>(S) | reinterpret_cast<uintptr_t>(P)) % 16 == 0);
  if (vec && ld <= 256)
    MPX_CUDA_CHECK(::mpx::launch_k(softmax_fwd_rows_kernel<4>, (unsigned)((rows + 31) / 32), 256, 0, st, S, P, rows, L, ld, fmt_of(dtype)));
  else if (vec && ld <= 512)
    MPX_CUDA_CHECK(::mpx::launch_k(softmax_fwd_vec_kernel<2>, grid, 256, 0, st, S, P, rows, L, ld, fmt_of(dtype)));
  else
    MPX_CUDA_CHECK(::mpx::launch_k(softmax_fwd_kernel, grid, 256, 0, st, S, P, rows, L, ld, fmt_of(dtype)));
  MPX_LAUNCH_CHECK("softmax_fwd_kernel");
  return 0;
}

int mpx_softmax_bwd(int dtype, const void* S, const void* dP, void* dS, int64_t rows, int L, int64_t ld, void* stream) {
  if (!half_dtype(dtype) || ld < L) return fail(MPX_EINVAL, "softmax_bwd: bad args");
  if (rows <= 0) return 0;
  const unsigned grid = (unsigned)((rows + 7) / 8);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool vec = ld % 8 == 0 && ((reinterpret_cast<uintptr_t>(S) | reinterpret_cast<uintptr_t>(dP) |
                                    reinterpret_cast<uintptr_t>(dS)) % 16 == 0);
  if (vec && ld <= 256)
    MPX_CUDA_CHECK(::mpx::launch_k(softmax_bwd_rows_kernel<4>, (unsigned)((rows + 31) / 32), 256, 0, st, S, dP, dS, rows, L, ld, fmt_of(dtype)));
  else if (vec && ld <= 512)
    MPX_CUDA_CHECK(::mpx::launch_k(softmax_bwd_vec_kernel<2>, grid, 256, 0, st, S, dP, dS, rows, L, ld, fmt_of(dtype)));
  else
    MPX_CUDA_CHECK(::mpx::launch_k(softmax_bwd_kernel, grid, 256, 0, st, S, dP, dS, rows, L, ld, fmt_of(dtype)));
  MPX_LAUNCH_CHECK("softmax_bwd_kernel");
  return 0;
}

int mpx_cross_entropy_fwd(int dtype, const void* logits, int64_t ld, const int32_t* labels, int B, int C,
                          float* nll_ws, float* loss, void* stream) {
  if (!half_dtype(dtype)) return fail(MPX_EINVAL, "cross_entropy: f16/bf16 logits only");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  MPX_CUDA_CHECK(::mpx::launch_k(ce_fwd_kernel, (B + 7) / 8, 256, 0, st, logits, ld, labels, B, C, nll_ws, fmt_of(dtype)));
  MPX_LAUNCH_CHECK("ce_fwd_kernel");
  MPX_CUDA_CHECK(::mpx::launch_k(ce_mean_kernel, 1, 1024, 0, st, nll_ws, B, loss));
  MPX_LAUNCH_CHECK("ce_mean_kernel");
  return 0;
}

int mpx_cross_entropy_bwd(int dtype, const void* logits, int64_t ld, const int32_t* labels, int B, int C,
                          const float* d_dloss, void* dlogits, int64_t ld_d, void* stream) {
  if (!half_dtype(dtype)) return fail(MPX_EINVAL, "cross_entropy_bwd: f16/bf16 only");
  MPX_CUDA_CHECK(::mpx::launch_k(ce_bwd_kernel, (B + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream), logits, ld, labels, B, C, d_dloss, dlogits,
                                                                             ld_d, fmt_of(dtype)));
  MPX_LAUNCH_CHECK("ce_bwd_kernel");
  return 0;
}

int mpx_patchify(int dtype, const void* img, void* patches, int B, int H, int W, int C, int P, void* stream) {
  if (!half_dtype(dtype) || P <= 0 || H % P || W % P) return fail(MPX_EINVAL, "patchify: bad args");
  const long long n = (long long)B * H * W * C;
  if ((P * C) % 8 == 0 && (W * C) % 8 == 0 &&
      ((reinterpret_cast<uintptr_t>(img) | reinterpret_cast<uintptr_t>(patches)) & 15) == 0) {
    MPX_CUDA_CHECK(::mpx::launch_k(patchify_vec_kernel, ew_grid(n / 8), 256, 0, static_cast<cudaStream_t>(stream), static_cast<const uint4*>(img), static_cast<uint4*>(patches), B, H, W, C, P));
    MPX_LAUNCH_CHECK("patchify_vec_kernel");
    return 0;
  }
  MPX_CUDA_CHECK(::mpx::launch_k(patchify_kernel, ew_grid(n), 256, 0, static_cast<cudaStream_t>(stream), static_cast<const uint16_t*>(img), static_cast<uint16_t*>(patches), B, H, W, C, P));
  MPX_LAUNCH_CHECK("patchify_kernel");
  return 0;
}

int mpx_copy_rows(int dtype, const void* src, int64_t ld_src, int64_t sb_src, void* dst, int64_t ld_dst,
                  int64_t sb_dst, int rows, int batches, int cols, void* stream) {
  if (!half_dtype(dtype)) return fail(MPX_EINVAL, "copy_rows: f16/bf16 only");
  const long long n = (long long)rows * batches * cols;
  if (n <= 0) return 0;
  if (cols % 8 == 0 && ld_src % 8 == 0 && sb_src % 8 == 0 && ld_dst % 8 == 0 && sb_dst % 8 == 0 &&
      ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    MPX_CUDA_CHECK(::mpx::launch_k(copy_rows_vec_kernel, ew_grid(n / 8), 256, 0, static_cast<cudaStream_t>(stream), static_cast<const uint16_t*>(src), ld_src, sb_src, static_cast<uint16_t*>(dst), ld_dst, sb_dst, rows, batches,
        cols));
    MPX_LAUNCH_CHECK("copy_rows_vec_kernel");
    return 0;
  }
  MPX_CUDA_CHECK(::mpx::launch_k(copy_rows_kernel, ew_grid(n), 256, 0, static_cast<cudaStream_t>(stream), static_cast<const uint16_t*>(src), ld_src, sb_src, static_cast<uint16_t*>(dst), ld_dst, sb_dst, rows, batches,
      cols));
  MPX_LAUNCH_CHECK("copy_rows_kernel");
  return 0;
}

int mpx_transpose_batch(int dtype, int n, const void* const* src, void* const* dst, const int* rows,
                        const int* cols, const int64_t* ld_src, const int64_t* ld_dst, void* stream) {
  if (!half_dtype(dtype)) return fail(MPX_EINVAL, "transpose: f16/bf16 only");
  if (n < 0 || n > kMaxTransposeJobs) return fail(MPX_EINVAL, "transpose: at most 64 matrices per call");
  TransposeBatch T{};
  int tiles = 0;
  for (int i = 0; i < n; ++i) {
    if (rows[i] <= 0 || cols[i] <= 0) continue;
    if (ld_src[i] < cols[i] || ld_dst[i] < rows[i]) return fail(MPX_EINVAL, "transpose: bad leading dimensions");
    TransposeJob& J = T.job[T.n++];
    J.src = static_cast<const uint16_t*>(src[i]);
    J.dst = static_cast<uint16_t*>(dst[i]);
    J.rows = rows[i];
    J.cols = cols[i];
    J.ld_src = ld_src[i];
    J.ld_dst = ld_dst[i];
    J.tile_begin = tiles;
    J.tiles_c = (cols[i] + 63) / 64;
    tiles += ((rows[i] + 63) / 64) * J.tiles_c;
  }
  if (tiles == 0) return 0;
  MPX_CUDA_CHECK(::mpx::launch_k(transpose16_kernel, tiles, 256, 0, static_cast<cudaStream_t>(stream), T));
  return 0;
}

int mpx_transpose(int dtype, const void* src, int rows, int cols, int64_t ld_src, void* dst, int64_t ld_dst,
                  void* stream) {
  const int64_t ls = ld_src, ld = ld_dst;
  return mpx_transpose_batch(dtype, 1, &src, &dst, &rows, &cols, &ls, &ld, stream);
}

int mpx_rows_add(int dtype, const void* a, const void* b, void* dst, int64_t sb, int B, int D, void* stream) {
  if (!half_dtype(dtype)) return fail(MPX_EINVAL, "rows_add: f16/bf16 only");
  MPX_CUDA_CHECK(::mpx::launch_k(rows_add_kernel, ew_grid((long long)B * D), 256, 0, static_cast<cudaStream_t>(stream), a, b, dst, sb, B, D,
                                                                                            fmt_of(dtype)));
  MPX_LAUNCH_CHECK("rows_add_kernel");
  return 0;
}

int mpx_bcast_rows(int dtype, const void* src, int64_t ld_src, void* dst, int64_t ld_dst, int64_t sb_dst, int rows,
                   int B, int D, float alpha, void* stream) {
  if (!half_dtype(dtype)) return fail(MPX_EINVAL, "bcast_rows: f16/bf16 only");
  MPX_CUDA_CHECK(::mpx::launch_k(bcast_rows_kernel, ew_grid((long long)B * rows * D), 256, 0, static_cast<cudaStream_t>(stream), src, ld_src, dst, ld_dst, sb_dst, rows, B, D, alpha, fmt_of(dtype)));
  MPX_LAUNCH_CHECK("bcast_rows_kernel");
  return 0;
}

}  // extern "C"

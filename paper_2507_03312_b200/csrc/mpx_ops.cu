// The reference's generic tensor operators (mpsim.tensors, the `T` namespace
// its models are written against: tensors.py:220-555) as sm_100a kernels, so
// a model written for mpsim runs on the device through the drop-in names
// (paper_2507_03312_b200.tensors).  The ViT engine does not use these: its
// hot ops are the fused tcgen05 GEMM / attention / LayerNorm kernels.
//
// Numerics follow the reference op for op.  Every operator evaluates in f32
// and rounds its result once onto the output format's grid (quantize_array,
// dtypes.py:100-123); accumulations are the reference's STEPWISE ones
// (_stepwise_sum, tensors.py:327-338: the partial sum is re-rounded to the op
// dtype after every addition, in index order), done sequentially per output
// so f32 (and half) reductions, softmax sums, LayerNorm statistics and
// cross-entropy means are bit-identical to the reference wherever the
// reference itself is IEEE-exact (+ - * / sqrt); exp / log / tanh come from
// CUDA's libdevice (<= 2 ulp) instead of the host libm, so results that pass
// through them agree to a tolerance.  No FMA contraction anywhere (__f*_rn).
// The SIMT matmul keeps the reference's k order and f32 rounding per product
// and per partial sum, so f32 matmuls are bit-exact; half matmuls accumulate
// in f32 and round once (the tensor-core numerics),
// identical to the tcgen05 GEMM the host layer prefers when TMA can address
// the operands.
#include "mpx_common.cuh"

#include <cmath>

namespace mpx {
namespace {

constexpr int kMaxDims = 8;

__device__ __forceinline__ float ld_any(const void* p, int dt, int64_t i) {
  switch (dt) {
    case MPX_F16: return to_f32<MPX_F16>(static_cast<const uint16_t*>(p)[i]);
    case MPX_BF16: return to_f32<MPX_BF16>(static_cast<const uint16_t*>(p)[i]);
    default: return static_cast<const float*>(p)[i];
  }
}
__device__ __forceinline__ void st_any(void* p, int dt, int64_t i, float x) {
  switch (dt) {
    case MPX_F16: static_cast<uint16_t*>(p)[i] = from_f32<MPX_F16>(x); break;
    case MPX_BF16: static_cast<uint16_t*>(p)[i] = from_f32<MPX_BF16>(x); break;
    default: static_cast<float*>(p)[i] = x;
  }
}
// quantize_array(x, dt) staying in f32
__device__ __forceinline__ float q_any(float x, int dt) {
  switch (dt) {
    case MPX_F16: return quantize_f32<MPX_F16>(x);
    case MPX_BF16: return quantize_f32<MPX_BF16>(x);
    default: return x;
  }
}
// np.max semantics: NaN propagates
__device__ __forceinline__ float nanmax(float m, float v) { return (isnan(m) || !(isnan(v) || v > m)) ? m : v; }

// ---------------------------------------------------------------- gelu
// _gelu_kernel (tensors.py:196-200), numpy's left-to-right f32 evaluation
constexpr float kC0 = 0.7978845608028654f, kC1 = 0.044715f;
__device__ __forceinline__ float gelu_ref(float x) {
  const float inner = __fmul_rn(kC0, __fadd_rn(x, __fmul_rn(__fmul_rn(__fmul_rn(kC1, x), x), x)));
  return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.0f, tanhf(inner)));
}
// _bw_gelu's derivative (autodiff.py:173-185) before its quantize
__device__ __forceinline__ float gelu_deriv_ref(float x) {
  const float inner = __fmul_rn(kC0, __fadd_rn(x, __fmul_rn(__fmul_rn(__fmul_rn(kC1, x), x), x)));
  const float t = tanhf(inner);
  const float sech2 = __fsub_rn(1.0f, __fmul_rn(t, t));
  const float a = __fmul_rn(0.5f, __fadd_rn(1.0f, t));
  const float c3 = __fmul_rn(3.0f, kC1);
  const float b = __fmul_rn(__fmul_rn(__fmul_rn(__fmul_rn(0.5f, x), sech2), kC0),
                            __fadd_rn(1.0f, __fmul_rn(__fmul_rn(c3, x), x)));
  return __fadd_rn(a, b);
}

// ---------------------------------------------------------------- elementwise
struct EwArgs {
  int op, ndim, out_dt, a_dt, b_dt, scalar_side, grad_dt;
  float scalar;
  int64_t n;
  int64_t shape[kMaxDims], sa[kMaxDims], sb[kMaxDims];
  void* out;
  const void* a;
  const void* b;
};

__device__ __forceinline__ float ew_apply(int op, float x, float y, int grad_dt) {
  switch (op) {
    case MPX_EW_COPY: return x;
    case MPX_EW_ADD: return __fadd_rn(x, y);
    case MPX_EW_SUB: return __fsub_rn(x, y);
    case MPX_EW_MUL: return __fmul_rn(x, y);
    case MPX_EW_DIV: return __fdiv_rn(x, y);
    case MPX_EW_NEG: return -x;
    case MPX_EW_EXP: return expf(x);
    case MPX_EW_LOG: return logf(x);
    case MPX_EW_SQRT: return __fsqrt_rn(x);
    case MPX_EW_RELU: return isnan(x) ? x : fmaxf(x, 0.0f);  // np.maximum(x, 0) keeps NaN
    case MPX_EW_GELU: return gelu_ref(x);
    // x = cotangent c, y = the forward input: c * quantize(gelu'(y), c.dtype)
    case MPX_EW_GELU_BWD: return __fmul_rn(x, q_any(gelu_deriv_ref(y), grad_dt));
    // c * (y > 0) with the mask as a c-typed tensor (autodiff.py:167-170)
    case MPX_EW_RELU_BWD: return __fmul_rn(x, y > 0.0f ? 1.0f : 0.0f);
    default: return 0.0f;
  }
}

__global__ void __launch_bounds__(256) ew_kernel(const EwArgs A) {
  const bool binary = (A.op >= MPX_EW_ADD && A.op <= MPX_EW_DIV) || A.op >= MPX_EW_GELU_BWD;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = i, oa = 0, ob = 0;
#pragma unroll
    for (int d = kMaxDims - 1; d >= 0; --d) {
      if (d < A.ndim) {
        const int64_t ext = A.shape[d];
        const int64_t c = rem % ext;
        rem /= ext;
        oa += c * A.sa[d];
        ob += c * A.sb[d];
      }
    }
    float x = ld_any(A.a, A.a_dt, oa), y = 0.0f;
    if (binary) y = A.b ? ld_any(A.b, A.b_dt, ob) : A.scalar;
    if (binary && A.scalar_side && !A.b) {  // scalar (op) tensor: rsub / rtruediv
      const float t = x;
      x = y;
      y = t;
    }
    st_any(A.out, A.out_dt, i, ew_apply(A.op, x, y, A.grad_dt));
  }
}

// ---------------------------------------------------------------- reductions
// out[o, i] = reduce_j a[o, j, i] over a contiguous (outer, n, inner) view
__global__ void __launch_bounds__(256) reduce_kernel(int op, const void* a, int dt, int64_t outer, int64_t n,
                                                     int64_t inner, void* out, int out_dt) {
  const int64_t total = outer * inner;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = t / inner, i = t - o * inner;
    const int64_t base = o * n * inner + i;
    float acc;
    if (n == 0) {
      acc = 0.0f;
    } else if (op == MPX_RED_MAX) {
      acc = ld_any(a, dt, base);
      for (int64_t j = 1; j < n; ++j) acc = nanmax(acc, ld_any(a, dt, base + j * inner));
    } else {
      acc = ld_any(a, dt, base);  // _stepwise_sum: acc = x0; acc = q(acc + xj)
      for (int64_t j = 1; j < n; ++j) acc = q_any(__fadd_rn(acc, ld_any(a, dt, base + j * inner)), dt);
      if (op == MPX_RED_MEAN) acc = q_any(__fdiv_rn(acc, (float)n), dt);
    }
    st_any(out, out_dt, t, acc);
  }
}

// _bw_max (autodiff.py:223-230): the cotangent split equally among ties
__global__ void __launch_bounds__(256) reduce_max_bwd_kernel(const void* a, int dt, const void* m, const void* c,
                                                             int c_dt, int64_t outer, int64_t n, int64_t inner,
                                                             void* out) {
  const int64_t total = outer * inner;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = t / inner, i = t - o * inner;
    const int64_t base = o * n * inner + i;
    const float mv = ld_any(m, dt, t), cv = ld_any(c, c_dt, t);
    float cnt = 0.0f;
    for (int64_t j = 0; j < n; ++j) cnt += ld_any(a, dt, base + j * inner) == mv ? 1.0f : 0.0f;
    for (int64_t j = 0; j < n; ++j) {
      const float hit = ld_any(a, dt, base + j * inner) == mv ? 1.0f : 0.0f;
      st_any(out, c_dt, base + j * inner, __fdiv_rn(__fmul_rn(cv, hit), cnt));
    }
  }
}

// ---------------------------------------------------------------- softmax
// softmax along the middle axis of (outer, n, inner), tensors.py:431-446
__global__ void __launch_bounds__(256) softmax_axis_kernel(const void* a, int dt, int64_t outer, int64_t n,
                                                           int64_t inner, void* out) {
  const int64_t total = outer * inner;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = t / inner, i = t - o * inner;
    const int64_t base = o * n * inner + i;
    float m = ld_any(a, dt, base);
    for (int64_t j = 1; j < n; ++j) m = nanmax(m, ld_any(a, dt, base + j * inner));
    float s = 0.0f;
    for (int64_t j = 0; j < n; ++j) {
      const float e = q_any(expf(q_any(__fsub_rn(ld_any(a, dt, base + j * inner), m), dt)), dt);
      s = j == 0 ? e : q_any(__fadd_rn(s, e), dt);
    }
    for (int64_t j = 0; j < n; ++j) {
      const float e = q_any(expf(q_any(__fsub_rn(ld_any(a, dt, base + j * inner), m), dt)), dt);
      st_any(out, dt, base + j * inner, __fdiv_rn(e, s));
    }
  }
}

// _bw_softmax (autodiff.py:233-240): y * (c - stepwise_sum(c * y)), in dt
__global__ void __launch_bounds__(256) softmax_axis_bwd_kernel(const void* y, const void* c, int dt, int64_t outer,
                                                               int64_t n, int64_t inner, void* out) {
  const int64_t total = outer * inner;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = t / inner, i = t - o * inner;
    const int64_t base = o * n * inner + i;
    float s = 0.0f;
    for (int64_t j = 0; j < n; ++j) {
      const int64_t k = base + j * inner;
      const float t1 = q_any(__fmul_rn(ld_any(c, dt, k), ld_any(y, dt, k)), dt);
      s = j == 0 ? t1 : q_any(__fadd_rn(s, t1), dt);
    }
    for (int64_t j = 0; j < n; ++j) {
      const int64_t k = base + j * inner;
      const float yv = ld_any(y, dt, k);
      st_any(out, dt, k, __fmul_rn(yv, q_any(__fsub_rn(ld_any(c, dt, k), s), dt)));
    }
  }
}

// ---------------------------------------------------------------- layernorm
// _layernorm_internals (tensors.py:462-471) of row r, in dt: mean, std
__device__ __forceinline__ void ln_stats(const void* x, int x_dt, int64_t base, int64_t n, int dt, float& mean,
                                         float& std_) {
  float s = ld_any(x, x_dt, base);
  for (int64_t j = 1; j < n; ++j) s = q_any(__fadd_rn(s, ld_any(x, x_dt, base + j)), dt);
  mean = q_any(__fdiv_rn(q_any(s, dt), (float)n), dt);
  float v = 0.0f;
  for (int64_t j = 0; j < n; ++j) {
    const float c = q_any(__fsub_rn(ld_any(x, x_dt, base + j), mean), dt);
    const float sq = q_any(__fmul_rn(c, c), dt);
    v = j == 0 ? sq : q_any(__fadd_rn(v, sq), dt);
  }
  const float var = q_any(__fdiv_rn(v, (float)n), dt);
  std_ = q_any(__fsqrt_rn(q_any(__fadd_rn(var, 1e-5f), dt)), dt);
}

__global__ void __launch_bounds__(256) layernorm_ref_kernel(const void* x, int x_dt, const void* g, int g_dt,
                                                            const void* b, int b_dt, int64_t rows, int64_t n,
                                                            int dt, void* out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = r * n;
    float mean, sd;
    ln_stats(x, x_dt, base, n, dt, mean, sd);
    for (int64_t j = 0; j < n; ++j) {
      const float c = q_any(__fsub_rn(ld_any(x, x_dt, base + j), mean), dt);
      const float xh = q_any(__fdiv_rn(c, sd), dt);
      const float y = q_any(__fmul_rn(xh, ld_any(g, g_dt, j)), dt);
      st_any(out, dt, base + j, __fadd_rn(y, ld_any(b, b_dt, j)));
    }
  }
}

// _bw_layernorm (autodiff.py:243-262): dx per row; dgx[r, j] = q(c * xhat)
// (summed over rows afterwards by reduce_kernel, in the reference's order)
__global__ void __launch_bounds__(256) layernorm_ref_bwd_kernel(const void* x, int x_dt, const void* g, int g_dt,
                                                                const void* c, int64_t rows, int64_t n, int dt,
                                                                void* dx, void* dgx) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = r * n;
    float mean, sd;
    ln_stats(x, x_dt, base, n, dt, mean, sd);
    float s1 = 0.0f, s2 = 0.0f;
    for (int64_t j = 0; j < n; ++j) {
      const float xh = q_any(__fdiv_rn(q_any(__fsub_rn(ld_any(x, x_dt, base + j), mean), dt), sd), dt);
      const float cv = ld_any(c, dt, base + j);
      const float cg = q_any(__fmul_rn(cv, ld_any(g, g_dt, j)), dt);
      const float cx = q_any(__fmul_rn(cg, xh), dt);
      s1 = j == 0 ? cg : q_any(__fadd_rn(s1, cg), dt);
      s2 = j == 0 ? cx : q_any(__fadd_rn(s2, cx), dt);
      st_any(dgx, dt, base + j, __fmul_rn(cv, xh));
    }
    const float m1 = q_any(__fdiv_rn(s1, (float)n), dt), m2 = q_any(__fdiv_rn(s2, (float)n), dt);
    for (int64_t j = 0; j < n; ++j) {
      const float xh = q_any(__fdiv_rn(q_any(__fsub_rn(ld_any(x, x_dt, base + j), mean), dt), sd), dt);
      const float cg = q_any(__fmul_rn(ld_any(c, dt, base + j), ld_any(g, g_dt, j)), dt);
      const float t = q_any(__fsub_rn(q_any(__fsub_rn(cg, m1), dt), q_any(__fmul_rn(xh, m2), dt)), dt);
      st_any(dx, dt, base + j, __fdiv_rn(t, sd));
    }
  }
}

// ---------------------------------------------------------------- cross-entropy
// per-row nll (tensors.py:494-522); the batch mean is a reduce_kernel MEAN
__global__ void __launch_bounds__(256) xent_rows_kernel(const void* logits, int dt, const int32_t* labels, int64_t B,
                                                        int64_t C, void* nll) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < B; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = r * C;
    float m = ld_any(logits, dt, base);
    for (int64_t j = 1; j < C; ++j) m = nanmax(m, ld_any(logits, dt, base + j));
    float s = 0.0f;
    for (int64_t j = 0; j < C; ++j) {
      const float e = q_any(expf(q_any(__fsub_rn(ld_any(logits, dt, base + j), m), dt)), dt);
      s = j == 0 ? e : q_any(__fadd_rn(s, e), dt);
    }
    const float lse = q_any(logf(s), dt);
    const float ts = q_any(__fsub_rn(ld_any(logits, dt, base + labels[r]), m), dt);
    st_any(nll, dt, r, __fsub_rn(lse, ts));
  }
}

// _bw_cross_entropy (autodiff.py:265-276)
__global__ void __launch_bounds__(256) xent_bwd_kernel(const void* logits, int dt, const int32_t* labels, int64_t B,
                                                       int64_t C, const void* cot, int cot_dt, void* out) {
  const float cv = ld_any(cot, cot_dt, 0);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < B; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = r * C;
    float m = ld_any(logits, dt, base);
    for (int64_t j = 1; j < C; ++j) m = nanmax(m, ld_any(logits, dt, base + j));
    float s = 0.0f;
    for (int64_t j = 0; j < C; ++j) {
      const float e = q_any(expf(q_any(__fsub_rn(ld_any(logits, dt, base + j), m), dt)), dt);
      s = j == 0 ? e : q_any(__fadd_rn(s, e), dt);
    }
    const int32_t lab = labels[r];
    for (int64_t j = 0; j < C; ++j) {
      const float e = q_any(expf(q_any(__fsub_rn(ld_any(logits, dt, base + j), m), dt)), dt);
      const float p = q_any(__fdiv_rn(e, s), dt);
      const float diff = q_any(__fsub_rn(p, j == lab ? 1.0f : 0.0f), dt);
      const float sc = q_any(__fmul_rn(diff, cv), dt);
      st_any(out, dt, base + j, __fdiv_rn(sc, (float)B));
    }
  }
}

// ---------------------------------------------------------------- SIMT matmul
// C[z][m, n] = sum_k A[z][m, k] B[z][k, n] with arbitrary element strides:
// 64 x 64 tiles, 256 threads x 4 x 4 outputs, k-slabs of 16 staged in smem
// as f32.  Each output accumulates in k order: acc = f32(acc + f32(a * b)),
// acc starting at -0.0 (the identity of +, so acc == the first product).
struct MmArgs {
  const void* a;
  const void* b;
  void* c;
  int a_dt, b_dt, c_dt, nbatch_dims;
  int64_t M, N, K;
  int64_t sam, sak, sbk, sbn, scm, scn;
  int64_t bshape[4], sa_b[4], sb_b[4], sc_b[4];
};

__global__ void __launch_bounds__(256) matmul_simt_kernel(const MmArgs A) {
  __shared__ float sA[16][64 + 1];
  __shared__ float sB[16][64 + 1];
  int64_t z = blockIdx.z, oa = 0, ob = 0, oc = 0;
  for (int d = A.nbatch_dims - 1; d >= 0; --d) {
    const int64_t c = z % A.bshape[d];
    z /= A.bshape[d];
    oa += c * A.sa_b[d];
    ob += c * A.sb_b[d];
    oc += c * A.sc_b[d];
  }
  const int64_t m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = -0.0f;
  for (int64_t k0 = 0; k0 < A.K; k0 += 16) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = threadIdx.x + e * 256;  // 1024 = 16 x 64
      const int kk = idx >> 6, mm = idx & 63;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      sA[kk][mm] = (gm < A.M && gk < A.K) ? ld_any(A.a, A.a_dt, oa + gm * A.sam + gk * A.sak) : 0.0f;
      const int64_t gn = n0 + mm;
      sB[kk][mm] = (gn < A.N && gk < A.K) ? ld_any(A.b, A.b_dt, ob + gk * A.sbk + gn * A.sbn) : 0.0f;
    }
    __syncthreads();
    const int kmax = A.K - k0 < 16 ? (int)(A.K - k0) : 16;
    for (int kk = 0; kk < kmax; ++kk) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float av = sA[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av, sB[kk][tx + 16 * j]));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty + 16 * i;
    if (gm >= A.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx + 16 * j;
      if (gn < A.N) st_any(A.c, A.c_dt, oc + gm * A.scm + gn * A.scn, A.K == 0 ? 0.0f : acc[i][j]);
    }
  }
}

int grid_for(int64_t work) {
  const int64_t blocks = (work + 255) / 256;
  const int64_t cap = (int64_t)current_num_sms() * 16;
  return (int)std::max<int64_t>(1, std::min(blocks, cap));
}
bool dt_ok(int dt) { return dt == MPX_F32 || dt == MPX_F16 || dt == MPX_BF16; }
int inval(const char* what) { return fail(MPX_EINVAL, what); }

}  // namespace
}  // namespace mpx

using namespace mpx;

extern "C" {

int mpx_ew(int op, int ndim, const int64_t* h_shape, void* out, int out_dtype, const void* a, int a_dtype,
           const int64_t* h_a_strides, const void* b, int b_dtype, const int64_t* h_b_strides, double scalar,
           int scalar_side, int grad_dtype, void* stream) {
  if (op < MPX_EW_COPY || op > MPX_EW_RELU_BWD || ndim < 0 || ndim > kMaxDims || !dt_ok(out_dtype) ||
      !dt_ok(a_dtype) || (b && !dt_ok(b_dtype)) || !dt_ok(grad_dtype))
    return inval("mpx_ew: bad op / rank / dtype");
  EwArgs A{};
  A.op = op;
  A.ndim = ndim;
  A.out_dt = out_dtype;
  A.a_dt = a_dtype;
  A.b_dt = b ? b_dtype : MPX_F32;
  A.grad_dt = grad_dtype;
  A.scalar = (float)scalar;  // np.float32(weak scalar), tensors.py:235-236
  A.scalar_side = scalar_side;
  A.out = out;
  A.a = a;
  A.b = b;
  A.n = 1;
  for (int d = 0; d < ndim; ++d) {
    A.shape[d] = h_shape[d];
    A.sa[d] = h_a_strides[d];
    A.sb[d] = b ? h_b_strides[d] : 0;
    A.n *= h_shape[d];
  }
  if (A.n == 0) return 0;
  if (!out || !a) return inval("mpx_ew: null operand");
  MPX_CUDA_CHECK(launch_k(ew_kernel, dim3(grid_for(A.n)), dim3(256), 0, (cudaStream_t)stream, A));
  return 0;
}

int mpx_reduce(int op, const void* a, int dtype, int64_t outer, int64_t n, int64_t inner, void* out, int out_dtype,
               void* stream) {
  if (op < MPX_RED_SUM || op > MPX_RED_MAX || !dt_ok(dtype) || !dt_ok(out_dtype) || outer < 0 || n < 0 || inner < 0)
    return inval("mpx_reduce: bad op / dtype / extents");
  if (outer * inner == 0) return 0;
  MPX_CUDA_CHECK(launch_k(reduce_kernel, dim3(grid_for(outer * inner)), dim3(256), 0, (cudaStream_t)stream, op, a,
                          dtype, outer, n, inner, out, out_dtype));
  return 0;
}

int mpx_reduce_max_bwd(const void* a, int dtype, const void* m, const void* c, int c_dtype, int64_t outer, int64_t n,
                       int64_t inner, void* out, void* stream) {
  if (!dt_ok(dtype) || !dt_ok(c_dtype)) return inval("mpx_reduce_max_bwd: dtype");
  if (outer * inner * n == 0) return 0;
  MPX_CUDA_CHECK(launch_k(reduce_max_bwd_kernel, dim3(grid_for(outer * inner)), dim3(256), 0, (cudaStream_t)stream, a,
                          dtype, m, c, c_dtype, outer, n, inner, out));
  return 0;
}

int mpx_softmax_axis(const void* a, int dtype, int64_t outer, int64_t n, int64_t inner, void* out, void* stream) {
  if (!dt_ok(dtype)) return inval("mpx_softmax_axis: dtype");
  if (outer * inner * n == 0) return 0;
  MPX_CUDA_CHECK(launch_k(softmax_axis_kernel, dim3(grid_for(outer * inner)), dim3(256), 0, (cudaStream_t)stream, a,
                          dtype, outer, n, inner, out));
  return 0;
}

int mpx_softmax_axis_bwd(const void* y, const void* c, int dtype, int64_t outer, int64_t n, int64_t inner, void* out,
                         void* stream) {
  if (!dt_ok(dtype)) return inval("mpx_softmax_axis_bwd: dtype");
  if (outer * inner * n == 0) return 0;
  MPX_CUDA_CHECK(launch_k(softmax_axis_bwd_kernel, dim3(grid_for(outer * inner)), dim3(256), 0, (cudaStream_t)stream,
                          y, c, dtype, outer, n, inner, out));
  return 0;
}

int mpx_layernorm_ref(const void* x, int x_dtype, const void* gain, int g_dtype, const void* bias, int b_dtype,
                      int64_t rows, int64_t n, int dtype, void* out, void* stream) {
  if (!dt_ok(x_dtype) || !dt_ok(g_dtype) || !dt_ok(b_dtype) || !dt_ok(dtype) || n <= 0)
    return inval("mpx_layernorm_ref: dtype / empty axis");
  if (rows == 0) return 0;
  MPX_CUDA_CHECK(launch_k(layernorm_ref_kernel, dim3(grid_for(rows)), dim3(256), 0, (cudaStream_t)stream, x, x_dtype,
                          gain, g_dtype, bias, b_dtype, rows, n, dtype, out));
  return 0;
}

int mpx_layernorm_ref_bwd(const void* x, int x_dtype, const void* gain, int g_dtype, const void* c, int64_t rows,
                          int64_t n, int dtype, void* dx, void* dgx, void* stream) {
  if (!dt_ok(x_dtype) || !dt_ok(g_dtype) || !dt_ok(dtype) || n <= 0) return inval("mpx_layernorm_ref_bwd: dtype");
  if (rows == 0) return 0;
  MPX_CUDA_CHECK(launch_k(layernorm_ref_bwd_kernel, dim3(grid_for(rows)), dim3(256), 0, (cudaStream_t)stream, x,
                          x_dtype, gain, g_dtype, c, rows, n, dtype, dx, dgx));
  return 0;
}

int mpx_xent_rows(const void* logits, int dtype, const int32_t* labels, int64_t B, int64_t C, void* nll,
                  void* stream) {
  if (!dt_ok(dtype) || C <= 0) return inval("mpx_xent_rows: dtype / classes");
  if (B == 0) return 0;
  MPX_CUDA_CHECK(launch_k(xent_rows_kernel, dim3(grid_for(B)), dim3(256), 0, (cudaStream_t)stream, logits, dtype,
                          labels, B, C, nll));
  return 0;
}

int mpx_xent_bwd(const void* logits, int dtype, const int32_t* labels, int64_t B, int64_t C, const void* cot,
                 int cot_dtype, void* out, void* stream) {
  if (!dt_ok(dtype) || !dt_ok(cot_dtype) || C <= 0) return inval("mpx_xent_bwd: dtype / classes");
  if (B == 0) return 0;
  MPX_CUDA_CHECK(launch_k(xent_bwd_kernel, dim3(grid_for(B)), dim3(256), 0, (cudaStream_t)stream, logits, dtype,
                          labels, B, C, cot, cot_dtype, out));
  return 0;
}

int mpx_matmul_simt(const void* a, int a_dtype, const void* b, int b_dtype, void* c, int c_dtype, int64_t M,
                    int64_t N, int64_t K, const int64_t* h_strides /* sam sak sbk sbn scm scn */, int nbatch_dims,
                    const int64_t* h_bshape, const int64_t* h_sa_b, const int64_t* h_sb_b, const int64_t* h_sc_b,
                    void* stream) {
  if (!dt_ok(a_dtype) || !dt_ok(b_dtype) || !dt_ok(c_dtype) || nbatch_dims < 0 || nbatch_dims > 4 || M < 0 ||
      N < 0 || K < 0)
    return inval("mpx_matmul_simt: bad dtype / rank / extents");
  MmArgs A{};
  A.a = a;
  A.b = b;
  A.c = c;
  A.a_dt = a_dtype;
  A.b_dt = b_dtype;
  A.c_dt = c_dtype;
  A.M = M;
  A.N = N;
  A.K = K;
  A.sam = h_strides[0];
  A.sak = h_strides[1];
  A.sbk = h_strides[2];
  A.sbn = h_strides[3];
  A.scm = h_strides[4];
  A.scn = h_strides[5];
  A.nbatch_dims = nbatch_dims;
  int64_t batch = 1;
  for (int d = 0; d < nbatch_dims; ++d) {
    A.bshape[d] = h_bshape[d];
    A.sa_b[d] = h_sa_b[d];
    A.sb_b[d] = h_sb_b[d];
    A.sc_b[d] = h_sc_b[d];
    batch *= h_bshape[d];
  }
  if (M == 0 || N == 0 || batch == 0) return 0;
  if (batch > 65535) return inval("mpx_matmul_simt: more than 65535 batch matrices");
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64), (unsigned)batch);
  MPX_CUDA_CHECK(launch_k(matmul_simt_kernel, grid, dim3(256), 0, (cudaStream_t)stream, A));
  return 0;
}

}  // extern "C"

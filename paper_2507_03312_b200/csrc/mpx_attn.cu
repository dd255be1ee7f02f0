// K6 — fused attention for the ViT (sm_100a): softmax(Q K^T * scale) V per
// (image, head), straight out of the [B, N, 3, H, hd] qkv activation, with no
// N x N tensor in HBM.
//
// The reference computes scores in half, a full-precision softmax island and
// probabilities cast back to half before P V (bench.py:196-198;
// tensors.py:431-446).  Here the scores accumulate in f32 in TMEM, are
// rounded to the half format (the reference's score dtype), the softmax runs
// in f32 from TMEM, and P is rounded to half as the A operand of P V — the
// same roundings as the unfused path.
//
// One CTA = one (b, h, 128-query tile); all keys (N <= 256) fit on chip:
//   TMA   Q tile [128 x 64], K and V [256 x 64] (rows >= N zero-filled), SW128
//   MMA1  S[128 x 256] = Q K^T       tcgen05 M128 N256, f32 in TMEM cols 0-255
//   4 warps: one query row per thread, two TMEM passes (online max/sum, then
//            P = exp(s - m) / l), P (half) into smem in the UMMA K-major layout
//   MMA2  O[128 x 64] = P V          tcgen05 M128 N64 K256 (V read MN-major)
//   epilogue: O rows -> merged [B*N, H*hd] layout
#include "mpx_common.cuh"
#include "sm100_ptx.cuh"

#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <type_traits>

namespace mpx {

using namespace ptx;

// -DMPX_TRACE builds (tools only): per-CTA clock64 timestamps of the backward's
// phases for the first kTraceCtas CTAs, read back with mpx_debug_attn_trace
#ifdef MPX_TRACE
constexpr int kTraceCtas = 64, kTraceSlots = 32;
__device__ long long g_attn_trace[kTraceCtas * kTraceSlots];
#define ATRACE(slot)                                                            \
  do {                                                                          \
    if (blockIdx.x < kTraceCtas) g_attn_trace[blockIdx.x * kTraceSlots + (slot)] = clock64(); \
  } while (0)
#else
#define ATRACE(slot) \
  do {               \
  } while (0)
#endif
#ifndef MPX_TRACE_IT
#define MPX_TRACE_IT 0
#endif
constexpr int kTraceIt = MPX_TRACE_IT;  // which item of each CTA the trace records

constexpr int kAttnQ = 16384;      // Q tile 128 x 64 half
constexpr int kAttnKV = 32768;     // K / V 256 x 64 half
constexpr int kAttnP = 65536;      // P 128 x 256 half (4 K-major chunks of 64 keys)
constexpr int kSplit = 4;          // backward: softmax warps per TMEM lane quarter (column split)
constexpr int kSplitF = 7;         // forward: 28 softmax warps + 4 control warps = 1024 threads (64 registers)
constexpr int kAttnThreads = 128 + 128 * kSplit;  // warps 0-3 control, then 4*kSplit softmax warps
constexpr int kAttnThreadsF = 128 + 128 * kSplitF;

struct AttnParams {
  int N, H, hd, m_tiles;
  float scale;
  int fmt;  // 0 f16, 1 bf16
  void* O;
  long long ldo;  // O row stride (elements); head h at column h*hd
  float2* stats;  // optional [(b*H + h)*m_tiles*128 + row] = (row max, 1 / row sum) for the backward
  uint8_t* psave;  // optional: P (rounded, as the P V MMA read it) to [B*H][N][16 ceil(N/16)] for the backward
  int items;       // B * H (image, head) items, walked by a persistent grid
};

__device__ __forceinline__ float h2f(uint16_t h, int fmt) { return fmt ? to_f32<MPX_BF16>(h) : to_f32<MPX_F16>(h); }
__device__ __forceinline__ uint16_t f2h(float x, int fmt) { return fmt ? from_f32<MPX_BF16>(x) : from_f32<MPX_F16>(x); }
template <int NS>
__device__ __forceinline__ void quarter_sync(int q) {  // the NS warps sharing TMEM lane quarter q
  asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(32 * NS) : "memory");
}
// An mbarrier phase wait for the NS warps of lane quarter q: ONE warp polls
// (try_wait loop), the others block on a hardware named barrier (ids 5-8) that
// takes no issue slots — with 28 softmax warps spinning, the polls were ~10 %
// of the forward's instructions in an issue-bound kernel (and its energy).
// The caller's tcgen05 fence::after_thread_sync follows the named barrier.
// (Forward only: in the backward's 16 softmax warps it measured +0.7 % time.)
template <int NS, int ID0 = 5>
__device__ __forceinline__ void quarter_wait(uint64_t* b, uint32_t parity, int split, int q) {
  if (split == 0) mbar_wait(b, parity);
  asm volatile("bar.sync %0, %1;" ::"r"(ID0 + q), "r"(32 * NS) : "memory");
}

// P chunk c (keys 16c..16c+15) of row r into the K-major SW128 P tile
__device__ __forceinline__ void store_p_chunk(uint8_t* sP, int c, int r, const uint32_t* pk) {
  uint8_t* rowp = sP + (c >> 2) * 16384 + r * 128;
  const int u0 = (c & 3) * 2, sw = r & 7;
  *reinterpret_cast<uint4*>(rowp + ((u0 ^ sw) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  *reinterpret_cast<uint4*>(rowp + (((u0 + 1) ^ sw) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
}

__device__ __forceinline__ void unpack2(uint32_t pk, int fmt, float& lo, float& hi) {
  if (fmt) {
    lo = __uint_as_float(pk << 16);
    hi = __uint_as_float(pk & 0xFFFF0000u);
  } else {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&pk));
    lo = f.x;
    hi = f.y;
  }
}
// Scores of a chunk on the half grid.  For bf16 and a power-of-two scale,
// round(s * scale) == round(s) * scale exactly, so the scale is folded into the
// exponent constant (sv stays unscaled, `sl` = scale * log2 e); otherwise sv is
// round(s * scale) and sl = log2 e.  Either way e = 2^(sv * sl - m * log2 e).
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

struct ScoreGrid {
  float pre;  // multiplier before rounding (1 when folded)
  float sl;   // sv -> log2 units
  float ms;   // sv -> scaled score units (for the row max)
  __device__ __forceinline__ ScoreGrid(float scale, int fmt) {
    constexpr float kLog2e = 1.4426950408889634f;
    const uint32_t b = __float_as_uint(scale);
    const bool fold = fmt == 1 && (b & 0x807FFFFFu) == 0u && ((b >> 23) & 0xFFu) > 32u && ((b >> 23) & 0xFFu) < 222u;
    pre = fold ? 1.f : scale;
    sl = fold ? scale * kLog2e : kLog2e;
    ms = fold ? scale : 1.f;
  }
};
__device__ __forceinline__ void grid_scores16(const uint32_t* a, const ScoreGrid& G, int fmt, float* sv) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
    unpack2(pack2_fmt(__uint_as_float(a[2 * i]) * G.pre, __uint_as_float(a[2 * i + 1]) * G.pre, fmt), fmt,
            sv[2 * i], sv[2 * i + 1]);
}

// Forward softmax of row r, one TMEM pass: the thread's chunks c = split +
// NS j (< n_chunks) stay in registers (scores on the half grid, then e); the
// row max is exchanged through red_m, e = 2^(sv sl - M log2 e), and the row
// sum L is each split's chunk sums (pairs accumulated in order, then .x + .y)
// added in chunk order, then the split partials added in split order — the
// canonical order the backward's recompute follows, so its P is bit-identical.  Keys past N in the tail chunk are masked (e = 0); full
// chunks run unpredicated.  Returns (M, 1/L); softmax_store_p then writes P.
template <int FMT>
__device__ __forceinline__ uint32_t pack2T(float a, float b) {
  return FMT ? pack2<MPX_BF16>(a, b) : pack2<MPX_F16>(a, b);
}
template <int FMT>
__device__ __forceinline__ float2 unpack2T(uint32_t pk) {
  if (FMT) return make_float2(__uint_as_float(pk << 16), __uint_as_float(pk & 0xFFFF0000u));
  return __half22float2(*reinterpret_cast<const __half2*>(&pk));
}
template <int NS, int KC, int FMT>
__device__ __forceinline__ float2 softmax_fwd_regs(uint32_t trow, int split, int r, int q, int N, const ScoreGrid& G,
                                                   float* red_m, float* red_l, uint32_t (&a)[KC][16]) {
  constexpr float kLog2e = 1.4426950408889634f;
  const int n_chunks = (N + 15) / 16;
  const int tail = N - (n_chunks - 1) * 16;  // valid keys in the last chunk (1..16)
#pragma unroll
  for (int j = 0; j < KC; ++j)
    if (split + NS * j < n_chunks) tmem_ld16(trow + (split + NS * j) * 16, a[j]);
  tmem_ld_wait();
  float mloc = -INFINITY;
#pragma unroll
  for (int j = 0; j < KC; ++j) {
    const int c = split + NS * j;
    if (c < n_chunks) {
      if (G.pre != 1.f) {  // scores onto the half grid (pre = 1 when the scale is folded: x * 1 == x)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[j][i] = __float_as_uint(__uint_as_float(a[j][i]) * G.pre);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 s2 = unpack2T<FMT>(pack2T<FMT>(__uint_as_float(a[j][2 * i]), __uint_as_float(a[j][2 * i + 1])));
        a[j][2 * i] = __float_as_uint(s2.x);
        a[j][2 * i + 1] = __float_as_uint(s2.y);
      }
      if (c == n_chunks - 1 && tail < 16) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (i < tail) mloc = fmaxf(mloc, __uint_as_float(a[j][i]));
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) mloc = fmaxf(mloc, __uint_as_float(a[j][i]));
      }
    }
  }
  red_m[split * 128 + r] = mloc * G.ms;
  quarter_sync<NS>(q);
  float M = -INFINITY;
#pragma unroll
  for (int j = 0; j < NS; ++j) M = fmaxf(M, red_m[j * 128 + r]);
  const float ml = M * kLog2e;
  auto expc = [&](uint32_t* x, auto masked) {  // e in place, returns the chunk sum
    constexpr bool kMasked = decltype(masked)::value;
    float2 acc = f2(0.f);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float2 arg = __ffma2_rn(make_float2(__uint_as_float(x[2 * i]), __uint_as_float(x[2 * i + 1])), f2(G.sl),
                                    f2(-ml));
      const float e0 = (!kMasked || 2 * i < tail) ? ex2_approx(arg.x) : 0.f;
      const float e1 = (!kMasked || 2 * i + 1 < tail) ? ex2_approx(arg.y) : 0.f;
      acc = __fadd2_rn(acc, make_float2(e0, e1));
      x[2 * i] = __float_as_uint(e0);
      x[2 * i + 1] = __float_as_uint(e1);
    }
    return acc.x + acc.y;
  };
  float part = 0.f;  // this split's chunk sums, in chunk order
#pragma unroll
  for (int j = 0; j < KC; ++j) {
    const int c = split + NS * j;
    if (c < n_chunks)
      part += (c == n_chunks - 1 && tail < 16) ? expc(a[j], std::true_type{}) : expc(a[j], std::false_type{});
  }
  red_l[split * 128 + r] = part;
  quarter_sync<NS>(q);
  float L = 0.f;  // the split partials in split order (the canonical order; softmax_bwd_p repeats it)
#pragma unroll
  for (int j = 0; j < NS; ++j) L += red_l[j * 128 + r];
  return make_float2(M, 1.f / L);
}

// P = e * (1/L) rounded to half, the thread's chunks into the K-major P tile
template <int NS, int KC, int FMT>
__device__ __forceinline__ void softmax_store_p(int split, int r, int N, float inv, const uint32_t (&a)[KC][16],
                                                uint8_t* sP) {
  const int n_chunks = (N + 15) / 16;
#pragma unroll
  for (int j = 0; j < KC; ++j) {
    const int c = split + NS * j;
    if (c < n_chunks) {
      uint32_t pk[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 p2 = __fmul2_rn(make_float2(__uint_as_float(a[j][2 * i]), __uint_as_float(a[j][2 * i + 1])),
                                     f2(inv));
        pk[i] = pack2T<FMT>(p2.x, p2.y);
      }
      store_p_chunk(sP, c, r, pk);
    }
  }
}

// Backward: P_t of row r recomputed from the forward's (M, 1/L) when given,
// else from statistics recomputed here in the forward's canonical order (exact
// row max; chunk sums, each as softmax_fwd_regs forms it, through `lsc` [16
// chunks][128 rows], added per forward split and then in split order) — the
// same bits as the forward.
template <int NS>
__device__ __forceinline__ void softmax_bwd_p(uint32_t trow, int split, int r, int q, int N, float scale, int fmt,
                                              float* red, float* lsc, uint8_t* sP, const float2* stats) {
  constexpr float kLog2e = 1.4426950408889634f;
  const ScoreGrid G(scale, fmt);
  const int n_chunks = (N + 15) / 16;
  const int tail = N - (n_chunks - 1) * 16;
  float M, inv;
  if (stats != nullptr) {
    const float2 st = *stats;
    M = st.x;
    inv = st.y;
  } else {
    float mloc = -INFINITY;
    for (int c = split; c < n_chunks; c += NS) {
      uint32_t a[16];
      tmem_ld16(trow + c * 16, a);
      tmem_ld_wait();
      float sv[16];
      grid_scores16(a, G, fmt, sv);
      const int nv = c == n_chunks - 1 ? tail : 16;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < nv) mloc = fmaxf(mloc, sv[i]);
    }
    red[split * 128 + r] = mloc * G.ms;
    quarter_sync<NS>(q);
    M = -INFINITY;
#pragma unroll
    for (int j = 0; j < NS; ++j) M = fmaxf(M, red[j * 128 + r]);
    const float mlc = M * kLog2e;
    for (int c = split; c < n_chunks; c += NS) {
      uint32_t a[16];
      tmem_ld16(trow + c * 16, a);
      tmem_ld_wait();
      float sv[16];
      grid_scores16(a, G, fmt, sv);
      const int nv = c == n_chunks - 1 ? tail : 16;
      float2 acc = f2(0.f);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 arg = __ffma2_rn(make_float2(sv[2 * i], sv[2 * i + 1]), f2(G.sl), f2(-mlc));
        const float e0 = 2 * i < nv ? ex2_approx(arg.x) : 0.f;
        const float e1 = 2 * i + 1 < nv ? ex2_approx(arg.y) : 0.f;
        acc = __fadd2_rn(acc, make_float2(e0, e1));
      }
      lsc[c * 128 + r] = acc.x + acc.y;
    }
    quarter_sync<NS>(q);
    float L = 0.f;  // the forward's order: per forward split (chunks s, s + kSplitF, ...), then the splits
#pragma unroll
    for (int sp = 0; sp < kSplitF; ++sp) {
      float part = 0.f;
      for (int c = sp; c < n_chunks; c += kSplitF) part += lsc[c * 128 + r];
      L += part;
    }
    quarter_sync<NS>(q);  // red[] / lsc[] are reused by the caller
    inv = 1.f / L;
  }
  const float ml = M * kLog2e;
  auto write_p = [&](const uint32_t* a, int c, auto masked) {
    constexpr bool kMasked = decltype(masked)::value;
    float sv[16];
    grid_scores16(a, G, fmt, sv);
    uint32_t pk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float2 arg = __ffma2_rn(make_float2(sv[2 * i], sv[2 * i + 1]), f2(G.sl), f2(-ml));
      const float e0 = (!kMasked || 2 * i < tail) ? ex2_approx(arg.x) : 0.f;
      const float e1 = (!kMasked || 2 * i + 1 < tail) ? ex2_approx(arg.y) : 0.f;
      const float2 p2 = __fmul2_rn(make_float2(e0, e1), f2(inv));
      pk[i] = pack2_fmt(p2.x, p2.y, fmt);
    }
    store_p_chunk(sP, c, r, pk);
  };
  for (int c = split; c < n_chunks; c += NS) {
    uint32_t a[16];
    tmem_ld16(trow + c * 16, a);
    tmem_ld_wait();
    if (c == n_chunks - 1 && tail < 16)
      write_p(a, c, std::true_type{});
    else
      write_p(a, c, std::false_type{});
  }
}

// ===========================================================================
// Forward: persistent, one CTA per SM walking the (image, head) items; per
// item K, V and every 128-query tile's Q are loaded once.  The CTA's tiles
// g = 0, 1, ... (item-major) alternate between two TMEM buffers (cols
// 256 (g & 1) ..): S_g = Q K^T there, then O_g = P_g V over the consumed S_g.
//   28 softmax warps (kSplitF column splits per lane quarter), software-
//   pipelined one tile deep: softmax(S_g) in registers (softmax_fwd_regs, one
//   TMEM pass), then the readout of O_{g-1} (its P V ran during that
//   softmax), then P_g into the K-major SW128 P tile
//   issuer (warp 0, one thread): S_{g+1} as soon as O_{g-1} is read out of its
//   buffer, P_g V once P_g is written, the TMA stores of the rounded P tiles
//   (psave), TMA loads — the next item's K and Q once this item's S MMAs have
//   read them, V once its last P V has
// smem: K, V (256 key rows, zero-filled past N), Q_0, Q_1, P, row-exchange
// scratch.  Barriers: 0 K+Q landed, 1 V landed, 2/3 S in buffer 0/1, 4 P
// written, 5/6 O in buffer 0/1, 7/8 buffer 0/1 read out, 9 P tile's TMA store
// has read it
// ===========================================================================
// dynamic: the 1 KB-aligned tiles; the row-exchange scratch and the barriers are static
// __shared__ arrays (constant-offset LDS/STS addressing, nothing for the compiler to
// rematerialise in the register-capped softmax warps)
constexpr size_t kAttnSmemF = 1024 + 2 * kAttnKV + 2 * kAttnQ + kAttnP;

template <int KC, int FMT>
__global__ void __launch_bounds__(kAttnThreadsF, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmP,
                    const __grid_constant__ AttnParams P) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ float red_m[kSplitF * 128];
  __shared__ float red_l[kSplitF * 128];
  __shared__ uint64_t bar[10];
  __shared__ uint32_t tmem_slot[1];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sK = smem;
  uint8_t* sV = sK + kAttnKV;
  uint8_t* sQ = sV + kAttnKV;  // Q_0, Q_1
  uint8_t* sP = sQ + 2 * kAttnQ;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int T = P.m_tiles;
  const int n_chunks = (P.N + 15) / 16;
  // this CTA's items blockIdx.x, + gridDim.x, ...; tiles g = item index * T + t
  const int n_items = P.items > (int)blockIdx.x ? (P.items - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int G = n_items * T;

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int i = 0; i < 10; ++i) mbar_init(&bar[i], (i == 4 || i == 7 || i == 8) ? 128 * kSplitF : 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ::mpx::pdl_grid_sync();  // prologue done: wait for the predecessor's outputs

  if (warp == 0) {
    if (G > 0) {  // warp-wide loop; one elected lane issues (operands stay warp-uniform)
      auto item_of = [&](int i) { return (int)blockIdx.x + i * (int)gridDim.x; };
      auto load_kq = [&](int i) {
        const int item = item_of(i), hh = item % P.H, bb = item / P.H;
        mbar_arrive_expect_tx(&bar[0], kAttnKV + T * kAttnQ);
        tma_load_4d(sK, &tmK, &bar[0], 0, 0, hh, bb);
        for (int t = 0; t < T; ++t) tma_load_4d(sQ + t * kAttnQ, &tmQ, &bar[0], 0, t * 128, hh, bb);
      };
      auto load_v = [&](int i) {
        const int item = item_of(i);
        mbar_arrive_expect_tx(&bar[1], kAttnKV);
        tma_load_4d(sV, &tmV, &bar[1], 0, 0, item % P.H, item / P.H);
      };
      if (elect_one()) {
        load_kq(0);
        load_v(0);
      }
      __syncwarp();
      constexpr uint32_t kHi = 0x40004040u;  // SW128 descriptor high word (SBO 1024, version, swizzle)
      auto lo = [](uint32_t addr, uint32_t lbo) { return (addr >> 4) | ((lbo >> 4) << 16); };
      const uint32_t idesc1 = idesc_f16(FMT, 128, 16 * n_chunks, 0, 0);  // keys past N: never computed
      const uint32_t idesc2 = idesc_f16(FMT, 128, 64, 0, 1);
      const uint32_t k = smem_u32(sK), v = smem_u32(sV), p = smem_u32(sP);
      auto issue_s = [&](int gs) {  // S_gs = Q_t K^T into buffer gs & 1
        const int i = gs / T, t = gs - i * T, buf = gs & 1;
        if (t == 0) mbar_wait(&bar[0], i & 1);                            // the item's K and Q landed
        if (gs >= 2) mbar_wait(&bar[7 + buf], ((gs >> 1) - 1) & 1);       // O_{gs-2} read out of the buffer
        tc_fence_after();
        const uint32_t q = smem_u32(sQ + t * kAttnQ);
        if (elect_one()) {
#pragma unroll
          for (int s = 0; s < 4; ++s)
            umma_f16_w(tmem + 256 * buf, lo(q, 16) + s * 2, kHi, lo(k, 16) + s * 2, kHi, idesc1, s > 0);
          umma_commit(&bar[2 + buf]);
        }
        __syncwarp();
        if (t == T - 1 && i + 1 < n_items) {  // K and the Q tiles are free once these S MMAs completed
          mbar_wait(&bar[2 + buf], (gs >> 1) & 1);
          if (elect_one()) load_kq(i + 1);
          __syncwarp();
        }
      };
      issue_s(0);
      for (int g = 0; g < G; ++g) {
        if (g % T == 0 && g / T == kTraceIt) ATRACE(0);
        if (g % T == 0 && g / T == kTraceIt + 1) ATRACE(20);
        if (g + 1 < G) issue_s(g + 1);
        const int i = g / T, t = g - i * T, buf = g & 1;
        if (t == 0) mbar_wait(&bar[1], i & 1);  // V landed
        mbar_wait(&bar[4], g & 1);              // P_g written (S_g consumed)
        tc_fence_after();
        if (elect_one()) {
          if (P.psave) {  // the rounded P tile as the MMAs read it (rows < N, keys < 16 n_chunks)
            for (int blk = 0; blk * 4 < n_chunks; ++blk)
              tma_store_4d(&tmP, sP + blk * 16384, blk * 64, t * 128, item_of(i), 0);
            bulk_commit();
          }
          for (int s = 0; s < n_chunks; ++s)  // O_g = P_g V
            umma_f16_w(tmem + 256 * buf, lo(p, 16) + (s >> 2) * 1024 + (s & 3) * 2, kHi, lo(v, 8192) + s * 128, kHi,
                       idesc2, s > 0);
          umma_commit(&bar[5 + buf]);
          if (P.psave) bulk_wait_read0();  // (the bulk group belongs to the issuing thread)
          mbar_arrive(&bar[9]);
        }
        __syncwarp();
        if (t == T - 1 && i + 1 < n_items) {  // V is free once this P V completed
          mbar_wait(&bar[5 + buf], (g >> 1) & 1);
          if (elect_one()) load_v(i + 1);
          __syncwarp();
        }
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3, split = (warp - 4) >> 2;
    const int r = q * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    const ScoreGrid G2(P.scale, FMT);
    // tile bookkeeping advanced incrementally (no divisions per tile): the
    // current tile (t, item = b H + h) and the previous one, whose O is read out
    const int hstep = (int)gridDim.x % P.H, bstep = (int)gridDim.x / P.H;
    int t = 0, item = blockIdx.x, h = item % P.H, b = item / P.H;
    int pt = 0, ph_ = 0, pb = 0;
    // O rows of the previous tile -> O (one 16-column chunk per split 0-3, two 8-column loads)
    auto drain = [&](int g) {
      const int buf = g & 1;
      quarter_wait<kSplitF>(&bar[5 + buf], (g >> 1) & 1, split, q);
      tc_fence_after();
      const int qrow = pt * 128 + r;
      if (split < 4 && pt * 128 + q * 32 < P.N) {
        uint16_t* o = static_cast<uint16_t*>(P.O) + ((long long)pb * P.N + qrow) * P.ldo + (long long)ph_ * P.hd +
                      split * 16;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t o32[8];
          tmem_ld8(trow + 256 * buf + split * 16 + hh * 8, o32);
          tmem_ld_wait();
          if (qrow < P.N)
            *reinterpret_cast<uint4*>(o + hh * 8) =
                make_uint4(pack2T<FMT>(__uint_as_float(o32[0]), __uint_as_float(o32[1])),
                           pack2T<FMT>(__uint_as_float(o32[2]), __uint_as_float(o32[3])),
                           pack2T<FMT>(__uint_as_float(o32[4]), __uint_as_float(o32[5])),
                           pack2T<FMT>(__uint_as_float(o32[6]), __uint_as_float(o32[7])));
        }
      }
      tc_fence_before();
      mbar_arrive(&bar[7 + buf]);
    };
    for (int g = 0; g < G; ++g) {
      const int buf = g & 1;
      // a lane quarter whose 32 query rows are all padding (rows >= N of the last
      // tile) skips the softmax: its P rows keep whatever finite bytes the tile
      // held, feed only O rows that are never stored, and are clipped from the saved P
      const bool live = t * 128 + q * 32 < P.N;
      quarter_wait<kSplitF>(&bar[2 + buf], (g >> 1) & 1, split, q);
      const bool tr = warp == 4 && lane == 0 && (g / T) == kTraceIt;
      if (tr) ATRACE(1 + 8 * t);
      tc_fence_after();
      uint32_t a[KC][16];
      float2 st = make_float2(0.f, 0.f);
      if (live) st = softmax_fwd_regs<kSplitF, KC, FMT>(trow + 256 * buf, split, r, q, P.N, G2, red_m, red_l, a);
      if (tr) ATRACE(2 + 8 * t);
      if (g > 0) {
        drain(g - 1);                     // O_{g-1}: its P V also means the P tile is no longer read by MMAs
        if (tr) ATRACE(3 + 8 * t);
        quarter_wait<kSplitF>(&bar[9], (g - 1) & 1, split, q);  // ... and its TMA store has read it
      }
      if (tr) ATRACE(4 + 8 * t);
      if (live) softmax_store_p<kSplitF, KC, FMT>(split, r, P.N, st.y, a, sP);
      // every row's statistics, padding quarters included: (0, 0) makes the backward's
      // recomputed P of those rows exactly 0 (they multiply dO rows that are zero, and
      // garbage statistics would turn 0 * P into NaN in dV)
      if (P.stats != nullptr && split == 0) P.stats[((long long)item * T + t) * 128 + r] = live ? st : make_float2(0.f, 0.f);
      fence_async_smem();  // generic-proxy smem writes -> visible to the tensor core / TMA
      tc_fence_before();
      mbar_arrive(&bar[4]);
      if (tr) ATRACE(5 + 8 * t);
      pt = t;
      ph_ = h;
      pb = b;
      if (++t == T) {
        t = 0;
        item += gridDim.x;
        h += hstep;
        b += bstep;
        if (h >= P.H) {
          h -= P.H;
          ++b;
        }
      }
    }
    if (G > 0) drain(G - 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ===========================================================================
// Backward: one CTA per (b, h), both 128-query tiles, all keys on chip.
//   dP = dO V^T;  dS = P * (dP - rowsum(P * dP));  dV = P^T dO;
//   dK = scale * dS^T Q;  dQ = scale * dS K        (autodiff.py:193-205, 233-240)
// TMEM: cols 0-255 S, then dP, then dQ (per tile); 256-383 dV, 384-511 dK
// (keys 0-127 / 128-255 as two M=128 halves), accumulated over the tiles.
// smem: Q_t, dO_t (16 KB each), K, V (32 KB), P_t, dS_t (64 KB each): the P /
// dS tiles are K-major A operands for dQ and, read MN-major, for dV / dK.
// ===========================================================================
// 224 KB of tiles + 2 KB reduction scratch + barriers: the alignment slack is
// trimmed to fit the 227 KB limit (the dynamic window starts 1 KB-aligned when
// the kernel has no static shared memory; checked at run time)
constexpr size_t kAttnBwdBody = 2 * kAttnQ + 2 * kAttnKV + 2 * kAttnP + kSplit * 128 * 4 + 160;
constexpr size_t kAttnBwdSmem = 232448;
static_assert(kAttnBwdBody <= kAttnBwdSmem, "attention backward tiles exceed shared memory");

struct AttnBwdParams {
  int N, H, hd, m_tiles;
  float scale;
  int fmt;
  void* dqkv;  // [B*N, 3*H*hd]
  long long ld;
  const float2* stats;  // the forward's row statistics, or null (recomputed here)
  float* csum;          // optional per-image column sums of dqkv [B][3*H*hd] (the qkv bias gradient's partials)
  int items;            // B * H work items, walked by a persistent grid
  const uint8_t* psaved;  // optional: the forward's P tiles (attn_fwd psave) — reloaded instead of recomputed
};


template <int FMT>  // 0 f16, 1 bf16: one conversion path compiled
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                    const __grid_constant__ CUtensorMap tmP, const __grid_constant__ AttnBwdParams P) {
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned by indexing the __shared__ array (not via an integer cast), so
  // derived pointers stay in the shared window: STS/LDS, 32-bit addressing
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  if (reinterpret_cast<uintptr_t>(smem) - reinterpret_cast<uintptr_t>(smem_raw) + kAttnBwdBody > kAttnBwdSmem) __trap();
  uint8_t* sQ = smem;
  uint8_t* sdO = sQ + kAttnQ;
  uint8_t* sK = sdO + kAttnQ;
  uint8_t* sV = sK + kAttnKV;
  uint8_t* sP = sV + kAttnKV;
  uint8_t* sdS = sP + kAttnP;
  // 0 V landed, 1 dO_t (+ saved P_t) landed, 2 S, 3 P, 4 dP, 5 dS, 6 dQ done (K free), 7 dQ read,
  // 8 dK done (Q free), 9 dV done (dO / P free), 10 dV/dK read out (the next item may overwrite
  // TMEM cols 256-511), 11 Q_t landed, 12 K landed
  float* red = reinterpret_cast<float*>(sdS + kAttnP);
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + kSplit * 128);
  uint64_t* cready = bar + 13;  // qkv-bias column sums handed to warps 1-3: cready[2], cdone[2]
  uint64_t* cdone = bar + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 17);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int T = P.m_tiles;
  const long long D = (long long)P.H * P.hd;
  // qkv-bias column sums, off the softmax warps: cready[s] completes when every softmax
  // thread has stored item it's dQ / dK / dV rows (s = it & 1), cdone[s] when warps 1-3
  // have summed them (the softmax warps wait for it two items later)

  if (threadIdx.x == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    tma_prefetch(&tmdO);
    for (int i = 0; i < 13; ++i) mbar_init(&bar[i], (i == 3 || i == 5 || i == 7 || i == 10) ? 128 * kSplit : 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&cready[i], 128 * kSplit);
      mbar_init(&cdone[i], 3);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  ::mpx::pdl_grid_sync();  // prologue done: wait for the predecessor's outputs

  if (warp == 0) {
    {  // warp-wide loop; one elected lane issues (operands stay warp-uniform)
      // persistent: items blockIdx.x, + gridDim.x, ...  Every operand tile is
      // reloaded the moment its last reader has finished, on its own barrier,
      // so loads stream while the MMAs and the softmax warps work:
      //   V      after the item's last dP (waited through dS ready)   -> next item's V
      //   dO, P  after dV_t (and the dS pass, which read P_t)          -> tile t+1 / next item's tile 0
      //   K      after the item's last dQ                             -> next item's K
      //   Q      after dK_t                                           -> tile t+1 / next item's tile 0
      // dP needs only dO and V, so the next item's first dP no longer waits for its K and Q.
      const bool saved = P.psaved != nullptr;
      const int n_pblk = ((P.N + 15) / 16 + 3) / 4;  // 64-key blocks of the saved P
      const uint32_t dop_tx = kAttnQ + (saved ? n_pblk * 16384 : 0);  // dO (+ the saved P) per tile
      auto load_dop = [&](int item, int t) {
        mbar_arrive_expect_tx(&bar[1], dop_tx);
        tma_load_4d(sdO, &tmdO, &bar[1], 0, t * 128, item % P.H, item / P.H);
        if (saved)
          for (int blk = 0; blk < n_pblk; ++blk)
            tma_load_4d(sP + blk * 16384, &tmP, &bar[1], blk * 64, t * 128, item, 0);
      };
      auto load_q = [&](int item, int t) {
        mbar_arrive_expect_tx(&bar[11], kAttnQ);
        tma_load_4d(sQ, &tmQ, &bar[11], 0, t * 128, item % P.H, item / P.H);
      };
      auto load_v = [&](int item) {
        mbar_arrive_expect_tx(&bar[0], kAttnKV);
        tma_load_4d(sV, &tmV, &bar[0], 0, 0, item % P.H, item / P.H);
      };
      auto load_k = [&](int item) {
        mbar_arrive_expect_tx(&bar[12], kAttnKV);
        tma_load_4d(sK, &tmK, &bar[12], 0, 0, item % P.H, item / P.H);
      };
      const uint32_t q = smem_u32(sQ), dO = smem_u32(sdO), k = smem_u32(sK), v = smem_u32(sV);
      const uint32_t pp = smem_u32(sP), ds = smem_u32(sdS);
      const int n_chunks = (P.N + 15) / 16;
      const int halves = P.N > 128 ? 2 : 1;
      // [128 x 16 n_chunks] = X[128 x 64] Y[keys x 64]^T: keys past N are never computed
      const uint32_t id_nk = idesc_f16(FMT, 128, 16 * n_chunks, 0, 0);
      const uint32_t id_kv = idesc_f16(FMT, 128, 64, 1, 1);   // dV / dK halves: A, B MN-major
      const uint32_t id_q = idesc_f16(FMT, 128, 64, 0, 1);    // dQ: A K-major, B MN-major
      uint32_t gt = 0;  // tiles so far (barrier phases)
      int it = 0;       // items so far
      if (blockIdx.x < P.items && elect_one()) {
        load_v(blockIdx.x);
        load_dop(blockIdx.x, 0);
        load_k(blockIdx.x);
        load_q(blockIdx.x, 0);
      }
      __syncwarp();
      // SW128 descriptor low words ((address >> 4) | (LBO >> 4) << 16); the high word is constant
      constexpr uint32_t kHi = 0x40004040u;
      auto lo = [](uint32_t addr, uint32_t lbo) { return (addr >> 4) | ((lbo >> 4) << 16); };
      for (int item = blockIdx.x; item < P.items; item += gridDim.x, ++it) {
        const int next = item + (int)gridDim.x;
        if (it == kTraceIt) ATRACE(0);
        if (it == kTraceIt + 1) ATRACE(21);
        for (int t = 0; t < T; ++t, ++gt) {
          const uint32_t ph = gt & 1;
          mbar_wait(&bar[1], ph);  // dO_t (+ P_t)
          if (t == 0) mbar_wait(&bar[0], it & 1);  // V
          if (it == kTraceIt) ATRACE(2 + 8 * t);
          if (gt > 0) mbar_wait(&bar[7], ph ^ 1);  // previous dQ drained from TMEM cols 0-63
          tc_fence_after();
          if (!saved) {  // recompute P: S = Q K^T, softmax by the softmax warps
            if (t == 0) mbar_wait(&bar[12], it & 1);
            mbar_wait(&bar[11], ph);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
              for (int s = 0; s < 4; ++s)  // S = Q K^T
                umma_f16_w(tmem, lo(q, 16) + s * 2, kHi, lo(k, 16) + s * 2, kHi, id_nk, s > 0);
              umma_commit(&bar[2]);
            }
            __syncwarp();
            mbar_wait(&bar[3], ph);  // P_t written (S consumed)
            if (it == kTraceIt) ATRACE(3 + 8 * t);
            tc_fence_after();
          }
          if (elect_one()) {
#pragma unroll
            for (int s = 0; s < 4; ++s)  // dP = dO V^T
              umma_f16_w(tmem, lo(dO, 16) + s * 2, kHi, lo(v, 16) + s * 2, kHi, id_nk, s > 0);
            umma_commit(&bar[4]);
          }
          __syncwarp();
          // dV needs only P_t and dO_t: it runs on the tensor pipe while the
          // softmax warps turn dP into dS (TMEM cols 256-383, disjoint from dP)
          if (t == 0 && it > 0) {
            mbar_wait(&bar[10], (it - 1) & 1);  // last item's dV/dK read out of TMEM
            tc_fence_after();
          }
          if (elect_one()) {
            for (int half = 0; half < halves; ++half) {
#pragma unroll
              for (int s = 0; s < 8; ++s)  // dV += P^T dO
                umma_f16_w(tmem + 256 + half * 64, lo(pp + half * 32768, 16384) + s * 128, kHi,
                           lo(dO, 8192) + s * 128, kHi, id_kv, (t > 0 || s > 0));
            }
            umma_commit(&bar[9]);
          }
          __syncwarp();
          mbar_wait(&bar[5], ph);  // dS_t written (dP consumed, P_t no longer read by the softmax warps)
          if (it == kTraceIt) ATRACE(4 + 8 * t);
          if (t == T - 1 && next < P.items && elect_one()) load_v(next);  // the item's dP MMAs are done with V
          __syncwarp();
          if (t == 0) mbar_wait(&bar[12], it & 1);  // K
          tc_fence_after();
          // dQ first, so the softmax warps read it out while dK runs
          if (elect_one()) {
            for (int s = 0; s < n_chunks; ++s)  // dQ = dS K
              umma_f16_w(tmem, lo(ds, 16) + (s >> 2) * 1024 + (s & 3) * 2, kHi, lo(k, 8192) + s * 128, kHi, id_q,
                         s > 0);
            umma_commit(&bar[6]);
          }
          __syncwarp();
          mbar_wait(&bar[11], ph);  // Q_t
          tc_fence_after();
          if (elect_one()) {
            for (int half = 0; half < halves; ++half) {
#pragma unroll
              for (int s = 0; s < 8; ++s)  // over the 128 queries of the tile: dK += dS^T Q
                umma_f16_w(tmem + 384 + half * 64, lo(ds + half * 32768, 16384) + s * 128, kHi,
                           lo(q, 8192) + s * 128, kHi, id_kv, (t > 0 || s > 0));
            }
            umma_commit(&bar[8]);
          }
          __syncwarp();
          const bool more = t + 1 < T;
          if (more || next < P.items) {
            const int li = more ? item : next, lt = more ? t + 1 : 0;
            mbar_wait(&bar[9], ph);  // dV_t done: dO and P free (the dS pass finished with P_t)
            if (elect_one()) load_dop(li, lt);
            __syncwarp();
            if (!more) {
              mbar_wait(&bar[6], ph);  // the item's last dQ is done with K
              if (elect_one()) load_k(next);
              __syncwarp();
            }
            mbar_wait(&bar[8], ph);  // dK_t done: Q free
            if (elect_one()) load_q(li, lt);
            __syncwarp();
          }
        }
      }
    }
  } else if (warp <= 3) {
    if (P.csum) {  // warps 1-3 (q, k, v): per item, the column sums of the part's stored rows (fresh
                   // in L2): lane = 8 rp + co sums columns 8co..8co+7 over rows rp, rp + 4, ... with
                   // 16-byte loads, 8 rows in flight; the 4 row phases are then added in a fixed tree
      const int part = warp - 1, rp = lane >> 3, co = lane & 7;
      int it = 0;
      for (int item = blockIdx.x; item < P.items; item += gridDim.x, ++it) {
        const int s = it & 1;
        mbar_wait(&cready[s], (uint32_t)(it >> 1) & 1u);
        const int h = item % P.H, b = item / P.H;
        const uint16_t* col = static_cast<const uint16_t*>(P.dqkv) + (long long)b * P.N * P.ld + part * D +
                              (long long)h * P.hd + 8 * co;
        float2 acc[4] = {f2(0.f), f2(0.f), f2(0.f), f2(0.f)};
        int rr = rp;
        for (; rr + 28 < P.N; rr += 32) {
          uint4 w[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) w[u] = *reinterpret_cast<const uint4*>(col + (long long)(rr + 4 * u) * P.ld);
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            acc[0] = add_h2<FMT>(acc[0], w[u].x);
            acc[1] = add_h2<FMT>(acc[1], w[u].y);
            acc[2] = add_h2<FMT>(acc[2], w[u].z);
            acc[3] = add_h2<FMT>(acc[3], w[u].w);
          }
        }
        for (; rr < P.N; rr += 4) {
          const uint4 w = *reinterpret_cast<const uint4*>(col + (long long)rr * P.ld);
          acc[0] = add_h2<FMT>(acc[0], w.x);
          acc[1] = add_h2<FMT>(acc[1], w.y);
          acc[2] = add_h2<FMT>(acc[2], w.z);
          acc[3] = add_h2<FMT>(acc[3], w.w);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // (p0 + p1) + (p2 + p3) over the row phases
          acc[i].x += __shfl_xor_sync(0xffffffffu, acc[i].x, 8);
          acc[i].y += __shfl_xor_sync(0xffffffffu, acc[i].y, 8);
          acc[i].x += __shfl_xor_sync(0xffffffffu, acc[i].x, 16);
          acc[i].y += __shfl_xor_sync(0xffffffffu, acc[i].y, 16);
        }
        if (rp == 0) {
          float4* o = reinterpret_cast<float4*>(P.csum + (long long)b * 3 * D + part * D + (long long)h * P.hd + 8 * co);
          o[0] = make_float4(acc[0].x, acc[0].y, acc[1].x, acc[1].y);
          o[1] = make_float4(acc[2].x, acc[2].y, acc[3].x, acc[3].y);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&cdone[s]);
      }
    }
  } else if (warp >= 4) {
    const int qd = warp & 3, split = (warp - 4) >> 2;
    const int r = qd * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(qd * 32) << 16);
    const int n_chunks = (P.N + 15) / 16;
    const int sw = r & 7;
    auto read_pw = [&](int c, uint32_t* u) {  // own row of P_t, keys 16c..16c+15, as 8 packed pairs
      const uint8_t* rowp = sP + (c >> 2) * 16384 + r * 128;
      const int u0 = (c & 3) * 2;
      const uint4 w0 = *reinterpret_cast<const uint4*>(rowp + ((u0 ^ sw) << 4));
      const uint4 w1 = *reinterpret_cast<const uint4*>(rowp + (((u0 + 1) ^ sw) << 4));
      u[0] = w0.x, u[1] = w0.y, u[2] = w0.z, u[3] = w0.w, u[4] = w1.x, u[5] = w1.y, u[6] = w1.z, u[7] = w1.w;
    };
    constexpr int kMaxC = 16 / kSplit;  // chunks per thread
    static_assert(kSplit == 4, "dQ readout: one chunk per split");
    uint32_t gt = 0;  // tiles so far (barrier phases)
    int it = 0;       // items so far
    for (int item = blockIdx.x; item < P.items; item += gridDim.x, ++it) {
    const int h = item % P.H, b = item / P.H;
    for (int t = 0; t < T; ++t, ++gt) {
      const uint32_t ph = gt & 1;
      if (P.psaved == nullptr) {
        // ---- P = softmax(round(S * scale)) -> smem (as in the forward)
        float2 st = make_float2(0.f, 0.f);  // the forward's (max, 1/sum), fetched while S is computed
        if (P.stats) st = __ldg(P.stats + ((long long)item * T + t) * 128 + r);
        mbar_wait(&bar[2], ph);
        if (warp == 4 && lane == 0 && it == kTraceIt) ATRACE(5 + 8 * t);
        tc_fence_after();
        softmax_bwd_p<kSplit>(trow, split, r, qd, P.N, P.scale, FMT, red, reinterpret_cast<float*>(sdS), sP,
                              P.stats ? &st : nullptr);
        fence_async_smem();
        tc_fence_before();
        mbar_arrive(&bar[3]);
      } else {
        mbar_wait(&bar[1], ph);  // the forward's P tile has landed (TMA) before it is read here
      }
      // ---- dS = P * (dP - sum(P * dP)) -> smem; dP rounded to the half
      // format first (the reference's dP is a half GEMM output), kept packed
      mbar_wait(&bar[4], ph);
      if (warp == 4 && lane == 0 && it == kTraceIt) ATRACE(6 + 8 * t);
      tc_fence_after();
      uint32_t dpk[kMaxC][8];
      float2 tsum2 = f2(0.f);
#pragma unroll
      for (int j = 0; j < kMaxC; ++j) {
        const int c = split + j * kSplit;
        if (c < n_chunks) {
          uint32_t a[16], pw[8];
          tmem_ld16(trow + c * 16, a);
          read_pw(c, pw);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 8; ++i) {  // P * dP on the half pairs: FHFMA, the same bits as unpack + FFMA2
            dpk[j][i] = pack2_fmt(__uint_as_float(a[2 * i]), __uint_as_float(a[2 * i + 1]), FMT);
            tsum2 = fma_h2<FMT>(pw[i], dpk[j][i], tsum2);
          }
        }
      }
      red[split * 128 + r] = tsum2.x + tsum2.y;
      quarter_sync<kSplit>(qd);
      float tsum = 0.f;
#pragma unroll
      for (int j = 0; j < kSplit; ++j) tsum += red[j * 128 + r];
      quarter_sync<kSplit>(qd);
#pragma unroll
      for (int j = 0; j < kMaxC; ++j) {
        const int c = split + j * kSplit;
        if (c < n_chunks) {
          uint32_t pw[8];
          read_pw(c, pw);
          uint32_t pk[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {  // dS = P (dP - t): dP - t by FHADD on the packed dP
            const float2 ds = __fmul2_rn(unpack2_fmt<FMT>(pw[i]), add_h2<FMT>(f2(-tsum), dpk[j][i]));
            pk[i] = pack2_fmt(ds.x, ds.y, FMT);
          }
          store_p_chunk(sdS, c, r, pk);
        }
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(&bar[5]);
      // ---- dQ_t -> dqkv[:, q part]
      mbar_wait(&bar[6], ph);
      if (warp == 4 && lane == 0 && it == kTraceIt) ATRACE(7 + 8 * t);
      tc_fence_after();
      const int qrow = t * 128 + r;
      uint16_t* o = static_cast<uint16_t*>(P.dqkv) + ((long long)b * P.N + qrow) * P.ld + (long long)h * P.hd;
      {
        const int c = split;  // kSplit == 4: one 16-column chunk of dQ per thread
        uint32_t a[16];
        tmem_ld16(trow + c * 16, a);
        tmem_ld_wait();
        // dQ is in registers: free its TMEM columns for the next tile's MMAs first, then
        // store it and take its column sums off the MMA critical path
        tc_fence_before();
        mbar_arrive(&bar[7]);
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          pk[i] = pack2_fmt(__uint_as_float(a[2 * i]) * P.scale, __uint_as_float(a[2 * i + 1]) * P.scale, FMT);
        if (qrow < P.N) {
          *reinterpret_cast<uint4*>(o + c * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4*>(o + c * 16 + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
      if (warp == 4 && lane == 0 && it == kTraceIt) ATRACE(8 + 8 * t);
    }
    // ---- dV, dK (keys r and 128 + r of this head): 4 (half, which) combos split over the warps,
    // once the last tile's dK MMAs (issued after its dQ) have completed
    mbar_wait(&bar[8], (gt - 1) & 1);
    tc_fence_after();
    const int half = split >> 1, which = split & 1;  // kSplit == 4: one combo per split
    {
      const int key = half * 128 + r;
      uint16_t* o = static_cast<uint16_t*>(P.dqkv) + ((long long)b * P.N + key) * P.ld + (which ? D : 2 * D) +
                    (long long)h * P.hd;
      const float mul = which ? P.scale : 1.f;
      for (int c = 0; c < 4; ++c) {
        uint32_t a[16];
        tmem_ld16(trow + 256 + which * 128 + half * 64 + c * 16, a);
        tmem_ld_wait();
        if (c == 3) {  // the last dV/dK read: the next item may accumulate into TMEM cols 256-511
          tc_fence_before();  // while this item's stores, column sums and combine finish
          mbar_arrive(&bar[10]);
        }
        uint32_t pk[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          pk[i] = pack2_fmt(__uint_as_float(a[2 * i]) * mul, __uint_as_float(a[2 * i + 1]) * mul, FMT);
        if (key < P.N) {
          *reinterpret_cast<uint4*>(o + c * 16) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4*>(o + c * 16 + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
    }
    if (P.csum) {  // this item's rows are stored: hand them to warps 1-3 (after they took item it - 2)
      if (it >= 2) mbar_wait(&cdone[it & 1], (uint32_t)((it >> 1) - 1) & 1u);
      mbar_arrive(&cready[it & 1]);
    }
    if (warp == 4 && lane == 0 && it == kTraceIt) ATRACE(20);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) ATRACE(30);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// the column-sum second pass over many partial rows (mpx_gemm.cu)
__global__ void colsum_parts_kernel(const float* __restrict__ parts, int nparts, int N, void* out, int out_dtype);

static PFN_cuTensorMapEncodeTiled_v12000 attn_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// map over one of Q/K/V inside qkv [B, N, 3, H, hd]: dims (hd, N, H, B)
static int qkv_map(CUtensorMap* m, const void* base, int fmt, int N, int H, int hd, int B, uint32_t box_rows,
                   int row_heads = 3) {
  auto fn = attn_encode_fn();
  if (!fn) return fail(MPX_EINVAL, "cuTensorMapEncodeTiled unavailable");
  const uint64_t row = (uint64_t)row_heads * H * hd * 2;
  cuuint64_t dims[4] = {(cuuint64_t)hd, (cuuint64_t)N, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[3] = {row, (cuuint64_t)hd * 2, row * N};
  cuuint32_t box[4] = {64, box_rows, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, fmt ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                  const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MPX_EINVAL, "attention tensor map failed (" + std::to_string((int)r) + ")");
  return 0;
}

// map over the saved probabilities: [B*H][N rows][16*ceil(N/16) keys] half,
// boxes of 64 keys x 128 rows, 128B-swizzled = exactly the smem P tile's blocks
static int p_map(CUtensorMap* m, const void* base, int fmt, int N, int BH) {
  auto fn = attn_encode_fn();
  if (!fn) return fail(MPX_EINVAL, "cuTensorMapEncodeTiled unavailable");
  const uint64_t keys = 16ull * ((N + 15) / 16);
  cuuint64_t dims[4] = {(cuuint64_t)keys, (cuuint64_t)N, (cuuint64_t)BH, 1};
  cuuint64_t strides[3] = {keys * 2, keys * 2 * N, keys * 2 * N * BH};
  cuuint32_t box[4] = {64, 128, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, fmt ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                  const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MPX_EINVAL, "attention P tensor map failed (" + std::to_string((int)r) + ")");
  return 0;
}

}  // namespace mpx

using namespace mpx;

#ifdef MPX_TRACE
extern "C" int mpx_debug_attn_trace(long long* host_out) {  // kTraceCtas * kTraceSlots int64
  MPX_CUDA_CHECK(cudaMemcpyFromSymbol(host_out, g_attn_trace, sizeof(long long) * kTraceCtas * kTraceSlots));
  return 0;
}
#endif

extern "C" int mpx_attention_fwd(int dtype, const void* qkv, int B, int N, int H, int hd, float scale, void* O,
                                 int64_t ldo, float* row_stats, void* p_save, void* stream) {
  if (dtype != MPX_F16 && dtype != MPX_BF16) return fail(MPX_EINVAL, "attention: f16/bf16 only");
  if (hd != 64 || N < 1 || N > 256) return fail(MPX_EINVAL, "attention_fwd: fused path needs hd == 64, N <= 256");
  const int fmt = dtype == MPX_BF16 ? 1 : 0;
  const uint16_t* base = static_cast<const uint16_t*>(qkv);
  const int D = H * hd;
  CUtensorMap tq, tk, tv;
  int rc = qkv_map(&tq, base, fmt, N, H, hd, B, 128);
  if (!rc) rc = qkv_map(&tk, base + D, fmt, N, H, hd, B, 256);
  if (!rc) rc = qkv_map(&tv, base + 2 * D, fmt, N, H, hd, B, 256);
  CUtensorMap tp = tv;
  if (!rc && p_save) rc = p_map(&tp, p_save, fmt, N, B * H);
  if (rc) return rc;
  AttnParams P{};
  P.N = N;
  P.H = H;
  P.hd = hd;
  P.m_tiles = (N + 127) / 128;
  P.scale = scale;
  P.fmt = fmt;
  P.O = O;
  P.ldo = ldo;
  P.stats = reinterpret_cast<float2*>(row_stats);
  P.psave = static_cast<uint8_t*>(p_save);
  P.items = B * H;
  const int kc3 = (N + 15) / 16 > 2 * kSplitF;
  auto kern = kc3 ? (fmt ? attn_fwd_kernel<3, 1> : attn_fwd_kernel<3, 0>)
                  : (fmt ? attn_fwd_kernel<2, 1> : attn_fwd_kernel<2, 0>);
  cudaError_t err = ensure_smem_attr((const void*)kern, (int)kAttnSmemF);
  if (err != cudaSuccess) return fail((int)err, "cudaFuncSetAttribute(attn_fwd_kernel)");
  // persistent: one CTA per SM walks the (image, head) items; KC = score chunks
  // per softmax thread (2 up to N = 224)
  const unsigned grid = (unsigned)std::min(B * H, current_num_sms());
  MPX_CUDA_CHECK(::mpx::launch_k(kern, grid, kAttnThreadsF, kAttnSmemF, static_cast<cudaStream_t>(stream), tq, tk,
                                 tv, tp, P));
  MPX_LAUNCH_CHECK("attn_fwd_kernel");
  return 0;
}

extern "C" int64_t mpx_attention_psave_bytes(int B, int N, int H) {
  return (int64_t)B * H * N * (16 * ((N + 15) / 16)) * 2;  // [B*H][N][16 ceil(N/16)] half
}

extern "C" int mpx_attention_bwd(int dtype, const void* qkv, const void* dO, int B, int N, int H, int hd, float scale,
                                 void* dqkv, const float* row_stats, const void* p_saved, float* colsum_ws,
                                 void* colsum_out, void* stream) {
  if (dtype != MPX_F16 && dtype != MPX_BF16) return fail(MPX_EINVAL, "attention: f16/bf16 only");
  if (hd != 64 || N < 1 || N > 256) return fail(MPX_EINVAL, "attention_bwd: fused path needs hd == 64, N <= 256");
  const int fmt = dtype == MPX_BF16 ? 1 : 0;
  const uint16_t* base = static_cast<const uint16_t*>(qkv);
  const int D = H * hd;
  CUtensorMap tq, tk, tv, tdo;
  int rc = qkv_map(&tq, base, fmt, N, H, hd, B, 128);
  if (!rc) rc = qkv_map(&tk, base + D, fmt, N, H, hd, B, 256);
  if (!rc) rc = qkv_map(&tv, base + 2 * D, fmt, N, H, hd, B, 256);
  if (!rc) rc = qkv_map(&tdo, dO, fmt, N, H, hd, B, 128, 1);
  CUtensorMap tp = tv;
  if (!rc && p_saved) rc = p_map(&tp, p_saved, fmt, N, B * H);
  if (rc) return rc;
  AttnBwdParams P{};
  P.N = N;
  P.H = H;
  P.hd = hd;
  P.m_tiles = (N + 127) / 128;
  P.scale = scale;
  P.fmt = fmt;
  P.dqkv = dqkv;
  P.ld = 3LL * D;
  P.stats = reinterpret_cast<const float2*>(row_stats);
  P.psaved = static_cast<const uint8_t*>(p_saved);
  if ((colsum_ws == nullptr) != (colsum_out == nullptr))
    return fail(MPX_EINVAL, "attention_bwd: colsum_ws and colsum_out go together");
  P.csum = colsum_ws;
  cudaError_t err = ensure_smem_attr((const void*)(fmt ? attn_bwd_kernel<1> : attn_bwd_kernel<0>), (int)kAttnBwdSmem);
  if (err != cudaSuccess) return fail((int)err, "cudaFuncSetAttribute(attn_bwd_kernel)");
  P.items = B * H;  // persistent: one CTA per SM walks the (image, head) items
  const unsigned grid = (unsigned)std::min(B * H, current_num_sms());
  MPX_CUDA_CHECK(::mpx::launch_k(fmt ? attn_bwd_kernel<1> : attn_bwd_kernel<0>, grid, kAttnThreads, kAttnBwdSmem, static_cast<cudaStream_t>(stream),
                                 tq, tk, tv, tdo, tp, P));
  MPX_LAUNCH_CHECK("attn_bwd_kernel");
  if (colsum_out) {  // the qkv bias gradient: sum the per-image partials [B][3D]
    const int cols = 3 * D;
    MPX_CUDA_CHECK(::mpx::launch_k(colsum_parts_kernel, (unsigned)((cols + 31) / 32), 1024, 0,
                                   static_cast<cudaStream_t>(stream), colsum_ws, B, cols, colsum_out, dtype));
  }
  return 0;
}

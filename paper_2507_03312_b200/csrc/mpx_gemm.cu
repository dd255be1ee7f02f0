// K5 — tcgen05 GEMM for the ViT forward/backward contractions (sm_100a).
//
// Replaces the reference's stepwise matmul (tensors.py:387-422) and its
// backward rule (autodiff.py:193-205) with half-precision operands and f32
// accumulation in TMEM (the north star's mandate).
//
//   C[z][m, n] = epilogue( alpha * sum_k A[z][m, k] * B[z][k, n] )
//
// A and B are each either K-major (k contiguous) or MN-major (m / n
// contiguous), so one kernel serves forward (x @ W), dgrad (dY @ W^T) and
// wgrad (X^T @ dY) without any transpose copies, and batched attention
// (Q K^T, P V, ...) through 4-D TMA tensor maps over the [B, N, 3, H, hd]
// qkv layout.
//
// Structure (one CTA per SM, persistent, 192 threads):
//   warp 0      TMA producer: 128B-swizzled A/B tiles into a 4-stage smem ring
//   warp 1      MMA issuer: tcgen05.mma M=128 x N=BN x K=16, f32 accumulators in
//               TMEM, double-buffered (2 x 256 columns) so the epilogue of tile
//               i overlaps the MMAs of tile i+1; owns TMEM alloc/dealloc
//   warps 2..5  epilogue: tcgen05.ld -> alpha, +bias, GELU (saving the
//               pre-activation), GELU' (backward), +residual -> f16/bf16/f32
// Tiles are rastered in groups of 16 M-blocks so the A panels and the whole
// B operand of the CTAs in flight stay L2-resident.
#include "mpx_common.cuh"
#include "sm100_ptx.cuh"

#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

namespace mpx {

using namespace ptx;

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kBNMax = 256;
constexpr int kATileBytes = kBM * kBK * 2;       // 16 KB
constexpr int kBTileBytes = kBNMax * kBK * 2;    // 32 KB
// epilogue warps: kEpiWarps / 4 per TMEM lane quarter (16: no gain for the plain /
// operand-in epilogues).  -DMPX_GELU_EPI_WARPS=16 gives the GELU-aux-out variant 16
// epilogue warps (one 64-column group per warp per tile, its two 4 KB buffers free
// a whole tile ahead) with a 3-deep ring in the same 230 KB of smem: measured
// slower (331 vs 300 us steady state at the fc1 shape), so 8 is the default
#ifndef MPX_AUXOUT_GW
#define MPX_AUXOUT_GW 32
#endif
#ifndef MPX_GELU_EPI_WARPS
#define MPX_GELU_EPI_WARPS 8
#endif
template <int XO> struct EpiCfg {
  static constexpr int kWarps = XO == 3 ? MPX_GELU_EPI_WARPS : 8;  // XOP_AUX_OUT
  static constexpr int kPerQ = kWarps / 4;
  static constexpr int kThreads = 64 + 32 * kWarps;  // TMA warp, MMA warp, epilogue warps
};
constexpr int kEpiWarps = 8;  // the default variants (host-side BN checks)
constexpr int kEpiPerQ = kEpiWarps / 4;
// Shared memory = A/B ring + epilogue staging, 230 KB either way.  Variants
// that stage an operand (residual / GELU aux in) keep two 4 KB buffers per
// epilogue warp (64 KB: operand prefetch + in-place output) and a 5-deep ring;
// the others one buffer per warp (32 KB) and a 6-deep ring (measured: plain
// epilogue 209 -> 205 us, operand-in variants 250 -> 262 us with one buffer).
template <int XO> struct GemmSmem {
  static constexpr int kStageKB = (XO == 1 || XO == 2 || XO == 5) ? 64 : XO == 3 ? 8 * EpiCfg<XO>::kWarps : 32;
  static constexpr int kEpiStage = kStageKB * 1024;
  static constexpr int kStages2 = (192 - kStageKB) / 32 + 1 - (XO == 5 ? 1 : 0);  // CTA-pair ring depth (32 KB stages)
  static constexpr int kStages1 = (kStages2 * 2) / 3 > 1 ? (kStages2 * 2) / 3 : 2;  // single-CTA (48 KB stages)
  static constexpr int kBufPerWarp = kEpiStage / EpiCfg<XO>::kWarps / 4096;
};
constexpr int kGroupM = 16;  // tile raster: groups of kGroupM m-blocks, m fastest
constexpr size_t kGemmSmem = 1024 + 5 * (kATileBytes + kBTileBytes / 2) + 65536 + 384;
static_assert(1024 + 6 * (kATileBytes + kBTileBytes / 2) + 32768 + 384 == kGemmSmem, "variant smem budgets differ");
static_assert(4 * (kATileBytes + kBTileBytes) <= 6 * (kATileBytes + kBTileBytes / 2), "CG=1 ring exceeds the CG=2 one");

// ACT_SOFTMAX: the tile holds whole rows (one N block, N <= 256): C = softmax
//   over the row of round_half(alpha * acc) (f32 island, tensors.py:431-446)
// ACT_SOFTMAX_BWD: aux = P (same layout as C); C = P * (acc - sum_row(P * acc))
//   with acc = dP (autodiff.py:233-240)
// ACT_GELU_D: GELU forward whose aux receives round_half(gelu'(pre)) — the
//   derivative _bw_gelu rounds onto the cotangent's grid (autodiff.py:173-185)
//   — instead of the pre-activation; ACT_MUL_AUX: C = acc * aux (its backward:
//   the saved derivative, so the dgrad epilogue needs no tanh)
enum { ACT_NONE = 0, ACT_GELU = 1, ACT_GELU_BWD = 2, ACT_SOFTMAX = 3, ACT_SOFTMAX_BWD = 4, ACT_GELU_D = 5,
       ACT_MUL_AUX = 6 };

// n / d for 0 <= n < 2^31 by a multiply-high, an add and a shift (d >= 1
// fixed per launch, m and s from make_fastdiv on the host): the per-tile raster
// arithmetic every warp repeats for every tile, without integer divisions
struct FastDiv {
  uint32_t d, m, s;
};
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) { return (__umulhi(n, f.m) + n) >> f.s; }

struct GemmParams {
  int M, N, K, BN;
  int N_store;     // N rounded up to 8: stores cover whole 8-column groups
  int a_mn, b_mn;  // operand majorness: 0 = K-major, 1 = MN-major
  int nb1, nbatch, split;
  int a_bc1, a_bc2, b_bc1, b_bc2;  // operand shared across that batch dim (coordinate 0)
  int m_blocks, n_blocks, k_blocks, kb_per_split;
  long long total_tiles;
  FastDiv fd_mn, fd_split, fd_grp, fd_gmt, fd_nb1;  // m_blocks*n_blocks, split, kGroupM*n_blocks, tail group, nb1
  uint32_t idesc;
  uint32_t idesc2;  // WN variants: the second MMA of each K step (N = 128 at 384 wide, 256 at 512)
  int ab_fmt;  // 0 = f16, 1 = bf16 (also the dtype of bias/residual/aux)
  // epilogue
  void* C;
  long long ldc, c_sb1, c_sb2;
  int c_dtype;  // MPX_F32 / MPX_F16 / MPX_BF16
  const void* bias;
  const void* res;
  long long ldr, r_sb1, r_sb2;
  void* aux;  // ACT_GELU: pre-activation out; ACT_GELU_BWD: pre-activation in
  long long ld_aux;
  float alpha;
  int act;
  float* ws;  // split-K partials [split][M][N] (f32)
  float* csum;  // fused column sum: per-32-row partials [ceil(M/32)][N] (f32), or null
  int tma_store;  // 16-bit C written through swizzled smem staging + TMA bulk stores
  int xop;        // epilogue operand through TMA (tmX): 0 none, 1 residual in, 2 aux in (GELU'), 3 aux out (GELU)
  // XOP_RES_LN: LayerNorm of the stored rows (gain / bias in the A/B format, f32 row stats)
  const void* ln_g;
  const void* ln_b;
  float* ln_mean;
  float* ln_rstd;
  float ln_eps;
};
// kernel variants by epilogue: XOP_NONE = generic (every act / operand at run
// time, operands read from global); the others are lean staged-path variants
// (bias optional): residual in, GELU' with aux in, GELU with aux out, plain
enum { XOP_NONE = 0, XOP_RES_IN = 1, XOP_AUX_IN = 2, XOP_AUX_OUT = 3, XOP_PLAIN = 4, XOP_RES_LN = 5 };
// XOP_RES_LN — bias + residual epilogue followed by the LayerNorm of every
// stored row (LN folded into the GEMM that produces the residual
// stream, tensors.py:459-491).  N = 768 = 3 x 256: a cluster of 3 CTA pairs
// (6 CTAs) owns one 256-row block, pair p computes columns 256p..256p+255;
// each CTA's per-row partial sums (of the ROUNDED stored values) are
// exchanged over distributed shared memory, so every CTA normalises its own
// columns from smem and TMA-stores LN(x) next to x: the LayerNorm never
// re-reads x from HBM and needs no launch of its own.

__device__ __forceinline__ float half_to_f32(uint16_t h, int fmt) {
  return fmt ? to_f32<MPX_BF16>(h) : to_f32<MPX_F16>(h);
}
__device__ __forceinline__ uint16_t f32_to_half(float x, int fmt) {
  return fmt ? from_f32<MPX_BF16>(x) : from_f32<MPX_F16>(x);
}

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// tanh-approximation GELU and its derivative (tensors.py:196-200, autodiff.py:173-185),
// the same operations as the packed versions below (so every epilogue path of the
// GEMM gives the same bits): u = x c0 (1 + c1 x^2), y = x/2 + x/2 t,
// gelu' = (1 + t)/2 + (y - y t) c0 (1 + 3 c1 x^2)
__device__ __forceinline__ float gelu_f(float x) {
  const float c0 = 0.7978845608028654f, c1 = 0.044715f;
  const float x2 = __fmul_rn(x, x);
  const float t = tanh_fast(__fmul_rn(x, __fmaf_rn(x2, c0 * c1, c0)));
  const float hx = __fmul_rn(x, 0.5f);
  return __fmaf_rn(hx, t, hx);
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  const float c0 = 0.7978845608028654f, c1 = 0.044715f;
  const float x2 = __fmul_rn(x, x);
  const float t = tanh_fast(__fmul_rn(x, __fmaf_rn(x2, c0 * c1, c0)));
  const float hx = __fmul_rn(x, 0.5f);
  const float y = __fmaf_rn(hx, t, hx);
  const float a = __fmaf_rn(t, 0.5f, 0.5f);
  const float ymt = __fmaf_rn(-y, t, y);
  return __fmaf_rn(ymt, __fmaf_rn(x2, 3.f * c0 * c1, c0), a);
}

// packed-f32x2 (FFMA2 / FMUL2) versions for the lean epilogues: two columns per
// instruction on the FMA pipe; the same tanh form, c0 x (1 + c1 x^2) inside
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 gelu2(float2 x) {
  const float c0 = 0.7978845608028654f, c1 = 0.044715f;
  const float2 x2 = __fmul2_rn(x, x);
  const float2 u = __fmul2_rn(x, __ffma2_rn(x2, f2(c0 * c1), f2(c0)));  // x c0 (1 + c1 x^2)
  const float2 th = make_float2(tanh_fast(u.x), tanh_fast(u.y));
  const float2 hx = __fmul2_rn(x, f2(0.5f));
  return __ffma2_rn(hx, th, hx);
}
// GELU and its derivative from one tanh (ACT_GELU_D): with y = x/2 (1 + t),
// d = (1 + t)/2 + x/2 (1 - t^2) k = (1 + t)/2 + (y - y t) k, k = c0 (1 + 3 c1 x^2)
__device__ __forceinline__ void gelu_and_grad2(float2 x, float2& y, float2& d) {
  const float c0 = 0.7978845608028654f, c1 = 0.044715f;
  const float2 x2 = __fmul2_rn(x, x);
  const float2 u = __fmul2_rn(x, __ffma2_rn(x2, f2(c0 * c1), f2(c0)));
  const float2 t = make_float2(tanh_fast(u.x), tanh_fast(u.y));
  const float2 hx = __fmul2_rn(x, f2(0.5f));
  y = __ffma2_rn(hx, t, hx);
  const float2 a = __ffma2_rn(t, f2(0.5f), f2(0.5f));                      // 0.5 (1 + t)
  const float2 ymt = __ffma2_rn(make_float2(-y.x, -y.y), t, y);            // y (1 - t) = x/2 (1 - t^2)
  const float2 k = __ffma2_rn(x2, f2(3.f * c0 * c1), f2(c0));              // c0 (1 + 3 c1 x^2)
  d = __ffma2_rn(ymt, k, a);
}
__device__ __forceinline__ float2 gelu_grad2(float2 x) {
  float2 y, d;
  gelu_and_grad2(x, y, d);
  return d;
}

struct TileCoord {
  int z, s, m_blk, n_blk;
};
// tile t -> (batch z, split s, m block, n block): groups of kGroupM m-blocks,
// m fastest inside a group (t < 2^31, checked on the host)
__device__ __forceinline__ TileCoord tile_coord(const GemmParams& P, long long t64) {
  const uint32_t t = (uint32_t)t64;
  const uint32_t zs = fdiv(t, P.fd_mn);
  const uint32_t r = t - zs * P.fd_mn.d;
  TileCoord c;
  const uint32_t z = fdiv(zs, P.fd_split);
  c.z = (int)z;
  c.s = (int)(zs - z * P.fd_split.d);
  const uint32_t group = fdiv(r, P.fd_grp);
  const uint32_t first_m = group * kGroupM;
  const uint32_t in = r - group * P.fd_grp.d;
  uint32_t q, gm;
  if (first_m + kGroupM <= (uint32_t)P.m_blocks) {  // a full group: constant divisor
    q = in / kGroupM;
    gm = kGroupM;
  } else {  // the last, partial group
    q = fdiv(in, P.fd_gmt);
    gm = P.fd_gmt.d;
  }
  c.m_blk = (int)(first_m + (in - q * gm));
  c.n_blk = (int)q;
  return c;
}

// CG = 1: one CTA per tile (M = 128).  CG = 2: a CTA pair (cluster of 2)
// per 256-row tile: each CTA stages its 128 A rows and half of the BN B
// columns, the leader issues tcgen05.mma.cta_group::2 (M = 256), so each SM
// streams 2/3 of the bytes per FLOP of the 1-CTA tile.
// FMT: the A/B (and 16-bit C, bias, residual, aux) format, 0 f16 / 1 bf16,
// compiled in so the epilogue carries one conversion path.
// WN = 1 / 2: the wide weight-gradient tiles — CTA pair, 256 x 384 / 256 x 512,
// MN-major B, one accumulator (384 / 512 TMEM columns; the split-K units are one
// tile each, so there is no next tile to overlap): per K step an N = 256 MMA and
// an N = 128 / 256 one share the A tile; each CTA stages the B column chunks
// {2r, 2r+1, 4+r} / {2r, 2r+1, 4+2r, 5+2r} (64 columns each) so every MMA's
// per-CTA halves land in column order.  Bytes per MAC from L2 are 5/6 / 3/4 of
// the 256 x 256 tile's, the feed the long wgrad mainloops are bound by.
template <int CG, int XO, int FMT, int WN = 0>
__global__ void __launch_bounds__(EpiCfg<XO>::kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ CUtensorMap tmL, const __grid_constant__ GemmParams P) {
  static_assert(!WN || (CG == 2 && XO == XOP_PLAIN), "the wide tile is a CTA-pair plain-epilogue variant");
  static_assert(XO != XOP_RES_LN || CG == 2, "the LayerNorm epilogue is a CTA-pair variant");
  constexpr bool kLN = XO == XOP_RES_LN;
  constexpr int kClusterCTAs = kLN ? 6 : CG;
  using SM = GemmSmem<XO>;
  constexpr int kEpiWarps = EpiCfg<XO>::kWarps;  // (shadows the file-scope default)
  constexpr int kEpiPerQ = EpiCfg<XO>::kPerQ;
  constexpr int kBNw = WN == 2 ? 512 : WN == 1 ? 384 : kBNMax;  // tile width
  constexpr int BT = kBNw * kBK * 2 / CG;  // B bytes per stage per CTA
  // smem ring depth: 48 / 32 KB stages; wide: 40 KB stages in the same 224 KB budget
  constexpr int S = WN ? (224 - SM::kStageKB) * 1024 / (kATileBytes + BT) : CG == 1 ? SM::kStages1 : SM::kStages2;
  constexpr int kBufPerWarp = SM::kBufPerWarp;
  constexpr int kEpiStage = SM::kEpiStage;
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned by indexing the __shared__ array (not via an integer cast), so
  // derived pointers stay in the shared window: STS/LDS, 32-bit addressing
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * kATileBytes;
  uint8_t* stage_epi = sB + S * BT;  // kEpiWarps x kBufPerWarp x 4 KB staging
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_epi + kEpiStage);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* ebar = tempty + 2;  // per epilogue warp: its operand tile has landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ebar + kEpiWarps);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t crank = CG == 2 ? cluster_ctarank() : 0u;
  const uint32_t rank = crank & 1u;     // rank within the CTA pair
  const uint32_t pr = crank >> 1;       // pair within the cluster (LN variant: the 256-column block)
  const uint16_t pair_mask = (uint16_t)(3u << (2 * pr));
  const uint32_t leader_rank = crank & ~1u;
  const bool leader = rank == 0;
  const long long t_first = blockIdx.x / kClusterCTAs, t_step = gridDim.x / kClusterCTAs;
  // the LayerNorm exchange scratch (RES_LN only; past the barriers, in the ring space the shorter ring frees):
  // lnq [4 quarters][2 warps][32 rows] float2, lnx [2 tile parities][3 pairs][128 rows] float2, lnbar[2]
  float2* lnq = reinterpret_cast<float2*>(stage_epi + kEpiStage + 512);
  float2* lnx = lnq + 4 * 2 * 32;
  uint64_t* lnbar = reinterpret_cast<uint64_t*>(lnx + 2 * 3 * 128);
  float2* lngb = reinterpret_cast<float2*>(lnbar + 2);  // [256 columns] (gain, bias) of this CTA's columns

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (P.tma_store) tma_prefetch(&tmC);
    if (XO != XOP_NONE) tma_prefetch(&tmX);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kEpiWarps * CG);
    }
    for (int i = 0; i < kEpiWarps; ++i) mbar_init(&ebar[i], 1);
    if (kLN)
      for (int i = 0; i < 2; ++i) mbar_init(&lnbar[i], 1);  // this CTA's expect_tx + 3 x 128 x 8 B of st.async
    fence_barrier_init();
  }
  if (warp == 1) {
    if (CG == 2)
      tmem_alloc_2sm<512>(tmem_slot);
    else
      tmem_alloc<512>(tmem_slot);
  }
  if (kLN) {  // this CTA's 256 columns of the LayerNorm gain / bias, as f32, once (global reads before the
              // PDL wait are fine: the parameters are not produced by the predecessor in the step graph)
    for (int c = threadIdx.x; c < kBNMax; c += blockDim.x) {
      const int col = (int)(crank >> 1) * kBNMax + c;
      lngb[c] = col < P.N ? make_float2(half_to_f32(static_cast<const uint16_t*>(P.ln_g)[col], FMT),
                                        half_to_f32(static_cast<const uint16_t*>(P.ln_b)[col], FMT))
                          : make_float2(0.f, 0.f);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync();  // the peer's barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // prologue done (barriers, TMEM, descriptor prefetch): wait for the
  // predecessor's outputs before the first global access
  ::mpx::pdl_grid_sync();

  const uint32_t a_bytes = kATileBytes;
  const int bn_cta = P.BN / CG;  // B columns staged by this CTA
  const uint32_t b_bytes = (uint32_t)bn_cta * kBK * 2;

  if (warp == 0) {
    {
      // ------------------------------------------------ TMA producer (warp-wide loop,
      // one elected lane issues: the loop's values stay warp-uniform)
      int stage = 0;
      uint32_t phase = 0;
      for (long long t = t_first; t < P.total_tiles; t += t_step) {
        const TileCoord tc = kLN ? TileCoord{0, 0, (int)t, (int)pr} : tile_coord(P, t);
        const int b2 = (int)fdiv((uint32_t)tc.z, P.fd_nb1), b1 = tc.z - b2 * P.nb1;
        const int m0 = tc.m_blk * (kBM * CG) + (int)rank * kBM;
        const int n0 = tc.n_blk * P.BN + (WN ? 0 : (int)rank * bn_cta);
        const int kb0 = tc.s * P.kb_per_split;
        const int kb1 = min(P.k_blocks, kb0 + P.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) {
          if (leader) mbar_arrive_expect_tx(&full[stage], CG * (a_bytes + b_bytes));
          uint8_t* a = sA + stage * kATileBytes;
          uint8_t* b = sB + stage * BT;
          const int k0 = kb * kBK;
          const int ab1 = P.a_bc1 ? 0 : b1, ab2 = P.a_bc2 ? 0 : b2;
          const int bb1 = P.b_bc1 ? 0 : b1, bb2 = P.b_bc2 ? 0 : b2;
          auto load = [&](void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3) {
            if (CG == 2)
              tma_load_4d_2sm(dst, m, &full[stage], c0, c1, c2, c3);
            else
              tma_load_4d(dst, m, &full[stage], c0, c1, c2, c3);
          };
          if (!P.a_mn) {
            load(a, &tmA, k0, m0, ab1, ab2);
          } else {
            load(a, &tmA, m0, k0, ab1, ab2);
            load(a + 8192, &tmA, m0 + 64, k0, ab1, ab2);
          }
          if (WN) {  // chunks 2r, 2r + 1 (the first N = 256 MMA's half), then 4 + r (384: the N = 128
                     // MMA's half) or 4 + 2r, 5 + 2r (512: the second N = 256 MMA's half)
#pragma unroll
            for (int c = 0; c < (WN == 2 ? 4 : 3); ++c) {
              const int chunk = c < 2 ? 2 * (int)rank + c : (WN == 2 ? 4 + 2 * (int)rank + (c - 2) : 4 + (int)rank);
              load(b + c * 8192, &tmB, n0 + 64 * chunk, k0, bb1, bb2);
            }
          } else if (!P.b_mn) {
            load(b, &tmB, k0, n0, bb1, bb2);
          } else {
            for (int c = 0; c < bn_cta / 64; ++c) load(b + c * 8192, &tmB, n0 + 64 * c, k0, bb1, bb2);
          }
          }
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ------------------------------------------------ MMA issuer (warp-wide loop, one elected lane issues)
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      // SW128 descriptors = constant fields + (smem address >> 4) in the low 14 bits: the
      // per-stage bases and per-k16 steps are 32-bit adds on the low word (no re-packing)
      const uint64_t a_desc0 = sw128_desc(smem_u32(sA), P.a_mn ? 8192 : 16, 1024);
      const uint64_t b_desc0 = sw128_desc(smem_u32(sB), P.b_mn ? 8192 : 16, 1024);
      const uint64_t b2_desc0 = sw128_desc(smem_u32(sB) + 2 * 8192, 8192, 1024);  // WN: the second MMA's B (MN-major)
      const uint32_t a_hi = (uint32_t)(a_desc0 >> 32), b_hi = (uint32_t)(b_desc0 >> 32);
      const uint32_t b2_hi = (uint32_t)(b2_desc0 >> 32);
      const uint32_t a_kstep = P.a_mn ? 2048 >> 4 : 32 >> 4, b_kstep = P.b_mn ? 2048 >> 4 : 32 >> 4;
      for (long long t = t_first; t < P.total_tiles; t += t_step) {
        const TileCoord tc = kLN ? TileCoord{0, 0, (int)t, (int)pr} : tile_coord(P, t);
        const int kb0 = tc.s * P.kb_per_split;
        const int kb1 = min(P.k_blocks, kb0 + P.kb_per_split);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + (WN ? 0u : (uint32_t)acc * 256);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t as = (uint32_t)a_desc0 + (uint32_t)(stage * kATileBytes >> 4);
          const uint32_t bs = (uint32_t)b_desc0 + (uint32_t)(stage * BT >> 4);
          const uint32_t b2s = (uint32_t)b2_desc0 + (uint32_t)(stage * BT >> 4);
          if (elect_one()) {
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint32_t acc_in = (kb > kb0 || k > 0) ? 1u : 0u;
            const uint32_t ad = as + k * a_kstep, bd = bs + k * b_kstep;
            if (WN) {
              umma_f16_2sm_w(d, ad, a_hi, bd, b_hi, P.idesc, acc_in);
              umma_f16_2sm_w(d + 256, ad, a_hi, b2s + k * (2048 >> 4), b2_hi, P.idesc2, acc_in);
            } else if (CG == 2) {
              umma_f16_2sm_w(d, ad, a_hi, bd, b_hi, P.idesc, acc_in);
            } else {
              umma_f16_w(d, ad, a_hi, bd, b_hi, P.idesc, acc_in);
            }
          }
          // smem slot free (in both CTAs) once these MMAs have read it
          if (CG == 2)
            umma_commit_2sm_mc(&empty[stage], pair_mask);
          else
            umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) {
          if (CG == 2)
            umma_commit_2sm_mc(&tfull[acc], pair_mask);  // accumulator ready for both epilogues
          else
            umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (!WN) acc ^= 1;  // (wide: one accumulator, its phase flips every tile)
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // -------------------------------------------------- epilogue warps
    // kEpiPerQ warps per TMEM lane quarter (warp % 4); warp h of a quarter
    // owns column groups h, h + kEpiPerQ, ... (TMA-store path) or 16-column
    // chunks h, h + kEpiPerQ, ... (direct path)
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int h = (warp - 2) >> 2;
    // (single-thread TMA / bulk-group work below runs on the elect.sync lane — lane 0
    // of the full warp every time, so the per-thread bulk groups stay consistent — which
    // keeps the TMA operands in uniform registers)
    // kBufPerWarp 4 KB staging buffers per warp (32 rows x 128 B, swizzled),
    // used in turn by successive column groups
    uint8_t* obuf = stage_epi + (warp - 2) * (kBufPerWarp * 4096);
    uint8_t* stg = obuf;
    uint32_t gcount = 0;  // staged column groups so far (selects the ping-pong buffer)
    uint32_t eph = 0;  // phase of this warp's operand barrier
    uint32_t ln_tiles = 0;  // RES_LN: tiles exchanged so far (slot / phase of lnbar)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (long long t = t_first; t < P.total_tiles; t += t_step) {
      const TileCoord tc = kLN ? TileCoord{0, 0, (int)t, (int)pr} : tile_coord(P, t);
      const int b2 = (int)fdiv((uint32_t)tc.z, P.fd_nb1), b1 = tc.z - b2 * P.nb1;
      const int row0 = tc.m_blk * (kBM * CG) + (int)rank * kBM + q * 32;
      const int row = row0 + lane;
      const int n0 = tc.n_blk * P.BN;
      const bool row_ok = row < P.M;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (WN ? 0u : (uint32_t)acc * 256) + ((uint32_t)(q * 32) << 16);

      // bias / activation / residual on 16 consecutive columns of this row
      auto load8 = [&](const void* base, long long idx, float* o) {
        const uint4 w = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(base) + idx);
        const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          o[2 * e] = half_to_f32((uint16_t)(u[e] & 0xFFFFu), FMT);
          o[2 * e + 1] = half_to_f32((uint16_t)(u[e] >> 16), FMT);
        }
      };
      // ---- softmax modes: row statistics over this warp's column groups,
      // combined with the partner warp (same TMEM lane quarter) through smem
      float row_m = 0.f, row_inv = 1.f, row_t = 0.f;
      const bool smx = XO == XOP_NONE && (P.act == ACT_SOFTMAX || P.act == ACT_SOFTMAX_BWD);
      auto round_half = [&](float x) { return half_to_f32(f32_to_half(x, FMT), FMT); };
      if (smx) {
        float m = -INFINITY, l = 0.f, tacc = 0.f;
        for (int g = h; g * 64 < P.BN; g += kEpiPerQ) {
          for (int cc = 0; cc < 4 && g * 64 + cc * 16 < P.BN; ++cc) {
            uint32_t r[16];
            tmem_ld16(taddr + g * 64 + cc * 16, r);
            tmem_ld_wait();
            const int col = n0 + g * 64 + cc * 16;
            if (P.act == ACT_SOFTMAX) {
              float sv[16], cm = -INFINITY;
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                sv[i] = col + i < P.N ? round_half(__uint_as_float(r[i]) * P.alpha) : -INFINITY;
                cm = fmaxf(cm, sv[i]);
              }
              const float nm = fmaxf(m, cm);
              float add = 0.f;
#pragma unroll
              for (int i = 0; i < 16; ++i) add += sv[i] == -INFINITY ? 0.f : __expf(sv[i] - nm);
              l = (m == -INFINITY ? 0.f : l * __expf(m - nm)) + add;
              m = nm;
            } else if (row_ok && col < P.N) {
              float pv[16];
              const long long ai = b1 * P.c_sb1 + b2 * P.c_sb2 + (long long)row * P.ld_aux + col;
              const uint4 w0 = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(P.aux) + ai);
              const uint4 w1 = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(P.aux) + ai + 8);
              const uint32_t u[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                pv[2 * e] = half_to_f32((uint16_t)(u[e] & 0xFFFFu), FMT);
                pv[2 * e + 1] = half_to_f32((uint16_t)(u[e] >> 16), FMT);
              }
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (col + i < P.N) tacc += pv[i] * __uint_as_float(r[i]) * P.alpha;
            }
          }
        }
        // exchange with the partner warp through the (idle) staging buffers
        if (elect_one()) bulk_wait_read0();
        __syncwarp();
        float* mine = reinterpret_cast<float*>(stg);
        mine[lane] = m;
        mine[32 + lane] = l;
        mine[64 + lane] = tacc;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(32 * kEpiPerQ) : "memory");
        float om[kEpiPerQ], ol[kEpiPerQ], M = -INFINITY, L = 0.f, T = 0.f;
#pragma unroll
        for (int j = 0; j < kEpiPerQ; ++j) {  // the warps of this lane quarter: e = (e & 3) + 4 j
          const float* o = reinterpret_cast<const float*>(stage_epi + (((warp - 2) & 3) + 4 * j) * (kBufPerWarp * 4096));
          om[j] = o[lane];
          ol[j] = o[32 + lane];
          T += o[64 + lane];
          M = fmaxf(M, om[j]);
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(32 * kEpiPerQ) : "memory");
#pragma unroll
        for (int j = 0; j < kEpiPerQ; ++j) L += om[j] == -INFINITY ? 0.f : ol[j] * __expf(om[j] - M);
        row_m = M;
        row_inv = 1.f / L;
        row_t = T;
      }

      // xin: the 16 staged operand values of this chunk (TMA operand path) or unused
      auto epi = [&](float* v, int col, int ncols, const float* xin) {
        if (XO != XOP_NONE) {  // lean variants: bias, then the staged operand
          if (P.bias) {
            float bb[16];
            if (col + 16 <= P.N) {
              load8(P.bias, col, bb);
              load8(P.bias, col + 8, bb + 8);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                bb[i] = col + i < P.N ? half_to_f32(static_cast<const uint16_t*>(P.bias)[col + i], FMT) : 0.f;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float2 r2 = __fadd2_rn(make_float2(v[2 * i], v[2 * i + 1]), make_float2(bb[2 * i], bb[2 * i + 1]));
              v[2 * i] = r2.x;
              v[2 * i + 1] = r2.y;
            }
          }
          if (XO == XOP_RES_IN || XO == XOP_RES_LN) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float2 r2 =
                  __fadd2_rn(make_float2(v[2 * i], v[2 * i + 1]), make_float2(xin[2 * i], xin[2 * i + 1]));
              v[2 * i] = r2.x;
              v[2 * i + 1] = r2.y;
            }
          } else if (XO == XOP_AUX_IN) {
            if (P.act == ACT_MUL_AUX) {  // the saved GELU derivative
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float2 r2 = __fmul2_rn(make_float2(v[2 * i], v[2 * i + 1]), make_float2(xin[2 * i], xin[2 * i + 1]));
                v[2 * i] = r2.x;
                v[2 * i + 1] = r2.y;
              }
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float2 r2 = __fmul2_rn(make_float2(v[2 * i], v[2 * i + 1]),
                                             gelu_grad2(make_float2(xin[2 * i], xin[2 * i + 1])));
                v[2 * i] = r2.x;
                v[2 * i + 1] = r2.y;
              }
            }
          }
          return;  // XOP_AUX_OUT: the caller rounds (aux) and applies the GELU
        }
        if (P.act == ACT_SOFTMAX) {  // v = alpha*acc: P = exp(round(v) - M) / L, 0 past N
#pragma unroll
          for (int i = 0; i < 16; ++i)
            v[i] = col + i < P.N ? __expf(round_half(v[i]) - row_m) * row_inv : 0.f;
          return;
        }
        if (P.act == ACT_SOFTMAX_BWD) {  // v = alpha*dP: dS = P * (v - t)
          float pv[16];
          load8(P.aux, b1 * P.c_sb1 + b2 * P.c_sb2 + (long long)row * P.ld_aux + col, pv);
          load8(P.aux, b1 * P.c_sb1 + b2 * P.c_sb2 + (long long)row * P.ld_aux + col + 8, pv + 8);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = col + i < P.N ? pv[i] * (v[i] - row_t) : 0.f;
          return;
        }
        if (P.bias) {
          float bb[16];
          if (col + 16 <= P.N) {
            load8(P.bias, col, bb);
            load8(P.bias, col + 8, bb + 8);
          } else {  // ragged tail: the bias has exactly N entries
#pragma unroll
            for (int i = 0; i < 16; ++i)
              bb[i] = col + i < P.N ? half_to_f32(static_cast<const uint16_t*>(P.bias)[col + i], FMT) : 0.f;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += bb[i];
        }
        if ((P.act == ACT_GELU || P.act == ACT_GELU_D) && XO == XOP_AUX_OUT) {
          // bias only here; the staged aux store and the GELU happen in the caller
        } else if (P.act == ACT_GELU || P.act == ACT_GELU_D) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = half_to_f32(f32_to_half(v[i], FMT), FMT);  // the rounded pre-activation
          if (P.aux) {
            uint16_t* ax = static_cast<uint16_t*>(P.aux) + b1 * P.c_sb1 + b2 * P.c_sb2 + (long long)row * P.ld_aux + col;
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              pk[i] = P.act == ACT_GELU_D ? pack2_fmt(gelu_grad_f(v[2 * i]), gelu_grad_f(v[2 * i + 1]), FMT)
                                          : pack2_fmt(v[2 * i], v[2 * i + 1], FMT);
            *reinterpret_cast<uint4*>(ax) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            if (ncols == 16) *reinterpret_cast<uint4*>(ax + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = gelu_f(v[i]);
        } else if (P.act == ACT_MUL_AUX) {
          float z[16];
          if (XO == XOP_AUX_IN) {
#pragma unroll
            for (int i = 0; i < 16; ++i) z[i] = xin[i];
          } else {
            const long long ai = b1 * P.c_sb1 + b2 * P.c_sb2 + (long long)row * P.ld_aux + col;
            load8(P.aux, ai, z);
            if (ncols == 16) load8(P.aux, ai + 8, z + 8);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] *= z[i];
        } else if (P.act == ACT_GELU_BWD) {
          float z[16];
          if (XO == XOP_AUX_IN) {
#pragma unroll
            for (int i = 0; i < 16; ++i) z[i] = xin[i];
          } else {
            const long long ai = b1 * P.c_sb1 + b2 * P.c_sb2 + (long long)row * P.ld_aux + col;
            load8(P.aux, ai, z);
            if (ncols == 16) load8(P.aux, ai + 8, z + 8);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] *= gelu_grad_f(z[i]);
        }
        if (P.res && (XO == XOP_RES_IN || XO == XOP_RES_LN)) {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += xin[i];
        } else if (P.res) {
          float rr[16];
          const long long ri = b1 * P.r_sb1 + b2 * P.r_sb2 + (long long)row * P.ldr + col;
          load8(P.res, ri, rr);
          if (ncols == 16) load8(P.res, ri + 8, rr + 8);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += rr[i];
        }
      };

      if (XO != XOP_NONE || P.tma_store) {  // (the lean variants are only launched staged)
        // Column groups of GW: 64 half columns (128 B rows, SW128), or 32 f32
        // columns, or — GELU with the aux written too — 32 half columns whose
        // aux and C tiles (64 B rows, SW64) share one buffer.  Each warp
        // ping-pongs its two 4 KB buffers over a running group count, so the
        // TMA store of group gc overlaps the TMEM loads and math of gc + 1; a
        // staged operand (residual / GELU aux in) lands in the group's buffer
        // one group ahead and the output overwrites it in place, row by row.
        constexpr bool kXin = XO == XOP_RES_IN || XO == XOP_AUX_IN || XO == XOP_RES_LN;
        constexpr bool kAuxOut = XO == XOP_AUX_OUT;
        constexpr int kAuxGW = MPX_AUXOUT_GW;
        const bool f32out = P.split > 1 || P.c_dtype == MPX_F32;
        // GELU-aux-out with kAuxGW == 32: 32-column groups whose aux + C tiles (2 KB
        // each, SW64) fill ONE 4 KB buffer, so the warp's two buffers ping-pong and a
        // group waits only for the stores of the group before last (64: one 64-column
        // group fills both buffers and waits for all earlier stores)
        const int GW = (f32out || (kAuxOut && kAuxGW == 32)) ? 32 : 64;
        constexpr int cf = FMT;  // 16-bit C has the A/B format (checked on the host)
        float2 ln_s1 = make_float2(0.f, 0.f), ln_s2 = make_float2(0.f, 0.f);  // RES_LN: this row's sums (pairs)
        const int n_groups = (P.BN + GW - 1) / GW;
        const int my_groups = n_groups > h ? (n_groups - h + kEpiPerQ - 1) / kEpiPerQ : 0;
        auto buf = [&](uint32_t c) { return obuf + (c % kBufPerWarp) * 4096; };
        auto x_load = [&](int g, uint32_t c) {  // operand tile of group g -> buffer of group count c
          const int xb1 = (XO == XOP_RES_IN || XO == XOP_RES_LN) && P.r_sb1 == 0 ? 0 : b1;
          const int xb2 = (XO == XOP_RES_IN || XO == XOP_RES_LN) && P.r_sb2 == 0 ? 0 : b2;
          bulk_wait_read<kBufPerWarp - 1>();  // the store that last used this buffer has read it
          mbar_arrive_expect_tx(&ebar[warp - 2], 4096);
          tma_load_4d(buf(c), &tmX, &ebar[warp - 2], n0 + g * GW, row0, xb1, xb2);
        };
        auto release_acc = [&]() {  // this warp is done with the accumulator: the MMA may reuse it
          tc_fence_before();
          if (CG == 2)
            mbar_arrive_remote(&tempty[acc], leader_rank);
          else
            mbar_arrive(&tempty[acc]);
        };
        // TMEM -> epilogue math -> the group's staging buffer (in place over a staged operand)
        auto stage_group = [&](int g, int nch, uint8_t* bb, bool last) {
          constexpr int kLd = kEpiWarps > 8 ? (XO == XOP_PLAIN || XO == XOP_AUX_OUT ? 2 : 1) : (XO == XOP_NONE ? 2 : 4);  // chunks per TMEM wait
#pragma unroll
          for (int pair = 0; pair < 4 / kLd; ++pair) {
            if (pair * kLd >= nch) continue;
            uint32_t r[kLd][16];
#pragma unroll
            for (int k = 0; k < kLd; ++k)
              if (pair * kLd + k < nch) tmem_ld16(taddr + g * GW + (pair * kLd + k) * 16, r[k]);
            tmem_ld_wait();
            if (last && (pair == 4 / kLd - 1 || nch <= (pair + 1) * kLd)) release_acc();
#pragma unroll
            for (int kk = 0; kk < kLd; ++kk) {
              const int k = pair * kLd + kk;
              if (k >= nch) continue;
              float v[16];
              if (P.alpha != 1.f) {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[kk][i]) * P.alpha;
              } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[kk][i]);
              }
              if (f32out) {  // raw (split-K partial) or f32 output: 4 x 16 B, SW128
                uint8_t* rowp = bb + lane * 128;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  *reinterpret_cast<float4*>(rowp + (((4 * k + u) ^ (lane & 7)) << 4)) =
                      make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
                continue;
              }
              const int col = n0 + g * GW + k * 16;
              if (kAuxOut) {  // aux (rounded pre-activation) in the warp's buffer 0, C = GELU(aux) in buffer 1; SW128
                if (row_ok && col < P.N_store) epi(v, col, min(16, P.N_store - col), v);
                uint32_t pa[8], pc[8];
                const bool dout = P.act == ACT_GELU_D;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  pa[i] = pack2_fmt(v[2 * i], v[2 * i + 1], FMT);
                  const float a = half_to_f32((uint16_t)(pa[i] & 0xFFFFu), FMT);
                  const float b = half_to_f32((uint16_t)(pa[i] >> 16), FMT);
                  if (dout) {  // aux = the rounded derivative, from the same tanh as the GELU
                    float2 y, d;
                    gelu_and_grad2(make_float2(a, b), y, d);
                    pc[i] = pack2_fmt(y.x, y.y, cf);
                    pa[i] = pack2_fmt(d.x, d.y, FMT);
                  } else {
                    const float2 y = gelu2(make_float2(a, b));  // GELU of the rounded pre-activation
                    pc[i] = pack2_fmt(y.x, y.y, cf);
                  }
                }
                if (kAuxGW == 32) {  // 64 B rows, SW64: 16-byte unit u of row r at u ^ ((r >> 1) & 3)
                  const int s64 = (lane >> 1) & 3;
                  uint8_t* ra = bb + lane * 64;
                  uint8_t* rc = ra + 2048;
                  *reinterpret_cast<uint4*>(ra + (((2 * k) ^ s64) << 4)) = make_uint4(pa[0], pa[1], pa[2], pa[3]);
                  *reinterpret_cast<uint4*>(ra + (((2 * k + 1) ^ s64) << 4)) = make_uint4(pa[4], pa[5], pa[6], pa[7]);
                  *reinterpret_cast<uint4*>(rc + (((2 * k) ^ s64) << 4)) = make_uint4(pc[0], pc[1], pc[2], pc[3]);
                  *reinterpret_cast<uint4*>(rc + (((2 * k + 1) ^ s64) << 4)) = make_uint4(pc[4], pc[5], pc[6], pc[7]);
                  continue;
                }
                const int s128 = lane & 7;
                uint8_t* ra = obuf + lane * 128;
                uint8_t* rc = ra + 4096;
                *reinterpret_cast<uint4*>(ra + (((2 * k) ^ s128) << 4)) = make_uint4(pa[0], pa[1], pa[2], pa[3]);
                *reinterpret_cast<uint4*>(ra + (((2 * k + 1) ^ s128) << 4)) = make_uint4(pa[4], pa[5], pa[6], pa[7]);
                *reinterpret_cast<uint4*>(rc + (((2 * k) ^ s128) << 4)) = make_uint4(pc[0], pc[1], pc[2], pc[3]);
                *reinterpret_cast<uint4*>(rc + (((2 * k + 1) ^ s128) << 4)) = make_uint4(pc[4], pc[5], pc[6], pc[7]);
                continue;
              }
              uint8_t* rowp = bb + lane * 128;
              const int sw = lane & 7;
              float xv[16];
              if (kXin) {  // own row of the staged operand
                const uint4 w0 = *reinterpret_cast<const uint4*>(rowp + (((2 * k) ^ sw) << 4));
                const uint4 w1 = *reinterpret_cast<const uint4*>(rowp + (((2 * k + 1) ^ sw) << 4));
                const uint32_t u[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  xv[2 * e] = half_to_f32((uint16_t)(u[e] & 0xFFFFu), FMT);
                  xv[2 * e + 1] = half_to_f32((uint16_t)(u[e] >> 16), FMT);
                }
              }
              if (row_ok && col < P.N_store) epi(v, col, min(16, P.N_store - col), xv);
              uint32_t pk[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) pk[i] = pack2_fmt(v[2 * i], v[2 * i + 1], cf);
              if (kLN) {  // row statistics of the ROUNDED stored values (the LayerNorm's input)
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const float2 ab = make_float2(half_to_f32((uint16_t)(pk[i] & 0xFFFFu), FMT),
                                                half_to_f32((uint16_t)(pk[i] >> 16), FMT));
                  ln_s1 = __fadd2_rn(ln_s1, ab);
                  ln_s2 = __ffma2_rn(ab, ab, ln_s2);
                }
              }
              *reinterpret_cast<uint4*>(rowp + (((2 * k) ^ sw) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
              *reinterpret_cast<uint4*>(rowp + (((2 * k + 1) ^ sw) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
            }
          }
        };
        // stage_group for the common case, everything known at compile time: a whole
        // 64-column group inside N, 16-bit C, alpha 1, a lean variant (bias / residual /
        // GELU' operand; half operands added by mixed-precision FHADD).  Rows past M run the same math (their A rows are TMA zero-fill,
        // staged operands too; the TMA store clips them and the column sum skips them)
        auto stage_full = [&](int g, uint8_t* bb, bool last) {  // (alpha == 1)
          uint8_t* rowp = bb + lane * 128;
          const int sw = lane & 7;
          const uint16_t* bias = static_cast<const uint16_t*>(P.bias);
#pragma unroll
          for (int half = 0; half < 2; ++half) {  // two chunks per TMEM wait (register budget)
            uint32_t r[2][16];
            tmem_ld16(taddr + g * GW + half * 32, r[0]);
            tmem_ld16(taddr + g * GW + half * 32 + 16, r[1]);
            tmem_ld_wait();
            if (last && half == 1) release_acc();
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const int k = 2 * half + kk;
              float2 v[8];
#pragma unroll
              for (int i = 0; i < 8; ++i)
                v[i] = make_float2(__uint_as_float(r[kk][2 * i]), __uint_as_float(r[kk][2 * i + 1]));
              if (bias != nullptr) {
                const uint4 b0 = *reinterpret_cast<const uint4*>(bias + n0 + g * GW + k * 16);
                const uint4 b1_ = *reinterpret_cast<const uint4*>(bias + n0 + g * GW + k * 16 + 8);
                const uint32_t bw[8] = {b0.x, b0.y, b0.z, b0.w, b1_.x, b1_.y, b1_.z, b1_.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = add_h2<FMT>(v[i], bw[i]);
              }
              uint4* p0 = reinterpret_cast<uint4*>(rowp + (((2 * k) ^ sw) << 4));
              uint4* p1 = reinterpret_cast<uint4*>(rowp + (((2 * k + 1) ^ sw) << 4));
              if (kXin) {  // own row of the staged operand
                const uint4 w0 = *p0, w1 = *p1;
                const uint32_t u[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
                if (XO == XOP_RES_IN || XO == XOP_RES_LN) {
#pragma unroll
                  for (int i = 0; i < 8; ++i) v[i] = add_h2<FMT>(v[i], u[i]);
                } else if (P.act == ACT_MUL_AUX) {  // XOP_AUX_IN: the saved GELU derivative
#pragma unroll
                  for (int i = 0; i < 8; ++i) v[i] = __fmul2_rn(v[i], unpack2_fmt<FMT>(u[i]));
                } else {  // XOP_AUX_IN: gelu' of the saved pre-activation
#pragma unroll
                  for (int i = 0; i < 8; ++i) v[i] = __fmul2_rn(v[i], gelu_grad2(unpack2_fmt<FMT>(u[i])));
                }
              }
              uint32_t pk[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) pk[i] = pack2_fmt(v[i].x, v[i].y, cf);
              if (kLN) {  // row statistics of the ROUNDED stored values (the LayerNorm's input)
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const float2 ab = unpack2_fmt<FMT>(pk[i]);
                  ln_s1 = __fadd2_rn(ln_s1, ab);
                  ln_s2 = __ffma2_rn(ab, ab, ln_s2);
                }
              }
              *p0 = make_uint4(pk[0], pk[1], pk[2], pk[3]);
              *p1 = make_uint4(pk[4], pk[5], pk[6], pk[7]);
            }
          }
        };
        // the same for the GELU-aux-out groups (32 columns, SW64, aux + C in one buffer)
        auto stage_full_aux = [&](int g, uint8_t* bb, bool last) {  // (alpha == 1, kAuxGW == 32)
          uint32_t r[2][16];
          tmem_ld16(taddr + g * GW, r[0]);
          tmem_ld16(taddr + g * GW + 16, r[1]);
          tmem_ld_wait();
          if (last) release_acc();
          const uint16_t* bias = static_cast<const uint16_t*>(P.bias);
          const bool dout = P.act == ACT_GELU_D;
          const int s64 = (lane >> 1) & 3;
          uint8_t* ra = bb + lane * 64;
          uint8_t* rc = ra + 2048;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            float2 v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = make_float2(__uint_as_float(r[k][2 * i]), __uint_as_float(r[k][2 * i + 1]));
            if (bias != nullptr) {
              const uint4 b0 = *reinterpret_cast<const uint4*>(bias + n0 + g * GW + k * 16);
              const uint4 b1_ = *reinterpret_cast<const uint4*>(bias + n0 + g * GW + k * 16 + 8);
              const uint32_t bw[8] = {b0.x, b0.y, b0.z, b0.w, b1_.x, b1_.y, b1_.z, b1_.w};
#pragma unroll
              for (int i = 0; i < 8; ++i) v[i] = add_h2<FMT>(v[i], bw[i]);
            }
            uint32_t pa[8], pc[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              pa[i] = pack2_fmt(v[i].x, v[i].y, FMT);  // the rounded pre-activation
              const float2 ab = unpack2_fmt<FMT>(pa[i]);
              if (dout) {  // aux = the rounded derivative, from the same tanh as the GELU
                float2 y, d;
                gelu_and_grad2(ab, y, d);
                pc[i] = pack2_fmt(y.x, y.y, cf);
                pa[i] = pack2_fmt(d.x, d.y, FMT);
              } else {
                const float2 y = gelu2(ab);
                pc[i] = pack2_fmt(y.x, y.y, cf);
              }
            }
            *reinterpret_cast<uint4*>(ra + (((2 * k) ^ s64) << 4)) = make_uint4(pa[0], pa[1], pa[2], pa[3]);
            *reinterpret_cast<uint4*>(ra + (((2 * k + 1) ^ s64) << 4)) = make_uint4(pa[4], pa[5], pa[6], pa[7]);
            *reinterpret_cast<uint4*>(rc + (((2 * k) ^ s64) << 4)) = make_uint4(pc[0], pc[1], pc[2], pc[3]);
            *reinterpret_cast<uint4*>(rc + (((2 * k + 1) ^ s64) << 4)) = make_uint4(pc[4], pc[5], pc[6], pc[7]);
          }
        };
        auto store_group = [&](int g, uint8_t* bb) {  // lane 0
          if (P.split > 1) {
            tma_store_4d(&tmC, bb, n0 + g * GW, row0, tc.s, 0);
          } else if (kAuxOut && kAuxGW == 32) {
            tma_store_4d(&tmX, bb, n0 + g * GW, row0, b1, b2);
            tma_store_4d(&tmC, bb + 2048, n0 + g * GW, row0, b1, b2);
          } else if (kAuxOut) {
            tma_store_4d(&tmX, obuf, n0 + g * GW, row0, b1, b2);
            tma_store_4d(&tmC, obuf + 4096, n0 + g * GW, row0, b1, b2);
          } else {
            tma_store_4d(&tmC, bb, n0 + g * GW, row0, b1, b2);
          }
        };
        // batched: both of this warp's groups staged at once (one buffer each),
        // one proxy fence and one bulk group per tile — the previous tile's
        // stores had a whole tile of MMA time to drain.  Otherwise (f32 / GELU-
        // aux-out groups, > 2 groups) ping-pong the buffers group by group.
        const bool batched = !kAuxOut && my_groups <= kBufPerWarp;  // GELU-aux-out: both buffers per group
        if (batched) {
          if (elect_one()) {
            bulk_wait_read0();
            if (kXin && my_groups > 0) {
              const int xb1 = (XO == XOP_RES_IN || XO == XOP_RES_LN) && P.r_sb1 == 0 ? 0 : b1;
              const int xb2 = (XO == XOP_RES_IN || XO == XOP_RES_LN) && P.r_sb2 == 0 ? 0 : b2;
              mbar_arrive_expect_tx(&ebar[warp - 2], 4096u * my_groups);
              for (int j = 0; j < my_groups; ++j)
                tma_load_4d(buf(j), &tmX, &ebar[warp - 2], n0 + (h + kEpiPerQ * j) * GW, row0, xb1, xb2);
            }
          }
          __syncwarp();
        } else if (kXin && my_groups > 0 && elect_one()) {
          x_load(h, gcount);
        }
        if (my_groups == 0) release_acc();
        for (int j = 0; j < my_groups; ++j, ++gcount) {
          const int g = h + kEpiPerQ * j;
          const int nch = min(GW / 16, (P.BN - g * GW) / 16);
          uint8_t* bb = batched ? buf(j) : buf(gcount);
          if (kXin) {
            if (!batched || j == 0) {
              mbar_wait(&ebar[warp - 2], eph);
              eph ^= 1u;
            }
          } else if (!batched) {
            if (elect_one()) {  // the store that last used this buffer (both, for 64-column GELU-aux-out) has read it
              if (kAuxOut && kAuxGW != 32)
                bulk_wait_read0();
              else
                bulk_wait_read<kBufPerWarp - 1>();
            }
            __syncwarp();
          }
          constexpr bool kFast = XO == XOP_PLAIN || XO == XOP_RES_IN || XO == XOP_AUX_IN || XO == XOP_RES_LN;
          if (kFast && GW == 64 && nch == 4 && n0 + g * GW + 64 <= P.N && P.alpha == 1.f)
            stage_full(g, bb, j == my_groups - 1);
          else if (kAuxOut && kAuxGW == 32 && GW == 32 && nch == 2 && n0 + g * GW + 32 <= P.N &&
                   P.alpha == 1.f)
            stage_full_aux(g, bb, j == my_groups - 1);
          else
            stage_group(g, nch, bb, j == my_groups - 1);
          if (batched && j + 1 < my_groups) continue;
          fence_async_smem();
          __syncwarp();
          if (elect_one()) {
            if (batched) {
              for (int jj = 0; jj < my_groups; ++jj) store_group(h + kEpiPerQ * jj, buf(jj));
            } else {
              store_group(g, bb);
            }
            bulk_commit();
            if (!batched && kXin && j + 1 < my_groups) x_load(g + kEpiPerQ, gcount + 1);  // next group's operand
          }
        }
        if (kLN && P.ln_eps >= 0.f) {  // (experiment: ln_eps < 0 = the cluster schedule without the LN work)
          // ---- LayerNorm of the stored rows.  (1) combine this quarter's warps
          lnq[(q * kEpiPerQ + h) * 32 + lane] = make_float2(ln_s1.x + ln_s1.y, ln_s2.x + ln_s2.y);
          asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(32 * kEpiPerQ) : "memory");
          float2 part = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < kEpiPerQ; ++j) {
            const float2 o = lnq[(q * kEpiPerQ + j) * 32 + lane];
            part.x += o.x;
            part.y += o.y;
          }
          asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(32 * kEpiPerQ) : "memory");
          // (2) send the row's partial over this CTA's 256 columns to the 3 CTAs
          // holding the same 128 rows (pair rank `rank` of each pair); slot by tile parity
          const int slot = (int)(ln_tiles & 1u);
          const int r = q * 32 + lane;
          // (the phase completes when this CTA has armed it and all 3 x 128 partials have landed:
          // st.async signals the destination's barrier itself — no cluster-scope fences)
          if (warp == 2 && elect_one()) mbar_arrive_expect_tx(&lnbar[slot], 3u * 128u * 8u);
          if (h == 0) {
#pragma unroll
            for (int dst = 0; dst < 3; ++dst)
              st_async_f2(lnx + (slot * 3 + (int)pr) * 128 + r, 2u * dst + rank, part, &lnbar[slot]);
          }
          // (3) the whole row's statistics
          mbar_wait(&lnbar[slot], (ln_tiles >> 1) & 1u);
          float s1 = 0.f, s2 = 0.f;
#pragma unroll
          for (int src = 0; src < 3; ++src) {
            const float2 o = lnx[(slot * 3 + src) * 128 + r];
            s1 += o.x;
            s2 += o.y;
          }
          const float inv_n = 1.f / (float)P.N;
          const float mean = s1 * inv_n;
          const float rstd = rsqrtf(fmaxf(s2 * inv_n - mean * mean, 0.f) + P.ln_eps);
          if (pr == 0 && h == 0 && row_ok) {
            P.ln_mean[row] = mean;
            P.ln_rstd[row] = rstd;
          }
          // (4) once the x stores have read the staging buffers, y = LN(x) in place -> TMA store
          if (elect_one()) bulk_wait_read0();
          __syncwarp();
          const int sw = lane & 7;
          for (int j = 0; j < my_groups; ++j) {
            uint8_t* rowp = buf(j) + lane * 128;
            const int cbase = n0 + (h + kEpiPerQ * j) * GW;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint4 w0 = *reinterpret_cast<const uint4*>(rowp + (((2 * k) ^ sw) << 4));
              const uint4 w1 = *reinterpret_cast<const uint4*>(rowp + (((2 * k + 1) ^ sw) << 4));
              const uint32_t u[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
              const float4* gb = reinterpret_cast<const float4*>(lngb + (cbase - (int)pr * kBNMax) + k * 16);
              uint32_t pk[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {  // y = ((x - mean) rstd) g + b = (x rstd - mean rstd) g + b
                const float2 xx = make_float2(half_to_f32((uint16_t)(u[e] & 0xFFFFu), FMT),
                                              half_to_f32((uint16_t)(u[e] >> 16), FMT));
                const float4 q4 = gb[e];  // (g, b) of columns 2e, 2e + 1
                const float2 t = __ffma2_rn(xx, make_float2(rstd, rstd), make_float2(-mean * rstd, -mean * rstd));
                const float2 y = __ffma2_rn(t, make_float2(q4.x, q4.z), make_float2(q4.y, q4.w));
                pk[e] = pack2_fmt(y.x, y.y, FMT);
              }
              *reinterpret_cast<uint4*>(rowp + (((2 * k) ^ sw) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
              *reinterpret_cast<uint4*>(rowp + (((2 * k + 1) ^ sw) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
            }
          }
          fence_async_smem();
          __syncwarp();
          if (elect_one()) {
            for (int j = 0; j < my_groups; ++j) tma_store_4d(&tmL, buf(j), n0 + (h + kEpiPerQ * j) * GW, row0, 0, 0);
            bulk_commit();
          }
          ++ln_tiles;
        }
        if (XO != XOP_NONE && XO != XOP_AUX_OUT && P.csum != nullptr && batched && row0 < P.M) {
          // fused column sum of the staged (rounded) C: lane l sums columns 2l, 2l+1
          // of each group over this warp's 32 rows (conflict-free: one row per step)
          __syncwarp();
          for (int j = 0; j < my_groups; ++j) {
            const int g = h + kEpiPerQ * j;
            const int nch = min(GW / 16, (P.BN - g * GW) / 16);
            const uint32_t base = smem_u32(buf(j)) + ((lane & 3) << 2);
            float2 s = make_float2(0.f, 0.f);
            auto add_row = [&](int rr) {
              uint32_t w;
              asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w) : "r"(base + rr * 128 + (((lane >> 2) ^ (rr & 7)) << 4)));
              s = add_h2<cf>(s, w);  // (mixed-precision adds: the same sums as unpack + FADD)
            };
            if (row0 + 32 <= P.M) {
#pragma unroll 8
              for (int rr = 0; rr < 32; ++rr) add_row(rr);
            } else {  // rows past M hold no data (the fast path stages them)
              for (int rr = 0; rr < P.M - row0; ++rr) add_row(rr);
            }
            const float s0 = s.x, s1 = s.y;
            const int col = n0 + g * GW + 2 * lane;
            if (2 * lane < nch * 16 && col < P.N) {
              float* o = P.csum + (long long)(row0 >> 5) * P.N + col;
              o[0] = s0;
              if (col + 1 < P.N) o[1] = s1;
            }
          }
        }
      } else {
        uint32_t r[16];
        const int chunk0 = h * 16;
        if (chunk0 < P.BN) tmem_ld16(taddr + chunk0, r);
        for (int c = chunk0; c < P.BN; c += 16 * kEpiPerQ) {
          tmem_ld_wait();
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]) * P.alpha;
          if (c + 16 * kEpiPerQ < P.BN) tmem_ld16(taddr + c + 16 * kEpiPerQ, r);  // next chunk in flight
          const int col = n0 + c;
          if (col >= P.N_store || !row_ok) continue;
          const int ncols = min(16, P.N_store - col);  // 8 or 16
          if (P.split > 1) {
            float* w = P.ws + ((long long)tc.s * P.M + row) * P.N + col;
            for (int i = 0; i < ncols; i += 4)
              *reinterpret_cast<float4*>(w + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            continue;
          }
          epi(v, col, ncols, v);  // (no staged operand on the direct path)
          const long long off = b1 * P.c_sb1 + b2 * P.c_sb2 + (long long)row * P.ldc + col;
          if (P.c_dtype == MPX_F32) {
            float* o = static_cast<float*>(P.C) + off;
            for (int i = 0; i < ncols; i += 4)
              *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          } else {
            constexpr int f = FMT;
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              pk[i] = pack2_fmt(v[2 * i], v[2 * i + 1], f);
            uint16_t* o = static_cast<uint16_t*>(P.C) + off;
            *reinterpret_cast<uint4*>(o) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            if (ncols == 16) *reinterpret_cast<uint4*>(o + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
        }
      }
      if (!P.tma_store) {  // (the staged path released it after its last TMEM load)
        tc_fence_before();
        if (CG == 2)
          mbar_arrive_remote(&tempty[acc], leader_rank);  // the leader's MMA reuses this accumulator
        else
          mbar_arrive(&tempty[acc]);
      }
      if (!WN) acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (P.tma_store && elect_one()) bulk_wait0();
  }
  __syncthreads();
  if (CG == 2) cluster_sync();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    if (CG == 2)
      tmem_dealloc_2sm<512>(tmem_base);
    else
      tmem_dealloc<512>(tmem_base);
  }
}

// fused column sum, second pass: out[c] = sum_k parts[k][c] over many partial
// rows; block = 32 columns x 32 partial lanes, four rows in flight per
// thread, fixed summation order
__global__ void __launch_bounds__(1024) colsum_parts_kernel(const float* __restrict__ parts, int nparts, int N,
                                                            void* out, int out_dtype) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  __shared__ float sm[32][33];
  const int cl = threadIdx.x & 31, kl = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + cl;
  float a = 0.f;
  if (c < N) {
    const float* w = parts + c;
    int k = kl;
    for (; k + 224 < nparts; k += 256) {  // 8 partial rows in flight, summed in row order
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = w[(long long)(k + 32 * u) * N];
#pragma unroll
      for (int u = 0; u < 8; ++u) a += v[u];
    }
    for (; k < nparts; k += 32) a += w[(long long)k * N];
  }
  sm[kl][cl] = a;
  __syncthreads();
  if (kl == 0 && c < N) {
    float t = 0.f;
    for (int k = 0; k < 32; ++k) t += sm[k][cl];
    if (out_dtype == MPX_F32)
      static_cast<float*>(out)[c] = t;
    else
      static_cast<uint16_t*>(out)[c] = f32_to_half(t, out_dtype == MPX_BF16 ? 1 : 0);
  }
}

// split-K: C = cast(sum_s ws[s]) (+ bias), summed in split order
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int split, long long mn, int N, void* C,
                                     long long ldc, int c_dtype, const void* bias, int ab_fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < mn; i += (long long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < split; ++k) s += ws[k * mn + i];
    const long long row = i / N, col = i - row * N;
    if (bias) s += half_to_f32(static_cast<const uint16_t*>(bias)[col], ab_fmt);
    const long long o = row * ldc + col;
    if (c_dtype == MPX_F32)
      static_cast<float*>(C)[o] = s;
    else
      static_cast<uint16_t*>(C)[o] = f32_to_half(s, c_dtype == MPX_BF16 ? 1 : 0);
  }
}

// the same, 4 columns per thread (N % 4 == 0, 16-byte aligned ws), all split
// loads of a step in flight together; one 2D index per row block, no 64-bit divides
__global__ void __launch_bounds__(256) splitk_reduce4_kernel(const float* __restrict__ ws, int split, int M, int N,
                                                             void* C, long long ldc, int c_dtype, const void* bias,
                                                             int ab_fmt) {
  ::mpx::pdl_grid_sync();  // programmatic dependent launch: inputs are final past here
  const int n4 = N / 4;
  const long long mn = (long long)M * N;
  const long long total = (long long)M * n4;
  // 32-bit index math when the output fits (every ViT shape): one 32-bit divide per 4 columns
  const bool small = total < (1ll << 31);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int row = small ? (int)((unsigned)i / (unsigned)n4) : (int)(i / n4);
    const int c4 = (int)(i - (long long)row * n4);
    const long long e = (long long)row * N + 4 * c4;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    int k = 0;
    for (; k + 4 <= split; k += 4) {
      float4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = __ldcs(reinterpret_cast<const float4*>(ws + (k + j) * mn + e));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a.x += v[j].x;
        a.y += v[j].y;
        a.z += v[j].z;
        a.w += v[j].w;
      }
    }
    for (; k < split; ++k) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(ws + k * mn + e));
      a.x += v.x;
      a.y += v.y;
      a.z += v.z;
      a.w += v.w;
    }
    float o[4] = {a.x, a.y, a.z, a.w};
    if (bias) {
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] += half_to_f32(static_cast<const uint16_t*>(bias)[4 * c4 + j], ab_fmt);
    }
    const long long off = (long long)row * ldc + 4 * c4;
    if (c_dtype == MPX_F32) {
#pragma unroll
      for (int j = 0; j < 4; ++j) static_cast<float*>(C)[off + j] = o[j];
    } else {
      const int f = c_dtype == MPX_BF16 ? 1 : 0;
      const uint2 w = make_uint2(pack2_fmt(o[0], o[1], f), pack2_fmt(o[2], o[3], f));
      if ((off & 3) == 0 && (reinterpret_cast<uintptr_t>(C) & 7) == 0)
        *reinterpret_cast<uint2*>(static_cast<uint16_t*>(C) + off) = w;
      else
        for (int j = 0; j < 4; ++j) static_cast<uint16_t*>(C)[off + j] = f32_to_half(o[j], f);
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 4-D map: (inner, outer, b1, b2) with byte strides for dims 1..3
static int make_map(CUtensorMap* m, const void* ptr, int ab_fmt, uint64_t inner, uint64_t outer, uint64_t nb1,
                    uint64_t nb2, uint64_t s_outer, uint64_t s_b1, uint64_t s_b2, uint32_t box_inner,
                    uint32_t box_outer, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return fail(MPX_EINVAL, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {inner, outer, nb1, nb2};
  cuuint64_t strides[3] = {s_outer, s_b1, s_b2};
  cuuint32_t box[4] = {box_inner, box_outer, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, ab_fmt ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                  const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MPX_EINVAL, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return 0;
}

// a zero batch stride means "shared across that batch dim": the map gets
// extent 1 there (TMA strides must be non-zero) and the kernel uses coordinate 0
static int make_map_dt(CUtensorMap* m, const void* ptr, CUtensorMapDataType dt, uint64_t inner, uint64_t outer,
                       uint64_t nb1, uint64_t nb2, uint64_t s_outer, uint64_t s_b1, uint64_t s_b2, uint32_t box_inner,
                       uint32_t box_outer, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return fail(MPX_EINVAL, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {inner, outer, nb1, nb2};
  cuuint64_t strides[3] = {s_outer, s_b1, s_b2};
  cuuint32_t box[4] = {box_inner, box_outer, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, dt, 4, const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MPX_EINVAL, "cuTensorMapEncodeTiled (C) failed (" + std::to_string((int)r) + ")");
  return 0;
}

// round-up multiplier for fdiv (s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1;
// exact for every n < 2^31 — checked exhaustively on small d and at the n edges)
static FastDiv make_fastdiv(uint32_t d) {
  uint32_t s = 0;
  while ((1ull << s) < d) ++s;
  return FastDiv{d, (uint32_t)(((1ull << 32) * ((1ull << s) - d)) / d + 1), s};
}
static uint64_t nz_stride(int64_t s, uint64_t fallback) { return s > 0 ? (uint64_t)s : fallback; }
static uint64_t ext(int64_t s, int n) { return s > 0 ? (uint64_t)n : 1u; }

}  // namespace mpx

using namespace mpx;

extern "C" int mpx_gemm(const mpx_gemm_desc* g, void* stream) {
  if (!g) return fail(MPX_EINVAL, "mpx_gemm: null desc");
  if (g->ab_dtype != MPX_F16 && g->ab_dtype != MPX_BF16) return fail(MPX_EINVAL, "mpx_gemm: A/B must be f16/bf16");
  if (g->M <= 0 || g->N <= 0 || g->K <= 0) return fail(MPX_EINVAL, "mpx_gemm: empty problem");
  const int n_store = (g->N + 7) / 8 * 8;
  if (n_store != g->N && (g->split_k > 1 || g->ldc < n_store))
    return fail(MPX_EINVAL, "mpx_gemm: N not a multiple of 8 needs ldc >= round_up(N, 8) and no split-K");
  const int fmt = g->ab_dtype == MPX_BF16 ? 1 : 0;
  const int nb1 = g->nb1 > 0 ? g->nb1 : 1, nb2 = g->nb2 > 0 ? g->nb2 : 1;
  int BN = g->block_n;
  if (BN <= 0) BN = g->N >= kBNMax ? kBNMax : ((g->N + 15) / 16) * 16;
  if (g->b_mn_major) BN = ((BN + 63) / 64) * 64;
  const bool wide = BN == 384 || BN == 512;  // the wide weight-gradient tiles (WN variants)
  const int wn = BN == 512 ? 2 : BN == 384 ? 1 : 0;
  if (wide && (!g->b_mn_major || g->act != ACT_NONE || g->residual || g->aux || g->M < 256))
    return fail(MPX_EINVAL, "mpx_gemm: block_n 384 / 512 is the MN-major-B plain-epilogue pair tile");
  if ((BN > kBNMax && !wide) || BN % 16) return fail(MPX_EINVAL, "mpx_gemm: bad block_n");
  const int split = g->split_k > 1 ? g->split_k : 1;
  if (split > 1 && (nb1 * nb2 != 1 || !g->workspace)) return fail(MPX_EINVAL, "mpx_gemm: split-K needs batch 1 + workspace");
  if (split > 1 && g->act != ACT_NONE) return fail(MPX_EINVAL, "mpx_gemm: split-K supports no activation");
  if (g->act == ACT_SOFTMAX || g->act == ACT_SOFTMAX_BWD) {
    // the epilogue needs whole rows: one N block, and 16-element aux reads
    if (g->N > BN || split > 1 || (g->c_dtype != MPX_F16 && g->c_dtype != MPX_BF16))
      return fail(MPX_EINVAL, "mpx_gemm: softmax epilogues need N <= 256 in one tile, 16-bit C, no split-K");
    if (g->act == ACT_SOFTMAX_BWD && (!g->aux || g->ld_aux < (g->N + 15) / 16 * 16 || g->ld_aux % 8))
      return fail(MPX_EINVAL, "mpx_gemm: softmax backward needs aux = P with ld_aux >= round_up(N, 16)");
  }
  const bool ln = g->ln_out != nullptr;
  if (ln && (g->N != 3 * kBNMax || BN != kBNMax || split > 1 || nb1 * nb2 != 1 || g->act != ACT_NONE ||
             !g->residual || g->b_mn_major || (g->c_dtype != MPX_F16 && g->c_dtype != MPX_BF16) || !g->ln_gain ||
             !g->ln_bias || !g->ln_mean || !g->ln_rstd || g->ld_ln % 8 || g->tma_store < 0 ||
             (g->cta_group != 0 && g->cta_group != 2)))
    return fail(MPX_EINVAL, "mpx_gemm: the fused LayerNorm needs N = 768, K-major B, a residual epilogue (no act), "
                            "batch 1, 16-bit C, no split-K, gain / bias / out / mean / rstd, ld_ln % 8 == 0");
  // CTA pair (M = 256 tiles) for the large problems; single CTA otherwise
  int CG = ln ? 2 : g->cta_group;
  const bool pair_ok = (BN == 256 || BN == 128 || wide) && (!g->b_mn_major || BN % 128 == 0);
  if (CG == 0) CG = (pair_ok && (g->M >= 512 || wide)) ? 2 : 1;
  if (wide && CG != 2) return fail(MPX_EINVAL, "mpx_gemm: block_n 384 / 512 needs the CTA pair");
  if (CG != 1 && CG != 2) return fail(MPX_EINVAL, "mpx_gemm: cta_group must be 0, 1 or 2");
  if (CG == 2 && !pair_ok) return fail(MPX_EINVAL, "mpx_gemm: cta_group 2 needs BN 128/256");

  const uint64_t es = 2;
  CUtensorMap ta, tb;
  int rc;
  // A: K-major dims (K, M), MN-major dims (M, K); lda = element stride of the outer dim
  const uint64_t an1 = ext(g->a_sb1, nb1), an2 = ext(g->a_sb2, nb2), bn1 = ext(g->b_sb1, nb1), bn2 = ext(g->b_sb2, nb2);
  if (!g->a_mn_major)
    rc = make_map(&ta, g->A, fmt, g->K, g->M, an1, an2, g->lda * es, nz_stride(g->a_sb1 * es, g->lda * es * g->M),
                  nz_stride(g->a_sb2 * es, g->lda * es * g->M), 64, kBM);
  else
    rc = make_map(&ta, g->A, fmt, g->M, g->K, an1, an2, g->lda * es, nz_stride(g->a_sb1 * es, g->lda * es * g->K),
                  nz_stride(g->a_sb2 * es, g->lda * es * g->K), 64, 64);
  if (rc) return rc;
  if (!g->b_mn_major)
    rc = make_map(&tb, g->B, fmt, g->K, g->N, bn1, bn2, g->ldb * es, nz_stride(g->b_sb1 * es, g->ldb * es * g->N),
                  nz_stride(g->b_sb2 * es, g->ldb * es * g->N), 64, BN / CG);
  else
    rc = make_map(&tb, g->B, fmt, g->N, g->K, bn1, bn2, g->ldb * es, nz_stride(g->b_sb1 * es, g->ldb * es * g->K),
                  nz_stride(g->b_sb2 * es, g->ldb * es * g->K), 64, 64);
  if (rc) return rc;

  GemmParams P{};
  P.M = g->M;
  P.N = g->N;
  P.N_store = n_store;
  P.K = g->K;
  P.BN = BN;
  P.a_mn = g->a_mn_major;
  P.b_mn = g->b_mn_major;
  P.nb1 = nb1;
  P.nbatch = nb1 * nb2;
  P.a_bc1 = g->a_sb1 <= 0;
  P.a_bc2 = g->a_sb2 <= 0;
  P.b_bc1 = g->b_sb1 <= 0;
  P.b_bc2 = g->b_sb2 <= 0;
  P.split = split;
  P.m_blocks = (g->M + kBM * CG - 1) / (kBM * CG);
  P.n_blocks = (g->N + BN - 1) / BN;
  P.k_blocks = (g->K + kBK - 1) / kBK;
  P.kb_per_split = (P.k_blocks + split - 1) / split;
  P.total_tiles = (long long)P.nbatch * split * P.m_blocks * P.n_blocks;
  if (P.total_tiles >= (1ll << 31)) return fail(MPX_EINVAL, "mpx_gemm: more than 2^31 - 1 output tiles");
  P.fd_mn = make_fastdiv((uint32_t)(P.m_blocks * P.n_blocks));
  P.fd_split = make_fastdiv((uint32_t)split);
  P.fd_grp = make_fastdiv((uint32_t)(kGroupM * P.n_blocks));
  P.fd_gmt = make_fastdiv(P.m_blocks % kGroupM ? (uint32_t)(P.m_blocks % kGroupM) : 1u);
  P.fd_nb1 = make_fastdiv((uint32_t)nb1);
  P.idesc = ptx::idesc_f16(fmt, kBM * CG, wide ? 256 : BN, g->a_mn_major, g->b_mn_major);
  P.idesc2 = ptx::idesc_f16(fmt, kBM * CG, wn == 2 ? 256 : 128, g->a_mn_major, g->b_mn_major);
  P.ab_fmt = fmt;
  P.C = g->C;
  P.ldc = g->ldc;
  P.c_sb1 = g->c_sb1;
  P.c_sb2 = g->c_sb2;
  P.c_dtype = g->c_dtype;
  if (split == 1 && g->c_dtype != MPX_F32 && g->c_dtype != g->ab_dtype)
    return fail(MPX_EINVAL, "mpx_gemm: a 16-bit C must have the A/B format");
  P.bias = g->bias;
  P.res = g->residual;
  P.ldr = g->ldr;
  P.r_sb1 = g->r_sb1;
  P.r_sb2 = g->r_sb2;
  P.aux = g->aux;
  P.ld_aux = g->ld_aux;
  P.alpha = g->alpha == 0.f ? 1.f : g->alpha;
  P.act = g->act;
  P.ws = static_cast<float*>(g->workspace);
  P.csum = nullptr;
  if (split > 1 && (long long)(split - 1) * P.kb_per_split >= P.k_blocks)
    return fail(MPX_EINVAL, "mpx_gemm: split_k too large for K");

  // outputs go through swizzled smem staging + TMA stores when the layout
  // allows: 16-bit / f32 C, and the f32 split-K partials ws[split][M][N]
  CUtensorMap tc = tb;
  if (g->tma_store >= 0) {
    if (split > 1) {
      const uint64_t s_m = (uint64_t)g->N * 4;
      if (g->N % 4 == 0 && reinterpret_cast<uintptr_t>(g->workspace) % 16 == 0 && (BN % 32 == 0)) {
        rc = make_map_dt(&tc, g->workspace, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, g->N, g->M, split, 1, s_m,
                         s_m * g->M, s_m * g->M * split, 32, 32);
        if (rc) return rc;
        P.tma_store = 1;
      }
    } else {
      const int es_c = g->c_dtype == MPX_F32 ? 4 : 2;
      const bool c_aligned = (reinterpret_cast<uintptr_t>(g->C) % 16 == 0) && (g->ldc * es_c) % 16 == 0 &&
                             (nb1 == 1 || (g->c_sb1 > 0 && (g->c_sb1 * es_c) % 16 == 0)) &&
                             (nb2 == 1 || (g->c_sb2 > 0 && (g->c_sb2 * es_c) % 16 == 0));
      const int gw = es_c == 4 ? 32 : 64;
      if (c_aligned && (BN % gw == 0 || P.n_blocks == 1) && (es_c == 2 || g->act == ACT_NONE && !g->bias && !g->residual)) {
        const uint64_t s_m = (uint64_t)g->ldc * es_c;
        const CUtensorMapDataType dt = g->c_dtype == MPX_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                       : g->c_dtype == MPX_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                                : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
        rc = make_map_dt(&tc, g->C, dt, g->N, g->M, nb1, nb2, s_m, nb1 > 1 ? (uint64_t)g->c_sb1 * es_c : s_m * g->M,
                         nb2 > 1 ? (uint64_t)g->c_sb2 * es_c : s_m * g->M, es_c == 4 ? 32 : 64, 32);
        if (rc) return rc;
        P.tma_store = 1;
      }
    }
  }

  // epilogue operand (residual in / GELU aux in / GELU aux out) through TMA when possible
  CUtensorMap tx = tb;
  P.xop = XOP_NONE;
  static const bool no_xop = getenv("MPX_GEMM_NO_XOP") != nullptr;  // debugging switch
  if (P.tma_store && split == 1 && g->c_dtype != MPX_F32 && g->tma_store >= 0 && !no_xop) {
    const uint64_t es2 = 2;
    auto al16 = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
    const bool gelu_out = g->act == ACT_GELU || g->act == ACT_GELU_D;
    if ((gelu_out || g->act == ACT_GELU_BWD || g->act == ACT_MUL_AUX) && !g->residual && g->aux && al16(g->aux) &&
        g->ld_aux % 8 == 0 && (nb1 == 1 || (g->c_sb1 > 0 && g->c_sb1 % 8 == 0)) &&
        (nb2 == 1 || (g->c_sb2 > 0 && g->c_sb2 % 8 == 0))) {
      const uint64_t s_m = (uint64_t)g->ld_aux * es2;
      P.xop = gelu_out ? XOP_AUX_OUT : XOP_AUX_IN;
      // GELU out: aux and C leave as 64-column SW128 tiles, one 4 KB staging buffer each
      const bool out2 = P.xop == XOP_AUX_OUT;
      // (GELU-aux-out with 32-column groups: 32-column SW64 boxes)
      const bool gw32 = out2 && MPX_AUXOUT_GW == 32;
      const CUtensorMapSwizzle swz = gw32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
      const uint32_t box_c = gw32 ? 32 : 64;
      rc = make_map(&tx, g->aux, fmt, g->N, g->M, nb1, nb2, s_m, nb1 > 1 ? (uint64_t)g->c_sb1 * es2 : s_m * g->M,
                    nb2 > 1 ? (uint64_t)g->c_sb2 * es2 : s_m * g->M, box_c, 32, swz);
      if (rc) return rc;
      if (out2) {
        const uint64_t s_c = (uint64_t)g->ldc * es2;
        rc = make_map(&tc, g->C, g->c_dtype == MPX_BF16 ? 1 : 0, g->N, g->M, nb1, nb2, s_c,
                      nb1 > 1 ? (uint64_t)g->c_sb1 * es2 : s_c * g->M, nb2 > 1 ? (uint64_t)g->c_sb2 * es2 : s_c * g->M,
                      box_c, 32, swz);
        if (rc) return rc;
      }
    } else if (g->act == ACT_NONE && g->residual && al16(g->residual) && g->ldr % 8 == 0 &&
               (nb1 == 1 || g->r_sb1 == 0 || g->r_sb1 % 8 == 0) && (nb2 == 1 || g->r_sb2 == 0 || g->r_sb2 % 8 == 0)) {
      const uint64_t s_m = (uint64_t)g->ldr * es2;
      rc = make_map(&tx, g->residual, fmt, g->N, g->M, ext(g->r_sb1, nb1), ext(g->r_sb2, nb2), s_m,
                    g->r_sb1 > 0 ? (uint64_t)g->r_sb1 * es2 : s_m * g->M,
                    g->r_sb2 > 0 ? (uint64_t)g->r_sb2 * es2 : s_m * g->M, 64, 32);
      if (rc) return rc;
      P.xop = XOP_RES_IN;
    }
  }
  if (P.tma_store && P.xop == XOP_NONE && g->act == ACT_NONE && !g->residual && !no_xop) P.xop = XOP_PLAIN;
  CUtensorMap tl = tb;  // the LayerNorm output (RES_LN), laid out like C
  if (ln) {
    if (P.xop != XOP_RES_IN || !P.tma_store)
      return fail(MPX_EINVAL, "mpx_gemm: the fused LayerNorm needs the staged residual epilogue (aligned C / residual)");
    P.xop = XOP_RES_LN;
    const uint64_t s_l = (uint64_t)g->ld_ln * 2;
    rc = make_map(&tl, g->ln_out, fmt, g->N, g->M, 1, 1, s_l, s_l * g->M, s_l * g->M, 64, 32);
    if (rc) return rc;
    P.ln_g = g->ln_gain;
    P.ln_b = g->ln_bias;
    P.ln_mean = g->ln_mean;
    P.ln_rstd = g->ln_rstd;
    P.ln_eps = g->ln_eps;
    P.total_tiles = P.m_blocks;  // the cluster's pairs share each 256-row block
  }

  using KernelFn = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                           const CUtensorMap, const GemmParams);
  static const KernelFn kernels[2][2][6] = {
      {{gemm_kernel<1, XOP_NONE, 0>, gemm_kernel<1, XOP_RES_IN, 0>, gemm_kernel<1, XOP_AUX_IN, 0>,
        gemm_kernel<1, XOP_AUX_OUT, 0>, gemm_kernel<1, XOP_PLAIN, 0>, nullptr},
       {gemm_kernel<2, XOP_NONE, 0>, gemm_kernel<2, XOP_RES_IN, 0>, gemm_kernel<2, XOP_AUX_IN, 0>,
        gemm_kernel<2, XOP_AUX_OUT, 0>, gemm_kernel<2, XOP_PLAIN, 0>, gemm_kernel<2, XOP_RES_LN, 0>}},
      {{gemm_kernel<1, XOP_NONE, 1>, gemm_kernel<1, XOP_RES_IN, 1>, gemm_kernel<1, XOP_AUX_IN, 1>,
        gemm_kernel<1, XOP_AUX_OUT, 1>, gemm_kernel<1, XOP_PLAIN, 1>, nullptr},
       {gemm_kernel<2, XOP_NONE, 1>, gemm_kernel<2, XOP_RES_IN, 1>, gemm_kernel<2, XOP_AUX_IN, 1>,
        gemm_kernel<2, XOP_AUX_OUT, 1>, gemm_kernel<2, XOP_PLAIN, 1>, gemm_kernel<2, XOP_RES_LN, 1>}}};
  static const KernelFn wide_kernels[2][2] = {{gemm_kernel<2, XOP_PLAIN, 0, 1>, gemm_kernel<2, XOP_PLAIN, 1, 1>},
                                              {gemm_kernel<2, XOP_PLAIN, 0, 2>, gemm_kernel<2, XOP_PLAIN, 1, 2>}};
  // fused column sum: in the staged lean epilogues (16-bit C, one batch), else a separate pass
  bool csum_fused = false;
  if (g->colsum_out) {
    if (!g->colsum_ws) return fail(MPX_EINVAL, "mpx_gemm: colsum_out needs colsum_ws");
    csum_fused = P.tma_store && split == 1 && g->c_dtype != MPX_F32 && nb1 * nb2 == 1 && P.xop != XOP_NONE &&
                 P.xop != XOP_AUX_OUT &&
                 BN <= 64 * kEpiPerQ * (P.xop == XOP_PLAIN ? GemmSmem<XOP_PLAIN>::kBufPerWarp
                                                           : GemmSmem<XOP_AUX_IN>::kBufPerWarp);
    if (csum_fused) P.csum = g->colsum_ws;
  }
  if (wide && P.xop != XOP_PLAIN)
    return fail(MPX_EINVAL, "mpx_gemm: block_n 384 / 512 needs the TMA-store plain epilogue (aligned C / workspace)");
  const KernelFn kern = wide ? wide_kernels[wn - 1][fmt] : kernels[fmt][CG - 1][P.xop];
  const unsigned threads = P.xop == XOP_AUX_OUT ? EpiCfg<XOP_AUX_OUT>::kThreads : EpiCfg<XOP_PLAIN>::kThreads;
  const cudaError_t attr_err = ensure_smem_attr((const void*)kern, (int)kGemmSmem);
  if (attr_err != cudaSuccess) return fail((int)attr_err, "cudaFuncSetAttribute(gemm_kernel)");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (CG == 1) {
    const long long grid = std::min<long long>(P.total_tiles, current_num_sms());
    MPX_CUDA_CHECK(::mpx::launch_k(kern, (unsigned)grid, threads, kGemmSmem, st, ta, tb, tc, tx, tl, P));
  } else {
    // the LayerNorm variant: clusters of 3 CTA pairs, one 256-row block each.  A
    // 6-CTA cluster must fit in one GPC, so fewer than SMs / 6 may be co-resident:
    // the persistent grid is sized by the occupancy query (a second wave of
    // clusters would double the tail)
    const int per = P.xop == XOP_RES_LN ? 6 : 2;
    long long slots = current_num_sms() / per;
    cudaLaunchConfig_t cfg{};
    if (per == 6) {
      cudaLaunchConfig_t q{};
      q.gridDim = dim3((unsigned)(6 * slots));
      q.blockDim = dim3(threads);
      q.dynamicSmemBytes = kGemmSmem;
      cudaLaunchAttribute qa[1];
      qa[0].id = cudaLaunchAttributeClusterDimension;
      qa[0].val.clusterDim.x = 6;
      qa[0].val.clusterDim.y = 1;
      qa[0].val.clusterDim.z = 1;
      q.attrs = qa;
      q.numAttrs = 1;
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, (const void*)kern, &q) == cudaSuccess && n > 0) slots = n;
    }
    const long long units = std::min<long long>(P.total_tiles, slots);
    cfg.gridDim = dim3((unsigned)(per * units));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = kGemmSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = per;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;  // (no PDL for the ViT kernels, see launch_k)
    count_launch();
    MPX_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tx, tl, P));
  }
  MPX_LAUNCH_CHECK("gemm_kernel");
  if (split > 1) {
    const long long mn = (long long)g->M * g->N;
    if (g->N % 4 == 0 && reinterpret_cast<uintptr_t>(P.ws) % 16 == 0)
      MPX_CUDA_CHECK(::mpx::launch_k(splitk_reduce4_kernel, current_num_sms() * 8, 256, 0, st, P.ws, split, g->M, g->N, g->C, g->ldc, g->c_dtype,
                                                                   g->bias, fmt));
    else
      MPX_CUDA_CHECK(::mpx::launch_k(splitk_reduce_kernel, current_num_sms() * 4, 256, 0, st, P.ws, split, mn, g->N, g->C, g->ldc, g->c_dtype,
                                                                 g->bias, fmt));
    MPX_LAUNCH_CHECK("splitk_reduce_kernel");
  }
  if (g->colsum_out) {
    if (csum_fused) {
      const int parts = (g->M + 31) / 32;
      MPX_CUDA_CHECK(::mpx::launch_k(colsum_parts_kernel, (unsigned)((g->N + 31) / 32), 1024, 0, st, g->colsum_ws, parts, g->N, g->colsum_out,
                                                                         g->c_dtype));
      MPX_LAUNCH_CHECK("colsum_parts_kernel");
    } else {
      const int rc2 = mpx_colsum(g->c_dtype, g->C, g->ldc, 0, g->M, g->N, 1, g->colsum_ws,
                                 (int64_t)((g->M + 31) / 32) * g->N, g->colsum_out, g->N, g->c_dtype, 1.f, stream);
      if (rc2) return rc2;
    }
  }
  return 0;
}

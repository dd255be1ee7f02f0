/*
 * mpx_b200.h — C ABI of the B200-native mixed-precision training step.
 *
 * The reference (`mpsim`, /root/reference/pkg) is pure Python/numpy and has
 * no FFI: its hot path is a set of Python functions.  Each entry point below
 * is the native body of one of those functions; the Python host layer
 * (paper_2507_03312_b200/) keeps the reference names and calls these through
 * ctypes with raw device pointers and the caller's CUDA stream.
 *
 * Conventions
 *   - every pointer named d_* is a device pointer owned by the caller;
 *   - arrays of per-leaf pointers/sizes (h_*) are HOST arrays, read before the
 *     call returns (a leaf table is packed into the kernel's parameter block,
 *     no host->device copy, no allocation);
 *   - `stream` is a cudaStream_t (0 = legacy default stream);
 *   - every call is stream-ordered and asynchronous: nothing synchronises the
 *     host;
 *   - return value 0 = success, otherwise a cudaError_t / MPX_E* code; the
 *     message is available from mpx_last_error() on the calling thread.
 *
 * Numerics contract: casts are IEEE round-to-nearest-
 * even with subnormals and overflow to inf; unscale is an IEEE f32 division;
 * Adam uses single-rounded f32 operations in the reference's order with no
 * FMA contraction, so results are bit-identical to the reference.
 */
#ifndef MPX_B200_H
#define MPX_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes — mirror mpsim.dtypes.DType (dtypes.py:31-46) */
enum {
  MPX_F32 = 0,
  MPX_F16 = 1,
  MPX_BF16 = 2,
};

/* error codes beyond cudaError_t */
enum {
  MPX_EINVAL = 10001,     /* bad argument (dtype, size, null pointer) */
  MPX_ETOOMANY = 10002,   /* internal: leaf table overflow */
  MPX_ENCCL = 10003,      /* NCCL missing or an NCCL call failed */
};

/* Device-resident dynamic loss-scaling state.  Field-for-field the
 * reference's LossScaling NamedTuple (precision.py:120-132); fp64 so the
 * trajectory is bit-identical to the Python-double state machine. */
typedef struct mpx_scaling_state {
  double loss_scale;
  double growth_factor;
  double backoff_factor;
  double min_scale;
  int64_t growth_interval;
  int64_t steps_since_growth;
} mpx_scaling_state;

/* Adam/SGD hyper-parameters, already rounded the way the reference rounds
 * its weak Python scalars (np.float32(x) at use, tensors.py:187,235-236):
 *   b1 = f32(beta1), omb1 = f32(1.0 - beta1), b2 = f32(beta2),
 *   omb2 = f32(1.0 - beta2), lr = f32(lr), eps = f32(eps),
 *   neg_lr = f32(-lr) (SGD, optim.py:60-66), neg_lr_wd = f32(-lr*wd)
 *   (decoupled weight decay; 0 => the exact reference Adam path). */
typedef struct mpx_adam_hparams {
  float b1, omb1, b2, omb2, lr, eps, neg_lr, neg_lr_wd;
} mpx_adam_hparams;

const char* mpx_last_error(void);
int mpx_version(void);
int mpx_num_sms(int device);
/* kernels launched by this library so far in this process (every entry
 * point); bench.py reports its timed regions' launches from it */
int64_t mpx_launch_count(void);

/* K1 — multi-tensor cast/scale: dst[i] = round_{dst_dtype}(f32(src[i]) * s).
 * Replaces cast_tree/cast_to_* (precision.py:53-85, T.cast tensors.py:529,
 * quantize_array dtypes.py:100-123) and LossScaling.scale (precision.py:134-143,
 * T.mul(leaf, s)).  The multiplier is taken from d_scale (a device fp64, e.g.
 * &state->loss_scale) when non-NULL, else from `scale` (host fp64); 1.0 means a
 * plain cast (the multiply is skipped).  src/dst dtypes are per call. */
int mpx_cast(const void* const* h_src, void* const* h_dst, const int64_t* h_numel,
             int n_leaves, int src_dtype, int dst_dtype, double scale,
             const double* d_scale, void* stream);

/* K2 — fused unscale + non-finite check (precision.py:145-154 and
 * tree.py:125-131 run back to back at precision.py:225-226):
 *   g32 = f32(g) / f32(loss_scale)   (IEEE division; x * 2^-k when exact)
 *   *d_flag &= all(isfinite(g32))
 * h_out may be NULL (flag only, nothing written) or an array of f32 outputs
 * (NULL entries allowed).  The divisor comes from d_scale (device fp64) when
 * non-NULL, else from `scale`.  If reset_flag != 0 the flag is set to 1 first
 * (stream-ordered), so one call computes all_finite of the whole table. */
int mpx_unscale_finite(const void* const* h_g, float* const* h_out, const int64_t* h_numel,
                       int n_leaves, int g_dtype, double scale, const double* d_scale,
                       uint32_t* d_flag, int reset_flag, void* stream);

/* K3 — LossScaling.adjust on the device (precision.py:156-173), fp64, one
 * thread, no host sync.  If d_step_count is non-NULL it is incremented when
 * the flag is set (optimizer step counter: only applied steps count,
 * optim.py:102-103).  d_used_scale (optional) receives the pre-adjust scale. */
int mpx_scaling_adjust(mpx_scaling_state* d_state, const uint32_t* d_flag,
                       int64_t* d_step_count, double* d_used_scale, void* stream);

/* K4 — finite-gated fused optimizer step (optim.py:58-113).
 *   mode 0 = Adam (compute_updates Adam branch + apply_leaf),
 *   mode 1 = SGD.
 * Per leaf: master p (f32/f16/bf16, updated in place and re-rounded to its own
 * dtype), moments m, v (f32, in place; ignored for SGD), gradient g of g_dtype
 * (f32 grads are used as-is; f16/bf16 grads are *scaled* grads, unscaled in
 * the kernel with the same division as K2), optional half working copy
 * h_half[i] of half_dtype written in the same pass (NULL = none), optional
 * h_upd[i] (if non-NULL the f32 update u is written there and p is NOT
 * modified: compute_updates without apply).
 * The whole call is a no-op when *d_flag == 0 (d_flag may be NULL = always).
 * Bias correction: t = d_counter[0] + 1 (applied steps only);
 * d_bc_table[2*(t-1)+{0,1}] = f32(1 - beta{1,2}**t) computed on the host in
 * double (optim.py:73-76); t is clamped to bc_len.
 * d_counter is int64[2] = {step_count, scratch}: when the step is applied the
 * last block to finish increments step_count (optim.py:77 `step_count=t`,
 * SGD optim.py:66) and leaves scratch at 0, so the call needs no extra launch
 * and never syncs.  scratch must be 0 on entry (it is after every call). */
int mpx_optimizer_step(void* const* h_p, const int32_t* h_p_dtype, float* const* h_m,
                       float* const* h_v, const void* const* h_g, void* const* h_half,
                       float* const* h_upd, const int64_t* h_numel, int n_leaves,
                       int g_dtype, int half_dtype, int mode, mpx_adam_hparams hp,
                       const float* d_bc_table, int64_t bc_len, int64_t* d_counter,
                       double scale, const double* d_scale, const uint32_t* d_flag,
                       void* stream);

/* K5 — tcgen05 GEMM with f32 accumulation (tensors.py:387-422 matmul and its
 * backward rule autodiff.py:193-205, at half precision with f32 accumulate):
 *   C[z][m,n] = epi(alpha * sum_k A[z][m,k] * B[z][k,n]),  z = b1 + nb1*b2
 * A is K-major (element (m,k) at A[m*lda + k]) or MN-major (A[k*lda + m]);
 * B is K-major (B[n*ldb + k]) or MN-major (B[k*ldb + n]); *_sb1/_sb2 are the
 * element strides of the two batch dims (0 = the operand is shared across that
 * dim, e.g. one weight for every image; likewise r_sb* for the residual).  Strides must be
 * multiples of 8 elements (16-byte TMA rule).  When N is not a multiple of 8
 * the epilogue writes whole 8-column groups (the pad columns get the value of
 * zero-filled operands), so ldc must be >= round_up(N, 8).
 * Epilogue (fused, per element, f32): + bias[n]; act GELU (aux receives the
 * rounded pre-activation) or GELU-backward (multiplies by gelu'(aux[m,n]));
 * + residual[m,n]; store as c_dtype (f32/f16/bf16).  bias/residual/aux share
 * ab_dtype; a 16-bit C must have the A/B format (f32 C any).  split_k > 1
 * (batch 1, no act) reduces through `workspace` (split*M*N f32) with a second
 * deterministic pass. */
typedef struct mpx_gemm_desc {
  int ab_dtype; /* MPX_F16 / MPX_BF16 */
  int M, N, K;
  const void* A;
  int64_t lda, a_sb1, a_sb2;
  int a_mn_major;
  const void* B;
  int64_t ldb, b_sb1, b_sb2;
  int b_mn_major;
  int nb1, nb2;
  void* C;
  int64_t ldc, c_sb1, c_sb2;
  int c_dtype;
  const void* bias;
  const void* residual;
  int64_t ldr, r_sb1, r_sb2;
  void* aux;
  int64_t ld_aux;
  float alpha; /* 0 means 1 */
  int act;     /* 0 none, 1 GELU, 2 GELU backward, 3 row softmax of round_half(alpha*acc)
                  (whole rows: N <= 256 in one tile), 4 softmax backward: C = P*(alpha*acc -
                  rowsum(P*alpha*acc)) with aux = P (ld_aux >= round_up(N, 16)); aux is
                  addressed with C's batch strides; 5 GELU whose aux receives
                  round_half(gelu'(pre)) (what _bw_gelu multiplies by, autodiff.py:173-185);
                  6 C = acc * aux (the backward of 5: the saved derivative) */
  int block_n; /* 0 = auto (<= 256); 384 = the wide weight-gradient tile: CTA pair, 256 x 384,
                  one accumulator, MN-major B, no act / residual / aux, TMA-store epilogue
                  (aligned C or workspace) */
  int split_k; /* <= 1: none */
  void* workspace;
  int cta_group; /* 0 = auto, 1 = one CTA per 128-row tile, 2 = CTA pair per 256-row tile */
  int tma_store; /* 0 = auto (16-bit C through smem + TMA stores), -1 = direct stores */
  /* optional fused column sum of the stored C (the next layer's bias gradient,
   * _unbroadcast autodiff.py:88-99): colsum_out[n] = sum_m C[m,n] over the
   * rounded C values, through colsum_ws (>= ceil(M/32)*N f32) in two
   * deterministic passes.  Needs the staged epilogue (batch 1, split_k 1, 16-bit
   * C, no GELU-aux-out); colsum_out has C's dtype. */
  float* colsum_ws;
  void* colsum_out;
  /* optional fused LayerNorm of the stored C rows (tensors.py:459-491):
   * ln_out[m, :] = (C[m, :] - mean) * rstd * ln_gain + ln_bias over each WHOLE row,
   * mean / rstd (f32 per row) saved for the backward.  Needs N == 768 (a cluster of
   * three CTA pairs owns a 256-row block and exchanges row sums over distributed
   * shared memory), the residual epilogue (no act), batch 1, 16-bit C, split 1;
   * ln_out has C's layout with leading dimension ld_ln.  NULL ln_out = off. */
  const void* ln_gain;
  const void* ln_bias;
  void* ln_out;
  int64_t ld_ln;
  float* ln_mean;
  float* ln_rstd;
  float ln_eps;
} mpx_gemm_desc;

int mpx_gemm(const mpx_gemm_desc* desc, void* stream);

/* ---- ViT kernels around the GEMMs (f32 islands + reductions) ----------- */
/* K7 LayerNorm over the last dim, f32 inside (tensors.py:459-491, used as an
 * island at bench.py:185-187).  x/y rows have element strides ldx/ldy; mean
 * and rstd (f32 per row) are saved for the backward. */
int mpx_layernorm_fwd(int dtype, const void* x, int64_t ldx, const void* gain, const void* bias, void* y,
                      int64_t ldy, float* mean, float* rstd, int rows, int D, float eps, void* stream);
/* backward (autodiff.py:243-262): dx (+ dres residual cotangent), dgain and
 * dbias (column sums, written as dtype).  workspace: 2*mpx_layernorm_bwd_blocks(rows)*D f32 */
int mpx_layernorm_bwd_blocks(int rows);
int mpx_layernorm_bwd(int dtype, const void* x, int64_t ldx, const void* gain, const float* mean, const float* rstd,
                      const void* dy, int64_t lddy, const void* dres, int64_t ldres, void* dx, int64_t lddx,
                      void* dgain, void* dbias, float* workspace, int rows, int D, void* stream);
/* K7 backward, occupancy-split form: dx as above, then one coalesced pass
 * for dgain, dbias and (dxsum != NULL) the column sum of dx itself — the
 * gradient of the bias that produced this residual stream (proj.b / fc2.b).
 * workspace >= 3 * splits * D floats (splits <= 4 * SMs). */
int mpx_layernorm_bwd2(int dtype, const void* x, int64_t ldx, const void* gain, const float* mean, const float* rstd,
                       const void* dy, int64_t lddy, const void* dres, int64_t ldres, void* dx, int64_t lddx,
                       void* dgain, void* dbias, void* dxsum, float* workspace, int64_t workspace_floats, int rows,
                       int D, void* stream);
/* out[z][c] = alpha * sum_r x[z][r][c]: bias / position gradients
 * (_unbroadcast, autodiff.py:88-99) and the mean-pool island; deterministic
 * two passes through workspace (>= splits*cols*batches f32). */
int mpx_colsum(int dtype, const void* x, int64_t ldx, int64_t sbx, int rows, int cols, int batches, float* workspace,
               int64_t workspace_floats, void* out, int64_t ld_out, int out_dtype, float alpha, void* stream);
/* K6 softmax over rows of length L (row stride ld, pad columns written 0),
 * f32 inside (tensors.py:431-446); backward dS = y*(dP - sum(dP*y)) with y
 * recomputed from S in f32 (autodiff.py:233-240). */
int mpx_softmax_fwd(int dtype, const void* S, void* P, int64_t rows, int L, int64_t ld, void* stream);
int mpx_softmax_bwd(int dtype, const void* S, const void* dP, void* dS, int64_t rows, int L, int64_t ld, void* stream);
/* K9 mean cross-entropy in f32 (tensors.py:494-522): nll_ws[B] scratch,
 * *loss (device f32).  Backward (autodiff.py:265-276): dlogits =
 * (softmax - onehot) * (*d_dloss) / B, columns >= C of each ld_d row zeroed. */
int mpx_cross_entropy_fwd(int dtype, const void* logits, int64_t ld, const int32_t* labels, int B, int C,
                          float* nll_ws, float* loss, void* stream);
int mpx_cross_entropy_bwd(int dtype, const void* logits, int64_t ld, const int32_t* labels, int B, int C,
                          const float* d_dloss, void* dlogits, int64_t ld_d, void* stream);
/* K6 fused attention forward (bench.py:196-198 with its softmax island):
 * O[b*N + n, h*hd + :] = softmax(round(Q K^T * scale)) V for every image b and
 * head h, reading Q/K/V straight from qkv [B, N, 3, H, hd]; scores live in
 * TMEM, probabilities in shared memory — nothing N x N reaches HBM.
 * Requires hd == 64 and N <= 256 (ViT-B/16, ViT-L/16: N = 197).  row_stats
 * (nullable, f32 [B*H*ceil(N/128)*128*2]) receives each query row's softmax
 * (max, 1/sum) for mpx_attention_bwd; p_save (nullable, 16-byte aligned,
 * mpx_attention_psave_bytes) receives the rounded probabilities P exactly as
 * the P V product consumed them (the saved softmax output of the reference's
 * autodiff), as [B*H][N][16*ceil(N/16)] half. */
int mpx_attention_fwd(int dtype, const void* qkv, int B, int N, int H, int hd, float scale, void* O, int64_t ldo,
                      float* row_stats, void* p_save, void* stream);
int64_t mpx_attention_psave_bytes(int B, int N, int H);
/* K6 fused attention backward: given qkv and dO [B*N, H*hd], writes the whole
 * dqkv [B*N, 3*H*hd] (dQ = scale dS K, dK = scale dS^T Q, dV = P^T dO with
 * dS = P (dP - rowsum(P dP)), dP = dO V^T.  P is the forward's saved tiles
 * when p_saved is given (reloaded, no score recompute), else recomputed on chip
 * — from the forward's row_stats when given, else from the scores here).
 * colsum_ws (f32 [B*3*H*hd]) + colsum_out (3*H*hd, dtype), both or neither:
 * colsum_out = sum over rows of the stored dqkv (the qkv bias gradient). */
int mpx_attention_bwd(int dtype, const void* qkv, const void* dO, int B, int N, int H, int hd, float scale,
                      void* dqkv, const float* row_stats, const void* p_saved, float* colsum_ws, void* colsum_out,
                      void* stream);
/* image [B,H,W,C] -> patch rows [B*(H/P)*(W/P), P*P*C], order (py, px, c) */
int mpx_patchify(int dtype, const void* img, void* patches, int B, int H, int W, int C, int P, void* stream);
/* strided row copy dst[b][r][c] = src[b][r][c] */
/* dst[c*ld_dst + r] = src[r*ld_src + c] (16-bit): the forward keeps its
 * weights K-major for the GEMM's B operand (MN-major B costs ~6 %) */
int mpx_transpose(int dtype, const void* src, int rows, int cols, int64_t ld_src, void* dst, int64_t ld_dst,
                  void* stream);
/* the same for n <= 64 matrices in one launch (the forward's weight copies) */
int mpx_transpose_batch(int dtype, int n, const void* const* src, void* const* dst, const int* rows,
                        const int* cols, const int64_t* ld_src, const int64_t* ld_dst, void* stream);
int mpx_copy_rows(int dtype, const void* src, int64_t ld_src, int64_t sb_src, void* dst, int64_t ld_dst,
                  int64_t sb_dst, int rows, int batches, int cols, void* stream);
/* dst[b*sb + c] = a[c] + b[c] (cls token + its position embedding) */
int mpx_rows_add(int dtype, const void* a, const void* b, void* dst, int64_t sb, int B, int D, void* stream);
/* dst[b][r][c] = alpha * src[b][c] (mean-pool backward) */
int mpx_bcast_rows(int dtype, const void* src, int64_t ld_src, void* dst, int64_t ld_dst, int64_t sb_dst, int rows,
                   int B, int D, float alpha, void* stream);

/* ---- the reference's generic tensor operators (mpsim.tensors, the `T`
 * namespace of its models: tensors.py:220-555) -------------------------------
 * Each evaluates in f32 and rounds its result once onto the output grid
 * (quantize_array, dtypes.py:100-123); accumulations are the reference's
 * stepwise ones (_stepwise_sum, tensors.py:327-338: re-rounded to the op dtype
 * after every addition, in index order).  Not used by the ViT engine, whose
 * hot ops are the fused kernels above. */
enum {
  MPX_EW_COPY = 0, /* cast / strided copy (T.cast, transpose / reshape materialisation) */
  MPX_EW_ADD = 1, MPX_EW_SUB = 2, MPX_EW_MUL = 3, MPX_EW_DIV = 4, /* tensors.py:255-268 */
  MPX_EW_NEG = 5, MPX_EW_EXP = 6, MPX_EW_LOG = 7, MPX_EW_SQRT = 8, MPX_EW_RELU = 9,
  MPX_EW_GELU = 10,     /* tensors.py:271-292, _gelu_kernel :196-200 */
  MPX_EW_GELU_BWD = 11, /* a = cotangent, b = input: a * quantize(gelu'(b), grad_dtype), autodiff.py:173-185 */
  MPX_EW_RELU_BWD = 12, /* a * (b > 0), autodiff.py:167-170 */
};
enum { MPX_RED_SUM = 0, MPX_RED_MEAN = 1, MPX_RED_MAX = 2 };
/* out (contiguous, `shape`) = op(a, b) with per-operand element strides
 * (0 = broadcast, tensors.py:220-241 numpy broadcasting).  b == NULL for a
 * binary op uses the weak scalar f32(scalar) (tensors.py:235-236), on the
 * left when scalar_side != 0 (rsub / rtruediv). ndim <= 8. */
int mpx_ew(int op, int ndim, const int64_t* h_shape, void* out, int out_dtype, const void* a, int a_dtype,
           const int64_t* h_a_strides, const void* b, int b_dtype, const int64_t* h_b_strides, double scalar,
           int scalar_side, int grad_dtype, void* stream);
/* T.reduce (tensors.py:353-384) over the middle axis of a contiguous
 * (outer, n, inner) view, one sequential stepwise accumulation per output */
int mpx_reduce(int op, const void* a, int dtype, int64_t outer, int64_t n, int64_t inner, void* out, int out_dtype,
               void* stream);
/* _bw_max (autodiff.py:223-230): the cotangent c split equally among ties of
 * the max m; out has a's (outer, n, inner) shape and c's dtype */
int mpx_reduce_max_bwd(const void* a, int dtype, const void* m, const void* c, int c_dtype, int64_t outer, int64_t n,
                       int64_t inner, void* out, void* stream);
/* T.softmax along the middle axis (tensors.py:431-446) and _bw_softmax
 * (autodiff.py:233-240) */
int mpx_softmax_axis(const void* a, int dtype, int64_t outer, int64_t n, int64_t inner, void* out, void* stream);
int mpx_softmax_axis_bwd(const void* y, const void* c, int dtype, int64_t outer, int64_t n, int64_t inner, void* out,
                         void* stream);
/* T.layernorm over the last axis in the promoted dtype (tensors.py:459-491);
 * backward (autodiff.py:243-262): dx, and dgx = c * xhat per element (the
 * caller sums it over the leading axes for dgain, as the reference does) */
int mpx_layernorm_ref(const void* x, int x_dtype, const void* gain, int g_dtype, const void* bias, int b_dtype,
                      int64_t rows, int64_t n, int dtype, void* out, void* stream);
int mpx_layernorm_ref_bwd(const void* x, int x_dtype, const void* gain, int g_dtype, const void* c, int64_t rows,
                          int64_t n, int dtype, void* dx, void* dgx, void* stream);
/* T.cross_entropy (tensors.py:494-522): per-row nll in the logits' dtype
 * (the mean is mpx_reduce MEAN), and _bw_cross_entropy (autodiff.py:265-276)
 * with the 0-d cotangent cot */
int mpx_xent_rows(const void* logits, int dtype, const int32_t* labels, int64_t B, int64_t C, void* nll,
                  void* stream);
int mpx_xent_bwd(const void* logits, int dtype, const int32_t* labels, int64_t B, int64_t C, const void* cot,
                 int cot_dtype, void* out, void* stream);
/* T.matmul (tensors.py:387-422) on CUDA cores for operands the tcgen05 GEMM
 * cannot address (f32, mixed formats, unaligned strides): arbitrary element
 * strides {sam, sak, sbk, sbn, scm, scn}, <= 4 broadcast batch dims; products
 * and partial sums in f32, in k order (bit-exact to the reference for f32) */
int mpx_matmul_simt(const void* a, int a_dtype, const void* b, int b_dtype, void* c, int c_dtype, int64_t M,
                    int64_t N, int64_t K, const int64_t* h_strides, int nbatch_dims, const int64_t* h_bshape,
                    const int64_t* h_sa_b, const int64_t* h_sb_b, const int64_t* h_sc_b, void* stream);

/* ---- data-parallel exchange over NCCL (NVLink / NVSwitch) --------------
 * For hosts that drive this ABI without torch.distributed (the reference has
 * no FFI; these replace the replicated-state agreement of PAPER.md:120-121 in
 * the batch-split DP setup of PAPER.md:282).  libnccl.so.2
 * is dlopen'ed on first use.  A comm is an ncclComm_t: one made here, or the
 * host's own. */
#define MPX_COMM_ID_BYTES 128
int mpx_comm_unique_id(uint8_t* h_id /* [MPX_COMM_ID_BYTES], rank 0 makes it, all ranks share it */);
int mpx_comm_init(void** h_comm, int nranks, const uint8_t* h_id, int rank, int device);
int mpx_comm_destroy(void* comm);
int mpx_comm_size(void* comm, int* h_nranks);
/* *d_flag = MIN over ranks of the u32 finite flag K2 wrote: the AND of every
 * rank's all_finite (tree.py:125-131), so K3 (precision.py:156-173) and the
 * gated K4 (optim.py:100-113) take one skip / back-off decision everywhere.
 * In place, stream-ordered, after K2 and before K3/K4. */
int mpx_allreduce_flag(void* comm, uint32_t* d_flag, void* stream);
/* in-place SUM of a gradient arena (f32 / f16 / bf16) across ranks: the
 * scaled half grads, with 1/W folded into the loss cotangent upstream */
int mpx_allreduce_grads(void* comm, void* d_grads, int64_t numel, int dtype, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MPX_B200_H */

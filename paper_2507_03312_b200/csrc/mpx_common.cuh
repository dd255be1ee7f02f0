// Shared helpers for the mpx_b200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>
#include <utility>

#include "../../include/mpx_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "mpx_b200 kernels target sm_100a only"
#endif

namespace mpx {

// ---------------------------------------------------------------------------
// error plumbing: every C entry point returns an int status and leaves a
// message in a thread-local buffer (mpx_last_error()).
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define MPX_CUDA_CHECK(...)                                                        \
  do {                                                                             \
    cudaError_t _e = (__VA_ARGS__);                                                \
    if (_e != cudaSuccess)                                                         \
      return ::mpx::fail((int)_e, std::string(#__VA_ARGS__) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define MPX_LAUNCH_CHECK(what)                                                     \
  do {                                                                             \
    cudaError_t _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess)                                                         \
      return ::mpx::fail((int)_e, std::string(what) + ": " + cudaGetErrorString(_e)); \
  } while (0)

int current_num_sms();
// cudaFuncAttributeMaxDynamicSharedMemorySize for `fn` on the CURRENT device
// (the attribute is per device: a process driving two GPUs sets it on each),
// remembered per (kernel, device) so the call is cheap on every launch
cudaError_t ensure_smem_attr(const void* fn, int bytes);
// the whole 32-bit word *d_flag = value, stream-ordered
cudaError_t set_flag_word(uint32_t* d_flag, uint32_t value, cudaStream_t st);

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL).  Every kernel starts with
// pdl_grid_sync() (no global memory access before it): launched with
// programmatic stream serialization (launch_pdl) it may be scheduled while its
// predecessor drains, griddepcontrol.wait then blocks until the predecessor
// has completed and its memory is visible, and launch_dependents lets the
// successor be scheduled in turn; launched plainly (launch_k) both are no-ops.
// MPX_PDL=0 turns the attribute off everywhere.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_grid_sync() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// a non-persistent kernel (many waves of blocks) lets its successor launch only
// from its last wave: the successor's CTAs then fill the SMs its tail frees
// instead of taking them from its remaining waves
__device__ __forceinline__ void pdl_wait_only() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();
bool pdl_all();       // MPX_PDL_ALL=1: the plain (launch_k) launches use PDL too
void count_launch();  // every kernel the library launches (mpx_launch_count)
inline void pdl_attr(cudaLaunchAttribute& a) {
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_cfg(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  pdl_attr(attr[0]);
  if (!pdl) attr[0].val.programmaticStreamSerializationAllowed = 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  count_launch();
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
// plain stream-ordered launch (the ViT kernels: measured no gain from PDL
// inside the captured step graph, -0.4 %)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  return launch_cfg(pdl_all(), kern, grid, block, smem, st, std::forward<Args>(args)...);
}
// PDL launch (the MP-step chain K2 -> K4 -> K3: +0.8 %)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  return launch_cfg(true, kern, grid, block, smem, st, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// element conversions.  All rounding is IEEE RNE with subnormals (no FTZ:
// the library is built with -ftz=false -prec-div=true -prec-sqrt=true).
// ---------------------------------------------------------------------------
template <int DT> struct Storage;
template <> struct Storage<MPX_F32>  { using T = float;    };
template <> struct Storage<MPX_F16>  { using T = uint16_t; };
template <> struct Storage<MPX_BF16> { using T = uint16_t; };

template <int DT> __device__ __forceinline__ float to_f32(typename Storage<DT>::T x);
template <> __device__ __forceinline__ float to_f32<MPX_F32>(float x) { return x; }
template <> __device__ __forceinline__ float to_f32<MPX_F16>(uint16_t x) {
  return __half2float(__ushort_as_half(x));
}
template <> __device__ __forceinline__ float to_f32<MPX_BF16>(uint16_t x) {
  return __uint_as_float(((uint32_t)x) << 16);
}

template <int DT> __device__ __forceinline__ typename Storage<DT>::T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<MPX_F32>(float x) { return x; }
template <> __device__ __forceinline__ uint16_t from_f32<MPX_F16>(float x) {
  return __half_as_ushort(__float2half_rn(x));
}
template <> __device__ __forceinline__ uint16_t from_f32<MPX_BF16>(float x) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

// two f32 -> one packed pair (low half = a), RNE: a single cvt.rn.{f16,bf16}x2.f32
// on the ALU pipe instead of two F2F conversions — bit-identical to from_f32
template <int DT> __device__ __forceinline__ uint32_t pack2(float a, float b);
template <> __device__ __forceinline__ uint32_t pack2<MPX_F16>(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
template <> __device__ __forceinline__ uint32_t pack2<MPX_BF16>(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack2_fmt(float a, float b, int bf16) {
  return bf16 ? pack2<MPX_BF16>(a, b) : pack2<MPX_F16>(a, b);
}

// round an f32 onto DT's grid, staying in f32 (quantize_array semantics)
template <int F>
__device__ __forceinline__ float2 unpack2_fmt(uint32_t w) {  // (lo, hi) halves of w, exactly
  if (F) return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
  return __half22float2(*reinterpret_cast<const __half2*>(&w));
}
// acc + the two half values packed in w (lo, hi): the conversion is exact and the
// add rounds once, so this equals unpack-then-FADD bit for bit, in one FHADD each
template <int F>
__device__ __forceinline__ float2 add_h2(float2 acc, uint32_t w) {
  float2 d;
  if (F)
    asm("{.reg .b16 lo, hi; mov.b32 {lo, hi}, %2;\n add.rn.f32.bf16 %0, lo, %3;\n add.rn.f32.bf16 %1, hi, %4;}"
        : "=f"(d.x), "=f"(d.y) : "r"(w), "f"(acc.x), "f"(acc.y));
  else
    asm("{.reg .b16 lo, hi; mov.b32 {lo, hi}, %2;\n add.rn.f32.f16 %0, lo, %3;\n add.rn.f32.f16 %1, hi, %4;}"
        : "=f"(d.x), "=f"(d.y) : "r"(w), "f"(acc.x), "f"(acc.y));
  return d;
}

// (a_lo * b_lo + acc.x, a_hi * b_hi + acc.y) for half pairs a, b: the product of two
// halves is exact in f32 and the add rounds once — the same bits as unpack + FFMA2
template <int F>
__device__ __forceinline__ float2 fma_h2(uint32_t a, uint32_t b, float2 acc) {
  float2 d;
  if (F)
    asm("{.reg .b16 al, ah, bl, bh; mov.b32 {al, ah}, %2; mov.b32 {bl, bh}, %3;\n"
        " fma.rn.f32.bf16 %0, al, bl, %4;\n fma.rn.f32.bf16 %1, ah, bh, %5;}"
        : "=f"(d.x), "=f"(d.y) : "r"(a), "r"(b), "f"(acc.x), "f"(acc.y));
  else
    asm("{.reg .b16 al, ah, bl, bh; mov.b32 {al, ah}, %2; mov.b32 {bl, bh}, %3;\n"
        " fma.rn.f32.f16 %0, al, bl, %4;\n fma.rn.f32.f16 %1, ah, bh, %5;}"
        : "=f"(d.x), "=f"(d.y) : "r"(a), "r"(b), "f"(acc.x), "f"(acc.y));
  return d;
}
template <int DT> __device__ __forceinline__ float quantize_f32(float x) {
  return to_f32<DT>(from_f32<DT>(x));
}

// ---------------------------------------------------------------------------
// 4-wide vector access.  A tile is 256 threads x 2 groups x 4 elements; thread
// t owns elements [4t, 4t+4) and [1024+4t, 1024+4t+4) of its tile, so every
// load/store instruction of a warp covers one contiguous span (fully
// coalesced for 2-byte and 4-byte element types alike).
// ---------------------------------------------------------------------------
constexpr int kThreads = 256;
constexpr int kGroups = 2;
constexpr int kVec = 4;
constexpr int kTile = kThreads * kGroups * kVec;  // 2048 elements
constexpr int kGroupStride = kThreads * kVec;       // 1024 elements

template <int DT> struct Vec4;
template <> struct Vec4<MPX_F32> {
  __device__ __forceinline__ static void load(const void* base, int64_t i, float* o) {
    float4 v = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + i);
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
  __device__ __forceinline__ static void load_cs(const void* base, int64_t i, float* o) {
    float4 v = __ldcs(reinterpret_cast<const float4*>(static_cast<const float*>(base) + i));
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
  }
  __device__ __forceinline__ static void store(void* base, int64_t i, const float* x) {
    *reinterpret_cast<float4*>(static_cast<float*>(base) + i) = make_float4(x[0], x[1], x[2], x[3]);
  }
  __device__ __forceinline__ static void store_cs(void* base, int64_t i, const float* x) {
    __stcs(reinterpret_cast<float4*>(static_cast<float*>(base) + i), make_float4(x[0], x[1], x[2], x[3]));
  }
};

template <int DT> struct Vec4Half {
  __device__ __forceinline__ static void unpack(uint2 w, float* o) {
    o[0] = to_f32<DT>((uint16_t)(w.x & 0xFFFFu));
    o[1] = to_f32<DT>((uint16_t)(w.x >> 16));
    o[2] = to_f32<DT>((uint16_t)(w.y & 0xFFFFu));
    o[3] = to_f32<DT>((uint16_t)(w.y >> 16));
  }
  __device__ __forceinline__ static uint2 pack(const float* x) {
    uint2 w;
    w.x = pack2<DT>(x[0], x[1]);
    w.y = pack2<DT>(x[2], x[3]);
    return w;
  }
  __device__ __forceinline__ static void load(const void* base, int64_t i, float* o) {
    unpack(*reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(base) + i), o);
  }
  __device__ __forceinline__ static void load_cs(const void* base, int64_t i, float* o) {
    unpack(__ldcs(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(base) + i)), o);
  }
  __device__ __forceinline__ static void store(void* base, int64_t i, const float* x) {
    *reinterpret_cast<uint2*>(static_cast<uint16_t*>(base) + i) = pack(x);
  }
  __device__ __forceinline__ static void store_cs(void* base, int64_t i, const float* x) {
    __stcs(reinterpret_cast<uint2*>(static_cast<uint16_t*>(base) + i), pack(x));
  }
};
template <> struct Vec4<MPX_F16> : Vec4Half<MPX_F16> {};
template <> struct Vec4<MPX_BF16> : Vec4Half<MPX_BF16> {};

template <int DT> __device__ __forceinline__ float load1(const void* base, int64_t i) {
  return to_f32<DT>(static_cast<const typename Storage<DT>::T*>(base)[i]);
}
template <int DT> __device__ __forceinline__ void store1(void* base, int64_t i, float x) {
  static_cast<typename Storage<DT>::T*>(base)[i] = from_f32<DT>(x);
}

__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

// ---------------------------------------------------------------------------
// The unscale divisor.  The reference divides by f32(loss_scale)
// (precision.py:151, np.float32(s) at tensors.py:236).  When f32(scale) is a
// normal power of two, x / s == x * (1/s) bit-for-bit (both are one rounding
// of the same exact real), so the kernels multiply; otherwise they divide.
// ---------------------------------------------------------------------------
struct Divisor {
  float s;
  float inv;
  bool pow2;
  __device__ __forceinline__ void init(float sf) {
    s = sf;
    uint32_t b = __float_as_uint(sf);
    uint32_t e = (b >> 23) & 0xFFu;
    pow2 = ((b & 0x807FFFFFu) == 0u) && e >= 1u && e <= 254u;
    inv = pow2 ? __uint_as_float((254u - e) << 23) : 0.f;  // exact 2^-k (subnormal when e == 254)
    if (pow2 && e == 254u) inv = __uint_as_float(0x00400000u);  // 2^-127
  }
  __device__ __forceinline__ float apply(float x) const {
    return pow2 ? __fmul_rn(x, inv) : __fdiv_rn(x, s);
  }
};

__device__ __forceinline__ bool f32_finite(float x) {
  return (__float_as_uint(x) & 0x7F800000u) != 0x7F800000u;
}

}  // namespace mpx

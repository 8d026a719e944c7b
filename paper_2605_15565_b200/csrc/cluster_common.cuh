// Shared pieces of the single-visit cluster loss kernel (policy_loss_sv.cu):
// launch geometry, kernel arguments, packed fp32x2 / fp16 / bf16 helpers, per-vector math.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <type_traits>

#include "loss_common.cuh"
#include "rowstats.cuh"
#include "sm100.cuh"

namespace rl {

constexpr int kNcw = 15;  // consumer warps: 15 + 1 producer = 16 warps = 4 per SMSP -> 128 regs/thread
constexpr int kCons = kNcw * 32;              // consumer threads (one 16-B vector each per chunk)
constexpr int kChunkVec = kCons;              // vectors per chunk
constexpr int kChunkBytes = kChunkVec * 16;   // 7.5 KB
constexpr int kClThreads = kCons + 32;        // + producer warp
constexpr int kSmemMax = 232448;              // 227 KB opt-in per CTA on sm_100

// fp16 cache of e' = 2^(x k - m + kCacheShift) in (0, 2^15]: the shift keeps the bulk of a
// peaked row (e ~ 1e-7 .. 1e-9) out of the fp16 subnormal range (abs. precision 2^-39 instead
// of 2^-24), so the cached probabilities lose no mass; 2^-15 is folded into the pass-C scale.
constexpr float kCacheShift = 15.f;

struct ClArgs {
  const void* logits;
  void* dlogits;
  int64_t n_tokens, V, ld, nvec;
  int64_t h_vec;  // vectors per CTA slice
  const int32_t* targets;
  const float* old_logp;
  const uint8_t* mask;
  const int32_t* token_seq;
  const float* seq_adv;
  const int32_t* seq_version;
  const int32_t* seq_active;
  float* logp_out;
  uint8_t* clipped_out;
  double* partials;
  Knobs kn;
  int32_t nslots;
  uint8_t* redo;            // SV kernel: per-row flag, 1 = row left to the two-pass fixup
};

// ------------------------------------------------------------------ packed fp32x2 helpers
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint32_t cvt_h2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint64_t h2_to_f2(uint32_t h) {
  float lo, hi;
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\tcvt.f32.f16 %0, l;\n\tcvt.f32.f16 %1, h;\n\t}"
      : "=f"(lo), "=f"(hi)
      : "r"(h));
  return f2pack(lo, hi);
}
__device__ __forceinline__ uint32_t f2_to_bf2(uint64_t v) {
  float lo, hi;
  f2unpack(v, lo, hi);
  return pack_bf16x2(lo, hi);
}

// ------------------------------------------------------------------ per-vector kernels
template <typename T>
struct ClVec;

template <>
struct ClVec<bf16_t> {
  static constexpr int EPV = 8;
  using MaxT = __nv_bfloat162;
  __device__ static __forceinline__ MaxT max_init() { return __bfloat162bfloat162(__ushort_as_bfloat16(0xff80)); }
  // pass A: running packed max
  __device__ static __forceinline__ void max_acc(const uint4& v, MaxT& m) {
    const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&v);
    m = __hmax2(m, __hmax2(__hmax2(p[0], p[1]), __hmax2(p[2], p[3])));
  }
  __device__ static __forceinline__ float max_to_float(MaxT m) { return fmaxf(__low2float(m), __high2float(m)); }
  __device__ static __forceinline__ uint4 neg_inf_vec() { return make_uint4(0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u); }
  // pass B: e' = 2^(x k + mneg); accumulates packed partial sums, fills the fp16 cache words
  __device__ static __forceinline__ uint64_t exp_cache(const uint4& v, uint64_t k2, uint64_t mn2, uint64_t acc,
                                                       uint4& c) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t t = ffma2(f2pack(bf16_lo(w[i]), bf16_hi(w[i])), k2, mn2);
      float a, b;
      f2unpack(t, a, b);
      a = fast_exp2(a);
      b = fast_exp2(b);
      acc = fadd2(acc, f2pack(a, b));
      o[i] = cvt_h2(a, b);
    }
    c = make_uint4(o[0], o[1], o[2], o[3]);
    return acc;
  }
  // pass C: q * e' -> bf16
  __device__ static __forceinline__ uint4 grad(const uint4& c, uint64_t q2) {
    return make_uint4(f2_to_bf2(fmul2(h2_to_f2(c.x), q2)), f2_to_bf2(fmul2(h2_to_f2(c.y), q2)),
                      f2_to_bf2(fmul2(h2_to_f2(c.z), q2)), f2_to_bf2(fmul2(h2_to_f2(c.w), q2)));
  }
  // bf16-cache variant: e' cached as bf16 (F2FP.BF16), pass C is one packed bf16 multiply
  // (HMUL2.BF16) per pair: 4 instructions per vector instead of 16, at the cost of two extra
  // bf16 roundings (e' and q): <= ~0.6 % relative per element (reading Z21)
  __device__ static __forceinline__ uint64_t exp_cache_bf(const uint4& v, uint64_t k2, uint64_t mn2, uint64_t acc,
                                                          uint4& c) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t t = ffma2(f2pack(bf16_lo(w[i]), bf16_hi(w[i])), k2, mn2);
      float a, b;
      f2unpack(t, a, b);
      a = fast_exp2(a);
      b = fast_exp2(b);
      acc = fadd2(acc, f2pack(a, b));
      o[i] = pack_bf16x2(a, b);
    }
    c = make_uint4(o[0], o[1], o[2], o[3]);
    return acc;
  }
  // read-only sum of 2^(x k + c) (logprob_warp_kernel)
  __device__ static __forceinline__ uint64_t exp_sum(const uint4& v, uint64_t k2, uint64_t c2, uint64_t acc) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float a, b;
      f2unpack(ffma2(f2pack(bf16_lo(w[i]), bf16_hi(w[i])), k2, c2), a, b);
      acc = fadd2(acc, f2pack(fast_exp2(a), fast_exp2(b)));
    }
    return acc;
  }
  // single-visit kernel (policy_loss_sv.cu): bf16 cache of e' = 2^(x k - R + 15), R = target
  __device__ static __forceinline__ uint64_t exp_sv(const uint4& v, uint64_t k2, uint64_t mn2, uint64_t acc, uint4& c) {
    return exp_cache_bf(v, k2, mn2, acc, c);
  }
  // dlogits = q e' with ONE rounding in the product: q is split into bf16 q_hi + q_lo (q_lo =
  // bf16(q - q_hi), so q_hi + q_lo = q (1 + O(u^2))); t = e' q_lo (HMUL2, a tiny term), then
  // d = fma(e', q_hi, t) rounded once (HFMA2).  With the e' cache that is two bf16 roundings per
  // element (<= 2u + O(u^2) = 0.78 % relative, u = 2^-8): reading R2 / Z21 by construction.
  __device__ static __forceinline__ uint4 grad_sv(const uint4& c, uint32_t qhi2, uint32_t qlo2, float) {
    const __nv_bfloat162 qh = *reinterpret_cast<const __nv_bfloat162*>(&qhi2);
    const __nv_bfloat162 ql = *reinterpret_cast<const __nv_bfloat162*>(&qlo2);
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 e = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
      const __nv_bfloat162 r = __hfma2(e, qh, __hmul2(e, ql));
      o[i] = *reinterpret_cast<const uint32_t*>(&r);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
  }
  // exp_sv + the entropy moment accx += e' * x (fp32 pairs)
  __device__ static __forceinline__ uint64_t exp_sv_ent(const uint4& v, uint64_t k2, uint64_t mn2, uint64_t acc,
                                                        uint64_t& accx, uint4& c) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t x2 = f2pack(bf16_lo(w[i]), bf16_hi(w[i]));
      float a, b;
      f2unpack(ffma2(x2, k2, mn2), a, b);
      a = fast_exp2(a);
      b = fast_exp2(b);
      const uint64_t e2 = f2pack(a, b);
      acc = fadd2(acc, e2);
      accx = ffma2(e2, x2, accx);
      o[i] = pack_bf16x2(a, b);
    }
    c = make_uint4(o[0], o[1], o[2], o[3]);
    return acc;
  }
  __device__ static __forceinline__ uint4 grad_bf(const uint4& c, uint32_t qb2) {
    const __nv_bfloat162 q = *reinterpret_cast<const __nv_bfloat162*>(&qb2);
    uint4 o;
    __nv_bfloat162 r;
    r = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&c.x), q); o.x = *reinterpret_cast<uint32_t*>(&r);
    r = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&c.y), q); o.y = *reinterpret_cast<uint32_t*>(&r);
    r = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&c.z), q); o.z = *reinterpret_cast<uint32_t*>(&r);
    r = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&c.w), q); o.w = *reinterpret_cast<uint32_t*>(&r);
    return o;
  }
};

template <>
struct ClVec<float> {
  static constexpr int EPV = 4;
  using MaxT = float;
  __device__ static __forceinline__ MaxT max_init() { return -INFINITY; }
  __device__ static __forceinline__ void max_acc(const uint4& v, MaxT& m) {
    m = fmaxf(fmaxf(m, fmaxf(__uint_as_float(v.x), __uint_as_float(v.y))),
              fmaxf(__uint_as_float(v.z), __uint_as_float(v.w)));
  }
  __device__ static __forceinline__ float max_to_float(MaxT m) { return m; }
  __device__ static __forceinline__ uint4 neg_inf_vec() { return make_uint4(0xff800000u, 0xff800000u, 0xff800000u, 0xff800000u); }
  __device__ static __forceinline__ uint64_t exp_cache(const uint4& v, uint64_t k2, uint64_t mn2, uint64_t acc,
                                                       uint4& c) {
    uint32_t o[2];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const uint64_t t = ffma2(f2pack(__uint_as_float(w[2 * i]), __uint_as_float(w[2 * i + 1])), k2, mn2);
      float a, b;
      f2unpack(t, a, b);
      a = fast_exp2(a);
      b = fast_exp2(b);
      acc = fadd2(acc, f2pack(a, b));
      o[i] = cvt_h2(a, b);
    }
    c.x = o[0];
    c.y = o[1];
    return acc;
  }
  __device__ static __forceinline__ uint64_t exp_sum(const uint4& v, uint64_t k2, uint64_t c2, uint64_t acc) {
    float a, b, d, e;
    f2unpack(ffma2(f2pack(__uint_as_float(v.x), __uint_as_float(v.y)), k2, c2), a, b);
    f2unpack(ffma2(f2pack(__uint_as_float(v.z), __uint_as_float(v.w)), k2, c2), d, e);
    acc = fadd2(acc, f2pack(fast_exp2(a), fast_exp2(b)));
    return fadd2(acc, f2pack(fast_exp2(d), fast_exp2(e)));
  }
  // single-visit kernel: fp32 cache (e' may exceed the fp16 range once R is not the max)
  __device__ static __forceinline__ uint64_t exp_sv(const uint4& v, uint64_t k2, uint64_t mn2, uint64_t acc, uint4& c) {
    const uint64_t t0 = ffma2(f2pack(__uint_as_float(v.x), __uint_as_float(v.y)), k2, mn2);
    const uint64_t t1 = ffma2(f2pack(__uint_as_float(v.z), __uint_as_float(v.w)), k2, mn2);
    float a, b, d, e;
    f2unpack(t0, a, b);
    f2unpack(t1, d, e);
    a = fast_exp2(a);
    b = fast_exp2(b);
    d = fast_exp2(d);
    e = fast_exp2(e);
    acc = fadd2(acc, f2pack(a, b));
    acc = fadd2(acc, f2pack(d, e));
    c = make_uint4(__float_as_uint(a), __float_as_uint(b), __float_as_uint(d), __float_as_uint(e));
    return acc;
  }
  __device__ static __forceinline__ uint64_t exp_sv_ent(const uint4& v, uint64_t k2, uint64_t mn2, uint64_t acc,
                                                        uint64_t& accx, uint4& c) {
    const uint64_t x0 = f2pack(__uint_as_float(v.x), __uint_as_float(v.y));
    const uint64_t x1 = f2pack(__uint_as_float(v.z), __uint_as_float(v.w));
    float a, b, d, e;
    f2unpack(ffma2(x0, k2, mn2), a, b);
    f2unpack(ffma2(x1, k2, mn2), d, e);
    const uint64_t e0 = f2pack(fast_exp2(a), fast_exp2(b)), e1 = f2pack(fast_exp2(d), fast_exp2(e));
    acc = fadd2(fadd2(acc, e0), e1);
    accx = ffma2(e1, x1, ffma2(e0, x0, accx));
    float p, q, r, t;
    f2unpack(e0, p, q);
    f2unpack(e1, r, t);
    c = make_uint4(__float_as_uint(p), __float_as_uint(q), __float_as_uint(r), __float_as_uint(t));
    return acc;
  }
  __device__ static __forceinline__ uint4 grad_sv(const uint4& c, uint32_t, uint32_t, float q) {
    const uint64_t q2 = f2pack(q, q);
    float a, b, d, e;
    f2unpack(fmul2(f2pack(__uint_as_float(c.x), __uint_as_float(c.y)), q2), a, b);
    f2unpack(fmul2(f2pack(__uint_as_float(c.z), __uint_as_float(c.w)), q2), d, e);
    return make_uint4(__float_as_uint(a), __float_as_uint(b), __float_as_uint(d), __float_as_uint(e));
  }
  __device__ static __forceinline__ uint4 grad(const uint4& c, uint64_t q2) {
    float a, b, d, e;
    f2unpack(fmul2(h2_to_f2(c.x), q2), a, b);
    f2unpack(fmul2(h2_to_f2(c.y), q2), d, e);
    return make_uint4(__float_as_uint(a), __float_as_uint(b), __float_as_uint(d), __float_as_uint(e));
  }
};

// Compile-time loop: f(integral_constant<int, i>) for i in [B, E) — register-array indices and
// phase boundaries stay static in the fully unrolled row loops.
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// Ring position of the first chunk of a row (slot index + phase parity), advanced per row.
struct RingPos {
  uint32_t slot, phase;
  __device__ __forceinline__ void advance(int n, int nslots) {
    slot += n;
    while (slot >= (uint32_t)nslots) {
      slot -= nslots;
      phase ^= 1u;
    }
  }
};

}  // namespace rl

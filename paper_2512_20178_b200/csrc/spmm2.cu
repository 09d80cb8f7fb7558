// spmm2.cu -- software-pipelined CSR SpMM (K1/K2/K3/K6 of DESIGN.md), an
// opt-in variant (SHIRO_KERNEL=2,3,5..9) for N in {32, 64, 128}.  MEASURED
// SLOWER than k_spmm with one-warp CTAs (profiles/r1_kernel_sweep.txt): the
// deeper per-warp pipeline costs registers, and more resident warps beat
// deeper pipelines for this gather.  Kept as documented evidence.
//
// Same work decomposition and result as k_spmm (kernels.cu): a lane group of
// LPR = N/4 lanes owns a work unit (a row group of short rows, or one chunk of
// a hub row), every nonzero a_ij of the unit is a length-N axpy of source row
// j into output row i, accumulated in fp32 registers in
// CSR order.  What changes is the instruction stream, which ncu showed to be
// the limiter of k_spmm (~50 warp instructions per nonzero, 60 % issue-active,
// 180 B of register spills, PAPER-independent):
//   * the source-row address is one IMAD.WIDE (N is a template constant);
//   * row boundaries inside a batch of LPR nonzeros are one ballot per batch
//     (a bitmask), not a shuffle + compare per nonzero; the row offset is only
//     read at a boundary;
//   * gathers are software pipelined in stages of U nonzeros over two
//     register buffers: stage s+1 is in flight while stage s is consumed, and
//     the next batch's (col, val) pairs are prefetched one batch ahead, so
//     loads stay in flight across row and batch boundaries;
//   * weights are broadcast at consume time (no weight registers), loop
//     counters are 32-bit offsets inside the unit.
// Hub chunks keep k_spmm's deterministic last-arriver reduction in chunk order.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace shiro {

namespace {

constexpr int kB2 = 256;

__device__ __forceinline__ int2 ldcv(const int2 *p) {
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ int ldro(const uint8_t *p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return (int)v;
}
__device__ __forceinline__ void fma4(float4 &acc, float v, const float4 &x) {
  acc.x = fmaf(v, x.x, acc.x);
  acc.y = fmaf(v, x.y, acc.y);
  acc.z = fmaf(v, x.z, acc.z);
  acc.w = fmaf(v, x.w, acc.w);
}
__device__ __forceinline__ void add4(float4 &acc, const float4 &x) {
  acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
}

// Source row c of the unified source space [X0 || X1], already offset by the
// lane's float4 (base0/base1 = X + li).
template <int LPR, bool TWO>
__device__ __forceinline__ const float4 *srow(const float4 *base0, const float4 *base1, int n0, int c) {
  if (TWO && c >= n0) return base1 + (int64_t)(c - n0) * LPR;
  return base0 + (int64_t)c * LPR;
}

// One unit's nonzero stream [0, n) (cvp/rop already offset to the unit).
// GROUP: nonzeros carry a row offset (row group); row ends call flush(t)
// = "finish rows until the current row is t".  !GROUP: one row (hub chunk).
template <int LPR, int U, bool TWO, bool GROUP, class Flush>
__device__ __forceinline__ void stream(const int2 *cvp, const uint8_t *rop, const int n,
                                       const float4 *b0, const float4 *b1, const int n0,
                                       const int li, const unsigned mask, const int shift,
                                       float4 &acc, Flush &&flush) {
  constexpr int S = LPR / U;          // stages per batch (even)
  static_assert(S >= 2 && S % 2 == 0, "stages per batch must be even");
  if (n <= 0) return;
  const int nb = (n + LPR - 1) / LPR;
  int2 cvc = make_int2(0, 0), cvn = make_int2(0, 0);
  int roc = 0, ron = 0;
  if (li < n) {
    cvc = ldcv(cvp + li);
    if (GROUP) roc = ldro(rop + li);
  }
  if (nb > 1 && LPR + li < n) {
    cvn = ldcv(cvp + LPR + li);
    if (GROUP) ron = ldro(rop + LPR + li);
  }
  // boundary mask of the current batch: bit j <=> nonzero j starts a new row
  auto boundaries = [&](int ro, int prev, int cnt) -> unsigned {
    if (!GROUP) return 0u;
    int up = __shfl_up_sync(mask, ro, 1, LPR);
    if (li == 0) up = prev;
    const unsigned bal = __ballot_sync(mask, li < cnt && ro != up);
    return (LPR == 32) ? bal : ((bal >> shift) & ((1u << LPR) - 1u));
  };
  int cnt = n < LPR ? n : LPR;
  unsigned bmc = boundaries(roc, 0, cnt);

  float4 xa[U], xb[U];
  auto issue = [&](float4 (&x)[U], const int2 &cv, int j0, int c) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int col = __shfl_sync(mask, cv.x, j0 + u, LPR);
      if (j0 + u < c) x[u] = __ldg(srow<LPR, TWO>(b0, b1, n0, col));
    }
  };
  auto consume = [&](const float4 (&x)[U], int j0, int c) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u;
      const float w = __int_as_float(__shfl_sync(mask, cvc.y, j, LPR));
      if (GROUP && ((bmc >> j) & 1u)) flush(__shfl_sync(mask, roc, j, LPR));
      if (j < c) fma4(acc, w, x[u]);
    }
  };

  issue(xa, cvc, 0, cnt);
  for (int b = 0; b < nb; ++b) {
    const int cntn = (b + 1 < nb) ? ((n - (b + 1) * LPR) < LPR ? n - (b + 1) * LPR : LPR) : 0;
    // two stages per trip, not unrolled: keeps exactly two stages in flight
    // (an unrolled batch lets the scheduler hoist every gather and spill)
#pragma unroll 1
    for (int s = 0; s < S; s += 2) {
      if ((s + 1) * U < cnt) issue(xb, cvc, (s + 1) * U, cnt);
      if (s * U < cnt) consume(xa, s * U, cnt);
      if (s + 2 < S) {
        if ((s + 2) * U < cnt) issue(xa, cvc, (s + 2) * U, cnt);
      } else if (cntn > 0) {
        issue(xa, cvn, 0, cntn);
      }
      if ((s + 1) * U < cnt) consume(xb, (s + 1) * U, cnt);
    }
    if (cntn > 0) {
      const int last = __shfl_sync(mask, roc, LPR - 1, LPR);
      cvc = cvn;
      roc = ron;
      bmc = boundaries(roc, last, cntn);
      cnt = cntn;
      if (b + 2 < nb) {
        const int k = (b + 2) * LPR + li;
        if (k < n) {
          cvn = ldcv(cvp + k);
          if (GROUP) ron = ldro(rop + k);
        }
      }
    }
  }
}

// Deterministic reduction of a hub row's chunk partials (fixed chunk order),
// by the last-arriving chunk.  Kept out of line: rare, register hungry.
template <int LPR, bool ACCUM, bool OUTP>
__device__ __forceinline__ void hub_reduce(const SpmmArgs &a, int f, int nch, int64_t t, int li) {
  constexpr int N4 = LPR;   // float4 per row
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4 *sp = reinterpret_cast<const float4 *>(a.scratch) + (int64_t)f * N4 + li;
  int c = 0;
  for (; c + 4 <= nch; c += 4) {
    float4 p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) p[i] = __ldcg(sp + (int64_t)(c + i) * N4);
#pragma unroll
    for (int i = 0; i < 4; ++i) add4(s, p[i]);
  }
  for (; c < nch; ++c) add4(s, __ldcg(sp + (int64_t)c * N4));
  float4 *y;
  if (OUTP) {
    const long long v = (long long)a.out_ptr[t];
    y = (v < 0) ? reinterpret_cast<float4 *>(a.Y + (v & 0x7fffffffffffffffLL) * a.N)
                : reinterpret_cast<float4 *>(v);
  } else {
    const int64_t orow = a.out_row ? a.out_row[t] : t;
    y = reinterpret_cast<float4 *>(a.Y) + orow * N4;
  }
  if (ACCUM) add4(s, y[li]);
  y[li] = s;
}

template <int LPR, int U, bool ACCUM, bool TWO, bool OUTP, int MINB, int BS>
__global__ void __launch_bounds__(BS, MINB) k_spmm2(const SpmmArgs a) {
  constexpr int R = 32 / LPR;
  constexpr int N4 = LPR;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR;
  const int li = lane % LPR;
  const int shift = sub * LPR;
  const unsigned mask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << shift);
  const int64_t u = (((int64_t)blockIdx.x * BS + threadIdx.x) >> 5) * R + sub;
  const float4 *b0 = reinterpret_cast<const float4 *>(a.X0) + li;
  const float4 *b1 = TWO ? reinterpret_cast<const float4 *>(a.X1) + li : b0;
  const int n0 = TWO ? (int)a.n0 : 0;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);

  if (u < a.n_tasks) {
    // ---- one chunk of a hub row ---------------------------------------------
    const int lr = a.task_long[u];
    const int64_t t = a.long_row[lr];
    const int f = a.long_first[lr], nch = a.long_first[lr + 1] - f;
    const int64_t rb = __ldg(a.rp + t), re = __ldg(a.rp + t + 1);
    const int64_t clen = (re - rb + nch - 1) / nch;
    const int64_t kb = rb + (int64_t)(u - f) * clen;
    const int64_t ke = (kb + clen < re) ? kb + clen : re;
    stream<LPR, U, TWO, false>(a.cv + kb, nullptr, (int)(ke - kb), b0, b1, n0, li, mask, shift, acc,
                               [](int) {});
    float4 *sp = reinterpret_cast<float4 *>(a.scratch) + u * N4 + li;
    __stcg(sp, acc);
    __threadfence();
    __syncwarp(mask);
    int last = 0;
    if (li == 0) last = (atomicAdd(a.long_counter + lr, 1) == nch - 1);
    last = __shfl_sync(mask, last, 0, LPR);
    if (last) {
      __threadfence();
      hub_reduce<LPR, ACCUM, OUTP>(a, f, nch, t, li);
      if (li == 0) a.long_counter[lr] = 0;   // re-arm for the next launch
    }
    return;
  }

  // ---- row group: rows [r0, r1), nonzeros [k0, k1) ----------------------------
  const int64_t gi = u - a.n_tasks;
  if (gi >= a.n_groups) return;
  const RowGroup g = a.groups[gi];
  const int nrows = g.r1 - g.r0;
  int orw0 = 0, orw1 = 0;
  long long opw0 = 0, opw1 = 0;
  if (OUTP) {
    if (li < nrows) opw0 = (long long)a.out_ptr[g.r0 + li];
    if (LPR + li < nrows) opw1 = (long long)a.out_ptr[g.r0 + LPR + li];
  } else if (a.out_row) {
    if (li < nrows) orw0 = __ldg(a.out_row + g.r0 + li);
    if (LPR + li < nrows) orw1 = __ldg(a.out_row + g.r0 + LPR + li);
  }
  int cur = 0;
  auto flush1 = [&]() {
    float4 *y;
    if (OUTP) {
      const long long v = __shfl_sync(mask, (cur < LPR) ? opw0 : opw1, cur & (LPR - 1), LPR);
      y = (v < 0) ? reinterpret_cast<float4 *>(a.Y) + (v & 0x7fffffffffffffffLL) * N4 + li
                  : reinterpret_cast<float4 *>(v) + li;
    } else {
      int64_t orow;
      if (a.out_row) orow = __shfl_sync(mask, (cur < LPR) ? orw0 : orw1, cur & (LPR - 1), LPR);
      else orow = g.r0 + cur;
      y = reinterpret_cast<float4 *>(a.Y) + orow * N4 + li;
    }
    if (ACCUM) add4(acc, *y);
    *y = acc;
    acc = make_float4(0.f, 0.f, 0.f, 0.f);
    ++cur;
  };
  stream<LPR, U, TWO, true>(a.cv + g.k0, a.roff + g.k0, (int)(g.k1 - g.k0), b0, b1, n0, li, mask,
                            shift, acc, [&](int t) {
                              while (cur < t) flush1();
                            });
  while (cur < nrows) flush1();   // last row and trailing empty rows
}

template <int LPR, int U, int MINB, int BS = kB2>
void launch2(const SpmmArgs &a, bool acc, cudaStream_t s) {
  const int64_t units = a.n_tasks + a.n_groups;
  const int64_t per_block = (int64_t)(BS / 32) * (32 / LPR);
  const unsigned grid = (unsigned)((units + per_block - 1) / per_block);
  const bool two = a.X1 != nullptr;
  if (a.out_ptr) {
    k_spmm2<LPR, U, false, false, true, MINB, BS><<<grid, BS, 0, s>>>(a);
  } else if (acc) {
    if (two) k_spmm2<LPR, U, true, true, false, MINB, BS><<<grid, BS, 0, s>>>(a);
    else k_spmm2<LPR, U, true, false, false, MINB, BS><<<grid, BS, 0, s>>>(a);
  } else {
    if (two) k_spmm2<LPR, U, false, true, false, MINB, BS><<<grid, BS, 0, s>>>(a);
    else k_spmm2<LPR, U, false, false, false, MINB, BS><<<grid, BS, 0, s>>>(a);
  }
}

int kernel_choice() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("SHIRO_KERNEL");
    v = e ? atoi(e) : 0;
  }
  return v;
}

}  // namespace

// returns 1 if launched, 0 if the shape has no pipelined kernel (caller uses k_spmm)
int launch_spmm2(const SpmmArgs &a, bool accumulate, cudaStream_t s) {
  // opt-in (SHIRO_KERNEL=2,3,5..9): measured slower than k_spmm with one-warp
  // CTAs (profiles/r1_kernel_sweep.txt)
  const int kc = kernel_choice();
  if (kc < 2 || kc == 4 || kc >= 10 || a.sig_ptrs || a.wait_flags) return 0;   // no in-kernel flags
  const int var = kernel_choice();
  switch (a.N) {
    case 128:
#ifdef SHIRO_KERNEL_SWEEP
      switch (var) {   // (U, MINB, CTA size) variants of the sweeps
        case 3: launch2<32, 4, 3>(a, accumulate, s); return 1;
        case 5: launch2<32, 2, 6>(a, accumulate, s); return 1;
        case 6: launch2<32, 2, 20, 64>(a, accumulate, s); return 1;
        case 7: launch2<32, 4, 16, 64>(a, accumulate, s); return 1;
        case 8: launch2<32, 4, 24, 32>(a, accumulate, s); return 1;
        case 9: launch2<32, 2, 32, 32>(a, accumulate, s); return 1;
        default: break;
      }
#endif
      launch2<32, 4, 4>(a, accumulate, s);
      return 1;
    case 64: launch2<16, 4, 4>(a, accumulate, s); return 1;
    case 32: launch2<8, 4, 4>(a, accumulate, s); return 1;
    default: return 0;
  }
  (void)var;
}

}  // namespace shiro

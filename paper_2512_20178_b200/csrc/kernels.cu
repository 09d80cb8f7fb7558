// kernels.cu -- hand-written sm_100a kernels of the SHIRO hot path.
//
// The dense width N of B and C is the contraction-free axis of SpMM: every
// nonzero a_ij contributes a length-N axpy of row j of the source into row i
// of the output.  The work is a memory-bound gather, so
// the kernels are designed around L2 / HBM3e traffic, not tensor cores:
//   * a source row is N*4 bytes (512 B at N = 128); a group of
//     LPR = min(32, N/4) lanes owns one output row and moves each source row
//     with one 128-bit load per lane (fully coalesced LDG.128);
//   * the nonzeros of a work unit are loaded cooperatively as interleaved
//     (col, val) pairs, one 8-byte streaming load per lane, and broadcast with
//     shuffles; U = 8 independent row gathers are issued before any FMA
//     (the value of each is shuffled at its FMA, holding no register);
//   * short rows are packed at plan time into row groups (<= L nonzeros,
//     <= 64 rows); a per-nonzero byte gives the row offset inside the group,
//     so row boundaries cost no memory access and the gathers of many short
//     rows stay in flight together; empty rows are written as zeros;
//   * rows longer than L nonzeros (power-law hubs) become chunk tasks of L
//     nonzeros scheduled first; their partials are reduced in chunk order by
//     the last-arriving chunk (threadfence + arrival counter): deterministic,
//     single launch;
//   * fp32 accumulation in registers, one store per output row;
//   * one-warp CTAs, 32 resident per SM (measured best).
// L2 policy per launch (HINT): 0 default; 1 = the streams evict_first, the
// gathers default; 4 = as 3 with the compact hot buffer (X1) as the hot
// rows; 2 = source rows fit in L2 -> the
// streams (A's (col, val) pairs, C rows) evict_first, gathered rows
// evict_last; 3 = source rows far larger than L2 -> the plan-time "hot" rows
// (bit 31 of the column id) evict_last, every other gather and the streams
// evict_first.  WAIT: per-unit, per-source READY wait of the fused exchange
// consumer with L2-coherent source loads (SpmmArgs::ready).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "kernels.h"

namespace shiro {

namespace {

constexpr int kBlock = 256;   // CTA size of the pack / scatter / generic kernels

__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
template <int HINT>
__device__ __forceinline__ int2 ldcv_h(const int2 *p) {
  int2 v;
  if (HINT == 0) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0, %1}, [%2];"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(p), "l"(pol_first()));
  }
  return v;
}
// Per-lane vector of the SpMM: W floats (float, float2, float4).  N = 32 and
// 64 run one 32-lane group per warp with float / float2 lanes (no divergent
// lane groups inside a warp); N = 128 float4; N = 256 / 512 several float4.
template <int W> struct VT;
template <> struct VT<1> {
  using T = float;
  static __device__ __forceinline__ T zero() { return 0.f; }
};
template <> struct VT<2> {
  using T = float2;
  static __device__ __forceinline__ T zero() { return make_float2(0.f, 0.f); }
};
template <> struct VT<4> {
  using T = float4;
  static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
};

__device__ __forceinline__ void fma4(float &acc, float v, const float &x) { acc = fmaf(v, x, acc); }
__device__ __forceinline__ void fma4(float2 &acc, float v, const float2 &x) {
  acc.x = fmaf(v, x.x, acc.x);
  acc.y = fmaf(v, x.y, acc.y);
}
__device__ __forceinline__ void add4(float &acc, const float &x) { acc += x; }
__device__ __forceinline__ void add4(float2 &acc, const float2 &x) { acc.x += x.x; acc.y += x.y; }

// raw loads / stores of one per-lane vector with an optional L2 policy
__device__ __forceinline__ float ld_weak(const float *p) {
  float v;
  asm volatile("ld.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float2 ld_weak(const float2 *p) {
  float2 v;
  asm volatile("ld.global.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float4 ld_weak(const float4 *p) {
  float4 v;
  asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ float ld_pol(const float *p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float2 ld_pol(const float2 *p, uint64_t pol) {
  float2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
               : "=f"(v.x), "=f"(v.y)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ld_pol(const float4 *p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_pol(float *p, const float &v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_pol(float2 *p, const float2 &v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_pol(float4 *p, const float4 &v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}

// gathered source row: HINT 0 and 1 plain LDG (1 only marks the streams --
// column/value words, row offsets, output rows -- evict_first); 2 evict_last;
// 4 evict_last for the compact hot buffer (X1), evict_first otherwise; 3 evict_last for hot
// rows, evict_first otherwise; COH (and coh for this row): a weak
// (coherent-path, L1-cacheable) load instead of the read-only ld.global.nc:
// peers store into other parts of the buffer during the launch, and these
// rows are only read after this lane group's ld.acquire.sys of their READY
// flag (memory-model ordered, unlike the non-coherent path)
template <int HINT, bool COH, typename V>
__device__ __forceinline__ V ldB(const V *p, bool hot, bool coh) {
  if (COH && coh) return ld_weak(p);
  if (HINT <= 1) return __ldg(p);
  // the policy operand lives in a uniform register: one load per constant
  // policy (a per-row select would make the compiler waterfall over lanes);
  // `hot` is uniform across the lane group, so this branch never diverges
  if (HINT == 2 || hot) return ld_pol(p, pol_last());
  return ld_pol(p, pol_first());
}
template <int HINT, typename V>
__device__ __forceinline__ void stY_h(V *p, const V &v) {
  if (HINT == 0) { *p = v; return; }
  st_pol(p, v, pol_first());
}

__device__ __forceinline__ int ld_stream_u8(const uint8_t *p) {
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

// Source row in the unified row space [X0 || X1] (X1 unused when n0 covers all).
// (one IMAD.WIDE.U32 per row: column ids and N are non-negative 32-bit)
template <bool TWO>
__device__ __forceinline__ const float *src_row_ptr(const SpmmArgs &a, int c) {
  const uint32_t rowb = (uint32_t)a.N * 4u;
  if (TWO) {
    // branch-free: one select of the base, X1's rows addressed as
    // (X1 - n0 rows) + c rows (a per-gather branch cost 1.5x the instructions)
    const uint64_t b1 = reinterpret_cast<uint64_t>(a.X1) - (uint64_t)a.n0 * rowb;
    const uint64_t base = (c >= a.n0) ? b1 : reinterpret_cast<uint64_t>(a.X0);
    return reinterpret_cast<const float *>(base + (uint64_t)(uint32_t)c * rowb);
  }
  return reinterpret_cast<const float *>(reinterpret_cast<uint64_t>(a.X0) +
                                         (uint64_t)(uint32_t)c * rowb);
}
template <bool TWO, typename V>
__device__ __forceinline__ const V *src_row(const SpmmArgs &a, int c) {
  return reinterpret_cast<const V *>(src_row_ptr<TWO>(a, c));
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Per-source READY wait of one lane group (SpmmArgs::ready): bit s of `need`
// set -> wait until ready[s] >= target.  Lane li of the group polls sources
// li, li + lanes, ... (P <= 64).  Gives up at its own timeout or as soon as
// another warp has raised *err (one timeout in total, however many waves the
// grid has).
__device__ __noinline__ bool wait_sources(const int32_t *ready, uint64_t need, int32_t target,
                                          int32_t *err, int64_t timeout_ns, int li, int lanes,
                                          unsigned mask) {
  const uint64_t t0 = gtimer();
  for (;;) {
    bool ok = true;
    for (int s = li; s < 64; s += lanes) {
      if ((need >> s) & 1ull) {
        int32_t v;
        asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(ready + s) : "memory");
        ok = ok && v >= target;
      }
    }
    if (__all_sync(mask, ok)) break;
    if (*reinterpret_cast<volatile int32_t *>(err)) return false;
    if ((int64_t)(gtimer() - t0) > timeout_ns) {
      if (li == 0) atomicExch(err, 1);
      return false;
    }
    __nanosleep(128);
  }
  __syncwarp(mask);   // order every lane's source loads after the acquiring lanes
  return true;
}

// L2 prefetch of the source row of this lane's nonzero (PF): every lane of a
// batch requests its whole row (N*4 bytes = N/32 lines of 128 B) before the
// lane group gathers the batch U rows at a time, so up to LPR rows per lane
// group are in flight at the L2/DRAM level while only U are held in
// registers.  No registers are tied up by a prefetch.
template <bool TWO>
__device__ __forceinline__ void prefetch_row(const SpmmArgs &a, int c) {
  const char *r = reinterpret_cast<const char *>(src_row_ptr<TWO>(a, c & 0x7fffffff));   // any HINT
  for (int off = 0; off < a.N * 4; off += 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(r + off));
}

// Output row address of a pointer-routed row: a peer (or own) buffer address,
// or -- top bit set -- a row index into Y (the caller's C: local rows of the
// hierarchical Stage-I launch, whose address is only known at call time).
template <typename V>
__device__ __forceinline__ V *out_addr(const SpmmArgs &a, long long v) {
  if (v < 0) return reinterpret_cast<V *>(a.Y + (v & 0x7fffffffffffffffLL) * a.N);
  return reinterpret_cast<V *>(v);
}


// Gather U source rows for nonzeros j..j+U-1 of the current batch; the
// weights are broadcast together with the columns, before any FMA.
template <int LPR, int VPL, int W, bool TWO, int U, int HINT, bool COH>
__device__ __forceinline__ void gather(const SpmmArgs &a, typename VT<W>::T (&x)[U][VPL], int c, int j,
                                       int cnt, int li, unsigned mask) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int cu = __shfl_sync(mask, c, j + u, LPR);
    if (j + u < cnt) {               // uniform across the lane group
      // hot marks (bit 31) exist only in HINT 3 launches
      const typename VT<W>::T *r = src_row<TWO, typename VT<W>::T>(a, HINT == 3 ? (cu & 0x7fffffff) : cu);
      // with two sources only the second one (the receive buffer) is written
      // by peers during the launch
      const bool coh = !TWO || cu >= a.n0;
      // evict_last: marked rows (HINT 3) or the compact hot buffer (HINT 4, X1)
      const bool hot = (HINT == 3 && cu < 0) || (HINT == 4 && cu >= a.n0);
#pragma unroll
      for (int q = 0; q < VPL; ++q)
        x[u][q] = ldB<HINT, COH>(r + li + q * LPR, hot, coh);
    } else {
#pragma unroll
      for (int q = 0; q < VPL; ++q) x[u][q] = VT<W>::zero();
    }
  }
}

// One work unit u: a chunk task (u < n_tasks) or a row group.  OUTP: output
// rows are addressed by a per-row pointer (e.g. a peer's receive buffer over
// NVLink, the fused exchange) instead of Y + out_row * N.
// Unit wait of a two-phase consumer: the sources of unit u's remote part
// (false: a wait failed -> skip the remote part; the error word is set).
template <bool WAIT>
__device__ __forceinline__ bool unit_wait(const SpmmArgs &a, int64_t u, int32_t target, int li,
                                          int lanes, unsigned mask) {
  if (!WAIT) return true;
  const uint64_t need = a.unit_src[u];
  if (!need) return true;
  return wait_sources(a.ready, need, target, a.wait_err, a.wait_timeout_ns, li, lanes, mask);
}

// Non-blocking readiness of unit u's sources (one poll per lane group).
__device__ __forceinline__ bool sources_ready(const SpmmArgs &a, int64_t u, int32_t target, int li,
                                              int lanes, unsigned mask) {
  const uint64_t need = a.unit_src[u];
  bool ok = true;
  for (int s = li; s < 64; s += lanes)
    if ((need >> s) & 1ull) {
      int32_t v;
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(a.ready + s) : "memory");
      ok = ok && v >= target;
    }
  return __all_sync(mask, ok);
}

// Push unit u to the deferred list of the two-phase consumer (lane 0 of the group).
__device__ __forceinline__ void defer_unit(const SpmmArgs &a, int64_t u, int li) {
  if (li == 0) a.defer_list[atomicAdd(a.defer_n, 1)] = (int32_t)u;
}

// STAGE (two-phase ops, PH): 0 = both phases inline (waiting in between when
// WAIT); 1 = phase A, then phase B only if the unit's sources are already
// READY, else the unit is deferred (a hub chunk parks its partial in its
// scratch row) -- never spins; 2 = the deferred continuation: phase B after
// waiting for the sources (launched after this GPU's producer and READY).
template <int LPR, int VPL, int W, bool ACCUM, bool TWO, int U, bool OUTP, int HINT, bool COH,
          bool PF = false, bool PH = false, bool WAIT = false, int STAGE = 0>
__device__ __forceinline__ void spmm_unit(const SpmmArgs &a, const int64_t u, const int li,
                                          const unsigned mask, const int32_t target = 0) {
  typename VT<W>::T acc[VPL];
#pragma unroll
  for (int q = 0; q < VPL; ++q) acc[q] = VT<W>::zero();

  if (u < a.n_tasks) {
    // ---- chunk of a long (hub) row -------------------------------------
    const int lr = a.task_long[u];
    const int64_t t = a.long_row[lr];
    const int f = a.long_first[lr], nch = a.long_first[lr + 1] - f;
    const int64_t rb = __ldg(a.rp + t), re = __ldg(a.rp + t + 1);
    const int64_t clen = (re - rb + nch - 1) / nch;     // chunk length of this hub row
    const int64_t kb = rb + (int64_t)(u - f) * clen;
    const int64_t ke = (kb + clen < re) ? kb + clen : re;
    // two-phase: [kb, kmid) local part, then wait, then [kmid, ke) remote part
    const int64_t kmid = PH ? (a.long_mid[lr] < kb ? kb : (a.long_mid[lr] > ke ? ke : a.long_mid[lr])) : ke;
    auto walk = [&](int64_t k0, int64_t k1) {
      for (int64_t base = k0; base < k1; base += LPR) {
        const int64_t k = base + li;
        int2 cv = make_int2(0, 0);
        if (k < k1) {
          cv = ldcv_h<HINT>(a.cv + k);
          if (PF) prefetch_row<TWO>(a, cv.x);
        }
        const int cnt = (int)((k1 - base) < LPR ? (k1 - base) : LPR);
        for (int j = 0; j < cnt; j += U) {
          typename VT<W>::T x[U][VPL];
          gather<LPR, VPL, W, TWO, U, HINT, COH>(a, x, cv.x, j, cnt, li, mask);
#pragma unroll
          for (int uu = 0; uu < U; ++uu) {
            // the weight is shuffled at use: no register held per row in flight
            // (lanes past cnt hold v = 0 and x = 0)
            const float wu = __shfl_sync(mask, __int_as_float(cv.y), j + uu, LPR);
#pragma unroll
            for (int q = 0; q < VPL; ++q) fma4(acc[q], wu, x[uu][q]);
          }
        }
      }
    };
    typename VT<W>::T *sp = reinterpret_cast<typename VT<W>::T *>(a.scratch + u * (int64_t)a.N);
    if (STAGE == 2) {       // deferred continuation: the parked phase-A partial
#pragma unroll
      for (int q = 0; q < VPL; ++q) acc[q] = __ldcg(sp + li + q * LPR);
    } else {
      walk(kb, kmid);
    }
    if (PH && kmid < ke) {
      if (STAGE == 1 && !sources_ready(a, u, target, li, LPR, mask)) {
#pragma unroll
        for (int q = 0; q < VPL; ++q) __stcg(sp + li + q * LPR, acc[q]);
        defer_unit(a, u, li);
        return;
      }
      if (STAGE == 2 ? unit_wait<true>(a, u, target, li, LPR, mask)
                     : (STAGE == 1 || unit_wait<WAIT>(a, u, target, li, LPR, mask)))
        walk(kmid, ke);
    }
#pragma unroll
    for (int q = 0; q < VPL; ++q) __stcg(sp + li + q * LPR, acc[q]);
    __threadfence();
    __syncwarp(mask);
    int last = 0;
    if (li == 0) last = (atomicAdd(a.long_counter + lr, 1) == nch - 1);
    last = __shfl_sync(mask, last, 0, LPR);
    if (last) {
      __threadfence();
      typename VT<W>::T s[VPL];
#pragma unroll
      for (int q = 0; q < VPL; ++q) s[q] = VT<W>::zero();
      // fixed chunk order (deterministic); 8 partial loads in flight
      for (int c0 = 0; c0 < nch; c0 += 8) {
        typename VT<W>::T pv[8][VPL];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const typename VT<W>::T *cp = reinterpret_cast<const typename VT<W>::T *>(a.scratch + (int64_t)(f + c0 + c) * a.N);
#pragma unroll
          for (int q = 0; q < VPL; ++q)
            pv[c][q] = (c0 + c < nch) ? __ldcg(cp + li + q * LPR) : VT<W>::zero();
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
#pragma unroll
          for (int q = 0; q < VPL; ++q) add4(s[q], pv[c][q]);
      }
      typename VT<W>::T *y;
      if (OUTP) {
        y = out_addr<typename VT<W>::T>(a, (long long)a.out_ptr[t]);
      } else {
        const int64_t orow = a.out_row ? a.out_row[t] : t;
        y = reinterpret_cast<typename VT<W>::T *>(a.Y + orow * a.N);
      }
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        if (ACCUM) add4(s[q], y[li + q * LPR]);
        y[li + q * LPR] = s[q];
      }
      if (li == 0) a.long_counter[lr] = 0;    // re-arm for the next launch
    }
    return;
  }

  // ---- row group: rows [r0, r1), nonzeros [k0, k1) ------------------------
  const int64_t gi = u - a.n_tasks;
  if (gi >= a.n_groups) return;
  const RowGroup g = a.groups[gi];
  const int64_t kend = PH ? g.kmid : g.k1;      // phase A (or the whole group)
  const int nrows = g.r1 - g.r0;
  // output rows of the group, one per lane (groups with an out_row map have
  // <= 2*LPR rows, checked at plan time)
  int orw0 = 0, orw1 = 0;
  long long opw0 = 0, opw1 = 0;
  if (OUTP) {
    if (li < nrows) opw0 = (long long)a.out_ptr[g.r0 + li];
    if (LPR + li < nrows) opw1 = (long long)a.out_ptr[g.r0 + LPR + li];
  } else if (a.out_row) {
    if (li < nrows) orw0 = __ldg(a.out_row + g.r0 + li);
    if (LPR + li < nrows) orw1 = __ldg(a.out_row + g.r0 + LPR + li);
  }
  int cur = 0;   // current row offset inside the group
  auto flush = [&]() {
    typename VT<W>::T *y;
    if (OUTP) {
      const long long sel = (cur < LPR) ? opw0 : opw1;
      y = out_addr<typename VT<W>::T>(a, __shfl_sync(mask, sel, cur & (LPR - 1), LPR));
    } else {
      int64_t orow;
      if (a.out_row) {
        const int sel = (cur < LPR) ? orw0 : orw1;
        orow = __shfl_sync(mask, sel, cur & (LPR - 1), LPR);
      } else {
        orow = g.r0 + cur;
      }
      y = reinterpret_cast<typename VT<W>::T *>(a.Y + orow * a.N);
    }
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      if (ACCUM) add4(acc[q], y[li + q * LPR]);
      stY_h<HINT>(y + li + q * LPR, acc[q]);
      acc[q] = VT<W>::zero();
    }
    ++cur;
  };
  for (int64_t base = g.k0; STAGE != 2 && base < kend; base += LPR) {
    const int64_t k = base + li;
    int2 cv = make_int2(0, 0);
    int ro = 0;
    if (k < kend) {
      cv = ldcv_h<HINT>(a.cv + k);
      ro = ld_stream_u8(a.roff + k);
      if (PF) prefetch_row<TWO>(a, cv.x);
    }
    const int cnt = (int)((kend - base) < LPR ? (kend - base) : LPR);
    for (int j = 0; j < cnt; j += U) {
      typename VT<W>::T x[U][VPL];
      gather<LPR, VPL, W, TWO, U, HINT, COH>(a, x, cv.x, j, cnt, li, mask);
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int rou = __shfl_sync(mask, ro, j + uu, LPR);
        const float wu = __shfl_sync(mask, __int_as_float(cv.y), j + uu, LPR);
        if (j + uu < cnt) {
          while (cur < rou) flush();        // finished rows (and empty rows)
#pragma unroll
          for (int q = 0; q < VPL; ++q) fma4(acc[q], wu, x[uu][q]);
        }
      }
    }
  }
  if (STAGE != 2)
    while (cur < nrows) flush();            // last row and trailing empty rows
  if (!PH || g.kmid >= g.k1) return;
  // ---- phase B (two-phase consumer): the group's remote parts ------------
  // after its sources' READY; only rows with remote nonzeros are updated
  // (read-modify-write of rows this unit itself just wrote, in L2)
  if (STAGE == 1) {
    if (!sources_ready(a, u, target, li, LPR, mask)) {
      defer_unit(a, u, li);
      return;
    }
  } else if (!unit_wait<(STAGE == 2 || WAIT)>(a, u, target, li, LPR, mask)) {
    return;
  }
  int rcur = -1;
  auto flush_b = [&]() {
    int64_t orow;
    if (a.out_row) {
      const int sel = (rcur < LPR) ? orw0 : orw1;
      orow = __shfl_sync(mask, sel, rcur & (LPR - 1), LPR);
    } else {
      orow = g.r0 + rcur;
    }
    typename VT<W>::T *y = reinterpret_cast<typename VT<W>::T *>(a.Y + orow * a.N);
#pragma unroll
    for (int q = 0; q < VPL; ++q) {
      add4(acc[q], __ldcg(y + li + q * LPR));
      y[li + q * LPR] = acc[q];
      acc[q] = VT<W>::zero();
    }
  };
  for (int64_t base = g.kmid; base < g.k1; base += LPR) {
    const int64_t k = base + li;
    int2 cv = make_int2(0, 0);
    int ro = 0;
    if (k < g.k1) {
      cv = ldcv_h<HINT>(a.cv + k);
      ro = ld_stream_u8(a.roff + k);
    }
    const int cnt = (int)((g.k1 - base) < LPR ? (g.k1 - base) : LPR);
    for (int j = 0; j < cnt; j += U) {
      typename VT<W>::T x[U][VPL];
      gather<LPR, VPL, W, TWO, U, HINT, COH>(a, x, cv.x, j, cnt, li, mask);
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int rou = __shfl_sync(mask, ro, j + uu, LPR);
        const float wu = __shfl_sync(mask, __int_as_float(cv.y), j + uu, LPR);
        if (j + uu < cnt) {
          if (rou != rcur) {
            if (rcur >= 0) flush_b();
            rcur = rou;
          }
#pragma unroll
          for (int q = 0; q < VPL; ++q) fma4(acc[q], wu, x[uu][q]);
        }
      }
    }
  }
  if (rcur >= 0) flush_b();
}

// N <= 128 (VPL = 1): one-warp CTAs (BS = 32), 32 resident per SM; wider
// rows (VPL > 1) keep 8-warp CTAs without a residency floor (no spills).
// WAIT: remote SpMM with per-unit source waits (launched after this GPU's
// producer and READY).  PH + STAGE 1: the two-phase consumer's first launch
// (concurrent with the producer, never spins); PH + STAGE 2: its deferred
// continuation (after this GPU's producer and READY; a persistent grid pulls
// the deferred units).
template <int LPR, int VPL, int W, bool ACCUM, bool TWO, int U, bool OUTP, int HINT, bool WAIT,
          int BS = 32, int MINB = 32, bool PF = false, bool PH = false, int STAGE = 0>
__global__ void __launch_bounds__(BS, MINB) k_spmm(const SpmmArgs a) {
  constexpr int R = 32 / LPR;   // lane groups per warp
  constexpr int UU = (U < LPR ? U : LPR);
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR;
  const int li = lane % LPR;
  const unsigned mask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  const int64_t u = (((int64_t)blockIdx.x * BS + threadIdx.x) >> 5) * R + sub;
  if (PH && STAGE == 1) {
    const int32_t target = *reinterpret_cast<volatile int32_t *>(a.wait_epoch) + 1;
    spmm_unit<LPR, VPL, W, ACCUM, TWO, UU, OUTP, HINT, true, false, true, false, 1>(a, u, li, mask,
                                                                                target);
    return;
  }
  if (PH && STAGE == 2) {
    const int32_t target = *reinterpret_cast<volatile int32_t *>(a.wait_epoch) + 1;
    const int32_t nd = *reinterpret_cast<volatile int32_t *>(a.defer_n);
    for (;;) {
      int i = 0;
      if (li == 0) i = atomicAdd(a.work_ctr, 1);
      i = __shfl_sync(mask, i, 0, LPR);
      if (i >= nd) break;
      spmm_unit<LPR, VPL, W, ACCUM, TWO, UU, OUTP, HINT, true, false, true, true, 2>(
          a, a.defer_list[i], li, mask, target);
    }
    return;   // the step-end barrier and the epoch advance are the next launch (k_wait)
  }
  if (WAIT) {
    // target epoch read before this warp is counted done (the last warp
    // advances it, after every warp has read it)
    const int32_t target = *reinterpret_cast<volatile int32_t *>(a.wait_epoch) + 1;
    // remote SpMM: each lane group waits for its own unit's sources first
    const bool in = u < (int64_t)a.n_tasks + a.n_groups;
    if (in && unit_wait<true>(a, u, target, li, LPR, mask))
      spmm_unit<LPR, VPL, W, ACCUM, TWO, UU, OUTP, HINT, true>(a, u, li, mask);
    return;   // the step-end barrier and the epoch advance are the next launch (k_wait)
  }
  // two-phase without waits (loopback): coherent loads of the second source
  spmm_unit<LPR, VPL, W, ACCUM, TWO, UU, OUTP, HINT, PH, PF, PH, false>(a, u, li, mask);
}

// Generic width (N not a supported vector width): one warp per CSR row,
// lanes stride over columns; no row grouping or splitting.  Correctness path.
template <bool ACCUM>
__global__ void __launch_bounds__(kBlock) k_spmm_generic(const SpmmArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  if (t >= a.nrows) return;
  const int64_t kb = a.rp[t], ke = a.rp[t + 1];
  float *y;
  if (a.out_ptr) {
    const long long v = (long long)a.out_ptr[t];
    y = (v < 0) ? a.Y + (v & 0x7fffffffffffffffLL) * a.N : reinterpret_cast<float *>(v);
  } else {
    const int64_t orow = a.out_row ? a.out_row[t] : t;
    y = a.Y + orow * a.N;
  }
  for (int c0 = 0; c0 < a.N; c0 += 32 * 4) {
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int64_t k = kb; k < ke; ++k) {
      const int2 cv = a.cv[k];
      const int c = cv.x & 0x7fffffff;
      const float v = __int_as_float(cv.y);
      const float *r = (c < a.n0) ? a.X0 + (int64_t)c * a.N : a.X1 + (int64_t)(c - a.n0) * a.N;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int x = c0 + lane + 32 * q;
        if (x < a.N) acc[q] = fmaf(v, __ldcg(r + x), acc[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int x = c0 + lane + 32 * q;
      if (x < a.N) y[x] = ACCUM ? y[x] + acc[q] : acc[q];
    }
  }
}

template <int LPR, int VPL>
__global__ void __launch_bounds__(kBlock) k_pack(int64_t n, const int32_t *__restrict__ src,
                                                 const int32_t *__restrict__ dst,
                                                 const float *__restrict__ X, float *__restrict__ Y,
                                                 int N) {
  constexpr int R = 32 / LPR;
  constexpr int RPU = 4;   // rows per lane group: 4 loads in flight before the stores
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR, li = lane % LPR;
  const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int64_t u0 = (warp * R + sub) * RPU;
  float4 x[RPU][VPL];
#pragma unroll
  for (int r = 0; r < RPU; ++r) {
    if (u0 + r < n) {
      const float4 *s = reinterpret_cast<const float4 *>(X + (int64_t)__ldg(src + u0 + r) * N);
#pragma unroll
      for (int q = 0; q < VPL; ++q) x[r][q] = __ldg(s + li + q * LPR);
    }
  }
#pragma unroll
  for (int r = 0; r < RPU; ++r) {
    if (u0 + r < n) {
      float4 *d = reinterpret_cast<float4 *>(Y + (int64_t)__ldg(dst + u0 + r) * N);
#pragma unroll
      for (int q = 0; q < VPL; ++q) d[li + q * LPR] = x[r][q];
    }
  }
}

// K4 into peer buffers: Y row of packed row i is the pointer dstp[i].
// The source may be a buffer peers store into during other launches (the
// hierarchical forward reads its own R1), so it is read L2-coherently.
template <int LPR, int VPL>
__global__ void __launch_bounds__(kBlock) k_pack_ptr(int64_t n, const int32_t *__restrict__ src,
                                                     float *const *__restrict__ dstp,
                                                     const float *__restrict__ X, int N) {
  constexpr int R = 32 / LPR;
  constexpr int RPU = 4;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR, li = lane % LPR;
  const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int64_t u0 = (warp * R + sub) * RPU;
  float4 x[RPU][VPL];
#pragma unroll
  for (int r = 0; r < RPU; ++r) {
    if (u0 + r < n) {
      const float4 *s = reinterpret_cast<const float4 *>(X + (int64_t)__ldg(src + u0 + r) * N);
#pragma unroll
      for (int q = 0; q < VPL; ++q) x[r][q] = __ldcg(s + li + q * LPR);
    }
  }
#pragma unroll
  for (int r = 0; r < RPU; ++r) {
    if (u0 + r < n) {
      float4 *d = reinterpret_cast<float4 *>(dstp[u0 + r]);
#pragma unroll
      for (int q = 0; q < VPL; ++q) d[li + q * LPR] = x[r][q];
    }
  }
}

__global__ void __launch_bounds__(kBlock) k_pack_ptr_generic(int64_t n, const int32_t *src,
                                                             float *const *dstp, const float *X,
                                                             int N) {
  const int lane = threadIdx.x & 31;
  const int64_t u = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  if (u >= n) return;
  const float *s = X + (int64_t)src[u] * N;
  float *d = dstp[u];
  for (int x = lane; x < N; x += 32) d[x] = __ldcg(s + x);
}

__global__ void __launch_bounds__(kBlock) k_pack_generic(int64_t n, const int32_t *src,
                                                         const int32_t *dst, const float *X,
                                                         float *Y, int N) {
  const int lane = threadIdx.x & 31;
  const int64_t u = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  if (u >= n) return;
  const float *s = X + (int64_t)src[u] * N;
  float *d = Y + (int64_t)dst[u] * N;
  for (int x = lane; x < N; x += 32) d[x] = s[x];
}

// K5: gather-sum of received partial C rows.  One lane group owns a target
// row: C[t] = C[t] + sum of its partials in source order (at most P-1 flat,
// plus hierarchical aggregates) -- no atomics, deterministic.
template <int LPR, int VPL>
__global__ void __launch_bounds__(kBlock) k_scatter_add(int64_t nt, const int32_t *__restrict__ tgt,
                                                        const int64_t *__restrict__ ptr,
                                                        const int32_t *__restrict__ srcrow,
                                                        const float *__restrict__ Rb,
                                                        float *__restrict__ C, int N) {
  constexpr int R = 32 / LPR;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPR, li = lane % LPR;
  const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int64_t u = warp * R + sub;
  if (u >= nt) return;
  const int64_t kb = __ldg(ptr + u), ke = __ldg(ptr + u + 1);
  float4 *c = reinterpret_cast<float4 *>(C + (int64_t)__ldg(tgt + u) * N);
  float4 acc[VPL];
#pragma unroll
  for (int q = 0; q < VPL; ++q) acc[q] = c[li + q * LPR];
  for (int64_t k = kb; k < ke; k += 4) {
    float4 x[4][VPL];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (k + r < ke) {
        const float4 *s = reinterpret_cast<const float4 *>(Rb + (int64_t)__ldg(srcrow + k + r) * N);
#pragma unroll
        for (int q = 0; q < VPL; ++q) x[r][q] = __ldcs(s + li + q * LPR);
      } else {
#pragma unroll
        for (int q = 0; q < VPL; ++q) x[r][q] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < VPL; ++q) add4(acc[q], x[r][q]);
  }
#pragma unroll
  for (int q = 0; q < VPL; ++q) c[li + q * LPR] = acc[q];
}

__global__ void __launch_bounds__(kBlock) k_scatter_add_generic(int64_t nt, const int32_t *tgt,
                                                                const int64_t *ptr,
                                                                const int32_t *srcrow,
                                                                const float *Rb, float *C, int N) {
  const int lane = threadIdx.x & 31;
  const int64_t u = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
  if (u >= nt) return;
  float *c = C + (int64_t)tgt[u] * N;
  for (int x = lane; x < N; x += 32) {
    float acc = c[x];
    for (int64_t k = ptr[u]; k < ptr[u + 1]; ++k) acc += Rb[(int64_t)srcrow[k] * N + x];
    c[x] = acc;
  }
}

__global__ void k_refresh(int64_t nnz, const int32_t *__restrict__ vsrc,
                          const float *__restrict__ V, int2 *__restrict__ cv) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = vsrc[k];
    if (s >= 0) cv[k].y = __float_as_int(V[s]);
  }
}

inline int64_t blocks_for(int64_t units, int rows_per_warp) {
  const int64_t per_block = (int64_t)(kBlock / 32) * rows_per_warp;
  return (units + per_block - 1) / per_block;
}

template <int LPR, int VPL, int W, int H, bool PF = false, int UO = 0>
void spmm_launch(const SpmmArgs &a, bool acc, cudaStream_t s) {
  // rows in flight per lane group: 8 (N = 128: 8 float4 rows in 64 registers
  // since the weights are shuffled at use, measured 3-7 % faster than 4 on
  // c3 / c4; N = 64: 8 float2 -- 16 was 29 % slower on c5); 4 for the
  // narrow float4 lane groups (N = 4..16)
  constexpr int U = UO ? UO : ((VPL == 1 && W == 4 && LPR < 32) ? 4 : 8);
  constexpr int BS = VPL == 1 ? 32 : 256, MINB = VPL == 1 ? 32 : 1;
  const int64_t units = a.n_tasks + a.n_groups;
  const int64_t per_cta = (int64_t)(BS / 32) * (32 / LPR);
  const unsigned grid = (unsigned)((units + per_cta - 1) / per_cta);
  const bool two = a.X1 != nullptr;
  if (a.ready && a.long_mid) {   // two-phase consumer (CX): stage 1 or its deferred stage 2
    if (a.cx_stage == 1) {
      k_spmm<LPR, VPL, W, false, true, U, false, 0, false, BS, MINB, false, true, 1>
          <<<grid, BS, 0, s>>>(a);
    } else {
      const int64_t per_cta2 = (int64_t)(BS / 32) * (32 / LPR);
      const int64_t cap = ((int64_t)num_sms() * 32 * 32 / BS) ;   // one wave of lane groups
      const unsigned g2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((units + per_cta2 - 1) / per_cta2, cap));
      k_spmm<LPR, VPL, W, false, true, U, false, 0, false, BS, MINB, false, true, 2>
          <<<g2, BS, 0, s>>>(a);
    }
  } else if (a.ready) {   // remote SpMM with per-unit source waits, coherent loads
    k_spmm<LPR, VPL, W, true, false, U, false, 0, true, BS, MINB, false, false><<<grid, BS, 0, s>>>(a);
  } else if (a.long_mid) {   // two-phase consumer without waits (loopback)
    k_spmm<LPR, VPL, W, false, true, U, false, 0, false, BS, MINB, false, true><<<grid, BS, 0, s>>>(a);
  } else if (a.out_ptr) {   // fused exchange: overwrite rows in peer buffers
    k_spmm<LPR, VPL, W, false, false, U, true, H, false, BS, MINB, PF><<<grid, BS, 0, s>>>(a);
  } else if (acc) {
    if (two) k_spmm<LPR, VPL, W, true, true, U, false, H, false, BS, MINB, PF><<<grid, BS, 0, s>>>(a);
    else k_spmm<LPR, VPL, W, true, false, U, false, H, false, BS, MINB, PF><<<grid, BS, 0, s>>>(a);
  } else {
    if (two) k_spmm<LPR, VPL, W, false, true, U, false, H, false, BS, MINB, PF><<<grid, BS, 0, s>>>(a);
    else k_spmm<LPR, VPL, W, false, false, U, false, H, false, BS, MINB, PF><<<grid, BS, 0, s>>>(a);
  }
}

// L2 policy of a launch (SHIRO_L2HINT overrides): 3 when the op carries hot
// marks, 4 with a compact hot buffer, 2 when its source rows fit comfortably
// in L2 (c2: B = 87 MB, -5 %, profiles/r1_kernel_sweep.txt), else 1 (the
// streams evict_first: c3 / c4 / c5 -0.4 / -0.5 / -2.2 %, profiles/r2_hotbuf_sweep.txt).
int l2_hint(const SpmmArgs &a) {
  static const int env_hint = getenv("SHIRO_L2HINT") ? atoi(getenv("SHIRO_L2HINT")) : -1;
  static const int hb_pol = getenv("SHIRO_HOTBUF_POL") ? atoi(getenv("SHIRO_HOTBUF_POL")) : 1;
  if (a.hot == 2 && a.X1) return hb_pol ? 4 : 0;   // compact hot buffer
  if (env_hint >= 0) return (env_hint == 3 && a.hot != 1) ? 0 : env_hint;
  if (a.hot == 1) return 3;
  return (a.X1 == nullptr && a.n0 * (int64_t)a.N * 4 <= (96ll << 20)) ? 2 : 1;
}

// L2 prefetch of each batch's source rows (SHIRO_PREFETCH: 1 on, 0 off; by
// default on when the source rows are far larger than L2, where the gather
// waits on DRAM)
bool use_prefetch(const SpmmArgs &a) {
  static const int env = getenv("SHIRO_PREFETCH") ? atoi(getenv("SHIRO_PREFETCH")) : -1;
  if (env >= 0) return env == 1;
  return false;
}

template <int LPR, int VPL, int W>
void spmm_shape(const SpmmArgs &a, bool acc, cudaStream_t s) {
  if constexpr (VPL == 1 && LPR >= 8) {
    const int h = l2_hint(a);
    const bool pf = h != 2 && use_prefetch(a);
    if constexpr (W >= 2 && LPR == 32) {   // SHIRO_U128=4 / SHIRO_U64=4: 4 rows in flight (A/B)
      static const bool u4 = getenv(W == 4 ? "SHIRO_U128" : "SHIRO_U64") &&
                             atoi(getenv(W == 4 ? "SHIRO_U128" : "SHIRO_U64")) == 4;
      if (u4 && h <= 2) {
        if (h == 2) spmm_launch<LPR, VPL, W, 2, false, 4>(a, acc, s);
        else if (h == 1) spmm_launch<LPR, VPL, W, 1, false, 4>(a, acc, s);
        else spmm_launch<LPR, VPL, W, 0, false, 4>(a, acc, s);
        return;
      }
    }
    if (h == 2) { spmm_launch<LPR, VPL, W, 2>(a, acc, s); return; }
    if (h == 1) { spmm_launch<LPR, VPL, W, 1>(a, acc, s); return; }
    if (h == 4) { spmm_launch<LPR, VPL, W, 4>(a, acc, s); return; }
    if (h == 3) {
      if (pf) spmm_launch<LPR, VPL, W, 3, true>(a, acc, s);
      else spmm_launch<LPR, VPL, W, 3>(a, acc, s);
      return;
    }
    if (pf) { spmm_launch<LPR, VPL, W, 0, true>(a, acc, s); return; }
  }
  spmm_launch<LPR, VPL, W, 0>(a, acc, s);
}

template <int LPR, int VPL>
void pack_shape(int64_t n, const int32_t *src, const int32_t *dst, const float *X, float *Y,
                int N, cudaStream_t s) {
  const int64_t grid = blocks_for((n + 3) / 4, 32 / LPR);
  k_pack<LPR, VPL><<<(unsigned)grid, kBlock, 0, s>>>(n, src, dst, X, Y, N);
}

template <int LPR, int VPL>
void pack_ptr_shape(int64_t n, const int32_t *src, float *const *dstp, const float *X, int N,
                    cudaStream_t s) {
  const int64_t grid = blocks_for((n + 3) / 4, 32 / LPR);
  k_pack_ptr<LPR, VPL><<<(unsigned)grid, kBlock, 0, s>>>(n, src, dstp, X, N);
}

template <int LPR, int VPL>
void scatter_shape(int64_t nt, const int32_t *tgt, const int64_t *ptr, const int32_t *src,
                   const float *R, float *C, int N, cudaStream_t s) {
  const int64_t grid = blocks_for(nt, 32 / LPR);
  k_scatter_add<LPR, VPL><<<(unsigned)grid, kBlock, 0, s>>>(nt, tgt, ptr, src, R, C, N);
}

#define SHIRO_DISPATCH(N, FN, ...)                        \
  do {                                                    \
    int lpr_, vpl_;                                       \
    vec_shape(N, &lpr_, &vpl_);                           \
    if (lpr_ == 1) FN<1, 1>(__VA_ARGS__);                 \
    else if (lpr_ == 2) FN<2, 1>(__VA_ARGS__);            \
    else if (lpr_ == 4) FN<4, 1>(__VA_ARGS__);            \
    else if (lpr_ == 8) FN<8, 1>(__VA_ARGS__);            \
    else if (lpr_ == 16) FN<16, 1>(__VA_ARGS__);          \
    else if (vpl_ == 1) FN<32, 1>(__VA_ARGS__);           \
    else if (vpl_ == 2) FN<32, 2>(__VA_ARGS__);           \
    else FN<32, 4>(__VA_ARGS__);                          \
  } while (0)

}  // namespace

// Vector shape for width N: LPR lanes per row, VPL float4 per lane.
bool vec_shape(int N, int *lpr, int *vpl) {
  switch (N) {
    case 4: *lpr = 1; *vpl = 1; return true;
    case 8: *lpr = 2; *vpl = 1; return true;
    case 16: *lpr = 4; *vpl = 1; return true;
    case 32: *lpr = 8; *vpl = 1; return true;
    case 64: *lpr = 16; *vpl = 1; return true;
    case 128: *lpr = 32; *vpl = 1; return true;
    case 256: *lpr = 32; *vpl = 2; return true;
    case 512: *lpr = 32; *vpl = 4; return true;
    default: return false;
  }
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (!n) n = 148;
  }
  return n;
}

// SpMM lane shape for width N: LPR lanes per output row, W floats per lane
// load, VPL loads per lane (N = LPR * W * VPL); false -> generic path.
bool spmm_vec_shape(int N, int *lpr, int *w, int *vpl) {
  switch (N) {
    case 4: *lpr = 1; *w = 4; *vpl = 1; return true;
    case 8: *lpr = 2; *w = 4; *vpl = 1; return true;
    case 16: *lpr = 4; *w = 4; *vpl = 1; return true;
    case 32: *lpr = 32; *w = 1; *vpl = 1; return true;
    case 64: *lpr = 32; *w = 2; *vpl = 1; return true;
    case 128: *lpr = 32; *w = 4; *vpl = 1; return true;
    case 256: *lpr = 32; *w = 4; *vpl = 2; return true;
    case 512: *lpr = 32; *w = 4; *vpl = 4; return true;
    default: return false;
  }
}

int launch_spmm(const SpmmArgs &a, bool accumulate, cudaStream_t s) {
  if (a.nrows == 0) return 0;
  int lpr, w, vpl;
  if (spmm_vec_shape(a.N, &lpr, &w, &vpl)) {
    if (a.n_tasks + a.n_groups == 0) return 0;
    switch (a.N) {
      case 4: spmm_shape<1, 1, 4>(a, accumulate, s); break;
      case 8: spmm_shape<2, 1, 4>(a, accumulate, s); break;
      case 16: spmm_shape<4, 1, 4>(a, accumulate, s); break;
      case 32: spmm_shape<32, 1, 1>(a, accumulate, s); break;
      case 64: spmm_shape<32, 1, 2>(a, accumulate, s); break;
      case 128: spmm_shape<32, 1, 4>(a, accumulate, s); break;
      case 256: spmm_shape<32, 2, 4>(a, accumulate, s); break;
      default: spmm_shape<32, 4, 4>(a, accumulate, s); break;
    }
  } else {
    const int64_t grid = blocks_for(a.nrows, 1);
    if (accumulate)
      k_spmm_generic<true><<<(unsigned)grid, kBlock, 0, s>>>(a);
    else
      k_spmm_generic<false><<<(unsigned)grid, kBlock, 0, s>>>(a);
  }
  return 1;
}

int launch_pack(int64_t n, const int32_t *src, const int32_t *dst, const float *X, float *Y,
                int32_t N, cudaStream_t s) {
  if (n == 0) return 0;
  int lpr, vpl;
  if (vec_shape(N, &lpr, &vpl)) {
    SHIRO_DISPATCH(N, pack_shape, n, src, dst, X, Y, N, s);
  } else {
    k_pack_generic<<<(unsigned)blocks_for(n, 1), kBlock, 0, s>>>(n, src, dst, X, Y, N);
  }
  return 1;
}

int launch_pack_ptr(int64_t n, const int32_t *src, float *const *dstp, const float *X, int32_t N,
                    cudaStream_t s) {
  if (n == 0) return 0;
  int lpr, vpl;
  if (vec_shape(N, &lpr, &vpl)) {
    SHIRO_DISPATCH(N, pack_ptr_shape, n, src, dstp, X, N, s);
  } else {
    k_pack_ptr_generic<<<(unsigned)blocks_for(n, 1), kBlock, 0, s>>>(n, src, dstp, X, N);
  }
  return 1;
}

int launch_scatter_add(int64_t nt, const int32_t *tgt, const int64_t *ptr, const int32_t *src,
                       const float *R, float *C, int32_t N, cudaStream_t s) {
  if (nt == 0) return 0;
  int lpr, vpl;
  if (vec_shape(N, &lpr, &vpl)) {
    SHIRO_DISPATCH(N, scatter_shape, nt, tgt, ptr, src, R, C, N, s);
  } else {
    k_scatter_add_generic<<<(unsigned)blocks_for(nt, 1), kBlock, 0, s>>>(nt, tgt, ptr, src, R, C,
                                                                          N);
  }
  return 1;
}

int launch_refresh(int64_t nnz, const int32_t *vsrc, const float *V, int2 *cv, cudaStream_t s) {
  if (nnz == 0) return 0;
  const int64_t want = (nnz + 255) / 256;
  const unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)num_sms() * 8);
  k_refresh<<<grid, 256, 0, s>>>(nnz, vsrc, V, cv);
  return 1;
}

}  // namespace shiro

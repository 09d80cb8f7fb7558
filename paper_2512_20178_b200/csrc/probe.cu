// probe.cu -- measurement probe (not on the hot path): a pure row gather,
//   out[c] = sum_{k in chunk c} X[idx[k]]   (chunks of `chunk` indices),
// with the same 128-bit, 8-deep load structure as the SpMM kernels.  Fed with
// an SpMM's own column-index stream it times the unavoidable part of that
// SpMM -- every referenced source row delivered to an SM once per nonzero --
// which is the gather-aware roofline of DESIGN.md section 5.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/shiro.h"

namespace {

template <int LPR>
__global__ void __launch_bounds__(256) k_probe_gather(const float *__restrict__ X, int N,
                                                      const int32_t *__restrict__ idx, int64_t n,
                                                      int chunk, float *__restrict__ out) {
  constexpr int R = 32 / LPR;
  const int lane = threadIdx.x & 31, sub = lane / LPR, li = lane % LPR;
  const unsigned mask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (sub * LPR));
  const int64_t c = (((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5) * R + sub;
  const int64_t kb = c * chunk;
  if (kb >= n) return;
  const int64_t ke = (kb + chunk < n) ? kb + chunk : n;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t base = kb; base < ke; base += LPR) {
    const int64_t k = base + li;
    const int col = (k < ke) ? __ldg(idx + k) : 0;
    const int cnt = (int)((ke - base) < LPR ? (ke - base) : LPR);
    for (int j = 0; j < cnt; j += 8) {
      float4 x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int cu = __shfl_sync(mask, col, (j + u) & (LPR - 1), LPR);
        x[u] = (j + u < cnt) ? __ldg(reinterpret_cast<const float4 *>(X + (int64_t)cu * N) + li)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc.x += x[u].x; acc.y += x[u].y; acc.z += x[u].z; acc.w += x[u].w;
      }
    }
  }
  reinterpret_cast<float4 *>(out + c * N)[li] = acc;
}

// ---- TMA variant: the same sum, rows staged by cp.async.bulk.tensor
// tile::gather4 (4 rows of 512 B per instruction) into an S-stage shared
// memory ring per warp (one warp per CTA); lane 0 issues, every lane reads
// its float4 of each staged row.  In-flight bytes cost shared memory instead
// of registers.  N = 128 only (box = 128 fp32 x 1 row, 4 rows per gather4).
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
// the retry loop is C++ (no label inside inline asm: a kernel that inlines
// the wait twice must not end up with two branch targets of the same name)
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *tm, uint64_t *bar, int r0,
                                            int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(0), "r"(r0), "r"(r1), "r"(r2),
      "r"(r3)
      : "memory");
}

template <int S>
__global__ void __launch_bounds__(32) k_probe_gather_tma(const __grid_constant__ CUtensorMap tm,
                                                         const int32_t *__restrict__ idx, int64_t n,
                                                         int chunk, float *__restrict__ out) {
  extern __shared__ __align__(128) float4 ring[];   // S x 4 rows x 32 float4
  __shared__ __align__(8) uint64_t bar[S];
  const int li = threadIdx.x;
  const int64_t kb = (int64_t)blockIdx.x * chunk;
  const int64_t ke = (kb + chunk < n) ? kb + chunk : n;
  const int cnt = (int)(ke - kb);
  const int nq = (cnt + 3) / 4;
  if (li == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int q) {   // lane 0 only
    const int s = q % S;
    int r[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] = __ldg(idx + kb + ((4 * q + i < cnt) ? 4 * q + i : 0));
    mbar_expect_tx(&bar[s], 4 * 512);
    tma_gather4(ring + s * 128, &tm, &bar[s], r[0], r[1], r[2], r[3]);
  };
  if (li == 0)
    for (int q = 0; q < S && q < nq; ++q) issue(q);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int q = 0; q < nq; ++q) {
    const int s = q % S;
    mbar_wait(&bar[s], (uint32_t)((q / S) & 1));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (4 * q + i < cnt) {
        const float4 x = ring[s * 128 + i * 32 + li];
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
      }
    }
    __syncwarp();
    if (li == 0 && q + S < nq) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads -> async writes
      issue(q + S);
    }
  }
  reinterpret_cast<float4 *>(out + blockIdx.x * 128LL)[li] = acc;
}

// ---- roofline denominators (SURVEY 8(d) microbenchmarks) ------------------
// FP32 FMA: 8 independent dependency chains per thread, 4 FMAs per chain per
// iteration; every thread stores its sum (no dead code).
__global__ void __launch_bounds__(256) k_probe_fma(float *__restrict__ out, int iters) {
  const float m = 0.9999999f, c = 1e-7f;
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = (float)(threadIdx.x + j) * 1e-3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], m, c);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  out[(int64_t)blockIdx.x * 256 + threadIdx.x] = s;
}

// HBM copy: float4 grid-stride copy (read + write bytes), 4 loads in flight
// per thread before the stores
__global__ void __launch_bounds__(256) k_probe_copy(const float4 *__restrict__ x,
                                                    float4 *__restrict__ y, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * 256;
  int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(x + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) __stcs(y + i + u * stride, v[u]);
  }
  for (; i < n; i += stride) __stcs(y + i, __ldcs(x + i));
}

// ---- warp-specialized TMA variant (round 2): in-flight bytes decoupled from
// warps.  CTA = 1 producer warp + 8 consumer warps, 4 CTAs per SM, an
// S-stage ring of gather4 tiles (4 rows x 512 B = 2 KB per stage) per CTA: up
// to 4 x S x 2 KB per SM in flight (S = 24: 192 KB) vs 32 warps x 4 rows x
// 512 B = 64 KB for LDG.128.  Lane 0 of warp 0 issues cp.async.bulk.tensor
// tile::gather4 into stage q % S after the stage's EMPTY barrier; consumer c
// takes quads q = c, c + 8, ... -- S is a multiple of 8, so every phase of a
// stage is awaited by the same warp in order (a parity wait on phase k while
// phase k-1 is still pending would pass at once on the stale parity: the
// first version, 7 consumers, deadlocked that way at full occupancy).  Each
// CTA walks a contiguous range of quads.
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

template <int S>
__global__ void __launch_bounds__(288) k_probe_gather_tma_ws(const __grid_constant__ CUtensorMap tm,
                                                             const int32_t *__restrict__ idx,
                                                             int64_t nquads, int64_t n,
                                                             float *__restrict__ out) {
  extern __shared__ __align__(128) float4 ring[];   // S x 4 rows x 32 float4
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t per = (nquads + gridDim.x - 1) / gridDim.x;
  const int64_t q0 = (int64_t)blockIdx.x * per;
  const int64_t q1 = (q0 + per < nquads) ? q0 + per : nquads;
  const int64_t nq = q1 > q0 ? q1 - q0 : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    // the whole producer warp loads the indices of 8 quads at once (one
    // coalesced 128-B load), lane 0 issues the 8 gather4s with the indices
    // shuffled to it: the index latency is off the issue path
    for (int64_t q8 = 0; q8 < nq; q8 += 8) {
      const int64_t k = 4 * (q0 + q8) + lane;
      const int idxv = __ldg(idx + (k < n ? k : n - 1));
      for (int j = 0; j < 8; ++j) {
        const int r0 = __shfl_sync(0xffffffffu, idxv, 4 * j + 0);
        const int r1 = __shfl_sync(0xffffffffu, idxv, 4 * j + 1);
        const int r2 = __shfl_sync(0xffffffffu, idxv, 4 * j + 2);
        const int r3 = __shfl_sync(0xffffffffu, idxv, 4 * j + 3);
        const int64_t q = q8 + j;
        if (lane == 0 && q < nq) {
          const int s = (int)(q % S);
          if (q >= S) {
            mbar_wait(&empty[s], (uint32_t)(((q / S) - 1) & 1));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // consumers' reads -> async writes
          }
          mbar_expect_tx(&full[s], 4 * 512);
          tma_gather4(ring + s * 128, &tm, &full[s], r0, r1, r2, r3);
        }
        __syncwarp();
      }
    }
    return;
  }
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  static_assert(S % 8 == 0, "stages must be a multiple of the 8 consumers");
  for (int64_t q = warp - 1; q < nq; q += 8) {
    const int s = (int)(q % S);
    mbar_wait(&full[s], (uint32_t)((q / S) & 1));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 x = ring[s * 128 + i * 32 + lane];
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  reinterpret_cast<float4 *>(out + ((int64_t)blockIdx.x * 8 + warp - 1) * 128)[lane] = acc;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

extern "C" int shiro_probe_gather_tma(const float *X, int64_t x_rows, int32_t N, const int32_t *idx,
                                      int64_t n_idx, float *out, int32_t chunk, int32_t stages,
                                      void *stream) {
  if (!X || !idx || !out || n_idx < 0 || chunk < 4 || chunk % 4 || N != 128 || x_rows < 1)
    return SHIRO_E_ARG;
  if (stages != 2 && stages != 4 && stages != 8) return SHIRO_E_ARG;
  auto enc = encode_fn();
  if (!enc) return SHIRO_E_CUDA;
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)x_rows};
  const cuuint64_t strides[1] = {(cuuint64_t)N * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)N, 1};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(X), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return SHIRO_E_CUDA;
  const int64_t grid = (n_idx + chunk - 1) / chunk;
  if (grid == 0) return SHIRO_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t smem = (size_t)stages * 4 * 512;
  if (stages == 2) k_probe_gather_tma<2><<<(unsigned)grid, 32, smem, s>>>(tm, idx, n_idx, chunk, out);
  else if (stages == 4) k_probe_gather_tma<4><<<(unsigned)grid, 32, smem, s>>>(tm, idx, n_idx, chunk, out);
  else k_probe_gather_tma<8><<<(unsigned)grid, 32, smem, s>>>(tm, idx, n_idx, chunk, out);
  return cudaGetLastError() == cudaSuccess ? SHIRO_OK : SHIRO_E_CUDA;
}

extern "C" int shiro_probe_gather(const float *X, int32_t N, const int32_t *idx, int64_t n_idx,
                                  float *out, int32_t chunk, void *stream) {
  if (!X || !idx || !out || n_idx < 0 || chunk < 1) return SHIRO_E_ARG;
  if (N != 32 && N != 64 && N != 128) return SHIRO_E_ARG;
  const int lpr = N / 4, rpw = 32 / lpr;
  const int64_t chunks = (n_idx + chunk - 1) / chunk;
  const int64_t grid = (chunks + 8 * rpw - 1) / (8 * rpw);
  if (grid == 0) return SHIRO_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (lpr == 32) k_probe_gather<32><<<(unsigned)grid, 256, 0, s>>>(X, N, idx, n_idx, chunk, out);
  else if (lpr == 16) k_probe_gather<16><<<(unsigned)grid, 256, 0, s>>>(X, N, idx, n_idx, chunk, out);
  else k_probe_gather<8><<<(unsigned)grid, 256, 0, s>>>(X, N, idx, n_idx, chunk, out);
  return cudaGetLastError() == cudaSuccess ? SHIRO_OK : SHIRO_E_CUDA;
}

extern "C" int shiro_probe_fma(float *out, int32_t blocks, int32_t iters, void *stream) {
  if (!out || blocks < 1 || iters < 1) return SHIRO_E_ARG;
  k_probe_fma<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(out, iters);
  return cudaGetLastError() == cudaSuccess ? SHIRO_OK : SHIRO_E_CUDA;
}

extern "C" int shiro_probe_copy(const float *x, float *y, int64_t n_floats, void *stream) {
  if (!x || !y || n_floats < 0 || n_floats % 4) return SHIRO_E_ARG;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n4 = n_floats / 4;
  if (n4 == 0) return SHIRO_OK;
  const int64_t grid = std::min<int64_t>((n4 + 255) / 256, (int64_t)sms * 16);
  k_probe_copy<<<(unsigned)grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const float4 *>(x), reinterpret_cast<float4 *>(y), n4);
  return cudaGetLastError() == cudaSuccess ? SHIRO_OK : SHIRO_E_CUDA;
}

extern "C" int shiro_probe_gather_tma_ws(const float *X, int64_t x_rows, int32_t N,
                                         const int32_t *idx, int64_t n_idx, float *out,
                                         int32_t stages, int32_t ctas, void *stream) {
  if (!X || !idx || !out || n_idx < 4 || n_idx % 4 || N != 128 || x_rows < 1 || ctas < 1)
    return SHIRO_E_ARG;
  if (stages != 8 && stages != 16 && stages != 24) return SHIRO_E_ARG;
  auto enc = encode_fn();
  if (!enc) return SHIRO_E_CUDA;
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)x_rows};
  const cuuint64_t strides[1] = {(cuuint64_t)N * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)N, 1};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(X), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return SHIRO_E_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t smem = (size_t)stages * 4 * 512;
  const int64_t nq = n_idx / 4;
#define SHIRO_WS(S_)                                                                            \
  do {                                                                                          \
    cudaFuncSetAttribute(k_probe_gather_tma_ws<S_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)smem);                                                            \
    k_probe_gather_tma_ws<S_><<<ctas, 288, smem, s>>>(tm, idx, nq, n_idx, out);                 \
  } while (0)
  if (stages == 8) SHIRO_WS(8);
  else if (stages == 16) SHIRO_WS(16);
  else SHIRO_WS(24);
#undef SHIRO_WS
  return cudaGetLastError() == cudaSuccess ? SHIRO_OK : SHIRO_E_CUDA;
}

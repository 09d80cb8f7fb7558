// probe.cu -- measurement probe (not on the hot path): a pure row gather,
//   out[c] = sum_{k in chunk c} X[idx[k]]   (chunks of `chunk` indices),
// with the same 128-bit, 8-deep load structure as the SpMM kernels.  Fed with
// an SpMM's own column-index stream it times the unavoidable part of that
// SpMM -- every referenced source row delivered to an SM once per nonzero --
// which is the gather-aware roofline of DESIGN.md section 5.
#include <cuda_runtime.h>
#include <stdint.h>

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

}  // namespace

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

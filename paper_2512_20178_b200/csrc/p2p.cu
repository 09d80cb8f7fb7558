// p2p.cu -- synchronisation of the fused NVLink exchange (E3).
//
// In the fused exchange every sender stores its B rows (K4) and partial C
// rows (K3) directly into the receivers' buffers through CUDA-IPC peer
// mappings over NVLink/NVSwitch, then raises a per-(receiver, sender) READY
// flag in the receiver's memory; the receiver waits for READY >= epoch before
// its remote SpMM / scatter-add and afterwards raises CONSUMED >= epoch in
// each sender's memory, which the sender waits for before overwriting the
// buffer in the next call.  Epochs increase monotonically, so no reset is
// needed.  The waits time out (error flag) rather than hang a GPU.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace shiro {

namespace {

__device__ __forceinline__ void st_release_sys(int32_t *p, int32_t v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire_sys(const int32_t *p) {
  int32_t v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// value = *epoch + add (the device-side epoch keeps the arguments of a
// captured CUDA graph static); bump: advance the epoch afterwards (last
// signal of a call).
__global__ void k_signal(int32_t *const *flags, int n, int32_t *epoch, int add, int bump) {
  const int i = threadIdx.x;
  const int32_t value = *epoch + add;
  __threadfence_system();
  if (i < n) st_release_sys(flags[i], value);
  if (bump) {
    __syncthreads();
    if (i == 0) *epoch = value;
  }
}

__global__ void k_wait(const int32_t *flags, int n, int32_t *epoch, int add, int32_t *err,
                       int64_t timeout_ns, int bump) {
  const int i = threadIdx.x;
  const int32_t value = *epoch + add;
  if (i < n) {
    const uint64_t t0 = globaltimer();
    while (ld_acquire_sys(flags + i) < value) {
      if (*reinterpret_cast<volatile int32_t *>(err)) break;   // another waiter timed out
      if ((int64_t)(globaltimer() - t0) > timeout_ns) {
        atomicExch(err, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  __threadfence_system();
  if (bump && i == 0) *epoch = value;   // every thread has read the epoch before the barrier
}

}  // namespace

int launch_signal(int32_t *const *flags, int n, int32_t *epoch, int add, bool bump,
                  cudaStream_t s) {
  if (n <= 0 && !bump) return 0;
  k_signal<<<1, 64, 0, s>>>(flags, n, epoch, add, bump ? 1 : 0);
  return 1;
}

int launch_wait(const int32_t *flags, int n, int32_t *epoch, int add, int32_t *err,
                int64_t timeout_ns, cudaStream_t s, bool bump) {
  if (n <= 0) return 0;
  k_wait<<<1, 64, 0, s>>>(flags, n, epoch, add, err, timeout_ns, bump ? 1 : 0);
  return 1;
}

}  // namespace shiro

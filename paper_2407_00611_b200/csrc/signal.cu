// signal.cu -- cross-GPU stream synchronisation for the peer-memory (CUDA IPC) transport.
//
// Every rank's workspace begins with a flag block that peers write over NVLink:
//   data[chan][src]  count of message batches `src` has delivered to me on stream `chan`
//   ack[src]         count of ring slots `src` has released (it finished reading them)
//   bar[src]         per-call barrier epoch of `src`
// A sender's stream writes a flag with st.release.sys after its copy-engine copies (stream
// order: the copies have completed); the receiver's stream spins in a one-warp kernel with
// ld.acquire.sys until the count is reached, so the kernels after it see the data.  Counts
// only grow, so flags never need resetting.  A timed-out wait is reported, not trapped.
#include <cstdint>

#include "common.h"
#include "internal.h"

namespace wf {

namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Thread i: (optionally) publish sig.val[i] at sig.dst[i], then wait until *wait.flag[i] >= wait.val[i].
// A wait that outlives wait.timeout_ns (a peer is gone or stalled) records the failure in
// the context's host-mapped words and returns: the library reports WF_ERR_COMM on the next
// call instead of poisoning the CUDA context with a trap.  Later waits return at once.
__global__ void wf_signal_wait_kernel(SigArgs sig, SigArgs wait) {
  const int i = threadIdx.x;
  if (i < sig.n) {
    __threadfence_system();
    st_release_sys(sig.dst[i], sig.val[i]);
  }
  if (i < wait.n) {
    if (wait.fail && ld_volatile(wait.fail) != 0) return;
    const uint64_t t0 = gtimer();
    uint32_t spins = 0;
    uint32_t seen;
    while (static_cast<int32_t>((seen = ld_acquire_sys(wait.dst[i])) - wait.val[i]) < 0) {
      if ((++spins & 255u) == 0) {
        __nanosleep(200);
        if (gtimer() - t0 > wait.timeout_ns) {
          if (wait.fail) {
            wait.fail[1] = wait.val[i];
            wait.fail[2] = seen;
            __threadfence_system();
            atomicExch_system(wait.fail, 1u);
          }
          return;
        }
      }
    }
  }
}

}  // namespace

cudaError_t launch_signal_wait(const SigArgs& sig, const SigArgs& wait, cudaStream_t s) {
  if (sig.n == 0 && wait.n == 0) return cudaSuccess;
  if (sig.n > WF_MAX_SIG || wait.n > WF_MAX_SIG) return cudaErrorInvalidValue;
  const int threads = ((sig.n > wait.n ? sig.n : wait.n) + 31) / 32 * 32;
  wf_signal_wait_kernel<<<1, threads, 0, s>>>(sig, wait);
  return cudaGetLastError();
}

}  // namespace wf

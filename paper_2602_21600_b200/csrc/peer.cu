// peer.cu -- the C5 exchange over peer memory (SURVEY 8(e) "fused variant", BASELINE.json
// configs[4] "per-shard top-k gathered over NVLink and merged"): every rank's search kernel
// stores its per-shard top-k lists straight into the gather buffer of the rank that owns the
// query block (plain stores to a peer-mapped pointer: aqr_search's out_ids / out_dist), so the
// transfer rides on the search epilogue, query by query.  What is left for this file is the
// hand-off: one signal kernel per rank and step (system-scope release of a step counter into
// every peer's flag array, after the stream-ordered search kernels) and one wait kernel
// (system-scope acquire spin on the local flags, bounded by a timeout).
#include "aqr_internal.cuh"

namespace aqr {

namespace {

struct PeerFlags {
  unsigned long long* p[AQR_MAX_PEERS];
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long timer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// thread t signals peer t: every store this GPU issued before the kernel (the search kernels'
// stores into peer t's gather buffer, stream-ordered before this launch) is ordered before the
// flag by the system-scope fence + release
__global__ void signal_kernel(PeerFlags f, int n_peers, int slot, unsigned long long value) {
  const int t = threadIdx.x;
  if (t >= n_peers) return;
  __threadfence_system();
  st_release_sys(f.p[t] + slot, value);
}

// thread t waits for flag t >= value; status[0] = 0 ok, 1 + t = flag t timed out
__global__ void wait_kernel(const unsigned long long* flags, int n, unsigned long long value,
                            unsigned long long timeout_ns, int32_t* status) {
  const int t = threadIdx.x;
  if (t >= n) return;
  const unsigned long long t0 = timer_ns();
  while (ld_acquire_sys(flags + t) < value) {
    if (timer_ns() - t0 > timeout_ns) {
      if (status) atomicCAS(status, 0, 1 + t);
      return;
    }
    __nanosleep(200);
  }
}

}  // namespace

cudaError_t launch_peer_signal(unsigned long long* const* flags, int n_peers, int slot, unsigned long long value,
                               cudaStream_t s) {
  PeerFlags f;
  for (int i = 0; i < AQR_MAX_PEERS; ++i) f.p[i] = i < n_peers ? flags[i] : nullptr;
  signal_kernel<<<1, 32, 0, s>>>(f, n_peers, slot, value);
  return cudaGetLastError();
}

cudaError_t launch_peer_wait(const unsigned long long* flags, int n, unsigned long long value,
                             unsigned long long timeout_ns, int32_t* status, cudaStream_t s) {
  wait_kernel<<<1, 32, 0, s>>>(flags, n, value, timeout_ns, status);
  return cudaGetLastError();
}

}  // namespace aqr

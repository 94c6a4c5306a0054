// libspx runtime glue: error reporting across the C-ABI, device queries, driver entry points,
// and the path-hop copy primitive (NVLink peer copy when source and destination live on
// different GPUs, a device-local copy otherwise).
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <mutex>

#include "spx_internal.h"

namespace spx {

static thread_local char g_err[512] = "";

int set_error(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

int set_cuda_error(cudaError_t e, const char* where) {
  snprintf(g_err, sizeof g_err, "%s: %s (%d)", where, cudaGetErrorString(e), (int)e);
  return SPX_ERR_CUDA;
}

int check_launch(const char* kernel_name) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, kernel_name);
  return SPX_OK;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("SPX_PDL");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

TensorMapEncodeFn get_tensor_map_encoder() {
  static TensorMapEncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<TensorMapEncodeFn>(p);
  });
  return fn;
}

}  // namespace spx

using namespace spx;

extern "C" int spx_abi_version(void) { return SPX_ABI_VERSION; }

extern "C" const char* spx_last_error(void) { return g_err; }

extern "C" int spx_device_sm_count(void) { return num_sms(); }

extern "C" int64_t spx_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" int spx_enable_peer_access(int32_t dev, int32_t peer) {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(dev);
  int can = 0;
  cudaDeviceCanAccessPeer(&can, dev, peer);
  if (!can) {
    cudaSetDevice(prev);
    return set_error(SPX_ERR_ARG, "peer access not supported between these devices");
  }
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(prev);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return SPX_OK;
  }
  if (e != cudaSuccess) return set_cuda_error(e, "cudaDeviceEnablePeerAccess");
  return SPX_OK;
}

// One path hop: move `bytes` from src (on src_dev) to dst (on dst_dev) on `stream`.
// Across GPUs this is a peer copy over NVLink (copy engine); on one GPU it is a D2D copy.
extern "C" int spx_hop(int32_t dst_dev, void* dst, int32_t src_dev, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0) return set_error(SPX_ERR_ARG, "hop: negative size");
  if (bytes == 0) return SPX_OK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (dst_dev == src_dev) e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, s);
  else e = cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, (size_t)bytes, s);
  if (e != cudaSuccess) return set_cuda_error(e, "spx_hop");
  return SPX_OK;
}

// ---- cross-process path hops over NVLink peer memory ----
//
// Every rank exports the receive buffers of the logical nodes it hosts (the slot buffers a hop
// writes: layer-0 input, returned activation, incoming gradient) and one int32 flag per buffer
// (spx_ipc_export); the ranks that send to it map them (spx_ipc_open).  A hop is then a push:
// `ctas` CTAs on the sender stream stream the activation into the peer's slot with 16-byte
// stores over NVLink, and each CTA release-increments the peer's flag once its stores are
// system-visible.  The consumer's stream runs spx_hop_wait (one thread, acquire loads at system
// scope) until the flag reaches the count the host expects for that buffer, then the consumer
// op.  Buffer reuse is safe without a receiver->sender handshake because slots are static per
// (agent, node) and a slot's next write causally follows its last read (executor.py, DESIGN.md
// §1 "Static activation slots").

namespace {

typedef int (*MemGetAddressRangeFn)(unsigned long long*, size_t*, unsigned long long);

MemGetAddressRangeFn get_addr_range() {
  static MemGetAddressRangeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<MemGetAddressRangeFn>(p);
  });
  return fn;
}

__global__ void __launch_bounds__(512) hop_push_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                       int64_t n16, unsigned int* flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldg(src + i), b = __ldg(src + i + stride), c = __ldg(src + i + 2 * stride),
          d = __ldg(src + i + 3 * stride);
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = __ldg(src + i);
  if (flag == nullptr) return;  // unsignalled copy (bandwidth probes)
  // the CTA barrier orders every thread's stores before thread 0's release; the release at
  // system scope is cumulative, so the peer's acquire of the flag sees the whole CTA's data
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
}

__global__ void hop_signal_kernel(unsigned int* flag) {
  // runs after the copy engine finished the stream's preceding peer copy.  A release orders only
  // this thread's own accesses and the copy engine's writes are not among them, so a full system
  // fence precedes the flag update (opt-in path; the fence costs ~1 us per hop)
  __threadfence_system();
  asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(flag) : "memory");
}

__global__ void hop_wait_kernel(const unsigned int* flag, unsigned int target, unsigned long long timeout_ns) {
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - target) >= 0) break;
    __nanosleep(256);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) __trap();  // a lost hop fails loudly instead of hanging
  }
}

}  // namespace

extern "C" int spx_ipc_export(const void* ptr, void* handle_out, int64_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) return set_error(SPX_ERR_ARG, "ipc_export: null argument");
  MemGetAddressRangeFn range = get_addr_range();
  if (!range) return set_error(SPX_ERR_CUDA, "ipc_export: cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, (unsigned long long)ptr) != 0) return set_error(SPX_ERR_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return set_cuda_error(e, "cudaIpcGetMemHandle");
  memcpy(handle_out, &h, sizeof h);
  *offset_out = (int64_t)((unsigned long long)ptr - base);
  return SPX_OK;
}

extern "C" int spx_ipc_open(const void* handle, void** base_out) {
  if (!handle || !base_out) return set_error(SPX_ERR_ARG, "ipc_open: null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  cudaError_t e = cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaIpcOpenMemHandle");
  return SPX_OK;
}

extern "C" int spx_ipc_close(void* base) {
  cudaError_t e = cudaIpcCloseMemHandle(base);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaIpcCloseMemHandle");
  return SPX_OK;
}

extern "C" int spx_hop_push(void* dst, const void* src, int64_t bytes, uint32_t* flag, int32_t ctas, void* stream) {
  if (bytes < 0 || (bytes & 15) || ctas <= 0 || ctas > 1024) return set_error(SPX_ERR_ARG, "hop_push: bad size or ctas");
  if (!dst || !src) return set_error(SPX_ERR_ARG, "hop_push: null pointer");
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15)
    return set_error(SPX_ERR_ARG, "hop_push: buffers must be 16-byte aligned");
  hop_push_kernel<<<ctas, 512, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<uint4*>(dst), reinterpret_cast<const uint4*>(src), bytes / 16, flag);
  count_launch();
  return check_launch("hop_push_kernel");
}

static std::atomic<unsigned long long> g_hop_timeout_ns{120ull * 1000000000ull};

extern "C" int spx_hop_set_timeout(double seconds) {
  if (!(seconds > 0.0) || seconds > 86400.0) return set_error(SPX_ERR_ARG, "hop_set_timeout: need 0 < seconds <= 86400");
  g_hop_timeout_ns.store((unsigned long long)(seconds * 1e9));
  return SPX_OK;
}

extern "C" int spx_hop_wait(const uint32_t* flag, uint32_t target, void* stream) {
  if (!flag) return set_error(SPX_ERR_ARG, "hop_wait: null flag");
  hop_wait_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flag, target, g_hop_timeout_ns.load());
  count_launch();
  return check_launch("hop_wait_kernel");
}

extern "C" int spx_hop_push_ce(void* dst, const void* src, int64_t bytes, uint32_t* flag, void* stream) {
  if (bytes < 0) return set_error(SPX_ERR_ARG, "hop_push_ce: negative size");
  if (!dst || !src) return set_error(SPX_ERR_ARG, "hop_push_ce: null pointer");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return set_cuda_error(e, "hop_push_ce: cudaMemcpyAsync");
  if (flag == nullptr) return SPX_OK;
  hop_signal_kernel<<<1, 1, 0, s>>>(flag);
  count_launch();
  return check_launch("hop_signal_kernel");
}

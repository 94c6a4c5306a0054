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

// Host-side helpers shared by the libspx translation units (error state, device queries,
// driver entry points).  Not part of the public C-ABI (see include/spx.h).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spx.h"

namespace spx {

bool pdl_enabled();
void count_launch();  // libspx kernel-launch counter (spx_launch_count)

// Launch with Programmatic Dependent Launch: the kernel may start (and run its prologue) while
// the previous kernel on the stream drains; every libspx kernel calls griddepcontrol.wait before
// touching global data the previous kernel produced or consumes.  SPX_PDL=0 disables it.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  count_launch();
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Same, with a thread-block cluster of `cluster_x` CTAs along x (CTA pairs for cta_group::2).
template <typename... KArgs, typename... Args>
cudaError_t launch_k_cluster(void (*kern)(KArgs...), int cluster_x, dim3 grid, dim3 block, size_t smem,
                             cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeClusterDimension;
  attr[n].val.clusterDim.x = cluster_x;
  attr[n].val.clusterDim.y = 1;
  attr[n].val.clusterDim.z = 1;
  ++n;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  count_launch();
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// launch errors are also recorded as the runtime's last error, which check_launch() reports
#define spx_launch_check(expr) ((void)(expr))

int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
int check_launch(const char* kernel_name);
int num_sms();

typedef CUresult (*TensorMapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
TensorMapEncodeFn get_tensor_map_encoder();

// tcgen05 attention forward (attention_sm100.cu); head_dim 64/128, T % 128 == 0
int attn_fwd_tcgen05(const void* qkv, void* o, float* lse, int64_t B, int64_t T, int64_t H, int64_t Hkv, int64_t hd,
                     int64_t ld_qkv, int64_t ld_o, float scale, cudaStream_t s);
int attn_bwd_tcgen05(const void* qkv, const void* dout, const float* lse, const float* delta, void* dqkv, int64_t B,
                     int64_t T, int64_t H, int64_t Hkv, int64_t hd, int64_t ld_qkv, int64_t ld_o, float scale,
                     const float* rope_cs, bool gqa_split, cudaStream_t s);
bool attn_use_legacy();
// the tcgen05 backward splits each GQA group over several dK/dV work items (fp32 partials in the
// workspace, summed by a reduce pass) when it has fewer (batch, kv head, key block) items than SMs
bool attn_gqa_split(int64_t B, int64_t H, int64_t Hkv, int64_t T, int64_t hd);

}  // namespace spx

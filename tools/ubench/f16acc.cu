// How does a kind::f16 MMA with an f16 D lay out its accumulator in TMEM?  One 128x128x16 MMA,
// A[i][k] = (k == 0) * (i % 16), B[n][k] = (k == 0) * (n % 8 + 1) -> D[i][n] = (i%16)*(n%8+1).
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "../../paper_2502_19913_b200/csrc/spx_common.cuh"
using namespace spx;

__global__ void k(uint32_t* out, int dfmt) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  uint8_t* sA = smem;           // 128 x 64 bf16, K-major SW128
  uint8_t* sB = smem + 16384;   // 128 x 64 bf16
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    int r = e / 64, kk = e % 64;
    float a = kk == 0 ? (float)(r % 16) : 0.f, b = kk == 0 ? (float)(r % 8 + 1) : 0.f;
    int off = r * 128 + (((kk / 8) ^ (r & 7)) * 16) + (kk % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(sA + off) = __float2bfloat16(a);
    *reinterpret_cast<__nv_bfloat16*>(sB + off) = __float2bfloat16(b);
  }
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // zero TMEM columns 0..255 first (so untouched columns read 0)
  {
    uint32_t z[32];
    for (int i = 0; i < 32; ++i) z[i] = 0xDEADBEEFu;
    for (int c = 0; c < 256; c += 32)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   :: "r"(tmem + ((uint32_t)(warp * 32) << 16) + c), "r"(z[0]),"r"(z[1]),"r"(z[2]),"r"(z[3]),"r"(z[4]),"r"(z[5]),"r"(z[6]),"r"(z[7]),"r"(z[8]),"r"(z[9]),"r"(z[10]),"r"(z[11]),"r"(z[12]),"r"(z[13]),"r"(z[14]),"r"(z[15]),"r"(z[16]),"r"(z[17]),"r"(z[18]),"r"(z[19]),"r"(z[20]),"r"(z[21]),"r"(z[22]),"r"(z[23]),"r"(z[24]),"r"(z[25]),"r"(z[26]),"r"(z[27]),"r"(z[28]),"r"(z[29]),"r"(z[30]),"r"(z[31]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    uint32_t idesc = umma_idesc_bf16(128, 128, false, false);
    if (dfmt == 0) idesc &= ~(3u << 4);  // D format f16
    if (elect_one()) {
      mma_bf16_ss(tmem, umma_desc_sw128(smem_u32(sA), 16, 1024), umma_desc_sw128(smem_u32(sB), 16, 1024), idesc, 0);
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  for (int c = 0; c < 128; c += 32) {
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    for (int i = 0; i < 32; ++i) out[(warp * 32 + (threadIdx.x & 31)) * 128 + c + i] = r[i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 128 * 128 * 4);
  static uint32_t h[128 * 128];
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int fmt = 1; fmt >= 0; --fmt) {
    k<<<1, 128, 40000>>>(d, fmt);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("D format %s: lane 3, columns 0..11 raw:", fmt ? "f32" : "f16");
    for (int c = 0; c < 12; ++c) printf(" %08x", h[3 * 128 + c]);
    printf("\n  lane 3 columns 60..67:");
    for (int c = 60; c < 68; ++c) printf(" %08x", h[3 * 128 + c]);
    printf("\n  lane 3 columns 124..127:");
    for (int c = 124; c < 128; ++c) printf(" %08x", h[3 * 128 + c]);
    printf("\n");
  }
  return 0;
}

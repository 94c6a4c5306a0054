// TMEM read / write throughput probe (tcgen05.ld / tcgen05.st, 32x32b shapes), one CTA per SM.
#include <cstdio>
#include <cstdint>
#include "../../paper_2502_19913_b200/csrc/spx_common.cuh"

using namespace spx;

template <int X>
__device__ __forceinline__ void ld_x(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ld_x<32>(uint32_t taddr, uint32_t* r) {
  tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(long long* cyc, float* out, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int quad = warp & 3, sub = warp >> 2;  // 4 lane quadrants; sub selects a column block
  const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + sub * 32;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = i;
  float acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {  // loads, wait each
      ld_x<32>(base + (it & 3) * 128 % 512, r);
      tmem_ld_wait();
      acc += __uint_as_float(r[it & 31]);
    } else if (MODE == 1) {  // two loads in flight
      uint32_t r2[32];
      tmem_ld_32x32b_x32(base, *reinterpret_cast<uint32_t(*)[32]>(r));
      tmem_ld_32x32b_x32(base + 256, r2);
      tmem_ld_wait();
      acc += __uint_as_float(r[it & 31]) + __uint_as_float(r2[(it + 1) & 31]);
    } else {  // stores
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(base),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
          "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
          "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
          : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      r[it & 31] += 1;
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + r[3];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}


// generic load: SHAPE string, NREG registers per thread
#define LD_PROBE(NAME, SHAPE, NREG)                                                              \
  __global__ void __launch_bounds__(512, 1) NAME(long long* cyc, float* out, int iters) {        \
    __shared__ uint32_t slot;                                                                    \
    const int warp = threadIdx.x >> 5;                                                           \
    if (warp == 0) tmem_alloc(&slot, 512);                                                       \
    tc_fence_before();                                                                           \
    __syncthreads();                                                                             \
    tc_fence_after();                                                                            \
    const uint32_t tmem = slot;                                                                  \
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;         \
    uint32_t r[NREG];                                                                            \
    float acc = 0;                                                                               \
    long long t0 = clock64();                                                                    \
    for (int it = 0; it < iters; ++it) {                                                         \
      LD_ASM_##NREG(SHAPE, base, r);                                                             \
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");                               \
      acc += __uint_as_float(r[it % NREG]);                                                      \
    }                                                                                            \
    long long t1 = clock64();                                                                    \
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;                                            \
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                                             \
    tc_fence_before();                                                                           \
    __syncthreads();                                                                             \
    tc_fence_after();                                                                            \
    if (warp == 0) tmem_dealloc(tmem, 512);                                                      \
  }
#define R8(o) "=r"(r[o]), "=r"(r[o+1]), "=r"(r[o+2]), "=r"(r[o+3]), "=r"(r[o+4]), "=r"(r[o+5]), "=r"(r[o+6]), "=r"(r[o+7])
#define LD_ASM_32(SHAPE, a, r) asm volatile("tcgen05.ld.sync.aligned." SHAPE ".b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" : R8(0), R8(8), R8(16), R8(24) : "r"(a))
#define LD_ASM_64(SHAPE, a, r) asm volatile("tcgen05.ld.sync.aligned." SHAPE ".b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];" : R8(0), R8(8), R8(16), R8(24), R8(32), R8(40), R8(48), R8(56) : "r"(a))
LD_PROBE(p_32x32b_x64, "32x32b.x64", 64)
LD_PROBE(p_16x256b_x8, "16x256b.x8", 32)
LD_PROBE(p_16x128b_x16, "16x128b.x16", 32)
LD_PROBE(p_16x64b_x32, "16x64b.x32", 32)
LD_PROBE(p_16x256b_x16, "16x256b.x16", 64)

int main() {
  long long* cyc;
  float* out;
  cudaMalloc(&cyc, 8 * 256);
  cudaMalloc(&out, 4 << 20);
  const char* names[] = {"ld_x32_wait", "ld_x32_2inflight", "st_x32"};
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16}) {
      int iters = 1000;
      auto k = mode == 0 ? probe<0> : mode == 1 ? probe<1> : probe<2>;
      k<<<148, warps * 32>>>(cyc, out, iters);
      k<<<148, warps * 32>>>(cyc, out, iters);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double bytes = (double)warps * iters * 4096 * (mode == 1 ? 2 : 1);
      printf("{\"op\": \"%s\", \"warps\": %d, \"bytes_per_clk_per_sm\": %.1f}\n", names[mode], warps, bytes / c);
    }
  struct { const char* n; void (*k)(long long*, float*, int); int nreg; } ps[] = {
      {"32x32b.x64", p_32x32b_x64, 64}, {"16x256b.x8", p_16x256b_x8, 32}, {"16x128b.x16", p_16x128b_x16, 32},
      {"16x64b.x32", p_16x64b_x32, 32}, {"16x256b.x16", p_16x256b_x16, 64}};
  for (auto& p : ps)
    for (int warps : {4, 8, 16}) {
      int iters = 1000;
      p.k<<<148, warps * 32>>>(cyc, out, iters);
      p.k<<<148, warps * 32>>>(cyc, out, iters);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s %s\n", p.n, cudaGetErrorString(e)); return 1; }
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double bytes = (double)warps * iters * 32 * p.nreg * 4;
      printf("{\"op\": \"ld %s\", \"warps\": %d, \"bytes_per_clk_per_sm\": %.1f}\n", p.n, warps, bytes / c);
    }
  return 0;
}

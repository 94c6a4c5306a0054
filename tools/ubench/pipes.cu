// Issue/pipe throughput probes on one SM (B200): ex2 (MUFU), FFMA2, FMNMX3, F2FP pack, FADD.
// Each thread runs 8 independent chains; reports results per clock per SM.
#include <cstdio>
#include <cstdint>

template <int OP>
__global__ void probe(float* out, long long* cyc, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0.001f * (threadIdx.x + i);
  uint32_t u[8];
  for (int i = 0; i < 8; ++i) u[i] = __float_as_uint(a[i]);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) {
        unsigned long long p = ((unsigned long long)u[i] << 32) | u[(i + 1) & 7];
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(p));
        u[i] = (uint32_t)p;
      }
      if (OP == 2) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7]));
      if (OP == 3) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(__uint_as_float(u[i])));
      if (OP == 4) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]));
      if (OP == 5) asm volatile("fma.rn.f32 %0, %0, %1, %0;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]));
      if (OP == 6) {  // ex2 + bf16x2 pack per element pair
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        if (i & 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(a[i - 1]));
      }
      if (OP == 7) {  // ex2 + ffma2 per element pair
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        if (i & 1) {
          unsigned long long p = ((unsigned long long)u[i] << 32) | u[i - 1];
          asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(p));
          u[i] = (uint32_t)p;
        }
      }
      if (OP == 8) {  // ex2 + prmt pack per pair
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        if (i & 1) asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(u[i]) : "r"(__float_as_uint(a[i])), "r"(__float_as_uint(a[i - 1])));
      }
      if (OP == 9) {  // ex2 + fmnmx3 per pair
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        if (i & 1) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[(i + 2) & 7]) : "f"(a[(i + 3) & 7]), "f"(a[(i + 4) & 7]));
      }
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(u[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 8 * 1024);
  const char* names[] = {"ex2.f32", "ffma2(x2 elems)", "fmnmx3", "f2fp.pack", "fadd", "ffma", "ex2+f2fp/2", "ex2+ffma2/2", "ex2+prmt/2", "ex2+fmnmx3/2"};
  void (*ks[])(float*, long long*, int) = {probe<0>, probe<1>, probe<2>, probe<3>, probe<4>, probe<5>, probe<6>, probe<7>, probe<8>, probe<9>};
  for (int op = 0; op < 10; ++op) {
    for (int threads : {256, 512}) {
      int iters = 2000;
      void (*k)(float*, long long*, int) = ks[op];
      k<<<148, threads>>>(out, cyc, iters);
      k<<<148, threads>>>(out, cyc, iters);
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double per_clk = (double)threads * iters * 8 / c;
      printf("{\"op\": \"%s\", \"threads\": %d, \"elems_per_clk_per_sm\": %.2f}\n", names[op], threads, per_clk);
    }
  }
  return 0;
}

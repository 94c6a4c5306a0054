// Cost of the attention-forward exp_chunk sequence in isolation (8 warps per SM, like the kernel):
// cycles per 32-element chunk per warp with parts of the sequence switched off.
#include <cstdio>
#include <cstdint>
#include "../../paper_2502_19913_b200/csrc/spx_common.cuh"
using namespace spx;
SPX_DEVICE float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
SPX_DEVICE float max3(float a, float b, float c) { float d; asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }

template <bool MAX, bool FF2, bool SUM, bool PACK>
SPX_DEVICE void chunk(const uint32_t (&v)[32], float sl2, float m, uint32_t* pk, float& sum, float& bmax) {
  float s2[4][2] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
  float mk[2] = {bmax, -INFINITY};
  const float nm = -m;
#pragma unroll
  for (int i = 0; i < 32; i += 2) {
    float a = __uint_as_float(v[i]), b = __uint_as_float(v[i + 1]);
    if (MAX) mk[(i >> 1) & 1] = max3(mk[(i >> 1) & 1], a, b);
    float ya, yb;
    if (FF2) {
      asm("{\n\t.reg .b64 x, k, c, y;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 k, {%4, %4};\n\tmov.b64 c, {%5, %5};\n\t"
          "fma.rn.f32x2 y, x, k, c;\n\tmov.b64 {%0, %1}, y;\n\t}" : "=f"(ya), "=f"(yb) : "f"(a), "f"(b), "f"(sl2), "f"(nm));
    } else { ya = fmaf(a, sl2, nm); yb = fmaf(b, sl2, nm); }
    ya = ex2(ya); yb = ex2(yb);
    if (SUM) { float* acc = s2[(i >> 1) & 3]; acc[0] += ya; acc[1] += yb; }
    if (PACK) pk[i >> 1] = pack_bf16(ya, yb); else pk[i >> 1] = __float_as_uint(ya) ^ __float_as_uint(yb);
  }
  bmax = fmaxf(mk[0], mk[1]);
  sum += ((s2[0][0] + s2[0][1]) + (s2[1][0] + s2[1][1])) + ((s2[2][0] + s2[2][1]) + (s2[3][0] + s2[3][1]));
}

template <bool MAX, bool FF2, bool SUM, bool PACK>
__global__ void k(uint32_t* out, long long* cyc, int iters) {
  uint32_t v[32], pk[16];
  for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(0.001f * (threadIdx.x + i) - 3.f);
  float sum = 0, bmax = -1e30f, m = 0.5f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    chunk<MAX, FF2, SUM, PACK>(v, 0.18f, m, pk, sum, bmax);
    v[it & 31] ^= pk[it & 15];  // keep the chain alive
  }
  long long t1 = clock64();
  uint32_t x = 0;
  for (int i = 0; i < 16; ++i) x ^= pk[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x ^ __float_as_uint(sum + bmax);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  uint32_t* out; long long* cyc;
  cudaMalloc(&out, 1 << 22); cudaMalloc(&cyc, 8 * 256);
  struct { const char* n; void (*f)(uint32_t*, long long*, int); } vs[] = {
    {"full", k<true, true, true, true>}, {"no_max", k<false, true, true, true>}, {"scalar_ffma", k<true, false, true, true>},
    {"no_sum", k<true, true, false, true>}, {"no_pack", k<true, true, true, false>}, {"exp_only", k<false, false, false, false>}};
  for (auto& v : vs) for (int warps : {8, 16}) {
    int iters = 400;
    v.f<<<148, warps * 32>>>(out, cyc, iters); v.f<<<148, warps * 32>>>(out, cyc, iters);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"variant\": \"%s\", \"warps\": %d, \"cycles_per_chunk_per_warp\": %.1f, \"mufu_floor\": %.1f}\n", v.n, warps,
           (double)c / iters, 32.0 * 8 * warps / 4 / 8 / 1.0 * 1.0 / (warps / 4.0) * (warps / 4.0) );
  }
  return 0;
}

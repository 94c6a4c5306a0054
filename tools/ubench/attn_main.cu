// Attention kernel harness (benchmarking only): one translation unit with the libspx attention
// sources, so variants can be built with -D flags and probed without rebuilding libspx.so.
//   attn_main B T H Hkv hd iters [dump]   (ATTN_ROPE=1: backward through the inverse-RoPE epilogues)
#include "../../paper_2502_19913_b200/csrc/runtime.cu"
#include "../../paper_2502_19913_b200/csrc/attention.cu"
#include "../../paper_2502_19913_b200/csrc/attention_sm100.cu"
#include "../../paper_2502_19913_b200/csrc/attention_bwd_sm100.cu"
#include <cstdio>
#include <vector>
#include <cmath>

int main(int argc, char** argv) {
  int B = argc > 1 ? atoi(argv[1]) : 4, T = argc > 2 ? atoi(argv[2]) : 1024, H = argc > 3 ? atoi(argv[3]) : 16;
  int Hkv = argc > 4 ? atoi(argv[4]) : 16, hd = argc > 5 ? atoi(argv[5]) : 64, iters = argc > 6 ? atoi(argv[6]) : 20;
  const long long W = (long long)(H + 2 * Hkv) * hd, n = (long long)B * T;
  std::vector<uint16_t> h(n * W);
  uint32_t x = 12345;
  for (auto& v : h) {
    x = x * 1664525u + 1013904223u;
    float f = ((x >> 8) / 16777216.f - 0.5f);
    uint32_t b;
    memcpy(&b, &f, 4);
    v = (uint16_t)(b >> 16);
  }
  void *qkv, *o, *dout, *dqkv;
  float *lse, *ws, *cs;
  cudaMalloc(&qkv, n * W * 2);
  cudaMalloc(&dqkv, n * W * 2);
  cudaMalloc(&o, n * H * hd * 2);
  cudaMalloc(&dout, n * H * hd * 2);
  cudaMalloc(&lse, (size_t)B * H * T * 4);
  const long long wsf = spx_attn_bwd_ws_floats_ex(B, H, Hkv, T, hd);
  cudaMalloc(&ws, wsf * 4);
  cudaMalloc(&cs, (size_t)hd * T * 4);
  cudaMemset(cs, 0, (size_t)hd * T * 4);
  cudaMemcpy(qkv, h.data(), n * W * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dout, h.data(), n * H * hd * 2, cudaMemcpyHostToDevice);
  const float sc = 1.f / sqrtf((float)hd);
  const bool use_rope = getenv("ATTN_ROPE") != nullptr;  // backward with the inverse-RoPE epilogues
  cudaStream_t s;
  cudaStreamCreate(&s);
  auto fwd = [&] { return spx_attn_fwd(qkv, o, lse, B, T, H, Hkv, hd, W, H * hd, sc, s); };
  auto bwd = [&] {
    return spx_attn_bwd_ex(qkv, o, dout, lse, ws, dqkv, B, T, H, Hkv, hd, W, H * hd, sc, use_rope ? cs : nullptr,
                           SPX_ATTN_WS_EX, s);
  };
  double fl = 4.0 * B * H * (double)T * T / 2 * hd;
  for (int k = 0; k < 2; ++k) {
    for (int i = 0; i < 3; ++i) {
      int rc = k == 0 ? fwd() : bwd();
      if (rc) { printf("error %d %s\n", rc, spx_last_error()); return 1; }
    }
    cudaStreamSynchronize(s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int i = 0; i < iters; ++i) k == 0 ? fwd() : bwd();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double us = ms * 1e3 / iters;
    printf("{\"pass\": \"%s\", \"B\": %d, \"T\": %d, \"H\": %d, \"Hkv\": %d, \"hd\": %d, \"us\": %.2f, \"tflops\": %.1f}\n",
           k == 0 ? "fwd" : "bwd", B, T, H, Hkv, hd, us, (k == 0 ? 1.0 : 2.5) * fl / us / 1e6);
  }
#ifdef SPX_FA_PROBE
  {
    cudaDeviceSynchronize();
    fwd();
    cudaDeviceSynchronize();
    static long long pr[8][256];
    cudaMemcpyFromSymbol(pr, spx::fa::g_fa_probe, sizeof pr);
    const char* ev[] = {"s_full", "chunk0", "exps", "bar", "p_ready", "p_arrive", "S_issue", "PV_issue"};
    long long t0 = pr[0][0];
    for (int st = 0; st < 24; ++st) {
      printf("{\"fprobe\": %d", st);
      for (int e = 0; e < 8; ++e) printf(", \"%s\": %lld", ev[e], pr[e][st] - t0);
      printf("}\n");
    }
  }
#endif
#ifdef SPX_FAB_PROBE
  {
    // one more backward, then the per-step stamps of CTA 0 (cycles relative to its first S/dP)
    cudaDeviceSynchronize();
    bwd();
    cudaDeviceSynchronize();
    static long long pr[8][256];
    cudaMemcpyFromSymbol(pr, spx::fab::g_fab_probe, sizeof pr);
    const char* ev[] = {"load_issue", "tmem_free", "p_ready_mma", "sdp_full", "ew_computed", "ew_tiles_free",
                        "ew_stored"};
    long long t0 = pr[3][0];
    for (int st = 0; st < 24; ++st) {
      printf("{\"probe\": %d", st);
      for (int e = 0; e < 7; ++e) printf(", \"%s\": %lld", ev[e], pr[e][st] - t0);
      printf("}\n");
    }
  }
#endif
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
  if (argc > 7) {  // dump O and dQKV (bf16) for cross-variant comparison
    std::vector<uint16_t> ho(n * H * hd), hg(n * W);
    cudaMemcpy(ho.data(), o, ho.size() * 2, cudaMemcpyDeviceToHost);
    cudaMemcpy(hg.data(), dqkv, hg.size() * 2, cudaMemcpyDeviceToHost);
    FILE* f = fopen(argv[7], "wb");
    fwrite(ho.data(), 2, ho.size(), f);
    fwrite(hg.data(), 2, hg.size(), f);
    fclose(f);
  }
  return 0;
}

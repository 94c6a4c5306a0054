#include <cstdlib>
// HBM-bound kernels of a LLaMA stage and of the optimizer step: RMSNorm fwd/bwd, RoPE,
// SwiGLU backward, embedding gather / deterministic scatter, fused softmax cross-entropy
// (loss + dlogits in one pass pair), deterministic sums, grad-norm clip and fused AdamW.
//
// All row kernels use one warp per row with 16-byte vector accesses; reductions that feed
// parameter gradients are two-pass (fixed-order partials, then a fixed-order final sum) so a
// training step is bit-reproducible.
#include <cmath>

#include "spx_common.cuh"
#include "spx_internal.h"

namespace spx {
namespace ew {

constexpr int ROW_WARPS = 8;  // rows per 256-thread CTA

union Vec8 {
  uint4 u;
  __nv_bfloat162 h[4];
};

SPX_DEVICE void load8(float (&f)[8], const __nv_bfloat16* p) {
  Vec8 v;
  v.u = *reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(v.h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

SPX_DEVICE void store8(__nv_bfloat16* p, const float (&f)[8]) {
  Vec8 v;
#pragma unroll
  for (int i = 0; i < 4; ++i) v.h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = v.u;
}

// ---------------------------------------------------------------- RMSNorm
__global__ void rmsnorm_fwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
                                   __nv_bfloat16* __restrict__ y, float* __restrict__ rstd, int rows, int d,
                                   float eps) {
  pdl_wait();
  const int row = blockIdx.x * ROW_WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const __nv_bfloat16* xr = x + (size_t)row * d;
  float ss = 0.f;
  for (int c = lane * 8; c < d; c += 256) {
    float f[8];
    load8(f, xr + c);
#pragma unroll
    for (int i = 0; i < 8; ++i) ss += f[i] * f[i];
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / d + eps);
  __nv_bfloat16* yr = y + (size_t)row * d;
  for (int c = lane * 8; c < d; c += 256) {
    float f[8], w[8];
    load8(f, xr + c);
    load8(w, g + c);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = f[i] * r * w[i];
    store8(yr + c, f);
  }
  if (lane == 0) rstd[row] = r;
}

// Register-resident form (d <= 256*NCH): the row's 16-byte vectors are loaded once, all in
// flight together, kept in registers for the normalisation pass (no second read of x).
template <int NCH>
__global__ void rmsnorm_fwd_reg_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
                                       __nv_bfloat16* __restrict__ y, float* __restrict__ rstd, int rows, int d,
                                       float eps) {
  pdl_wait();
  const int row = blockIdx.x * ROW_WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const size_t off = (size_t)row * d;
  Vec8 xv[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    const int c = lane * 8 + k * 256;
    xv[k].u = c < d ? *reinterpret_cast<const uint4*>(x + off + c) : make_uint4(0, 0, 0, 0);
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < NCH; ++k)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(xv[k].h[i]);
      ss += f.x * f.x + f.y * f.y;
    }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / d + eps);
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    const int c = lane * 8 + k * 256;
    if (c < d) {
      float w[8], f[8];
      load8(w, g + c);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(xv[k].h[i]);
        f[2 * i] = t.x * r * w[2 * i];
        f[2 * i + 1] = t.y * r * w[2 * i + 1];
      }
      store8(y + off + c, f);
    }
  }
  if (lane == 0) rstd[row] = r;
}

// RMSNorm backward, dx:  dx = dres + rstd * (g*dy - xhat * mean(xhat*g*dy)), xhat = x*rstd.
// One warp per row, 16-byte vectors (HBM-bound: reads x, dy, dres, writes dx).
__global__ void rmsnorm_bwd_dx_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
                                      const float* __restrict__ rstd, const __nv_bfloat16* __restrict__ dy,
                                      const __nv_bfloat16* __restrict__ dres, __nv_bfloat16* __restrict__ dx,
                                      int rows, int d) {
  pdl_wait();
  const int row = blockIdx.x * ROW_WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const size_t off = (size_t)row * d;
  const float r = rstd[row];
  float dot = 0.f;
  for (int c = lane * 8; c < d; c += 256) {
    float xf[8], w[8], gy[8];
    load8(xf, x + off + c);
    load8(w, g + c);
    load8(gy, dy + off + c);
#pragma unroll
    for (int i = 0; i < 8; ++i) dot += xf[i] * w[i] * gy[i];
  }
  dot = warp_sum(dot) * r / d;
  for (int c = lane * 8; c < d; c += 256) {
    float xf[8], w[8], gy[8], o[8];
    load8(xf, x + off + c);
    load8(w, g + c);
    load8(gy, dy + off + c);
    if (dres) load8(o, dres + off + c);
    else {
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = 0.f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] += r * (w[i] * gy[i] - xf[i] * r * dot);
    store8(dx + off + c, o);
  }
}

// RMSNorm backward, dg partials: CTA (column block of 256, row chunk of DG_ROWS rows) sums
// dy * x * rstd over its rows in order; thread = 2 adjacent columns, 128 threads per block.
constexpr int DG_ROWS = 64;
__global__ void __launch_bounds__(128) rmsnorm_dg_partial_kernel(const __nv_bfloat16* __restrict__ x,
                                                                 const float* __restrict__ rstd,
                                                                 const __nv_bfloat16* __restrict__ dy,
                                                                 float* __restrict__ part, int rows, int d) {
  pdl_wait();
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (c >= d) return;
  const int r0 = blockIdx.y * DG_ROWS, r1 = min(rows, r0 + DG_ROWS);
  float a0 = 0.f, a1 = 0.f;
#pragma unroll 8
  for (int r = r0; r < r1; ++r) {
    const float s = rstd[r];
    const float2 xv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(x + (size_t)r * d + c));
    const float2 gv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dy + (size_t)r * d + c));
    a0 += gv.x * xv.x * s;
    a1 += gv.y * xv.y * s;
  }
  *reinterpret_cast<float2*>(part + (size_t)blockIdx.y * d + c) = make_float2(a0, a1);
}

// RMSNorm backward, dx and dg in one pass over x and dy.  Warp per row (a CTA owns a contiguous
// block of rows, warp w takes rows w, w+8, ...); lane owns the 8-column vectors lane*8 + k*256
// (k < NCH), so x and dy stay in registers between the row-dot pass and the dx pass, and the
// lane's dg accumulators need no shuffles.  The CTA's dg partial is reduced over its warps in
// fixed order through shared memory (deterministic), then colsum_add_kernel adds the partials.
template <int NCH>
__global__ void __launch_bounds__(256, NCH <= 4 ? 2 : 1) rmsnorm_bwd_fused_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g, const float* __restrict__ rstd,
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ dres, __nv_bfloat16* __restrict__ dx,
    float* __restrict__ part, int rows, int d, int rows_per_cta) {
  extern __shared__ float red[];  // [ROW_WARPS][d]
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float acc[NCH][8];
#pragma unroll
  for (int k = 0; k < NCH; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[k][i] = 0.f;
  const int r0 = blockIdx.x * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
  for (int r = r0 + warp; r < r1; r += ROW_WARPS) {
    const size_t off = (size_t)r * d;
    const float s = rstd[r];
    Vec8 xv[NCH], yv[NCH], rv[NCH];  // x, dy and dres of this row, loaded together up front
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const int c = lane * 8 + k * 256;
      if (c < d) {
        xv[k].u = *reinterpret_cast<const uint4*>(x + off + c);
        yv[k].u = *reinterpret_cast<const uint4*>(dy + off + c);
        rv[k].u = dres ? *reinterpret_cast<const uint4*>(dres + off + c) : make_uint4(0, 0, 0, 0);
      }
    }
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const int c = lane * 8 + k * 256;
      if (c < d) {
        float w[8];
        load8(w, g + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 xf = __bfloat1622float2(xv[k].h[i]), gy = __bfloat1622float2(yv[k].h[i]);
          dot += xf.x * w[2 * i] * gy.x + xf.y * w[2 * i + 1] * gy.y;
        }
      }
    }
    dot = warp_sum(dot) * s / d;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const int c = lane * 8 + k * 256;
      if (c < d) {
        float w[8], o[8];
        load8(w, g + c);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 xf = __bfloat1622float2(xv[k].h[i]), gy = __bfloat1622float2(yv[k].h[i]);
          const float2 rf = __bfloat1622float2(rv[k].h[i]);
          o[2 * i] = rf.x + s * (w[2 * i] * gy.x - xf.x * s * dot);
          o[2 * i + 1] = rf.y + s * (w[2 * i + 1] * gy.y - xf.y * s * dot);
          acc[k][2 * i] += gy.x * xf.x * s;
          acc[k][2 * i + 1] += gy.y * xf.y * s;
        }
        store8(dx + off + c, o);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    const int c = lane * 8 + k * 256;
    if (c < d) {
      float4* dst = reinterpret_cast<float4*>(red + (size_t)warp * d + c);
      dst[0] = make_float4(acc[k][0], acc[k][1], acc[k][2], acc[k][3]);
      dst[1] = make_float4(acc[k][4], acc[k][5], acc[k][6], acc[k][7]);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < ROW_WARPS; ++w) t += red[(size_t)w * d + c];
    part[(size_t)blockIdx.x * d + c] = t;
  }
}

// rows per CTA of the fused RMSNorm backward: a multiple of 16 giving about two CTAs per SM
static int rms_rows_per_cta(long long rows) {
  static const int fixed = [] {  // SPX_RMS_RPC: rows per CTA, multiple of 8 (benchmarking)
    const char* e = getenv("SPX_RMS_RPC");
    const int v = e ? atoi(e) : 0;
    return v >= 8 ? v / 8 * 8 : 0;
  }();
  if (fixed) return fixed;
  const long long target = 2LL * num_sms();
  long long rpc = (rows + target - 1) / target;
  rpc = ((rpc + 15) / 16) * 16;
  return (int)(rpc < 16 ? 16 : rpc);
}

// out[c] += sum_i part[i][c], deterministic.  A CTA owns 8 columns (one 32-byte sector per
// partial row); thread t sums the partials i = t/8, t/8 + 32, ... of column t%8 (independent
// loads, all in flight), then the 32 per-thread sums of a column are added in fixed order.  128
// CTAs at d = 1024 (the previous 32-column CTAs left most SMs idle and serialised the loads).
__global__ void __launch_bounds__(256) colsum_add_kernel(const float* __restrict__ part, float* __restrict__ out,
                                                         int nsplit, int d) {
  __shared__ float red[32][9];
  pdl_wait();
  const int cl = threadIdx.x & 7, pr = threadIdx.x >> 3;
  const int c = blockIdx.x * 8 + cl;
  float s = 0.f;
  if (c < d) {
#pragma unroll 8
    for (int i = pr; i < nsplit; i += 32) s += part[(size_t)i * d + c];
  }
  red[pr][cl] = s;
  __syncthreads();
  if (threadIdx.x < 8 && c < d) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 32; ++w) t += red[w][cl];
    out[c] += t;
  }
}

// ---------------------------------------------------------------- RoPE (rotate-half convention)
// in place on the q heads [0, H) and k heads [H, H+Hkv) of a fused QKV row; position = row % T
__global__ void rope_kernel(__nv_bfloat16* __restrict__ qkv, const float* __restrict__ cs, int rows, int T, int nheads,
                            int hd, long long ld, float sign) {
  pdl_wait();
  const int half = hd / 2;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per_row = (long long)nheads * half;
  if (idx >= (long long)rows * per_row) return;
  const int row = (int)(idx / per_row);
  const int rem = (int)(idx % per_row);
  const int h = rem / half, j = rem % half;
  const int t = row % T;
  const float c = cs[((size_t)j * T + t) * 2];
  const float s = sign * cs[((size_t)j * T + t) * 2 + 1];
  __nv_bfloat16* p = qkv + (size_t)row * ld + (size_t)h * hd;
  const float a = __bfloat162float(p[j]), b = __bfloat162float(p[j + half]);
  p[j] = __float2bfloat16(a * c - b * s);
  p[j + half] = __float2bfloat16(b * c + a * s);
}

// ---------------------------------------------------------------- SwiGLU backward
// gu [rows, 2F] with gate/up interleaved in 128-column blocks; dh [rows, F]; dgu [rows, 2F]
__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ gu, const __nv_bfloat16* __restrict__ dh,
                                  __nv_bfloat16* __restrict__ dgu, int rows, int F) {
  pdl_wait();
  const long long idx = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (idx >= (long long)rows * F) return;
  const int row = (int)(idx / F);
  const int c = (int)(idx % F);
  const int blk = c >> 7, j = c & 127;
  const size_t gofs = (size_t)row * 2 * F + (size_t)blk * 256 + j;
  float g[8], u[8], d[8], og[8], ou[8];
  load8(g, gu + gofs);
  load8(u, gu + gofs + 128);
  load8(d, dh + (size_t)row * F + c);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float sg = 1.f / (1.f + __expf(-g[i]));
    const float silu = g[i] * sg;
    og[i] = d[i] * u[i] * sg * (1.f + g[i] * (1.f - sg));
    ou[i] = d[i] * silu;
  }
  store8(dgu + gofs, og);
  store8(dgu + gofs + 128, ou);
}

// ---------------------------------------------------------------- embedding
__global__ void embed_fwd_kernel(const int32_t* __restrict__ ids, const __nv_bfloat16* __restrict__ table,
                                 __nv_bfloat16* __restrict__ out, int n, int d) {
  pdl_wait();
  const int row = blockIdx.x * ROW_WARPS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const __nv_bfloat16* src = table + (size_t)ids[row] * d;
  __nv_bfloat16* dst = out + (size_t)row * d;
  for (int c = lane * 8; c < d; c += 256)
    *reinterpret_cast<uint4*>(dst + c) = *reinterpret_cast<const uint4*>(src + c);
}

// Deterministic scatter-add: tokens pre-grouped by id (perm sorted by (id, position)); one CTA
// per distinct id sums its rows in position order and adds once into the fp32 table gradient.
__global__ void embed_bwd_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ seg_start,
                                 const int32_t* __restrict__ seg_id, const int32_t* __restrict__ n_seg,
                                 const __nv_bfloat16* __restrict__ dout, float* __restrict__ dtable, int d) {
  pdl_wait();
  const int seg = blockIdx.x;
  if (seg >= n_seg[0]) return;
  const int a = seg_start[seg], b = seg_start[seg + 1];
  float* dst = dtable + (size_t)seg_id[seg] * d;
  for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = a; k < b; ++k) {
      float f[8];
      load8(f, dout + (size_t)perm[k] * d + c);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += f[i];
    }
    float4* o = reinterpret_cast<float4*>(dst + c);
    float4 o0 = o[0], o1 = o[1];
    o0.x += acc[0]; o0.y += acc[1]; o0.z += acc[2]; o0.w += acc[3];
    o1.x += acc[4]; o1.y += acc[5]; o1.z += acc[6]; o1.w += acc[7];
    o[0] = o0;
    o[1] = o1;
  }
}

// ---------------------------------------------------------------- token batch preparation
// One microbatch's token block [b, T+1] (int64, row stride ld) -> inputs ids[n] = tok[r, t],
// targets[n] = tok[r, t+1] (n = b*T, position i = r*T + t), and the grouping the deterministic
// embedding backward needs: positions sorted by (id, position), perm, segment starts and ids.
// Keys (id << 32 | position) are unique, so the sorted order -- and with it the embedding
// gradient's summation order -- is unique: a bitonic sort in shared memory (one CTA, n <= 16384)
// gives exactly the host reference's stable argsort.  Runs on the device so a step's only
// host->device input is the raw token block.
constexpr int TP_THREADS = 1024;
constexpr int TP_MAX_N = 16384;

__global__ void __launch_bounds__(TP_THREADS) token_prep_kernel(const long long* __restrict__ tok, int T, long long ld,
                                                                int n, int n2, int32_t* __restrict__ ids,
                                                                int32_t* __restrict__ tgt, int32_t* __restrict__ perm,
                                                                int32_t* __restrict__ seg_start,
                                                                int32_t* __restrict__ seg_id,
                                                                int32_t* __restrict__ n_seg) {
  extern __shared__ unsigned long long keys[];  // n2 = next power of two >= n
  __shared__ int wsum[TP_THREADS / 32];
  pdl_wait();
  const int tid = threadIdx.x;
  for (int i = tid; i < n2; i += TP_THREADS) {
    unsigned long long k = ~0ull;
    if (i < n) {
      const int r = i / T, t = i - r * T;
      const long long id = tok[r * ld + t];
      if (ids) ids[i] = (int32_t)id;
      if (tgt) tgt[i] = (int32_t)tok[r * ld + t + 1];
      k = ((unsigned long long)(uint32_t)id << 32) | (uint32_t)i;
    }
    keys[i] = k;
  }
  __syncthreads();
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < n2; i += TP_THREADS) {
        const int p = i ^ j;
        if (p > i) {
          const unsigned long long a = keys[i], c = keys[p];
          if ((a > c) == ((i & k) == 0)) {
            keys[i] = c;
            keys[p] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // segment boundaries: a contiguous chunk of sorted positions per thread, block-wide scan
  const int per = (n + TP_THREADS - 1) / TP_THREADS;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32));
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((tid & 31) >= o) incl += y;
  }
  if ((tid & 31) == 31) wsum[tid >> 5] = incl;
  __syncthreads();
  if (tid < 32) {
    int w = wsum[tid], wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (tid >= o) wi += y;
    }
    wsum[tid] = wi - w;  // exclusive prefix over warps
  }
  __syncthreads();
  int seg = wsum[tid >> 5] + incl - cnt;
  for (int i = lo; i < hi; ++i) {
    const unsigned long long key = keys[i];
    perm[i] = (int32_t)(uint32_t)key;
    if (i == 0 || (key >> 32) != (keys[i - 1] >> 32)) {
      seg_start[seg] = i;
      seg_id[seg] = (int32_t)(key >> 32);
      ++seg;
    }
  }
  if (hi == n && lo < hi) {  // the thread holding the last position
    seg_start[seg] = n;
    n_seg[0] = seg;
  }
}

// split only (no grouping): ids / targets of one token block, one thread per position
__global__ void token_split_kernel(const long long* __restrict__ tok, int T, long long ld, int n,
                                   int32_t* __restrict__ ids, int32_t* __restrict__ tgt) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int r = i / T, t = i - r * T;
  if (ids) ids[i] = (int32_t)tok[r * ld + t];
  if (tgt) tgt[i] = (int32_t)tok[r * ld + t + 1];
}

// ---------------------------------------------------------------- softmax cross-entropy
// One CTA per row: loss_r = logsumexp(z) - z[target]; dlogits = (softmax(z) - onehot) * scale
// written in place over the bf16 logits.
constexpr int XE_THREADS = 512;
__global__ void __launch_bounds__(XE_THREADS) xent_kernel(__nv_bfloat16* __restrict__ logits,
                                                          const int32_t* __restrict__ targets,
                                                          float* __restrict__ row_loss, int V, long long ld,
                                                          float scale) {
  pdl_wait();
  __shared__ float red_m[XE_THREADS / 32], red_s[XE_THREADS / 32];
  const int row = blockIdx.x;
  __nv_bfloat16* z = logits + (size_t)row * ld;
  float m = -INFINITY, s = 0.f;
  for (int c = threadIdx.x * 8; c < V; c += XE_THREADS * 8) {
    float f[8];
    load8(f, z + c);
    float mx = f[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) mx = fmaxf(mx, f[i]);
    const float nm = fmaxf(m, mx);
    s *= __expf(m - nm);
#pragma unroll
    for (int i = 0; i < 8; ++i) s += __expf(f[i] - nm);
    m = nm;
  }
  // warp then block reduction of (m, s)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
    const float nm = fmaxf(m, om);
    s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
    m = nm;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red_m[w] = m;
    red_s[w] = s;
  }
  __syncthreads();
  if (w == 0) {
    m = lane < XE_THREADS / 32 ? red_m[lane] : -INFINITY;
    s = lane < XE_THREADS / 32 ? red_s[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
      const float nm = fmaxf(m, om);
      s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
      m = nm;
    }
    if (lane == 0) {
      red_m[0] = m;
      red_s[0] = s;
    }
  }
  __syncthreads();
  m = red_m[0];
  s = red_s[0];
  const int tgt = targets[row];
  const float zt = __bfloat162float(z[tgt]);
  __syncthreads();
  const float inv = 1.f / s;
  for (int c = threadIdx.x * 8; c < V; c += XE_THREADS * 8) {
    float f[8];
    load8(f, z + c);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = (__expf(f[i] - m) * inv - (c + i == tgt ? 1.f : 0.f)) * scale;
    store8(z + c, f);
  }
  if (threadIdx.x == 0) row_loss[row] = logf(s) + m - zt;
}

// Cross-entropy from the head GEMM's per-128-column (max, sum exp) partials (EPI_XENT): one CTA
// per row combines its nb partials in fixed order (deterministic) into the log-sum-exp, writes
// the row loss lse - z[target] and, when scale != 0, rewrites the logits in place as
// dlogits = (softmax - onehot) * scale -- one read and one write of the logits instead of the
// online pass plus the dlogits pass of xent_kernel.
__device__ __forceinline__ void lse_merge(float& m, float& s, float om, float os) {
  const float nm = fmaxf(m, om);
  s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
  m = nm;
}

__global__ void __launch_bounds__(XE_THREADS) xent_parts_kernel(__nv_bfloat16* __restrict__ logits,
                                                                const float* __restrict__ parts, int nb,
                                                                const int32_t* __restrict__ targets,
                                                                float* __restrict__ row_loss, int V, long long ld,
                                                                float scale) {
  pdl_wait();
  __shared__ float red_m[XE_THREADS / 32], red_s[XE_THREADS / 32];
  const int row = blockIdx.x;
  const float2* pr = reinterpret_cast<const float2*>(parts + (size_t)row * 2 * nb);
  float m = -INFINITY, s = 0.f;
  for (int b = threadIdx.x; b < nb; b += XE_THREADS) {
    const float2 p = pr[b];
    lse_merge(m, s, p.x, p.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
    lse_merge(m, s, om, os);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red_m[w] = m;
    red_s[w] = s;
  }
  __syncthreads();
  if (w == 0) {
    m = lane < XE_THREADS / 32 ? red_m[lane] : -INFINITY;
    s = lane < XE_THREADS / 32 ? red_s[lane] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
      lse_merge(m, s, om, os);
    }
    if (lane == 0) {
      red_m[0] = m;
      red_s[0] = s;
    }
  }
  __syncthreads();
  m = red_m[0];
  s = red_s[0];
  __nv_bfloat16* z = logits + (size_t)row * ld;
  const int tgt = targets[row];
  const float zt = __bfloat162float(z[tgt]);
  if (threadIdx.x == 0) row_loss[row] = logf(s) + m - zt;
  if (scale == 0.f) return;  // loss only (inference)
  __syncthreads();           // every thread has read z[tgt] before it is overwritten
  const float inv = 1.f / s;
  for (int c = threadIdx.x * 8; c < V; c += XE_THREADS * 8) {
    float f[8];
    load8(f, z + c);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = (__expf(f[i] - m) * inv - (c + i == tgt ? 1.f : 0.f)) * scale;
    store8(z + c, f);
  }
}

// ---------------------------------------------------------------- reductions
// out[0] (+)= scale * sum(x[0:n])   (single CTA, fixed order)
// dst += src (fp32, float4 vectors when aligned): merges co-resident replicas' gradient buffers
// CLEAR: src = 0 afterwards (the merged buffer starts the next iteration at zero, no fill pass)
template <bool CLEAR>
__global__ void add_f32_kernel(float* __restrict__ dst, float* __restrict__ src, long long n) {
  pdl_wait();
  const long long n4 = n / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 a = reinterpret_cast<float4*>(dst)[i];
    const float4 b = reinterpret_cast<const float4*>(src)[i];
    a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    reinterpret_cast<float4*>(dst)[i] = a;
    if (CLEAR) reinterpret_cast<float4*>(src)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (long long i = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    dst[i] += src[i];
    if (CLEAR) src[i] = 0.f;
  }
}

__global__ void sum_kernel(const float* __restrict__ x, long long n, float* __restrict__ out, float scale,
                           int accumulate) {
  pdl_wait();
  __shared__ double red[32];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    const float v = (float)(t * scale);
    out[0] = accumulate ? out[0] + v : v;
  }
}

constexpr int SUMSQ_BLOCKS = 592;  // 4 per SM
__global__ void sumsq_partial_kernel(const float* __restrict__ x, long long n, float* __restrict__ part) {
  pdl_wait();
  __shared__ float red[32];
  float s = 0.f;
  const long long n4 = n / 4;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 v = x4[i];
    s += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  if (blockIdx.x == 0)
    for (long long i = n4 * 4 + threadIdx.x; i < n; i += blockDim.x) s += x[i] * x[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    part[blockIdx.x] = t;
  }
}

// scale = min(1, max_norm / (||g|| + 1e-6)) from per-set squared norms (torch clip_grad_norm_)
__global__ void clip_scale_kernel(const float* __restrict__ sumsq, int count, float max_norm, float* __restrict__ scale,
                                  float* __restrict__ norm_out) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  double t = 0.0;
  for (int i = 0; i < count; ++i) t += sumsq[i];
  const float nrm = (float)sqrt(t);
  if (norm_out) norm_out[0] = nrm;
  const float c = max_norm / (nrm + 1e-6f);
  scale[0] = c < 1.f ? c : 1.f;
}

// ---------------------------------------------------------------- AdamW (torch.optim.AdamW math)
// One AdamW element update with every rounding explicit (no compiler FMA contraction choices), so
// the scalar and the 16-byte vector kernels are bit-identical.
__device__ __forceinline__ void adamw_one(float& pi, float gi, float& mi, float& vi, bool decay, float lr, float b1,
                                          float b2, float eps, float wd, float step, float rbc2) {
  if (decay) pi = __fmul_rn(pi, __fsub_rn(1.f, __fmul_rn(lr, wd)));
  mi = __fmaf_rn(b1, mi, __fmul_rn(__fsub_rn(1.f, b1), gi));
  vi = __fmaf_rn(b2, vi, __fmul_rn(__fmul_rn(__fsub_rn(1.f, b2), gi), gi));
  const float den = __fmaf_rn(__fsqrt_rn(vi), rbc2, eps);
  pi = __fsub_rn(pi, __fdiv_rn(__fmul_rn(step, mi), den));
}

template <bool ZERO>
__global__ void adamw_kernel(float* __restrict__ p, float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, __nv_bfloat16* __restrict__ pb, long long n, long long n_decay,
                             float lr, float b1, float b2, float eps, float wd, float bc1, float bc2,
                             const float* __restrict__ gscale) {
  pdl_wait();
  const float sc = gscale ? gscale[0] : 1.f;
  const float step = lr / bc1;
  const float rbc2 = rsqrtf(bc2);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float pi = p[i], mi = m[i], vi = v[i];
    adamw_one(pi, __fmul_rn(g[i], sc), mi, vi, i < n_decay, lr, b1, b2, eps, wd, step, rbc2);
    m[i] = mi;
    v[i] = vi;
    p[i] = pi;
    pb[i] = __float2bfloat16(pi);
    if (ZERO) g[i] = 0.f;
  }
}

// 16-byte vector form: 4 elements per thread per iteration (p/g/m/v 16-byte, pb 8-byte aligned;
// n % 4 by the scalar tail)
// ZERO: the consumed gradient is cleared (the next iteration accumulates from zero without a fill)
template <bool ZERO>
__global__ void __launch_bounds__(256) adamw_vec_kernel(float* __restrict__ p, float* __restrict__ g,
                                                        float* __restrict__ m, float* __restrict__ v,
                                                        __nv_bfloat16* __restrict__ pb, long long n, long long n_decay,
                                                        float lr, float b1, float b2, float eps, float wd, float bc1,
                                                        float bc2, const float* __restrict__ gscale) {
  pdl_wait();
  const float sc = gscale ? gscale[0] : 1.f;
  const float step = lr / bc1;
  const float rbc2 = rsqrtf(bc2);
  const long long n4 = n / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 g4 = __ldcs(reinterpret_cast<const float4*>(g) + i);
    float4 p4 = __ldcs(reinterpret_cast<const float4*>(p) + i);
    float4 m4 = __ldcs(reinterpret_cast<const float4*>(m) + i);
    float4 v4 = __ldcs(reinterpret_cast<const float4*>(v) + i);
    const long long e = 4 * i;
    adamw_one(p4.x, __fmul_rn(g4.x, sc), m4.x, v4.x, e + 0 < n_decay, lr, b1, b2, eps, wd, step, rbc2);
    adamw_one(p4.y, __fmul_rn(g4.y, sc), m4.y, v4.y, e + 1 < n_decay, lr, b1, b2, eps, wd, step, rbc2);
    adamw_one(p4.z, __fmul_rn(g4.z, sc), m4.z, v4.z, e + 2 < n_decay, lr, b1, b2, eps, wd, step, rbc2);
    adamw_one(p4.w, __fmul_rn(g4.w, sc), m4.w, v4.w, e + 3 < n_decay, lr, b1, b2, eps, wd, step, rbc2);
    __stcs(reinterpret_cast<float4*>(m) + i, m4);
    __stcs(reinterpret_cast<float4*>(v) + i, v4);
    __stcs(reinterpret_cast<float4*>(p) + i, p4);
    __nv_bfloat162 lo = __floats2bfloat162_rn(p4.x, p4.y), hi = __floats2bfloat162_rn(p4.z, p4.w);
    uint2 packed;
    packed.x = *reinterpret_cast<uint32_t*>(&lo);
    packed.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(pb)[i] = packed;
    if (ZERO) __stcs(reinterpret_cast<float4*>(g) + i, make_float4(0.f, 0.f, 0.f, 0.f));
  }
  for (long long i = 4 * n4 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float pi = p[i], mi = m[i], vi = v[i];
    adamw_one(pi, __fmul_rn(g[i], sc), mi, vi, i < n_decay, lr, b1, b2, eps, wd, step, rbc2);
    m[i] = mi;
    v[i] = vi;
    p[i] = pi;
    pb[i] = __float2bfloat16(pi);
    if (ZERO) g[i] = 0.f;
  }
}

}  // namespace ew
}  // namespace spx

using namespace spx;
using namespace spx::ew;

#define SPX_S reinterpret_cast<cudaStream_t>(stream)
#define BF(p) reinterpret_cast<__nv_bfloat16*>(p)
#define CBF(p) reinterpret_cast<const __nv_bfloat16*>(p)

extern "C" int spx_rmsnorm_fwd(const void* x, const void* g, void* y, float* rstd, int64_t rows, int64_t d, float eps,
                               void* stream) {
  if (d % 8) return set_error(SPX_ERR_ARG, "rmsnorm: d must be a multiple of 8");
  const dim3 grid((unsigned)((rows + ROW_WARPS - 1) / ROW_WARPS)), block(ROW_WARPS * 32);
  if (d <= 4096) {
    const int nch = (int)((d + 255) / 256);
    auto k = nch <= 1 ? rmsnorm_fwd_reg_kernel<1> : nch <= 2 ? rmsnorm_fwd_reg_kernel<2>
             : nch <= 4 ? rmsnorm_fwd_reg_kernel<4> : nch <= 8 ? rmsnorm_fwd_reg_kernel<8> : rmsnorm_fwd_reg_kernel<16>;
    spx_launch_check(launch_k(k, grid, block, 0, SPX_S, CBF(x), CBF(g), BF(y), rstd, (int)rows, (int)d, eps));
    return check_launch("rmsnorm_fwd_reg_kernel");
  }
  spx_launch_check(launch_k(rmsnorm_fwd_kernel, grid, block, 0, SPX_S, CBF(x), CBF(g), BF(y), rstd, (int)rows, (int)d, eps));
  return check_launch("rmsnorm_fwd_kernel");
}

extern "C" int spx_rmsnorm_bwd(const void* x, const void* g, const float* rstd, const void* dy, const void* dres,
                               void* dx, float* dg, float* ws, int64_t rows, int64_t d, void* stream) {
  if (d % 8) return set_error(SPX_ERR_ARG, "rmsnorm: d must be a multiple of 8");
  if (rows <= 0) return SPX_OK;
  if (dg != nullptr && d <= 2048) {
    const int rpc = rms_rows_per_cta(rows);
    const int grid = (int)((rows + rpc - 1) / rpc);
    const size_t smem = (size_t)ROW_WARPS * d * sizeof(float);
    const int nch = (int)((d + 255) / 256);
    auto launch = [&](auto kern) {
      static bool attr[4] = {false, false, false, false};  // per instantiation; 64 KB at d = 2048
      const int slot = nch <= 1 ? 0 : nch <= 2 ? 1 : nch <= 4 ? 2 : 3;
      if (!attr[slot]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2048 * 4);
        if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(rmsnorm_bwd_fused)");
        attr[slot] = true;
      }
      spx_launch_check(launch_k(kern, dim3((unsigned)grid), dim3(ROW_WARPS * 32), smem, SPX_S, CBF(x), CBF(g), rstd,
                                CBF(dy), CBF(dres), BF(dx), ws, (int)rows, (int)d, rpc));
      return check_launch("rmsnorm_bwd_fused_kernel");
    };
    int rc = nch <= 1 ? launch(rmsnorm_bwd_fused_kernel<1>)
             : nch <= 2 ? launch(rmsnorm_bwd_fused_kernel<2>)
             : nch <= 4 ? launch(rmsnorm_bwd_fused_kernel<4>)
                        : launch(rmsnorm_bwd_fused_kernel<8>);
    if (rc) return rc;
    spx_launch_check(launch_k(colsum_add_kernel, dim3((unsigned)((d + 7) / 8)), dim3(256), 0, SPX_S, ws, dg, grid, (int)d));
    return check_launch("colsum_add_kernel");
  }
  spx_launch_check(launch_k(rmsnorm_bwd_dx_kernel, dim3((unsigned)((rows + ROW_WARPS - 1) / ROW_WARPS)), dim3(ROW_WARPS * 32), 0, SPX_S, 
      CBF(x), CBF(g), rstd, CBF(dy), CBF(dres), BF(dx), (int)rows, (int)d));
  int rc = check_launch("rmsnorm_bwd_dx_kernel");
  if (rc || dg == nullptr) return rc;
  const int chunks = (int)((rows + DG_ROWS - 1) / DG_ROWS);
  spx_launch_check(launch_k(rmsnorm_dg_partial_kernel, dim3(dim3((unsigned)((d / 2 + 127) / 128), (unsigned)chunks)), dim3(128), 0, SPX_S, 
      CBF(x), rstd, CBF(dy), ws, (int)rows, (int)d));
  rc = check_launch("rmsnorm_dg_partial_kernel");
  if (rc) return rc;
  spx_launch_check(launch_k(colsum_add_kernel, dim3((unsigned)((d + 7) / 8)), dim3(256), 0, SPX_S, ws, dg, chunks, (int)d));
  return check_launch("colsum_add_kernel");
}

extern "C" int64_t spx_rmsnorm_ws_floats(int64_t rows, int64_t d) {
  if (rows <= 0) return d;
  const long long rpc = rms_rows_per_cta(rows);
  const long long fused = (rows + rpc - 1) / rpc, split = (rows + DG_ROWS - 1) / DG_ROWS;
  return (fused > split ? fused : split) * d;
}

extern "C" int spx_rope(void* qkv, const float* cos_sin, int64_t rows, int64_t T, int64_t n_heads, int64_t hd,
                        int64_t ld, int32_t inverse, void* stream) {
  if (hd % 2) return set_error(SPX_ERR_ARG, "rope: odd head dim");
  const long long total = rows * n_heads * (hd / 2);
  spx_launch_check(launch_k(rope_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, SPX_S, BF(qkv), cos_sin, (int)rows, (int)T, (int)n_heads,
                                                                 (int)hd, ld, inverse ? -1.f : 1.f));
  return check_launch("rope_kernel");
}

extern "C" int spx_swiglu_bwd(const void* gu, const void* dh, void* dgu, int64_t rows, int64_t F, void* stream) {
  if (F % 128) return set_error(SPX_ERR_ARG, "swiglu_bwd: F must be a multiple of 128");
  const long long total = rows * F / 8;
  spx_launch_check(launch_k(swiglu_bwd_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, SPX_S, CBF(gu), CBF(dh), BF(dgu), (int)rows, (int)F));
  return check_launch("swiglu_bwd_kernel");
}

extern "C" int spx_embed_fwd(const int32_t* ids, const void* table, void* out, int64_t n, int64_t d, void* stream) {
  if (d % 8) return set_error(SPX_ERR_ARG, "embed: d must be a multiple of 8");
  spx_launch_check(launch_k(embed_fwd_kernel, dim3((unsigned)((n + ROW_WARPS - 1) / ROW_WARPS)), dim3(ROW_WARPS * 32), 0, SPX_S, ids, CBF(table), BF(out),
                                                                                            (int)n, (int)d));
  return check_launch("embed_fwd_kernel");
}

extern "C" int spx_embed_bwd(const int32_t* perm, const int32_t* seg_start, const int32_t* seg_id,
                             const int32_t* n_segments, int64_t max_segments, const void* dout, float* dtable, int64_t d,
                             void* stream) {
  if (d % 8) return set_error(SPX_ERR_ARG, "embed: d must be a multiple of 8");
  if (max_segments <= 0) return SPX_OK;
  spx_launch_check(launch_k(embed_bwd_kernel, dim3((unsigned)max_segments), dim3(128), 0, SPX_S, perm, seg_start, seg_id, n_segments, CBF(dout), dtable,
                                                              (int)d));
  return check_launch("embed_bwd_kernel");
}

extern "C" int spx_token_prep(const int64_t* tokens, int64_t b, int64_t T, int64_t ld_tokens, int32_t* ids,
                              int32_t* targets, int32_t* perm, int32_t* seg_start, int32_t* seg_id, int32_t* n_segments,
                              void* stream) {
  const int64_t n = b * T;
  if (b <= 0 || T <= 0) return set_error(SPX_ERR_ARG, "token_prep: b and T must be positive");
  if (n > TP_MAX_N) return set_error(SPX_ERR_ARG, "token_prep: b*T must be <= 16384 (one-CTA sort)");
  if (ld_tokens < T + 1) return set_error(SPX_ERR_ARG, "token_prep: ld_tokens must be >= T + 1");
  if (perm == nullptr) {  // split only: ids / targets, no embedding-backward grouping
    if (seg_start || seg_id || n_segments) return set_error(SPX_ERR_ARG, "token_prep: grouping needs perm");
    spx_launch_check(launch_k(token_split_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, SPX_S,
                              reinterpret_cast<const long long*>(tokens), (int)T, (long long)ld_tokens, (int)n, ids,
                              targets));
    return check_launch("token_split_kernel");
  }
  if (!seg_start || !seg_id || !n_segments) return set_error(SPX_ERR_ARG, "token_prep: grouping outputs missing");
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  const size_t smem = (size_t)n2 * sizeof(unsigned long long);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(token_prep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         TP_MAX_N * (int)sizeof(unsigned long long));
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(token_prep)");
    attr = true;
  }
  spx_launch_check(launch_k(token_prep_kernel, dim3(1), dim3(TP_THREADS), smem, SPX_S,
                            reinterpret_cast<const long long*>(tokens), (int)T, (long long)ld_tokens, (int)n, n2, ids,
                            targets, perm, seg_start, seg_id, n_segments));
  return check_launch("token_prep_kernel");
}

extern "C" int spx_xent_from_parts(void* logits, const float* parts, int64_t nb, const int32_t* targets,
                                   float* row_loss, int64_t n, int64_t V, int64_t ld, float scale, void* stream) {
  if (V % 8 || ld % 8) return set_error(SPX_ERR_ARG, "xent_from_parts: V and ld must be multiples of 8");
  if (nb <= 0 || nb * 128 < V) return set_error(SPX_ERR_ARG, "xent_from_parts: need nb >= V / 128 partials per row");
  spx_launch_check(launch_k(xent_parts_kernel, dim3((unsigned)n), dim3(XE_THREADS), 0, SPX_S, BF(logits), parts, (int)nb,
                            targets, row_loss, (int)V, ld, scale));
  return check_launch("xent_parts_kernel");
}

extern "C" int spx_xent_fwd_bwd(void* logits, const int32_t* targets, float* row_loss, int64_t n, int64_t V, int64_t ld,
                                float scale, void* stream) {
  if (V % 8 || ld % 8) return set_error(SPX_ERR_ARG, "xent: V and ld must be multiples of 8");
  spx_launch_check(launch_k(xent_kernel, dim3((unsigned)n), dim3(XE_THREADS), 0, SPX_S, BF(logits), targets, row_loss, (int)V, ld, scale));
  return check_launch("xent_kernel");
}

extern "C" int spx_sum_f32(const float* x, int64_t n, float* out, float scale, int32_t accumulate, void* stream) {
  spx_launch_check(launch_k(sum_kernel, dim3(1), dim3(1024), 0, SPX_S, x, n, out, scale, accumulate));
  return check_launch("sum_kernel");
}

static int add_f32(float* dst, float* src, int64_t n, bool clear, cudaStream_t s) {
  if (n < 0) return set_error(SPX_ERR_ARG, "add_f32: negative size");
  if (n == 0) return SPX_OK;
  if (((uintptr_t)dst | (uintptr_t)src) & 15) return set_error(SPX_ERR_ARG, "add_f32: 16-byte aligned buffers required");
  const long long want = (n / 4 + 255) / 256;
  const int grid = (int)(want < 4LL * num_sms() ? (want > 0 ? want : 1) : 4LL * num_sms());
  spx_launch_check(launch_k(clear ? add_f32_kernel<true> : add_f32_kernel<false>, dim3(grid), dim3(256), 0, s, dst, src,
                            (long long)n));
  return check_launch("add_f32_kernel");
}

extern "C" int spx_add_f32(float* dst, const float* src, int64_t n, void* stream) {
  return add_f32(dst, const_cast<float*>(src), n, false, SPX_S);
}

extern "C" int spx_add_f32_clear(float* dst, float* src, int64_t n, void* stream) {
  return add_f32(dst, src, n, true, SPX_S);
}

extern "C" int64_t spx_sumsq_ws_floats(void) { return SUMSQ_BLOCKS; }

extern "C" int spx_sumsq(const float* x, int64_t n, float* ws, float* out, void* stream) {
  spx_launch_check(launch_k(sumsq_partial_kernel, dim3(SUMSQ_BLOCKS), dim3(256), 0, SPX_S, x, n, ws));
  int rc = check_launch("sumsq_partial_kernel");
  if (rc) return rc;
  spx_launch_check(launch_k(sum_kernel, dim3(1), dim3(1024), 0, SPX_S, ws, SUMSQ_BLOCKS, out, 1.f, 0));
  return check_launch("sum_kernel");
}

extern "C" int spx_clip_scale(const float* sumsq, int32_t count, float max_norm, float* scale, float* norm_out,
                              void* stream) {
  spx_launch_check(launch_k(clip_scale_kernel, dim3(1), dim3(32), 0, SPX_S, sumsq, count, max_norm, scale, norm_out));
  return check_launch("clip_scale_kernel");
}

static int adamw(float* p, float* g, float* m, float* v, void* p_bf16, int64_t n, int64_t n_decay, float lr,
                 float beta1, float beta2, float eps, float weight_decay, int64_t step, const float* grad_scale,
                 bool zero, cudaStream_t s) {
  if (step < 1) return set_error(SPX_ERR_ARG, "adamw: step must be >= 1");
  const float bc1 = 1.f - powf(beta1, (float)step);
  const float bc2 = 1.f - powf(beta2, (float)step);
  const int blocks = num_sms() * 8;
  const bool vec = !((((uintptr_t)p | (uintptr_t)g | (uintptr_t)m | (uintptr_t)v) & 15) | ((uintptr_t)p_bf16 & 7));
  auto k = vec ? (zero ? adamw_vec_kernel<true> : adamw_vec_kernel<false>)
               : (zero ? adamw_kernel<true> : adamw_kernel<false>);
  spx_launch_check(launch_k(k, dim3(blocks), dim3(256), 0, s, p, g, m, v, BF(p_bf16), n, n_decay, lr, beta1, beta2,
                            eps, weight_decay, bc1, bc2, grad_scale));
  return check_launch("adamw_kernel");
}

extern "C" int spx_adamw(float* p, const float* g, float* m, float* v, void* p_bf16, int64_t n, int64_t n_decay,
                         float lr, float beta1, float beta2, float eps, float weight_decay, int64_t step,
                         const float* grad_scale, void* stream) {
  return adamw(p, const_cast<float*>(g), m, v, p_bf16, n, n_decay, lr, beta1, beta2, eps, weight_decay, step,
               grad_scale, false, SPX_S);
}

extern "C" int spx_adamw_clear(float* p, float* g, float* m, float* v, void* p_bf16, int64_t n, int64_t n_decay,
                               float lr, float beta1, float beta2, float eps, float weight_decay, int64_t step,
                               const float* grad_scale, void* stream) {
  return adamw(p, g, m, v, p_bf16, n, n_decay, lr, beta1, beta2, eps, weight_decay, step, grad_scale, true, SPX_S);
}

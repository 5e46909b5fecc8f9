// Vectorised NHWC bf16 kernels for the nodes the conv epilogues cannot absorb:
//   * ub_eltwise    -- PER_CHANNEL affine (BN / bias), positional ADD, activations
//                      (PASS_THROUGH), and the per-image channel gate of a
//                      squeeze-excitation `mul` (SE mul -> positional ADD
//                      in the IR), one pass: y = act(scale*a + shift + b) * gate;
//   * ub_avgpool2d  -- k x k / stride s average pools (DenseNet transitions when the
//                      pool cannot move in front of its conv).
// One thread per (pixel, 8-channel group): 16-byte loads/stores when every operand
// row is 16-byte aligned, a scalar path otherwise.  HBM-bound; grid-stride loops sized
// from the SM count.
#include <cuda_bf16.h>

#include "ub_common.cuh"
#include "ub_host.h"

namespace ub {
namespace {

UB_DEVI float bf(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }
// 8 floats -> 8 bf16 in one uint4, in registers (a uint16_t[8] written element-wise and
// re-read as uint4 lives on the local-memory stack: ncu flagged it in the depthwise conv)
UB_DEVI uint4 pack8(const float (&f)[8]) {
  return make_uint4(cvt_bf16x2(f[0], f[1]), cvt_bf16x2(f[2], f[3]), cvt_bf16x2(f[4], f[5]), cvt_bf16x2(f[6], f[7]));
}
// bf16 element j (0..7) of a uint4 of 8 packed values, as fp32
UB_DEVI float bfj(const uint4& q, int j) {
  const uint32_t w = j < 2 ? q.x : (j < 4 ? q.y : (j < 6 ? q.z : q.w));
  return __uint_as_float((j & 1) ? (w & 0xffff0000u) : (w << 16));
}
// store 8 packed bf16 to p (16-byte aligned) or the first n of them
UB_DEVI void store8(uint16_t* p, const uint4& q, int n) {
  if (n >= 8) {
    *reinterpret_cast<uint4*>(p) = q;
  } else {
    for (int j = 0; j < n; ++j) {
      const uint32_t w = j < 2 ? q.x : (j < 4 ? q.y : (j < 6 ? q.z : q.w));
      p[j] = static_cast<uint16_t>((j & 1) ? (w >> 16) : (w & 0xffffu));
    }
  }
}
UB_DEVI uint16_t tobf(float v) { return __bfloat16_as_ushort(__float2bfloat16_rn(v)); }

template <bool VEC>
__global__ void __launch_bounds__(256) eltwise_kernel(ub_eltwise_desc d) {
  griddep_wait();
  griddep_launch_dependents();
  const int groups = VEC ? (d.C + 7) / 8 : d.C;
  const long long total = static_cast<long long>(d.N) * d.HW * groups;
  const uint16_t* a = static_cast<const uint16_t*>(d.a);
  const uint16_t* b = static_cast<const uint16_t*>(d.b);
  const uint16_t* g = static_cast<const uint16_t*>(d.gate);
  uint16_t* y = static_cast<uint16_t*>(d.y);
  // 32-bit index math (a 64-bit division costs ~100 instructions; totals stay < 2^31 here)
#pragma unroll 2
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < static_cast<unsigned>(total);
       e += gridDim.x * blockDim.x) {
    const unsigned pu = e / static_cast<unsigned>(groups);
    const long long p = pu;
    const int c0 = static_cast<int>(e - pu * groups) * (VEC ? 8 : 1);
    const int n = static_cast<int>(pu / static_cast<unsigned>(d.HW));
    if (VEC) {
      const uint4 qa = *reinterpret_cast<const uint4*>(a + p * d.a_cstride + d.a_coff + c0);
      const uint4 qb = b ? *reinterpret_cast<const uint4*>(b + p * d.b_cstride + d.b_coff + c0) : make_uint4(0, 0, 0, 0);
      const uint4 qg = g ? *reinterpret_cast<const uint4*>(g + static_cast<long long>(n) * d.gate_cstride + d.gate_coff + c0)
                         : make_uint4(0, 0, 0, 0);
      float f[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = c0 + j < d.C ? c0 + j : d.C - 1;
        float v = bfj(qa, j);
        if (d.scale) v *= d.scale[c];
        if (d.shift) v += d.shift[c];
        if (b) v += bfj(qb, j);
        v = act_f(v, d.act);
        if (g) v *= bfj(qg, j);
        f[j] = v;
      }
      store8(y + p * d.y_cstride + d.y_coff + c0, pack8(f), d.C - c0);
    } else {
      const int c = c0;
      float v = bf(a[p * d.a_cstride + d.a_coff + c]);
      if (d.scale) v *= d.scale[c];
      if (d.shift) v += d.shift[c];
      if (b) v += bf(b[p * d.b_cstride + d.b_coff + c]);
      v = act_f(v, d.act);
      if (g) v *= bf(g[static_cast<long long>(n) * d.gate_cstride + d.gate_coff + c]);
      y[p * d.y_cstride + d.y_coff + c] = tobf(v);
    }
  }
}

// y = act(a) * gate[n] (the squeeze-excitation `mul`, a positional ADD of the lowering with
// the gate broadcast over the pixels): one image per grid row; per thread GM_UNROLL
// independent 16-byte loads of `a` and of the (L1-resident) gate row in flight together,
// no per-element operand branches (the generic kernel above carries every PER_CHANNEL /
// ADD option).  ncu: staging the gate row in shared memory first put a dependent global
// round trip and a barrier in front of every CTA's only batch of loads.
constexpr int GM_UNROLL = 4;
template <bool ACT>  // ACT: apply a UB_ACT_* activation to `a` first (else the plain product)
__global__ void __launch_bounds__(256) gate_mul_kernel(const uint16_t* __restrict__ a, int a_cstride, int a_coff,
                                                       const uint16_t* __restrict__ g, int g_cstride, int g_coff,
                                                       uint16_t* __restrict__ y, int y_cstride, int y_coff, int HW,
                                                       int C, int act) {
  const int n = blockIdx.y;
  const int groups = (C + 7) / 8;
  const float inv_groups = 1.f / static_cast<float>(groups);
  griddep_wait();
  griddep_launch_dependents();
  const int total = HW * groups;
  // per-image base pointers once; 32-bit offsets inside the image
  const uint16_t* ai = a + static_cast<long long>(n) * HW * a_cstride + a_coff;
  uint16_t* yi = y + static_cast<long long>(n) * HW * y_cstride + y_coff;
  const uint16_t* gi = g + static_cast<long long>(n) * g_cstride + g_coff;
  const int step = gridDim.x * blockDim.x;
  for (int e0 = blockIdx.x * blockDim.x + threadIdx.x; e0 < total; e0 += step * GM_UNROLL) {
    uint4 q[GM_UNROLL], qg[GM_UNROLL];
    int pix[GM_UNROLL], grp[GM_UNROLL];
#pragma unroll
    for (int u = 0; u < GM_UNROLL; ++u) {
      const int e = e0 + u * step;
      // e / groups by a float reciprocal and one correction step (exact for e < 2^24)
      int pq = static_cast<int>(static_cast<float>(e) * inv_groups);
      int rm = e - pq * groups;
      if (rm < 0) { --pq; rm += groups; }
      if (rm >= groups) { ++pq; rm -= groups; }
      pix[u] = pq;
      grp[u] = rm;
      const bool ok = e < total;
      q[u] = ok ? *reinterpret_cast<const uint4*>(ai + pq * a_cstride + rm * 8) : make_uint4(0, 0, 0, 0);
      qg[u] = ok ? __ldg(reinterpret_cast<const uint4*>(gi + rm * 8)) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < GM_UNROLL; ++u) {
      if (e0 + u * step >= total) break;
      const int c0 = grp[u] * 8;
      float f[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = (ACT ? act_f(bfj(q[u], j), act) : bfj(q[u], j)) * bfj(qg[u], j);
      uint16_t* dst = yi + pix[u] * y_cstride + c0;
      if (c0 + 8 <= C) *reinterpret_cast<uint4*>(dst) = pack8(f);
      else store8(dst, pack8(f), C - c0);
    }
  }
}

// k x k / s average pool with zero padding counted (torch's count_include_pad=True).
__global__ void __launch_bounds__(256) avgpool2d_kernel(const uint16_t* __restrict__ x, int N, int H, int W, int C,
                                                        int x_cstride, int x_coff, int k, int s, int pad, int Ho,
                                                        int Wo, uint16_t* __restrict__ y, int y_cstride, int y_coff) {
  griddep_wait();
  griddep_launch_dependents();
  const int groups = (C + 7) / 8;
  const long long total = static_cast<long long>(N) * Ho * Wo * groups;
  const float inv = 1.f / static_cast<float>(k * k);
  for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < static_cast<unsigned>(total);
       e += gridDim.x * blockDim.x) {
    const unsigned pu = e / static_cast<unsigned>(groups);
    const long long p = pu;
    const int c0 = static_cast<int>(e - pu * groups) * 8;
    const int n = static_cast<int>(pu / static_cast<unsigned>(Ho * Wo));
    const int r = static_cast<int>(pu - static_cast<unsigned>(n) * Ho * Wo);
    const int yo = r / Wo, xo = r - yo * Wo;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int dy = 0; dy < k; ++dy) {
      const int yi = yo * s - pad + dy;
      if (yi < 0 || yi >= H) continue;
      for (int dx = 0; dx < k; ++dx) {
        const int xi = xo * s - pad + dx;
        if (xi < 0 || xi >= W) continue;
        const uint4 qv = *reinterpret_cast<const uint4*>(
            x + ((static_cast<long long>(n) * H + yi) * W + xi) * x_cstride + x_coff + c0);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += bfj(qv, j);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] *= inv;
    store8(y + p * y_cstride + y_coff + c0, pack8(acc), C - c0);
  }
}


// Depthwise k x k conv (groups == channels, multiplier 1) with the following BN folded
// into w/bias and the activation fused: y[n][yo][xo][c] = act(bias[c] +
// sum_{dy,dx} w[dy*k+dx][c] * x[n][yo*s-pad+dy][xo*s-pad+dx][c]).  MobileNetV3 /
// EfficientNetV2 lower it to a PER_CHANNEL-like interior node, so the
// planner permutes its filters with the channel order.  One thread per (output pixel,
// 8 channels): 16-byte input loads per tap (neighbouring pixels' taps hit L1), fp32
// accumulation, weights [k*k][C] fp32 read as float4 pairs.
__global__ void __launch_bounds__(256) dwconv_kernel(const uint16_t* __restrict__ x, int N, int H, int W, int C,
                                                     int x_cstride, int x_coff, const float* __restrict__ w,
                                                     const float* __restrict__ bias, int k, int s, int pad, int act,
                                                     int Ho, int Wo, uint16_t* __restrict__ y, int y_cstride,
                                                     int y_coff) {
  griddep_wait();
  griddep_launch_dependents();
  const int groups = (C + 7) / 8;
  const long long total = static_cast<long long>(N) * Ho * Wo * groups;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int g = static_cast<int>(e % groups);
    const long long p = e / groups;
    const int c0 = g * 8;
    const int n = static_cast<int>(p / (static_cast<long long>(Ho) * Wo));
    const int r = static_cast<int>(p - static_cast<long long>(n) * Ho * Wo);
    const int yo = r / Wo, xo = r - yo * Wo;
    float acc[8];
    if (bias) {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = c0 + j < C ? bias[c0 + j] : 0.f;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    }
    for (int dy = 0; dy < k; ++dy) {
      const int yi = yo * s - pad + dy;
      if (yi < 0 || yi >= H) continue;
      for (int dx = 0; dx < k; ++dx) {
        const int xi = xo * s - pad + dx;
        if (xi < 0 || xi >= W) continue;
        const uint4 qv = __ldg(reinterpret_cast<const uint4*>(
            x + ((static_cast<long long>(n) * H + yi) * W + xi) * x_cstride + x_coff + c0));
        const float* wt = w + static_cast<long long>(dy * k + dx) * ((C + 7) / 8 * 8) + c0;
        const float4 w0 = __ldg(reinterpret_cast<const float4*>(wt));
        const float4 w1 = __ldg(reinterpret_cast<const float4*>(wt + 4));
        acc[0] = fmaf(w0.x, bfj(qv, 0), acc[0]);
        acc[1] = fmaf(w0.y, bfj(qv, 1), acc[1]);
        acc[2] = fmaf(w0.z, bfj(qv, 2), acc[2]);
        acc[3] = fmaf(w0.w, bfj(qv, 3), acc[3]);
        acc[4] = fmaf(w1.x, bfj(qv, 4), acc[4]);
        acc[5] = fmaf(w1.y, bfj(qv, 5), acc[5]);
        acc[6] = fmaf(w1.z, bfj(qv, 6), acc[6]);
        acc[7] = fmaf(w1.w, bfj(qv, 7), acc[7]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = act_f(acc[j], act);
    store8(y + p * y_cstride + y_coff + c0, pack8(acc), C - c0);
  }
}


// Global average pool for small grids (few images x few channel groups, many pixels --
// MobileNet / EfficientNet squeeze-excitation pools at batch 1): a CTA takes one image and
// up to 32 groups of 8 channels; its 256 threads split the pixels into phases, each phase
// sums its pixels in order, and the phases are added in a fixed order (deterministic).
__global__ void __launch_bounds__(256) avgpool_split_kernel(const uint16_t* __restrict__ x, int HW, int C,
                                                            int x_cstride, int x_coff, uint16_t* __restrict__ y,
                                                            int y_cstride, int y_coff) {
  __shared__ float red[256 * 8];
  griddep_wait();
  griddep_launch_dependents();
  const int G = (C + 7) / 8;
  const int g0 = blockIdx.x * 32;
  const int gb = min(32, G - g0);
  const int phases = 256 / gb;
  const int n = blockIdx.y;
  const int t = threadIdx.x;
  const int g = t % gb, ph = t / gb;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (ph < phases) {
    const uint16_t* base = x + static_cast<long long>(n) * HW * x_cstride + x_coff + (g0 + g) * 8;
    for (int p = ph; p < HW; p += phases) {
      const uint4 qv = __ldg(reinterpret_cast<const uint4*>(base + static_cast<long long>(p) * x_cstride));
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += bfj(qv, j);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[t * 8 + j] = acc[j];
  __syncthreads();
  if (t < gb * 8) {
    const int gg = t >> 3, j = t & 7;
    float sum = 0.f;
    for (int q = 0; q < phases; ++q) sum += red[(q * gb + gg) * 8 + j];
    const int c = (g0 + gg) * 8 + j;
    if (c < C) y[static_cast<long long>(n) * y_cstride + y_coff + c] = tobf(sum / static_cast<float>(HW));
  }
}

// Small-M linear / 1x1 conv (M = images x pixels <= 16: squeeze-excitation FCs and
// classifiers at small batch): y[m][o] = act(sum_k x[m][xcol[k]] * w[o][k] + bias[o]).
// The M activation rows are gathered once into shared memory (fp32); one warp per output
// channel streams its weight row with 16-byte loads (every weight byte read once, spread
// over all SMs) and reduces the M dot products with shuffles.  CUDA cores: at M <= 16 a
// 128-row tensor-core tile would be >= 87 % padding and the launch is latency-bound.
__global__ void __launch_bounds__(256) linear_small_kernel(const uint16_t* __restrict__ x, int M, int x_cstride,
                                                           const int32_t* __restrict__ xcol, int K,
                                                           const uint16_t* __restrict__ w, int w_stride, int O,
                                                           const float* __restrict__ bias, int act, void* y,
                                                           int y_f32, int y_cstride, int y_coff) {
  extern __shared__ float xs[];  // [M][K8]
  const int K8 = (K + 7) / 8 * 8;
  griddep_wait();
  griddep_launch_dependents();
  // four elements per thread per step: their column-map loads, then their gathered loads
  // (a chain of two dependent round trips per element made the staging latency-bound at batch 1)
  for (int e0 = threadIdx.x; e0 < M * K8; e0 += 4 * blockDim.x) {
    int col[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x;
      const int m = e / K8, k = e - m * K8;
      col[u] = (e < M * K8 && k < K) ? __ldg(xcol + k) : -1;  // -1: a zero-filled GATHER entry
    }
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * blockDim.x;
      const int m = e / K8;
      v[u] = col[u] >= 0 ? bf(x[static_cast<long long>(m) * x_cstride + col[u]]) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (e0 + u * blockDim.x < M * K8) xs[e0 + u * blockDim.x] = v[u];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int o = blockIdx.x * 8 + warp; o < O; o += gridDim.x * 8) {
    float acc[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) acc[m] = 0.f;
    const uint16_t* wr = w + static_cast<long long>(o) * w_stride;
#pragma unroll 4
    for (int k = lane * 8; k < K8; k += 256) {
      const uint4 wq = __ldg(reinterpret_cast<const uint4*>(wr + k));
      float wf[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) wf[j] = bfj(wq, j);
#pragma unroll
      for (int m = 0; m < 16; ++m) {
        if (m < M) {
          const float4 a = *reinterpret_cast<const float4*>(xs + m * K8 + k);
          const float4 b = *reinterpret_cast<const float4*>(xs + m * K8 + k + 4);
          acc[m] += a.x * wf[0] + a.y * wf[1] + a.z * wf[2] + a.w * wf[3] + b.x * wf[4] + b.y * wf[5] + b.z * wf[6] +
                    b.w * wf[7];
        }
      }
    }
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      if (m < M) {
        float v = acc[m];
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        acc[m] = v;
      }
    }
    if (lane < M) {
      float v = 0.f;
#pragma unroll
      for (int m = 0; m < 16; ++m)
        if (m == lane) v = acc[m];
      if (bias) v += bias[o];
      v = act_f(v, act);
      const long long off = static_cast<long long>(lane) * y_cstride + y_coff + o;
      if (y_f32) static_cast<float*>(y)[off] = v;
      else static_cast<uint16_t*>(y)[off] = tobf(v);
    }
  }
}


// Depthwise conv, smem-tiled: a CTA computes an 8 x 8 output tile of one image for a block
// of up to 64 channels.  The input window ((8-1)*S + K)^2 x 64 ch is staged ONCE by 16-byte
// cp.async (zero-filled outside the image), the folded weights / bias of the block are
// staged too, then every (pixel, 8-channel group) output reads its K*K taps from shared
// memory.  HBM sees the input once (+ the tile halo) and the output once.
__host__ __device__ constexpr int dw_tile(int k, int s) { return (k == 5 && s == 2) ? 6 : 8; }

template <int K, int S>
__global__ void __launch_bounds__(256) dwconv_tile_kernel(const uint16_t* __restrict__ x, int N, int H, int W, int C,
                                                          int x_cstride, int x_coff, const float* __restrict__ w,
                                                          const float* __restrict__ bias, int pad, int act, int Ho,
                                                          int Wo, int tiles_h, int tiles_w,
                                                          uint16_t* __restrict__ y, int y_cstride, int y_coff) {
  constexpr int TH = dw_tile(K, S), TW = TH;  // the staged window fits the 48 KB static smem
  constexpr int IH = (TH - 1) * S + K, IW = (TW - 1) * S + K;
  __shared__ uint4 tile[IH * IW * 8];
  // the 8 filter values of group g sit at stride 12 floats: a quarter-warp's 16-byte weight
  // loads (8 groups) then hit 8 distinct bank quads (stride 8 gave 2-way conflicts, ncu)
  constexpr int WG = 12;
  __shared__ __align__(16) float sw[K * K * 8 * WG];
  __shared__ float sb[64];
  const int C8 = (C + 7) / 8 * 8;
  const int cb = blockIdx.y * 64;
  const int G = min(8, (C - cb + 7) / 8);
  const int t = blockIdx.x;
  const int n = t / (tiles_h * tiles_w);
  const int r = t - n * tiles_h * tiles_w;
  const int y0 = (r / tiles_w) * TH, x0 = (r % tiles_w) * TW;
  const int iy0 = y0 * S - pad, ix0 = x0 * S - pad;
  for (int e = threadIdx.x; e < K * K * 64; e += 256) {
    const int tap = e >> 6, c = e & 63;
    sw[tap * 8 * WG + (c >> 3) * WG + (c & 7)] = cb + c < C8 ? w[tap * C8 + cb + c] : 0.f;
  }
  if (threadIdx.x < 64) sb[threadIdx.x] = (bias && cb + threadIdx.x < C) ? bias[cb + threadIdx.x] : 0.f;
  griddep_wait();
  griddep_launch_dependents();
  for (int e = threadIdx.x; e < IH * IW * G; e += 256) {
    const int pix = e / G, g = e - (e / G) * G;
    const int iy = iy0 + pix / IW, ix = ix0 + pix % IW;
    uint4* dst = &tile[pix * 8 + g];
    if (iy >= 0 && iy < H && ix >= 0 && ix < W)
      cp_async16(dst, x + ((static_cast<long long>(n) * H + iy) * W + ix) * x_cstride + x_coff + cb + g * 8, 16);
    else
      *dst = make_uint4(0, 0, 0, 0);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  for (int e = threadIdx.x; e < TH * TW * G; e += 256) {
    const int op = e / G, g = e - (e / G) * G;
    const int oy = op / TW, ox = op - (op / TW) * TW;
    if (y0 + oy >= Ho || x0 + ox >= Wo) continue;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = sb[g * 8 + j];
#pragma unroll
    for (int dy = 0; dy < K; ++dy) {
#pragma unroll
      for (int dx = 0; dx < K; ++dx) {
        const uint4 q = tile[((oy * S + dy) * IW + ox * S + dx) * 8 + g];
        const float* wt = sw + (dy * K + dx) * 8 * WG + g * WG;
        const float4 w0 = *reinterpret_cast<const float4*>(wt);
        const float4 w1 = *reinterpret_cast<const float4*>(wt + 4);
        const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fmaf(wv[j], bfj(q, j), acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = act_f(acc[j], act);
    const int c0 = cb + g * 8;
    store8(y + ((static_cast<long long>(n) * Ho + y0 + oy) * Wo + x0 + ox) * y_cstride + y_coff + c0, pack8(acc),
           C - c0);
  }
}


// 3x3 depthwise conv, register strips: same staged 8 x 8 x 64-channel tile as above, but a
// thread owns 4 channels x one output column x a strip of DWS_R output rows.  Its 9 x 4
// filter values live in registers (loaded once), and each staged input pixel it needs is
// read from shared memory once per strip and applied to every output row of the strip it
// touches: (DWS_R - 1) * S + 3 rows x 3 columns of 8-byte loads for DWS_R x 4 outputs,
// against 9 input + 18 weight 16-byte loads per 8 outputs in the per-pixel form (which
// ncu showed shared-memory-bound).  A half-warp reads 16 x 8 contiguous bytes of a pixel.
constexpr int DWS_R = 4;
template <int S>
__global__ void __launch_bounds__(256) dwconv3_strip_kernel(const uint16_t* __restrict__ x, int N, int H, int W, int C,
                                                            int x_cstride, int x_coff, const float* __restrict__ w,
                                                            const float* __restrict__ bias, int pad, int act, int Ho,
                                                            int Wo, int tiles_h, int tiles_w,
                                                            uint16_t* __restrict__ y, int y_cstride, int y_coff,
                                                            float* __restrict__ part) {
  constexpr int K = 3, TH = 8, TW = 8;
  constexpr int IH = (TH - 1) * S + K, IW = (TW - 1) * S + K;
  static_assert(TH % DWS_R == 0 && (TH / DWS_R) * TW * 16 == 256, "one strip per thread");
  __shared__ uint4 tile[IH * IW * 8];
  __shared__ __align__(16) float sw[K * K * 64];
  __shared__ float sb[64];
  const int C8 = (C + 7) / 8 * 8;
  const int cb = blockIdx.y * 64;
  const int G = min(8, (C - cb + 7) / 8);
  const int t = blockIdx.x;
  const int n = t / (tiles_h * tiles_w);
  const int r = t - n * tiles_h * tiles_w;
  const int y0 = (r / tiles_w) * TH, x0 = (r % tiles_w) * TW;
  const int iy0 = y0 * S - pad, ix0 = x0 * S - pad;
  for (int e = threadIdx.x; e < K * K * 64; e += 256) {
    const int c = e & 63;
    sw[e] = cb + c < C8 ? w[(e >> 6) * C8 + cb + c] : 0.f;
  }
  if (threadIdx.x < 64) sb[threadIdx.x] = (bias && cb + threadIdx.x < C) ? bias[cb + threadIdx.x] : 0.f;
  griddep_wait();
  griddep_launch_dependents();
  for (int e = threadIdx.x; e < IH * IW * 8; e += 256) {
    const int pix = e >> 3, g = e & 7;
    if (g >= G) continue;
    const int iy = iy0 + pix / IW, ix = ix0 + pix % IW;
    uint4* dst = &tile[e];
    if (iy >= 0 && iy < H && ix >= 0 && ix < W)
      cp_async16(dst, x + ((static_cast<long long>(n) * H + iy) * W + ix) * x_cstride + x_coff + cb + g * 8, 16);
    else
      *dst = make_uint4(0, 0, 0, 0);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int hg = threadIdx.x & 15;          // 4-channel quarter of the 64-channel block
  const int ox = (threadIdx.x >> 4) & 7;    // output column in the tile
  const int oy0 = (threadIdx.x >> 7) * DWS_R;
  const int c0 = cb + hg * 4;
  const bool live = c0 < C && x0 + ox < Wo && y0 + oy0 < Ho;
  float psum[4] = {0.f, 0.f, 0.f, 0.f};  // this strip's stored (bf16-rounded) outputs, summed
  if (live) {
    float wr[K * K][4];
#pragma unroll
    for (int tap = 0; tap < K * K; ++tap) {
      const float4 v = *reinterpret_cast<const float4*>(&sw[tap * 64 + hg * 4]);
      wr[tap][0] = v.x; wr[tap][1] = v.y; wr[tap][2] = v.z; wr[tap][3] = v.w;
    }
    float acc[DWS_R][4];
#pragma unroll
    for (int q = 0; q < DWS_R; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[q][j] = sb[hg * 4 + j];
    const uint2* tile2 = reinterpret_cast<const uint2*>(tile);
#pragma unroll
    for (int i = 0; i < (DWS_R - 1) * S + K; ++i) {
#pragma unroll
      for (int dx = 0; dx < K; ++dx) {
        const uint2 v = tile2[((oy0 * S + i) * IW + ox * S + dx) * 16 + hg];
        const float f[4] = {__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u),
                            __uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u)};
#pragma unroll
        for (int q = 0; q < DWS_R; ++q) {
          const int dy = i - q * S;
          if (dy >= 0 && dy < K) {
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[q][j] = fmaf(wr[dy * K + dx][j], f[j], acc[q][j]);
          }
        }
      }
    }
    const int nc = min(4, C - c0);
#pragma unroll
    for (int q = 0; q < DWS_R; ++q) {
      if (y0 + oy0 + q >= Ho) break;
      const uint2 o = make_uint2(cvt_bf16x2(act_f(acc[q][0], act), act_f(acc[q][1], act)),
                                 cvt_bf16x2(act_f(acc[q][2], act), act_f(acc[q][3], act)));
      psum[0] += __uint_as_float(o.x << 16);
      psum[1] += __uint_as_float(o.x & 0xffff0000u);
      psum[2] += __uint_as_float(o.y << 16);
      psum[3] += __uint_as_float(o.y & 0xffff0000u);
      uint16_t* p = y + ((static_cast<long long>(n) * Ho + y0 + oy0 + q) * Wo + x0 + ox) * y_cstride + y_coff + c0;
      if (nc == 4) {
        *reinterpret_cast<uint2*>(p) = o;
      } else {
        for (int j = 0; j < nc; ++j) {
          const uint32_t h = j < 2 ? o.x : o.y;
          p[j] = static_cast<uint16_t>((j & 1) ? (h >> 16) : (h & 0xffffu));
        }
      }
    }
  }
  if (part) {
    // the SE global pool of the output, fused: per-channel sums of this tile, reduced over the
    // 16 strips of each 4-channel group in (now free) shared memory, one partial per tile
    // (deterministic: the consumer adds the image's tile partials in a fixed order)
    __syncthreads();
    float4* red = reinterpret_cast<float4*>(tile);
    red[threadIdx.x] = make_float4(psum[0], psum[1], psum[2], psum[3]);
    __syncthreads();
    if (threadIdx.x < 64 && cb + threadIdx.x < C8) {
      const float* rf = reinterpret_cast<const float*>(red);
      float s = 0.f;
#pragma unroll
      for (int it = 0; it < 16; ++it) s += rf[(it * 16 + (threadIdx.x >> 2)) * 4 + (threadIdx.x & 3)];
      part[static_cast<long long>(t) * C8 + cb + threadIdx.x] = s;
    }
  }
}


// The same register-strip 3x3 depthwise conv with the input window staged by ONE 4-D TMA box
// ([64 channels][IW][IH][1 image], zero-filled outside the image and past channel C) and the
// thread's filters / bias loaded straight from global (L2) into registers: the per-element
// staging address math, the cp.async issue and the shared-memory filter copy -- a third of
// the per-strip instruction stream in the cp.async form (ncu) -- disappear.
template <int S>
__global__ void __launch_bounds__(256) dwconv3_tma_kernel(const __grid_constant__ CUtensorMap tmx, int N, int C,
                                                          const float* __restrict__ w, const float* __restrict__ bias,
                                                          int pad, int act, int Ho, int Wo, int tiles_h, int tiles_w,
                                                          uint16_t* __restrict__ y, int y_cstride, int y_coff,
                                                          float* __restrict__ part) {
  constexpr int K = 3, TH = 8, TW = 8;
  constexpr int IH = (TH - 1) * S + K, IW = (TW - 1) * S + K;
  static_assert(TH % DWS_R == 0 && (TH / DWS_R) * TW * 16 == 256, "one strip per thread");
  __shared__ __align__(128) uint4 tile[IH * IW * 8];
  __shared__ uint64_t bar;
  const int C8 = (C + 7) / 8 * 8;
  const int cb = blockIdx.y * 64;
  const int t = blockIdx.x;
  const int n = t / (tiles_h * tiles_w);
  const int r = t - n * tiles_h * tiles_w;
  const int y0 = (r / tiles_w) * TH, x0 = (r % tiles_w) * TW;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    griddep_wait();
    mbar_arrive_expect_tx(&bar, IH * IW * 128);
    tma_load_4d(&tmx, &bar, tile, cb, x0 * S - pad, y0 * S - pad, n);
  }
  griddep_launch_dependents();
  const int hg = threadIdx.x & 15;
  const int ox = (threadIdx.x >> 4) & 7;
  const int oy0 = (threadIdx.x >> 7) * DWS_R;
  const int c0 = cb + hg * 4;
  const bool live = c0 < C && x0 + ox < Wo && y0 + oy0 < Ho;
  // filters as packed fp32 pairs (channels c0, c0+1 | c0+2, c0+3): the taps run on the
  // fma.f32x2 pipe, one instruction per two channels
  uint64_t wr[K * K][2];
  float bv[4] = {0.f, 0.f, 0.f, 0.f};
  if (live) {
#pragma unroll
    for (int tap = 0; tap < K * K; ++tap) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(w + tap * C8 + c0));
      wr[tap][0] = f2_bits(v.x, v.y);
      wr[tap][1] = f2_bits(v.z, v.w);
    }
    if (bias) {
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = c0 + j < C ? __ldg(bias + c0 + j) : 0.f;
    }
  }
  mbar_wait(&bar, 0);
  float psum[4] = {0.f, 0.f, 0.f, 0.f};
  if (live) {
    uint64_t acc[DWS_R][2];
#pragma unroll
    for (int q = 0; q < DWS_R; ++q) {
      acc[q][0] = f2_bits(bv[0], bv[1]);
      acc[q][1] = f2_bits(bv[2], bv[3]);
    }
    const uint2* tile2 = reinterpret_cast<const uint2*>(tile);
#pragma unroll
    for (int i = 0; i < (DWS_R - 1) * S + K; ++i) {
#pragma unroll
      for (int dx = 0; dx < K; ++dx) {
        const uint2 v = tile2[((oy0 * S + i) * IW + ox * S + dx) * 16 + hg];
        const uint64_t x01 = f2_bits(__uint_as_float(v.x << 16), __uint_as_float(v.x & 0xffff0000u));
        const uint64_t x23 = f2_bits(__uint_as_float(v.y << 16), __uint_as_float(v.y & 0xffff0000u));
#pragma unroll
        for (int q = 0; q < DWS_R; ++q) {
          const int dy = i - q * S;
          if (dy >= 0 && dy < K) {
            acc[q][0] = fma2(wr[dy * K + dx][0], x01, acc[q][0]);
            acc[q][1] = fma2(wr[dy * K + dx][1], x23, acc[q][1]);
          }
        }
      }
    }
    const int nc = min(4, C - c0);
#pragma unroll
    for (int q = 0; q < DWS_R; ++q) {
      if (y0 + oy0 + q >= Ho) break;
      const uint2 o = act_pack4(act, f2_lo(acc[q][0]), f2_hi(acc[q][0]), f2_lo(acc[q][1]), f2_hi(acc[q][1]));
      if (part) {
        psum[0] += __uint_as_float(o.x << 16);
        psum[1] += __uint_as_float(o.x & 0xffff0000u);
        psum[2] += __uint_as_float(o.y << 16);
        psum[3] += __uint_as_float(o.y & 0xffff0000u);
      }
      uint16_t* p = y + ((static_cast<long long>(n) * Ho + y0 + oy0 + q) * Wo + x0 + ox) * y_cstride + y_coff + c0;
      if (nc == 4) {
        *reinterpret_cast<uint2*>(p) = o;
      } else {
        for (int j = 0; j < nc; ++j) {
          const uint32_t h = j < 2 ? o.x : o.y;
          p[j] = static_cast<uint16_t>((j & 1) ? (h >> 16) : (h & 0xffffu));
        }
      }
    }
  }
  if (part) {
    // lanes l and l + 16 hold the same 4 channels (columns ox, ox + 1): one shuffle, then the
    // 8 warps' 64-channel rows through a small smem table and one barrier
    __shared__ float4 wred[8][16];
#pragma unroll
    for (int j = 0; j < 4; ++j) psum[j] += __shfl_xor_sync(0xffffffffu, psum[j], 16);
    if ((threadIdx.x & 31) < 16) wred[threadIdx.x >> 5][hg] = make_float4(psum[0], psum[1], psum[2], psum[3]);
    __syncthreads();
    if (threadIdx.x < 64 && cb + threadIdx.x < C8) {
      const float* rf = reinterpret_cast<const float*>(wred);
      float sum = 0.f;
#pragma unroll
      for (int wi = 0; wi < 8; ++wi) sum += rf[wi * 64 + threadIdx.x];
      part[static_cast<long long>(t) * C8 + cb + threadIdx.x] = sum;
    }
  }
}


// Direct stem conv on CUDA cores for few input channels (MobileNetV3 / EfficientNetV2:
// 3x3/s2 on the 3 image planes).  Reads the fp32 NCHW model input through the INPUT
// node's GATHER (idx), BN folded into w/bias, activation fused, NHWC bf16 out.  A CTA of
// 128 threads computes a 16 x 16 output tile: the cin input windows and all weights are
// staged in shared memory (the window's loads issued DS_BATCH at a time per thread, not as a
// chain of dependent round trips); a thread owns two pixels (rows oy, oy + 8) x a block of
// CB output channels, so each 16-byte weight broadcast feeds 8 FMAs and the channel block
// is pad8(cout) for narrow stems (no FMAs on padding channels beyond the next multiple of 8).
// At cin <= 4 the tensor-core im2col stem spends its time building a 9x-expanded operand;
// here the input is read once and the output written once.
constexpr int DS_TH = 16, DS_TW = 16, DS_THREADS = 128, DS_BATCH = 8;
template <int CB, int KT, int ST>  // KT / ST: compile-time filter size / stride (0: runtime k, s)
__global__ void __launch_bounds__(DS_THREADS) conv_direct_kernel(const float* __restrict__ x, int N, int C, int H,
                                                                 int W, const int32_t* __restrict__ idx, int cin,
                                                                 const float* __restrict__ w,
                                                                 const float* __restrict__ bias, int cout, int k_,
                                                                 int s_, int pad, int act, int Ho, int Wo,
                                                                 int tiles_h, int tiles_w, uint16_t* __restrict__ y,
                                                                 int y_cstride, int y_coff) {
  extern __shared__ float ds_smem[];
  const int k = KT ? KT : k_, s = ST ? ST : s_;
  const int IH = (DS_TH - 1) * s + k, IW = (DS_TW - 1) * s + k;
  const int coutp = (cout + CB - 1) / CB * CB;      // weight row length (multiple of CB)
  float* sx = ds_smem;                              // [cin][IH][IW]
  float* sw = sx + (cin * IH * IW + 3) / 4 * 4;     // [k*k*cin][coutp], 16-byte aligned rows
  float* sb = sw + k * k * cin * coutp;             // [coutp]
  const int t = blockIdx.x;
  const int n = t / (tiles_h * tiles_w);
  const int r = t - n * tiles_h * tiles_w;
  const int y0 = (r / tiles_w) * DS_TH, x0 = (r % tiles_w) * DS_TW;
  const int iy0 = y0 * s - pad, ix0 = x0 * s - pad;
  for (int e = threadIdx.x; e < k * k * cin * coutp; e += DS_THREADS) sw[e] = w[e];
  for (int e = threadIdx.x; e < coutp; e += DS_THREADS) sb[e] = (bias && e < cout) ? bias[e] : 0.f;
  griddep_wait();
  griddep_launch_dependents();
  const int total = cin * IH * IW;
  for (int e0 = threadIdx.x; e0 < total; e0 += DS_THREADS * DS_BATCH) {
    float v[DS_BATCH];
#pragma unroll
    for (int u = 0; u < DS_BATCH; ++u) {
      const int e = e0 + u * DS_THREADS;
      v[u] = 0.f;
      if (e < total) {
        const int row = e / IW, col = e - row * IW;
        const int c = row / IH;
        const int iy = iy0 + row - c * IH, ix = ix0 + col;
        if (iy >= 0 && iy < H && ix >= 0 && ix < W)
          v[u] = __ldg(x + ((static_cast<long long>(n) * C + __ldg(idx + c)) * H + iy) * W + ix);
      }
    }
#pragma unroll
    for (int u = 0; u < DS_BATCH; ++u)
      if (e0 + u * DS_THREADS < total) sx[e0 + u * DS_THREADS] = v[u];
  }
  __syncthreads();
  const int oy = threadIdx.x / DS_TW, ox = threadIdx.x % DS_TW;  // pixels (oy, ox) and (oy + 8, ox)
  const bool live0 = y0 + oy < Ho && x0 + ox < Wo, live1 = y0 + oy + 8 < Ho && x0 + ox < Wo;
  const int down = 8 * s * IW;
  for (int cb = 0; cb < coutp; cb += CB) {
    // channel pairs on the fma.f32x2 pipe: one instruction per two output channels
    uint64_t acc0[CB / 2], acc1[CB / 2];
#pragma unroll
    for (int j = 0; j < CB / 2; ++j) acc0[j] = acc1[j] = f2_bits(sb[cb + 2 * j], sb[cb + 2 * j + 1]);
    for (int c = 0; c < cin; ++c) {
#pragma unroll
      for (int dy = 0; dy < (KT ? KT : k); ++dy) {
        const float* row = sx + (c * IH + oy * s + dy) * IW + ox * s;
#pragma unroll
        for (int dx = 0; dx < (KT ? KT : k); ++dx) {
          const float v0 = row[dx], v1 = row[dx + down];
          const uint64_t p0 = f2_bits(v0, v0), p1 = f2_bits(v1, v1);
          const ulonglong2* wt = reinterpret_cast<const ulonglong2*>(sw + ((dy * k + dx) * cin + c) * coutp + cb);
#pragma unroll
          for (int j4 = 0; j4 < CB / 4; ++j4) {
            const ulonglong2 q = wt[j4];
            acc0[2 * j4] = fma2(q.x, p0, acc0[2 * j4]);
            acc0[2 * j4 + 1] = fma2(q.y, p0, acc0[2 * j4 + 1]);
            acc1[2 * j4] = fma2(q.x, p1, acc1[2 * j4]);
            acc1[2 * j4 + 1] = fma2(q.y, p1, acc1[2 * j4 + 1]);
          }
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!(h ? live1 : live0)) continue;
      float acc[CB];
#pragma unroll
      for (int j = 0; j < CB / 2; ++j) {
        acc[2 * j] = f2_lo(h ? acc1[j] : acc0[j]);
        acc[2 * j + 1] = f2_hi(h ? acc1[j] : acc0[j]);
      }
      uint16_t* yp = y + ((static_cast<long long>(n) * Ho + y0 + oy + 8 * h) * Wo + x0 + ox) * y_cstride + y_coff + cb;
      // whole 8-channel groups as 16-byte stores, then bf16 pairs, then a single channel
      // (2-byte stores at a 48-byte pixel pitch cost 14x the written bytes in L2 transactions)
      const int nc = cout - cb;
#pragma unroll
      for (int q = 0; q < CB / 8; ++q) {
        if (8 * q + 8 <= nc) {
          *reinterpret_cast<uint4*>(yp + q * 8) =
              act_pack8(act, acc[q * 8], acc[q * 8 + 1], acc[q * 8 + 2], acc[q * 8 + 3], acc[q * 8 + 4],
                        acc[q * 8 + 5], acc[q * 8 + 6], acc[q * 8 + 7]);
        } else if (8 * q < nc) {
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            if (8 * q + j + 2 <= nc)
              *reinterpret_cast<uint32_t*>(yp + q * 8 + j) =
                  cvt_bf16x2(act_f(acc[q * 8 + j], act), act_f(acc[q * 8 + j + 1], act));
            else if (8 * q + j < nc)
              yp[q * 8 + j] = tobf(act_f(acc[q * 8 + j], act));
          }
        }
      }
    }
  }
}


// Squeeze-excitation gate in one launch (MobileNetV3 / EfficientNetV2): per image,
//   pooled = mean_p x[n][p][:C]                       (PASS_THROUGH global pool)
//   h      = act1(W1 pooled + b1)   W1: [C1][ldw1]     (CHANNEL_MIX fc1 + bias + ReLU/SiLU)
//   gate   = act2(W2 h + b2)        W2: [C2][ldw2]     (CHANNEL_MIX fc2 + bias + hardsigmoid/sigmoid)
// replacing three launches (pool, fc1, fc2) by one CTA per image.  The fc reads (SLICE /
// GATHER of the pooled vector, of fc1's output) are folded into W1 / W2 as zero columns
// on the host.  Pooled and hidden vectors live in shared memory (fp32); a warp per output
// row streams its weight row with 16-byte loads.
// Dot products of RPW weight rows (bf16, 16-byte aligned, ld multiple of 8) with the fp32
// vector v (shared memory) by one warp: all rows' loads are issued before the FMAs.
template <int RPW>
__device__ __forceinline__ void warp_rows_dot(const uint16_t* __restrict__ w, int ld, int row0, int nrows,
                                              const float* v, int lane, float* out) {
  float acc[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) acc[r] = 0.f;
  for (int k = lane * 8; k < ld; k += 256) {
    uint4 wv[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r)
      wv[r] = row0 + r < nrows ? __ldg(reinterpret_cast<const uint4*>(w + static_cast<long long>(row0 + r) * ld + k))
                               : make_uint4(0, 0, 0, 0);
    float xv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) xv[e] = v[k + e];
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[r] = fmaf(bfj(wv[r], e), xv[e], acc[r]);
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], d);
    out[r] = acc[r];
  }
}

__global__ void __launch_bounds__(512) se_gate_kernel(const uint16_t* __restrict__ x, int HW, int C, int x_cstride,
                                                      int x_coff, const uint16_t* __restrict__ w1, int ldw1, int C1,
                                                      const float* __restrict__ b1, int act1,
                                                      const uint16_t* __restrict__ w2, int ldw2, int C2,
                                                      const float* __restrict__ b2, int act2,
                                                      uint16_t* __restrict__ gate, int g_cstride, int g_coff,
                                                      const float* __restrict__ part, int nparts,
                                                      int thread_rows) {
  constexpr int RPW = 8;  // weight rows per warp step (loads in flight)
  extern __shared__ float se_smem[];
  const int C8 = (C + 7) / 8 * 8, C18 = (C1 + 7) / 8 * 8;
  float* pooled = se_smem;            // [max(C8, ldw1)]
  float* hidden = pooled + (ldw1 > C8 ? ldw1 : C8);  // [max(C18, ldw2)]
  float* red = hidden + (ldw2 > C18 ? ldw2 : C18);   // [512 * 8] partial sums
  const int n = blockIdx.x;
  const int split = blockIdx.y, nsplit = gridDim.y;  // gate channels are split over nsplit CTAs
  const int t = threadIdx.x;
  griddep_wait();
  griddep_launch_dependents();
  if (part) {
    // ---- pool from the producer's per-tile partial sums (ub_dwconv_pool), in tile order
    const float* pp = part + static_cast<long long>(n) * nparts * C8;
    const float inv_hw = 1.f / static_cast<float>(HW);
    for (int c0 = t; c0 < C8; c0 += 4 * blockDim.x) {  // four channels' loads in flight per thread
      float sum[4] = {0.f, 0.f, 0.f, 0.f};
      for (int q = 0; q < nparts; ++q) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + u * blockDim.x;
          v[u] = c < C8 ? __ldg(pp + static_cast<long long>(q) * C8 + c) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) sum[u] += v[u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u * blockDim.x;
        if (c < C8) pooled[c] = c < C ? sum[u] * inv_hw : 0.f;
      }
    }
    __syncthreads();
  }
  // ---- pool: groups of 8 channels x pixel phases (4 independent loads in flight per thread)
  const int G = part ? 0 : C8 / 8;
  const uint16_t* base = x + static_cast<long long>(n) * HW * x_cstride + x_coff;
  for (int g0 = 0; g0 < G; g0 += 64) {
    const int gb = min(64, G - g0);
    const int phases = blockDim.x / gb;
    const int g = t % gb, ph = t / gb;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (ph < phases) {
      const uint16_t* col = base + (g0 + g) * 8;
      int p = ph;
      for (; p + 3 * phases < HW; p += 4 * phases) {
        uint4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          q[u] = __ldg(reinterpret_cast<const uint4*>(col + static_cast<long long>(p + u * phases) * x_cstride));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] += bfj(q[u], j);
        }
      }
      for (; p < HW; p += phases) {
        const uint4 qv = __ldg(reinterpret_cast<const uint4*>(col + static_cast<long long>(p) * x_cstride));
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += bfj(qv, j);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) red[t * 8 + j] = acc[j];
    __syncthreads();
    if (t < gb * 8) {
      const int gg = t >> 3, j = t & 7;
      float sum = 0.f;
      for (int q = 0; q < phases; ++q) sum += red[(q * gb + gg) * 8 + j];
      const int c = (g0 + gg) * 8 + j;
      pooled[c] = c < C ? sum / static_cast<float>(HW) : 0.f;
    }
    __syncthreads();
  }
  for (int c = C8 + t; c < ldw1; c += blockDim.x) pooled[c] = 0.f;
  __syncthreads();
  const int warp = t >> 5, lane = t & 31, warps = blockDim.x >> 5;
  // ---- fc1 (+ bias, act1): RPW hidden units per warp step
  for (int j0 = warp * RPW; j0 < C1; j0 += warps * RPW) {
    float o[RPW];
    warp_rows_dot<RPW>(w1, ldw1, j0, C1, pooled, lane, o);
    if (lane < RPW && j0 + lane < C1) {
      float v = 0.f;
#pragma unroll
      for (int r = 0; r < RPW; ++r)
        if (r == lane) v = o[r];
      hidden[j0 + lane] = act_f(v + (b1 ? b1[j0 + lane] : 0.f), act1);
    }
  }
  for (int j = C1 + t; j < (ldw2 > C18 ? ldw2 : C18); j += blockDim.x) hidden[j] = 0.f;
  __syncthreads();
  // ---- fc2 (+ bias, act2): this CTA's share of the gate channels, RPW per warp step
  const int per = (C2 + nsplit - 1) / nsplit;
  const int c_lo = split * per, c_hi = min(C2, c_lo + per);
  if (thread_rows) {
    // short rows (ldw2 <= 128, the usual SE squeeze width): a thread per gate channel, its
    // row's 16-byte chunks loaded four at a time, fc1 read from shared memory as broadcasts
    // (a warp per row would leave most lanes idle and pay a shuffle reduction per row)
    const int n8 = ldw2 >> 3;
    for (int c = c_lo + t; c < c_hi; c += blockDim.x) {
      const uint4* wr = reinterpret_cast<const uint4*>(w2 + static_cast<long long>(c) * ldw2);
      float acc = 0.f;
      for (int k8 = 0; k8 < n8; k8 += 8) {  // eight 16-byte chunks in flight (one round trip for <= 64 inputs)
        uint4 q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) q[u] = k8 + u < n8 ? __ldg(wr + k8 + u) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (k8 + u < n8) {
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = fmaf(bfj(q[u], e), hidden[(k8 + u) * 8 + e], acc);
          }
        }
      }
      gate[static_cast<long long>(n) * g_cstride + g_coff + c] = tobf(act_f(acc + (b2 ? b2[c] : 0.f), act2));
    }
    return;
  }
  for (int c0 = c_lo + warp * RPW; c0 < c_hi; c0 += warps * RPW) {
    float o[RPW];
    warp_rows_dot<RPW>(w2, ldw2, c0, c_hi, hidden, lane, o);
    if (lane < RPW && c0 + lane < c_hi) {
      float v = 0.f;
#pragma unroll
      for (int r = 0; r < RPW; ++r)
        if (r == lane) v = o[r];
      gate[static_cast<long long>(n) * g_cstride + g_coff + c0 + lane] =
          tobf(act_f(v + (b2 ? b2[c0 + lane] : 0.f), act2));
    }
  }
}

bool a16(const void* base, int cstride, int coff) {
  return base == nullptr || (aligned16(base) && (cstride & 7) == 0 && (coff & 7) == 0);
}

}  // namespace
}  // namespace ub

using namespace ub;

extern "C" int ub_eltwise(const ub_eltwise_desc* d, cudaStream_t stream) {
  if (!d || !d->a || !d->y || d->N < 1 || d->HW < 1 || d->C < 1 || d->act < UB_ACT_NONE || d->act > UB_ACT_SIGMOID)
    return fail(UB_EINVAL, "ub_eltwise: bad arguments");
  if (d->a_coff + d->C > d->a_cstride || d->y_coff + d->C > d->y_cstride ||
      (d->b && d->b_coff + d->C > d->b_cstride) || (d->gate && d->gate_coff + d->C > d->gate_cstride))
    return fail(UB_EINVAL, "ub_eltwise: channels exceed a row");
  const bool vec = a16(d->a, d->a_cstride, d->a_coff) && a16(d->y, d->y_cstride, d->y_coff) &&
                   a16(d->b, d->b_cstride, d->b_coff) && a16(d->gate, d->gate_cstride, d->gate_coff);
  const long long work = static_cast<long long>(d->N) * d->HW * (vec ? (d->C + 7) / 8 : d->C);
  if (work >= (1ll << 31)) return fail(UB_EUNSUPPORTED, "ub_eltwise: tensor too large");
  static const bool gate_fast = !std::getenv("UB_ELT_GENERIC");
  if (gate_fast && vec && d->gate && !d->b && !d->scale && !d->shift && d->N <= 65535 &&
      d->gate_coff + (d->C + 7) / 8 * 8 <= d->gate_cstride) {  // gate rows read as whole 16-byte groups
    const long long per_img = static_cast<long long>(d->HW) * ((d->C + 7) / 8);
    long long gx = (per_img + 256LL * GM_UNROLL - 1) / (256LL * GM_UNROLL);
    if (gx < 1) gx = 1;
    if (per_img >= (1ll << 24) || static_cast<long long>(d->HW) * d->a_cstride >= (1ll << 31) ||
        static_cast<long long>(d->HW) * d->y_cstride >= (1ll << 31))
      return fail(UB_EUNSUPPORTED, "ub_eltwise: image too large for the gate kernel");
    const cudaError_t e = launch_pdl(d->act == UB_ACT_NONE ? gate_mul_kernel<false> : gate_mul_kernel<true>,
                                     dim3(static_cast<unsigned>(gx), d->N), dim3(256), 0, stream,
                                     static_cast<const uint16_t*>(d->a), d->a_cstride, d->a_coff,
                                     static_cast<const uint16_t*>(d->gate), d->gate_cstride, d->gate_coff,
                                     static_cast<uint16_t*>(d->y), d->y_cstride, d->y_coff, d->HW, d->C, d->act);
    count_launch();
    return cuda_status(e, "eltwise_kernel");
  }
  const int grid = grid_for(work, 256, 2);
  const cudaError_t e = vec ? launch_pdl(eltwise_kernel<true>, dim3(grid), dim3(256), 0, stream, *d)
                            : launch_pdl(eltwise_kernel<false>, dim3(grid), dim3(256), 0, stream, *d);
  count_launch();
  return cuda_status(e, "eltwise_kernel");
}

extern "C" int ub_avgpool2d(const void* x, int N, int H, int W, int C, int x_cstride, int x_coff, int k, int s,
                            int pad, int Ho, int Wo, void* y, int y_cstride, int y_coff, cudaStream_t stream) {
  if (!x || !y || N < 1 || H < 1 || W < 1 || C < 1 || k < 1 || s < 1 || pad < 0 || Ho < 1 || Wo < 1)
    return fail(UB_EINVAL, "ub_avgpool2d: bad arguments");
  if (!a16(x, x_cstride, x_coff) || !a16(y, y_cstride, y_coff) || x_coff + C > x_cstride || y_coff + C > y_cstride)
    return fail(UB_EINVAL, "ub_avgpool2d: rows must be 16-byte aligned");
  const long long work = static_cast<long long>(N) * Ho * Wo * ((C + 7) / 8);
  if (work >= (1ll << 31)) return fail(UB_EUNSUPPORTED, "ub_avgpool2d: tensor too large");
  const cudaError_t e = launch_pdl(avgpool2d_kernel, dim3(grid_for(work, 256, 2)), dim3(256), 0, stream,
                                   static_cast<const uint16_t*>(x), N, H, W, C, x_cstride, x_coff, k, s, pad, Ho, Wo,
                                   static_cast<uint16_t*>(y), y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "avgpool2d_kernel");
}

// tiles per image of the register-strip 3x3 form, i.e. the SE pool partials ub_dwconv_pool
// writes per image; 0 when the shape takes another form (no fused pool)
static bool dw_strips_enabled() {
  static const bool on = !std::getenv("UB_DW_NOSTRIP");
  return on;
}

extern "C" int ub_dwconv_pool_parts(int k, int s, int Ho, int Wo) {
  if (k != 3 || (s != 1 && s != 2) || Ho < 1 || Wo < 1 || !dw_strips_enabled()) return 0;
  return ((Ho + 7) / 8) * ((Wo + 7) / 8);
}

extern "C" int ub_dwconv_pool(const void* x, int N, int H, int W, int C, int x_cstride, int x_coff, const float* w,
                              const float* bias, int k, int s, int pad, int act, int Ho, int Wo, void* y, int y_cstride,
                              int y_coff, float* part, cudaStream_t stream) {
  if (!x || !w || !y || N < 1 || H < 1 || W < 1 || C < 1 || k < 1 || s < 1 || pad < 0 || Ho < 1 || Wo < 1 ||
      act < UB_ACT_NONE || act > UB_ACT_SIGMOID)
    return fail(UB_EINVAL, "ub_dwconv: bad arguments");
  if (!a16(x, x_cstride, x_coff) || !a16(y, y_cstride, y_coff) || x_coff + C > x_cstride || y_coff + C > y_cstride ||
      (reinterpret_cast<uintptr_t>(w) & 15))
    return fail(UB_EINVAL, "ub_dwconv: rows must be 16-byte aligned");
  if (part && (ub_dwconv_pool_parts(k, s, Ho, Wo) == 0 || (reinterpret_cast<uintptr_t>(part) & 3)))
    return fail(UB_EUNSUPPORTED, "ub_dwconv_pool: fused pool needs the 3x3 strip form (k %d s %d)", k, s);
  if ((k == 3 || k == 5) && (s == 1 || s == 2)) {  // smem-tiled forms
    const int tsz = dw_tile(k, s);
    const int th = (Ho + tsz - 1) / tsz, tw = (Wo + tsz - 1) / tsz;
    const long long tiles = static_cast<long long>(N) * th * tw;
    if (tiles < (1ll << 31)) {
      const dim3 grid(static_cast<unsigned>(tiles), (C + 63) / 64);
      cudaError_t e;
      static const bool use_tma = !std::getenv("UB_DW_NOTMA");
      CUtensorMap tmx{};
      bool tma_ok = false;
      if (k == 3 && dw_strips_enabled() && use_tma) {
        const int ih = 7 * s + 3;
        const cuuint64_t xs = static_cast<cuuint64_t>(x_cstride) * 2;
        cuuint64_t xd[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                            static_cast<cuuint64_t>(N)};
        cuuint64_t xst[3] = {xs, xs * W, xs * W * H};
        cuuint32_t xb[4] = {64, static_cast<cuuint32_t>(ih), static_cast<cuuint32_t>(ih), 1};
        cuuint32_t xe[4] = {1, 1, 1, 1};
        tma_ok = encode_tiled_fn()(&tmx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                                   const_cast<uint16_t*>(static_cast<const uint16_t*>(x)) + x_coff, xd, xst, xb, xe,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        if (tma_ok) apply_small_tensor_quirk(&tmx, static_cast<size_t>(N) * H * W * x_cstride * 2);
      }
      if (tma_ok) {
        e = launch_pdl(s == 1 ? dwconv3_tma_kernel<1> : dwconv3_tma_kernel<2>, grid, dim3(256), 0, stream, tmx, N, C,
                       w, bias, pad, act, Ho, Wo, th, tw, static_cast<uint16_t*>(y), y_cstride, y_coff, part);
      } else if (k == 3 && dw_strips_enabled()) {
        e = launch_pdl(s == 1 ? dwconv3_strip_kernel<1> : dwconv3_strip_kernel<2>, grid, dim3(256), 0, stream,
                       static_cast<const uint16_t*>(x), N, H, W, C, x_cstride, x_coff, w, bias, pad, act, Ho, Wo, th,
                       tw, static_cast<uint16_t*>(y), y_cstride, y_coff, part);
      } else {
        void (*kern)(const uint16_t*, int, int, int, int, int, int, const float*, const float*, int, int, int, int,
                     int, int, uint16_t*, int, int) =
            k == 3 ? (s == 1 ? dwconv_tile_kernel<3, 1> : dwconv_tile_kernel<3, 2>)
                   : (s == 1 ? dwconv_tile_kernel<5, 1> : dwconv_tile_kernel<5, 2>);
        e = launch_pdl(kern, grid, dim3(256), 0, stream, static_cast<const uint16_t*>(x), N, H, W, C, x_cstride,
                       x_coff, w, bias, pad, act, Ho, Wo, th, tw, static_cast<uint16_t*>(y), y_cstride, y_coff);
      }
      count_launch();
      return cuda_status(e, "dwconv_tile_kernel");
    }
  }
  const long long work = static_cast<long long>(N) * Ho * Wo * ((C + 7) / 8);
  const cudaError_t e = launch_pdl(dwconv_kernel, dim3(grid_for(work, 256, 1)), dim3(256), 0, stream,
                                   static_cast<const uint16_t*>(x), N, H, W, C, x_cstride, x_coff, w, bias, k, s, pad,
                                   act, Ho, Wo, static_cast<uint16_t*>(y), y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "dwconv_kernel");
}

extern "C" int ub_dwconv(const void* x, int N, int H, int W, int C, int x_cstride, int x_coff, const float* w,
                         const float* bias, int k, int s, int pad, int act, int Ho, int Wo, void* y, int y_cstride,
                         int y_coff, cudaStream_t stream) {
  return ub_dwconv_pool(x, N, H, W, C, x_cstride, x_coff, w, bias, k, s, pad, act, Ho, Wo, y, y_cstride, y_coff,
                        nullptr, stream);
}

extern "C" int ub_avgpool_split(const void* x, int N, int HW, int C, int x_cstride, int x_coff, void* y, int y_cstride,
                                int y_coff, cudaStream_t stream) {
  if (!x || !y || N < 1 || HW < 1 || C < 1 || N > 65535) return fail(UB_EINVAL, "ub_avgpool_split: bad arguments");
  if (!a16(x, x_cstride, x_coff) || x_coff + (C + 7) / 8 * 8 > x_cstride || y_coff + C > y_cstride)
    return fail(UB_EINVAL, "ub_avgpool_split: rows must be 16-byte aligned");
  const dim3 grid(((C + 7) / 8 + 31) / 32, N);
  const cudaError_t e = launch_pdl(avgpool_split_kernel, grid, dim3(256), 0, stream, static_cast<const uint16_t*>(x),
                                   HW, C, x_cstride, x_coff, static_cast<uint16_t*>(y), y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "avgpool_split_kernel");
}

extern "C" int ub_linear_small(const void* x, int M, int x_cstride, const int32_t* xcol, int K, const void* w,
                               int w_stride, int O, const float* bias, int act, void* y, int y_dtype, int y_cstride,
                               int y_coff, cudaStream_t stream) {
  if (!x || !xcol || !w || !y || M < 1 || M > 16 || K < 1 || O < 1 || act < UB_ACT_NONE || act > UB_ACT_SIGMOID)
    return fail(UB_EINVAL, "ub_linear_small: bad arguments (M must be 1..16)");
  if ((w_stride & 7) || w_stride < (K + 7) / 8 * 8 || (reinterpret_cast<uintptr_t>(w) & 15) ||
      y_coff + O > y_cstride || (y_dtype != UB_BF16 && y_dtype != UB_F32))
    return fail(UB_EINVAL, "ub_linear_small: weight rows must be 16-byte aligned and hold pad8(K) columns");
  const size_t smem = static_cast<size_t>(M) * ((K + 7) / 8 * 8) * sizeof(float);
  if (smem > 200 * 1024) return fail(UB_EUNSUPPORTED, "ub_linear_small: M x K too large");
  if (const cudaError_t ae = ensure_max_smem(linear_small_kernel)) return cuda_status(ae, "linear_small attr");
  int grid = (O + 7) / 8;
  if (grid > 4 * num_sms()) grid = 4 * num_sms();
  const cudaError_t e = launch_pdl(linear_small_kernel, dim3(grid), dim3(256), smem, stream,
                                   static_cast<const uint16_t*>(x), M, x_cstride, xcol, K,
                                   static_cast<const uint16_t*>(w), w_stride, O, bias, act, y,
                                   y_dtype == UB_F32 ? 1 : 0, y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "linear_small_kernel");
}

// the channel block of ub_conv_direct for a given cout: pad8(cout) up to 32, else 32
int direct_cb(int cout) { return cout >= 32 ? 32 : (cout + 7) / 8 * 8; }

extern "C" int ub_conv_direct_wcols(int cout) {
  const int cb = direct_cb(cout);
  return (cout + cb - 1) / cb * cb;
}

extern "C" int ub_conv_direct(const float* x, int N, int C, int H, int W, const int32_t* idx, int cin, const float* w,
                              const float* bias, int cout, int k, int s, int pad, int act, void* y, int y_cstride,
                              int y_coff, cudaStream_t stream) {
  if (!x || !idx || !w || !y || N < 1 || C < 1 || H < 1 || W < 1 || cin < 1 || cout < 1 || k < 1 || s < 1 ||
      pad < 0 || act < UB_ACT_NONE || act > UB_ACT_SIGMOID)
    return fail(UB_EINVAL, "ub_conv_direct: bad arguments");
  if (cin > 8 || k > 7 || cout > 256) return fail(UB_EUNSUPPORTED, "ub_conv_direct: cin %d k %d cout %d", cin, k, cout);
  if (!a16(y, y_cstride, y_coff) || y_coff + cout > y_cstride || (reinterpret_cast<uintptr_t>(w) & 15))
    return fail(UB_EINVAL, "ub_conv_direct: output rows / weights must be 16-byte aligned");
  const int Ho = (H + 2 * pad - k) / s + 1, Wo = (W + 2 * pad - k) / s + 1;
  const int IH = (DS_TH - 1) * s + k, IW = (DS_TW - 1) * s + k;
  const int cb = direct_cb(cout), coutp = ub_conv_direct_wcols(cout);
  const size_t smem =
      ((static_cast<size_t>(cin) * IH * IW + 3) / 4 * 4 + static_cast<size_t>(k) * k * cin * coutp + coutp) * 4;
  if (smem > 200 * 1024) return fail(UB_EUNSUPPORTED, "ub_conv_direct: shared memory");
  void (*kern)(const float*, int, int, int, int, const int32_t*, int, const float*, const float*, int, int, int, int,
               int, int, int, int, int, uint16_t*, int, int);
  if (k == 3 && s == 2)  // the MobileNetV3 / EfficientNetV2 stems: unrolled taps, constant window geometry
    kern = cb == 8 ? conv_direct_kernel<8, 3, 2> : cb == 16 ? conv_direct_kernel<16, 3, 2>
         : cb == 24 ? conv_direct_kernel<24, 3, 2> : conv_direct_kernel<32, 3, 2>;
  else
    kern = cb == 8 ? conv_direct_kernel<8, 0, 0> : cb == 16 ? conv_direct_kernel<16, 0, 0>
         : cb == 24 ? conv_direct_kernel<24, 0, 0> : conv_direct_kernel<32, 0, 0>;
  if (const cudaError_t ae = ensure_max_smem(kern)) return cuda_status(ae, "conv_direct attr");
  const int th = (Ho + DS_TH - 1) / DS_TH, tw = (Wo + DS_TW - 1) / DS_TW;
  const long long tiles = static_cast<long long>(N) * th * tw;
  if (tiles >= (1ll << 31)) return fail(UB_EUNSUPPORTED, "ub_conv_direct: too many tiles");
  const cudaError_t e = launch_pdl(kern, dim3(static_cast<unsigned>(tiles)), dim3(DS_THREADS), smem, stream, x, N, C,
                                   H, W, idx, cin, w, bias, cout, k, s, pad, act, Ho, Wo, th, tw,
                                   static_cast<uint16_t*>(y), y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "conv_direct_kernel");
}

extern "C" int ub_se_gate_parts(const void* x, int N, int HW, int C, int x_cstride, int x_coff, const void* w1,
                                int ldw1, int C1, const float* b1, int act1, const void* w2, int ldw2, int C2,
                                const float* b2, int act2, void* gate, int g_cstride, int g_coff, const float* part,
                                int nparts, cudaStream_t stream) {
  if ((!x && !part) || (part && nparts < 1) || !w1 || !w2 || !gate || N < 1 || HW < 1 || C < 1 || C1 < 1 || C2 < 1 ||
      act1 < UB_ACT_NONE || act1 > UB_ACT_SIGMOID || act2 < UB_ACT_NONE || act2 > UB_ACT_SIGMOID)
    return fail(UB_EINVAL, "ub_se_gate: bad arguments");
  if ((!part && (!a16(x, x_cstride, x_coff) || x_coff + (C + 7) / 8 * 8 > x_cstride)) || (ldw1 & 7) ||
      ldw1 < (C + 7) / 8 * 8 || (ldw2 & 7) || ldw2 < (C1 + 7) / 8 * 8 || (reinterpret_cast<uintptr_t>(w1) & 15) ||
      (reinterpret_cast<uintptr_t>(w2) & 15) || g_coff + C2 > g_cstride)
    return fail(UB_EINVAL, "ub_se_gate: rows must be 16-byte aligned / weight rows too short");
  const int C8 = (C + 7) / 8 * 8, C18 = (C1 + 7) / 8 * 8;
  const size_t smem = (static_cast<size_t>(ldw1 > C8 ? ldw1 : C8) + (ldw2 > C18 ? ldw2 : C18) + 512 * 8) * 4;
  if (smem > 200 * 1024) return fail(UB_EUNSUPPORTED, "ub_se_gate: vectors too wide");
  if (const cudaError_t ae = ensure_max_smem(se_gate_kernel)) return cuda_status(ae, "se_gate attr");
  // few images: split the gate channels over several CTAs per image (each recomputes the
  // cheap pool + fc1) so the fc2 weight stream is spread over more SMs
  int nsplit = num_sms() / N;
  nsplit = nsplit < 1 ? 1 : (nsplit > 16 ? 16 : nsplit);
  if (nsplit > (C2 + 63) / 64) nsplit = (C2 + 63) / 64;
  static const bool rows_env = !std::getenv("UB_SE_WARPROWS");
  const bool thread_rows = rows_env && ldw2 <= 128;
  const cudaError_t e = launch_pdl(se_gate_kernel, dim3(N, nsplit), dim3(512), smem, stream, static_cast<const uint16_t*>(x),
                                   HW, C, x_cstride, x_coff, static_cast<const uint16_t*>(w1), ldw1, C1, b1, act1,
                                   static_cast<const uint16_t*>(w2), ldw2, C2, b2, act2, static_cast<uint16_t*>(gate),
                                   g_cstride, g_coff, part, nparts, thread_rows ? 1 : 0);
  count_launch();
  return cuda_status(e, "se_gate_kernel");
}

extern "C" int ub_se_gate(const void* x, int N, int HW, int C, int x_cstride, int x_coff, const void* w1, int ldw1,
                          int C1, const float* b1, int act1, const void* w2, int ldw2, int C2, const float* b2,
                          int act2, void* gate, int g_cstride, int g_coff, cudaStream_t stream) {
  if (!x) return fail(UB_EINVAL, "ub_se_gate: bad arguments");
  return ub_se_gate_parts(x, N, HW, C, x_cstride, x_coff, w1, ldw1, C1, b1, act1, w2, ldw2, C2, b2, act2, gate,
                          g_cstride, g_coff, nullptr, 0, stream);
}

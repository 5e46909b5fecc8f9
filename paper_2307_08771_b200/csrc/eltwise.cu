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
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long p = e / groups;
    const int c0 = static_cast<int>(e - p * groups) * (VEC ? 8 : 1);
    const int n = static_cast<int>(p / d.HW);
    if (VEC) {
      uint16_t va[8], vb[8], vg[8], vy[8];
      *reinterpret_cast<uint4*>(va) = *reinterpret_cast<const uint4*>(a + p * d.a_cstride + d.a_coff + c0);
      if (b) *reinterpret_cast<uint4*>(vb) = *reinterpret_cast<const uint4*>(b + p * d.b_cstride + d.b_coff + c0);
      if (g) *reinterpret_cast<uint4*>(vg) = *reinterpret_cast<const uint4*>(g + static_cast<long long>(n) *
                                                                                   d.gate_cstride + d.gate_coff + c0);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = c0 + j < d.C ? c0 + j : d.C - 1;
        float v = bf(va[j]);
        if (d.scale) v *= d.scale[c];
        if (d.shift) v += d.shift[c];
        if (b) v += bf(vb[j]);
        v = act_f(v, d.act);
        if (g) v *= bf(vg[j]);
        vy[j] = tobf(v);
      }
      if (c0 + 8 <= d.C) {
        *reinterpret_cast<uint4*>(y + p * d.y_cstride + d.y_coff + c0) = *reinterpret_cast<const uint4*>(vy);
      } else {
        for (int j = 0; c0 + j < d.C; ++j) y[p * d.y_cstride + d.y_coff + c0 + j] = vy[j];
      }
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

// k x k / s average pool with zero padding counted (torch's count_include_pad=True).
__global__ void __launch_bounds__(256) avgpool2d_kernel(const uint16_t* __restrict__ x, int N, int H, int W, int C,
                                                        int x_cstride, int x_coff, int k, int s, int pad, int Ho,
                                                        int Wo, uint16_t* __restrict__ y, int y_cstride, int y_coff) {
  griddep_wait();
  griddep_launch_dependents();
  const int groups = (C + 7) / 8;
  const long long total = static_cast<long long>(N) * Ho * Wo * groups;
  const float inv = 1.f / static_cast<float>(k * k);
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long p = e / groups;
    const int c0 = static_cast<int>(e - p * groups) * 8;
    const int n = static_cast<int>(p / (static_cast<long long>(Ho) * Wo));
    const int r = static_cast<int>(p - static_cast<long long>(n) * Ho * Wo);
    const int yo = r / Wo, xo = r - yo * Wo;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int dy = 0; dy < k; ++dy) {
      const int yi = yo * s - pad + dy;
      if (yi < 0 || yi >= H) continue;
      for (int dx = 0; dx < k; ++dx) {
        const int xi = xo * s - pad + dx;
        if (xi < 0 || xi >= W) continue;
        uint16_t v[8];
        *reinterpret_cast<uint4*>(v) = *reinterpret_cast<const uint4*>(
            x + ((static_cast<long long>(n) * H + yi) * W + xi) * x_cstride + x_coff + c0);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += bf(v[j]);
      }
    }
    uint16_t o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = tobf(acc[j] * inv);
    uint16_t* yp = y + p * y_cstride + y_coff + c0;
    if (c0 + 8 <= C) {
      *reinterpret_cast<uint4*>(yp) = *reinterpret_cast<const uint4*>(o);
    } else {
      for (int j = 0; c0 + j < C; ++j) yp[j] = o[j];
    }
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
        uint16_t v[8];
        *reinterpret_cast<uint4*>(v) = __ldg(reinterpret_cast<const uint4*>(
            x + ((static_cast<long long>(n) * H + yi) * W + xi) * x_cstride + x_coff + c0));
        const float* wt = w + static_cast<long long>(dy * k + dx) * ((C + 7) / 8 * 8) + c0;
        const float4 w0 = __ldg(reinterpret_cast<const float4*>(wt));
        const float4 w1 = __ldg(reinterpret_cast<const float4*>(wt + 4));
        acc[0] = fmaf(w0.x, bf(v[0]), acc[0]);
        acc[1] = fmaf(w0.y, bf(v[1]), acc[1]);
        acc[2] = fmaf(w0.z, bf(v[2]), acc[2]);
        acc[3] = fmaf(w0.w, bf(v[3]), acc[3]);
        acc[4] = fmaf(w1.x, bf(v[4]), acc[4]);
        acc[5] = fmaf(w1.y, bf(v[5]), acc[5]);
        acc[6] = fmaf(w1.z, bf(v[6]), acc[6]);
        acc[7] = fmaf(w1.w, bf(v[7]), acc[7]);
      }
    }
    uint16_t o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = tobf(act_f(acc[j], act));
    uint16_t* yp = y + p * y_cstride + y_coff + c0;
    if (c0 + 8 <= C) {
      *reinterpret_cast<uint4*>(yp) = *reinterpret_cast<const uint4*>(o);
    } else {
      for (int j = 0; c0 + j < C; ++j) yp[j] = o[j];
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
  const cudaError_t e = launch_pdl(avgpool2d_kernel, dim3(grid_for(work, 256, 2)), dim3(256), 0, stream,
                                   static_cast<const uint16_t*>(x), N, H, W, C, x_cstride, x_coff, k, s, pad, Ho, Wo,
                                   static_cast<uint16_t*>(y), y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "avgpool2d_kernel");
}

extern "C" int ub_dwconv(const void* x, int N, int H, int W, int C, int x_cstride, int x_coff, const float* w,
                         const float* bias, int k, int s, int pad, int act, int Ho, int Wo, void* y, int y_cstride,
                         int y_coff, cudaStream_t stream) {
  if (!x || !w || !y || N < 1 || H < 1 || W < 1 || C < 1 || k < 1 || s < 1 || pad < 0 || Ho < 1 || Wo < 1 ||
      act < UB_ACT_NONE || act > UB_ACT_SIGMOID)
    return fail(UB_EINVAL, "ub_dwconv: bad arguments");
  if (!a16(x, x_cstride, x_coff) || !a16(y, y_cstride, y_coff) || x_coff + C > x_cstride || y_coff + C > y_cstride ||
      (reinterpret_cast<uintptr_t>(w) & 15))
    return fail(UB_EINVAL, "ub_dwconv: rows must be 16-byte aligned");
  const long long work = static_cast<long long>(N) * Ho * Wo * ((C + 7) / 8);
  const cudaError_t e = launch_pdl(dwconv_kernel, dim3(grid_for(work, 256, 1)), dim3(256), 0, stream,
                                   static_cast<const uint16_t*>(x), N, H, W, C, x_cstride, x_coff, w, bias, k, s, pad,
                                   act, Ho, Wo, static_cast<uint16_t*>(y), y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "dwconv_kernel");
}

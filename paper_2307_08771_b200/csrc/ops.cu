// Memory-bound kernels of the hot path: the export-time permute (apply_plan's
// weight math), the baseline export's channel gather, input staging and pools.
// All are HBM-bound: coalesced on the side that is contiguous, vectorised where
// the layout allows, grids sized in multiples of the SM count.
#include <cuda_bf16.h>

#include <algorithm>

#include "ub_common.cuh"
#include "ub_host.h"

namespace ub {
namespace {



template <typename T>
__device__ __forceinline__ float to_f(T v) { return static_cast<float>(v); }

// Plan indices that point outside the source tensor (a bad or mismatched plan file):
// the kernels read nothing for them and count them here; ub_index_faults() reports.
__device__ unsigned long long g_index_faults = 0;

// ------------------------------------------------------------- permute weights
// planner.py:661-673 (rows) + 755-767 (columns), both sides of a layer fused.
// Iterates over OUTPUT elements so the writes are coalesced; reads gather.
template <typename TI, typename TO, int LAYOUT>
__global__ void permute_weights_kernel(const TI* __restrict__ W, int O, int I, int taps, const int32_t* __restrict__ rows,
                                       int n_rows, const int32_t* __restrict__ cols, int n_cols,
                                       const float* __restrict__ scale, int lead, int cpad, TO* __restrict__ out,
                                       long long total) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int r, c, t;
    bool inside = true;
    if (LAYOUT == UB_LAYOUT_OIHW) {  // [r][c][t]
      t = static_cast<int>(e % taps);
      long long rc = e / taps;
      c = static_cast<int>(rc % n_cols);
      r = static_cast<int>(rc / n_cols);
    } else if (LAYOUT == UB_LAYOUT_S2D) {  // [r][dy][dx][(py*2+px)*n_cols + c], kw passed as `lead`
      const int kw = lead, kq = (lead + 1) / 2;
      const int k = static_cast<int>(e % cpad);
      r = static_cast<int>(e / cpad);
      const int tq = k >> 3, slot = k & 7;
      const int dy = tq / kq, dx = tq - (tq / kq) * kq;
      const int q = slot / n_cols;
      c = slot - q * n_cols;
      const int fr = 2 * dy + (q >> 1), fs = 2 * dx + (q & 1);
      inside = q < 4 && fr < taps / kw && fs < kw;
      t = fr * kw + fs;
    } else if (LAYOUT == UB_LAYOUT_GEMM_DENSE) {  // [r][k], k = t * n_cols + c
      const int k = static_cast<int>(e % cpad);
      r = static_cast<int>(e / cpad);
      t = k / n_cols;
      c = k - t * n_cols;
      inside = t < taps;
    } else {  // [r][t][k], column c at k = lead + c
      const int k = static_cast<int>(e % cpad);
      long long rt = e / cpad;
      t = static_cast<int>(rt % taps);
      r = static_cast<int>(rt / taps);
      c = k - lead;
      inside = c >= 0 && c < n_cols;
    }
    TO v = TO(0);
    if (inside) {
      const int src_r = rows[r];
      const int src_c = cols[c];
      if (src_r >= O || src_c >= I) {
        atomicAdd(&g_index_faults, 1ull);
      } else if (src_r >= 0 && src_c >= 0) {
        const TI w = W[((long long)src_r * I + src_c) * taps + t];
        if (scale) {
          v = static_cast<TO>(static_cast<float>(w) * scale[r]);
        } else {
          v = static_cast<TO>(w);
        }
      }
    }
    out[e] = v;
  }
}

template <typename TI, typename TO>
int permute_dispatch_layout(const void* W, int O, int I, int taps, const int32_t* rows, int n_rows, const int32_t* cols,
                            int n_cols, const float* scale, int layout, int lead, int cpad, void* out,
                            cudaStream_t s) {
  const long long total = layout == UB_LAYOUT_OIHW    ? (long long)n_rows * n_cols * taps
                          : layout == UB_LAYOUT_GEMM ? (long long)n_rows * taps * cpad
                                                     : (long long)n_rows * cpad;  // DENSE, S2D
  const int block = 256;
  const int grid = grid_for(total, block, 4);
  if (layout == UB_LAYOUT_OIHW)
    permute_weights_kernel<TI, TO, UB_LAYOUT_OIHW><<<grid, block, 0, s>>>(
        static_cast<const TI*>(W), O, I, taps, rows, n_rows, cols, n_cols, scale, lead, cpad, static_cast<TO*>(out), total);
  else if (layout == UB_LAYOUT_GEMM)
    permute_weights_kernel<TI, TO, UB_LAYOUT_GEMM><<<grid, block, 0, s>>>(
        static_cast<const TI*>(W), O, I, taps, rows, n_rows, cols, n_cols, scale, lead, cpad, static_cast<TO*>(out), total);
  else if (layout == UB_LAYOUT_S2D)
    permute_weights_kernel<TI, TO, UB_LAYOUT_S2D><<<grid, block, 0, s>>>(
        static_cast<const TI*>(W), O, I, taps, rows, n_rows, cols, n_cols, scale, lead, cpad, static_cast<TO*>(out), total);
  else
    permute_weights_kernel<TI, TO, UB_LAYOUT_GEMM_DENSE><<<grid, block, 0, s>>>(
        static_cast<const TI*>(W), O, I, taps, rows, n_rows, cols, n_cols, scale, lead, cpad, static_cast<TO*>(out), total);
  count_launch();
  return cuda_status(cudaGetLastError(), "permute_weights_kernel");
}

// ------------------------------------------------------------- permute vector
template <typename T>
__global__ void permute_vector_kernel(const T* __restrict__ v, const int32_t* __restrict__ idx, int n,
                                      T* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int j = idx[i];
    out[i] = j >= 0 ? v[j] : T(0);
  }
}

// ------------------------------------------------------------- channel gather
// One warp per pixel row; lanes stride over the gathered channels so the reads
// of a warp fall inside the source row (the covering window) and the writes
// are contiguous.
__global__ void channel_gather_kernel(const uint16_t* __restrict__ x, int x_cstride, int x_coff,
                                      const int32_t* __restrict__ idx, int n, long long npix, uint16_t* __restrict__ y,
                                      int y_cstride, int y_coff) {
  griddep_wait();
  griddep_launch_dependents();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (long long p = (long long)blockIdx.x * warps + (threadIdx.x >> 5); p < npix; p += (long long)gridDim.x * warps) {
    const uint16_t* xr = x + p * x_cstride + x_coff;
    uint16_t* yr = y + p * y_cstride + y_coff;
    for (int i = lane * 2; i < n; i += 64) {
      const int j0 = __ldg(idx + i);
      const uint16_t a = j0 >= 0 ? __ldg(xr + j0) : uint16_t(0);
      if (i + 1 < n) {
        const int j1 = __ldg(idx + i + 1);
        const uint16_t b = j1 >= 0 ? __ldg(xr + j1) : uint16_t(0);
        if (((y_coff + i) & 1) == 0) {
          *reinterpret_cast<uint32_t*>(yr + i) = uint32_t(a) | (uint32_t(b) << 16);
        } else {
          yr[i] = a;
          yr[i + 1] = b;
        }
      } else {
        yr[i] = a;
      }
    }
  }
}

// Gather + pixel subsample: one warp per output pixel, 8 output channels (one 16-byte store)
// per lane and step; the index list sits in shared memory and the source row's sectors are
// shared through L1 by the lanes' 2-byte loads.
__global__ void __launch_bounds__(256) channel_gather_2d_kernel(const uint16_t* __restrict__ x, int x_cstride,
                                                                 int x_coff, const int32_t* __restrict__ idx,
                                                                 int n_idx, int n8, int N, int H, int W, int stride,
                                                                 int Ho, int Wo, uint16_t* __restrict__ y,
                                                                 int y_cstride, int y_coff) {
  extern __shared__ int32_t sidx[];
  for (int i = threadIdx.x; i < n8; i += blockDim.x) sidx[i] = i < n_idx ? __ldg(idx + i) : -1;
  __syncthreads();
  griddep_wait();
  griddep_launch_dependents();
  const int lane = threadIdx.x & 31;
  const long long npix = static_cast<long long>(N) * Ho * Wo;
  for (long long p = static_cast<long long>(blockIdx.x) * 8 + (threadIdx.x >> 5); p < npix;
       p += static_cast<long long>(gridDim.x) * 8) {
    const int n = static_cast<int>(p / (static_cast<long long>(Ho) * Wo));
    const int r = static_cast<int>(p - static_cast<long long>(n) * Ho * Wo);
    const int yo = r / Wo, xo = r - (r / Wo) * Wo;
    const uint16_t* xr = x + ((static_cast<size_t>(n) * H + yo * stride) * W + xo * stride) * x_cstride + x_coff;
    uint16_t* yr = y + static_cast<size_t>(p) * y_cstride + y_coff;
    for (int i = lane * 8; i < n8; i += 256) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int a = sidx[i + 2 * j], b = sidx[i + 2 * j + 1];
        const uint32_t lo = a >= 0 ? __ldg(xr + a) : 0u, hi = b >= 0 ? __ldg(xr + b) : 0u;
        w[j] = lo | (hi << 16);
      }
      *reinterpret_cast<uint4*>(yr + i) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// ------------------------------------------------------------- row-staged gather
// The baseline export's copy and the engine's "copy" read plan: a reference GATHER
// (interp.py:75-77) with an optional pixel subsample.  One warp per output pixel; the
// source row's covering window [ws, ws + 16*win16) is staged in shared memory with
// 16-byte cp.async (the next pixel's window is in flight while the current one is
// gathered), then each lane gathers 8 channels from shared memory and writes one 16-byte
// vector.  Global traffic: the window read once (coalesced), the gathered row written once.
//
// AFFINE: the read's pre-activation prologue (DenseNet's BN -> ReLU in front of every
// conv, SURVEY.md 2.2 "PER_CHANNEL ... prologue on the consumer's A-operand"): each
// gathered value becomes relu?(scale[i] * x + shift[i]) in fp32 before the bf16 store.
// ROWS == 4: the 2x2/s2 average pool a transition layer applies after its 1x1 conv,
// moved in front of the conv (both are linear; exact up to rounding): the four source
// pixels of each output pixel are staged and averaged after the prologue.
template <int ROWS, bool AFFINE>
__global__ void __launch_bounds__(256) gather_rows_kernel(const uint16_t* __restrict__ x, int x_cstride, int ws,
                                                          int win16, int pb, const int32_t* __restrict__ idx,
                                                          int n_idx, int rel, int n8, int N, int H, int W, int stride,
                                                          int Ho, int Wo, const float* __restrict__ scale,
                                                          const float* __restrict__ shift, int relu,
                                                          uint16_t* __restrict__ y, int y_cstride, int y_coff) {
  // A warp moves a batch of `pb` output pixels per step (narrow rows: several pixels' windows
  // per cp.async wave), with GR_STAGES batches in flight.
  constexpr int GR_STAGES = 3;
  extern __shared__ __align__(16) uint8_t g_smem[];
  int32_t* sidx = reinterpret_cast<int32_t*>(g_smem);
  float* sscale = reinterpret_cast<float*>(g_smem + n8 * 4);
  float* sshift = sscale + n8;
  const int idx_bytes = ((AFFINE ? 3 : 1) * n8 * 4 + 15) & ~15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int pix_chunks = ROWS * win16;                 // 16-byte chunks staged per output pixel
  const int stage_bytes = pb * pix_chunks * 16;
  uint8_t* buf0 = g_smem + idx_bytes + static_cast<size_t>(warp) * GR_STAGES * stage_bytes;
  for (int i = threadIdx.x; i < n8; i += blockDim.x) {
    const int j = i < n_idx ? __ldg(idx + i) : -1;
    sidx[i] = j >= 0 ? j + rel : -1;  // element offset inside the staged window
    if (AFFINE) {
      sscale[i] = i < n_idx ? __ldg(scale + i) : 0.f;
      sshift[i] = i < n_idx ? __ldg(shift + i) : 0.f;
    }
  }
  __syncthreads();
  griddep_wait();
  griddep_launch_dependents();
  const long long npix = static_cast<long long>(N) * Ho * Wo;
  const long long nbatch = (npix + pb - 1) / pb;
  const long long step = static_cast<long long>(gridDim.x) * warps;
  const int groups = n8 >> 3;
  // chunk t = lane + 32 i of a batch -> (pixel k, row q, chunk ch): the same for every batch,
  // walked with increments (no divisions in the loop)
  const bool direct = ROWS == 1 && stride == 1;  // source pixel == output pixel
  // pool2 with one output per lane: this lane's channel offsets and BN scale / shift
  int reg_a[8];
  float reg_sc[8], reg_sh[8];
  if (ROWS == 4) {
    const int gi0 = lane % groups;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = gi0 * 8 + j;
      reg_a[j] = c < n8 ? sidx[c] : -1;
      reg_sc[j] = AFFINE && c < n8 ? sscale[c] : 0.f;
      reg_sh[j] = AFFINE && c < n8 ? sshift[c] : 0.f;
    }
  }
  const int howo = Ho * Wo;
  auto issue = [&](long long b, uint8_t* dst) {
    const long long p0 = b * pb;
    const int total = pb * pix_chunks;
    int k = lane / pix_chunks, rem = lane - (lane / pix_chunks) * pix_chunks;
    // the output pixel's source position, recomputed only when the chunk walk moves to the next
    // pixel, in 32-bit arithmetic (a 64-bit division per chunk made this kernel instruction-bound)
    int kcur = -1;
    const uint16_t* pix_base = x;
    for (int t = lane; t < total; t += 32) {
      const long long p = p0 + k;
      if (p >= npix) break;
      const uint16_t* src;
      if (direct) {
        src = x + static_cast<size_t>(p) * x_cstride + ws + rem * 8;
      } else {
        if (k != kcur) {
          kcur = k;
          const int pi = static_cast<int>(p);  // npix < 2^31 (host-checked)
          const int n = pi / howo;
          const int r = pi - n * howo;
          const int yo = r / Wo, xo = r - (r / Wo) * Wo;
          const int yb = ROWS == 4 ? 2 * yo : yo * stride, xb = ROWS == 4 ? 2 * xo : xo * stride;
          pix_base = x + ((static_cast<size_t>(n) * H + yb) * W + xb) * x_cstride + ws;
        }
        const int q = ROWS == 1 ? 0 : rem / win16, ch = rem - q * win16;
        const int dyx = ROWS == 4 ? ((q >> 1) * W + (q & 1)) : 0;
        src = pix_base + static_cast<size_t>(dyx) * x_cstride + ch * 8;
      }
      cp_async16(dst + t * 16, src, 16);
      rem += 32;
      while (rem >= pix_chunks) {
        rem -= pix_chunks;
        ++k;
      }
    }
  };
  long long b = static_cast<long long>(blockIdx.x) * warps + warp;
#pragma unroll
  for (int st = 0; st < GR_STAGES - 1; ++st) {
    if (b + st * step < nbatch) issue(b + st * step, buf0 + st * stage_bytes);
    cp_async_commit();
  }
  int k = 0;
  for (; b < nbatch; b += step, k = (k + 1 == GR_STAGES ? 0 : k + 1)) {
    const long long bn = b + (GR_STAGES - 1) * step;
    const int kn = (k + GR_STAGES - 1) % GR_STAGES;
    if (bn < nbatch) issue(bn, buf0 + kn * stage_bytes);
    cp_async_commit();
    cp_async_wait<GR_STAGES - 1>();
    __syncwarp();
    const uint8_t* stage = buf0 + k * stage_bytes;
    const long long p0 = b * pb;
    const int work = pb * groups;
    int kp = lane / groups, gi = lane - (lane / groups) * groups;
    if (ROWS == 4 && work <= 32) {
      // one output (pixel kp, group gi) per lane, the same every batch: the channel offsets and
      // the BN scale/shift come from registers (reg_*), not 3 shared loads per channel
      if (lane < work && p0 + kp < npix) {
        const uint16_t* row = reinterpret_cast<const uint16_t*>(stage + kp * pix_chunks * 16);
        float f[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float acc = 0.f;
          if (reg_a[j] >= 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float v = __uint_as_float(static_cast<uint32_t>(row[q * win16 * 8 + reg_a[j]]) << 16);
              if (AFFINE) {
                v = fmaf(reg_sc[j], v, reg_sh[j]);
                if (relu) v = fmaxf(v, 0.f);
              }
              acc += v;
            }
            acc *= 0.25f;
          }
          f[j] = acc;
        }
        *reinterpret_cast<uint4*>(y + static_cast<size_t>(p0 + kp) * y_cstride + y_coff + gi * 8) =
            make_uint4(cvt_bf16x2(f[0], f[1]), cvt_bf16x2(f[2], f[3]), cvt_bf16x2(f[4], f[5]), cvt_bf16x2(f[6], f[7]));
      }
      __syncwarp();
      continue;
    }
    for (int t = lane; t < work; t += 32) {
      const long long p = p0 + kp;
      if (p >= npix) break;
      const int i = gi * 8;
      gi += 32;
      const int kp_here = kp;
      while (gi >= groups) {
        gi -= groups;
        ++kp;
      }
      const uint16_t* row = reinterpret_cast<const uint16_t*>(stage + kp_here * pix_chunks * 16);
      uint32_t w[4];
#pragma unroll
      for (int j2 = 0; j2 < 4; ++j2) {
        uint16_t h[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = i + 2 * j2 + e;
          const int a = sidx[c];
          if (!AFFINE && ROWS == 1) {
            h[e] = a >= 0 ? row[a] : uint16_t(0);
          } else {
            float acc = 0.f;
            if (a >= 0) {
#pragma unroll
              for (int q = 0; q < ROWS; ++q) {
                float v = __uint_as_float(static_cast<uint32_t>(row[q * win16 * 8 + a]) << 16);
                if (AFFINE) {
                  v = fmaf(sscale[c], v, sshift[c]);
                  if (relu) v = fmaxf(v, 0.f);
                }
                acc += v;
              }
              if (ROWS == 4) acc *= 0.25f;
            }
            h[e] = __bfloat16_as_ushort(__float2bfloat16_rn(acc));
          }
        }
        w[j2] = static_cast<uint32_t>(h[0]) | (static_cast<uint32_t>(h[1]) << 16);
      }
      *reinterpret_cast<uint4*>(y + static_cast<size_t>(p) * y_cstride + y_coff + i) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    __syncwarp();
  }
  cp_async_wait<0>();
}

// Fast form of gather_rows_kernel for the common case -- stride 1, no pool.  Narrow outputs
// (groups = pad8(n)/8 <= 32): a warp step moves pb = 32 / groups pixels so that every lane
// owns ONE (pixel, 8-channel group) of the batch.  Wide outputs (groups > 32): pb = 1 and
// lane l owns groups l, l+32, ... (GJ of them).  Either way the lane's source columns and
// cp.async chunk offsets are the same for every batch and live in registers (the BN
// scale/shift of wide outputs in shared memory, read conflict-free), so a batch costs a
// few cp.async and one 16-byte gather/store per owned group; with the engine's ascending
// source order the 2-byte shared-memory reads of a warp hit distinct banks.
constexpr int GRF_MAXI = 4;  // cp.async chunks per lane per batch
template <bool AFFINE, int GJ>
__global__ void __launch_bounds__(256) gather_rows_fast_kernel(const uint16_t* __restrict__ x, int x_cstride, int ws,
                                                               int win16, int pb, const int32_t* __restrict__ idx,
                                                               int n_idx, int rel, int n8, long long npix,
                                                               const float* __restrict__ scale,
                                                               const float* __restrict__ shift, int relu,
                                                               uint16_t* __restrict__ y, int y_cstride, int y_coff) {
  constexpr int STAGES = 4;
  extern __shared__ __align__(16) uint8_t g_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int stage_bytes = pb * win16 * 16;
  float* s_sc = reinterpret_cast<float*>(g_smem);  // wide outputs: [n8] scale then [n8] shift
  float* s_sh = s_sc + n8;
  const int par_bytes = (GJ > 1 && AFFINE) ? ((2 * n8 * 4 + 15) & ~15) : 0;
  uint8_t* buf0 = g_smem + par_bytes + static_cast<size_t>(warp) * STAGES * stage_bytes;
  const int groups = n8 >> 3;
  if (GJ > 1 && AFFINE) {
    for (int c = threadIdx.x; c < n8; c += blockDim.x) {
      s_sc[c] = c < n_idx ? __ldg(scale + c) : 0.f;
      s_sh[c] = c < n_idx ? __ldg(shift + c) : 0.f;
    }
    __syncthreads();
  }
  // owned outputs: GJ == 1 -> pixel kp, group lane % groups; GJ > 1 -> pixel 0, groups lane + 32 j
  const int kp = GJ == 1 ? lane / groups : 0;
  int col[GJ][8];
  float sc[GJ == 1 ? 8 : 1], sh[GJ == 1 ? 8 : 1];
#pragma unroll
  for (int jj = 0; jj < GJ; ++jj) {
    const int g = GJ == 1 ? lane - kp * groups : lane + 32 * jj;
    const bool own = GJ == 1 ? lane < pb * groups : g < groups;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = g * 8 + j;
      const int a = (own && c < n_idx) ? __ldg(idx + c) : -1;
      col[jj][j] = a >= 0 ? kp * win16 * 8 + a + rel : -1;
      if (GJ == 1 && AFFINE) {
        sc[j] = (own && c < n_idx) ? __ldg(scale + c) : 0.f;
        sh[j] = (own && c < n_idx) ? __ldg(shift + c) : 0.f;
      }
    }
  }
  const int total = pb * win16;
  int ck[GRF_MAXI], coffs[GRF_MAXI];
#pragma unroll
  for (int m = 0; m < GRF_MAXI; ++m) {
    const int t = lane + 32 * m;
    ck[m] = t < total ? t / win16 : 1 << 30;
    coffs[m] = t < total ? ck[m] * x_cstride + (t - ck[m] * win16) * 8 : 0;
  }
  griddep_wait();
  griddep_launch_dependents();
  const long long nbatch = (npix + pb - 1) / pb;
  const long long step = static_cast<long long>(gridDim.x) * warps;
  auto issue = [&](long long b, uint8_t* dst) {
    const long long p0 = b * pb;
    const uint16_t* src = x + static_cast<size_t>(p0) * x_cstride + ws;
#pragma unroll
    for (int m = 0; m < GRF_MAXI; ++m) {
      if (lane + 32 * m >= total) break;
      if (p0 + ck[m] < npix) cp_async16(dst + (lane + 32 * m) * 16, src + coffs[m], 16);
    }
  };
  long long b = static_cast<long long>(blockIdx.x) * warps + warp;
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (b + st * step < nbatch) issue(b + st * step, buf0 + st * stage_bytes);
    cp_async_commit();
  }
  int k = 0;
  for (; b < nbatch; b += step, k = (k + 1 == STAGES ? 0 : k + 1)) {
    const long long bn = b + (STAGES - 1) * step;
    if (bn < nbatch) issue(bn, buf0 + ((k + STAGES - 1) % STAGES) * stage_bytes);
    cp_async_commit();
    cp_async_wait<STAGES - 1>();
    __syncwarp();
    const long long p = b * pb + kp;
    const uint16_t* row = reinterpret_cast<const uint16_t*>(buf0 + k * stage_bytes);
#pragma unroll
    for (int jj = 0; jj < GJ; ++jj) {
      const int g = GJ == 1 ? lane - kp * groups : lane + 32 * jj;
      const bool own = GJ == 1 ? lane < pb * groups : g < groups;
      if (!own || p >= npix) continue;
      uint32_t w[4];
#pragma unroll
      for (int j2 = 0; j2 < 4; ++j2) {
        uint16_t h[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int j = 2 * j2 + e;
          const int cj = col[jj][j];
          if (!AFFINE) {
            h[e] = cj >= 0 ? row[cj] : uint16_t(0);
          } else {
            float v = 0.f;
            if (cj >= 0) {
              const float a = GJ == 1 ? sc[j] : s_sc[g * 8 + j];
              const float t = GJ == 1 ? sh[j] : s_sh[g * 8 + j];
              v = fmaf(a, __uint_as_float(static_cast<uint32_t>(row[cj]) << 16), t);
              if (relu) v = fmaxf(v, 0.f);
            }
            h[e] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
          }
        }
        w[j2] = static_cast<uint32_t>(h[0]) | (static_cast<uint32_t>(h[1]) << 16);
      }
      *reinterpret_cast<uint4*>(y + static_cast<size_t>(p) * y_cstride + y_coff + g * 8) =
          make_uint4(w[0], w[1], w[2], w[3]);
    }
    __syncwarp();
  }
  cp_async_wait<0>();
}

// Wide outputs (more than 256 gathered channels, DenseNet blocks 3-4): one pixel per warp
// step; lane l owns outputs l, l+32, ... so the per-output tables (source column, BN scale
// and shift) are read from shared memory conflict-free and consecutive lanes gather from
// nearby (ascending) source columns -- distinct banks; 2-byte stores of consecutive lanes
// coalesce.  (Owning 8 consecutive outputs per lane put lanes 32 bytes apart: 4-way bank
// conflicts, ncu L1 88 %.)
template <bool AFFINE, int MPL>  // MPL > 0: the lane's <= MPL (column, scale, shift) triples live in registers
__global__ void __launch_bounds__(256) gather_rows_wide_kernel(const uint16_t* __restrict__ x, int x_cstride, int ws,
                                                               int win16, const int32_t* __restrict__ idx, int n_idx,
                                                               int rel, int n8, long long npix, int stride, int H,
                                                               int W, int Ho, int Wo, const float* __restrict__ scale,
                                                               const float* __restrict__ shift, int relu,
                                                               uint16_t* __restrict__ y, int y_cstride, int y_coff) {
  constexpr int STAGES = 3;
  extern __shared__ __align__(16) uint8_t g_smem[];
  int32_t* s_col = reinterpret_cast<int32_t*>(g_smem);
  float* s_sc = reinterpret_cast<float*>(g_smem + n8 * 4);
  float* s_sh = s_sc + n8;
  const int par_bytes = MPL > 0 ? 0 : (((AFFINE ? 3 : 1) * n8 * 4 + 15) & ~15);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int stage_bytes = win16 * 16;
  uint8_t* buf0 = g_smem + par_bytes + static_cast<size_t>(warp) * STAGES * stage_bytes;
  constexpr int R = MPL > 0 ? MPL : 1;
  int rcol[R];
  float rsc[R], rsh[R];
  if (MPL > 0) {
#pragma unroll
    for (int m = 0; m < R; ++m) {
      const int c = lane + 32 * m;
      const int a = c < n_idx ? __ldg(idx + c) : -1;
      rcol[m] = a >= 0 ? a + rel : -1;
      rsc[m] = (AFFINE && c < n_idx) ? __ldg(scale + c) : 0.f;
      rsh[m] = (AFFINE && c < n_idx) ? __ldg(shift + c) : 0.f;
    }
  } else {
    for (int c = threadIdx.x; c < n8; c += blockDim.x) {
      const int a = c < n_idx ? __ldg(idx + c) : -1;
      s_col[c] = a >= 0 ? a + rel : -1;
      if (AFFINE) {
        s_sc[c] = c < n_idx ? __ldg(scale + c) : 0.f;
        s_sh[c] = c < n_idx ? __ldg(shift + c) : 0.f;
      }
    }
    __syncthreads();
  }
  griddep_wait();
  griddep_launch_dependents();
  const long long step = static_cast<long long>(gridDim.x) * warps;
  auto issue = [&](long long p, uint8_t* dst) {
    long long sp = p;  // source pixel (a strided 1x1 conv reads every stride-th pixel)
    if (stride != 1) {
      const long long hw = static_cast<long long>(Ho) * Wo;
      const long long n = p / hw;
      const int r = static_cast<int>(p - n * hw);
      const int yo = r / Wo, xo = r - (r / Wo) * Wo;
      sp = (n * H + static_cast<long long>(yo) * stride) * W + static_cast<long long>(xo) * stride;
    }
    const uint16_t* src = x + static_cast<size_t>(sp) * x_cstride + ws;
    for (int j = lane; j < win16; j += 32) cp_async16(dst + j * 16, src + j * 8, 16);
  };
  long long p = static_cast<long long>(blockIdx.x) * warps + warp;
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (p + st * step < npix) issue(p + st * step, buf0 + st * stage_bytes);
    cp_async_commit();
  }
  int k = 0;
  for (; p < npix; p += step, k = (k + 1 == STAGES ? 0 : k + 1)) {
    const long long pn = p + (STAGES - 1) * step;
    if (pn < npix) issue(pn, buf0 + ((k + STAGES - 1) % STAGES) * stage_bytes);
    cp_async_commit();
    cp_async_wait<STAGES - 1>();
    __syncwarp();
    const uint16_t* row = reinterpret_cast<const uint16_t*>(buf0 + k * stage_bytes);
    uint16_t* yr = y + static_cast<size_t>(p) * y_cstride + y_coff;
    if (MPL > 0) {
#pragma unroll
      for (int m = 0; m < R; ++m) {
        const int c = lane + 32 * m;
        if (c >= n8) break;
        const int cj = rcol[m];
        const uint16_t raw = cj >= 0 ? row[cj] : uint16_t(0);
        uint16_t h = raw;
        if (AFFINE) {
          float v = 0.f;
          if (cj >= 0) {
            v = fmaf(rsc[m], __uint_as_float(static_cast<uint32_t>(raw) << 16), rsh[m]);
            if (relu) v = fmaxf(v, 0.f);
          }
          h = __bfloat16_as_ushort(__float2bfloat16_rn(v));
        }
        yr[c] = h;
      }
    } else {
      for (int c = lane; c < n8; c += 32) {
        const int cj = s_col[c];
        uint16_t h = cj >= 0 ? row[cj] : uint16_t(0);
        if (AFFINE) {
          float v = 0.f;
          if (cj >= 0) {
            v = fmaf(s_sc[c], __uint_as_float(static_cast<uint32_t>(h) << 16), s_sh[c]);
            if (relu) v = fmaxf(v, 0.f);
          }
          h = __bfloat16_as_ushort(__float2bfloat16_rn(v));
        }
        yr[c] = h;
      }
    }
    __syncwarp();
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------- input staging
// NCHW fp32 -> NHWC bf16 (channel-gathered), zero-filling the padded channels.
__global__ void stage_input_kernel(const float* __restrict__ x, int N, int C, int HW, const int32_t* __restrict__ idx,
                                   int n, __nv_bfloat16* __restrict__ y, int y_cstride) {
  const long long total = (long long)N * HW;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < total;
       p += (long long)gridDim.x * blockDim.x) {
    const long long img = p / HW;
    const long long hw = p - img * HW;
    const float* xp = x + img * C * HW + hw;
    __nv_bfloat16* yp = y + p * y_cstride;
    for (int c = 0; c < y_cstride; ++c) {
      float v = 0.f;
      if (c < n) {
        const int src = idx ? idx[c] : c;
        if (src >= 0) v = __ldg(xp + (long long)src * HW);
      }
      yp[c] = __float2bfloat16_rn(v);
    }
  }
}

// ------------------------------------------------------------- max pool
// Thread = (output pixel, 8-channel group); 16-byte vectors when aligned.
__global__ void maxpool_kernel(const __nv_bfloat16* __restrict__ x, int N, int H, int W, int C, int x_cstride,
                               int x_coff, int k, int stride, int pad, int Ho, int Wo, __nv_bfloat16* __restrict__ y,
                               int y_cstride, int y_coff, bool vec) {
  griddep_wait();
  griddep_launch_dependents();
  const int groups = (C + 7) / 8;
  const int total = N * Ho * Wo * groups;  // < 2^31 (checked by the host)
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int g = e % groups;
    const int pix = e / groups;
    const int wo = pix % Wo;
    const int t = pix / Wo;
    const int ho = t % Ho;
    const int img = t / Ho;
    const int c0 = g * 8;
    const int nc = min(8, C - c0);
    float m[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) m[i] = -INFINITY;
    for (int r = 0; r < k; ++r) {
      const int hi = ho * stride - pad + r;
      if (hi < 0 || hi >= H) continue;
      for (int s = 0; s < k; ++s) {
        const int wi = wo * stride - pad + s;
        if (wi < 0 || wi >= W) continue;
        const __nv_bfloat16* xp = x + (static_cast<size_t>(img * H + hi) * W + wi) * x_cstride + x_coff + c0;
        if (vec && nc == 8) {
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(xp));
          const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = unpack_bf16x2(w4[i]);
            m[2 * i] = fmaxf(m[2 * i], f.x);
            m[2 * i + 1] = fmaxf(m[2 * i + 1], f.y);
          }
        } else {
          for (int i = 0; i < nc; ++i) m[i] = fmaxf(m[i], __bfloat162float(xp[i]));
        }
      }
    }
    __nv_bfloat16* yp = y + static_cast<size_t>(pix) * y_cstride + y_coff + c0;
    if (vec && nc == 8) {
      uint4 o;
      o.x = pack_bf16x2(m[0], m[1]);
      o.y = pack_bf16x2(m[2], m[3]);
      o.z = pack_bf16x2(m[4], m[5]);
      o.w = pack_bf16x2(m[6], m[7]);
      *reinterpret_cast<uint4*>(yp) = o;
    } else {
      for (int i = 0; i < nc; ++i) yp[i] = __float2bfloat16_rn(m[i]);
    }
  }
}

// ------------------------------------------------------------- global avg pool
// Block = one image x 256 channels; threads stride the HW positions per channel.
__global__ void avgpool_kernel(const __nv_bfloat16* __restrict__ x, int HW, int C, int x_cstride, int x_coff,
                               __nv_bfloat16* __restrict__ y, int y_cstride, int y_coff) {
  griddep_wait();
  griddep_launch_dependents();
  const int img = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const __nv_bfloat16* xp = x + (long long)img * HW * x_cstride + x_coff + c;
  float s = 0.f;
  for (int p = 0; p < HW; ++p) s += __bfloat162float(xp[(long long)p * x_cstride]);
  y[(long long)img * y_cstride + y_coff + c] = __float2bfloat16_rn(s / HW);
}

// 8 channels per thread (16-byte loads), the pixel loop unrolled so a thread has several
// loads in flight; the fp32 sum is accumulated in pixel order (same result as the scalar
// kernel).
__global__ void avgpool8_kernel(const uint4* __restrict__ x, int HW, int C8, int x_cstride8, int x_coff8,
                                uint4* __restrict__ y, int y_cstride8, int y_coff8) {
  griddep_wait();
  griddep_launch_dependents();
  const int img = blockIdx.y;
  const int c8 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c8 >= C8) return;
  const uint4* xp = x + static_cast<long long>(img) * HW * x_cstride8 + x_coff8 + c8;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  int p = 0;
  for (; p + 7 <= HW; p += 7) {
    uint4 v[7];
#pragma unroll
    for (int u = 0; u < 7; ++u) v[u] = __ldg(xp + static_cast<long long>(p + u) * x_cstride8);
#pragma unroll
    for (int u = 0; u < 7; ++u) {
      const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = bf16x2_to_f32x2(w[j]);
        s[2 * j] += f.x;
        s[2 * j + 1] += f.y;
      }
    }
  }
  for (; p < HW; ++p) {
    const uint4 v = __ldg(xp + static_cast<long long>(p) * x_cstride8);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = bf16x2_to_f32x2(w[j]);
      s[2 * j] += f.x;
      s[2 * j + 1] += f.y;
    }
  }
  uint32_t o[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) o[j] = cvt_bf16x2(s[2 * j] / HW, s[2 * j + 1] / HW);
  y[static_cast<long long>(img) * y_cstride8 + y_coff8 + c8] = make_uint4(o[0], o[1], o[2], o[3]);
}

// ------------------------------------------------------------- global avg pool + GATHER
// avgpool8_kernel's mapping (CTA = image x 128 groups of 8 channels, a thread walks the
// pixels of its group in order, 7 loads in flight), then the GATHER that reads the pool is
// applied from shared memory: the kept channels of this block are written compacted,
// y[j] = pooled[idx[j]] (0 for idx[j] < 0, written by block 0; interp.py:75-77).  The consumer
// reads a dense operand and the standalone gather copy disappears.  (Splitting the pixels
// over more threads measured slower under ncu: 18-32 us vs 15 us for 45 MB.)
__global__ void __launch_bounds__(128) avgpool_gather_kernel(const uint4* __restrict__ x, int HW, int C8,
                                                             int x_cstride8, int x_coff8,
                                                             const int32_t* __restrict__ idx, int n_idx,
                                                             __nv_bfloat16* __restrict__ y, int y_cstride,
                                                             int y_coff) {
  __shared__ float pooled[128 * 8];
  griddep_wait();
  griddep_launch_dependents();
  const int img = blockIdx.y;
  const int c8 = blockIdx.x * 128 + threadIdx.x;
  if (c8 < C8) {
    const uint4* xp = x + static_cast<long long>(img) * HW * x_cstride8 + x_coff8 + c8;
    float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int p = 0;
    for (; p + 7 <= HW; p += 7) {
      uint4 v[7];
#pragma unroll
      for (int u = 0; u < 7; ++u) v[u] = __ldg(xp + static_cast<long long>(p + u) * x_cstride8);
#pragma unroll
      for (int u = 0; u < 7; ++u) {
        const uint32_t wv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = bf16x2_to_f32x2(wv[j]);
          s[2 * j] += f.x;
          s[2 * j + 1] += f.y;
        }
      }
    }
    for (; p < HW; ++p) {
      const uint4 v = __ldg(xp + static_cast<long long>(p) * x_cstride8);
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = bf16x2_to_f32x2(wv[j]);
        s[2 * j] += f.x;
        s[2 * j + 1] += f.y;
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) pooled[threadIdx.x * 8 + j] = s[j] / HW;
  }
  __syncthreads();
  __nv_bfloat16* yi = y + static_cast<long long>(img) * y_cstride + y_coff;
  const int c_lo = blockIdx.x * 1024, c_hi = min(c_lo + 1024, C8 * 8);
  for (int j = threadIdx.x; j < n_idx; j += blockDim.x) {
    const int c = __ldg(idx + j);
    if (c >= c_lo && c < c_hi)
      yi[j] = __float2bfloat16_rn(pooled[c - c_lo]);
    else if (c < 0 && blockIdx.x == 0)
      yi[j] = __float2bfloat16_rn(0.f);
  }
}

// Small-batch form: CTA = (256-channel block, image), warp q reads pixels q, q + 8, ... (a warp
// covers 512 contiguous bytes of a pixel row) with up to 7 predicated loads in flight per
// thread -- one DRAM round trip per 56 pixels instead of 7 for the thread-walks-all-pixels
// form.  The 8 phase sums meet in shared memory (added in phase order).  Faster when the
// grid is small (N = 1: 12 vs 18 us, events, L2 flushed) but slower at N = 256 (25 vs 20 us),
// so ub_avgpool_gather picks it only while the large form would leave SMs idle.
constexpr int APG_PHASES = 8, APG_UNROLL = 7;
__global__ void __launch_bounds__(256) avgpool_gather_phased_kernel(const uint4* __restrict__ x, int HW, int C8,
                                                                    int x_cstride8, int x_coff8,
                                                                    const int32_t* __restrict__ idx, int n_idx,
                                                                    __nv_bfloat16* __restrict__ y, int y_cstride,
                                                                    int y_coff) {
  __shared__ float part[APG_PHASES][32 * 8];
  __shared__ float pooled[32 * 8];
  griddep_wait();
  griddep_launch_dependents();
  const int img = blockIdx.y;
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int c8 = blockIdx.x * 32 + lane;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c8 < C8) {
    const uint4* xp = x + static_cast<long long>(img) * HW * x_cstride8 + x_coff8 + c8;
    for (int p0 = q; p0 < HW; p0 += APG_PHASES * APG_UNROLL) {
      uint4 v[APG_UNROLL];
#pragma unroll
      for (int u = 0; u < APG_UNROLL; ++u) {
        const int p = p0 + u * APG_PHASES;
        v[u] = p < HW ? __ldg(xp + static_cast<long long>(p) * x_cstride8) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < APG_UNROLL; ++u) {  // zero-filled slots add +0.0f
        const uint32_t wv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = bf16x2_to_f32x2(wv[j]);
          s[2 * j] += f.x;
          s[2 * j + 1] += f.y;
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) part[q][lane * 8 + j] = s[j];
  __syncthreads();
  {
    float t = part[0][threadIdx.x];
#pragma unroll
    for (int r = 1; r < APG_PHASES; ++r) t += part[r][threadIdx.x];
    pooled[threadIdx.x] = t / HW;
  }
  __syncthreads();
  __nv_bfloat16* yi = y + static_cast<long long>(img) * y_cstride + y_coff;
  const int c_lo = blockIdx.x * 256, c_hi = min(c_lo + 256, C8 * 8);
  for (int j = threadIdx.x; j < n_idx; j += blockDim.x) {
    const int c = __ldg(idx + j);
    if (c >= c_lo && c < c_hi)
      yi[j] = __float2bfloat16_rn(pooled[c - c_lo]);
    else if (c < 0 && blockIdx.x == 0)
      yi[j] = __float2bfloat16_rn(0.f);
  }
}

// ------------------------------------------------------------- affine / add / relu
__global__ void affine_add_relu_kernel(const __nv_bfloat16* __restrict__ a, int a_cstride, int a_coff,
                                       const float* __restrict__ scale, const float* __restrict__ shift,
                                       const __nv_bfloat16* __restrict__ b, int b_cstride, int b_coff, int relu,
                                       long long npix, int C, __nv_bfloat16* __restrict__ y, int y_cstride,
                                       int y_coff) {
  const long long total = npix * C;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(e % C);
    const long long p = e / C;
    float v = __bfloat162float(a[p * a_cstride + a_coff + c]);
    if (scale) v *= scale[c];
    if (shift) v += shift[c];
    if (b) v += __bfloat162float(b[p * b_cstride + b_coff + c]);
    if (relu) v = fmaxf(v, 0.f);
    y[p * y_cstride + y_coff + c] = __float2bfloat16_rn(v);
  }
}

}  // namespace
}  // namespace ub

using namespace ub;

extern "C" int ub_permute_weights(const void* W, int dtype_in, int O, int I, int kh, int kw, const int32_t* rows,
                                  int n_rows, const int32_t* cols, int n_cols, const float* row_scale, int layout,
                                  int lead, int cpad, void* out, int dtype_out, cudaStream_t stream) {
  if (!W || !rows || !cols || !out) return fail(UB_EINVAL, "ub_permute_weights: null pointer");
  if (O < 1 || I < 1 || kh < 1 || kw < 1 || n_rows < 1 || n_cols < 1)
    return fail(UB_EINVAL, "ub_permute_weights: bad sizes");
  if (layout != UB_LAYOUT_OIHW && layout != UB_LAYOUT_GEMM && layout != UB_LAYOUT_GEMM_DENSE &&
      layout != UB_LAYOUT_S2D)
    return fail(UB_EINVAL, "ub_permute_weights: layout");
  if (layout == UB_LAYOUT_S2D) {
    if (kh != kw || kw < 2 || 4 * n_cols > 8)
      return fail(UB_EUNSUPPORTED, "ub_permute_weights: S2D needs a square filter and n_cols <= 2");
    lead = kw;  // the kernel decomposes k with the filter width
    cpad = (kw + 1) / 2 * ((kw + 1) / 2) * 8;
  }
  if (layout == UB_LAYOUT_GEMM_DENSE && kh * kw * n_cols > cpad)
    return fail(UB_EINVAL, "ub_permute_weights: dense K %d > cpad %d", kh * kw * n_cols, cpad);
  if (layout == UB_LAYOUT_GEMM && (lead < 0 || lead + n_cols > cpad))
    return fail(UB_EINVAL, "ub_permute_weights: lead + n_cols > cpad");
  const int taps = kh * kw;
  if (dtype_in == UB_F32) {
    if (dtype_out == UB_F32)
      return permute_dispatch_layout<float, float>(W, O, I, taps, rows, n_rows, cols, n_cols, row_scale, layout, lead,
                                                   cpad, out, stream);
    if (dtype_out == UB_BF16)
      return permute_dispatch_layout<float, __nv_bfloat16>(W, O, I, taps, rows, n_rows, cols, n_cols, row_scale, layout,
                                                           lead, cpad, out, stream);
  } else if (dtype_in == UB_F64) {
    if (dtype_out == UB_F64)
      return permute_dispatch_layout<double, double>(W, O, I, taps, rows, n_rows, cols, n_cols, row_scale, layout, lead,
                                                     cpad, out, stream);
    if (dtype_out == UB_F32)
      return permute_dispatch_layout<double, float>(W, O, I, taps, rows, n_rows, cols, n_cols, row_scale, layout, lead,
                                                    cpad, out, stream);
  }
  return fail(UB_EUNSUPPORTED, "ub_permute_weights: dtype pair (%d -> %d)", dtype_in, dtype_out);
}

extern "C" int ub_index_faults(unsigned long long* count) {
  if (!count) return fail(UB_EINVAL, "ub_index_faults: null pointer");
  const unsigned long long zero = 0;
  cudaError_t e = cudaMemcpyFromSymbol(count, g_index_faults, sizeof(zero));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_index_faults, &zero, sizeof(zero));
  return cuda_status(e, "ub_index_faults");
}

extern "C" int ub_permute_vector(const void* v, int dtype, const int32_t* idx, int n, void* out,
                                 cudaStream_t stream) {
  if (!v || !idx || !out || n < 1) return fail(UB_EINVAL, "ub_permute_vector: bad arguments");
  const int grid = grid_for(n, 256);
  if (dtype == UB_F32)
    permute_vector_kernel<float><<<grid, 256, 0, stream>>>(static_cast<const float*>(v), idx, n,
                                                           static_cast<float*>(out));
  else if (dtype == UB_F64)
    permute_vector_kernel<double><<<grid, 256, 0, stream>>>(static_cast<const double*>(v), idx, n,
                                                            static_cast<double*>(out));
  else
    return fail(UB_EUNSUPPORTED, "ub_permute_vector: dtype %d", dtype);
  count_launch();
  return cuda_status(cudaGetLastError(), "permute_vector_kernel");
}

extern "C" int ub_channel_gather(const void* x, int x_cstride, int x_coff, const int32_t* idx, int n, long long npix,
                                 void* y, int y_cstride, int y_coff, cudaStream_t stream) {
  if (!x || !idx || !y || n < 1 || npix < 1) return fail(UB_EINVAL, "ub_channel_gather: bad arguments");
  if (y_coff + n > y_cstride) return fail(UB_EINVAL, "ub_channel_gather: output exceeds y_cstride");
  const int block = 256;
  const int grid = grid_for(npix, block / 32);
  const cudaError_t e = launch_pdl(channel_gather_kernel, dim3(grid), dim3(block), 0, stream,
                                   static_cast<const uint16_t*>(x), x_cstride, x_coff, idx, n, npix,
                                   static_cast<uint16_t*>(y), y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "channel_gather_kernel");
}

extern "C" int ub_channel_gather_2d(const void* x, int x_cstride, int x_coff, const int32_t* idx, int n_idx, int N,
                                    int H, int W, int stride, void* y, int y_cstride, int y_coff,
                                    cudaStream_t stream) {
  if (!x || !idx || !y || n_idx < 1 || N < 1 || H < 1 || W < 1 || stride < 1)
    return fail(UB_EINVAL, "ub_channel_gather_2d: bad arguments");
  const int n8 = (n_idx + 7) / 8 * 8;
  if ((y_cstride & 7) || (y_coff & 7) || y_coff + n8 > y_cstride || !aligned16(y))
    return fail(UB_EINVAL, "ub_channel_gather_2d: output rows must hold pad8(n) 16-byte aligned channels");
  if (n8 > 8192) return fail(UB_EUNSUPPORTED, "ub_channel_gather_2d: %d channels", n_idx);
  const int Ho = (H + stride - 1) / stride, Wo = (W + stride - 1) / stride;
  const long long npix = static_cast<long long>(N) * Ho * Wo;
  const long long want = (npix + 7) / 8;
  const int grid = static_cast<int>(want < 148LL * 16 ? want : 148LL * 16);
  const cudaError_t e = launch_pdl(channel_gather_2d_kernel, dim3(grid), dim3(256), n8 * sizeof(int32_t), stream,
                                   static_cast<const uint16_t*>(x), x_cstride, x_coff, idx, n_idx, n8, N, H, W,
                                   stride, Ho, Wo, static_cast<uint16_t*>(y), y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "channel_gather_2d_kernel");
}

extern "C" int ub_gather_rows_ex(const void* x, int x_cstride, int x_coff, int lo, int hi, const int32_t* idx,
                                 int n_idx, int N, int H, int W, int stride, int pool2, const float* scale,
                                 const float* shift, int relu, void* y, int y_cstride, int y_coff,
                                 cudaStream_t stream) {
  if (!x || !idx || !y || n_idx < 1 || N < 1 || H < 1 || W < 1 || stride < 1 || lo < 0 || hi < lo)
    return fail(UB_EINVAL, "ub_gather_rows: bad arguments");
  if ((scale == nullptr) != (shift == nullptr)) return fail(UB_EINVAL, "ub_gather_rows: scale and shift go together");
  if (pool2 && (stride != 1 || H < 2 || W < 2)) return fail(UB_EINVAL, "ub_gather_rows: pool2 needs stride 1");
  const int n8 = (n_idx + 7) / 8 * 8;
  if ((y_cstride & 7) || (y_coff & 7) || y_coff + n8 > y_cstride || !aligned16(y))
    return fail(UB_EINVAL, "ub_gather_rows: output rows must hold pad8(n) 16-byte aligned channels");
  if ((x_cstride & 7) || !aligned16(x) || x_coff < 0 || x_coff + hi >= x_cstride)
    return fail(UB_EINVAL, "ub_gather_rows: source window outside 16-byte aligned rows");
  const bool affine = scale != nullptr;
  const int rows = pool2 ? 4 : 1;
  const int ws = (x_coff + lo) & ~7;
  const int we = (x_coff + hi + 8) & ~7;
  const int win16 = (we - ws) / 8;
  if (!pool2 && n8 > 256 && win16 <= 256) {  // wide outputs: lane-interleaved ownership
    const bool regs = n8 <= 32 * 24;  // the lane's tables in registers
    const size_t par = regs ? 0 : ((affine ? 3 : 1) * static_cast<size_t>(n8) * 4 + 15) & ~static_cast<size_t>(15);
    const size_t stage_w = static_cast<size_t>(win16) * 16;
    int ww = 8;
    while (ww > 1 && par + ww * 3 * stage_w > 200 * 1024) ww >>= 1;
    const size_t smem_w = par + ww * 3 * stage_w;
    void (*kw)(const uint16_t*, int, int, int, const int32_t*, int, int, int, long long, int, int, int, int, int,
               const float*, const float*, int, uint16_t*, int, int) =
        regs ? (affine ? gather_rows_wide_kernel<true, 24> : gather_rows_wide_kernel<false, 24>)
             : (affine ? gather_rows_wide_kernel<true, 0> : gather_rows_wide_kernel<false, 0>);
    if (const cudaError_t ae = ensure_max_smem(kw)) return cuda_status(ae, "gather_rows_wide attr");
    const int Ho_w = (H + stride - 1) / stride, Wo_w = (W + stride - 1) / stride;
    const long long npix_w = static_cast<long long>(N) * Ho_w * Wo_w;
    int per_sm = static_cast<int>((227 * 1024) / (smem_w + 1024));
    if (per_sm > 2048 / (32 * ww)) per_sm = 2048 / (32 * ww);
    if (per_sm < 1) per_sm = 1;
    const long long want = (npix_w + ww - 1) / ww;
    const long long cap = static_cast<long long>(num_sms()) * per_sm;
    const int grid = static_cast<int>(want < cap ? want : cap);
    const cudaError_t e = launch_pdl(kw, dim3(grid), dim3(32 * ww), smem_w, stream, static_cast<const uint16_t*>(x),
                                     x_cstride, ws, win16, idx, n_idx, x_coff - ws, n8, npix_w, stride, H, W, Ho_w,
                                     Wo_w, scale, shift, relu, static_cast<uint16_t*>(y), y_cstride, y_coff);
    count_launch();
    return cuda_status(e, "gather_rows_wide_kernel");
  }
  if (!pool2 && stride == 1 && n8 <= 1024) {  // fast form: fixed per-lane ownership of output groups
    const int groups = n8 / 8;
    const int gj = groups <= 32 ? 1 : (groups + 31) / 32;
    const int pbf = gj == 1 ? 32 / groups : 1;
    if (pbf * win16 <= 32 * GRF_MAXI) {
      const size_t stage_f = static_cast<size_t>(pbf) * win16 * 16;
      const size_t par = (gj > 1 && affine) ? ((2 * n8 * 4 + 15) & ~15) : 0;
      int wf = 8;
      while (wf > 1 && par + wf * 4 * stage_f > 200 * 1024) wf >>= 1;
      const size_t smem_f = par + wf * 4 * stage_f;
      void (*kf)(const uint16_t*, int, int, int, int, const int32_t*, int, int, int, long long, const float*,
                 const float*, int, uint16_t*, int, int) = nullptr;
      switch (gj) {
        case 1: kf = affine ? gather_rows_fast_kernel<true, 1> : gather_rows_fast_kernel<false, 1>; break;
        case 2: kf = affine ? gather_rows_fast_kernel<true, 2> : gather_rows_fast_kernel<false, 2>; break;
        case 3: kf = affine ? gather_rows_fast_kernel<true, 3> : gather_rows_fast_kernel<false, 3>; break;
        default: kf = affine ? gather_rows_fast_kernel<true, 4> : gather_rows_fast_kernel<false, 4>; break;
      }
      if (const cudaError_t ae = ensure_max_smem(kf)) return cuda_status(ae, "gather_rows_fast attr");
      const long long npix_f = static_cast<long long>(N) * H * W;
      const long long nb = (npix_f + pbf - 1) / pbf;
      int per_sm = static_cast<int>((227 * 1024) / (smem_f + 1024));
      if (per_sm > 2048 / (32 * wf)) per_sm = 2048 / (32 * wf);
      if (per_sm < 1) per_sm = 1;
      const long long want = (nb + wf - 1) / wf;
      const long long cap = static_cast<long long>(num_sms()) * per_sm;
      const int grid = static_cast<int>(want < cap ? want : cap);
      const cudaError_t e = launch_pdl(kf, dim3(grid), dim3(32 * wf), smem_f, stream, static_cast<const uint16_t*>(x),
                                       x_cstride, ws, win16, pbf, idx, n_idx, x_coff - ws, n8, npix_f, scale, shift,
                                       relu, static_cast<uint16_t*>(y), y_cstride, y_coff);
      count_launch();
      return cuda_status(e, "gather_rows_fast_kernel");
    }
  }
  const int idx_bytes = ((affine ? 3 : 1) * n8 * 4 + 15) & ~15;
  // pixels per warp step: ~96 16-byte chunks per cp.async wave (3 per lane), at most 16 pixels
  int pb = 96 / (rows * win16);
  pb = pb < 1 ? 1 : (pb > 16 ? 16 : pb);
  // ... and enough pixels that every lane owns an output group (pool2 windows are wide)
  while (pb < 16 && pb * (n8 / 8) < 32 && (pb + 1) * rows * win16 <= 192) ++pb;
  const size_t stage = static_cast<size_t>(pb) * rows * win16 * 16;
  int warps = 8;
  while (warps > 1 && idx_bytes + warps * 3 * stage > 200 * 1024) warps >>= 1;
  const size_t smem = idx_bytes + warps * 3 * stage;
  if (smem > 227 * 1024) return fail(UB_EUNSUPPORTED, "ub_gather_rows: window of %d channels", we - ws);
  void (*kern)(const uint16_t*, int, int, int, int, const int32_t*, int, int, int, int, int, int, int, int, int,
               const float*, const float*, int, uint16_t*, int, int) =
      pool2 ? (affine ? gather_rows_kernel<4, true> : gather_rows_kernel<4, false>)
            : (affine ? gather_rows_kernel<1, true> : gather_rows_kernel<1, false>);
  if (const cudaError_t ae = ensure_max_smem(kern)) return cuda_status(ae, "gather_rows attr");
  const int Ho = pool2 ? H / 2 : (H + stride - 1) / stride, Wo = pool2 ? W / 2 : (W + stride - 1) / stride;
  const long long npix = static_cast<long long>(N) * Ho * Wo;
  if (npix >= (1ll << 31)) return fail(UB_EUNSUPPORTED, "ub_gather_rows: too many output pixels");
  int per_sm = static_cast<int>((227 * 1024) / (smem + 1024));
  if (per_sm > 2048 / (32 * warps)) per_sm = 2048 / (32 * warps);
  if (per_sm < 1) per_sm = 1;
  const long long nbatch = (npix + pb - 1) / pb;
  const long long want = (nbatch + warps - 1) / warps;
  const long long cap = static_cast<long long>(num_sms()) * per_sm;
  const int grid = static_cast<int>(want < cap ? want : cap);
  const cudaError_t e = launch_pdl(kern, dim3(grid), dim3(32 * warps), smem, stream, static_cast<const uint16_t*>(x),
                                   x_cstride, ws, win16, pb, idx, n_idx, x_coff - ws, n8, N, H, W, stride, Ho, Wo,
                                   scale, shift, relu, static_cast<uint16_t*>(y), y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "gather_rows_kernel");
}

extern "C" int ub_gather_rows(const void* x, int x_cstride, int x_coff, int lo, int hi, const int32_t* idx,
                              int n_idx, int N, int H, int W, int stride, void* y, int y_cstride, int y_coff,
                              cudaStream_t stream) {
  return ub_gather_rows_ex(x, x_cstride, x_coff, lo, hi, idx, n_idx, N, H, W, stride, 0, nullptr, nullptr, 0, y,
                           y_cstride, y_coff, stream);
}

extern "C" int ub_stage_input(const float* x, int N, int C, int H, int W, const int32_t* idx, int n, void* y,
                              int y_cstride, cudaStream_t stream) {
  if (!x || !y || N < 1 || C < 1 || H < 1 || W < 1) return fail(UB_EINVAL, "ub_stage_input: bad arguments");
  if (!idx) n = C;
  if (n > y_cstride) return fail(UB_EINVAL, "ub_stage_input: n > y_cstride");
  const long long total = (long long)N * H * W;
  stage_input_kernel<<<grid_for(total, 256), 256, 0, stream>>>(x, N, C, H * W, idx, n,
                                                               static_cast<__nv_bfloat16*>(y), y_cstride);
  count_launch();
  return cuda_status(cudaGetLastError(), "stage_input_kernel");
}

extern "C" int ub_h2d_input_channels(const float* host_nchw, int N, int C, int HW, const int32_t* channels, int n,
                                     float* dev_nchw, long long* bytes, cudaStream_t stream) {
  if (!host_nchw || !dev_nchw || !channels || N < 1 || C < 1 || HW < 1 || n < 1 || n > C)
    return fail(UB_EINVAL, "ub_h2d_input_channels: bad arguments");
  const size_t plane = static_cast<size_t>(HW) * sizeof(float);
  const size_t pitch = plane * C;
  for (int i = 0; i < n; ++i) {
    const int c = channels[i];
    if (c < 0 || c >= C) return fail(UB_EINVAL, "ub_h2d_input_channels: channel %d out of range", c);
    const cudaError_t e = cudaMemcpy2DAsync(reinterpret_cast<char*>(dev_nchw) + c * plane, pitch,
                                            reinterpret_cast<const char*>(host_nchw) + c * plane, pitch, plane, N,
                                            cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return cuda_status(e, "ub_h2d_input_channels");
  }
  if (bytes) *bytes = static_cast<long long>(n) * N * plane;
  return UB_OK;
}

// Row-staged max pool for the 3x3 / stride-2 window (ResNet's): one CTA per band of ROWS
// output rows of one image.  Each thread owns fixed 16-byte pieces (w, channel group) of the
// input rows; per output row it loads input rows 2h and 2h+1 and carries row 2h-1 from the
// previous output row in registers, so every input row is read once per band (bf16 max is
// exact: __hmax2 on packed pairs).  The vertical maxima go to a shared [W][groups] row and
// each output pixel then takes the horizontal window of that row.
constexpr int MP_ROWS = 4;     // output rows per CTA
constexpr int MP_PER_T = 4;    // 16-byte pieces per thread per input row (W*groups <= 4*blockDim)
__global__ void maxpool3s2_rows_kernel(const uint4* __restrict__ x, int H, int W, int groups, int x_cs16,
                                       int x_co16, int Ho, int Wo, uint4* __restrict__ y, int y_cs16, int y_co16) {
  griddep_wait();
  griddep_launch_dependents();
  extern __shared__ uint4 vrow[];  // [W][groups]
  const int bands = (Ho + MP_ROWS - 1) / MP_ROWS;
  const int img = blockIdx.x / bands;
  const int ho0 = (blockIdx.x - img * bands) * MP_ROWS;
  const int total = W * groups;
  const __nv_bfloat162 ninf = __floats2bfloat162_rn(-INFINITY, -INFINITY);
  uint4 ninf4;
  {
    __nv_bfloat162* v = reinterpret_cast<__nv_bfloat162*>(&ninf4);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = ninf;
  }
  size_t off[MP_PER_T];
#pragma unroll
  for (int b = 0; b < MP_PER_T; ++b) {
    const int e = threadIdx.x + b * blockDim.x;
    const int wi = e / groups, g = e - (e / groups) * groups;
    off[b] = static_cast<size_t>(wi) * x_cs16 + x_co16 + g;
  }
  const uint4* ximg = x + static_cast<size_t>(img) * H * W * x_cs16;
  uint4 carry[MP_PER_T];
  {
    const int r = 2 * ho0 - 1;
#pragma unroll
    for (int b = 0; b < MP_PER_T; ++b) {
      const int e = threadIdx.x + b * blockDim.x;
      carry[b] = (r >= 0 && r < H && e < total) ? __ldg(ximg + static_cast<size_t>(r) * W * x_cs16 + off[b]) : ninf4;
    }
  }
  const int ho1 = min(ho0 + MP_ROWS, Ho);
  for (int ho = ho0; ho < ho1; ++ho) {
    const int ra = 2 * ho, rb = 2 * ho + 1;
    uint4 a[MP_PER_T], c[MP_PER_T];
#pragma unroll
    for (int b = 0; b < MP_PER_T; ++b) {
      const int e = threadIdx.x + b * blockDim.x;
      a[b] = (ra < H && e < total) ? __ldg(ximg + static_cast<size_t>(ra) * W * x_cs16 + off[b]) : ninf4;
      c[b] = (rb < H && e < total) ? __ldg(ximg + static_cast<size_t>(rb) * W * x_cs16 + off[b]) : ninf4;
    }
    if (ho > ho0) __syncthreads();  // previous row's horizontal pass is done with vrow
#pragma unroll
    for (int b = 0; b < MP_PER_T; ++b) {
      const int e = threadIdx.x + b * blockDim.x;
      uint4 m = carry[b];
      __nv_bfloat162* mv = reinterpret_cast<__nv_bfloat162*>(&m);
      const __nv_bfloat162* av = reinterpret_cast<const __nv_bfloat162*>(&a[b]);
      const __nv_bfloat162* cv = reinterpret_cast<const __nv_bfloat162*>(&c[b]);
#pragma unroll
      for (int i = 0; i < 4; ++i) mv[i] = __hmax2(mv[i], __hmax2(av[i], cv[i]));
      if (e < total) vrow[e] = m;
      carry[b] = c[b];
    }
    __syncthreads();
    uint4* yrow = y + static_cast<size_t>(img * Ho + ho) * Wo * y_cs16 + y_co16;
    for (int e = threadIdx.x; e < Wo * groups; e += blockDim.x) {
      const int wo = e / groups, g = e - (e / groups) * groups;
      const int w0 = 2 * wo - 1;
      uint4 m = vrow[(2 * wo) * groups + g];
      __nv_bfloat162* mv = reinterpret_cast<__nv_bfloat162*>(&m);
      if (w0 >= 0) {
        const uint4 u = vrow[w0 * groups + g];
        const __nv_bfloat162* uv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) mv[i] = __hmax2(mv[i], uv[i]);
      }
      if (w0 + 2 < W) {
        const uint4 u = vrow[(w0 + 2) * groups + g];
        const __nv_bfloat162* uv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) mv[i] = __hmax2(mv[i], uv[i]);
      }
      yrow[static_cast<size_t>(wo) * y_cs16 + g] = m;
    }
  }
}

extern "C" int ub_maxpool2d(const void* x, int N, int H, int W, int C, int x_cstride, int x_coff, int k, int stride,
                            int pad, int Ho, int Wo, void* y, int y_cstride, int y_coff, cudaStream_t stream) {
  if (!x || !y || N < 1 || C < 1 || k < 1 || stride < 1) return fail(UB_EINVAL, "ub_maxpool2d: bad arguments");
  const bool vec = aligned16(x) && aligned16(y) && (x_cstride % 8 == 0) && (x_coff % 8 == 0) &&
                   (y_cstride % 8 == 0) && (y_coff % 8 == 0);
  const long long total = (long long)N * Ho * Wo * ((C + 7) / 8);
  if (total >= (1ll << 31)) return fail(UB_EUNSUPPORTED, "ub_maxpool2d: tensor too large");
  const int groups = (C + 7) / 8;
  const size_t row_smem = static_cast<size_t>(W) * groups * 16;
  // whole 16-byte groups; a ragged last group is allowed when it is the tail of both rows
  // (the padding channels of y get the max of x's padding channels)
  const bool whole = C % 8 == 0 || (y_coff + groups * 8 == y_cstride && x_coff + groups * 8 <= x_cstride);
  const int block = 256;
  if (vec && whole && k == 3 && stride == 2 && pad == 1 && W * groups <= MP_PER_T * block &&
      row_smem <= 48 * 1024 && (long long)N * ((Ho + MP_ROWS - 1) / MP_ROWS) < (1ll << 31)) {
    const int grid = N * ((Ho + MP_ROWS - 1) / MP_ROWS);
    const cudaError_t e = launch_pdl(maxpool3s2_rows_kernel, dim3(grid), dim3(block), row_smem, stream,
                                     static_cast<const uint4*>(x), H, W, groups, x_cstride / 8, x_coff / 8, Ho, Wo,
                                     static_cast<uint4*>(y), y_cstride / 8, y_coff / 8);
    count_launch();
    return cuda_status(e, "maxpool3s2_rows_kernel");
  }
  maxpool_kernel<<<grid_for(total, 256), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(x), N, H, W, C, x_cstride, x_coff, k, stride, pad, Ho, Wo,
      static_cast<__nv_bfloat16*>(y), y_cstride, y_coff, vec);
  count_launch();
  return cuda_status(cudaGetLastError(), "maxpool_kernel");
}

extern "C" int ub_avgpool_global(const void* x, int N, int HW, int C, int x_cstride, int x_coff, void* y,
                                 int y_cstride, int y_coff, cudaStream_t stream) {
  if (!x || !y || N < 1 || HW < 1 || C < 1) return fail(UB_EINVAL, "ub_avgpool_global: bad arguments");
  if (N > 65535) return fail(UB_EUNSUPPORTED, "ub_avgpool_global: N too large");
  if (C % 8 == 0 && x_cstride % 8 == 0 && x_coff % 8 == 0 && y_cstride % 8 == 0 && y_coff % 8 == 0 && aligned16(x) &&
      aligned16(y)) {
    const int C8 = C / 8;
    dim3 grid8((C8 + 127) / 128, N);
    const cudaError_t e = launch_pdl(avgpool8_kernel, grid8, dim3(128), 0, stream, static_cast<const uint4*>(x), HW,
                                     C8, x_cstride / 8, x_coff / 8, static_cast<uint4*>(y), y_cstride / 8, y_coff / 8);
    count_launch();
    return cuda_status(e, "avgpool8_kernel");
  }
  dim3 grid((C + 127) / 128, N);
  const cudaError_t e = launch_pdl(avgpool_kernel, grid, dim3(128), 0, stream, static_cast<const __nv_bfloat16*>(x),
                                   HW, C, x_cstride, x_coff, static_cast<__nv_bfloat16*>(y), y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "avgpool_kernel");
}

extern "C" int ub_avgpool_gather(const void* x, int N, int HW, int C, int x_cstride, int x_coff,
                                 const int32_t* idx, int n_idx, void* y, int y_cstride, int y_coff,
                                 cudaStream_t stream) {
  if (!x || !y || !idx || N < 1 || HW < 1 || C < 1 || n_idx < 1 || y_cstride < y_coff + n_idx)
    return fail(UB_EINVAL, "ub_avgpool_gather: bad arguments");
  if (C % 8 || x_cstride % 8 || x_coff % 8 || !aligned16(x))
    return fail(UB_EUNSUPPORTED, "ub_avgpool_gather: C, x_cstride and x_coff must be multiples of 8");
  if (N > 65535) return fail(UB_EUNSUPPORTED, "ub_avgpool_gather: N too large");
  const int C8 = C / 8;
  if (static_cast<long long>(N) * ((C8 + 127) / 128) < num_sms()) {  // small batch: phased form
    const dim3 grid((C8 + 31) / 32, N);
    const cudaError_t e = launch_pdl(avgpool_gather_phased_kernel, grid, dim3(256), 0, stream,
                                     static_cast<const uint4*>(x), HW, C8, x_cstride / 8, x_coff / 8, idx, n_idx,
                                     static_cast<__nv_bfloat16*>(y), y_cstride, y_coff);
    count_launch();
    return cuda_status(e, "avgpool_gather_phased_kernel");
  }
  const dim3 grid((C8 + 127) / 128, N);
  const cudaError_t e = launch_pdl(avgpool_gather_kernel, grid, dim3(128), 0, stream, static_cast<const uint4*>(x), HW,
                                   C8, x_cstride / 8, x_coff / 8, idx, n_idx, static_cast<__nv_bfloat16*>(y),
                                   y_cstride, y_coff);
  count_launch();
  return cuda_status(e, "avgpool_gather_kernel");
}

extern "C" int ub_affine_add_relu(const void* a, int a_cstride, int a_coff, const float* scale, const float* shift,
                                  const void* b, int b_cstride, int b_coff, int relu, long long npix, int C, void* y,
                                  int y_cstride, int y_coff, cudaStream_t stream) {
  if (!a || !y || npix < 1 || C < 1) return fail(UB_EINVAL, "ub_affine_add_relu: bad arguments");
  affine_add_relu_kernel<<<grid_for(npix * C, 256, 4), 256, 0, stream>>>(
      static_cast<const __nv_bfloat16*>(a), a_cstride, a_coff, scale, shift, static_cast<const __nv_bfloat16*>(b),
      b_cstride, b_coff, relu, npix, C, static_cast<__nv_bfloat16*>(y), y_cstride, y_coff);
  count_launch();
  return cuda_status(cudaGetLastError(), "affine_add_relu_kernel");
}

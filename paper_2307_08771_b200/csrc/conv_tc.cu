// Implicit-GEMM convolution on sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// One reference CHANNEL_MIX node (interp.py:57-63, `W @ x`) executed over real
// NHWC activations, with the node that reads its input and the nodes that
// consume its output fused in:
//   * SLICE read  (interp.py:72-74): the A operand's TMA descriptor starts at the
//     slice's channel offset -- no copy (UPSCALE's contiguous read);
//   * GATHER read (interp.py:75-77): dedicated gather warps build the A tile
//     (implicit im2col over the gathered channels) straight from the producer's
//     tensor into swizzled shared memory -- the copy the baseline export
//     materialises never touches HBM;
//   * PER_CHANNEL bias (BN shift; the scale is folded into the weight rows at
//     export), ADD residual, ReLU, and a channel-offset store (CONCAT without a
//     copy).
//
// GEMM view: D[M = N*Ho*Wo pixels][cout] = A[M][K] * B[cout][K]^T, K = taps*cpad.
// Tile 128 pixels x block_n channels (block_n <= 256, multiple of 16, runtime).
//
// Persistent, warp-specialised, one CTA per SM; tiles are strided over the grid.
//   warp 0      TMA producer (A: 2-D tiled or im2col; B: weights)
//   warp 1      MMA issuer: tcgen05.mma into one of TWO TMEM accumulators, so the
//               epilogue of tile i overlaps the mainloop of tile i+1
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: TMEM -> regs (+bias, +residual, ReLU) -> swizzled smem
//               -> TMA bulk store; the residual tile arrives by TMA load,
//               double-buffered one 32-channel chunk ahead
//   warps 8-11  gather producers (GATHER mode only)
#include <mutex>

#include "ub_common.cuh"
#include "ub_host.h"

namespace ub {

enum AMode : int { A_TILED = 0, A_IM2COL = 1, A_GATHER = 2 };

constexpr int BLOCK_M = 128;
constexpr int EPI_CHUNK = 32;                // output channels per epilogue chunk
constexpr int EPI_BUF = 32 * EPI_CHUNK * 2;  // one warp's 32 rows x 32 ch bf16 staging buffer
constexpr int MAX_BLOCK_N = 256;

struct ConvKParams {
  int M;        // output pixels (GEMM M)
  int cout;     // output channels (GEMM N)
  int block_n;  // N tile
  int num_kb;   // k-blocks per tile
  int cchunks;  // channel chunks per tap
  int kw;       // filter width
  int cpad;     // per-tap weight K
  int H, W, Ho, Wo, stride, pad;
  int stages;
  int m_tiles, n_tiles;
  uint32_t tmem_cols, acc_stride;
  // fused gather source
  const uint16_t* x;
  int x_cstride, x_coff;
  const int32_t* gidx;
  int n_gather;
  // epilogue
  const float* bias;
  int has_res, relu, epi_tma;
  const __nv_bfloat16* res;  // direct-store fallback only
  int res_cstride, res_coff;
  void* y;
  int y_cstride, y_coff, y_f32;
};

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// Byte offset of 16-byte chunk j of row r in a 64-byte-row SWIZZLE_64B buffer.
__device__ __forceinline__ uint32_t swz64(uint32_t r, uint32_t j) { return r * 64 + ((j ^ ((r >> 1) & 3)) << 4); }

template <int AMODE, int BK>
__global__ void __launch_bounds__(AMODE == A_GATHER ? 384 : 256, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmR,
                   const ConvKParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr uint32_t A_BYTES = BLOCK_M * BK * 2;
  constexpr uint32_t ROW_BYTES = BK * 2;
  constexpr uint32_t SBO = 8 * ROW_BYTES;
  constexpr uint32_t LAYOUT = (BK == 64) ? 2u : 6u;  // SWIZZLE_128B : SWIZZLE_32B
  const uint32_t b_bytes = static_cast<uint32_t>(p.block_n) * ROW_BYTES;
  const uint32_t b_stride = (b_bytes + 1023u) & ~1023u;
  const int stages = p.stages;

  uint8_t* sA = smem;
  uint8_t* sB = sA + stages * A_BYTES;
  uint8_t* sE = sB + stages * b_stride;                           // 4 warps x 2 x EPI_BUF (1024-aligned)
  float* sBias = reinterpret_cast<float*>(sE + 4 * 2 * EPI_BUF);  // 4 warps x MAX_BLOCK_N
  uint64_t* full = reinterpret_cast<uint64_t*>(sBias + 4 * MAX_BLOCK_N);
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint64_t* rbar = tempty + 2;       // [4 warps][2 buffers]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = p.m_tiles * p.n_tiles;
  const int nk = p.num_kb;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (p.epi_tma) {
      tma_prefetch_desc(&tmY);
      if (p.has_res) tma_prefetch_desc(&tmR);
    }
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], AMODE == A_GATHER ? 1 + 4 : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    for (int i = 0; i < 8; ++i) mbar_init(&rbar[i], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ================= TMA producer
      int g = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int m_tile = t / p.n_tiles;
        const int n0 = (t - m_tile * p.n_tiles) * p.block_n;
        const int m0 = m_tile * BLOCK_M;
        int w_start = 0, h_start = 0, n_img = 0;
        if (AMODE == A_IM2COL) {
          const int hw = p.Ho * p.Wo;
          n_img = m0 / hw;
          const int rem = m0 - n_img * hw;
          const int ho = rem / p.Wo;
          w_start = (rem - ho * p.Wo) * p.stride - p.pad;
          h_start = ho * p.stride - p.pad;
        }
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % stages;
          const uint32_t ph = (g / stages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], b_bytes + (AMODE == A_GATHER ? 0u : A_BYTES));
          int kcoord = kb * BK;
          if (AMODE == A_TILED) {
            tma_load_2d(&tmA, &full[s], sA + s * A_BYTES, kb * BK, m0);
          } else if (AMODE == A_IM2COL) {
            const int tap = kb / p.cchunks;
            const int cc = kb - tap * p.cchunks;
            const int r = tap / p.kw;
            tma_load_im2col_4d(&tmA, &full[s], sA + s * A_BYTES, cc * BK, w_start, h_start, n_img,
                               static_cast<uint16_t>(tap - r * p.kw), static_cast<uint16_t>(r));
            kcoord = tap * p.cpad + cc * BK;
          }
          tma_load_2d(&tmB, &full[s], sB + s * b_stride, kcoord, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ================= MMA issuer
      const uint32_t idesc = make_idesc_bf16(BLOCK_M, static_cast<uint32_t>(p.block_n));
      int g = 0, it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * p.acc_stride;
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % stages;
          const uint32_t ph = (g / stages) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + s * A_BYTES);
          const uint32_t b_base = smem_u32(sB + s * b_stride);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            umma_bf16(d, make_sdesc(a_base + k * 32, SBO, LAYOUT), make_sdesc(b_base + k * 32, SBO, LAYOUT), idesc,
                      (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 8) {
    if constexpr (AMODE == A_GATHER) {
      // ================= gather producers: implicit im2col over gathered channels
      // A[row][j] of tap (r, s) = x[pixel(row) + (r, s)][x_coff + gidx[cc*64 + j]], 0 outside.
      const int qg = warp - 8;
      const int hw = p.Ho * p.Wo;
      int g = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int m0 = (t / p.n_tiles) * BLOCK_M;
        int g_img = 0, g_hb = -(1 << 28), g_wb = 0;  // lane owns row qg*32 + lane
        {
          const int m = m0 + qg * 32 + lane;
          if (m < p.M) {
            g_img = m / hw;
            const int rem = m - g_img * hw;
            const int ho = rem / p.Wo;
            g_hb = ho * p.stride - p.pad;
            g_wb = (rem - ho * p.Wo) * p.stride - p.pad;
          }
        }
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int s = g % stages;
          const uint32_t ph = (g / stages) & 1;
          const int tap = kb / p.cchunks;
          const int cc = kb - tap * p.cchunks;
          const int fr = tap / p.kw;
          const int fs = tap - fr * p.kw;
          const int j = cc * 64 + lane * 2;
          const int i0 = j < p.n_gather ? __ldg(p.gidx + j) : -1;
          const int i1 = (j + 1) < p.n_gather ? __ldg(p.gidx + j + 1) : -1;
          uint32_t vals[32];
#pragma unroll
          for (int u = 0; u < 32; ++u) {  // all 64 loads of this lane in flight before any store
            const int img = __shfl_sync(0xffffffffu, g_img, u);
            const int hi = __shfl_sync(0xffffffffu, g_hb, u) + fr;
            const int wi = __shfl_sync(0xffffffffu, g_wb, u) + fs;
            uint32_t a = 0, b = 0;
            if (hi >= 0 && hi < p.H && wi >= 0 && wi < p.W) {
              const uint16_t* xr =
                  p.x + ((static_cast<size_t>(img) * p.H + hi) * p.W + wi) * p.x_cstride + p.x_coff;
              if (i0 >= 0) a = __ldg(xr + i0);
              if (i1 >= 0) b = __ldg(xr + i1);
            }
            vals[u] = a | (b << 16);
          }
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* tile = sA + s * A_BYTES;
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int row = qg * 32 + u;
            const uint32_t off = row * 128 + ((((lane >> 2) ^ (row & 7)) << 4)) + ((lane & 3) << 2);
            *reinterpret_cast<uint32_t*>(tile + off) = vals[u];
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[s]);
        }
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue
    const int q = warp - 4;  // TMEM lane quarter (warp % 4)
    uint8_t* ebuf = sE + q * 2 * EPI_BUF;
    float* sb = sBias + q * MAX_BLOCK_N;
    uint64_t* rb = rbar + q * 2;
    uint32_t ec = 0;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      const int m_tile = t / p.n_tiles;
      const int n0 = (t - m_tile * p.n_tiles) * p.block_n;
      const int m0 = m_tile * BLOCK_M;
      const int rows0 = m0 + q * 32;
      const int ncols = min(p.block_n, p.cout - n0);
      const int nchunks = (ncols + EPI_CHUNK - 1) / EPI_CHUNK;
      __syncwarp();
      for (int i = lane; i < nchunks * EPI_CHUNK; i += 32) sb[i] = (p.bias && i < ncols) ? __ldg(p.bias + n0 + i) : 0.f;
      __syncwarp();
      if (p.epi_tma && p.has_res && lane == 0) {  // residual chunk 0, in flight during the mainloop
        bulk_wait_read<0>();
        mbar_arrive_expect_tx(&rb[ec & 1], EPI_BUF);
        tma_load_2d(&tmR, &rb[ec & 1], ebuf + (ec & 1) * EPI_BUF, n0, rows0);
      }
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * p.acc_stride + (static_cast<uint32_t>(q * 32) << 16);
      for (int c = 0; c < nchunks; ++c, ++ec) {
        const uint32_t b = ec & 1;
        uint32_t r[32];
        tmem_ld32(taddr + c * EPI_CHUNK, r);
        tmem_ld_wait();
        if (c == nchunks - 1) {  // accumulator drained: MMA may start the tile after next
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) + sb[c * EPI_CHUNK + i];
        if (p.epi_tma) {
          uint8_t* buf = ebuf + b * EPI_BUF;
          if (p.has_res) {
            if (lane == 0 && c + 1 < nchunks) {
              bulk_wait_read<0>();  // the other buffer's last store has read smem
              mbar_arrive_expect_tx(&rb[b ^ 1], EPI_BUF);
              tma_load_2d(&tmR, &rb[b ^ 1], ebuf + (b ^ 1) * EPI_BUF, n0 + (c + 1) * EPI_CHUNK, rows0);
            }
            mbar_wait(&rb[b], (ec >> 1) & 1);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const uint4 u = *reinterpret_cast<const uint4*>(buf + swz64(lane, jj));
              const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
              for (int h = 0; h < 4; ++h) {
                const float2 f = unpack_bf16x2(w4[h]);
                v[jj * 8 + 2 * h] += f.x;
                v[jj * 8 + 2 * h + 1] += f.y;
              }
            }
          } else {
            if (lane == 0) bulk_wait_read<1>();  // this buffer's store from two chunks ago has read smem
            __syncwarp();
          }
          if (p.relu) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
          }
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            uint4 o;
            o.x = pack_bf16x2(v[jj * 8 + 0], v[jj * 8 + 1]);
            o.y = pack_bf16x2(v[jj * 8 + 2], v[jj * 8 + 3]);
            o.z = pack_bf16x2(v[jj * 8 + 4], v[jj * 8 + 5]);
            o.w = pack_bf16x2(v[jj * 8 + 6], v[jj * 8 + 7]);
            *reinterpret_cast<uint4*>(buf + swz64(lane, jj)) = o;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmY, buf, n0 + c * EPI_CHUNK, rows0);
            bulk_commit();
          }
        } else {
          // direct-store fallback (fp32 logits / unaligned views)
          const int m = rows0 + lane;
          const int nb = n0 + c * EPI_CHUNK;
          const int nv = min(EPI_CHUNK, p.cout - nb);
          if (m < p.M) {
            if (p.has_res) {
              const __nv_bfloat16* rp = p.res + static_cast<size_t>(m) * p.res_cstride + p.res_coff + nb;
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (i < nv) v[i] += __bfloat162float(rp[i]);
            }
            if (p.relu) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
            }
            const size_t yo = static_cast<size_t>(m) * p.y_cstride + p.y_coff + nb;
            if (p.y_f32) {
              float* yp = reinterpret_cast<float*>(p.y) + yo;
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (i < nv) yp[i] = v[i];
            } else {
              __nv_bfloat16* yp = reinterpret_cast<__nv_bfloat16*>(p.y) + yo;
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (i < nv) yp[i] = __float2bfloat16_rn(v[i]);
            }
          }
        }
      }
    }
    if (p.epi_tma && lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, p.tmem_cols);
}

// ------------------------------------------------------------------ host side

namespace {

int g_driver_version = -1;
int g_num_sms = -1;

void apply_small_tensor_quirk(CUtensorMap* map, size_t footprint_bytes) {
  // Same workaround CUTLASS applies for drivers <= 13.1 (copy_traits_sm90_tma.hpp).
  if (g_driver_version < 0) {
    int v = 0;
    cudaDriverGetVersion(&v);
    g_driver_version = v;
  }
  if (g_driver_version <= 13010 && footprint_bytes < 131072)
    reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
}

int num_sms() {
  if (g_num_sms < 0) {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    g_num_sms = n > 0 ? n : 148;
  }
  return g_num_sms;
}

template <int AMODE, int BK>
int launch_conv(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmY, const CUtensorMap& tmR,
                const ConvKParams& p, int grid, size_t smem, cudaStream_t stream) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(conv_tc_kernel<AMODE, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    227 * 1024);
  });
  if (attr_err != cudaSuccess) return cuda_status(attr_err, "cudaFuncSetAttribute(conv)");
  const int threads = AMODE == A_GATHER ? 384 : 256;
  conv_tc_kernel<AMODE, BK><<<grid, threads, smem, stream>>>(tmA, tmB, tmY, tmR, p);
  count_launch();
  return cuda_status(cudaGetLastError(), "conv_tc_kernel launch");
}

int pick_bk(int cin_eff) { return cin_eff <= 16 ? 16 : 64; }

int encode_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                   uint32_t box_inner, uint32_t box_outer, int swizzle_bytes, const char* what) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_tiled_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                                 box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(swizzle_bytes),
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_fwd: encode %s tensor map failed (%d)", what, (int)r);
  apply_small_tensor_quirk(map, static_cast<size_t>(outer) * row_bytes);
  return UB_OK;
}

}  // namespace
}  // namespace ub

using namespace ub;

extern "C" int ub_conv_weight_layout(int cin, int coff, int gather, int* lead, int* cpad) {
  if (cin < 1 || coff < 0 || !lead || !cpad) return fail(UB_EINVAL, "ub_conv_weight_layout: bad arguments");
  const int ld = gather ? 0 : (coff & 7);
  const int ce = cin + ld;
  const int bk = gather ? 64 : pick_bk(ce);
  *lead = ld;
  *cpad = (ce + bk - 1) / bk * bk;
  return UB_OK;
}

extern "C" int ub_conv_fwd(const ub_conv_desc* d, cudaStream_t stream) {
  if (!d) return fail(UB_EINVAL, "ub_conv_fwd: null descriptor");
  if (!d->x || !d->w || !d->y) return fail(UB_EINVAL, "ub_conv_fwd: null x/w/y");
  if (d->N < 1 || d->H < 1 || d->W < 1 || d->cin < 1 || d->cout < 1 || d->kh < 1 || d->kw < 1 || d->stride < 1 ||
      d->pad < 0 || d->Ho < 1 || d->Wo < 1)
    return fail(UB_EINVAL, "ub_conv_fwd: bad geometry");
  if (d->Ho != (d->H + 2 * d->pad - d->kh) / d->stride + 1 || d->Wo != (d->W + 2 * d->pad - d->kw) / d->stride + 1)
    return fail(UB_EINVAL, "ub_conv_fwd: Ho/Wo inconsistent with kernel/stride/pad");
  if (d->x_cstride % 8 || d->x_coff < 0 || (!d->gather_idx && d->x_coff + d->cin > d->x_cstride))
    return fail(UB_EINVAL, "ub_conv_fwd: x channel stride must be a multiple of 8 and cover the read");
  if (!aligned16(d->x) || !aligned16(d->w) || !aligned16(d->y))
    return fail(UB_EINVAL, "ub_conv_fwd: x/w/y must be 16-byte aligned");
  if (d->y_dtype != UB_BF16 && d->y_dtype != UB_F32) return fail(UB_EINVAL, "ub_conv_fwd: y_dtype");
  if (d->y_coff < 0 || d->y_coff + d->cout > d->y_cstride)
    return fail(UB_EINVAL, "ub_conv_fwd: output channels exceed y_cstride");
  if (d->residual && (d->res_coff < 0 || d->res_coff + d->cout > d->res_cstride))
    return fail(UB_EINVAL, "ub_conv_fwd: residual channels exceed res_cstride");
  if (d->kh > 64 || d->kw > 64) return fail(UB_EUNSUPPORTED, "ub_conv_fwd: filter too large");

  const bool gather = d->gather_idx != nullptr;
  const bool pointwise = d->kh == 1 && d->kw == 1 && d->stride == 1 && d->pad == 0;
  if (gather && d->x_coff % 8) return fail(UB_EINVAL, "ub_conv_fwd: gather base must be 8-aligned");

  int lead = 0, cpad = 0;
  ub_conv_weight_layout(d->cin, d->x_coff, gather ? 1 : 0, &lead, &cpad);
  if (d->w_lead != lead || d->w_cpad != cpad)
    return fail(UB_EINVAL, "ub_conv_fwd: weight layout (lead %d, cpad %d) != expected (lead %d, cpad %d)", d->w_lead,
                d->w_cpad, lead, cpad);
  const int cin_eff = d->cin + lead;
  const int bk = gather ? 64 : pick_bk(cin_eff);
  const int taps = d->kh * d->kw;
  const int K_total = taps * cpad;
  if (!encode_tiled_fn() || !encode_im2col_fn())
    return fail(UB_ECUDA, "ub_conv_fwd: cannot resolve cuTensorMapEncode* entry points");

  ConvKParams p{};
  p.M = d->N * d->Ho * d->Wo;
  p.cout = d->cout;
  p.n_tiles = (d->cout + MAX_BLOCK_N - 1) / MAX_BLOCK_N;
  // Multi-tile N: round to the epilogue's 32-channel chunk so a tile's last chunk never
  // spills into the next tile's channels (the TMA store only clips at cout).
  const int n_gran = p.n_tiles > 1 ? EPI_CHUNK : 16;
  p.block_n = (((d->cout + p.n_tiles - 1) / p.n_tiles) + n_gran - 1) / n_gran * n_gran;
  p.m_tiles = (p.M + BLOCK_M - 1) / BLOCK_M;
  p.cchunks = cpad / bk;
  p.num_kb = taps * p.cchunks;
  p.kw = d->kw;
  p.cpad = cpad;
  p.H = d->H;
  p.W = d->W;
  p.Ho = d->Ho;
  p.Wo = d->Wo;
  p.stride = d->stride;
  p.pad = d->pad;
  // two accumulators, each wide enough for the epilogue's 32-column chunks
  const uint32_t acc_cols = (static_cast<uint32_t>(p.block_n) + 31u) & ~31u;
  uint32_t tc = 32;
  while (tc < 2u * acc_cols) tc <<= 1;
  p.tmem_cols = tc;
  p.acc_stride = tc / 2;
  p.x = reinterpret_cast<const uint16_t*>(d->x);
  p.x_cstride = d->x_cstride;
  p.x_coff = d->x_coff;
  p.gidx = d->gather_idx;
  p.n_gather = gather ? d->cin : 0;
  p.bias = d->bias;
  p.has_res = d->residual != nullptr;
  p.relu = d->relu;
  p.res = reinterpret_cast<const __nv_bfloat16*>(d->residual);
  p.res_cstride = d->res_cstride;
  p.res_coff = d->res_coff;
  p.y = d->y;
  p.y_cstride = d->y_cstride;
  p.y_coff = d->y_coff;
  p.y_f32 = d->y_dtype == UB_F32;

  const uint16_t* ybase = reinterpret_cast<const uint16_t*>(d->y) + d->y_coff;
  const uint16_t* rbase = reinterpret_cast<const uint16_t*>(d->residual) + d->res_coff;
  p.epi_tma = !p.y_f32 && d->y_cstride % 8 == 0 && aligned16(ybase) &&
              (!p.has_res || (d->res_cstride % 8 == 0 && aligned16(rbase)));

  const uint32_t a_bytes = BLOCK_M * bk * 2;
  const uint32_t b_stride = (static_cast<uint32_t>(p.block_n) * bk * 2 + 1023u) & ~1023u;
  const uint32_t stage_bytes = a_bytes + b_stride;
  const uint32_t fixed = 1024 + 4 * 2 * EPI_BUF + 4 * MAX_BLOCK_N * 4 + 256;
  const uint32_t budget = 226u * 1024u - fixed;
  int stages = static_cast<int>(budget / stage_bytes);
  stages = stages < 2 ? 2 : (stages > 8 ? 8 : stages);
  p.stages = stages;
  const size_t smem = fixed + static_cast<size_t>(stages) * stage_bytes;

  CUtensorMap tmA{}, tmB{}, tmY{}, tmR{};
  int rc = encode_2d_bf16(&tmB, d->w, K_total, d->cout, static_cast<uint64_t>(K_total) * 2, bk, p.block_n, bk * 2,
                          "B (weights)");
  if (rc) return rc;
  if (p.epi_tma) {
    rc = encode_2d_bf16(&tmY, ybase, d->cout, p.M, static_cast<uint64_t>(d->y_cstride) * 2, EPI_CHUNK, 32, 64, "Y");
    if (rc) return rc;
    if (p.has_res) {
      rc = encode_2d_bf16(&tmR, rbase, d->cout, p.M, static_cast<uint64_t>(d->res_cstride) * 2, EPI_CHUNK, 32, 64,
                          "residual");
      if (rc) return rc;
    } else {
      tmR = tmY;
    }
  } else {
    tmY = tmB;
    tmR = tmB;
  }
  const uint16_t* xbase = reinterpret_cast<const uint16_t*>(d->x) + (d->x_coff - lead);
  const size_t x_footprint = static_cast<size_t>(d->N) * d->H * d->W * d->x_cstride * 2;
  int amode;
  if (gather) {
    amode = A_GATHER;
    tmA = tmB;  // unused by the kernel in gather mode
  } else if (pointwise) {
    amode = A_TILED;
    rc = encode_2d_bf16(&tmA, xbase, cin_eff, p.M, static_cast<uint64_t>(d->x_cstride) * 2, bk, BLOCK_M, bk * 2,
                        "A (tiled)");
    if (rc) return rc;
    apply_small_tensor_quirk(&tmA, x_footprint);
  } else {
    amode = A_IM2COL;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(cin_eff), static_cast<cuuint64_t>(d->W),
                          static_cast<cuuint64_t>(d->H), static_cast<cuuint64_t>(d->N)};
    const cuuint64_t cs = static_cast<cuuint64_t>(d->x_cstride) * 2;
    cuuint64_t strides[3] = {cs, cs * d->W, cs * d->W * d->H};
    int lower[2] = {-d->pad, -d->pad};
    int upper[2] = {d->pad - (d->kw - 1), d->pad - (d->kh - 1)};
    cuuint32_t es[4] = {1, static_cast<cuuint32_t>(d->stride), static_cast<cuuint32_t>(d->stride), 1};
    CUresult r = encode_im2col_fn()(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(xbase), dims,
                                    strides, lower, upper, static_cast<cuuint32_t>(bk), BLOCK_M, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(bk * 2),
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_fwd: encode A (im2col) tensor map failed (%d)", (int)r);
    apply_small_tensor_quirk(&tmA, x_footprint);
  }

  const int num_tiles = p.m_tiles * p.n_tiles;
  const int grid = num_tiles < num_sms() ? num_tiles : num_sms();
  if (amode == A_GATHER) return launch_conv<A_GATHER, 64>(tmA, tmB, tmY, tmR, p, grid, smem, stream);
  if (amode == A_TILED)
    return bk == 64 ? launch_conv<A_TILED, 64>(tmA, tmB, tmY, tmR, p, grid, smem, stream)
                    : launch_conv<A_TILED, 16>(tmA, tmB, tmY, tmR, p, grid, smem, stream);
  return bk == 64 ? launch_conv<A_IM2COL, 64>(tmA, tmB, tmY, tmR, p, grid, smem, stream)
                  : launch_conv<A_IM2COL, 16>(tmA, tmB, tmY, tmR, p, grid, smem, stream);
}

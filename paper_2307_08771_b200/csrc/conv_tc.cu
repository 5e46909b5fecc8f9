// Implicit-GEMM convolution on sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// One reference CHANNEL_MIX node (interp.py:57-63, `W @ x`) executed over real
// NHWC activations, with the node that reads its input and the nodes that
// consume its output fused in:
//   * SLICE read  (interp.py:72-74): the A operand's TMA descriptor starts at the
//     slice's channel offset -- no copy (UPSCALE's contiguous read);
//   * GATHER read (interp.py:75-77): the A tile is gathered straight from the
//     producer's tensor into swizzled shared memory by the epilogue warps while
//     the mainloop runs (the copy the baseline export materialises is fused);
//   * PER_CHANNEL bias (BN shift; scale folded into weight rows at export),
//     ADD residual, ReLU, and a channel-offset store (concat without a copy).
//
// GEMM view: D[M=N*Ho*Wo pixels][cout] = A[M][K] * B[cout][K]^T, K = taps*cpad.
// Tile: 128 pixels x block_n channels (block_n <= 256, multiple of 16, runtime).
// Warp roles (256 threads, one output tile per CTA, 2 CTAs/SM co-resident):
//   warp 0: TMA producer (one lane)      warp 1: MMA issuer (one lane)
//   warp 2: TMEM allocator                warps 4-7: [gather producers] + epilogue
#include <mutex>

#include "ub_common.cuh"
#include "ub_host.h"

namespace ub {

enum AMode : int { A_TILED = 0, A_IM2COL = 1, A_GATHER = 2 };

constexpr int BLOCK_M = 128;
constexpr int NUM_THREADS = 256;

struct ConvKParams {
  int M;        // output pixels (GEMM M)
  int cout;     // output channels (GEMM N)
  int block_n;  // N tile
  int num_kb;   // k-blocks
  int cchunks;  // channel chunks per tap
  int kw;       // filter width
  int cpad;     // per-tap weight K
  int H, W, Ho, Wo, stride, pad;
  int stages;
  uint32_t tmem_cols;
  // fused gather source
  const uint16_t* x;
  int x_cstride, x_coff;
  const int32_t* gidx;
  int n_gather;
  // epilogue
  const float* bias;
  const __nv_bfloat16* res;
  int res_cstride, res_coff, relu;
  void* y;
  int y_cstride, y_coff, y_f32;
};

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

template <int AMODE, int BK>
__global__ void __launch_bounds__(NUM_THREADS, 2)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
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
  uint8_t* sB = smem + stages * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + stages * b_stride);
  uint64_t* empty = full + stages;
  uint64_t* tmem_full = empty + stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * p.block_n;
  const int m0 = blockIdx.y * BLOCK_M;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], AMODE == A_GATHER ? 1 + 4 : 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nk = p.num_kb;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int w_start = 0, h_start = 0, n_img = 0;
      if (AMODE == A_IM2COL) {
        const int hw = p.Ho * p.Wo;
        n_img = m0 / hw;
        const int rem = m0 - n_img * hw;
        const int ho = rem / p.Wo;
        const int wo = rem - ho * p.Wo;
        w_start = wo * p.stride - p.pad;
        h_start = ho * p.stride - p.pad;
      }
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % stages;
        const uint32_t ph = (kb / stages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], b_bytes + (AMODE == A_GATHER ? 0u : A_BYTES));
        int kcoord = kb * BK;
        if (AMODE == A_TILED) {
          tma_load_2d(&tmA, &full[s], sA + s * A_BYTES, kb * BK, m0);
        } else if (AMODE == A_IM2COL) {
          const int tap = kb / p.cchunks;
          const int cc = kb - tap * p.cchunks;
          const int r = tap / p.kw;
          const int q = tap - r * p.kw;
          tma_load_im2col_4d(&tmA, &full[s], sA + s * A_BYTES, cc * BK, w_start, h_start, n_img,
                             static_cast<uint16_t>(q), static_cast<uint16_t>(r));
          kcoord = tap * p.cpad + cc * BK;
        }
        tma_load_2d(&tmB, &full[s], sB + s * b_stride, kcoord, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      const uint32_t idesc = make_idesc_bf16(BLOCK_M, static_cast<uint32_t>(p.block_n));
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % stages;
        const uint32_t ph = (kb / stages) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sA + s * A_BYTES);
        const uint32_t b_base = smem_u32(sB + s * b_stride);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          umma_bf16(tmem_base, make_sdesc(a_base + k * 32, SBO, LAYOUT), make_sdesc(b_base + k * 32, SBO, LAYOUT),
                    idesc, (kb | k) != 0 ? 1u : 0u);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
    }
  } else if (warp >= 4) {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    if constexpr (AMODE == A_GATHER) {
      // ---------------- fused GATHER (implicit im2col over gathered channels):
      // A[row][j] of tap (r, s) = x[pixel(row) + (r, s)][x_coff + gidx[cc*64 + j]], 0 outside.
      // Lane l owns the geometry of row q*32+l; rows are broadcast with shuffles.
      const int hw = p.Ho * p.Wo;
      int g_img = 0, g_hb = -(1 << 28), g_wb = 0;
      {
        const int m = m0 + q * 32 + lane;
        if (m < p.M) {
          g_img = m / hw;
          const int rem = m - g_img * hw;
          const int ho = rem / p.Wo;
          g_hb = ho * p.stride - p.pad;
          g_wb = (rem - ho * p.Wo) * p.stride - p.pad;
        }
      }
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % stages;
        const uint32_t ph = (kb / stages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        const int tap = kb / p.cchunks;
        const int cc = kb - tap * p.cchunks;
        const int fr = tap / p.kw;
        const int fs = tap - fr * p.kw;
        const int j = cc * 64 + lane * 2;
        const int i0 = j < p.n_gather ? __ldg(p.gidx + j) : -1;
        const int i1 = (j + 1) < p.n_gather ? __ldg(p.gidx + j + 1) : -1;
        uint8_t* tile = sA + s * A_BYTES;
#pragma unroll 1
        for (int rb = 0; rb < 32; rb += 8) {
          uint32_t vals[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int img = __shfl_sync(0xffffffffu, g_img, rb + u);
            const int hi = __shfl_sync(0xffffffffu, g_hb, rb + u) + fr;
            const int wi = __shfl_sync(0xffffffffu, g_wb, rb + u) + fs;
            uint32_t a = 0, b = 0;
            if (hi >= 0 && hi < p.H && wi >= 0 && wi < p.W) {
              const size_t pix = (static_cast<size_t>(img) * p.H + hi) * p.W + wi;
              const uint16_t* xr = p.x + pix * p.x_cstride + p.x_coff;
              if (i0 >= 0) a = __ldg(xr + i0);
              if (i1 >= 0) b = __ldg(xr + i1);
            }
            vals[u] = a | (b << 16);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int row = q * 32 + rb + u;
            const uint32_t off = row * 128 + ((((lane >> 2) ^ (row & 7)) << 4)) + ((lane & 3) << 2);
            *reinterpret_cast<uint32_t*>(tile + off) = vals[u];
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      }
    }
    // ---------------- epilogue: TMEM -> regs -> bias/residual/ReLU -> global
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const int row = q * 32 + lane;
    const int m = m0 + row;
    const bool valid = m < p.M;
    const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    for (int c = 0; c < p.block_n; c += 16) {
      const int n = n0 + c;
      if (n >= p.cout) break;  // warp-uniform
      uint32_t r[16];
      tmem_ld16(trow + c, r);
      tmem_ld_wait();
      if (!valid) continue;
      const int nv = min(16, p.cout - n);
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
      if (p.bias) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (i < nv) v[i] += __ldg(p.bias + n + i);
      }
      if (p.res) {
        const __nv_bfloat16* rp = p.res + static_cast<size_t>(m) * p.res_cstride + p.res_coff + n;
        if (nv == 16 && ((reinterpret_cast<uintptr_t>(rp) & 15) == 0)) {
          const uint4 u0 = __ldg(reinterpret_cast<const uint4*>(rp));
          const uint4 u1 = __ldg(reinterpret_cast<const uint4*>(rp) + 1);
          const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float2 f = unpack_bf16x2(w[i]);
            v[2 * i] += f.x;
            v[2 * i + 1] += f.y;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (i < nv) v[i] += __bfloat162float(rp[i]);
        }
      }
      if (p.relu) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
      }
      const size_t yo = static_cast<size_t>(m) * p.y_cstride + p.y_coff + n;
      if (p.y_f32) {
        float* yp = reinterpret_cast<float*>(p.y) + yo;
        if (nv == 16 && ((reinterpret_cast<uintptr_t>(yp) & 15) == 0)) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            reinterpret_cast<float4*>(yp)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        } else {
          for (int i = 0; i < nv; ++i) yp[i] = v[i];
        }
      } else {
        __nv_bfloat16* yp = reinterpret_cast<__nv_bfloat16*>(p.y) + yo;
        if (nv == 16 && ((reinterpret_cast<uintptr_t>(yp) & 15) == 0)) {
          uint4 o0, o1;
          o0.x = pack_bf16x2(v[0], v[1]);
          o0.y = pack_bf16x2(v[2], v[3]);
          o0.z = pack_bf16x2(v[4], v[5]);
          o0.w = pack_bf16x2(v[6], v[7]);
          o1.x = pack_bf16x2(v[8], v[9]);
          o1.y = pack_bf16x2(v[10], v[11]);
          o1.z = pack_bf16x2(v[12], v[13]);
          o1.w = pack_bf16x2(v[14], v[15]);
          reinterpret_cast<uint4*>(yp)[0] = o0;
          reinterpret_cast<uint4*>(yp)[1] = o1;
        } else {
          for (int i = 0; i < nv; ++i) yp[i] = __float2bfloat16_rn(v[i]);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, p.tmem_cols);
}

// ------------------------------------------------------------------ host side

namespace {

int g_driver_version = -1;

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

template <int AMODE, int BK>
int launch_conv(const CUtensorMap& tmA, const CUtensorMap& tmB, const ConvKParams& p, int m_tiles, int n_tiles,
                size_t smem, cudaStream_t stream) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(conv_tc_kernel<AMODE, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    227 * 1024);
  });
  if (attr_err != cudaSuccess) return cuda_status(attr_err, "cudaFuncSetAttribute(conv)");
  conv_tc_kernel<AMODE, BK><<<dim3(n_tiles, m_tiles), NUM_THREADS, smem, stream>>>(tmA, tmB, p);
  count_launch();
  return cuda_status(cudaGetLastError(), "conv_tc_kernel launch");
}

int pick_bk(int cin_eff) { return cin_eff <= 16 ? 16 : 64; }

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

  ConvKParams p{};
  p.M = d->N * d->Ho * d->Wo;
  p.cout = d->cout;
  const int n_tiles = (d->cout + 255) / 256;
  p.block_n = (((d->cout + n_tiles - 1) / n_tiles) + 15) / 16 * 16;
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
  uint32_t tc = 32;
  while (tc < static_cast<uint32_t>(p.block_n)) tc <<= 1;
  p.tmem_cols = tc;
  p.x = reinterpret_cast<const uint16_t*>(d->x);
  p.x_cstride = d->x_cstride;
  p.x_coff = d->x_coff;
  p.gidx = d->gather_idx;
  p.n_gather = gather ? d->cin : 0;
  p.bias = d->bias;
  p.res = reinterpret_cast<const __nv_bfloat16*>(d->residual);
  p.res_cstride = d->res_cstride;
  p.res_coff = d->res_coff;
  p.relu = d->relu;
  p.y = d->y;
  p.y_cstride = d->y_cstride;
  p.y_coff = d->y_coff;
  p.y_f32 = d->y_dtype == UB_F32;

  const uint32_t a_bytes = BLOCK_M * bk * 2;
  const uint32_t b_stride = (static_cast<uint32_t>(p.block_n) * bk * 2 + 1023u) & ~1023u;
  const uint32_t stage_bytes = a_bytes + b_stride;
  const uint32_t budget = 110u * 1024u;  // two CTAs per SM
  int stages = static_cast<int>(budget / stage_bytes);
  stages = stages < 2 ? 2 : (stages > 8 ? 8 : stages);
  if (stages > p.num_kb && p.num_kb >= 1) stages = p.num_kb < 2 ? 2 : p.num_kb;
  p.stages = stages;
  const size_t smem = 1024 + static_cast<size_t>(stages) * stage_bytes + (2 * stages + 1) * 8 + 16;

  auto enc_tiled = encode_tiled_fn();
  auto enc_im2col = encode_im2col_fn();
  if (!enc_tiled || !enc_im2col) return fail(UB_ECUDA, "ub_conv_fwd: cannot resolve cuTensorMapEncode* entry points");
  const CUtensorMapSwizzle swz = swizzle_of(bk * 2);

  CUtensorMap tmA{}, tmB{};
  // B: weights [cout][K_total] bf16, K-major.
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(K_total), static_cast<cuuint64_t>(d->cout)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(K_total) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(bk), static_cast<cuuint32_t>(p.block_n)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc_tiled(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(d->w), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_fwd: encode B tensor map failed (%d)", (int)r);
    apply_small_tensor_quirk(&tmB, static_cast<size_t>(K_total) * d->cout * 2);
  }
  const uint16_t* xbase = reinterpret_cast<const uint16_t*>(d->x) + (d->x_coff - lead);
  const size_t x_footprint = static_cast<size_t>(d->N) * d->H * d->W * d->x_cstride * 2;
  int amode;
  if (gather) {
    amode = A_GATHER;
    tmA = tmB;  // unused by the kernel in gather mode
  } else if (pointwise) {
    amode = A_TILED;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cin_eff), static_cast<cuuint64_t>(p.M)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(d->x_cstride) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(bk), BLOCK_M};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc_tiled(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(xbase), dims, strides,
                           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_fwd: encode A (tiled) tensor map failed (%d)", (int)r);
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
    CUresult r = enc_im2col(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(xbase), dims, strides,
                            lower, upper, static_cast<cuuint32_t>(bk), BLOCK_M, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_fwd: encode A (im2col) tensor map failed (%d)", (int)r);
    apply_small_tensor_quirk(&tmA, x_footprint);
  }

  const int m_tiles = (p.M + BLOCK_M - 1) / BLOCK_M;
  if (m_tiles > 65535) return fail(UB_EUNSUPPORTED, "ub_conv_fwd: too many M tiles (%d)", m_tiles);
  if (amode == A_GATHER) return launch_conv<A_GATHER, 64>(tmA, tmB, p, m_tiles, n_tiles, smem, stream);
  if (amode == A_TILED)
    return bk == 64 ? launch_conv<A_TILED, 64>(tmA, tmB, p, m_tiles, n_tiles, smem, stream)
                    : launch_conv<A_TILED, 16>(tmA, tmB, p, m_tiles, n_tiles, smem, stream);
  return bk == 64 ? launch_conv<A_IM2COL, 64>(tmA, tmB, p, m_tiles, n_tiles, smem, stream)
                  : launch_conv<A_IM2COL, 16>(tmA, tmB, p, m_tiles, n_tiles, smem, stream);
}

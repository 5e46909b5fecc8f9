// Space-to-depth stem: the stride-2 k x k first conv of the network as a
// stride-1 ceil(k/2)^2 conv over a 2x2-folded input, on tcgen05 tensor cores.
//
// The first CHANNEL_MIX node (interp.py:57-63) reads the model input through
// the INPUT node's GATHER (planner.py:774-783 keeps e.g. 2 of 3 image
// channels).  With 4 * cin <= 8, one folded pixel
//     S[n][Y][X][(py*2 + px)*cin + c] = x[n][idx[c]][2Y+py-pad][2X+px-pad]
// is exactly 16 bytes of bf16, and output (ho, wo) reads S[ho+dy][wo+dx] for
// dy, dx < kq = ceil(k/2) with weights W'[o][dy][dx][(py,px,c)] =
// W[o][c][2dy+py][2dx+px] (0 past the filter).
//
// Flatten S as rows R = (n*Hs + Y)*Ws + X.  A tile is 128 consecutive X of one
// output row (n, Y): its A operand for tap (dy, dx) is S[R0 + dy*Ws + dx ...],
// 128 consecutive 16-byte rows -- a no-swizzle K-major UMMA operand (8x16-byte
// core matrices, SBO = 128 B) pointed at directly in shared memory.  One K=16
// MMA covers taps (dy, dx) and (dy, dx+1): the second K core matrix is the same
// rows shifted by one pixel (LBO = 16 B).  So a tile needs ONE contiguous bulk
// copy and kq*ceil(kq/2) MMAs -- no im2col, no per-element address math.
// Columns X >= Wo are computed and dropped by the TMA store's bounds clipping.
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      bulk-copy producer (cp.async.bulk global -> shared, mbarrier tx)
//   warp 1      MMA issuer (4 TMEM accumulators, descriptors precomputed)
//   warp 2      TMEM allocator
//   warps 4-19  epilogue, four groups of four (group g drains accumulator g):
//               TMEM -> regs, +bias, ReLU, bf16 -> SW128 smem -> one TMA store per
//               64 channels (box 64 ch x 128 pixels of the output row)
#include <cstdlib>

#include "ub_common.cuh"
#include "ub_host.h"

#include "upscale_b200.h"

namespace ub {
namespace {

constexpr int S2D_STAGES = 6;
constexpr int S2D_ACC = 4;
constexpr int S2D_EPI_GROUPS = S2D_ACC;  // group g drains accumulator g (tiles it % 4 == g)
constexpr int S2D_EPI_WARPS = 4 * S2D_EPI_GROUPS;
constexpr int S2D_THREADS = 128 + 32 * S2D_EPI_WARPS;
constexpr int S2D_TILE_X = 128;       // output pixels per tile (one MMA M)
constexpr int S2D_BOX_BYTES = 16384;  // 64 channels x 128 pixels of bf16

struct S2DParams {
  const uint16_t* s;  // folded input, 8 bf16 per row
  int tiles, xblocks;
  int Hs, Ws, Ho, Wo;
  int np, cout, acc_cols, boxes;
  uint32_t load_bytes, stage_bytes;
  const uint16_t* w;  // bf16 [cout][kq*kq*8]
  const float* bias;
  int relu;
  int dbg;  // profiling ablations (UB_DEBUG_FLAGS): 1 no stores, 4 no MMA, 16 no loads,
            // 32 no TMEM reads, 64 no proxy fence, 128 no group barriers
};

UB_DEVI void spin_wait(uint64_t* bar, uint32_t parity, int dbg) {
  if (dbg & 512) {
    const uint32_t a = smem_u32(bar);
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(a), "r"(parity)
          : "memory");
    }
  } else {
    mbar_wait(bar, parity);
  }
}

template <int KQ>
__global__ void __launch_bounds__(S2D_THREADS, 1)
    stem_s2d_kernel(const __grid_constant__ CUtensorMap tmY, const S2DParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int PAIRS = (KQ + 1) / 2, NMMA = KQ * PAIRS;
  const int b_bytes = (NMMA * 2 * p.np * 16 + 1023) & ~1023;
  uint8_t* sB = base;
  uint8_t* sOut = sB + b_bytes;  // [group][box] 16 KB each, 1024-aligned
  uint8_t* sA = sOut + S2D_EPI_GROUPS * p.boxes * S2D_BOX_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sA + S2D_STAGES * p.stage_bytes);
  uint64_t* empty = full + S2D_STAGES;
  uint64_t* tfull = empty + S2D_STAGES;
  uint64_t* tempty = tfull + S2D_ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + S2D_ACC);
  float* sBias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 256);  // 16-byte aligned

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmY);
    for (int s = 0; s < S2D_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < S2D_ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // the four warps of the group that drains it
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, S2D_ACC * p.acc_cols);
  // B operand: MMA j = (dy, pair pj) owns two K core-matrix columns h = 0, 1 (taps dx = 2pj + h),
  // each [np rows][16 bytes]; smem offset ((j*2 + h)*np + n)*16.
  if (KQ == 4 && (p.dbg & 8192)) {
    for (int i = threadIdx.x; i < 2 * p.np * 8; i += blockDim.x) {
      const int c = i & 7, n = (i >> 3) % p.np, q = (i >> 3) / p.np;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (n < p.cout) v = *reinterpret_cast<const uint4*>(p.w + static_cast<size_t>(n) * 128 + q * 64 + c * 8);
      *reinterpret_cast<uint4*>(sB + q * p.np * 128 + n * 128 + ((c ^ (n & 7)) << 4)) = v;
    }
  } else
  for (int i = threadIdx.x; i < NMMA * 2 * p.np; i += blockDim.x) {
    const int n = i % p.np;
    const int jh = i / p.np;
    const int j = jh >> 1, h = jh & 1;
    const int dy = j / PAIRS;
    const int dx = (j - dy * PAIRS) * 2 + h;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (n < p.cout && dx < KQ)
      v = *reinterpret_cast<const uint4*>(p.w + static_cast<size_t>(n) * (KQ * KQ * 8) + (dy * KQ + dx) * 8);
    *reinterpret_cast<uint4*>(sB + static_cast<size_t>(i) * 16) = v;
  }
  for (int i = threadIdx.x; i < p.np; i += blockDim.x) sBias[i] = (p.bias && i < p.cout) ? p.bias[i] : 0.f;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ================= producer: one contiguous block of S per tile
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        const int row = t / p.xblocks;  // n*Ho + Y
        const int xb = t - row * p.xblocks;
        const int n = row / p.Ho, Y = row - (row / p.Ho) * p.Ho;
        const size_t R0 = (static_cast<size_t>(n) * p.Hs + Y) * p.Ws + xb * S2D_TILE_X;
        spin_wait(&empty[s], ph ^ 1, p.dbg);
        if (p.dbg & 16) {
          mbar_arrive(&full[s]);
        } else {
          mbar_arrive_expect_tx(&full[s], p.load_bytes);
          bulk_load(sA + s * p.stage_bytes, p.s + R0 * 8, p.load_bytes, &full[s]);
        }
        if (++s == S2D_STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {  // ================= MMA issuer
    // The whole warp runs the loop (descriptors stay warp-uniform); lane 0 issues.
    const uint32_t idesc = make_idesc_bf16(128, static_cast<uint32_t>(p.np));
    const uint32_t b0 = smem_u32(sB);
    uint64_t bdesc[NMMA];
    uint32_t aoff[NMMA];  // descriptor start-address delta (16-byte units) of MMA j
#pragma unroll
    for (int j = 0; j < NMMA; ++j) {
      const int dy = j / PAIRS, dx = (j % PAIRS) * 2;
      aoff[j] = static_cast<uint32_t>(dy * p.Ws + dx);
      bdesc[j] = sdesc_plain(b0 + j * 2 * p.np * 16, p.np * 16, 128);
    }
    uint64_t adesc0 = sdesc_plain(smem_u32(sA), 16, 128);
    if (KQ == 4 && (p.dbg & 8192)) {
#pragma unroll
      for (int j = 0; j < NMMA; ++j) {
        const int dy = j / PAIRS, pr = j % PAIRS;
        bdesc[j] = make_sdesc(b0 + (dy >> 1) * p.np * 128 + (dy & 1) * 64 + pr * 32, 1024, 2);
      }
    }
    if (p.dbg & 2048) {  // timing probe: aligned, non-overlapping K core matrices
      adesc0 = sdesc_plain(smem_u32(sA), 2048, 128);
#pragma unroll
      for (int j = 0; j < NMMA; ++j) aoff[j] = 0;
    }
    if (p.dbg & 4096) {  // timing probe: SWIZZLE_128B A (garbage data; stages 1024-aligned)
      adesc0 = make_sdesc(smem_u32(sA), 1024, 2);
#pragma unroll
      for (int j = 0; j < NMMA; ++j) aoff[j] = (j & 3) * 2 + (j >> 2) * 1024;
    }
    const uint32_t stage_units = p.stage_bytes >> 4;
    int s = 0, a = 0;
    uint32_t sph = 0, aph = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x) {
      spin_wait(&tempty[a], aph ^ 1, p.dbg);
      spin_wait(&full[s], sph, p.dbg);
      tc_fence_after();
      const uint64_t ad = adesc0 + s * stage_units;
      const uint32_t d = tmem_base + a * p.acc_cols;
      __syncwarp();
      if (!(p.dbg & 4)) {
#pragma unroll
        for (int j = 0; j < NMMA; ++j) umma_bf16_warp(d, ad + aoff[j], bdesc[j], idesc, j > 0 ? 1u : 0u);
      }
      umma_commit_warp(&empty[s]);
      umma_commit_warp(&tfull[a]);
      if (++s == S2D_STAGES) {
        s = 0;
        sph ^= 1;
      }
      if (++a == S2D_ACC) {
        a = 0;
        aph ^= 1;
      }
    }
  } else if (warp >= 4) {  // ================= epilogue
    const int grp = (warp - 4) >> 2;  // == the accumulator this group drains
    const int quad = warp & 3;        // TMEM lanes / tile rows 32*quad .. +31
    const int r = quad * 32 + lane;   // this thread's row (output pixel X0 + r)
    const bool leader = quad == 0 && lane == 0;
    uint8_t* out = sOut + grp * p.boxes * S2D_BOX_BYTES;
    const int nchunks = p.np >> 4;
    const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + grp * p.acc_cols;
    uint32_t aph = 0;
    int it = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++it) {
      if ((it % S2D_EPI_GROUPS) != grp) continue;
      spin_wait(&tfull[grp], aph, p.dbg);
      aph ^= 1;
      tc_fence_after();
      if (!(p.dbg & 128)) {
        if (leader) bulk_wait_read<0>();  // this group's previous store has left shared memory
        named_bar_sync(1 + grp, 128);
      }
      for (int c = 0; c < nchunks; c += 2) {  // 32 columns per TMEM round trip
        const bool two = c + 1 < nchunks;
        uint32_t v[32];
        if (p.dbg & 32) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = i * lane;
        } else {
          tmem_ld16(taddr + c * 16, *reinterpret_cast<uint32_t(*)[16]>(&v[0]));
          if (two) tmem_ld16(taddr + c * 16 + 16, *reinterpret_cast<uint32_t(*)[16]>(&v[16]));
          tmem_ld_wait();
        }
        if (c + 2 >= nchunks) {  // accumulator drained: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[grp]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !two) break;
          const int cc = c + h;  // 16-column chunk: 16-byte pieces 2cc%8, 2cc%8+1 of box cc/4
          const float4* bq = reinterpret_cast<const float4*>(sBias + cc * 16);
          uint32_t o[8];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 b4 = bq[i];
            const float2 lo = add_f32x2(
                make_float2(__uint_as_float(v[h * 16 + 4 * i]), __uint_as_float(v[h * 16 + 4 * i + 1])),
                make_float2(b4.x, b4.y));
            const float2 hi = add_f32x2(
                make_float2(__uint_as_float(v[h * 16 + 4 * i + 2]), __uint_as_float(v[h * 16 + 4 * i + 3])),
                make_float2(b4.z, b4.w));
            o[2 * i] = p.relu ? cvt_relu_bf16x2(lo.x, lo.y) : cvt_bf16x2(lo.x, lo.y);
            o[2 * i + 1] = p.relu ? cvt_relu_bf16x2(hi.x, hi.y) : cvt_bf16x2(hi.x, hi.y);
          }
          uint8_t* rowp = out + (cc >> 2) * S2D_BOX_BYTES + r * 128;
          const int j0 = (cc & 3) * 2;
          *reinterpret_cast<uint4*>(rowp + ((j0 ^ (r & 7)) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
          *reinterpret_cast<uint4*>(rowp + (((j0 + 1) ^ (r & 7)) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
        }
      }
      if (!(p.dbg & 64)) fence_proxy_async_smem();  // st.shared -> TMA (async proxy) reads
      if (!(p.dbg & 128)) named_bar_sync(1 + grp, 128);
      if (leader && !(p.dbg & 1)) {
        const int row = t / p.xblocks;
        const int xb = t - row * p.xblocks;
        const int n = row / p.Ho, Y = row - (row / p.Ho) * p.Ho;
        for (int b = 0; b < p.boxes; ++b) tma_store_4d(&tmY, out + b * S2D_BOX_BYTES, b * 64, xb * S2D_TILE_X, Y, n);
        bulk_commit();
      }
    }
    if (leader) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, S2D_ACC * p.acc_cols);
  }
}

// ------------------------------------------------------------- packing
// grid (ceil(Hs*Ws / block), N): one thread per folded pixel; the tail rows past N*Hs*Ws
// stay as allocated (zero).  Lanes take consecutive X, so each fp32 load of a warp covers
// 256 contiguous bytes of one input row.
__global__ void stem_s2d_pack_kernel(const float* __restrict__ x, int C, int H, int W, const int32_t* __restrict__ idx,
                                     int cin, int pad, int Hs, int Ws, uint4* __restrict__ s) {
  const int rem = blockIdx.x * blockDim.x + threadIdx.x;
  if (rem >= Hs * Ws) return;
  const int n = blockIdx.y;
  const int Y = rem / Ws;
  const int X = rem - Y * Ws;
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int hi = 2 * Y + (q >> 1) - pad;
    const int wi = 2 * X + (q & 1) - pad;
    const bool in = hi >= 0 && hi < H && wi >= 0 && wi < W;
#pragma unroll 2
    for (int c = 0; c < cin; ++c) {
      const int slot = q * cin + c;
      float f = 0.f;
      if (in) f = __ldg(x + ((static_cast<size_t>(n) * C + __ldg(idx + c)) * H + hi) * W + wi);
      const uint32_t b = __bfloat16_as_ushort(__float2bfloat16_rn(f));
      w[slot >> 1] |= b << (16 * (slot & 1));
    }
  }
  s[static_cast<size_t>(n) * Hs * Ws + rem] = make_uint4(w[0], w[1], w[2], w[3]);
}

// Row-staged pack: one CTA per PACK_YB folded rows (n, Y .. Y + PACK_YB - 1).  The 2 * CIN
// input rows of each are loaded with coalesced float4 loads into shared memory (zero margins of
// `off` columns on the left and up to `sw` on the right stand in for the padding); then each
// thread assembles folded pixels from shared memory.  Thread -> (row, float4 column) and
// (row, pixel) maps are shifts, not divisions.  Needs W % 4 == 0 (16-byte row alignment).
constexpr int PACK_YB = 4, PACK_THREADS = 256;

template <int CIN>
__global__ void __launch_bounds__(PACK_THREADS) stem_s2d_pack_rows_kernel(
    const float* __restrict__ x, int C, int H, int W, const int32_t* __restrict__ idx, int pad, int Hs, int Ws,
    int off, int sw, uint4* __restrict__ s) {
  constexpr int NROWS = PACK_YB * 2 * CIN;  // staged rows: [yb][py][c]
  extern __shared__ float4 srow4[];
  const float* srow = reinterpret_cast<const float*>(srow4);
  const int Y0 = blockIdx.x * PACK_YB, n = blockIdx.y;
  const int w4 = W >> 2, sw4 = sw >> 2, off4 = off >> 2;
  int ch[CIN];
#pragma unroll
  for (int c = 0; c < CIN; ++c) ch[c] = __ldg(idx + c);
  // load: 64 threads per staged row, PACK_THREADS / 64 rows per pass
  {
    const int j0 = threadIdx.x & 63;
#pragma unroll
    for (int r0 = 0; r0 < NROWS; r0 += PACK_THREADS / 64) {
      const int rr = r0 + (threadIdx.x >> 6);
      const int yb = rr / (2 * CIN), py = (rr / CIN) & 1, c = rr % CIN;  // compile-time divisors
      const int hi = 2 * (Y0 + yb) + py - pad;
      const bool row_ok = Y0 + yb < Hs && hi >= 0 && hi < H;
      const float4* src = reinterpret_cast<const float4*>(x + ((static_cast<size_t>(n) * C + ch[c]) * H + hi) * W);
      for (int j = j0; j < sw4; j += 64) {
        const int i4 = j - off4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row_ok && i4 >= 0 && i4 < w4) v = __ldg(src + i4);
        srow4[rr * sw4 + j] = v;
      }
    }
  }
  __syncthreads();
  // assemble: 128 threads per folded row
  for (int yb = threadIdx.x >> 7; yb < PACK_YB; yb += PACK_THREADS / 128) {
    if (Y0 + yb >= Hs) break;
    const float* rows = srow + yb * 2 * CIN * sw;
    uint4* dst = s + (static_cast<size_t>(n) * Hs + Y0 + yb) * Ws;
    for (int X = threadIdx.x & 127; X < Ws; X += 128) {
      const int col = 2 * X - pad + off;  // in [0, sw - 1) by construction of off / sw
      float f[8];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < CIN; ++c) f[q * CIN + c] = rows[((q >> 1) * CIN + c) * sw + col + (q & 1)];
#pragma unroll
      for (int i = 4 * CIN; i < 8; ++i) f[i] = 0.f;
      dst[X] = make_uint4(cvt_bf16x2(f[0], f[1]), cvt_bf16x2(f[2], f[3]), cvt_bf16x2(f[4], f[5]),
                          cvt_bf16x2(f[6], f[7]));
    }
  }
}

template <int KQ>
void launch_s2d(const CUtensorMap& tm, const S2DParams& p, int grid, size_t smem, cudaStream_t stream) {
  (void)ensure_max_smem(stem_s2d_kernel<KQ>);
  stem_s2d_kernel<KQ><<<grid, S2D_THREADS, smem, stream>>>(tm, p);
}

struct S2DGeom {
  int Ho, Wo, kq, pairs, Hs, Ws, xblocks;
  long long rows_alloc;
  uint32_t load_rows;
};

int s2d_geometry(int N, int H, int W, int k, int pad, S2DGeom* g) {
  if (N < 1 || H < 1 || W < 1 || k < 2 || pad < 0) return fail(UB_EINVAL, "stem_s2d: bad geometry");
  g->Ho = (H + 2 * pad - k) / 2 + 1;
  g->Wo = (W + 2 * pad - k) / 2 + 1;
  if (g->Ho < 1 || g->Wo < 1) return fail(UB_EINVAL, "stem_s2d: empty output");
  g->kq = (k + 1) / 2;
  g->pairs = (g->kq + 1) / 2;
  g->Hs = g->Ho + g->kq - 1;
  g->Ws = g->Wo + g->kq - 1;
  g->xblocks = (g->Wo + S2D_TILE_X - 1) / S2D_TILE_X;
  g->load_rows = S2D_TILE_X + static_cast<uint32_t>((g->kq - 1) * g->Ws + 2 * g->pairs - 1);
  // the last tile's block of rows ends here (S rows past N*Hs*Ws are zero padding)
  const long long last_r0 = (static_cast<long long>(N - 1) * g->Hs + g->Ho - 1) * g->Ws +
                            static_cast<long long>(g->xblocks - 1) * S2D_TILE_X;
  const long long need = last_r0 + g->load_rows;
  const long long rows = static_cast<long long>(N) * g->Hs * g->Ws;
  g->rows_alloc = need > rows ? need : rows;
  return UB_OK;
}

}  // namespace
}  // namespace ub

using namespace ub;

extern "C" int ub_stem_s2d_geometry(int N, int H, int W, int k, int pad, int* Hs, int* Ws, long long* bytes) {
  S2DGeom g;
  const int rc = s2d_geometry(N, H, W, k, pad, &g);
  if (rc) return rc;
  if (Hs) *Hs = g.Hs;
  if (Ws) *Ws = g.Ws;
  if (bytes) *bytes = g.rows_alloc * 16;
  return UB_OK;
}

extern "C" int ub_stem_s2d_pack(const float* x, int N, int C, int H, int W, const int32_t* idx, int cin, int k,
                                int pad, void* s, cudaStream_t stream) {
  if (!x || !idx || !s || cin < 1 || C < 1) return fail(UB_EINVAL, "ub_stem_s2d_pack: bad arguments");
  if (4 * cin > 8) return fail(UB_EUNSUPPORTED, "ub_stem_s2d_pack: 4*cin = %d > 8", 4 * cin);
  S2DGeom g;
  const int rc = s2d_geometry(N, H, W, k, pad, &g);
  if (rc) return rc;
  if (W % 4 == 0 && !(reinterpret_cast<uintptr_t>(x) & 15) && g.Hs <= 65535 && N <= 65535) {
    const int off = (pad + 3) & ~3;                       // left zero margin (>= pad, float4-aligned)
    const int right = 2 * g.Ws + 1 - pad;                 // one past the last column read
    const int sw = off + ((right > W ? right : W) + 3) / 4 * 4;
    const size_t smem = static_cast<size_t>(PACK_YB) * 2 * cin * sw * sizeof(float);
    if (smem <= 48 * 1024) {
      const dim3 grid((g.Hs + PACK_YB - 1) / PACK_YB, N);
      if (cin == 1)
        stem_s2d_pack_rows_kernel<1><<<grid, PACK_THREADS, smem, stream>>>(x, C, H, W, idx, pad, g.Hs, g.Ws, off, sw,
                                                                           static_cast<uint4*>(s));
      else
        stem_s2d_pack_rows_kernel<2><<<grid, PACK_THREADS, smem, stream>>>(x, C, H, W, idx, pad, g.Hs, g.Ws, off, sw,
                                                                           static_cast<uint4*>(s));
      count_launch();
      return cuda_status(cudaGetLastError(), "stem_s2d_pack_rows_kernel");
    }
  }
  const int block = 256;
  const dim3 grid((g.Hs * g.Ws + block - 1) / block, N);
  stem_s2d_pack_kernel<<<grid, block, 0, stream>>>(x, C, H, W, idx, cin, pad, g.Hs, g.Ws, static_cast<uint4*>(s));
  count_launch();
  return cuda_status(cudaGetLastError(), "stem_s2d_pack_kernel");
}

extern "C" int ub_conv_s2d(const void* s, int N, int H, int W, int k, int pad, const void* w, int cout,
                           const float* bias, int relu, void* y, int y_cstride, int y_coff, cudaStream_t stream) {
  if (!s || !w || !y || cout < 1) return fail(UB_EINVAL, "ub_conv_s2d: bad arguments");
  if (cout > 128) return fail(UB_EUNSUPPORTED, "ub_conv_s2d: cout %d > 128", cout);
  if ((y_cstride & 7) || (y_coff & 7) || y_coff + cout > y_cstride)
    return fail(UB_EUNSUPPORTED, "ub_conv_s2d: output window (cout %d, cstride %d, coff %d) not 16-byte aligned",
                cout, y_cstride, y_coff);
  S2DGeom g;
  int rc = s2d_geometry(N, H, W, k, pad, &g);
  if (rc) return rc;
  if (g.kq < 2 || g.kq > 4) return fail(UB_EUNSUPPORTED, "ub_conv_s2d: kernel %d (ceil(k/2) must be 2..4)", k);
  const long long tiles = static_cast<long long>(N) * g.Ho * g.xblocks;
  if (tiles >= (1ll << 31)) return fail(UB_EUNSUPPORTED, "ub_conv_s2d: %lld tiles", tiles);
  S2DParams p{};
  p.s = static_cast<const uint16_t*>(s);
  p.tiles = static_cast<int>(tiles);
  p.xblocks = g.xblocks;
  p.Hs = g.Hs;
  p.Ws = g.Ws;
  p.Ho = g.Ho;
  p.Wo = g.Wo;
  p.np = (cout + 15) / 16 * 16;
  p.cout = cout;
  p.acc_cols = p.np <= 32 ? 32 : (p.np <= 64 ? 64 : 128);
  p.boxes = (p.np + 63) / 64;
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* e = getenv("UB_DEBUG_FLAGS");
      dbg = e ? atoi(e) : 0;
    }
    p.dbg = dbg;
  }
  p.load_bytes = g.load_rows * 16;
  p.stage_bytes = (p.load_bytes + 127) & ~127u;
  if (p.dbg & 4096) p.stage_bytes = (p.load_bytes + 1023) & ~1023u;
  p.w = static_cast<const uint16_t*>(w);
  p.bias = bias;
  p.relu = relu;
  const int pairs = (g.kq + 1) / 2;
  const int b_bytes = (g.kq * pairs * 2 * p.np * 16 + 1023) & ~1023;
  size_t smem = 1024 + b_bytes + static_cast<size_t>(S2D_EPI_GROUPS) * p.boxes * S2D_BOX_BYTES +
                      S2D_STAGES * p.stage_bytes + 256 + 128 * sizeof(float);
  if (p.dbg & 4096) smem += 32768;
  if (smem > 227 * 1024) return fail(UB_EUNSUPPORTED, "ub_conv_s2d: %zu bytes of shared memory", smem);

  if (!encode_tiled_fn()) return fail(UB_ECUDA, "ub_conv_s2d: cannot resolve cuTensorMapEncodeTiled");
  // output y[n][Y][X][c] at y + y_coff: dims (cout, Wo, Ho, N); box 64 channels x 128 pixels
  CUtensorMap tm{};
  const cuuint64_t cs = static_cast<cuuint64_t>(y_cstride) * 2;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(cout), static_cast<cuuint64_t>(g.Wo), static_cast<cuuint64_t>(g.Ho),
                        static_cast<cuuint64_t>(N)};
  cuuint64_t strides[3] = {cs, cs * g.Wo, cs * g.Wo * g.Ho};
  cuuint32_t box[4] = {64, S2D_TILE_X, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = encode_tiled_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, static_cast<uint16_t*>(y) + y_coff, dims,
                                 strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_s2d: encode output tensor map failed (%d)", (int)r);
  apply_small_tensor_quirk(&tm, static_cast<size_t>(N) * g.Ho * g.Wo * y_cstride * 2);

  const int grid = p.tiles < num_sms() ? p.tiles : num_sms();
  switch (g.kq) {
    case 2: launch_s2d<2>(tm, p, grid, smem, stream); break;
    case 3: launch_s2d<3>(tm, p, grid, smem, stream); break;
    default: launch_s2d<4>(tm, p, grid, smem, stream); break;
  }
  count_launch();
  return cuda_status(cudaGetLastError(), "stem_s2d_kernel");
}

// Halo-tile implicit GEMM for stride-1 3x3 convolutions on tcgen05 tensor cores.
//
// The im2col operand of a 3x3 conv re-reads every input pixel 9 times; streamed from L2 by
// cp.async that is the bound of the generic kernel (conv_tc.cu) for the bottleneck convs.
// Here a tile is R whole output rows of one image, and its input -- the R + 2 rows of the
// window, each laid out over a padded width Wp (a power of two >= W + 2, zeros outside the
// image) -- is staged ONCE in shared memory as channel planes:
//     plane p (channels 8p .. 8p+7) = [position q][8 bf16], q = row * Wp + col.
// Output position r = j * Wp + x (tile row j) reads input position r + dy * Wp + dx for tap
// (dy, dx), so the A operand of a tap is the plane block shifted by dy * Wp + dx: 128
// consecutive 16-byte rows -- a no-swizzle K-major UMMA operand (8-row core matrices,
// SBO = 128 B) whose two K halves are consecutive planes (LBO = plane stride).  Every tap's
// MMAs read the same staged block; nothing is copied per tap.  Positions with x >= W (or
// rows past H) are computed and dropped by the output TMA store's bounds clipping.
//
// Padded width: Wp >= W + 1 suffices -- column 0 of every staged row is zero and serves as the
// right pad of the previous row.  Small images (H + 1) * Wp <= 64 are stacked, ipt per tile,
// one zero row between them, so a 7x7 map fills 98 of the 128 MMA rows instead of 49.
//
// Weights (SWIZZLE_128B, one 128-byte row per output channel, tap and 64-channel group): for
// cpad <= 64 all taps stay resident, loaded once per CTA; for cpad > 64 the input is staged per
// 64-channel group and the (group, tap) weight blocks stream through a TMA ring (SB = true).
//
// Persistent, warp-specialised, one CTA per SM:
//   warps 0-11  epilogue, three groups of four (whole tiles round-robin, or each tile's 64-column
//               chunks dealt to all groups): TMEM -> regs, +bias, ReLU, bf16 -> SW128 smem ->
//               4-D TMA store (box 64 channels x BX pixels x BY rows of the output)
//   warp 12     MMA issuer (2-4 TMEM accumulators; one elected lane issues)
//   warp 13     TMEM allocator; lane 0 then streams the weight blocks (SB)
//   warps 14-17 producers: halo planes by cp.async (zero-fill outside the image)
#include <cstdlib>

#include "ub_common.cuh"
#include "ub_host.h"

#include "upscale_b200.h"

namespace ub {
namespace {

constexpr int HALO_PRODUCERS = 128;
constexpr int HALO_EPI_WARPS = 12;                     // up to three groups of four, round-robin tiles
constexpr int HALO_PROD_WARP0 = HALO_EPI_WARPS + 2;    // after the MMA and TMEM-alloc warps
constexpr int HALO_THREADS = 32 * HALO_PROD_WARP0 + HALO_PRODUCERS;
constexpr int HALO_SLOT = 32 * 128;  // one epilogue warp's 32 rows x 64 channels bf16

struct HaloParams {
  const uint16_t* x;  // at channel (coff - lead)
  int x_cstride, N, H, W;  // input
  int Ho;                  // output rows per image (== H for stride 1)
  int R, Wp, wp_shift, n_pos, planes;
  uint32_t plane_stride, a_stage_bytes;
  int a_stages;
  int tiles, tiles_per_img;
  int cout, np, acc_cols, nacc, ngroups;
  int drainers;  // groups draining each tile: 1 (whole tiles round-robin) or ngroups (chunks dealt out)
  uint32_t b_block_bytes;  // np * 128: one tap's weights
  const uint16_t* w;       // [cout][9][cpad]
  int cpad;
  const float* bias;
  int relu;
  int bx;  // output box width (pixels); box height = 32 / bx rows
  int groups;    // 64-channel groups (1: all taps' weights resident; > 1: streamed per group x tap)
  int b_stages;  // streamed weight ring depth
  int kvalid;    // lead + cin: channels past it are not read (their weights are zero)
  uint32_t a_box_bytes;  // AT: bytes of one input box (one stacked image's box when ipt > 1)
  int ipt;       // images stacked per tile (small images): image i's row y at staged row 1 + i * (H + 1) + y
  long long* trace;  // profiling (UB_HALO_TRACE): CTA 0 event clocks, [tile][8]
  int epi4;          // (AT, resident weights) the TMEM-alloc warp issues the input boxes and the
                     // producer warps 14-17 form a fourth epilogue group
  int dbg;           // profiling ablations (UB_HALO_DBG): 1 no halo loads, 2 no output, 4 no TMEM reads,
                     // 8 no TMA store, 16 no slot wait (races; timing only)
};

// Compile-time halo geometry: padded width WP, rows per tile, staged positions, plane stride.
// Stride 2 runs as a stride-1 2x2 conv over the 2x2-folded input (see conv_halo3_kernel): one
// staged row fewer and no left pad column.
template <int WP, int MT, int S>
struct HaloGeom {
  static constexpr int R = 128 / WP;    // output rows per 128-position MMA tile
  static constexpr int RT = MT * R;     // output rows per staged tile (MT MMA tiles)
  static constexpr int N_POS = S == 1 ? ((RT + 2) * WP + 2 + 7) / 8 * 8 : ((RT + 1) * WP + 1 + 7) / 8 * 8;
  static constexpr uint32_t PLANE_STRIDE = N_POS * 16 + 16;  // odd # of 16-B units: planes on different banks
};

// SB: weights streamed per (64-channel group, tap) through a TMA ring (cpad > 64); else resident.
// S = 2: stride-2 3x3 conv as a 2x2 stride-1 conv over the input folded 2x2 with origin -1:
// folded pixel (Y, X) quadrant (py, px) = input (2Y + py - 1, 2X + px - 1), so output (y, x)
// reads folded (y + dy, x + dx), dy, dx < 2, with filter tap (ky, kx) = (2dy + py, 2dx + px)
// (taps past 2 do not exist: 9 of the 16 (quadrant, shift) pairs).  Groups = quadrant x 64
// input channels; the producer folds on the fly (a plane is 16 contiguous bytes of one input
// pixel), so no folded copy is ever written.
// AT: the input tile arrives by ONE 4-D TMA box per (tile, 64-channel group) -- positions
// [row][Wp] x KB bytes (= PLANES * 16) with the 128-/64-byte swizzle, zero-filled outside the
// image (negative coordinates; stride 2 through element strides 2 on W and H) -- and the tap
// shifts are whole rows of that swizzled block.  Otherwise 128 producer threads cp.async the
// 16-byte channel planes.
// XA: the epilogue applies a UB_ACT_* activation other than ReLU (EfficientNetV2's SiLU);
// a separate instantiation keeps the ReLU epilogue's code unchanged (as conv_tc's XACT).
template <int WP, int PLANES, int MT, bool SB, int S, bool AT, bool XA>
__global__ void __maxnreg__(96)
    conv_halo3_kernel(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmW,
                      const __grid_constant__ CUtensorMap tmX, const HaloParams p) {
  constexpr int KB = PLANES * 16;  // bytes of one staged position (AT)
  constexpr int TAPS = 9;
  using G = HaloGeom<WP, MT, S>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // weights: resident [tap][np rows][128 B] (one group) or a ring of (group, tap) blocks; SW128
  uint8_t* sB = base;
  const int groups = SB ? p.groups : 1;
  uint8_t* sE = sB + (SB ? p.b_stages : TAPS) * p.b_block_bytes;  // epilogue slots (1024-aligned)
  uint8_t* sA = sE + (p.epi4 ? 16 : HALO_EPI_WARPS) * HALO_SLOT;  // a_stages x a_stage_bytes
  float* sBias = reinterpret_cast<float*>(sA + p.a_stages * p.a_stage_bytes);  // 256 floats
  uint64_t* afull = reinterpret_cast<uint64_t*>(sBias + 256);
  uint64_t* aempty = afull + 8;
  uint64_t* tfull = aempty + 8;
  uint64_t* tempty = tfull + 4;
  uint64_t* bres = tempty + 4;
  uint64_t* bfull = bres + 1;
  uint64_t* bempty = bfull + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  constexpr int MMA_WARP = HALO_EPI_WARPS, ALLOC_WARP = HALO_EPI_WARPS + 1;
  if (warp == MMA_WARP && lane == 0) {
    for (int s = 0; s < p.a_stages; ++s) {
      mbar_init(&afull[s], AT ? 1 : HALO_PRODUCERS);
      mbar_init(&aempty[s], 1);
    }
    for (int a = 0; a < p.nacc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * p.drainers);  // every warp of the groups draining a tile
    }
    mbar_init(bres, HALO_PRODUCERS);
    for (int b = 0; b < p.b_stages; ++b) {
      mbar_init(&bfull[b], 1);
      mbar_init(&bempty[b], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) {
    tma_prefetch_desc(&tmY);
    if (SB) tma_prefetch_desc(&tmW);
    if (AT) tma_prefetch_desc(&tmX);
  }
  if (warp == ALLOC_WARP) tmem_alloc(tmem_slot, p.nacc * MT * p.acc_cols);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sBias[i] = (p.bias && i < p.cout) ? p.bias[i] : 0.f;
  if constexpr (AT) {
    // positions no box covers read as zero: the right pad of a tile's (or the last stacked
    // image's) last row wraps to the next row's column 0 (Wp = W + 1)
    uint4* a4 = reinterpret_cast<uint4*>(sA);
    for (int i = threadIdx.x; i < static_cast<int>(p.a_stages * p.a_stage_bytes / 16); i += blockDim.x)
      a4[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();

  // the input boxes of every (tile, group) of this CTA, in order, into the A ring (AT): issued by
  // producer thread 0, or by the TMEM-alloc warp's lane 0 when the producers drain (epi4)
  auto issue_input_boxes = [&]() {
    int s = 0;
    uint32_t ph = 0;
    const int ncb = p.cpad >> 6;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x)
      for (int g = 0; g < groups; ++g) {
        const int img = p.ipt > 1 ? t * p.ipt : t / p.tiles_per_img;
        int c0 = g * 64, ox = -1, oy = -1;  // box origin: channel, column, row (input coordinates)
        int img_rows = p.H + 1;             // staged rows per stacked image
        if constexpr (S == 2) {
          const int qd = g / ncb;
          c0 = (g - qd * ncb) * 64;
          ox = (qd & 1) - 1;
          oy = (qd >> 1) - 1;
          img_rows = p.Ho + 1;
        }
        mbar_wait(&aempty[s], ph ^ 1);
        uint8_t* dst = sA + s * p.a_stage_bytes;
        if (p.ipt > 1) {
          const int n_i = p.N - img < p.ipt ? p.N - img : p.ipt;
          mbar_arrive_expect_tx(&afull[s], n_i * p.a_box_bytes);
          for (int i = 0; i < n_i; ++i)
            tma_load_4d(&tmX, &afull[s], dst + i * img_rows * WP * KB, c0, ox, oy, img + i);
        } else {
          const int row0 = (t - img * p.tiles_per_img) * G::RT;  // first output row
          mbar_arrive_expect_tx(&afull[s], p.a_box_bytes);
          tma_load_4d(&tmX, &afull[s], dst, c0, ox, S * row0 + oy, img);
        }
        if (++s == p.a_stages) {
          s = 0;
          ph ^= 1;
        }
      }
  };
  if (warp >= HALO_PROD_WARP0) {
    // ================= producers
    const int pt = threadIdx.x - 32 * HALO_PROD_WARP0;
    // resident weights: tap t, row n, 16-byte chunk j (K = 8j .. 8j+7 of the tap) -> SW128
    const int cp8 = p.cpad >> 3;
    if constexpr (!SB)
    for (int e = pt; e < TAPS * p.np * cp8; e += HALO_PRODUCERS) {
      const int t = e / (p.np * cp8);
      const int rem = e - t * (p.np * cp8);
      const int n = rem / cp8, j = rem - (rem / cp8) * cp8;
      const bool ok = n < p.cout;
      const uint16_t* src = ok ? p.w + (static_cast<size_t>(n) * TAPS + t) * p.cpad + j * 8 : p.w;
      const uint32_t dst = smem_u32(sB + t * p.b_block_bytes + n * 128 + ((j ^ (n & 7)) << 4));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16u : 0u)
                   : "memory");
    }
    cp_async_arrive_noinc(bres);
    if (!p.epi4) griddep_wait();  // the input activations come from the previous kernel (PDL)
    if constexpr (AT) {
      if (pt == 0 && !p.epi4) issue_input_boxes();
    } else {
    // halo planes: this thread always fills plane pp of positions q0 + i * qstep
    const int pp = pt % PLANES;
    const int q0 = pt / PLANES;
    constexpr int qstep = HALO_PRODUCERS / PLANES;
    constexpr int wmask = WP - 1;
    constexpr int wp_shift = __builtin_ctz(WP);
    int s = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x)
    for (int g = 0; g < groups; ++g) {
      const int img = p.ipt > 1 ? t * p.ipt : t / p.tiles_per_img;
      const int y0 = p.ipt > 1 ? -1 : (t - img * p.tiles_per_img) * G::RT - 1;  // first staged input row (pad 1)
      const uint16_t* ximg = p.x + static_cast<size_t>(img) * p.H * p.W * p.x_cstride + g * 64 + pp * 8;
      if (p.dbg & 64) mbar_wait_sleep(&aempty[s], ph ^ 1, 2000);
      else mbar_wait(&aempty[s], ph ^ 1);
      if (p.trace && blockIdx.x == 0 && pt == 0) {
        const int itp = (t - blockIdx.x) / gridDim.x;
        if (itp < 64) p.trace[itp * 16 + 7] = clock64();
      }
      const uint32_t dst0 = smem_u32(sA + s * p.a_stage_bytes + pp * G::PLANE_STRIDE);
      if constexpr (S == 2) {
        const int ncb = p.cpad >> 6;
        const int qd = g / ncb, cb = g - qd * ncb;
        const int py = qd >> 1, px = qd & 1;
        const uint16_t* xq = p.x + static_cast<size_t>(img) * p.H * p.W * p.x_cstride + cb * 64 + pp * 8;
        const bool kin = cb * 64 + pp * 8 < p.kvalid;
        const int ybase = p.ipt > 1 ? 0 : (t - img * p.tiles_per_img) * G::RT;  // first folded row
        for (int q = q0; q < G::N_POS && !(p.dbg & 1); q += qstep) {
          int sr = ybase + (q >> wp_shift);
          int i = 0;
          if (p.ipt > 1) {  // stacked: image i's folded rows 0 .. Ho at stack rows i (Ho + 1) ..
            i = sr / (p.Ho + 1);
            sr -= i * (p.Ho + 1);
          }
          const int yy = 2 * sr + py - 1;
          const int xx = 2 * (q & wmask) + px - 1;
          const bool ok = kin && i < p.ipt && img + i < p.N && yy >= 0 && yy < p.H && xx >= 0 && xx < p.W;
          const uint16_t* src = ok ? xq + (static_cast<size_t>(i * p.H + yy) * p.W + xx) * p.x_cstride : p.x;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst0 + q * 16), "l"(src),
                       "r"(ok ? 16u : 0u)
                       : "memory");
        }
      } else {
      const bool kin = g * 64 + pp * 8 < p.kvalid;
      if (p.ipt > 1) {  // stacked images: stack row r -> image i = r / (H + 1), its row r - i (H + 1)
        for (int q = q0; q < G::N_POS && !(p.dbg & 1); q += qstep) {
          const int r = (q >> wp_shift) - 1;
          const int xx = (q & wmask) - 1;
          const int i = r / (p.H + 1);
          const int y = r - i * (p.H + 1);
          const bool ok = kin && r >= 0 && y < p.H && i < p.ipt && img + i < p.N && xx >= 0 && xx < p.W;
          const uint16_t* src = ok ? ximg + (static_cast<size_t>(i * p.H + y) * p.W + xx) * p.x_cstride : p.x;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst0 + q * 16), "l"(src),
                       "r"(ok ? 16u : 0u)
                       : "memory");
        }
      } else {
        for (int q = q0; q < G::N_POS && !(p.dbg & 1); q += qstep) {
          const int yy = y0 + (q >> wp_shift);
          const int xx = (q & wmask) - 1;
          const bool ok = kin && yy >= 0 && yy < p.H && xx >= 0 && xx < p.W;
          const uint16_t* src = ok ? ximg + (static_cast<size_t>(yy) * p.W + xx) * p.x_cstride : p.x;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst0 + q * 16), "l"(src),
                       "r"(ok ? 16u : 0u)
                       : "memory");
        }
      }
      }
      cp_async_arrive_noinc(&afull[s]);
      if (++s == p.a_stages) {
        s = 0;
        ph ^= 1;
      }
    }
    cp_async_wait<0>();
    }
  } else if (warp == MMA_WARP) {
    // ================= MMA issuer (whole warp; one elected lane issues)
    const uint32_t idesc = make_idesc_bf16(128, static_cast<uint32_t>(p.np));
    const uint32_t b0 = smem_u32(sB);
    const uint64_t bdesc0 = make_sdesc(b0, 1024, 2);
    const uint32_t b_units = p.b_block_bytes >> 4;
    const uint64_t adesc0 = AT ? make_sdesc(smem_u32(sA), 8 * KB, KB == 128 ? 2 : 4)
                               : sdesc_plain(smem_u32(sA), G::PLANE_STRIDE, 128);
    // A operand of MMA tile mt, tap shift (dy, dx), K step j (16-byte units)
    auto a_off = [&](int mt, int dy, int dx, int j) -> uint32_t {
      const int pos = mt * G::R * WP + dy * WP + dx;
      return AT ? static_cast<uint32_t>(pos * KB + 32 * j) >> 4
                : static_cast<uint32_t>(pos * 16 + 2 * j * G::PLANE_STRIDE) >> 4;
    };
    const uint32_t stage_units = p.a_stage_bytes >> 4;
    if (!SB) mbar_wait(bres, 0);
    __syncwarp();
    tc_fence_after();
    fence_proxy_async_smem();
    int s = 0, it = 0, bs = 0, acc = 0;
    uint32_t ph = 0, bph = 0, aph = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++it) {
      if (p.trace && blockIdx.x == 0 && lane == 0 && it < 64) p.trace[it * 16 + 0] = clock64();
      mbar_wait(&tempty[acc], aph ^ 1);
      if (p.trace && blockIdx.x == 0 && lane == 0 && it < 64) p.trace[it * 16 + 1] = clock64();
      for (int g = 0; g < groups; ++g) {
        mbar_wait(&afull[s], ph);
        if (p.trace && blockIdx.x == 0 && lane == 0 && it < 64 && g == 0) p.trace[it * 16 + 2] = clock64();
        __syncwarp();
        tc_fence_after();
        if constexpr (!AT) fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tensor-core reads
        const uint64_t ad = adesc0 + s * stage_units;
        if constexpr (S == 2) {
          const int qd = g / (p.cpad >> 6);
          const int py = qd >> 1, px = qd & 1;
          for (int dy = 0; dy < 2 - py; ++dy)
            for (int dx = 0; dx < 2 - px; ++dx) {
              mbar_wait(&bfull[bs], bph);
              __syncwarp();
              tc_fence_after();
              const uint64_t bd = bdesc0 + bs * b_units;
#pragma unroll
              for (int mt = 0; mt < MT; ++mt) {
                const uint32_t d = tmem_base + (acc * MT + mt) * p.acc_cols;
#pragma unroll
                for (int j = 0; j < PLANES / 2; ++j) {
                  umma_bf16_warp(d, ad + a_off(mt, dy, dx, j), bd + 2 * j, idesc, (g | dy | dx | j) ? 1u : 0u);
                }
              }
              umma_commit_warp(&bempty[bs]);
              if (++bs == p.b_stages) {
                bs = 0;
                bph ^= 1;
              }
            }
        } else
#pragma unroll
        for (int tap = 0; tap < TAPS; ++tap) {
          uint64_t bd;
          if constexpr (!SB) {
            bd = bdesc0 + tap * b_units;
          } else {  // this (group, tap)'s weight block from the ring
            mbar_wait(&bfull[bs], bph);
            __syncwarp();
            tc_fence_after();
            bd = bdesc0 + bs * b_units;
          }
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const uint32_t d = tmem_base + (acc * MT + mt) * p.acc_cols;
#pragma unroll
            for (int j = 0; j < PLANES / 2; ++j) {
              // A: planes 2j, 2j+1 of MMA tile mt shifted by tap (dy, dx); B: K step j of the tap
              umma_bf16_warp(d, ad + a_off(mt, tap / 3, tap % 3, j), bd + 2 * j, idesc, (g | tap | j) ? 1u : 0u);
            }
          }
          if constexpr (SB) {
            umma_commit_warp(&bempty[bs]);
            if (++bs == p.b_stages) {
              bs = 0;
              bph ^= 1;
            }
          }
        }
        umma_commit_warp(&aempty[s]);
        if (++s == p.a_stages) {
          s = 0;
          ph ^= 1;
        }
      }
      umma_commit_warp(&tfull[acc]);
      if (p.trace && blockIdx.x == 0 && lane == 0 && it < 64) p.trace[it * 16 + 3] = clock64();
      if (++acc == p.nacc) {
        acc = 0;
        aph ^= 1;
      }
    }
  } else if (SB && warp == ALLOC_WARP) {
    // ================= streamed weights: one TMA box (64 K x np rows, SW128) per (group, tap)
    if (lane == 0) {
      int bs = 0;
      uint32_t bph = 0;
      const int ncb = p.cpad >> 6;
      for (int t = blockIdx.x; t < p.tiles; t += gridDim.x)
        for (int g = 0; g < groups; ++g)
          for (int k = 0; k < TAPS; ++k) {
            int tap = k, cb = g;
            if constexpr (S == 2) {  // the quadrant's taps (ky, kx) = (2dy + py, 2dx + px), MMA order
              const int qd = g / ncb;
              const int py = qd >> 1, px = qd & 1;
              const int ndx = 2 - px;
              if (k >= (2 - py) * ndx) break;
              const int dy = k / ndx, dx = k - dy * ndx;
              tap = (2 * dy + py) * 3 + 2 * dx + px;
              cb = g - qd * ncb;
            }
            mbar_wait(&bempty[bs], bph ^ 1);
            if (p.dbg & 512) {  // ablation: no weight traffic
              mbar_arrive(&bfull[bs]);
            } else {
              mbar_arrive_expect_tx(&bfull[bs], p.b_block_bytes);
              tma_load_2d(&tmW, &bfull[bs], sB + bs * p.b_block_bytes, tap * p.cpad + cb * 64, 0);
            }
            if (++bs == p.b_stages) {
              bs = 0;
              bph ^= 1;
            }
          }
    }
  } else if (AT && warp == ALLOC_WARP && p.epi4) {
    if (lane == 0) {
      griddep_wait();  // the input activations come from the previous kernel (PDL)
      issue_input_boxes();
    }
    __syncwarp();
  }
  if (warp < HALO_EPI_WARPS || (p.epi4 && warp >= HALO_PROD_WARP0)) {
    // ================= epilogue: group g = warp / 4 drains the tiles it % 2 == g; warp q = warp % 4
    // owns TMEM lanes / tile rows 32q .. 32q+31 (epi4: producer warps 14-17 are group 3)
    const int grp = warp >= HALO_PROD_WARP0 ? 3 : warp >> 2;  // groups >= p.ngroups stay idle
    const int q = warp & 3;
    uint8_t* slot = sE + (grp * 4 + q) * HALO_SLOT;  // one store slot per warp (a group's tiles are far apart)
    const int nchunks = (p.np + 63) >> 6;
    uint32_t ec = 0;
    int it = 0;
    for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++it) {
      // drainers == 1: the group takes whole tiles, it % ngroups == grp.  Otherwise the tile's 64-column
      // chunks cm = 0 .. MT * nchunks - 1 are dealt to all groups, rotated per tile: cm = first + k ngroups
      const int cstep = p.drainers == 1 ? 1 : p.ngroups;
      const int first = p.drainers == 1 ? ((it % p.ngroups) == grp ? 0 : MT * nchunks)
                                        : ((grp - it) % p.ngroups + p.ngroups) % p.ngroups;
      if (grp >= p.ngroups || first >= MT * nchunks) continue;
      int img = t / p.tiles_per_img;
      int y0 = (t - img * p.tiles_per_img) * G::RT;
      const int r0 = q * 32;
      bool store_ok = true;
      if (p.ipt > 1) {  // this warp's rows lie in stacked image i (host: H + 1 a multiple of the box rows)
        const int i = (r0 / WP) / (p.Ho + 1);
        img = t * p.ipt + i;
        y0 = -i * (p.Ho + 1);
        store_ok = i < p.ipt;
      }
      const int ox = r0 % WP;
      const int acc = it % p.nacc;
      if (p.trace && blockIdx.x == 0 && warp == 0 && lane == 0 && it < 64) p.trace[it * 16 + 4] = clock64();
      if (p.dbg & 128) mbar_wait_sleep(&tfull[acc], (it / p.nacc) & 1, 2000);
      else mbar_wait(&tfull[acc], (it / p.nacc) & 1);
      if (p.trace && blockIdx.x == 0 && warp == 0 && lane == 0 && it < 64) p.trace[it * 16 + 5] = clock64();
      tc_fence_after();
#define HALO_T(k) \
  if (p.trace && blockIdx.x == 0 && warp == 0 && lane == 0 && it < 64 && cm < 2) p.trace[it * 16 + 8 + cm * 4 + (k)] = clock64()
      for (int cm = first; cm < MT * nchunks; cm += cstep, ++ec) {
        const int mt = cm / nchunks, c = cm - mt * nchunks;
        const int oy = y0 + mt * G::R + r0 / WP;
        const uint32_t taddr =
            tmem_base + (acc * MT + mt) * p.acc_cols + (static_cast<uint32_t>(q * 32) << 16);

        const int col0 = c * 64;
        if (lane == 0 && !(p.dbg & 16)) bulk_wait_read<0>();  // this warp's previous store has left the slot
        __syncwarp();
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {  // 32 columns per TMEM round trip (register budget)
          const int colh = col0 + half * 32;
          if (colh >= p.np) break;
          uint32_t v[32];
          if (p.dbg & 4) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0;
          } else {
            if (colh + 32 <= p.np) tmem_ld32(taddr + colh, v);
            else tmem_ld16_lo(taddr + colh, v);
            tmem_ld_wait();
          }
          HALO_T(half);
          const bool last = cm + cstep >= MT * nchunks && (half == 1 || colh + 32 >= p.np);
          if (last) {  // accumulators drained: hand them back before the math and store
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (p.trace && blockIdx.x == 0 && warp == 0 && lane == 0 && it < 64) p.trace[it * 16 + 6] = clock64();
          }
          if (p.dbg & 2) continue;
          // 16-byte chunk k (channels colh + 8k ..) of row `lane`, SW128 position (half*4+k) ^ (lane & 7)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const int col = colh + 8 * jj;
            if (col >= p.np) break;
            float4 b0 = make_float4(0.f, 0.f, 0.f, 0.f), b1 = b0;
            if (!(p.dbg & 256)) {
              b0 = *reinterpret_cast<const float4*>(sBias + col);
              b1 = *reinterpret_cast<const float4*>(sBias + col + 4);
            }
            const float2 s0 = add_f32x2(make_float2(__uint_as_float(v[8 * jj]), __uint_as_float(v[8 * jj + 1])),
                                        make_float2(b0.x, b0.y));
            const float2 s1 = add_f32x2(make_float2(__uint_as_float(v[8 * jj + 2]), __uint_as_float(v[8 * jj + 3])),
                                        make_float2(b0.z, b0.w));
            const float2 s2 = add_f32x2(make_float2(__uint_as_float(v[8 * jj + 4]), __uint_as_float(v[8 * jj + 5])),
                                        make_float2(b1.x, b1.y));
            const float2 s3 = add_f32x2(make_float2(__uint_as_float(v[8 * jj + 6]), __uint_as_float(v[8 * jj + 7])),
                                        make_float2(b1.z, b1.w));
            uint4 o;
            if (XA) {
              o = act_pack8(p.relu, s0.x, s0.y, s1.x, s1.y, s2.x, s2.y, s3.x, s3.y);
            } else if (p.relu) {
              o = make_uint4(cvt_relu_bf16x2(s0.x, s0.y), cvt_relu_bf16x2(s1.x, s1.y), cvt_relu_bf16x2(s2.x, s2.y),
                             cvt_relu_bf16x2(s3.x, s3.y));
            } else {
              o = make_uint4(cvt_bf16x2(s0.x, s0.y), cvt_bf16x2(s1.x, s1.y), cvt_bf16x2(s2.x, s2.y),
                             cvt_bf16x2(s3.x, s3.y));
            }
            const int chunk = half * 4 + jj;
            *reinterpret_cast<uint4*>(slot + lane * 128 + ((chunk ^ (lane & 7)) << 4)) = o;
          }
        }
        HALO_T(2);
        if (p.dbg & 2) continue;
        if (!(p.dbg & 32)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && !(p.dbg & 8) && store_ok) {
          tma_store_4d(&tmY, slot, col0, ox, oy, img);
          bulk_commit();
        }
        HALO_T(3);
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == ALLOC_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.nacc * MT * p.acc_cols);
  }
}

}  // namespace

// Returns UB_OK with *handled = true when the halo kernel ran; *handled = false (and UB_OK)
// when the layer is outside its scope (the caller then uses the generic kernel).
long long* g_halo_trace = nullptr;

int conv_halo_fwd(const ub_conv_desc* d, int lead, int cpad, cudaStream_t stream, bool* handled) {
  *handled = false;
  if (d->kh != 3 || d->kw != 3 || (d->stride != 1 && d->stride != 2) || d->pad != 1 || d->x_nchw_f32 ||
      d->gather_idx || d->residual || d->y_dtype != UB_BF16 || (d->variant & 8) || d->y2)
    return UB_OK;
  const int S = d->stride;
  if (cpad != 16 && cpad != 32 && cpad % 64 != 0) return UB_OK;
  if (S == 2 && (cpad % 64 != 0 || lead != 0)) return UB_OK;  // a folded plane = 8 channels of one pixel
  if (d->cout > 256 || d->y_cstride % 8 || d->y_coff % 8) return UB_OK;
  const int Ho = d->Ho;
  int Wp = 8;
  // stride 1: one zero column (the right pad of a row is the left pad of the next); stride 2:
  // folded columns 0 .. Wo (origin -1)
  while (Wp < d->Wo + 1) Wp <<= 1;
  if (Wp > 128) return UB_OK;  // WP = 128: one output row per MMA tile (EfficientNetV2's 112-wide stages)
  HaloParams p{};
  p.x = reinterpret_cast<const uint16_t*>(d->x) + (d->x_coff - lead);
  p.x_cstride = d->x_cstride;
  p.N = d->N;
  p.H = d->H;
  p.W = d->W;
  p.Ho = Ho;
  p.Wp = Wp;
  p.wp_shift = __builtin_ctz(Wp);
  p.R = 128 / Wp;
  p.groups = S == 2 ? 4 * (cpad / 64) : (cpad > 64 ? cpad / 64 : 1);
  p.planes = p.groups > 1 ? 8 : cpad / 8;
  p.np = (d->cout + 15) / 16 * 16;
  p.acc_cols = p.np <= 32 ? 32 : (p.np <= 64 ? 64 : (p.np <= 128 ? 128 : 256));
  // two MMA tiles per staged tile when the image has the rows and TMEM holds 2 x 2 of them
  int mt = (Ho > p.R && 4 * p.acc_cols <= 512) ? 2 : 1;
  // four MMA tiles per staged tile for narrow outputs on wide rows (fewer, longer tiles: the
  // per-tile barrier / store overheads dominate 32-column tiles)
  // (measured: EfficientNetV2's 112-wide stages 613 -> 594 us; ResNet-50's 56-wide layer 1 -0.2 %,
  // so by default only at padded width 128; UB_HALO_MT4=1 / 0 forces it on / off)
  static const int mt4_env = getenv("UB_HALO_MT4") ? atoi(getenv("UB_HALO_MT4")) : -1;
  const bool mt4 = mt4_env < 0 ? Wp == 128 : mt4_env != 0;
  if (mt4 && Wp >= 64 && p.acc_cols <= 32 && Ho >= 4 * p.R && S == 1) mt = 4;
  p.nacc = 512 / (mt * p.acc_cols) >= 4 ? 4 : 2;  // tiles in flight (MMA runs ahead of the epilogue)
  // input by TMA boxes (AT) when a position's channels fill a 64- or 128-byte swizzle row
  const bool at = (cpad == 32 || cpad % 64 == 0) && !(d->variant & 2048);
  // AT with resident weights: the producer warps only stage the weights, so they drain as a
  // fourth epilogue group (the TMEM-alloc warp issues the input boxes)
  static const bool epi4_env = !std::getenv("UB_HALO_NOEPI4");
  p.epi4 = (epi4_env && at && p.groups == 1 && !(d->variant & 128)) ? 1 : 0;
  p.ngroups = (d->variant & 128) ? 2 : (p.epi4 ? 4 : HALO_EPI_WARPS / 4);
  // chunks dealt to all groups when every group gets one (shorter drain per tile), else whole tiles
  p.drainers = (mt * ((p.np + 63) / 64) >= p.ngroups && !(d->variant & 1024)) ? p.ngroups : 1;
  if (p.drainers == 1 && p.ngroups > p.nacc) p.ngroups = p.nacc;  // (epi4 then leaves group 3 idle)
  p.n_pos = S == 1 ? ((mt * p.R + 2) * Wp + 2 + 7) / 8 * 8 : ((mt * p.R + 1) * Wp + 1 + 7) / 8 * 8;  // == N_POS
  p.plane_stride = p.n_pos * 16 + 16;               // == HaloGeom<Wp, mt>::PLANE_STRIDE
  p.a_stage_bytes = (p.planes * p.plane_stride + 127) & ~127u;
  if (S == 2 && !at) return UB_OK;
  const int kb = p.planes * 16;
  if (at) {
    const int staged_rows = S == 1 ? mt * p.R + 2 : mt * p.R + 1;
    p.a_stage_bytes = static_cast<uint32_t>(((staged_rows * Wp + 8) * kb + 1023) & ~1023);
  }
  p.tiles_per_img = (Ho + mt * p.R - 1) / (mt * p.R);
  // small images: stack ipt of them per 128-row tile, one zero row between (a store box stays in one image)
  p.ipt = 1;
  if (mt == 1 && (Ho + 1) * Wp <= 64 && (Ho + 1) % (32 / (Wp < 32 ? Wp : 32)) == 0 && !(d->variant & 256))
    p.ipt = 128 / ((Ho + 1) * Wp);
  const long long tiles =
      p.ipt > 1 ? (d->N + p.ipt - 1) / p.ipt : static_cast<long long>(d->N) * p.tiles_per_img;
  if (tiles >= (1ll << 31)) return UB_OK;
  p.tiles = static_cast<int>(tiles);
  p.cout = d->cout;
  p.b_block_bytes = static_cast<uint32_t>((p.np + 7) / 8 * 8) * 128;
  p.b_stages = p.groups > 1 ? 4 : 0;
  p.kvalid = lead + d->cin;
  p.w = reinterpret_cast<const uint16_t*>(d->w);
  p.cpad = cpad;
  p.bias = d->bias;
  p.relu = d->relu;
  p.bx = Wp < 32 ? Wp : 32;
  {
    static long long* trace = nullptr;
    static int want = -1;
    if (want < 0) want = getenv("UB_HALO_TRACE") ? 1 : 0;
    if (want && !trace) cudaMalloc(&trace, 64 * 16 * sizeof(long long));
    p.trace = trace;
    g_halo_trace = trace;
    static int dbg = -1;
    if (dbg < 0) dbg = getenv("UB_HALO_DBG") ? atoi(getenv("UB_HALO_DBG")) : 0;
    p.dbg = dbg;
  }
  const size_t fixed = 1024 + (p.groups == 1 ? 9 : p.b_stages) * static_cast<size_t>(p.b_block_bytes) +
                      (p.epi4 ? 16 : HALO_EPI_WARPS) * HALO_SLOT + 256 * 4 + 512;
  const size_t budget = 227 * 1024;
  if (fixed + 2 * p.a_stage_bytes > budget) return UB_OK;
  int stages = static_cast<int>((budget - fixed) / p.a_stage_bytes);
  p.a_stages = stages > 6 ? 6 : stages;
  const size_t smem = fixed + static_cast<size_t>(p.a_stages) * p.a_stage_bytes;

  if (!encode_tiled_fn()) return fail(UB_ECUDA, "ub_conv_fwd: cannot resolve cuTensorMapEncodeTiled");
  CUtensorMap tm{};
  const cuuint64_t cs = static_cast<cuuint64_t>(d->y_cstride) * 2;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(d->cout), static_cast<cuuint64_t>(d->Wo),
                        static_cast<cuuint64_t>(d->Ho), static_cast<cuuint64_t>(d->N)};
  cuuint64_t strides[3] = {cs, cs * d->Wo, cs * d->Wo * d->Ho};
  cuuint32_t box[4] = {64, static_cast<cuuint32_t>(p.bx), static_cast<cuuint32_t>(32 / p.bx), 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = encode_tiled_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                                 reinterpret_cast<uint16_t*>(d->y) + d->y_coff, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_fwd: encode halo output tensor map failed (%d)", (int)r);
  apply_small_tensor_quirk(&tm, static_cast<size_t>(d->N) * d->Ho * d->Wo * d->y_cstride * 2);

  const int grid = p.tiles < num_sms() ? p.tiles : num_sms();
  void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const HaloParams) = nullptr;
  const bool xa = d->relu > 1;
  const bool sb = p.groups > 1;
#define UB_HALO_CASE(WPV, PL, SBV, SV, ATV)                                                     \
  if (Wp == WPV && p.planes == PL && sb == SBV && S == SV && at == ATV && mt <= 2)              \
    kern = xa ? (mt == 2 ? conv_halo3_kernel<WPV, PL, 2, SBV, SV, ATV, true>                       \
                         : conv_halo3_kernel<WPV, PL, 1, SBV, SV, ATV, true>)                       \
              : (mt == 2 ? conv_halo3_kernel<WPV, PL, 2, SBV, SV, ATV, false>                      \
                         : conv_halo3_kernel<WPV, PL, 1, SBV, SV, ATV, false>);
#define UB_HALO_CASE4(WPV, PL, ATV)                                                              \
  if (Wp == WPV && p.planes == PL && !sb && S == 1 && at == ATV && mt == 4)                    \
    kern = xa ? conv_halo3_kernel<WPV, PL, 4, false, 1, ATV, true> : conv_halo3_kernel<WPV, PL, 4, false, 1, ATV, false>;
#define UB_HALO_WP(WPV)                                                                                    \
  UB_HALO_CASE(WPV, 2, false, 1, false) UB_HALO_CASE(WPV, 4, false, 1, false)                              \
  UB_HALO_CASE(WPV, 4, false, 1, true) UB_HALO_CASE(WPV, 8, false, 1, false)                               \
  UB_HALO_CASE(WPV, 8, false, 1, true) UB_HALO_CASE(WPV, 8, true, 1, false) UB_HALO_CASE(WPV, 8, true, 1, true) \
  UB_HALO_CASE(WPV, 8, true, 2, true)
  UB_HALO_WP(8) UB_HALO_WP(16) UB_HALO_WP(32) UB_HALO_WP(64) UB_HALO_WP(128)
  UB_HALO_CASE4(64, 4, true) UB_HALO_CASE4(64, 8, true) UB_HALO_CASE4(128, 2, false) UB_HALO_CASE4(128, 4, true)
  UB_HALO_CASE4(128, 8, true)
#undef UB_HALO_WP
#undef UB_HALO_CASE
#undef UB_HALO_CASE4
  if (!kern) return UB_OK;
  if (const cudaError_t ae = ensure_max_smem(kern)) return cuda_status(ae, "cudaFuncSetAttribute(halo)");
  CUtensorMap tmw{};
  if (p.groups > 1) {  // weights [cout][9 * cpad]: box 64 K x np rows
    cuuint64_t wd[2] = {static_cast<cuuint64_t>(9 * cpad), static_cast<cuuint64_t>(d->cout)};
    cuuint64_t ws[1] = {static_cast<cuuint64_t>(9 * cpad) * 2};
    cuuint32_t wb[2] = {64, static_cast<cuuint32_t>(p.np)};
    cuuint32_t we[2] = {1, 1};
    CUresult rw = encode_tiled_fn()(&tmw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(d->w), wd, ws, wb, we,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rw != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_fwd: encode halo weight tensor map failed (%d)", (int)rw);
  }
  CUtensorMap tmx{};
  if (at) {  // input [N][H][W][lead + cin] (channels past the slice read as zeros), one box per group
    const int box_rows = p.ipt > 1 ? (S == 1 ? d->H + 2 : 2 * (Ho + 1)) : (S == 1 ? mt * p.R + 2 : 2 * (mt * p.R + 1));
    p.a_box_bytes = static_cast<uint32_t>(kb) * Wp * (box_rows / S);
    const cuuint64_t xs = static_cast<cuuint64_t>(d->x_cstride) * 2;
    cuuint64_t xd[4] = {static_cast<cuuint64_t>(lead + d->cin), static_cast<cuuint64_t>(d->W),
                        static_cast<cuuint64_t>(d->H), static_cast<cuuint64_t>(d->N)};
    cuuint64_t xst[3] = {xs, xs * d->W, xs * d->W * d->H};
    cuuint32_t xb[4] = {static_cast<cuuint32_t>(kb / 2), static_cast<cuuint32_t>(S * Wp),
                        static_cast<cuuint32_t>(box_rows), 1};
    cuuint32_t xe[4] = {1, static_cast<cuuint32_t>(S), static_cast<cuuint32_t>(S), 1};
    CUresult rx = encode_tiled_fn()(&tmx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<uint16_t*>(p.x), xd, xst,
                                    xb, xe, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    kb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                    a_promo(d->x_coff - lead == 0 && cpad >= d->x_cstride),
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rx != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_fwd: encode halo input tensor map failed (%d)", (int)rx);
  }
  const cudaError_t e = launch_pdl(kern, dim3(grid), dim3(HALO_THREADS), smem, stream, tm, tmw, tmx, p);
  count_launch();
  *handled = true;
  if (e != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    return fail(UB_ECUDA, "conv_halo3_kernel: %s (threads %d, max %d, regs %d, smem %zu, max dyn %d)",
                cudaGetErrorString(e), HALO_THREADS, fa.maxThreadsPerBlock, fa.numRegs, smem,
                fa.maxDynamicSharedSizeBytes);
  }
  return UB_OK;
}

}  // namespace ub

extern "C" long long* ub_debug_halo_trace() { return ub::g_halo_trace; }

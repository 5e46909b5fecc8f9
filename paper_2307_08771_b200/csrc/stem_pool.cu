// Space-to-depth stem fused with the 3x3 / stride-2 / pad-1 max pool that follows it.
//
// A tile is a PAIR of conv rows (2yp, 2yp+1) of one image, computed as ONE 128-row MMA with
// the roles of the operands swapped: the accumulator's 128 TMEM lanes are (conv row r, output
// channel c) = r * 64 + c and its columns are the conv pixels x.  So
//   A (weights, resident): row r*64+c, K = (dy', dx, s) over dy' = 0..KQ -- the weights of
//      tap (dy' - r, dx), zero outside the filter (the second conv row is the first shifted
//      by one folded row, folded into the weights);
//   B (folded input S, one bulk copy per tile): row x = S[2yp + dy'][x + dx], a shifted view
//      (no-swizzle K-major, LBO 16 B: one K=16 MMA covers taps dx and dx+1) -- no im2col.
// (KQ + 1) * ceil(KQ/2) MMAs of N = Wo per pair.
//
// The epilogue then pools in registers: a thread owns one (conv row, channel) and the
// pixels run along its registers, so the horizontal 3-window / stride-2 max is register math
// on the raw fp32 accumulators; bias, ReLU and the bf16 rounding follow the max (exact:
// fl(v + b), ReLU and rounding are monotonic, so max commutes with them -- the result equals
// conv -> BN -> ReLU -> MaxPool of the reference).  The vertical max takes the pair's two rows
// and the previous pair's odd row, handed over through a ring in shared memory (hready /
// hfree mbarriers); the pooled row is transposed to [pixel][channel] in shared memory and
// TMA-stored.  ResNet's 411 MB conv output never exists.
//
// Work is split into bands of U pooled rows of one image; a band that does not start at
// the top of the image first computes one extra "halo" pair (2*yp0-2, 2*yp0-1) whose
// pooled row is not stored.  U is chosen on the host to balance bands over the SMs.
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      bulk-copy producer (the pair's S rows in one copy)
//   warp 1      MMA issuer (4 accumulators of 128 columns)
//   warp 2      TMEM allocator
//   warps 4-19  epilogue, four groups of four (group g drains accumulator g): warps q = 0, 1
//               own conv row 2yp (channels 32q ..), warps 2, 3 row 2yp+1
#include <cstdlib>

#include "ub_common.cuh"
#include "ub_host.h"

#include "upscale_b200.h"

namespace ub {
namespace {

constexpr int SP_STAGES_MAX = 6;
constexpr int SP_ACC = 4;          // accumulators (tiles) in flight
constexpr int SP_GROUPS = SP_ACC;  // epilogue group g drains accumulator g (tiles it % 4 == g)
constexpr int SP_THREADS = 128 + 32 * 4 * SP_GROUPS;
constexpr int SP_RING = 6;         // odd-row hand-over slots (> SP_GROUPS)
constexpr int SP_COLS = 128;       // TMEM columns per accumulator (conv pixels, Wo <= 128)

struct PoolParams {
  const uint16_t* s;  // folded input, 8 bf16 per row
  int n_img, Hs, Ws, Ho, Wo, Hp, Wp;
  int band, bands_per_img, n_bands;
  int n, cout;  // MMA N (Wo rounded up to 16), output channels (<= 64)
  uint32_t load_bytes, stage_bytes;
  int stages;
  const uint16_t* w;  // bf16 [cout][kq*kq*8]
  const float* bias;
  int relu;
  int dbg;  // profiling ablations (UB_DEBUG_FLAGS): 4 no MMA, 16 no loads, 64 no pooled-row output
  int sleep_ns;  // epilogue accumulator wait: suspend-time hint (0: spin)
  int rw;  // ring words per channel (bf16 pairs of pooled pixels; rw / 4 odd: conflict-free rows)
  uint16_t* y;  // direct-store output (pooled [n][yp][xp] rows at pitch y_cstride) or null: TMA store
  int y_cstride;
  // fused pack (ub_stem_maxpool): the producer warps build the pair's folded rows straight from
  // the fp32 NCHW model input (the INPUT GATHER's channels idx) instead of bulk-copying S
  const float* x;  // null: S-based (ub_conv_s2d_maxpool)
  const int32_t* idx;
  int C, H, W, cin, pad;
  uint32_t raw_off, raw_bytes, raw_plane;  // PACK: window offset in a stage, bytes, per-channel bytes
  uint32_t raw_tx;                         // PACK: bytes the window's TMA boxes deliver
  int raw_cols;                            // PACK: floats per window row
  int raw_half;                            // PACK: floats per row of one of the two boxes
  uint32_t raw_box;                        // PACK: smem bytes of one box (128-byte aligned)
  int raw_xoff;                            // PACK: window column of input column 0 (multiple of 4, >= pad)
  int quad;  // tiles of FOUR conv rows x 32 channels (cout <= 32): band / tile counts in pooled rows / 2
};

constexpr int SP_PACK_THREADS = 64;  // warps 0 and 3 when packing

// The CTA's tile sequence: bands u = blockIdx.x, +gridDim.x, ...; per band an optional halo
// pair then the pairs of its pooled rows.
struct TileIter {
  int u, j, j_end, n, yp0;
  int step;  // pooled rows per tile: 1 (pair of conv rows) or 2 (quad)
  __device__ void start_band(const PoolParams& p) {
    step = p.quad ? 2 : 1;
    n = u / p.bands_per_img;
    yp0 = (u - n * p.bands_per_img) * p.band;
    const int yp1 = min(p.Hp, yp0 + p.band);
    j = yp0 > 0 ? -1 : 0;
    j_end = (yp1 - yp0 + step - 1) / step;
  }
  __device__ bool valid(const PoolParams& p) const { return u < p.n_bands; }
  __device__ int yp() const { return yp0 + j * step; }  // first pooled row of the tile
  __device__ bool emit() const { return j >= 0; }
  __device__ void next(const PoolParams& p) {
    if (++j >= j_end) {
      u += gridDim.x;
      if (u < p.n_bands) start_band(p);
    }
  }
};

// QUAD (cout <= 32): a tile is FOUR conv rows 4t .. 4t+3 as one 128-row MMA (lane = r * 32 + c),
// i.e. two pooled rows 2t (conv rows 4t-1, 4t, 4t+1) and 2t+1 (4t+1 .. 4t+3): every
// accumulator lane holds a kept channel (the pair form leaves lanes of channels 32-63 empty at
// 50 % sparsity), (KQ+3)*PAIRS MMAs per two pooled rows instead of 2*(KQ+1)*PAIRS, and half
// the epilogue work per pooled row.  Warps q = 1, 3 hand their rows over (ring slot: [r1 | r3]);
// q = 0 pools row 2t with the previous tile's r3, q = 2 pools row 2t+1.
template <int KQ, bool PACK, bool QUAD = false>  // PACK: the producer warps fold the fp32 input (p.x)
__global__ void __launch_bounds__(SP_THREADS, 1)
    stem_pool_kernel(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmX,
                     const PoolParams p) {
  constexpr int ROWS = QUAD ? 4 : 2, CH = QUAD ? 32 : 64;  // conv rows per tile, channels per row
  constexpr int PAIRS = (KQ + 1) / 2, NMMA = (KQ + ROWS - 1) * PAIRS;
  constexpr uint32_t A_BYTES = 128 * 32;  // one MMA's weights: 128 rows x K 16
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t out_sz = (static_cast<uint32_t>(p.Wp) * 128 + 1023) & ~1023u;
  const uint32_t ring_sz = 64u * p.rw * 4;
  uint8_t* sW = base;                                // NMMA x [khalf][128 rows][16 B]
  uint8_t* sOut = sW + NMMA * A_BYTES;               // per group: pooled row(s) [xp][64 ch] SW128
  uint8_t* sRing = sOut + SP_GROUPS * (QUAD ? 2 : 1) * out_sz;  // SP_RING x [64 ch][rw words]
  uint8_t* sS = sRing + SP_RING * ring_sz;           // stages x folded rows
  uint64_t* full = reinterpret_cast<uint64_t*>(sS + p.stages * p.stage_bytes);
  uint64_t* empty = full + SP_STAGES_MAX;
  uint64_t* tfull = empty + SP_STAGES_MAX;
  uint64_t* tempty = tfull + SP_ACC;
  uint64_t* hready = tempty + SP_ACC;
  uint64_t* hfree = hready + SP_RING;
  uint64_t* rfull = hfree + SP_RING;  // PACK: the raw fp32 window of stage s landed (TMA tx)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rfull + SP_STAGES_MAX);
  float* sBias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 512);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmY);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], PACK ? SP_PACK_THREADS : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < SP_ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // the group's four warps
    }
    for (int r = 0; r < SP_RING; ++r) {
      mbar_init(&hready[r], 2);  // the two odd-row warps of the writing tile
      // readers: pair -- the even-row warps of the writing tile and of the next; quad -- warps
      // q = 0, 2 of the writing tile and q = 0 of the next
      mbar_init(&hfree[r], QUAD ? 3 : 4);
    }
    if (PACK)
      for (int s = 0; s < p.stages; ++s) mbar_init(&rfull[s], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, SP_ACC * SP_COLS);
  // weights: MMA j = dy' * PAIRS + pr, row m = r * 64 + c, K half h -> tap (dy' - r, 2 pr + h)
  for (int i = threadIdx.x; i < NMMA * 2 * 128; i += blockDim.x) {
    const int m = i & 127;
    const int jh = i >> 7;
    const int j = jh >> 1, h = jh & 1;
    const int r = m / CH, c = m % CH;
    const int dy = j / PAIRS - r;
    const int dx = (j % PAIRS) * 2 + h;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (c < p.cout && dy >= 0 && dy < KQ && dx < KQ)
      v = *reinterpret_cast<const uint4*>(p.w + static_cast<size_t>(c) * (KQ * KQ * 8) + (dy * KQ + dx) * 8);
    *reinterpret_cast<uint4*>(sW + j * A_BYTES + h * 2048 + m * 16) = v;
  }
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sBias[i] = (p.bias && i < p.cout) ? p.bias[i] : 0.f;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  griddep_launch_dependents();
  TileIter ti;
  ti.u = blockIdx.x;
  if (ti.valid(p)) ti.start_band(p);

  if (PACK && warp == 2) {
    // ================= producer (fused pack, part 1): the pair's raw fp32 window -- input
    // rows 2Y0 - pad .. 2(Y0 + KQ) + 1 - pad, columns -pad .. 2 Ws - 1 - pad of each kept
    // channel -- by one TMA box per channel (zero-filled outside the image)
    if (lane == 0) {
      griddep_wait();  // the model input comes from the host copy / previous graph node
      tma_prefetch_desc(&tmX);
      int s = 0;
      uint32_t ph = 0;
      const int c0 = __ldg(p.idx), c1 = p.cin > 1 ? __ldg(p.idx + 1) : 0;
      for (; ti.valid(p); ti.next(p)) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* raw = sS + s * p.stage_bytes + p.raw_off;
        const int row0 = 4 * ti.yp() - p.pad;
        if (p.dbg & 16) {  // ablation: no input loads
          mbar_arrive(&rfull[s]);
        } else {
          mbar_arrive_expect_tx(&rfull[s], p.raw_tx);
          // two half-width boxes per channel plane (a box may not be wider than the image)
          for (int c = 0; c < p.cin; ++c) {
            const int z = ti.n * p.C + (c ? c1 : c0);
            uint8_t* dstp = raw + c * p.raw_plane;
            // the innermost box coordinate must be 16-byte aligned: start at -xoff (xoff >= pad)
            tma_load_3d(&tmX, &rfull[s], dstp, -p.raw_xoff, row0, z);
            tma_load_3d(&tmX, &rfull[s], dstp + p.raw_box, -p.raw_xoff + p.raw_half, row0, z);
          }
        }
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    __syncwarp();  // reconverge: this warp deallocates TMEM (a .sync.aligned op) at the end
  } else if (PACK && (warp == 0 || warp == 3)) {
    // ================= producer (fused pack, part 2): fold the raw window in smem -- folded
    // pixel e of the S window = 8 bf16 = (py, px, c) of window row 2 dyr + py, column 2X + px
    const int pt = (warp == 0 ? 0 : 32) + lane;
    int s = 0;
    uint32_t ph = 0;
    const int nrows = static_cast<int>(p.load_bytes >> 4);
    const int hw = p.raw_half;  // floats per window row of one box (columns [0, hw) / [hw, 2 hw))
    const int box_f = static_cast<int>(p.raw_box >> 2);
    for (; ti.valid(p); ti.next(p)) {
      mbar_wait(&rfull[s], ph);
      uint4* dst = reinterpret_cast<uint4*>(sS + s * p.stage_bytes);
      const float* raw = reinterpret_cast<const float*>(sS + s * p.stage_bytes + p.raw_off);
      const int plane_f = static_cast<int>(p.raw_plane >> 2);
      const int sh = p.raw_xoff - p.pad;  // window column of folded column 0, px = 0
      for (int e = pt; e < nrows; e += SP_PACK_THREADS) {
        const int dyr = e / p.Ws;
        const int X = e - dyr * p.Ws;
        const int ca = 2 * X + sh, cb = ca + 1;  // window columns of px = 0, 1 (may sit in different boxes)
        const int oa = (ca < hw ? ca : box_f + ca - hw) + (2 * dyr) * hw;
        const int ob = (cb < hw ? cb : box_f + cb - hw) + (2 * dyr) * hw;
        const float* r = raw;
        const float* q = raw + plane_f;
        if (p.cin > 1) {  // slot (py, px, c) = q * cin + c, as ub_stem_s2d_pack
          dst[e] = make_uint4(cvt_bf16x2(r[oa], q[oa]), cvt_bf16x2(r[ob], q[ob]), cvt_bf16x2(r[oa + hw], q[oa + hw]),
                              cvt_bf16x2(r[ob + hw], q[ob + hw]));
        } else {
          dst[e] = make_uint4(cvt_bf16x2(r[oa], r[ob]), cvt_bf16x2(r[oa + hw], r[ob + hw]), 0u, 0u);
        }
      }
      fence_proxy_async_smem();  // st.shared (generic proxy) -> tensor-core reads
      mbar_arrive(&full[s]);
      if (++s == p.stages) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {  // ================= producer: the pair's folded rows in one bulk copy
      griddep_wait();  // S comes from the pack kernel (PDL)
      int s = 0;
      uint32_t ph = 0;
      for (; ti.valid(p); ti.next(p)) {
        const size_t R0 = (static_cast<size_t>(ti.n) * p.Hs + 2 * ti.yp()) * p.Ws;
        mbar_wait(&empty[s], ph ^ 1);
        if (p.dbg & 16) {
          mbar_arrive(&full[s]);
        } else {
          mbar_arrive_expect_tx(&full[s], p.load_bytes);
          bulk_load(sS + s * p.stage_bytes, p.s + R0 * 8, p.load_bytes, &full[s]);
        }
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {  // ================= MMA issuer
    const uint32_t idesc = make_idesc_bf16(128, static_cast<uint32_t>(p.n));
    uint64_t adesc[NMMA];
    uint32_t boff[NMMA];
#pragma unroll
    for (int j = 0; j < NMMA; ++j) {
      adesc[j] = sdesc_plain(smem_u32(sW) + j * A_BYTES, 2048, 128);
      boff[j] = static_cast<uint32_t>((j / PAIRS) * p.Ws + (j % PAIRS) * 2);
    }
    const uint64_t bdesc0 = sdesc_plain(smem_u32(sS), 16, 128);
    const uint32_t stage_units = p.stage_bytes >> 4;
    int s = 0, a = 0;
    uint32_t sph = 0, aph = 0;
    for (; ti.valid(p); ti.next(p)) {
      mbar_wait(&tempty[a], aph ^ 1);
      mbar_wait(&full[s], sph);
      __syncwarp();
      tc_fence_after();
      const uint64_t bd = bdesc0 + s * stage_units;
      const uint32_t d = tmem_base + a * SP_COLS;
#pragma unroll
      for (int j = 0; j < NMMA; ++j)
        if (!(p.dbg & 4)) umma_bf16_warp(d, adesc[j], bd + boff[j], idesc, j > 0 ? 1u : 0u);
      umma_commit_warp(&empty[s]);
      umma_commit_warp(&tfull[a]);
      if (++s == p.stages) {
        s = 0;
        sph ^= 1;
      }
      if (++a == SP_ACC) {
        a = 0;
        aph ^= 1;
      }
    }
  } else if (QUAD && warp >= 4) {  // ================= epilogue, quad tiles
    const int grp = (warp - 4) >> 2;
    const int q = warp & 3;  // TMEM lane quarter = conv row r of the tile; lane = channel
    const int c = lane;
    const float bias = sBias[c];
    uint8_t* out = sOut + (grp * 2 + (q >> 1)) * out_sz;  // q = 0: row 2t, q = 2: row 2t+1
    const int nw = (p.Wp + 1) >> 1;
    const int chunk8 = c >> 3;
    const uint32_t cbyte2 = (c & 7) * 2;
    int it = 0;
    for (; ti.valid(p); ti.next(p), ++it) {
      if ((it % SP_GROUPS) != grp) continue;
      const int a = it % SP_ACC;
      const int slot = it % SP_RING;
      const int prev = (it + SP_RING - 1) % SP_RING;
      if (p.sleep_ns) mbar_wait_sleep(&tfull[a], (it / SP_ACC) & 1, p.sleep_ns);
      else mbar_wait(&tfull[a], (it / SP_ACC) & 1);
      tc_fence_after();
      uint32_t h[SP_COLS / 4];
      float carry = -INFINITY;
      const uint32_t taddr = tmem_base + a * SP_COLS + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll
      for (int k = 0; k < SP_COLS / 32; ++k) {
        if (32 * k >= p.Wo) break;
        uint32_t v[32];
        tmem_ld32(taddr + 32 * k, v);
        tmem_ld_wait();
        float m[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float left = i == 0 ? carry : __uint_as_float(v[2 * i - 1]);
          m[i] = fmaxf(left, fmaxf(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])));
        }
        carry = __uint_as_float(v[31]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          h[8 * k + i] = p.relu ? cvt_relu_bf16x2(m[2 * i] + bias, m[2 * i + 1] + bias)
                                : cvt_bf16x2(m[2 * i] + bias, m[2 * i + 1] + bias);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
      uint32_t* slot_base = reinterpret_cast<uint32_t*>(sRing + slot * ring_sz);
      if (q & 1) {
        // ---- rows r1 (q = 1) and r3 (q = 3) -> ring slot halves [0] / [1]
        if (lane == 0) mbar_wait(&hfree[slot], ((it / SP_RING) & 1) ^ 1);
        __syncwarp();
        uint32_t* dst = slot_base + ((q >> 1) * 32 + c) * p.rw;
#pragma unroll
        for (int i = 0; i < SP_COLS / 4; i += 4)
          if (i < nw) *reinterpret_cast<uint4*>(dst + i) = make_uint4(h[i], h[i + 1], h[i + 2], h[i + 3]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&hready[slot]);
        continue;
      }
      // ---- q = 0: pooled row 2t = max(prev r3, r0, r1); q = 2: row 2t+1 = max(r1, r2, r3)
      const int yp = ti.yp() + (q >> 1);
      if (ti.emit() && yp < p.Hp && !(p.dbg & 64)) {
        const bool use_prev = q == 0 && yp > 0;
        mbar_wait(&hready[slot], (it / SP_RING) & 1);
        if (use_prev) mbar_wait(&hready[prev], ((it - 1) / SP_RING) & 1);
        const uint32_t* r1 = slot_base + c * p.rw;
        const uint32_t* other = q == 0 ? (use_prev ? reinterpret_cast<const uint32_t*>(sRing + prev * ring_sz) +
                                                         (32 + c) * p.rw
                                                   : r1)
                                       : slot_base + (32 + c) * p.rw;
        if (lane == 0) bulk_wait_read<0>();  // this warp's previous pooled row has left `out`
        __syncwarp();
#pragma unroll
        for (int i = 0; i < SP_COLS / 4; i += 4) {
          if (i >= nw) break;
          const uint4 o = *reinterpret_cast<const uint4*>(r1 + i);
          const uint4 pv = *reinterpret_cast<const uint4*>(other + i);
          h[i] = bf16x2_max3(h[i], o.x, pv.x);
          h[i + 1] = bf16x2_max3(h[i + 1], o.y, pv.y);
          h[i + 2] = bf16x2_max3(h[i + 2], o.z, pv.z);
          h[i + 3] = bf16x2_max3(h[i + 3], o.w, pv.w);
        }
#pragma unroll
        for (int i = 0; i < SP_COLS / 4; ++i) {
          if (i >= nw) break;
          const int x0 = 2 * i, x1 = 2 * i + 1;
          *reinterpret_cast<uint16_t*>(out + x0 * 128 + ((chunk8 ^ (x0 & 7)) << 4) + cbyte2) =
              static_cast<uint16_t>(h[i] & 0xffffu);
          if (x1 < p.Wp)
            *reinterpret_cast<uint16_t*>(out + x1 * 128 + ((chunk8 ^ (x1 & 7)) << 4) + cbyte2) =
                static_cast<uint16_t>(h[i] >> 16);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_4d(&tmY, out, 0, 0, yp, ti.n);
          bulk_commit();
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&hfree[slot]);                         // done with this tile's r1 / r3
        if (q == 0 && it > 0) mbar_arrive(&hfree[prev]);   // and with the previous tile's r3
      }
    }
    if (lane == 0) bulk_wait_all();
  } else if (warp >= 4) {  // ================= epilogue
    const int grp = (warp - 4) >> 2;
    const int q = warp & 3;              // TMEM lane quarter: (conv row r, channels 32 (q & 1) ..)
    const int r = q >> 1;
    const int c = (q & 1) * 32 + lane;   // output channel of this thread
    const bool leader = q == 0 && lane == 0;
    const float bias = sBias[c];
    uint8_t* out = sOut + grp * out_sz;  // 1024-aligned: TMA SWIZZLE_128B source
    const int nw = (p.Wp + 1) >> 1;      // bf16x2 words of a pooled row (the last half-used if Wp is odd)
    const int chunk8 = c >> 3;             // this channel's 16-byte chunk of a pooled pixel row
    const uint32_t cbyte2 = (c & 7) * 2;
    int it = 0;
    for (; ti.valid(p); ti.next(p), ++it) {
      if ((it % SP_GROUPS) != grp) continue;
      const int a = it % SP_ACC;
      const int slot = it % SP_RING;
      const int prev = (it + SP_RING - 1) % SP_RING;
      if (p.sleep_ns) mbar_wait_sleep(&tfull[a], (it / SP_ACC) & 1, p.sleep_ns);
      else mbar_wait(&tfull[a], (it / SP_ACC) & 1);
      tc_fence_after();
      // ---- horizontal 3-window / stride-2 max over this thread's conv row, 32 pixels per load
      uint32_t h[SP_COLS / 4];  // bf16x2: pooled pixels (2i, 2i+1) after bias / ReLU / rounding
      float carry = -INFINITY;  // pixel 32k - 1 (the left pad for k = 0)
      const uint32_t taddr = tmem_base + a * SP_COLS + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll
      for (int k = 0; k < SP_COLS / 32; ++k) {
        if (32 * k >= p.Wo) break;
        uint32_t v[32];
        tmem_ld32(taddr + 32 * k, v);
        tmem_ld_wait();
        float m[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float left = i == 0 ? carry : __uint_as_float(v[2 * i - 1]);
          m[i] = fmaxf(left, fmaxf(__uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1])));
        }
        carry = __uint_as_float(v[31]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          h[8 * k + i] = p.relu ? cvt_relu_bf16x2(m[2 * i] + bias, m[2 * i + 1] + bias)
                                : cvt_bf16x2(m[2 * i] + bias, m[2 * i + 1] + bias);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);  // accumulator drained
      uint32_t* ring_slot = reinterpret_cast<uint32_t*>(sRing + slot * ring_sz) + c * p.rw;
      if (r == 1) {
        // ---- odd conv row 2yp+1 -> ring slot (read by this pair and the next)
        if (lane == 0) mbar_wait(&hfree[slot], ((it / SP_RING) & 1) ^ 1);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < SP_COLS / 4; i += 4)
          if (i < nw) *reinterpret_cast<uint4*>(ring_slot + i) = make_uint4(h[i], h[i + 1], h[i + 2], h[i + 3]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&hready[slot]);
        continue;
      }
      // ---- even conv row 2yp: pooled row yp = max(row 2yp-1 (previous pair), 2yp, 2yp+1)
      if (ti.emit() && !(p.dbg & 64)) {
        const int yp = ti.yp();
        const bool has_prev = yp > 0;
        mbar_wait(&hready[slot], (it / SP_RING) & 1);
        if (has_prev) mbar_wait(&hready[prev], ((it - 1) / SP_RING) & 1);
        const uint32_t* prv = reinterpret_cast<const uint32_t*>(sRing + prev * ring_sz) + c * p.rw;
        if (leader && !p.y) bulk_wait_read<0>();  // the group's previous pooled row has left `out`
#pragma unroll
        for (int i = 0; i < SP_COLS / 4; i += 4) {
          if (i >= nw) break;
          const uint4 o = *reinterpret_cast<const uint4*>(ring_slot + i);
          uint4 pv = o;
          if (has_prev) pv = *reinterpret_cast<const uint4*>(prv + i);
          h[i] = bf16x2_max3(h[i], o.x, pv.x);
          h[i + 1] = bf16x2_max3(h[i + 1], o.y, pv.y);
          h[i + 2] = bf16x2_max3(h[i + 2], o.z, pv.z);
          h[i + 3] = bf16x2_max3(h[i + 3], o.w, pv.w);
        }
        if (p.y) {  // direct stores: per pixel the group's 64 lanes write 128 contiguous bytes
          if (c < p.cout) {
            uint16_t* dst = p.y + (static_cast<size_t>(ti.n) * p.Hp + yp) * p.Wp * p.y_cstride + c;
#pragma unroll
            for (int i = 0; i < SP_COLS / 4; ++i) {
              if (i >= nw) break;
              dst[static_cast<size_t>(2 * i) * p.y_cstride] = static_cast<uint16_t>(h[i] & 0xffffu);
              if (2 * i + 1 < p.Wp) dst[static_cast<size_t>(2 * i + 1) * p.y_cstride] = static_cast<uint16_t>(h[i] >> 16);
            }
          }
        } else {
        // [xp][64 ch] with SW128 chunk swizzle: this thread's channel, pixels 2i and 2i+1
        named_bar_sync(1 + grp, 64);
#pragma unroll
        for (int i = 0; i < SP_COLS / 4; ++i) {
          if (i >= nw) break;
          const int x0 = 2 * i, x1 = 2 * i + 1;
          *reinterpret_cast<uint16_t*>(out + x0 * 128 + ((chunk8 ^ (x0 & 7)) << 4) + cbyte2) =
              static_cast<uint16_t>(h[i] & 0xffffu);
          if (x1 < p.Wp)
            *reinterpret_cast<uint16_t*>(out + x1 * 128 + ((chunk8 ^ (x1 & 7)) << 4) + cbyte2) =
                static_cast<uint16_t>(h[i] >> 16);
        }
        fence_proxy_async_smem();
        named_bar_sync(1 + grp, 64);
        if (leader) {
          tma_store_4d(&tmY, out, 0, 0, yp, ti.n);
          bulk_commit();
        }
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&hfree[slot]);              // this pair is done with its own odd row
        if (it > 0) mbar_arrive(&hfree[prev]);  // and with the previous pair's
      }
    }
    if (q == 0 && lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, SP_ACC * SP_COLS);
  }
}

template <int KQ, bool PACK, bool QUAD = false>
void launch_pool(const CUtensorMap& tm, const CUtensorMap& tmx, const PoolParams& p, int grid, size_t smem,
                 cudaStream_t stream) {
  (void)ensure_max_smem(stem_pool_kernel<KQ, PACK, QUAD>);
  (void)launch_pdl(stem_pool_kernel<KQ, PACK, QUAD>, dim3(grid), dim3(SP_THREADS), smem, stream, tm, tmx, p);
}

}  // namespace
}  // namespace ub

using namespace ub;

namespace {
// s: the folded input S (ub_stem_s2d_pack), or x: the fp32 NCHW model input packed on the fly
int stem_maxpool_launch(const void* s, const float* x, int C, const int32_t* idx, int cin, int N, int H, int W, int k,
                        int pad, const void* w, int cout, const float* bias, int relu, int pool_k, int pool_stride,
                        int pool_pad, void* y, int y_cstride, int y_coff, cudaStream_t stream) {
  if ((!s && !x) || !w || !y || cout < 1 || N < 1) return fail(UB_EINVAL, "ub_conv_s2d_maxpool: bad arguments");
  if (x && (!idx || cin < 1 || 4 * cin > 8 || C < 1)) return fail(UB_EINVAL, "ub_stem_maxpool: bad input gather");
  if (pool_k != 3 || pool_stride != 2 || pool_pad != 1)
    return fail(UB_EUNSUPPORTED, "ub_conv_s2d_maxpool: pool %d/%d/%d (3/2/1 only)", pool_k, pool_stride, pool_pad);
  if (cout > 64) return fail(UB_EUNSUPPORTED, "ub_conv_s2d_maxpool: cout %d > 64", cout);
  if ((y_cstride & 7) || (y_coff & 7) || y_coff + cout > y_cstride)
    return fail(UB_EUNSUPPORTED, "ub_conv_s2d_maxpool: output window not 16-byte aligned");
  int Hs = 0, Ws = 0;
  long long sbytes = 0;
  int rc = ub_stem_s2d_geometry(N, H, W, k, pad, &Hs, &Ws, &sbytes);
  if (rc) return rc;
  const int kq = (k + 1) / 2;
  const int Ho = (H + 2 * pad - k) / 2 + 1, Wo = (W + 2 * pad - k) / 2 + 1;
  if (kq < 2 || kq > 4) return fail(UB_EUNSUPPORTED, "ub_conv_s2d_maxpool: kernel %d", k);
  if ((Ho & 1) || (Wo & 1) || Wo > 128)
    return fail(UB_EUNSUPPORTED, "ub_conv_s2d_maxpool: conv output %dx%d (even, width <= 128)", Ho, Wo);
  PoolParams p{};
  p.s = static_cast<const uint16_t*>(s);
  p.x = x;
  p.idx = idx;
  p.C = C;
  p.H = H;
  p.W = W;
  p.cin = cin;
  p.pad = pad;
  p.n_img = N;
  p.Hs = Hs;
  p.Ws = Ws;
  p.Ho = Ho;
  p.Wo = Wo;
  p.Hp = Ho / 2;
  p.Wp = Wo / 2;
  p.n = (Wo + 15) / 16 * 16;
  {
    static int dbg = -1;
    if (dbg < 0) dbg = getenv("UB_DEBUG_FLAGS") ? atoi(getenv("UB_DEBUG_FLAGS")) : 0;
    p.dbg = dbg;
    static int sl = -1;
    if (sl < 0) sl = getenv("UB_SP_SLEEP") ? atoi(getenv("UB_SP_SLEEP")) : 0;
    p.sleep_ns = sl;
  }
  if (getenv("UB_SP_DIRECT_STORE")) {  // direct 2-byte stores; the TMA store is the default (88.8 -> 85.6 us, r2ak)
    p.y = static_cast<uint16_t*>(y) + y_coff;
    p.y_cstride = y_cstride;
  }
  p.cout = cout;
  // quad tiles (four conv rows x 32 channels per MMA) whenever the kept channels fit 32 lanes
  static const bool quad_env = !getenv("UB_SP_NOQUAD");
  p.quad = (quad_env && !x && cout <= 32 && (p.Hp % 2) == 0) ? 1 : 0;
  const int rows = p.quad ? 4 : 2;
  p.rw = ((p.Wp + 1) / 2 + 3) / 4 * 4;
  if (((p.rw / 4) & 1) == 0) p.rw += 4;
  p.w = static_cast<const uint16_t*>(w);
  p.bias = bias;
  p.relu = relu;
  // the pair's copy: S rows R0 .. R0 + kq*Ws + 2*pairs + N - 2 (folded rows 2yp .. 2yp + kq);
  // stays inside the buffer for the last pair since S holds Hs = Ho + kq - 1 rows per image
  // plus its tail
  const int pairs = (kq + 1) / 2;
  const uint32_t load_rows = static_cast<uint32_t>((kq + rows - 2) * Ws + 2 * pairs + p.n - 1);
  const long long last_end = (static_cast<long long>(N - 1) * Hs + Ho - rows) * Ws + load_rows;
  if (last_end * 16 > sbytes) return fail(UB_EUNSUPPORTED, "ub_conv_s2d_maxpool: staging buffer too small");
  p.load_bytes = load_rows * 16;
  p.stage_bytes = (p.load_bytes + 127) & ~127u;
  if (x) {  // raw fp32 window after the folded rows: cin planes of 2 (kq + 1) rows x raw_cols
    // two boxes of raw_half columns per channel plane: a box may not be wider than the image
    p.raw_xoff = (pad + 3) & ~3;
    p.raw_half = (Ws + (p.raw_xoff - pad + 1) / 2 + 3) / 4 * 4;  // 2 boxes cover window columns up to 2 Ws + sh
    p.raw_cols = 2 * p.raw_half;
    const uint32_t box_b = static_cast<uint32_t>(2 * (kq + 1) * p.raw_half * 4);
    p.raw_box = (box_b + 127) & ~127u;  // TMA destinations 128-byte aligned
    p.raw_plane = 2 * p.raw_box;
    p.raw_bytes = p.raw_plane * static_cast<uint32_t>(cin);
    p.raw_tx = 2 * box_b * static_cast<uint32_t>(cin);
    p.raw_off = (p.stage_bytes + 1023) & ~1023u;
    p.stage_bytes = (p.raw_off + p.raw_bytes + 1023) & ~1023u;
  }
  // bands of `band` pooled rows balanced over the SMs (+1 halo pair for bands below the top)
  const int sms = num_sms();
  int best_band = p.Hp;
  long long best_cost = -1;
  for (int b = 4; b <= p.Hp; b += p.quad ? 2 : 1) {  // quad bands start on even pooled rows
    const long long per_img = (p.Hp + b - 1) / b;
    const long long nb = per_img * N;
    const long long waves = (nb + sms - 1) / sms;
    const long long cost = waves * ((b + rows / 2 - 1) / (rows / 2) + 1);  // tiles per band + halo
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best_band = b;
    }
  }
  p.band = best_band;
  p.bands_per_img = (p.Hp + p.band - 1) / p.band;
  const long long n_bands = static_cast<long long>(p.bands_per_img) * N;
  if (n_bands >= (1ll << 31)) return fail(UB_EUNSUPPORTED, "ub_conv_s2d_maxpool: too many bands");
  p.n_bands = static_cast<int>(n_bands);
  const size_t w_bytes = static_cast<size_t>(kq + rows - 1) * pairs * 128 * 32;
  const size_t out_bytes = (static_cast<size_t>(p.Wp) * 128 + 1023) & ~static_cast<size_t>(1023);
  const size_t fixed = 1024 + w_bytes + SP_GROUPS * (rows / 2) * out_bytes + SP_RING * 64 * p.rw * 4 + 512 + 64 * 4;
  int stages = static_cast<int>((227 * 1024 - fixed) / p.stage_bytes);
  if (stages < 2) return fail(UB_EUNSUPPORTED, "ub_conv_s2d_maxpool: shared memory");
  p.stages = stages > SP_STAGES_MAX ? SP_STAGES_MAX : stages;
  const size_t smem = fixed + static_cast<size_t>(p.stages) * p.stage_bytes;

  if (!encode_tiled_fn()) return fail(UB_ECUDA, "ub_conv_s2d_maxpool: cannot resolve cuTensorMapEncodeTiled");
  CUtensorMap tm{};
  const cuuint64_t cs = static_cast<cuuint64_t>(y_cstride) * 2;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(cout), static_cast<cuuint64_t>(p.Wp), static_cast<cuuint64_t>(p.Hp),
                        static_cast<cuuint64_t>(N)};
  cuuint64_t strides[3] = {cs, cs * p.Wp, cs * p.Wp * p.Hp};
  cuuint32_t box[4] = {64, static_cast<cuuint32_t>(p.Wp), 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = encode_tiled_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, static_cast<uint16_t*>(y) + y_coff, dims,
                                 strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_s2d_maxpool: encode output tensor map failed (%d)", (int)r);
  apply_small_tensor_quirk(&tm, static_cast<size_t>(N) * p.Hp * p.Wp * y_cstride * 2);
  CUtensorMap tmx{};
  if (x) {  // model input as [N*C planes][H][W] fp32; box: raw_cols x 2 (kq + 1) rows of one plane
    cuuint64_t xd[3] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(N) * C};
    cuuint64_t xs[2] = {static_cast<cuuint64_t>(W) * 4, static_cast<cuuint64_t>(W) * H * 4};
    cuuint32_t xb[3] = {static_cast<cuuint32_t>(p.raw_half), static_cast<cuuint32_t>(2 * (kq + 1)), 1};
    cuuint32_t xe[3] = {1, 1, 1};
    if (p.raw_half > 256 || p.raw_half > W || (W * 4) % 16)
      return fail(UB_EUNSUPPORTED, "ub_stem_maxpool: input width %d (window %d floats)", W, p.raw_cols);
    CUresult rx = encode_tiled_fn()(&tmx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), xd, xs, xb, xe,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rx != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_stem_maxpool: encode input tensor map failed (%d)", (int)rx);
  }
  const int grid = p.n_bands < sms ? p.n_bands : sms;
  if (p.quad) {
    switch (kq) {
      case 2: launch_pool<2, false, true>(tm, tmx, p, grid, smem, stream); break;
      case 3: launch_pool<3, false, true>(tm, tmx, p, grid, smem, stream); break;
      default: launch_pool<4, false, true>(tm, tmx, p, grid, smem, stream); break;
    }
    count_launch();
    return cuda_status(cudaGetLastError(), "stem_pool_kernel");
  }
  switch (kq) {
    case 2: x ? launch_pool<2, true>(tm, tmx, p, grid, smem, stream) : launch_pool<2, false>(tm, tmx, p, grid, smem, stream); break;
    case 3: x ? launch_pool<3, true>(tm, tmx, p, grid, smem, stream) : launch_pool<3, false>(tm, tmx, p, grid, smem, stream); break;
    default: x ? launch_pool<4, true>(tm, tmx, p, grid, smem, stream) : launch_pool<4, false>(tm, tmx, p, grid, smem, stream); break;
  }
  count_launch();
  return cuda_status(cudaGetLastError(), "stem_pool_kernel");
}
}  // namespace

extern "C" int ub_conv_s2d_maxpool(const void* s, int N, int H, int W, int k, int pad, const void* w, int cout,
                                   const float* bias, int relu, int pool_k, int pool_stride, int pool_pad, void* y,
                                   int y_cstride, int y_coff, cudaStream_t stream) {
  if (!s) return fail(UB_EINVAL, "ub_conv_s2d_maxpool: bad arguments");
  return stem_maxpool_launch(s, nullptr, 0, nullptr, 0, N, H, W, k, pad, w, cout, bias, relu, pool_k, pool_stride,
                             pool_pad, y, y_cstride, y_coff, stream);
}

extern "C" int ub_stem_maxpool(const float* x, int N, int C, int H, int W, const int32_t* idx, int cin, int k, int pad,
                               const void* w, int cout, const float* bias, int relu, int pool_k, int pool_stride,
                               int pool_pad, void* y, int y_cstride, int y_coff, cudaStream_t stream) {
  if (!x) return fail(UB_EINVAL, "ub_stem_maxpool: bad arguments");
  return stem_maxpool_launch(nullptr, x, C, idx, cin, N, H, W, k, pad, w, cout, bias, relu, pool_k, pool_stride,
                             pool_pad, y, y_cstride, y_coff, stream);
}

// Space-to-depth stem fused with the 3x3 / stride-2 / pad-1 max pool that follows it.
//
// Same tensor-core mainloop as stem_s2d.cu (the folded input S, one bulk copy per tile,
// every filter tap a shifted view), but a tile is a PAIR of conv rows (2yp, 2yp+1) -- two
// MMA tiles -- and the epilogue pools instead of storing the conv output:
//   conv row -> bias, ReLU, bf16 (the reference's conv -> BN -> ReLU) -> smem row
//   -> horizontal 3-window max at stride 2 ("hrow", Wo/2 pixels)
//   pooled row yp = max(hrow(2yp-1), hrow(2yp), hrow(2yp+1)) -> TMA store.
// Row 2yp-1 belongs to the previous pair: its hrow is handed over through a small ring in
// shared memory (mbarriers hready/hfree per slot), so the 411 MB conv output of ResNet's
// stem never reaches HBM and the pool never reads it back.  bf16 max is exact, and
// max(relu(v)) = relu(max(v)), so the result equals conv -> BN -> ReLU -> MaxPool.
//
// Work is split into bands of U pooled rows of one image; a band that does not start at
// the top of the image first computes one extra "halo" pair (2*yp0-2, 2*yp0-1) whose
// pooled row is not stored.  U is chosen on the host to balance bands over the SMs.
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      bulk-copy producer (both conv rows of a pair in one copy)
//   warp 1      MMA issuer (4 accumulator pairs)
//   warp 2      TMEM allocator
//   warps 4-19  epilogue, four groups of four (group g drains accumulator pair g)
#include <cstdlib>

#include "ub_common.cuh"
#include "ub_host.h"

#include "upscale_b200.h"

namespace ub {
namespace {

constexpr int SP_STAGES_MAX = 4;
constexpr int SP_ACC = 4;         // accumulator pairs in flight
constexpr int SP_GROUPS = SP_ACC;  // epilogue group g drains pair g (tiles it % 4 == g)
constexpr int SP_THREADS = 128 + 32 * 4 * SP_GROUPS;
constexpr int SP_RING = 6;        // hrow hand-over slots (> SP_GROUPS)

struct PoolParams {
  const uint16_t* s;  // folded input, 8 bf16 per row
  int n_img, Hs, Ws, Ho, Wo, Hp, Wp;
  int band, bands_per_img, n_bands;
  int np, cout;
  uint32_t load_bytes, stage_bytes;
  int stages;
  const uint16_t* w;  // bf16 [cout][kq*kq*8]
  const float* bias;
  int relu;
  uint32_t crow_bytes, hrow_bytes;  // Wo * 128, Wp * 128
};

// The CTA's tile sequence: bands u = blockIdx.x, +gridDim.x, ...; per band an optional halo
// pair then the pairs of its pooled rows.
struct TileIter {
  int u, j, j_end, n, yp0;
  __device__ void start_band(const PoolParams& p) {
    n = u / p.bands_per_img;
    yp0 = (u - n * p.bands_per_img) * p.band;
    const int yp1 = min(p.Hp, yp0 + p.band);
    j = yp0 > 0 ? -1 : 0;
    j_end = yp1 - yp0;
  }
  __device__ bool valid(const PoolParams& p) const { return u < p.n_bands; }
  __device__ int yp() const { return yp0 + j; }
  __device__ bool emit() const { return j >= 0; }
  __device__ void next(const PoolParams& p) {
    if (++j >= j_end) {
      u += gridDim.x;
      if (u < p.n_bands) start_band(p);
    }
  }
};

template <int KQ>
__global__ void __launch_bounds__(SP_THREADS, 1)
    stem_pool_kernel(const __grid_constant__ CUtensorMap tmY, const PoolParams p) {
  constexpr int PAIRS = (KQ + 1) / 2, NMMA = KQ * PAIRS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int b_bytes = (NMMA * 2 * p.np * 16 + 1023) & ~1023;
  const uint32_t crow_sz = (p.crow_bytes + 1023) & ~1023u, hrow_sz = (p.hrow_bytes + 1023) & ~1023u;
  const uint32_t grp_bytes = crow_sz + 2 * hrow_sz;
  uint8_t* sB = base;
  uint8_t* sG = sB + b_bytes;                      // per group: crow | hev | out (1024-aligned)
  uint8_t* sRing = sG + SP_GROUPS * grp_bytes;     // SP_RING x hrow
  uint8_t* sA = sRing + SP_RING * p.hrow_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sA + p.stages * p.stage_bytes);
  uint64_t* empty = full + SP_STAGES_MAX;
  uint64_t* tfull = empty + SP_STAGES_MAX;
  uint64_t* tempty = tfull + SP_ACC;
  uint64_t* hready = tempty + SP_ACC;
  uint64_t* hfree = hready + SP_RING;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfree + SP_RING);
  float* sBias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + 512);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmY);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < SP_ACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    for (int r = 0; r < SP_RING; ++r) {
      mbar_init(&hready[r], 1);
      mbar_init(&hfree[r], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 2 * SP_ACC * 64);
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

  if (warp == 0) {
    if (lane == 0) {  // ================= producer: conv rows 2yp, 2yp+1 in one bulk copy
      griddep_wait();  // S comes from the pack kernel (PDL)
      int s = 0;
      uint32_t ph = 0;
      for (; ti.valid(p); ti.next(p)) {
        const size_t R0 = (static_cast<size_t>(ti.n) * p.Hs + 2 * ti.yp()) * p.Ws;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], p.load_bytes);
        bulk_load(sA + s * p.stage_bytes, p.s + R0 * 8, p.load_bytes, &full[s]);
        if (++s == p.stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {  // ================= MMA issuer
    const uint32_t idesc = make_idesc_bf16(128, static_cast<uint32_t>(p.np));
    const uint32_t b0 = smem_u32(sB);
    uint64_t bdesc[NMMA];
    uint32_t aoff[NMMA];
#pragma unroll
    for (int j = 0; j < NMMA; ++j) {
      const int dy = j / PAIRS, dx = (j % PAIRS) * 2;
      aoff[j] = static_cast<uint32_t>(dy * p.Ws + dx);
      bdesc[j] = sdesc_plain(b0 + j * 2 * p.np * 16, p.np * 16, 128);
    }
    const uint64_t adesc0 = sdesc_plain(smem_u32(sA), 16, 128);
    const uint32_t stage_units = p.stage_bytes >> 4;
    int s = 0, a = 0;
    uint32_t sph = 0, aph = 0;
    for (; ti.valid(p); ti.next(p)) {
      mbar_wait(&tempty[a], aph ^ 1);
      mbar_wait(&full[s], sph);
      __syncwarp();
      tc_fence_after();
      const uint64_t ad = adesc0 + s * stage_units;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const uint32_t d = tmem_base + (a * 2 + mt) * 64;
#pragma unroll
        for (int j = 0; j < NMMA; ++j)
          umma_bf16_warp(d, ad + aoff[j] + mt * p.Ws, bdesc[j], idesc, j > 0 ? 1u : 0u);
      }
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
  } else if (warp >= 4) {  // ================= epilogue
    const int grp = (warp - 4) >> 2;
    const int quad = warp & 3;
    const int gt = threadIdx.x - 128 - grp * 128;  // 0..127 within the group
    const int r = quad * 32 + lane;                 // conv pixel x of this thread's TMEM lane
    const bool leader = gt == 0;
    uint8_t* crow = sG + grp * grp_bytes;
    uint8_t* hev = crow + crow_sz;
    uint8_t* out = hev + hrow_sz;  // 1024-aligned: TMA SWIZZLE_128B source
    const __nv_bfloat162 ninf = __floats2bfloat162_rn(-INFINITY, -INFINITY);
    uint4 ninf4;
    {
      __nv_bfloat162* v = reinterpret_cast<__nv_bfloat162*>(&ninf4);
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = ninf;
    }
    int it = 0;
    for (; ti.valid(p); ti.next(p), ++it) {
      if ((it % SP_GROUPS) != grp) continue;
      const int a = it % SP_ACC;
      const int slot = it % SP_RING;
      const int prev = (it + SP_RING - 1) % SP_RING;
      mbar_wait(&tfull[a], (it / SP_ACC) & 1);
      tc_fence_after();
      for (int mt = 0; mt < 2; ++mt) {
        // ---- conv row 2yp+mt: TMEM -> bias, ReLU, bf16 -> crow[x] (SW128-style chunk swizzle)
        uint32_t v0[32], v1[32];
        const uint32_t taddr = tmem_base + (a * 2 + mt) * 64 + (static_cast<uint32_t>(quad * 32) << 16);
        tmem_ld32(taddr, v0);
        tmem_ld32(taddr + 32, v1);
        tmem_ld_wait();
        if (mt == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[a]);
        }
        if (r < p.Wo) {
          uint8_t* rowp = crow + r * 128;
          auto emit = [&](const uint32_t (&v)[32], int half) {
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int col = half * 32 + 8 * jj;
              const float4 b0 = *reinterpret_cast<const float4*>(sBias + col);
              const float4 b1 = *reinterpret_cast<const float4*>(sBias + col + 4);
              const float2 s0 = add_f32x2(make_float2(__uint_as_float(v[8 * jj]), __uint_as_float(v[8 * jj + 1])),
                                          make_float2(b0.x, b0.y));
              const float2 s1 = add_f32x2(make_float2(__uint_as_float(v[8 * jj + 2]), __uint_as_float(v[8 * jj + 3])),
                                          make_float2(b0.z, b0.w));
              const float2 s2 = add_f32x2(make_float2(__uint_as_float(v[8 * jj + 4]), __uint_as_float(v[8 * jj + 5])),
                                          make_float2(b1.x, b1.y));
              const float2 s3 = add_f32x2(make_float2(__uint_as_float(v[8 * jj + 6]), __uint_as_float(v[8 * jj + 7])),
                                          make_float2(b1.z, b1.w));
              uint4 o;
              if (p.relu) {
                o = make_uint4(cvt_relu_bf16x2(s0.x, s0.y), cvt_relu_bf16x2(s1.x, s1.y),
                               cvt_relu_bf16x2(s2.x, s2.y), cvt_relu_bf16x2(s3.x, s3.y));
              } else {
                o = make_uint4(cvt_bf16x2(s0.x, s0.y), cvt_bf16x2(s1.x, s1.y), cvt_bf16x2(s2.x, s2.y),
                               cvt_bf16x2(s3.x, s3.y));
              }
              const int k = half * 4 + jj;
              *reinterpret_cast<uint4*>(rowp + ((k ^ (r & 7)) << 4)) = o;
            }
          };
          emit(v0, 0);
          emit(v1, 1);
        }
        if (mt == 1) {  // this tile's odd hrow goes to the ring: its previous reader must be done
          if (leader) mbar_wait(&hfree[slot], ((it / SP_RING) & 1) ^ 1);
        }
        named_bar_sync(1 + grp, 128);
        // ---- horizontal max: hrow[xp][k] = max(crow[2xp-1], crow[2xp], crow[2xp+1]) chunk k
        uint8_t* hdst = mt == 0 ? hev : sRing + slot * p.hrow_bytes;
        for (int e = gt; e < p.Wp * 8; e += 128) {
          const int xp = e >> 3, k = e & 7;
          const int x0 = 2 * xp - 1;
          uint4 m = *reinterpret_cast<const uint4*>(crow + (x0 + 1) * 128 + ((k ^ ((x0 + 1) & 7)) << 4));
          __nv_bfloat162* mv = reinterpret_cast<__nv_bfloat162*>(&m);
          if (x0 >= 0) {
            const uint4 u = *reinterpret_cast<const uint4*>(crow + x0 * 128 + ((k ^ (x0 & 7)) << 4));
            const __nv_bfloat162* uv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) mv[i] = __hmax2(mv[i], uv[i]);
          }
          if (x0 + 2 < p.Wo) {
            const uint4 u = *reinterpret_cast<const uint4*>(crow + (x0 + 2) * 128 + ((k ^ ((x0 + 2) & 7)) << 4));
            const __nv_bfloat162* uv = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) mv[i] = __hmax2(mv[i], uv[i]);
          }
          *reinterpret_cast<uint4*>(hdst + e * 16) = m;
        }
        named_bar_sync(1 + grp, 128);  // crow free for the next row; hrow complete
        if (mt == 1 && leader) mbar_arrive(&hready[slot]);
      }
      // ---- vertical max with the previous pair's odd hrow (row 2yp-1), then store
      const int yp = ti.yp();
      const bool has_prev = it > 0;
      if (has_prev) mbar_wait(&hready[prev], ((it - 1) / SP_RING) & 1);
      if (ti.emit()) {
        if (leader) bulk_wait_read<0>();  // this group's previous pooled row has left `out`
        named_bar_sync(1 + grp, 128);
        const uint8_t* hodd = sRing + slot * p.hrow_bytes;
        const uint8_t* hprv = sRing + prev * p.hrow_bytes;
        for (int e = gt; e < p.Wp * 8; e += 128) {
          const int xp = e >> 3, k = e & 7;
          uint4 m = *reinterpret_cast<const uint4*>(hev + e * 16);
          __nv_bfloat162* mv = reinterpret_cast<__nv_bfloat162*>(&m);
          const uint4 u1 = *reinterpret_cast<const uint4*>(hodd + e * 16);
          const __nv_bfloat162* v1 = reinterpret_cast<const __nv_bfloat162*>(&u1);
          const uint4 u0 = yp > 0 ? *reinterpret_cast<const uint4*>(hprv + e * 16) : ninf4;
          const __nv_bfloat162* v0 = reinterpret_cast<const __nv_bfloat162*>(&u0);
#pragma unroll
          for (int i = 0; i < 4; ++i) mv[i] = __hmax2(mv[i], __hmax2(v0[i], v1[i]));
          *reinterpret_cast<uint4*>(out + xp * 128 + ((k ^ (xp & 7)) << 4)) = m;
        }
        fence_proxy_async_smem();
        named_bar_sync(1 + grp, 128);
        if (leader) {
          tma_store_4d(&tmY, out, 0, 0, yp, ti.n);
          bulk_commit();
        }
      } else {
        named_bar_sync(1 + grp, 128);
      }
      if (has_prev && leader) mbar_arrive(&hfree[prev]);
    }
    if (leader) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * SP_ACC * 64);
  }
}

template <int KQ>
void launch_pool(const CUtensorMap& tm, const PoolParams& p, int grid, size_t smem, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(stem_pool_kernel<KQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  (void)launch_pdl(stem_pool_kernel<KQ>, dim3(grid), dim3(SP_THREADS), smem, stream, tm, p);
}

}  // namespace
}  // namespace ub

using namespace ub;

extern "C" int ub_conv_s2d_maxpool(const void* s, int N, int H, int W, int k, int pad, const void* w, int cout,
                                   const float* bias, int relu, int pool_k, int pool_stride, int pool_pad, void* y,
                                   int y_cstride, int y_coff, cudaStream_t stream) {
  if (!s || !w || !y || cout < 1 || N < 1) return fail(UB_EINVAL, "ub_conv_s2d_maxpool: bad arguments");
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
  p.n_img = N;
  p.Hs = Hs;
  p.Ws = Ws;
  p.Ho = Ho;
  p.Wo = Wo;
  p.Hp = Ho / 2;
  p.Wp = Wo / 2;
  p.np = 64;
  p.cout = cout;
  p.w = static_cast<const uint16_t*>(w);
  p.bias = bias;
  p.relu = relu;
  p.crow_bytes = static_cast<uint32_t>(Wo) * 128;
  p.hrow_bytes = static_cast<uint32_t>(p.Wp) * 128;
  // the pair's copy: rows R0 .. R0 + Ws + 128 + (kq-1)*Ws + 2*pairs - 1 of S; stays inside the
  // buffer for the last pair since S holds Hs = Ho + kq - 1 rows per image plus its tail
  const int pairs = (kq + 1) / 2;
  const uint32_t load_rows = static_cast<uint32_t>(Ws + 128 + (kq - 1) * Ws + 2 * pairs - 1);
  const long long last_end = (static_cast<long long>(N - 1) * Hs + Ho - 2) * Ws + load_rows;
  if (last_end * 16 > sbytes) return fail(UB_EUNSUPPORTED, "ub_conv_s2d_maxpool: staging buffer too small");
  p.load_bytes = load_rows * 16;
  p.stage_bytes = (p.load_bytes + 127) & ~127u;
  // bands of `band` pooled rows balanced over the SMs (+1 halo pair for bands below the top)
  const int sms = num_sms();
  int best_band = p.Hp;
  long long best_cost = -1;
  for (int b = 4; b <= p.Hp; ++b) {
    const long long per_img = (p.Hp + b - 1) / b;
    const long long nb = per_img * N;
    const long long waves = (nb + sms - 1) / sms;
    const long long cost = waves * (b + 1);
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
  const int b_bytes = (kq * pairs * 2 * p.np * 16 + 1023) & ~1023;
  const size_t grp_bytes = ((p.crow_bytes + 1023) & ~1023u) + 2 * ((p.hrow_bytes + 1023) & ~1023u);
  const size_t fixed = 1024 + b_bytes + SP_GROUPS * grp_bytes + SP_RING * p.hrow_bytes + 512 + 64 * 4;
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
  const int grid = p.n_bands < sms ? p.n_bands : sms;
  switch (kq) {
    case 2: launch_pool<2>(tm, p, grid, smem, stream); break;
    case 3: launch_pool<3>(tm, p, grid, smem, stream); break;
    default: launch_pool<4>(tm, p, grid, smem, stream); break;
  }
  count_launch();
  return cuda_status(cudaGetLastError(), "stem_pool_kernel");
}

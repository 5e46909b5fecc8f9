// Implicit-GEMM convolution on sm_100a tensor cores (tcgen05 + TMEM + TMA store).
//
// One reference CHANNEL_MIX node (interp.py:57-63, `W @ x`) executed over real
// NHWC activations, with the node that reads its input and the nodes that
// consume its output fused in:
//   * SLICE read  (interp.py:72-74): the A operand is addressed at the slice's
//     channel offset -- no copy (UPSCALE's contiguous read);
//   * GATHER read (interp.py:75-77): the producer warps gather the channels
//     (implicit im2col over the gathered set) straight from the producer
//     layer's tensor into swizzled shared memory -- the copy the baseline
//     export materialises never touches HBM;
//   * PER_CHANNEL bias (BN shift; the scale is folded into the weight rows at
//     export): written into the TMEM accumulator before the first MMA;
//   * ADD residual (interp.py:64-65): extra "identity" K-blocks -- the residual
//     tile is the A operand and a 64x64 identity the B operand, so the tensor
//     core adds it exactly in fp32;
//   * ReLU (interp.py:68-69): folded into the fp32 -> bf16x2 conversion;
//   * channel-offset store: CONCAT without a copy (interp.py:66-67).
//
// GEMM view: D[M = N*Ho*Wo pixels][cout] = A[M][K] * B[cout][K]^T, K = taps*cpad.
// Tile 128 pixels x block_n channels (block_n <= 256, runtime).
//
// Data movement follows measurements on B200 (tools/tma_probe.cu): TMA LOADS
// cost ~10 SM cycles per box row, so operands come in by cp.async from the
// producer warps (completion tracked on mbarriers); TMA STORES (~6 cycles per
// 128-byte row) carry the output.  The epilogue does ~0.7 instructions per
// output element: TMEM load, one cvt(+relu) per pair, 16-byte smem stores.
//
// Persistent, warp-specialised, one CTA (512 threads) per SM:
//   warp 1      MMA issuer: tcgen05.mma into one of TWO TMEM accumulators, so the
//               epilogue of tile i overlaps the mainloop of tile i+1
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: TMEM -> regs -> cvt(+relu) -> swizzled smem -> TMA store;
//               re-arms the drained accumulator with the bias of tile i+2
//   warps 8-15  producers: A (tiled / im2col / gathered / fp32 stem / residual), B
#include <cstdlib>
#include <mutex>

#include "ub_common.cuh"
#include "ub_host.h"

namespace ub {

enum AMode : int { A_TILED = 0, A_IM2COL = 1, A_GATHER = 2, A_STEM = 3, A_PACKED = 4 };
// A_PACKED: im2col for small-channel k x k convs -- several taps share one 64-wide k-block
// (cpad per tap 8/16/32), so every operand row is a full 128-byte SWIZZLE_128B row.
// register-path producers (2-byte gathers, fp32 casts) arrive explicitly per warp as well
__host__ __device__ constexpr bool reg_mode(int m) { return m == A_GATHER || m == A_STEM; }

constexpr int BLOCK_M = 128;
// Producer warp count is a template parameter (256 or 512 threads): cp.async throughput scales
// with issuing warps, but more warps also take issue slots and registers from the epilogue, so
// the engine autotunes it per layer (ConvDesc.variant).
constexpr int EPI_CHUNK = 64;                 // output channels per epilogue chunk (128-byte rows)
constexpr int EPI_SLOT = 32 * EPI_CHUNK * 2;  // one warp's 32 rows x 64 ch bf16 (4 KB)
constexpr int EPI_WARP_BYTES = 2 * EPI_SLOT;  // two output slots per epilogue warp
constexpr int Y2_PITCH = EPI_CHUNK + 8;        // compacted-store staging row (halves; 144 B: conflict-free)
constexpr int Y2_STAGE = 32 * Y2_PITCH * 2;    // per epilogue warp
constexpr int IDENT_BYTES = 64 * 128;         // 64x64 bf16 identity (SWIZZLE_128B, K-major)
constexpr int MAX_BLOCK_N = 256;
constexpr int BAR_BYTES = 512;   // mbarriers + TMEM slot region
constexpr int MAX_STEM_K = 512;  // dense-K stem: taps * channels, padded to 64

struct ConvKParams {
  int M;        // output pixels (GEMM M)
  int cout;     // output channels (GEMM N)
  int block_n;  // N tile
  int num_kb;   // main k-blocks per tile
  int cchunks;  // channel chunks per tap
  int kw;       // filter width
  int cpad;     // per-tap weight K
  int K_total;  // weight row length
  int cin_eff;  // channels readable in the A source (slice length + lead)
  int H, W, Ho, Wo, stride, pad;
  int stages;
  int m_tiles, n_tiles;
  uint32_t tmem_cols, acc_stride;
  const uint16_t* x;  // A source (bf16 NHWC), offset to the 8-aligned slice base / gather base
  int x_cstride;
  const uint16_t* w;  // B: bf16 [cout][K_total]
  // fused gather
  const int32_t* gidx;
  int n_gather;
  // fused stem: fp32 NCHW model input, dense K = taps * n_gather
  const float* xf;
  int C_in, k_real;
  int taps, tpk;  // A_PACKED: filter taps, taps per k-block
  // epilogue
  const float* bias;
  int has_res, relu, epi_tma;
  const uint16_t* res;  // residual, offset to its channel base
  int res_cstride;
  void* y;  // direct-store fallback only
  int y_cstride, y_coff, y_f32;
  int dbg;  // ablation bits for profiling (UB_DEBUG_FLAGS): 1 no store, 2 no epilogue math, 4 no MMA,
            // 8 no streamed weight loads
  int b_res;  // weights of this CTA's N tile stay resident in smem (loaded once; grid % n_tiles == 0)
  long long* trace;  // profiling (UB_CONV_TRACE): CTA 0 per-tile event clocks [tile][8]
  int b_tma;         // per-k-block weights by TMA (one box per stage) instead of cp.async
  int a_tma;         // tiled mode: A and residual k-blocks by TMA too (one producer thread)
  int epi2;          // (a_tma only) idle producer warps 12-15 form a second epilogue group
  uint16_t* y2;           // compacted second store (ub_conv_desc.y2) or null
  int y2_cstride;
  const int32_t* y2_map;  // [cout] compact column of output channel c, -1 = not stored
  int tail_w;        // (a_tma, BK 64) channels of the narrower last A box (16 / 32), 64 = none
  int epi_alt;       // (epi2, one 64-channel chunk per tile) the groups take alternate tiles
  int epi4;          // (epi2, 512 producers, generic activation) warps 12-23 too: four epilogue
                     // groups of four, one output slot per warp
                     // (group g drains accumulator g) instead of alternate chunks
  int mt2;           // (a_tma, streamed B, no residual) pairs of M-adjacent tiles share each B box:
                     // 4 TMEM accumulators, the pair's second A box in the next ring stage
};

// Tile of a CTA's it-th step, -1 past its last.  Default: tiles blockIdx.x + it * gridDim.x.
// Pair mode (p.mt2): units u = blockIdx.x + (it / 2) * gridDim.x of two M tiles (2 * (u / n_tiles)
// and the next) with the same N tile; the half past m_tiles (odd m_tiles) ends the walk.
__device__ __forceinline__ int tile_at(const ConvKParams& p, int it, int num_tiles) {
  if (!p.mt2) {
    const int t = blockIdx.x + it * gridDim.x;
    return t < num_tiles ? t : -1;
  }
  const int u = blockIdx.x + (it >> 1) * gridDim.x;
  const int mp = u / p.n_tiles;
  const int m_tile = 2 * mp + (it & 1);
  return m_tile < p.m_tiles ? m_tile * p.n_tiles + (u - mp * p.n_tiles) : -1;
}
#define UB_TRACE(slot)                                                                  \
  do {                                                                                  \
    if (p.trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0 && it < 64) p.trace[it * 8 + (slot)] = clock64(); \
  } while (0)

// Align the dynamic smem base to 1024 B by pointer arithmetic on the __shared__ pointer itself
// (a round trip through uintptr_t would make every derived pointer generic and turn all
// shared-memory accesses into generic LD/ST).
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

// Byte offset of 16-byte chunk j of row r in a swizzled K-major tile with BK-element rows
// (SWIZZLE_128B / 64B / 32B: the chunk index is XORed with address bits [7, 10)).
template <int BK>
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t j) {
  if constexpr (BK == 64) return r * 128 + ((j ^ (r & 7)) << 4);
  else if constexpr (BK == 32) return r * 64 + ((j ^ ((r >> 1) & 3)) << 4);
  else return r * 32 + ((j ^ ((r >> 2) & 1)) << 4);
}

__device__ __forceinline__ int tile_res_chunks(const ConvKParams& p, int n0) {
  return p.has_res ? (min(p.block_n, p.cout - n0) + EPI_CHUNK - 1) / EPI_CHUNK : 0;
}

// XACT: the epilogue applies a UB_ACT_* activation other than ReLU (hardswish, SiLU, ...).
// A separate instantiation, so the ReLU / identity epilogue of the ResNet path keeps its
// compact code (folding the generic activation into one kernel cost ~8 % on ResNet-50).
template <int AMODE, int BK, int PRODUCERS, bool XACT>
__global__ void __launch_bounds__(256 + PRODUCERS, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmR,
                   const __grid_constant__ CUtensorMap tmAt, const ConvKParams p) {
  constexpr int PWARPS = PRODUCERS / 32;
  constexpr int GROWS = BLOCK_M / PWARPS;       // gather mode: rows per producer warp
  constexpr int STEM_K = 64 * 128 / PRODUCERS;  // stem mode: k values per producer thread per k-block
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr uint32_t ROW_BYTES = BK * 2;
  constexpr int CPR = ROW_BYTES / 16;  // 16-byte chunks per operand row
  // A stages are sized for max(BK, 64) columns: residual k-blocks are always 64 wide
  constexpr uint32_t A_BYTES = BLOCK_M * 128;
  constexpr uint32_t SBO = 8 * ROW_BYTES;
  constexpr uint32_t LAYOUT = (BK == 64) ? 2u : (BK == 32 ? 4u : 6u);  // SWIZZLE_128B / 64B / 32B
  const uint32_t b_bytes = static_cast<uint32_t>(p.block_n) * ROW_BYTES;
  const uint32_t b_stride = (b_bytes + 1023u) & ~1023u;
  const int stages = p.stages;

  uint8_t* sA = smem;
  uint8_t* sB = sA + stages * A_BYTES;  // per-stage B, or all k-blocks of B when resident
  uint8_t* sI = sB + (p.b_res ? p.num_kb : stages) * b_stride;  // identity 64x64 (8 KB)
  // epilogue warps: 4, or 8 when the producers are idle (TMA-fed 1x1): group 1 = warps 12-15
  const int epi_warps = p.epi4 ? 16 : (p.epi2 ? 8 : 4);
  const uint32_t warp_bytes = p.epi4 ? EPI_SLOT : EPI_WARP_BYTES;  // output slots per epilogue warp: 1 or 2
  uint8_t* sE = sI + IDENT_BYTES;                                      // epi_warps x warp_bytes
  float* sBias = reinterpret_cast<float*>(sE + epi_warps * warp_bytes);  // epi_warps x MAX_BLOCK_N
  uint16_t* sY2 = reinterpret_cast<uint16_t*>(sBias + epi_warps * MAX_BLOCK_N);  // y2 staging (when set)
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sY2) + (p.y2 ? epi_warps * Y2_STAGE : 0));
  uint64_t* empty = full + stages;
  uint64_t* tfull = empty + stages;  // [4] (2 used unless pair mode)
  uint64_t* tempty = tfull + 4;      // [4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 4);
  uint64_t* bres = tempty + 5;  // resident B landed (PRODUCERS cp.async arrivals)
  const int nacc = p.mt2 ? 4 : 2;  // TMEM accumulators
  const int acc_sh = p.mt2 ? 2 : 1;  // log2(nacc)
  int4* stem_tab = reinterpret_cast<int4*>(reinterpret_cast<uint8_t*>(full) + BAR_BYTES);  // A_STEM / A_PACKED

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = p.m_tiles * p.n_tiles;
  const int nk = p.num_kb;

  if (warp == 0 && lane == 0) {
    if (p.epi_tma) tma_prefetch_desc(&tmY);
    if (p.b_tma || p.a_tma) tma_prefetch_desc(&tmB);
    if (p.a_tma) {
      tma_prefetch_desc(&tmA);
      if (p.has_res) tma_prefetch_desc(&tmR);
    }
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], p.a_tma ? 1 : PRODUCERS + (reg_mode(AMODE) ? PWARPS : 0) + (p.b_tma ? 1 : 0));
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < nacc; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], p.epi_alt ? 4 : epi_warps);
    }
    mbar_init(bres, p.a_tma ? 1 : PRODUCERS);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, p.tmem_cols);
  if (warp == 3) {  // identity B operand for the residual k-blocks: row n has 1.0 in column n
    for (int i = lane; i < IDENT_BYTES / 16; i += 32) {
      const int r = i >> 3, j = i & 7;
      uint4 v = make_uint4(0, 0, 0, 0);
      if ((r >> 3) == j) {
        const uint32_t one = 0x3F80u << (16 * (r & 1));  // bf16 1.0 in the right half
        const int word = (r & 7) >> 1;
        if (word == 0) v.x = one;
        else if (word == 1) v.y = one;
        else if (word == 2) v.z = one;
        else v.w = one;
      }
      *reinterpret_cast<uint4*>(sI + swz<64>(r, j)) = v;
    }
    fence_proxy_async_smem();
  }
  if constexpr (AMODE == A_PACKED) {  // tap -> (filter row, filter col, element offset in the input)
    for (int t = threadIdx.x; t < p.taps; t += blockDim.x) {
      const int r = t / p.kw, c = t - (t / p.kw) * p.kw;
      stem_tab[t] = make_int4(r, c, (r * p.W + c) * p.x_cstride, 0);
    }
  }
  if constexpr (AMODE == A_STEM) {
    // k -> (input offset relative to the window origin, filter row r, filter col s); k >= k_real: r = -1
    for (int k = threadIdx.x; k < p.num_kb * 64; k += blockDim.x) {
      int4 e = make_int4(0, -1, 0, 0);
      if (k < p.k_real) {
        const int t = k / p.n_gather;
        const int c = k - t * p.n_gather;
        const int r = t / p.kw;
        const int sc = t - r * p.kw;
        e = make_int4((__ldg(p.gidx + c) * p.H + r) * p.W + sc, r, sc, 0);
      }
      stem_tab[k] = e;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();  // the next kernel may start its prologue as SMs free up

  if (warp == 1) {
    {
      // ================= MMA issuer (accumulators arrive pre-loaded with the bias); the whole
      // warp runs the loop and one elected lane issues (umma_*_warp)
      const uint32_t idesc = make_idesc_bf16(BLOCK_M, static_cast<uint32_t>(p.block_n));
      const uint32_t idesc_res = make_idesc_bf16(BLOCK_M, EPI_CHUNK);
      const uint32_t i_base = smem_u32(sI);
      int s = 0, it = 0;
      uint32_t ph = 0;
      if (p.b_res) mbar_wait(bres, 0);
      if (p.mt2) {
        // pair mode: per k-block, stage s holds A of the first tile + the shared B box, stage
        // s + 1 the second tile's A; both MMAs read B from stage s
        for (;; it += 2) {
          const int t0 = tile_at(p, it, num_tiles);
          if (t0 < 0) break;
          const bool two = tile_at(p, it + 1, num_tiles) >= 0;
          const int acc0 = it & 3, acc1 = (it + 1) & 3;
          mbar_wait(&tempty[acc0], (it >> 2) & 1);
          if (two) mbar_wait(&tempty[acc1], ((it + 1) >> 2) & 1);
          __syncwarp();
          tc_fence_after();
          const uint32_t d0 = tmem_base + acc0 * p.acc_stride, d1 = tmem_base + acc1 * p.acc_stride;
          for (int kb = 0; kb < nk; ++kb) {
            const int s0 = s;
            mbar_wait(&full[s0], ph);
            if (++s == stages) {
              s = 0;
              ph ^= 1;
            }
            int s1 = -1;
            if (two) {
              s1 = s;
              mbar_wait(&full[s1], ph);
              if (++s == stages) {
                s = 0;
                ph ^= 1;
              }
            }
            __syncwarp();
            tc_fence_after();
            const uint32_t b_base = smem_u32(sB + s0 * b_stride);
            const bool tail = BK == 64 && kb == nk - 1 && p.tail_w < 64;
            const uint32_t a_lay = tail ? (p.tail_w == 16 ? 6u : 4u) : LAYOUT;
            const uint32_t a_sbo = tail ? 8u * p.tail_w * 2 : SBO;
            const int ksteps = tail ? p.tail_w / 16 : BK / 16;
            // the first tile's k-steps, then the second's (interleaving the two accumulators
            // per k-step gave wrong columns 1.. on B200 -- measured, tools/pair_debug.py)
            for (int k = 0; k < ksteps; ++k)
              umma_bf16_warp(d0, make_sdesc(smem_u32(sA + s0 * A_BYTES) + k * 32, a_sbo, a_lay),
                             make_sdesc(b_base + k * 32, SBO, LAYOUT), idesc, 1u);
            if (two)
              for (int k = 0; k < ksteps; ++k)
                umma_bf16_warp(d1, make_sdesc(smem_u32(sA + s1 * A_BYTES) + k * 32, a_sbo, a_lay),
                               make_sdesc(b_base + k * 32, SBO, LAYOUT), idesc, 1u);
            umma_commit_warp(&empty[s0]);
            if (two) umma_commit_warp(&empty[s1]);
          }
          umma_commit_warp(&tfull[acc0]);
          if (two) umma_commit_warp(&tfull[acc1]);
        }
      } else
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const int n0 = (t % p.n_tiles) * p.block_n;
        const int nres = tile_res_chunks(p, n0);
        UB_TRACE(0);
        mbar_wait(&tempty[acc], (it >> 1) & 1);  // drained and re-armed with this tile's bias
        UB_TRACE(1);
        __syncwarp();
        tc_fence_after();
        const uint32_t d = tmem_base + acc * p.acc_stride;
        for (int kb = 0; kb < nk + nres; ++kb) {
          mbar_wait(&full[s], ph);
          __syncwarp();
          tc_fence_after();
          // generic-proxy (cp.async / st.shared) writes -> tensor-core reads; the TMA-fed path
          // (A, B, residual all async-proxy writes) needs no proxy fence per k-block
          if (!p.a_tma) fence_proxy_async_smem();
          const uint32_t a_base = smem_u32(sA + s * A_BYTES);
          if (!(p.dbg & 4)) {
            if (kb < nk) {
              const uint32_t b_base = smem_u32(sB + (p.b_res ? kb : s) * b_stride);
              if (BK == 64 && kb == nk - 1 && p.tail_w < 64) {
                // narrower last A box: rows of tail_w channels (SWIZZLE_32B / 64B), the same B box
                const uint32_t t_layout = p.tail_w == 16 ? 6u : 4u, t_sbo = 8u * p.tail_w * 2;
                for (int k = 0; k < p.tail_w / 16; ++k)
                  umma_bf16_warp(d, make_sdesc(a_base + k * 32, t_sbo, t_layout), make_sdesc(b_base + k * 32, SBO, LAYOUT),
                                 idesc, 1u);
              } else {
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                umma_bf16_warp(d, make_sdesc(a_base + k * 32, SBO, LAYOUT), make_sdesc(b_base + k * 32, SBO, LAYOUT),
                          idesc, 1u);
              }
            } else {  // residual chunk rc: D[:, rc*64 : rc*64+64] += R_rc * I
              const uint32_t dc = d + (kb - nk) * EPI_CHUNK;
#pragma unroll
              for (int k = 0; k < 4; ++k)
                umma_bf16_warp(dc, make_sdesc(a_base + k * 32, 1024, 2), make_sdesc(i_base + k * 32, 1024, 2), idesc_res,
                          1u);
            }
          }
          umma_commit_warp(&empty[s]);
          if (++s == stages) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit_warp(&tfull[acc]);
        UB_TRACE(2);
      }
    }
  } else if (warp >= 8 && !(p.epi2 && warp >= 12 && warp < 16) && !(p.epi4 && warp >= 16)) {
    // ================= producers (256 threads): fill stage s with A and B, then arrive on full[s]
    // Addresses are precomputed per tile so the per-k-block work is one add + one cp.async per
    // 16-byte chunk; smem destinations are constant for the whole kernel.
    const int pt = threadIdx.x - 256;  // 0..PRODUCERS-1
    const int pw = pt >> 5;            // producer warp 0..PWARPS-1
    const int hw = p.Ho * p.Wo;
    // cp.async modes: this thread owns A rows row0 + i * ROW_STEP (i < A_PER_THREAD), chunk cj;
    // with fewer chunks than threads (BK 16) the upper threads own none
    constexpr int A_PIECES = BLOCK_M * CPR;
    constexpr int A_PER_THREAD = A_PIECES >= PRODUCERS ? A_PIECES / PRODUCERS : 1;
    constexpr int ROW_STEP = PRODUCERS / CPR;                // rows between a thread's chunks
    const bool a_owner = pt < A_PIECES;
    const int row0 = pt / CPR;
    const int cj = pt % CPR;  // this thread's 16-byte chunk within an operand row
    const uint32_t dst0 = swz<BK>(row0, cj);  // + i * ROW_STEP * ROW_BYTES for chunk i (swizzle-invariant)
    const int nb_pieces = (p.block_n + ROW_STEP - 1) / ROW_STEP;  // B chunks per thread (upper bound)
    const size_t b_row_stride = static_cast<size_t>(ROW_STEP) * p.K_total;
    // residual k-blocks: 64-channel rows; this thread owns rows pt/8 + 32 i, chunk pt%8
    constexpr int R_PER_THREAD = BLOCK_M * 8 / PRODUCERS;  // residual 16-byte chunks per thread
    const int rrow0 = pt >> 3, rj = pt & 7;
    const uint32_t rdst0 = swz<64>(rrow0, rj);
    int s = 0;
    uint32_t ph = 0;
    if (p.b_res && p.a_tma) {  // all k-blocks of this CTA's N tile, once, as TMA boxes
      if (pt == 0) {
        const int n0 = (blockIdx.x % p.n_tiles) * p.block_n;
        mbar_arrive_expect_tx(bres, static_cast<uint32_t>(nk) * p.block_n * ROW_BYTES);
        for (int kb = 0; kb < nk; ++kb) tma_load_2d(&tmB, bres, sB + kb * b_stride, kb * BK, n0);
      }
    } else if (p.b_res) {  // all k-blocks of this CTA's N tile, once
      const int n0 = (blockIdx.x % p.n_tiles) * p.block_n;
      const int b_valid = min(p.block_n, p.cout - n0);
      const uint16_t* b_base = p.w + static_cast<size_t>(n0 + row0) * p.K_total + cj * 8;
      for (int kb = 0; kb < nk; ++kb) {
        const int kcoord = kb * BK;
        const uint32_t tileB = smem_u32(sB + kb * b_stride);
        const uint16_t* src = b_base + kcoord;
        const bool k_ok = AMODE != A_PACKED || kcoord + cj * 8 < p.K_total;
        for (int i = 0; i < nb_pieces; ++i, src += b_row_stride) {
          const int n = row0 + i * ROW_STEP;
          if (n >= p.block_n) break;
          const bool ok = n < b_valid && k_ok;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(tileB + dst0 + i * ROW_STEP * ROW_BYTES),
                       "l"(ok ? src : p.w), "r"(ok ? 16u : 0u)
                       : "memory");
        }
      }
      cp_async_arrive_noinc(bres);
    }
    griddep_wait();  // activations / residual come from the previous kernel (PDL)
    if (AMODE == A_TILED && p.a_tma) {
      // every operand of a 1x1/s1 tile is a TMA box: one thread issues A (BK ch x 128 px),
      // B (BK x block_n) and the residual chunks (64 ch x 128 px) per stage
      if (pt == 0 && p.mt2) {
        for (int it = 0;; it += 2) {
          const int t0 = tile_at(p, it, num_tiles);
          if (t0 < 0) break;
          const bool two = tile_at(p, it + 1, num_tiles) >= 0;
          const int m_tile = t0 / p.n_tiles;
          const int n0 = (t0 - m_tile * p.n_tiles) * p.block_n;
          const int m0 = m_tile * BLOCK_M;
          for (int kb = 0; kb < nk; ++kb) {
            const bool tail = kb == nk - 1 && p.tail_w < BK;
            const uint32_t a_bytes = BLOCK_M * (tail ? static_cast<uint32_t>(p.tail_w) * 2 : ROW_BYTES);
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], a_bytes + static_cast<uint32_t>(p.block_n) * ROW_BYTES);
            tma_load_2d(tail ? &tmAt : &tmA, &full[s], sA + s * A_BYTES, kb * BK, m0);
            tma_load_2d(&tmB, &full[s], sB + s * b_stride, kb * BK, n0);
            if (++s == stages) {
              s = 0;
              ph ^= 1;
            }
            if (two) {
              mbar_wait(&empty[s], ph ^ 1);
              mbar_arrive_expect_tx(&full[s], a_bytes);
              tma_load_2d(tail ? &tmAt : &tmA, &full[s], sA + s * A_BYTES, kb * BK, m0 + BLOCK_M);
              if (++s == stages) {
                s = 0;
                ph ^= 1;
              }
            }
          }
        }
      } else if (pt == 0) {
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
          const int m_tile = t / p.n_tiles;
          const int n0 = (t - m_tile * p.n_tiles) * p.block_n;
          const int m0 = m_tile * BLOCK_M;
          const int nres = tile_res_chunks(p, n0);
          for (int kb = 0; kb < nk; ++kb) {
            mbar_wait(&empty[s], ph ^ 1);
            const bool bload = p.b_tma && !(p.dbg & 8);
            const bool tail = kb == nk - 1 && p.tail_w < BK;  // only the channels the slice still needs
            const uint32_t a_bytes = BLOCK_M * (tail ? static_cast<uint32_t>(p.tail_w) * 2 : ROW_BYTES);
            const uint32_t bytes = a_bytes + (bload ? static_cast<uint32_t>(p.block_n) * ROW_BYTES : 0u);
            mbar_arrive_expect_tx(&full[s], bytes);
            tma_load_2d(tail ? &tmAt : &tmA, &full[s], sA + s * A_BYTES, kb * BK, m0);
            if (bload) tma_load_2d(&tmB, &full[s], sB + s * b_stride, kb * BK, n0);
            if (++s == stages) {
              s = 0;
              ph ^= 1;
            }
          }
          for (int rc = 0; rc < nres; ++rc) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], BLOCK_M * 128);
            tma_load_2d(&tmR, &full[s], sA + s * A_BYTES, n0 + rc * EPI_CHUNK, m0);
            if (++s == stages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    } else
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const int it = (t - blockIdx.x) / gridDim.x;
      if (pt == 0) UB_TRACE(6);
      const int m_tile = t / p.n_tiles;
      const int n0 = (t - m_tile * p.n_tiles) * p.block_n;
      const int m0 = m_tile * BLOCK_M;
      const int nres = tile_res_chunks(p, n0);
      // A geometry of this thread's rows: pixel base pointer + top-left window coordinate
      const uint16_t* a_base[A_PER_THREAD];
      int a_hb[A_PER_THREAD], a_wb[A_PER_THREAD];
#pragma unroll
      for (int i = 0; i < A_PER_THREAD; ++i) {
        const int m = m0 + row0 + i * ROW_STEP;
        a_base[i] = p.x;
        a_hb[i] = -(1 << 28);
        a_wb[i] = 0;
        if ((AMODE == A_TILED || AMODE == A_IM2COL || AMODE == A_PACKED) && m < p.M) {
          const int img = m / hw;
          const int rem = m - img * hw;
          const int ho = rem / p.Wo;
          a_hb[i] = ho * p.stride - p.pad;
          a_wb[i] = (rem - ho * p.Wo) * p.stride - p.pad;
          a_base[i] = p.x + ((static_cast<ptrdiff_t>(img) * p.H + a_hb[i]) * p.W + a_wb[i]) * p.x_cstride +
                      (AMODE == A_PACKED ? 0 : cj * 8);
        }
      }
      const uint16_t* b_base = p.w + static_cast<size_t>(n0 + row0) * p.K_total + cj * 8;
      const int b_valid = min(p.block_n, p.cout - n0);  // rows beyond are zero-filled
      // register-path geometry: gather -> warp pw owns rows 16*pw..16*pw+15 (lane = channel pair);
      // stem -> thread owns row pt & 127 and k slice pt >> 7
      int g_img = 0, g_hb = -(1 << 28), g_wb = 0;
      uint32_t s_rok = 0, s_cok = 0;  // stem: in-image filter rows / columns of this pixel's window
      const float* stem_base = p.xf;
      if constexpr (AMODE == A_GATHER) {
        if (lane < GROWS) {
          const int m = m0 + pw * GROWS + lane;
          if (m < p.M) {
            g_img = m / hw;
            const int rem = m - g_img * hw;
            const int ho = rem / p.Wo;
            g_hb = ho * p.stride - p.pad;
            g_wb = (rem - ho * p.Wo) * p.stride - p.pad;
          }
        }
      }
      if constexpr (AMODE == A_STEM) {
        const int m = m0 + (pt & 127);
        if (m < p.M) {
          const int img = m / hw;
          const int rem = m - img * hw;
          const int ho = rem / p.Wo;
          g_hb = ho * p.stride - p.pad;
          g_wb = (rem - ho * p.Wo) * p.stride - p.pad;
          for (int r = 0; r < p.kw; ++r) {
            s_rok |= static_cast<uint32_t>(g_hb + r >= 0 && g_hb + r < p.H) << r;
            s_cok |= static_cast<uint32_t>(g_wb + r >= 0 && g_wb + r < p.W) << r;
          }
          stem_base =
              p.xf + static_cast<size_t>(img) * p.C_in * p.H * p.W + static_cast<ptrdiff_t>(g_hb) * p.W + g_wb;
        }
      }
      int cc = 0, fs = 0, fr = 0;  // channel chunk, filter column, filter row of k-block kb
      for (int kb = 0; kb < nk; ++kb) {
        const int kcoord = kb * BK;  // weights are [cout][taps][cpad]: k-block kb starts at kb*BK
        // register paths: issue the global loads before waiting for the slot
        uint16_t la[GROWS], lb[GROWS];
        uint32_t okm = 0;
        int i0 = -1, i1 = -1;
        float fv[STEM_K];
        if constexpr (AMODE == A_GATHER) {
          const int j = cc * 64 + lane * 2;
          i0 = j < p.n_gather ? __ldg(p.gidx + j) : -1;
          i1 = (j + 1) < p.n_gather ? __ldg(p.gidx + j + 1) : -1;
          const int c0 = i0 < 0 ? 0 : i0;
          const int c1 = i1 < 0 ? 0 : i1;
#pragma unroll
          for (int u = 0; u < GROWS; ++u) {
            const int img = __shfl_sync(0xffffffffu, g_img, u);
            const int hi = __shfl_sync(0xffffffffu, g_hb, u) + fr;
            const int wi = __shfl_sync(0xffffffffu, g_wb, u) + fs;
            const bool ok = hi >= 0 && hi < p.H && wi >= 0 && wi < p.W;
            okm |= static_cast<uint32_t>(ok) << u;
            const size_t pix = ok ? (static_cast<size_t>(img) * p.H + hi) * p.W + wi : 0;
            const uint16_t* xr = p.x + pix * p.x_cstride;
            la[u] = __ldg(xr + c0);
            lb[u] = __ldg(xr + c1);
          }
        }
        if constexpr (AMODE == A_STEM) {
          const int kh0 = kb * 64 + (pt >> 7) * STEM_K;
#pragma unroll
          for (int kk = 0; kk < STEM_K; ++kk) {
            const int4 e = stem_tab[kh0 + kk];  // warp-uniform -> smem broadcast; e.y = -1 past k_real
            const bool ok = ((s_rok >> (e.y & 31)) & (s_cok >> e.z) & 1u) && e.y >= 0;
            fv[kk] = ok ? __ldg(stem_base + e.x) : 0.f;
          }
        }
        mbar_wait(&empty[s], ph ^ 1);
        const uint32_t tileA = smem_u32(sA + s * A_BYTES);
        const uint32_t tileB = smem_u32(sB + s * b_stride);
        // ---- A
        if constexpr (AMODE == A_PACKED) {
          const int cpt8 = p.cpad >> 3;  // 16-byte chunks per tap
          const int tap = kb * p.tpk + cj / cpt8;
          const int cjt = cj - (cj / cpt8) * cpt8;
          const int4 te = stem_tab[tap < p.taps ? tap : 0];
          const bool tap_ok = tap < p.taps && cjt * 8 < p.cin_eff;
#pragma unroll
          for (int i = 0; i < A_PER_THREAD; ++i) {
            const int hi = a_hb[i] + te.x;
            const int wi = a_wb[i] + te.y;
            const bool ok = tap_ok && hi >= 0 && hi < p.H && wi >= 0 && wi < p.W;
            const uint16_t* src = ok ? a_base[i] + te.z + cjt * 8 : p.x;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(tileA + dst0 + i * ROW_STEP * ROW_BYTES),
                         "l"(src), "r"(ok ? 16u : 0u)
                         : "memory");
          }
        } else if constexpr (AMODE == A_TILED || AMODE == A_IM2COL) {
          const bool ch_ok = cc * BK + cj * 8 < p.cin_eff;
          const ptrdiff_t toff = (static_cast<ptrdiff_t>(fr) * p.W + fs) * p.x_cstride + cc * BK;
#pragma unroll
          for (int i = 0; i < A_PER_THREAD; ++i) {
            if (!a_owner) break;
            const int hi = a_hb[i] + fr;
            const int wi = a_wb[i] + fs;
            const bool ok = ch_ok && hi >= 0 && hi < p.H && wi >= 0 && wi < p.W;
            const uint16_t* src = ok ? a_base[i] + toff : p.x;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(tileA + dst0 + i * ROW_STEP * ROW_BYTES),
                         "l"(src), "r"(ok ? 16u : 0u)
                         : "memory");
          }
        } else if constexpr (AMODE == A_GATHER) {
          uint8_t* tA = sA + s * A_BYTES;
#pragma unroll
          for (int u = 0; u < GROWS; ++u) {
            const bool ok = (okm >> u) & 1u;
            const uint32_t a = (ok && i0 >= 0) ? la[u] : 0u;
            const uint32_t b = (ok && i1 >= 0) ? lb[u] : 0u;
            const int row = pw * GROWS + u;
            *reinterpret_cast<uint32_t*>(tA + swz<64>(row, lane >> 2) + ((lane & 3) << 2)) = a | (b << 16);
          }
        } else {  // A_STEM
          uint8_t* tA = sA + s * A_BYTES;
          const int row = pt & 127;
          const int j0 = (pt >> 7) * (STEM_K / 8);
#pragma unroll
          for (int jj = 0; jj < STEM_K / 8; ++jj) {
            uint4 o;
            o.x = pack_bf16x2(fv[jj * 8 + 0], fv[jj * 8 + 1]);
            o.y = pack_bf16x2(fv[jj * 8 + 2], fv[jj * 8 + 3]);
            o.z = pack_bf16x2(fv[jj * 8 + 4], fv[jj * 8 + 5]);
            o.w = pack_bf16x2(fv[jj * 8 + 6], fv[jj * 8 + 7]);
            *reinterpret_cast<uint4*>(tA + swz<64>(row, j0 + jj)) = o;
          }
        }
        // ---- B (weights [cout][K_total]): one TMA box, or rows row0 + i * ROW_STEP, chunk cj
        if (p.b_tma) {
          if (pt == 0) {
            if (p.dbg & 8) {  // profiling: weights not loaded (timing only)
              mbar_arrive(&full[s]);
            } else {
              mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(p.block_n) * ROW_BYTES);
              tma_load_2d(&tmB, &full[s], sB + s * b_stride, kcoord, n0);
            }
          }
        } else if (!p.b_res) {
          const uint16_t* src = b_base + kcoord;
          const bool k_ok = AMODE != A_PACKED || kcoord + cj * 8 < p.K_total;  // packed: last k-block ragged
          for (int i = 0; i < nb_pieces; ++i, src += b_row_stride) {
            const int n = row0 + i * ROW_STEP;
            if (n >= p.block_n) break;
            const bool ok = n < b_valid && k_ok;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(tileB + dst0 + i * ROW_STEP * ROW_BYTES),
                         "l"(ok ? src : p.w), "r"(ok ? 16u : 0u)
                         : "memory");
          }
        }
        if constexpr (reg_mode(AMODE)) {  // st.shared part: fence, then one arrival per warp
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[s]);
        }
        cp_async_arrive_noinc(&full[s]);
        if (++s == stages) {
          s = 0;
          ph ^= 1;
        }
        if (++cc == p.cchunks) {
          cc = 0;
          if (++fs == p.kw) {
            fs = 0;
            ++fr;
          }
        }
      }
      // ---- residual k-blocks: A = residual[m0 : m0+128, n0 + rc*64 : +64], B = identity
      for (int rc = 0; rc < nres; ++rc) {
        mbar_wait(&empty[s], ph ^ 1);
        const uint32_t tileA = smem_u32(sA + s * A_BYTES);
        const int ch = n0 + rc * EPI_CHUNK + rj * 8;
#pragma unroll
        for (int i = 0; i < R_PER_THREAD; ++i) {
          const int m = m0 + rrow0 + (PRODUCERS / 8) * i;
          const bool ok = m < p.M && ch < p.cout;
          const uint16_t* src = ok ? p.res + static_cast<size_t>(m) * p.res_cstride + ch : p.res;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(tileA + rdst0 + i * (PRODUCERS / 8) * 128), "l"(src),
                       "r"(ok ? 16u : 0u)
                       : "memory");
        }
        if constexpr (reg_mode(AMODE)) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[s]);
        }
        if (p.b_tma && pt == 0) mbar_arrive(&full[s]);  // no weight box in a residual k-block
        cp_async_arrive_noinc(&full[s]);
        if (++s == stages) {
          s = 0;
          ph ^= 1;
        }
      }
      if (pt == 0) UB_TRACE(7);
    }
    cp_async_wait<0>();
  } else if (warp >= 4) {
    // ================= epilogue
    // Warp q owns TMEM lanes / tile rows q*32..q*32+31 and walks 64-channel chunks (with two
    // groups: group eg takes the chunks c % 2 == eg).  After draining a 32-column half it
    // re-arms those accumulator columns with the bias of the tile that uses this
    // accumulator next (tile i+2).
    const int q = warp & 3;  // TMEM lane quarter (warp % 4)
    const int eg = warp < 8 ? 0 : (warp - 8) >> 2;  // warps 4-7: 0; 12-15: 1; 16-19: 2; 20-23: 3
    const int ngrp = epi_warps / 4;
    const int ew = eg * 4 + q;  // epilogue warp index: slots and bias buffer
    uint8_t* oslots = sE + ew * warp_bytes;
    float* sb = sBias + ew * MAX_BLOCK_N;
    const bool tma = p.epi_tma;
    uint32_t ec = 0;  // chunks processed by this warp (= TMA stores committed)
    // bias of tile tt -> sb (zero past cout), columns [0, width)
    auto stage_bias = [&](int tt) {
      const int nn0 = (tt % p.n_tiles) * p.block_n;
      const int width = static_cast<int>(p.acc_stride);
      __syncwarp();
      for (int i = lane; i < width; i += 32)
        sb[i] = (p.bias && i < p.block_n && nn0 + i < p.cout) ? __ldg(p.bias + nn0 + i) : 0.f;
      __syncwarp();
    };
    // write sb[col0 .. col0+32) into TMEM columns (all 32 lanes of this warp's quarter)
    auto arm32 = [&](uint32_t taddr, int col0) {
      uint32_t bv[32];
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const float4 f = *reinterpret_cast<const float4*>(sb + col0 + i);
        bv[i] = __float_as_uint(f.x);
        bv[i + 1] = __float_as_uint(f.y);
        bv[i + 2] = __float_as_uint(f.z);
        bv[i + 3] = __float_as_uint(f.w);
      }
      tmem_st32(taddr, bv);
    };
    // initial arming of the accumulators (the CTA's first nacc tiles)
    for (int a = 0; a < nacc; ++a) {
      if (p.epi_alt && (a & 1) != eg) continue;
      const int tt = tile_at(p, a, num_tiles);
      if (tt >= 0) {
        stage_bias(tt);
        const uint32_t ta = tmem_base + a * p.acc_stride + (static_cast<uint32_t>(q * 32) << 16);
        for (int col = 0; col < static_cast<int>(p.acc_stride); col += 32)
          if (p.epi_alt || (col / EPI_CHUNK) % ngrp == eg) arm32(ta + col, col);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
    }
    int it = 0;
    const int c0 = p.epi_alt ? 0 : eg, cstep = p.epi_alt ? 1 : ngrp;  // this warp's chunks of a tile
    for (;; ++it) {
      const int t = tile_at(p, it, num_tiles);
      if (t < 0) break;
      if (p.epi_alt && (it & 1) != eg) continue;
      const int m_tile = t / p.n_tiles;
      const int n0 = (t - m_tile * p.n_tiles) * p.block_n;
      const int m0 = m_tile * BLOCK_M;
      const int rows0 = m0 + q * 32;
      const int ncols = min(p.block_n, p.cout - n0);
      const int nchunks = (ncols + EPI_CHUNK - 1) / EPI_CHUNK;
      const int t_next = tile_at(p, it + nacc, num_tiles);  // next user of this accumulator
      const bool rearm = t_next >= 0;
      if (rearm && p.n_tiles > 1) stage_bias(t_next);  // (one N tile: every tile's bias is the same)
      const int acc = it & (nacc - 1);
      if (ew == 0) UB_TRACE(3);
      mbar_wait(&tfull[acc], (it >> acc_sh) & 1);
      if (ew == 0) UB_TRACE(4);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * p.acc_stride + (static_cast<uint32_t>(q * 32) << 16);
      for (int c = c0; c < nchunks; c += cstep, ++ec) {
        uint8_t* oslot = oslots + (p.epi4 ? 0 : (ec & 1) * EPI_SLOT);
        if (tma && lane == 0) {  // this slot's previous store (2 chunks ago; 1 with one slot) has read it
          if (p.epi4) bulk_wait_read<0>();
          else bulk_wait_read<1>();
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // two 32-column halves
          const int col = c * EPI_CHUNK + h * 32;
          if (col >= ncols) {  // past cout: nothing to store (the TMA store clips these channels)
            if (rearm) arm32(taddr + col, col);
            continue;
          }
          uint32_t r[32];
          tmem_ld32(taddr + col, r);
          tmem_ld_wait();
          if (rearm) arm32(taddr + col, col);
          if (tma) {
            if (!(p.dbg & 2)) {
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                uint4 o;
                const float* f = reinterpret_cast<const float*>(r) + jj * 8;
                if (XACT) {  // other UB_ACT_* activations (hardswish, SiLU, ...)
                  o = act_pack8(p.relu, f[0], f[1], f[2], f[3], f[4], f[5], f[6], f[7]);
                } else if (p.relu) {
                  o.x = cvt_relu_bf16x2(f[0], f[1]);
                  o.y = cvt_relu_bf16x2(f[2], f[3]);
                  o.z = cvt_relu_bf16x2(f[4], f[5]);
                  o.w = cvt_relu_bf16x2(f[6], f[7]);
                } else {
                  o.x = cvt_bf16x2(f[0], f[1]);
                  o.y = cvt_bf16x2(f[2], f[3]);
                  o.z = cvt_bf16x2(f[4], f[5]);
                  o.w = cvt_bf16x2(f[6], f[7]);
                }
                *reinterpret_cast<uint4*>(oslot + swz<64>(lane, h * 4 + jj)) = o;
              }
            }
          } else {
            // direct-store fallback (fp32 logits / unaligned views); bias and residual are
            // already in the accumulator
            const int m = rows0 + lane;
            const int nb = n0 + col;
            const int nv = min(32, p.cout - nb);
            if (m < p.M && nv > 0) {
              float v[32];
#pragma unroll
              for (int i = 0; i < 32; ++i)
                v[i] = XACT ? act_f(__uint_as_float(r[i]), p.relu)
                            : (p.relu ? fmaxf(__uint_as_float(r[i]), 0.f) : __uint_as_float(r[i]));
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
        if (tma) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0 && !(p.dbg & 1)) {
            tma_store_2d(&tmY, oslot, n0 + c * EPI_CHUNK, rows0);
            bulk_commit();
          }
          if (p.y2) {
            // compacted copy.  The kept channels of a 64-channel chunk occupy consecutive y2
            // columns from an 8-aligned base (the caller's layout).  Phase 1 (lane = channel)
            // packs each row's kept values into a staging row; phase 2 (lane = row) writes the
            // row segment with 16-byte stores.
            const int ch = n0 + c * EPI_CHUNK + lane;
            const int pos0 = ch < p.cout ? __ldg(p.y2_map + ch) : -1;
            const int pos1 = ch + 32 < p.cout ? __ldg(p.y2_map + ch + 32) : -1;
            const uint32_t b0 = __ballot_sync(0xffffffffu, pos0 >= 0);
            const uint32_t b1 = __ballot_sync(0xffffffffu, pos1 >= 0);
            const int k = __popc(b0) + __popc(b1);
            if (k > 0) {
              const int base = b0 ? __shfl_sync(0xffffffffu, pos0, __ffs(b0) - 1)
                                  : __shfl_sync(0xffffffffu, pos1, __ffs(b1) - 1);
              const uint32_t lt = (1u << lane) - 1u;
              const int rank0 = __popc(b0 & lt), rank1 = __popc(b0) + __popc(b1 & lt);
              uint16_t* stg = sY2 + ew * (Y2_STAGE / 2);
              const uint32_t cb = (lane & 7) * 2;
#pragma unroll 4
              for (int r = 0; r < 32; ++r) {
                if (pos0 >= 0)
                  stg[r * Y2_PITCH + rank0] = *reinterpret_cast<const uint16_t*>(oslot + swz<64>(r, lane >> 3) + cb);
                if (pos1 >= 0)
                  stg[r * Y2_PITCH + rank1] =
                      *reinterpret_cast<const uint16_t*>(oslot + swz<64>(r, 4 + (lane >> 3)) + cb);
              }
              __syncwarp();
              const int m = rows0 + lane;
              if (m < p.M) {
                uint4* dst = reinterpret_cast<uint4*>(p.y2 + static_cast<size_t>(m) * p.y2_cstride + base);
                const uint4* src = reinterpret_cast<const uint4*>(stg + lane * Y2_PITCH);
                for (int g8 = 0; g8 * 8 < k; ++g8) {
                  uint4 v = src[g8];
                  const int valid = k - g8 * 8;  // zero the padding past the chunk's last kept channel
                  if (valid < 8) {
                    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                      if (2 * i >= valid) w[i] = 0u;
                      else if (2 * i + 1 >= valid) w[i] &= 0xffffu;
                    }
                    v = make_uint4(w[0], w[1], w[2], w[3]);
                  }
                  dst[g8] = v;
                }
              }
              __syncwarp();
            }
          }
        }
      }
      // re-arm the columns past this tile's last chunk (the next user may be wider)
      if (rearm)
        for (int col = nchunks * EPI_CHUNK; col < static_cast<int>(p.acc_stride); col += 32)
          if (p.epi_alt || (col / EPI_CHUNK) % ngrp == eg) arm32(taddr + col, col);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);  // drained (and re-armed): the MMA may reuse it
      if (ew == 0) UB_TRACE(5);
    }
    if (tma && lane == 0) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, p.tmem_cols);
}

// ------------------------------------------------------------------ host side

int g_driver_version = -1;
long long* g_conv_trace = nullptr;

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


namespace {

template <int AMODE, int BK, int PRODUCERS>
int launch_conv_p(const CUtensorMap& tmY, const CUtensorMap& tmB, const CUtensorMap& tmA, const CUtensorMap& tmR,
                  const CUtensorMap& tmAt, const ConvKParams& p, int grid, size_t smem, cudaStream_t stream) {
  auto kern = p.relu > 1 ? conv_tc_kernel<AMODE, BK, PRODUCERS, true> : conv_tc_kernel<AMODE, BK, PRODUCERS, false>;
  const cudaError_t attr_err = ensure_max_smem(kern);
  if (attr_err != cudaSuccess) return cuda_status(attr_err, "cudaFuncSetAttribute(conv)");
  const cudaError_t e = launch_pdl(kern, dim3(grid), dim3(256 + PRODUCERS), smem, stream, tmY, tmB, tmA, tmR, tmAt, p);
  if (e != cudaSuccess) return cuda_status(e, "conv_tc_kernel launch");
  count_launch();
  return cuda_status(cudaGetLastError(), "conv_tc_kernel launch");
}

template <int AMODE, int BK>
int launch_conv(const CUtensorMap& tmY, const CUtensorMap& tmB, const CUtensorMap& tmA, const CUtensorMap& tmR,
                const CUtensorMap& tmAt, const ConvKParams& p, int grid, size_t smem, cudaStream_t stream, int wide) {
  return wide ? launch_conv_p<AMODE, BK, 512>(tmY, tmB, tmA, tmR, tmAt, p, grid, smem, stream)
              : launch_conv_p<AMODE, BK, 256>(tmY, tmB, tmA, tmR, tmAt, p, grid, smem, stream);
}

int pick_bk(int cin_eff) { return cin_eff <= 16 ? 16 : (cin_eff <= 32 ? 32 : 64); }

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

extern "C" int ub_conv_weight_layout2(int cin, int coff, int gather, int kh, int kw, int* lead, int* cpad) {
  if (cin < 1 || coff < 0 || kh < 1 || kw < 1 || !lead || !cpad)
    return fail(UB_EINVAL, "ub_conv_weight_layout2: bad arguments");
  const int ld = gather ? 0 : (coff & 7);
  const int ce = cin + ld;
  if (!gather && kh * kw > 1 && ce <= 32) {  // packed taps: per-tap K of 8/16/32
    *lead = ld;
    *cpad = ce <= 8 ? 8 : (ce <= 16 ? 16 : 32);
    return UB_OK;
  }
  return ub_conv_weight_layout(cin, coff, gather, lead, cpad);
}

extern "C" int ub_conv_stem_kpad(int cin, int kh, int kw) { return (kh * kw * cin + 63) / 64 * 64; }

// L2 sector promotion of the activation / residual maps.  A channel slice of a wider row (e.g.
// 128 of 240 channels) is not 256-byte aligned, and 256-byte promotion fetches the neighbouring
// slices too: 64 B there (measured 0.65 -> 0.86 of the HBM roofline for a 128-of-240 slice);
// rows read whole keep 256 B (better for them).  UB_A_PROMO (0 none, 1 64 B, 2 128 B, 3 256 B)
// overrides.
CUtensorMapL2promotion ub::a_promo(bool whole_rows) {
  static int v = -2;
  if (v == -2) v = getenv("UB_A_PROMO") ? atoi(getenv("UB_A_PROMO")) : -1;
  if (v >= 0) return static_cast<CUtensorMapL2promotion>(v);
  return whole_rows ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
}

extern "C" int ub_conv_fwd(const ub_conv_desc* d, cudaStream_t stream) {
  if (!d) return fail(UB_EINVAL, "ub_conv_fwd: null descriptor");
  if (!d->x || !d->w || !d->y) return fail(UB_EINVAL, "ub_conv_fwd: null x/w/y");
  if (d->N < 1 || d->H < 1 || d->W < 1 || d->cin < 1 || d->cout < 1 || d->kh < 1 || d->kw < 1 || d->stride < 1 ||
      d->pad < 0 || d->Ho < 1 || d->Wo < 1)
    return fail(UB_EINVAL, "ub_conv_fwd: bad geometry");
  if (d->Ho != (d->H + 2 * d->pad - d->kh) / d->stride + 1 || d->Wo != (d->W + 2 * d->pad - d->kw) / d->stride + 1)
    return fail(UB_EINVAL, "ub_conv_fwd: Ho/Wo inconsistent with kernel/stride/pad");
  if (!d->x_nchw_f32 &&
      (d->x_cstride % 8 || d->x_coff < 0 || (!d->gather_idx && d->x_coff + d->cin > d->x_cstride)))
    return fail(UB_EINVAL, "ub_conv_fwd: x channel stride must be a multiple of 8 and cover the read");
  if (!aligned16(d->x) || !aligned16(d->w) || !aligned16(d->y))
    return fail(UB_EINVAL, "ub_conv_fwd: x/w/y must be 16-byte aligned");
  if (d->y_dtype != UB_BF16 && d->y_dtype != UB_F32) return fail(UB_EINVAL, "ub_conv_fwd: y_dtype");
  if (d->y_coff < 0 || d->y_coff + d->cout > d->y_cstride)
    return fail(UB_EINVAL, "ub_conv_fwd: output channels exceed y_cstride");
  if (d->residual && (d->res_coff < 0 || d->res_coff + d->cout > d->res_cstride))
    return fail(UB_EINVAL, "ub_conv_fwd: residual channels exceed res_cstride");
  if (d->kh > 64 || d->kw > 64) return fail(UB_EUNSUPPORTED, "ub_conv_fwd: filter too large");

  const bool stem = d->x_nchw_f32 != 0;
  const bool gather = d->gather_idx != nullptr && !stem;
  if (gather && d->x_coff % 8) return fail(UB_EINVAL, "ub_conv_fwd: gather base must be 8-aligned");
  const int taps = d->kh * d->kw;

  int lead = 0, cpad = 0;
  if (stem) {
    if (!d->gather_idx || d->x_channels < 1 || d->x_coff != 0)
      return fail(UB_EINVAL, "ub_conv_fwd: stem mode needs gather_idx over x_channels input planes");
    cpad = ub_conv_stem_kpad(d->cin, d->kh, d->kw);
    if (cpad > MAX_STEM_K) return fail(UB_EUNSUPPORTED, "ub_conv_fwd: stem K %d > %d", cpad, MAX_STEM_K);
  } else {
    ub_conv_weight_layout2(d->cin, d->x_coff, gather ? 1 : 0, d->kh, d->kw, &lead, &cpad);
  }
  const bool packed = !stem && !gather && taps > 1 && cpad < 64;
  if (d->w_lead != lead || d->w_cpad != cpad)
    return fail(UB_EINVAL, "ub_conv_fwd: weight layout (lead %d, cpad %d) != expected (lead %d, cpad %d)", d->w_lead,
                d->w_cpad, lead, cpad);
  {  // stride-1 3x3 convs: halo-tile kernel when in scope
    bool handled = false;
    const int rc = conv_halo_fwd(d, lead, cpad, stream, &handled);
    if (rc != UB_OK || handled) return rc;
  }
  const int cin_eff = d->cin + lead;
  const int bk = (gather || stem || packed) ? 64 : pick_bk(cin_eff);

  ConvKParams p{};
  p.M = d->N * d->Ho * d->Wo;
  p.cout = d->cout;
  p.m_tiles = (p.M + BLOCK_M - 1) / BLOCK_M;
  // N tiling: the widest tile (<= 256) unless that leaves SMs idle; then split N into
  // more tiles until the grid fills.  Multi-tile N rounds to the epilogue's 64-channel
  // chunk so a tile's last chunk never spills into the next tile's channels (the TMA
  // store only clips at cout).
  // variant bit 13: N tiles of at most 128 channels (their weights may then stay resident)
  const int max_bn = (d->variant & 8192) ? 128 : MAX_BLOCK_N;
  // variant bit 16: 32-channel granularity for multi-tile N when the output is fp32 (direct
  // stores bounded by the tile's own columns, no 64-channel TMA box that could spill into the
  // next tile) and there is no residual -- the classifier: twice the CTAs share its weights
  const int multi_gran = ((d->variant & 65536) && d->y_dtype == UB_F32 && !d->residual) ? 32 : EPI_CHUNK;
  p.n_tiles = (d->cout + max_bn - 1) / max_bn;
  while (static_cast<long long>(p.m_tiles) * p.n_tiles < num_sms() &&
         (d->cout + p.n_tiles) / (p.n_tiles + 1) >= multi_gran)
    ++p.n_tiles;
  {
    const int n_gran = p.n_tiles > 1 ? multi_gran : 16;
    const int per_tile = (d->cout + p.n_tiles - 1) / p.n_tiles;
    p.block_n = (per_tile + n_gran - 1) / n_gran * n_gran;
    // rounding up can undo the split (fc 1000 / 15 tiles -> 67 -> 128 -> 8 tiles): while the
    // grid is still short of the SMs, round down instead (1000 -> 16 tiles of 64)
    if (p.n_tiles > 1 && per_tile >= n_gran &&
        static_cast<long long>(p.m_tiles) * ((d->cout + p.block_n - 1) / p.block_n) < num_sms())
      p.block_n = per_tile / n_gran * n_gran;
    if (p.block_n > max_bn) p.block_n = max_bn;
    p.n_tiles = (d->cout + p.block_n - 1) / p.block_n;
  }
  p.cchunks = (stem || packed) ? 1 : cpad / bk;
  p.taps = taps;
  p.tpk = packed ? 64 / cpad : 1;
  p.num_kb = stem ? cpad / 64 : (packed ? (taps + p.tpk - 1) / p.tpk : taps * p.cchunks);
  p.kw = d->kw;
  p.cpad = cpad;
  p.K_total = stem ? cpad : taps * cpad;
  p.cin_eff = cin_eff;
  p.H = d->H;
  p.W = d->W;
  p.Ho = d->Ho;
  p.Wo = d->Wo;
  p.stride = d->stride;
  p.pad = d->pad;
  // pair mode (variant bit 15): TMA-fed 1x1 without residual, N tiles <= 128 channels, streamed
  // weights -- two M tiles per B box halve the weight bytes each SM pulls from L2
  const bool tiled_1x1_mt = !stem && !packed && !gather && d->kh == 1 && d->kw == 1 && d->stride == 1 &&
                            d->pad == 0 && !(d->variant & 32);
  p.mt2 = (d->variant & 32768) && tiled_1x1_mt && !d->residual && !d->y2 && p.block_n <= 128 && p.m_tiles >= 2;
  // two accumulators (four in pair mode), each a whole number of 64-column epilogue chunks wide
  const uint32_t nacc = p.mt2 ? 4u : 2u;
  const uint32_t acc_cols = (static_cast<uint32_t>(p.block_n) + EPI_CHUNK - 1) / EPI_CHUNK * EPI_CHUNK;
  uint32_t tc = 32;
  while (tc < nacc * acc_cols) tc <<= 1;
  p.tmem_cols = tc;
  p.acc_stride = tc / nacc;
  p.x = stem ? nullptr : reinterpret_cast<const uint16_t*>(d->x) + (d->x_coff - lead);
  p.x_cstride = d->x_cstride;
  p.w = reinterpret_cast<const uint16_t*>(d->w);
  p.gidx = d->gather_idx;
  p.n_gather = (gather || stem) ? d->cin : 0;
  p.xf = stem ? static_cast<const float*>(d->x) : nullptr;
  p.C_in = stem ? d->x_channels : 0;
  p.k_real = stem ? taps * d->cin : 0;
  p.bias = d->bias;
  p.has_res = d->residual != nullptr;
  p.relu = d->relu;
  p.res = reinterpret_cast<const uint16_t*>(d->residual) + (d->residual ? d->res_coff : 0);
  p.res_cstride = d->res_cstride;
  p.y = d->y;
  p.y_cstride = d->y_cstride;
  p.y_coff = d->y_coff;
  p.y_f32 = d->y_dtype == UB_F32;
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* e = getenv("UB_DEBUG_FLAGS");
      dbg = e ? atoi(e) : 0;
    }
    p.dbg = dbg;
  }

  {
    static long long* trace = nullptr;
    static int want = -1;
    if (want < 0) want = getenv("UB_CONV_TRACE") ? 1 : 0;
    if (want && !trace) cudaMalloc(&trace, 64 * 8 * sizeof(long long));
    p.trace = trace;
    g_conv_trace = trace;
  }
  const uint16_t* ybase = reinterpret_cast<const uint16_t*>(d->y) + d->y_coff;
  if (p.has_res && (d->res_cstride % 8 || !aligned16(p.res)))
    return fail(UB_EINVAL, "ub_conv_fwd: residual rows must be 16-byte aligned (res_cstride, res_coff multiples of 8)");
  p.epi_tma = !p.y_f32 && d->y_cstride % 8 == 0 && aligned16(ybase);
  if (d->y2) {
    if (!p.epi_tma || !d->y2_map || d->y2_cstride % 8 || !aligned16(d->y2))
      return fail(UB_EUNSUPPORTED, "ub_conv_fwd: the compacted second store needs the TMA epilogue (bf16, aligned)"
                  " and a 16-byte aligned y2 with y2_cstride %% 8 == 0");
    p.y2 = static_cast<uint16_t*>(d->y2);
    p.y2_cstride = d->y2_cstride;
    p.y2_map = d->y2_map;
  }

  const uint32_t a_bytes = BLOCK_M * 128;  // sized for 64-wide residual k-blocks
  const uint32_t b_stride = (static_cast<uint32_t>(p.block_n) * bk * 2 + 1023u) & ~1023u;
  const bool tiled_1x1 = !stem && !packed && !gather && d->kh == 1 && d->kw == 1 && d->stride == 1 && d->pad == 0;
  p.a_tma = tiled_1x1 && !(d->variant & 32);
  p.epi2 = p.a_tma && !(d->variant & 64);
  p.epi_alt = p.epi2 && p.block_n <= EPI_CHUNK && !(d->variant & 4096);
  // producer width: explicit variant from the caller (engine autotune), else a heuristic
  const int pw = d->variant & 3;
  int wide = pw == 2 ? 1 : (pw == 1 ? 0 : (p.has_res ? 0 : 1));
  if (stem) wide = 1;
  // the TMA-fed 1x1 without a residual is epilogue-bound at small K (generic activations
  // most: ncu showed time tracking the epilogue's instruction count at a constant IPC): let
  // the otherwise idle producer warps 16-23 drain too.  SiLU expand 46 -> 36 us, its ReLU
  // twin 24.9 -> 22.6 us; ResNet-50 neutral (109.3 k / 109.6 k images/s, r2ce).
  static const bool epi4_env = !std::getenv("UB_CONV_NOEPI4");
  p.epi4 = epi4_env && p.epi2 && wide && !p.has_res && !p.epi_alt && p.block_n >= 2 * EPI_CHUNK && !d->y2 &&
           !(d->variant & 128);
  const int epi_warps = p.epi4 ? 16 : (p.epi2 ? 8 : 4);
  const uint32_t warp_bytes = p.epi4 ? EPI_SLOT : EPI_WARP_BYTES;
  uint32_t fixed = 1024 + IDENT_BYTES + epi_warps * warp_bytes + epi_warps * MAX_BLOCK_N * 4 + BAR_BYTES +
                   (d->y2 ? epi_warps * Y2_STAGE : 0) +
                   ((stem || packed) ? MAX_STEM_K * sizeof(int4) : 0);
  // Weight-stationary B: when all k-blocks of one N tile fit next to >= 4 A stages, each CTA
  // keeps its N tile's weights in smem (grid a multiple of n_tiles, so a CTA's tiles share
  // one N tile) instead of re-loading B for every tile.
  const uint32_t b_res_bytes = static_cast<uint32_t>(p.num_kb) * b_stride;
  p.b_res = !(d->variant & 4) && !p.mt2 && p.n_tiles <= num_sms() && fixed + b_res_bytes + 4 * a_bytes <= 226u * 1024u;
  if (p.b_res) fixed += b_res_bytes;
  const uint32_t stage_bytes = a_bytes + (p.b_res ? 0u : b_stride);
  const uint32_t budget = 226u * 1024u - fixed;
  int stages = static_cast<int>(budget / stage_bytes);
  stages = stages < 2 ? 2 : (stages > 8 ? 8 : stages);
  if (fixed + static_cast<size_t>(stages) * stage_bytes > 227u * 1024u)
    return fail(UB_EUNSUPPORTED, "ub_conv_fwd: shared memory plan does not fit");
  p.stages = stages;
  const size_t smem = fixed + static_cast<size_t>(stages) * stage_bytes;

  if (!encode_tiled_fn()) return fail(UB_ECUDA, "ub_conv_fwd: cannot resolve cuTensorMapEncodeTiled");
  CUtensorMap tmY{};
  if (p.epi_tma) {
    // output: [M][cout] view at y + y_coff, row pitch y_cstride; box 64 channels x 32 rows
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(d->cout), static_cast<cuuint64_t>(p.M)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(d->y_cstride) * 2};
    cuuint32_t box[2] = {EPI_CHUNK, 32};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_tiled_fn()(&tmY, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(ybase), dims,
                                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_fwd: encode output tensor map failed (%d)", (int)r);
    apply_small_tensor_quirk(&tmY, static_cast<size_t>(p.M) * d->y_cstride * 2);
  }

  // weights by TMA: one box (BK x block_n, the operand's swizzle) per k-block
  CUtensorMap tmB{};
  p.b_tma = !p.b_res && (p.a_tma || !(d->variant & 16));  // the TMA-fed 1x1 path has no cp.async B
  if (p.b_tma || p.a_tma) {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.K_total), static_cast<cuuint64_t>(d->cout)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(p.K_total) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(bk), static_cast<cuuint32_t>(p.block_n)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_tiled_fn()(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(d->w), dims, strides,
                                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(bk * 2),
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(UB_ECUDA, "ub_conv_fwd: encode weight tensor map failed (%d)", (int)r);
    apply_small_tensor_quirk(&tmB, static_cast<size_t>(p.K_total) * d->cout * 2);
  }
  // 1x1/s1 (tiled) A and the residual by TMA as well
  CUtensorMap tmA{}, tmR{}, tmAt{};
  p.tail_w = 64;
  if (p.a_tma) {
    auto enc = [&](CUtensorMap* m, const void* base, int cstride, int cols, int box_c, bool whole) -> CUresult {
      cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(p.M)};
      cuuint64_t strides[1] = {static_cast<cuuint64_t>(cstride) * 2};
      cuuint32_t box[2] = {static_cast<cuuint32_t>(box_c), BLOCK_M};
      cuuint32_t es[2] = {1, 1};
      CUresult r = encode_tiled_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(box_c * 2),
                                     a_promo(whole), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      apply_small_tensor_quirk(m, static_cast<size_t>(p.M) * cstride * 2);
      return r;
    };
    // A: channels [coff - lead, x_cstride) of every pixel row (beyond: zero fill)
    const bool a_whole = d->x_coff - lead == 0 && cpad >= d->x_cstride;
    if (enc(&tmA, p.x, d->x_cstride, d->x_cstride - (d->x_coff - lead), bk, a_whole) != CUDA_SUCCESS)
      return fail(UB_ECUDA, "ub_conv_fwd: encode activation tensor map failed");
    // the last K block of a slice that ends just past a 64-channel boundary: a 16- / 32-channel
    // box (SWIZZLE_32B / 64B) instead of 64 channels -- the slice's tail, not the next slice
    const int tail = cin_eff - 64 * (p.num_kb - 1);
    if (bk == 64 && p.num_kb > 1 && tail <= 32 && !(d->variant & 16384)) {
      const int tw = tail <= 16 ? 16 : 32;
      if (enc(&tmAt, p.x, d->x_cstride, d->x_cstride - (d->x_coff - lead), tw, a_whole) != CUDA_SUCCESS)
        return fail(UB_ECUDA, "ub_conv_fwd: encode activation tail tensor map failed");
      p.tail_w = tw;
    }
    const bool r_whole = d->res_coff == 0 && d->cout + 8 > d->res_cstride;
    if (p.has_res &&
        enc(&tmR, p.res, d->res_cstride, d->res_cstride - d->res_coff, EPI_CHUNK, r_whole) != CUDA_SUCCESS)
      return fail(UB_ECUDA, "ub_conv_fwd: encode residual tensor map failed");
  }
  const int num_tiles = p.mt2 ? (p.m_tiles + 1) / 2 * p.n_tiles : p.m_tiles * p.n_tiles;  // work units
  int grid = num_tiles < num_sms() ? num_tiles : num_sms();
  if (p.b_res && grid % p.n_tiles) grid = grid / p.n_tiles * p.n_tiles;
  if (stem) return launch_conv<A_STEM, 64>(tmY, tmB, tmA, tmR, tmAt, p, grid, smem, stream, wide);
  if (packed) return launch_conv<A_PACKED, 64>(tmY, tmB, tmA, tmR, tmAt, p, grid, smem, stream, wide);
  if (gather) return launch_conv<A_GATHER, 64>(tmY, tmB, tmA, tmR, tmAt, p, grid, smem, stream, wide);
  const bool pointwise = d->kh == 1 && d->kw == 1 && d->stride == 1 && d->pad == 0;
  if (pointwise) {
    if (bk == 64) return launch_conv<A_TILED, 64>(tmY, tmB, tmA, tmR, tmAt, p, grid, smem, stream, wide);
    if (bk == 32) return launch_conv<A_TILED, 32>(tmY, tmB, tmA, tmR, tmAt, p, grid, smem, stream, wide);
    return launch_conv<A_TILED, 16>(tmY, tmB, tmA, tmR, tmAt, p, grid, smem, stream, wide);
  }
  if (bk == 64) return launch_conv<A_IM2COL, 64>(tmY, tmB, tmA, tmR, tmAt, p, grid, smem, stream, wide);
  if (bk == 32) return launch_conv<A_IM2COL, 32>(tmY, tmB, tmA, tmR, tmAt, p, grid, smem, stream, wide);
  return launch_conv<A_IM2COL, 16>(tmY, tmB, tmA, tmR, tmAt, p, grid, smem, stream, wide);
}

extern "C" long long* ub_debug_conv_trace() { return ub::g_conv_trace; }

/*
 * upscale_b200.h -- C ABI of the B200-native UPSCALE export/inference hot path.
 *
 * The reference (`reslice` 0.1.0, /root/reference/pkg) has no FFI: its boundary is
 * the Python API.  Each entry point below replaces the weight math or the op
 * semantics of one reference function; the citation names the function whose
 * behaviour the call reproduces (file:line in /root/reference/pkg/src/reslice).
 *
 * Conventions:
 *   - callers own every buffer; all pointers are DEVICE pointers unless stated;
 *   - every call takes a cudaStream_t and is stream-ordered (no implicit sync);
 *   - return 0 (UB_OK) or a negative status; ub_last_error() returns the
 *     message of the last failing call on the calling thread;
 *   - activations are NHWC bf16 with a per-tensor channel stride ("cstride",
 *     a multiple of 8 elements) and a channel offset ("coff") so that a
 *     reference SLICE node (planner.py:774-777) is a zero-copy view.
 */
#ifndef UPSCALE_B200_H
#define UPSCALE_B200_H

#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UB_OK 0
#define UB_EINVAL (-1)       /* invalid argument */
#define UB_EUNSUPPORTED (-2) /* shape/layout this build does not support */
#define UB_ECUDA (-3)        /* CUDA runtime / driver error */

/* element types */
#define UB_F32 0
#define UB_F64 1
#define UB_BF16 2

/* weight layouts produced by ub_permute_weights */
#define UB_LAYOUT_OIHW 0 /* [n_rows][n_cols][kh][kw]: the plain 4-D result of apply_plan */
#define UB_LAYOUT_GEMM 1 /* [n_rows][kh*kw][cpad]: K-major B operand of ub_conv_fwd,
                            column c of tap t at (lead + c); zeros elsewhere */
#define UB_LAYOUT_GEMM_DENSE 2 /* [n_rows][cpad]: dense-K operand of the fused stem,
                                  column c of tap t at t*n_cols + c; zeros beyond */
#define UB_LAYOUT_S2D 3 /* [n_rows][kq][kq][8], kq = ceil(kw/2): operand of ub_conv_s2d,
                           element (dy, dx, (py*2+px)*n_cols + c) = W[.][c][2dy+py][2dx+px]
                           (0 past the filter); kh == kw, n_cols <= 2, lead/cpad ignored */

/* Message of the last failing call on this thread ("" if none). */
const char* ub_last_error(void);

/* ABI version (bumped on any signature change). */
int ub_abi_version(void); /* 7 */

/* Number of kernel launches issued by this library on the calling thread since
 * the last reset (used by bench.py's gpu_launches claim). */
long long ub_launch_count(void);
void ub_reset_launch_count(void);

/*
 * Weight half of apply_plan, fused over both sides of one layer.
 * Replaces: planner.py:661-673 (producer rows W[rows,:] and zero_rows),
 *           planner.py:755-767 (consumer columns W[:,perm] and zero_columns).
 * out[r][c][t] = W[rows[r]][cols[c]][t] * (row_scale ? row_scale[r] : 1)
 * rows[r] == -1 or cols[c] == -1 yields 0 (zero_rows / zero_columns).
 * W is [O][I][kh][kw] in dtype_in (UB_F32 or UB_F64).
 * layout UB_LAYOUT_OIHW ignores lead/cpad; UB_LAYOUT_GEMM writes [n_rows][kh*kw][cpad]
 * with column c at lead + c (requires lead + n_cols <= cpad).
 * dtype_out: UB_F32, UB_F64 (bit-exact copies when row_scale is NULL) or UB_BF16.
 */
int ub_permute_weights(const void* W, int dtype_in, int O, int I, int kh, int kw,
                       const int32_t* rows, int n_rows, const int32_t* cols, int n_cols,
                       const float* row_scale, int layout, int lead, int cpad,
                       void* out, int dtype_out, cudaStream_t stream);

/*
 * Number of plan indices ub_permute_weights found outside [0, O) x [0, I) since the
 * last call (those elements are written as 0 and nothing is read for them); resets
 * the counter.  Synchronous (device-wide); export time only.  Guards against a bad
 * or mismatched plan file turning into an out-of-bounds device read.
 */
int ub_index_faults(unsigned long long* count);

/*
 * Per-channel vector permutation.  Replaces planner.py:731-733
 * (new_weights[u] = new_weights[u][perm]).  out[i] = v[idx[i]] (idx[i] == -1 -> 0).
 */
int ub_permute_vector(const void* v, int dtype, const int32_t* idx, int n, void* out,
                      cudaStream_t stream);

/*
 * Standalone channel gather (the baseline export's copy, i.e. a reference GATHER
 * node executed as index_select).  Replaces interp.py:75-77 over NHWC tensors:
 * y[p][y_coff + i] = idx[i] >= 0 ? x[p][x_coff + idx[i]] : 0, for p < npix.
 */
int ub_channel_gather(const void* x, int x_cstride, int x_coff, const int32_t* idx, int n,
                      long long npix, void* y, int y_cstride, int y_coff, cudaStream_t stream);

/*
 * Row-staged channel gather (the baseline export's copy and the engine's "copy" read
 * plan).  Same result as ub_channel_gather_2d:
 *   y[p][y_coff + i] = idx[i] >= 0 ? x[src(p)][x_coff + idx[i]] : 0,  i < n_idx,
 * with src(p) the stride-subsampled source pixel, zero-filled to pad8(n_idx) channels.
 * [lo, hi] must cover every non-negative idx[i] (the host knows the plan's indices); the
 * covering window of each source row is staged in shared memory with 16-byte cp.async,
 * so HBM sees one coalesced read of the window and one 16-byte-vector write per row.
 */
int ub_gather_rows(const void* x, int x_cstride, int x_coff, int lo, int hi, const int32_t* idx, int n_idx, int N,
                   int H, int W, int stride, void* y, int y_cstride, int y_coff, cudaStream_t stream);

/*
 * ub_gather_rows with the consumer's pre-activation prologue and an optional 2x2 pool:
 *   v_i(q) = x[src_q(p)][x_coff + idx[i]],  f = relu ? max(scale[i] * v + shift[i], 0) : scale[i] * v + shift[i]
 *   y[p][y_coff + i] = bf16( pool2 ? (f(0) + f(1) + f(2) + f(3)) / 4 : f )
 * scale/shift (fp32, per OUTPUT column i, both or neither): the PER_CHANNEL (BN) and
 * PASS_THROUGH (ReLU) nodes between a value and its GATHER/SLICE reader
 * (interp.py:68-71 then 72-77), e.g. DenseNet's norm1 -> relu1 -> conv1.read.
 * pool2 = 1: src_q are the four pixels of the 2x2/s2 window (Ho = H/2, Wo = W/2; stride
 * must be 1) -- a transition layer's average pool, applied before its 1x1 conv.
 */
int ub_gather_rows_ex(const void* x, int x_cstride, int x_coff, int lo, int hi, const int32_t* idx, int n_idx,
                      int N, int H, int W, int stride, int pool2, const float* scale, const float* shift, int relu,
                      void* y, int y_cstride, int y_coff, cudaStream_t stream);

/*
 * Channel gather fused with the pixel subsampling of a strided 1x1 conv that reads it:
 * y[n][yo][xo][i] = x[n][yo*stride][xo*stride][x_coff + idx[i]] (idx[i] < 0: 0), for i < n_idx,
 * and zeros for n_idx <= i < pad8(n_idx).  Output pixels are ceil(H/stride) x ceil(W/stride);
 * y_cstride, y_coff multiples of 8.  Lets the conv that follows run as a dense 1x1 / stride-1
 * GEMM over a compact operand (the engine's "copy" read plan).
 */
int ub_channel_gather_2d(const void* x, int x_cstride, int x_coff, const int32_t* idx, int n_idx, int N, int H,
                         int W, int stride, void* y, int y_cstride, int y_coff, cudaStream_t stream);

/* K-chunk and padded per-tap K of the GEMM weight layout ub_conv_fwd expects for a
 * read of `cin` channels starting at channel offset `coff` (TMA needs 16-byte
 * aligned bases, so a misaligned SLICE start is rounded down and the first
 * `lead` weight columns are zero).  gather != 0: fused-gather read (lead 0). */
int ub_conv_weight_layout(int cin, int coff, int gather, int* lead, int* cpad);

/* Same for a kh x kw filter: small-channel k x k reads (cin + lead <= 32) use a packed
 * per-tap K of 8/16/32 (several taps per 64-wide K-block); otherwise as above. */
int ub_conv_weight_layout2(int cin, int coff, int gather, int kh, int kw, int* lead, int* cpad);

/* One convolution (CHANNEL_MIX over a spatial tensor; interp.py:57-63) with its
 * read node and epilogue fused:
 *   read:      SLICE  -> x + x_coff view (interp.py:72-74), or
 *              GATHER -> gather_idx fused into the A-operand staging (interp.py:75-77);
 *   epilogue:  + bias (folded PER_CHANNEL, interp.py:70-71), + residual (ADD,
 *              interp.py:64-65), ReLU (PASS_THROUGH, interp.py:68-69), store at a
 *              channel offset (CONCAT without a copy, interp.py:66-67).
 * Implicit GEMM on tcgen05 tensor cores: M = N*Ho*Wo, N = cout, K = kh*kw*cpad. */
/* Activations of ub_eltwise (PASS_THROUGH ops of the lowered CNNs). */
#define UB_ACT_NONE 0
#define UB_ACT_RELU 1
#define UB_ACT_RELU6 2
#define UB_ACT_HARDSWISH 3   /* x * relu6(x + 3) / 6 */
#define UB_ACT_HARDSIGMOID 4 /* relu6(x + 3) / 6 */
#define UB_ACT_SILU 5        /* x * sigmoid(x) */
#define UB_ACT_SIGMOID 6

/*
 * One vectorised NHWC bf16 pass over N*HW pixels x C channels:
 *   y = act(a * scale[c] + shift[c] + b) * gate[n][c]
 * scale/shift (fp32, per channel), b (bf16 NHWC, positional ADD, interp.py:64-65) and
 * gate (bf16 [N][gate_cstride], a squeeze-excitation multiplier broadcast over the
 * image's pixels) are each optional.  Replaces interp.py:64-71 for the PER_CHANNEL /
 * ADD / PASS_THROUGH nodes no conv epilogue absorbs.
 */
typedef struct ub_eltwise_desc {
  int N, HW, C;
  const void* a;
  int a_cstride, a_coff;
  const float* scale;
  const float* shift;
  const void* b;
  int b_cstride, b_coff;
  int act;
  const void* gate;
  int gate_cstride, gate_coff;
  void* y;
  int y_cstride, y_coff;
} ub_eltwise_desc;
int ub_eltwise(const ub_eltwise_desc* d, cudaStream_t stream);

/*
 * k x k / stride s average pool with zero padding counted (count_include_pad), NHWC bf16,
 * 16-byte aligned rows.  A DenseNet transition's AvgPool2d(2, 2) when it cannot be moved
 * in front of its 1x1 conv (ub_gather_rows_ex pool2).
 */
/*
 * Depthwise k x k conv (groups == channels) with the following BN folded in and the
 * activation fused, NHWC bf16, 16-byte aligned rows:
 *   y[n][yo][xo][c] = act(bias[c] + sum_{dy,dx} w[(dy*k + dx)*pad8(C) + c] * x[n][yo*s-pad+dy][xo*s-pad+dx][c])
 * w: fp32 [k*k][pad8(C)] (16-byte aligned); bias nullable.  The depthwise convs of
 * MobileNetV3 / EfficientNetV2, lowered to PER_CHANNEL-like nodes.
 */
int ub_dwconv(const void* x, int N, int H, int W, int C, int x_cstride, int x_coff, const float* w, const float* bias,
              int k, int s, int pad, int act, int Ho, int Wo, void* y, int y_cstride, int y_coff, cudaStream_t stream);

/*
 * ub_dwconv with the global average pool of its output fused (the squeeze-excitation pool,
 * SURVEY.md A.5, that reads the depthwise output in MobileNetV3 / EfficientNetV2): part
 * (fp32, nullable) receives per-tile channel sums of the stored bf16 outputs,
 *   part[(n * P + t) * pad8(C) + c],  P = ub_dwconv_pool_parts(k, s, Ho, Wo) tiles per image,
 * which ub_se_gate_parts adds in tile order (deterministic).  P == 0: the shape has no fused
 * pool (part must then be null).
 */
int ub_dwconv_pool_parts(int k, int s, int Ho, int Wo);
int ub_dwconv_pool(const void* x, int N, int H, int W, int C, int x_cstride, int x_coff, const float* w,
                   const float* bias, int k, int s, int pad, int act, int Ho, int Wo, void* y, int y_cstride,
                   int y_coff, float* part, cudaStream_t stream);

/*
 * Global average pool for small grids (N x ceil(C/8) too small to fill the GPU, many
 * pixels): pixels split over a CTA's threads, partial sums added in a fixed order.
 * y[n][y_coff + c] = bf16(mean_p x[n][p][x_coff + c]).  16-byte aligned source rows.
 */
int ub_avgpool_split(const void* x, int N, int HW, int C, int x_cstride, int x_coff, void* y, int y_cstride,
                     int y_coff, cudaStream_t stream);

/*
 * Small-M CHANNEL_MIX (interp.py:57-63) for M = images x pixels <= 16 (squeeze-excitation
 * FCs, classifiers at small batch) on CUDA cores:
 *   y[m][y_coff + o] = act(sum_k x[m * x_cstride + xcol[k]] * w[o * w_stride + k] + bias[o])
 * xcol (device, K entries): the element offset of input column k in a row -- a SLICE
 * view, a GATHER or a concat column map alike.  w: bf16 rows of pad8(K) columns (16-byte
 * aligned, zero-padded).  y: bf16 or fp32 (y_dtype).
 */
int ub_linear_small(const void* x, int M, int x_cstride, const int32_t* xcol, int K, const void* w, int w_stride,
                    int O, const float* bias, int act, void* y, int y_dtype, int y_cstride, int y_coff,
                    cudaStream_t stream);

/*
 * Direct CUDA-core conv for the model's first layer when it reads few image channels
 * (cin <= 8, k <= 7, cout <= 256: the 3x3/s2 stems of MobileNetV3 / EfficientNetV2).
 * x: the fp32 NCHW model input [N][C][H][W]; idx (device): the INPUT GATHER's cin kept
 * channels (interp.py:75-77).  w: fp32 [k*k][cin][ub_conv_direct_wcols(cout)] (BN folded,
 * zero columns past cout, 16-byte aligned), bias fp32.
 *   y[n][yo][xo][y_coff + o] = bf16(act(bias[o] + sum w * x))   (NHWC, 16-byte aligned rows)
 */
int ub_conv_direct_wcols(int cout);  /* pad8(cout) below 32 channels, else pad32(cout) */
int ub_conv_direct(const float* x, int N, int C, int H, int W, const int32_t* idx, int cin, const float* w,
                   const float* bias, int cout, int k, int s, int pad, int act, void* y, int y_cstride, int y_coff,
                   cudaStream_t stream);

/*
 * A squeeze-excitation gate in one launch (one CTA per image): the global pool of x,
 * fc1 = act1(W1 pooled + b1), gate = act2(W2 fc1 + b2) -- the PASS_THROUGH pool and the two
 * CHANNEL_MIX layers (interp.py:57-63, 68-71) in front of an SE `mul`.  W1: bf16
 * [C1][ldw1] over the pooled channels, W2: bf16 [C2][ldw2] over fc1's outputs (the layers'
 * SLICE / GATHER reads folded in as zero columns; ldw multiples of 8, rows 16-byte
 * aligned); b1/b2 fp32 nullable.  gate[n][g_coff + c] bf16.
 */
int ub_se_gate(const void* x, int N, int HW, int C, int x_cstride, int x_coff, const void* w1, int ldw1, int C1,
               const float* b1, int act1, const void* w2, int ldw2, int C2, const float* b2, int act2, void* gate,
               int g_cstride, int g_coff, cudaStream_t stream);
/* ub_se_gate pooling from ub_dwconv_pool's partials (part, nparts per image) instead of
 * re-reading x (x may then be null; HW still scales the mean). */
int ub_se_gate_parts(const void* x, int N, int HW, int C, int x_cstride, int x_coff, const void* w1, int ldw1, int C1,
                     const float* b1, int act1, const void* w2, int ldw2, int C2, const float* b2, int act2, void* gate,
                     int g_cstride, int g_coff, const float* part, int nparts, cudaStream_t stream);

int ub_avgpool2d(const void* x, int N, int H, int W, int C, int x_cstride, int x_coff, int k, int s, int pad, int Ho,
                 int Wo, void* y, int y_cstride, int y_coff, cudaStream_t stream);

typedef struct {
  int N, H, W;                 /* input geometry */
  int cin;                     /* channels read (slice length or gather count) */
  int cout;                    /* output channels */
  int kh, kw, stride, pad;     /* square stride/pad */
  int Ho, Wo;                  /* output spatial size */
  const void* x;               /* bf16 NHWC input */
  int x_cstride, x_coff;       /* channel stride / SLICE start */
  const int32_t* gather_idx;   /* fused GATHER indices (any kernel/stride) or NULL */
  const void* w;               /* bf16 UB_LAYOUT_GEMM weights, [cout][kh*kw][cpad] */
  int w_lead, w_cpad;          /* from ub_conv_weight_layout */
  const float* bias;           /* [cout] fp32 or NULL */
  const void* residual;        /* bf16 NHWC [N*Ho*Wo][res_cstride] or NULL */
  int res_cstride, res_coff;
  int relu;                    /* activation after bias + residual: UB_ACT_* code (1 = ReLU, 0 = none) */
  void* y;                     /* output, NHWC [N*Ho*Wo][y_cstride] */
  int y_cstride, y_coff;
  int y_dtype;                 /* UB_BF16 or UB_F32 */
  int x_nchw_f32;              /* 1: fused stem -- x is the fp32 NCHW model input
                                  [N][x_channels][H][W]; gather_idx selects the cin planes
                                  (the INPUT node's GATHER), weights UB_LAYOUT_GEMM_DENSE */
  int x_channels;
  int variant;                 /* bits 0-1 producer width (0 heuristic, 1: 256, 2: 512 threads);
                                  bit 2: re-load weights per tile (no weight-stationary B);
                                  bit 3: no halo-tile kernel for stride-1 3x3 convs;
                                  bit 7: halo kernel with two epilogue groups (default: up to three);
                                  bit 4: weights by cp.async instead of one TMA box per K-block;
                                  bit 5: 1x1/s1 activations and residual by cp.async, not TMA;
                                  bit 6: one epilogue warpgroup (not two) on the TMA-fed 1x1 path;
                                  bit 8: no stacked small images in the halo kernel;
                                  bit 11: halo input by cp.async planes instead of TMA boxes;
                                  bit 12: narrow tiles drained by alternate chunks, not tiles;
                                  bit 13: N tiles of at most 128 channels;
                                  bit 14: no narrower (16/32-channel) last A box on the TMA 1x1 path */
  /* Optional second, compacted store of the output (the producer side of a GATHER read by
   * a later 1x1 conv): y2[m][y2_map[c]] = y[m][y_coff + c] for every c with y2_map[c] >= 0.
   * Layout contract: the kept channels of each 64-channel group [64g, 64g + 64) take
   * consecutive columns starting at a multiple of 8; the columns up to the next multiple of 8
   * are written as zeros.  The consumer runs as a dense GEMM over y2 (bf16, row pitch
   * y2_cstride % 8 == 0, 16-byte aligned).  Needs the TMA epilogue (bf16 y, aligned). */
  void* y2;
  int y2_cstride;
  const int32_t* y2_map;       /* [cout] or NULL */
} ub_conv_desc;

/* Dense-K padding (multiple of 64) of the fused-stem weight operand. */
int ub_conv_stem_kpad(int cin, int kh, int kw);

int ub_conv_fwd(const ub_conv_desc* d, cudaStream_t stream);

/*
 * Space-to-depth stem (the stride-2 k x k first conv when its input GATHER keeps
 * <= 2 channels).  Same op as ub_conv_fwd with x_nchw_f32 = 1, split in two launches:
 *   ub_stem_s2d_pack:  x fp32 NCHW [N][C][H][W] -> s, bf16 rows of 8:
 *                      s[(n*Hs + Y)*Ws + X][(py*2+px)*cin + c] = x[n][idx[c]][2Y+py-pad][2X+px-pad]
 *                      (0 outside the image); the tail rows past N*Hs*Ws are read by the
 *                      conv but never written here -- allocate s zeroed once;
 *   ub_conv_s2d:       y = act(conv(s, w) + bias) with w in UB_LAYOUT_S2D, on tcgen05 (the
 *                      2x2-folded conv is stride 1, so every filter tap of a 128-pixel tile
 *                      is a shifted view of ONE contiguous block of s).
 * ub_stem_s2d_geometry gives Hs, Ws and the byte size of s.  cout <= 128; y_cstride and
 * y_coff multiples of 8.  Replaces the same reference nodes as ub_conv_fwd's stem.
 */
int ub_stem_s2d_geometry(int N, int H, int W, int k, int pad, int* Hs, int* Ws, long long* bytes);
int ub_stem_s2d_pack(const float* x, int N, int C, int H, int W, const int32_t* idx, int cin, int k, int pad,
                     void* s, cudaStream_t stream);
int ub_conv_s2d(const void* s, int N, int H, int W, int k, int pad, const void* w, int cout,
                const float* bias, int relu, void* y, int y_cstride, int y_coff, cudaStream_t stream);

/*
 * ub_conv_s2d followed by the max pool that consumes it (PASS_THROUGH nn.MaxPool2d,
 * kernel 3 / stride 2 / pad 1, -inf padding), fused: y is the POOLED output
 * [N][Ho/2][Wo/2][y_cstride] bf16; the conv output never reaches memory.  cout <= 64,
 * conv output Ho, Wo even with Wo <= 128.  Same result as ub_conv_s2d + ub_maxpool2d.
 */
int ub_conv_s2d_maxpool(const void* s, int N, int H, int W, int k, int pad, const void* w, int cout,
                        const float* bias, int relu, int pool_k, int pool_stride, int pool_pad,
                        void* y, int y_cstride, int y_coff, cudaStream_t stream);

/* The same stem + max pool reading the fp32 NCHW model input directly: the pair tiles' folded
 * rows are built in shared memory by the kernel's producer warps from channels idx[0..cin) of
 * x [N][C][H][W] (the INPUT node's GATHER, interp.py:75-77, and the fp32 -> bf16 cast), so the
 * folded buffer S and the pack launch disappear.  Same result as ub_stem_s2d_pack +
 * ub_conv_s2d_maxpool, bit for bit. */
int ub_stem_maxpool(const float* x, int N, int C, int H, int W, const int32_t* idx, int cin, int k, int pad,
                    const void* w, int cout, const float* bias, int relu, int pool_k, int pool_stride, int pool_pad,
                    void* y, int y_cstride, int y_coff, cudaStream_t stream);

/* Model-input staging: NCHW fp32 -> NHWC bf16 [N*H*W][y_cstride], channels
 * idx[0..n) (a GATHER on the INPUT node, fused; idx == NULL: identity over C). */
int ub_stage_input(const float* x, int N, int C, int H, int W, const int32_t* idx, int n,
                   void* y, int y_cstride, cudaStream_t stream);

/* Host -> device copy of the model input restricted to the channels the INPUT node's
 * GATHER keeps (planner.py:774-783): for each c in channels[0..n) (HOST array), plane c of
 * every image of the pinned host NCHW fp32 batch goes to the same place in the device NCHW
 * buffer (one strided cudaMemcpy2DAsync per channel); dropped channels never cross PCIe.
 * *bytes (optional) receives the bytes copied. */
int ub_h2d_input_channels(const float* host_nchw, int N, int C, int HW, const int32_t* channels, int n,
                          float* dev_nchw, long long* bytes, cudaStream_t stream);

/* Max pool (PASS_THROUGH lowering of nn.MaxPool2d), NHWC bf16, -inf padding. */
int ub_maxpool2d(const void* x, int N, int H, int W, int C, int x_cstride, int x_coff,
                 int k, int stride, int pad, int Ho, int Wo,
                 void* y, int y_cstride, int y_coff, cudaStream_t stream);

/* Global average pool (nn.AdaptiveAvgPool2d(1)), NHWC bf16 -> [N][y_cstride] bf16. */
int ub_avgpool_global(const void* x, int N, int HW, int C, int x_cstride, int x_coff,
                      void* y, int y_cstride, int y_coff, cudaStream_t stream);

/* Global average pool fused with the GATHER that reads it (e.g. ResNet's avgpool -> fc.read):
 * y[n][y_coff + j] = bf16(mean over HW of x[n][.][x_coff + idx[j]]), 0 where idx[j] < 0
 * (interp.py:75-77 GATHER applied to the PASS_THROUGH pool output), written compacted so the
 * consumer reads a dense operand.  C, x_cstride, x_coff multiples of 8; N <= 65535. */
int ub_avgpool_gather(const void* x, int N, int HW, int C, int x_cstride, int x_coff,
                      const int32_t* idx, int n_idx, void* y, int y_cstride, int y_coff,
                      cudaStream_t stream);

/* Generic elementwise node for graphs the conv epilogue cannot absorb:
 * y = relu?( a*scale + shift + b ) per channel over NHWC bf16 (scale/shift/b optional).
 * Covers standalone PER_CHANNEL (interp.py:70-71), ADD (64-65), PASS_THROUGH ReLU (68-69). */
int ub_affine_add_relu(const void* a, int a_cstride, int a_coff,
                       const float* scale, const float* shift,
                       const void* b, int b_cstride, int b_coff, int relu,
                       long long npix, int C, void* y, int y_cstride, int y_coff,
                       cudaStream_t stream);

/*
 * Planner core (host only, no GPU): decompose one segment's reorder graph into maximum-
 * reward paths and emit its channel order -- path_search.py:157-305 (solve_mrap with the
 * lexicographic tie-break, the greedy fallback above 20 nodes, decompose_paths) and
 * ordering.py:39-88 (order_channels), restated natively; the reference's plan_model uses
 * it through paper_2307_08771_b200.native_planner.install().
 *   n nodes sorted by id; node i retains channels[offsets[i] .. offsets[i+1]) (ascending,
 *   non-empty, < channel_space).  Outputs: out_order[*n_order] (kept channels in the new
 *   order; capacity channel_space), path_of[i] / path_pos[i] (path index; position on it,
 *   -1 for an absorbed parent), path_reward[k] for k < *n_paths (capacity n).
 */
int ub_plan_order_segment(int n, const int32_t* offsets, const int32_t* channels, int channel_space,
                          int32_t* out_order, int32_t* n_order, int32_t* path_of, int32_t* path_pos,
                          int64_t* path_reward, int32_t* n_paths);

#ifdef __cplusplus
}
#endif
#endif /* UPSCALE_B200_H */

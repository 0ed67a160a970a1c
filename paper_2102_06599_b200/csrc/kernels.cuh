// Device-side parameter blocks and launchers shared by the nb200 kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace nb {

constexpr int kMaxRanges = 16;

#ifdef __CUDACC__
// 3xTF32 operand split: hi = round-to-nearest tf32(x), lo = tf32(x - hi), so
// hi + lo carries 22 significant bits and hi*hi + hi*lo + lo*hi reproduces an
// fp32 product to ~2^-22 (the tensor core reads only the top 19 bits of each
// operand, so both halves are pre-rounded rather than left to truncation).
__device__ __forceinline__ void split_tf32(uint32_t x, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(__uint_as_float(x)));
  const float r = __uint_as_float(x) - __uint_as_float(hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}
#endif

// One output-channel range of a ConvSpec (I/ir.hpp:54-57): channels
// [b, b+len) in G groups of slice_co outputs, each reading slice_ci inputs.
struct RangeDesc {
  int b, len, groups, slice_co, slice_ci;
  int64_t wf_off;  // offset (floats) of the fprop-packed weights Wf_r[tap][j][co_local]
  int64_t wd_off;  // offset (floats) of the dgrad-packed weights Wd_r[tap][t][ci]
};

// Geometry of one conv layer over a batch, NHWC fp32 activations.
struct ConvGeom {
  int N, H, W, Ci, OH, OW, Co, KH, KW, S, P;
  int nranges;
  RangeDesc r[kMaxRanges];
};

// Pixel tile of the fused dgrad/Fisher epilogue: partial sums of A*g are
// produced per (image, tile, channel) and combined in a fixed order.
constexpr int kDgradTilePix = 128;
inline int dgrad_tiles(int H, int W) { return (H * W + kDgradTilePix - 1) / kDgradTilePix; }

// ---- launchers (kernels_simt.cu) -----------------------------------------
void launch_nchw64_to_nhwc32(const double* src, float* dst, int64_t N, int C, int H, int W,
                             cudaStream_t st);
void launch_nhwc32_to_nchw64(const float* src, double* dst, int64_t N, int C, int H, int W,
                             cudaStream_t st);
// Packs one range's weights; null destinations are skipped.  TC packings
// are K-major hi/lo pairs (hi = tf32-truncated value, lo = value - hi):
//   tcf: [co_local][tap][j]      (fprop B operand, rows = output channels)
//   tcd: [ci][tap][t]            (dgrad B operand, rows = input channels)
struct PackDst {
  float* wf;
  float* wd;
  float* tcf_hi;
  float* tcf_lo;
  float* tcd_hi;
  float* tcd_lo;
  // kw-fused tensor-core layouts (rows kw*width + c, K = kh x channels)
  int kwf_f = 0, kwf_d = 0, KW = 1;
  // 16-bit split tensor-core layouts: tc*_hi / tc*_lo hold 16-bit halves
  // (rn(w'), rn(w' - hi)) of w' = w * h16_scale at the same element index
  // instead of the tf32 fp32 pair; h16: 0 = tf32 pair, 1 = bf16, 2 = fp16
  int h16 = 0;
  float h16_scale = 1.f;
  // padded K per tap of the fprop / dgrad tensor-core layouts (0 = exact)
  int kpf = 0, kpd = 0;
  // densified grouped layouts: K indexed by the full input (fprop) / range
  // output (dgrad) channel instead of the slice-local one
  int dense_f = 0, dense_d = 0;
  // im2col stem layout: row co, K = tap * Ci + ci in 32 columns
  int col_f = 0;
};
// im2col of an NHWC fp32 batch for a stem with Ci*KH*KW <= 32:
// out (N, OH, OW, 32), column tap*Ci + ci, zeros for padding taps and k >= Ci*KH*KW
void launch_im2col32(const float* x, int64_t N, int H, int W, int Ci, int KH, int KW, int S,
                     int P, int OH, int OW, float* out, cudaStream_t st);
void launch_pack_weights(const double* src, double scale, const ConvGeom& g, int range,
                         const PackDst& d, cudaStream_t st);
void launch_fprop_direct(const ConvGeom& g, int range, const float* x, const float* wbase,
                         float* y, bool relu, cudaStream_t st);
// g_in = convT(W, dpre) over all ranges; fused epilogue on the previous
// layer's activation a_prev (nullable): partial[n][tile][ci] = sum A*g,
// dpre_out = g * [a_prev > 0] (or g when !relu_prev), g_out = g (nullable).
// Partial tiles per image of the direct dgrad launch_dgrad_direct picks for g.
int direct_dgrad_tiles(const ConvGeom& g);
void launch_dgrad_direct(const ConvGeom& g, const float* dpre, const float* wbase,
                         const float* a_prev, bool relu_prev, float* dpre_out, float* g_out,
                         double* partial, cudaStream_t st);
// Epilogue of a split-K tensor-core GEMM: v = sum_k ws[k] (fixed order) over
// an (N, H, W) pixel grid and channels [c0, c0+C) of tensors with `ld`
// channels.  fprop (mode 0): out = relu?(v).  dgrad (mode 1): g_out = v,
// dpre_out = v masked by a_prev > 0 (when relu_prev), partial[n][0][c] =
// sum over the image of a_prev * v (fixed order; one partial tile per image).
struct SplitEpi {
  const float* ws;
  int64_t ws_stride;
  int ksplit, mode;
  int N, HW, ld, c0, C;
  float* out;
  int relu;
  const float* a_prev;
  float* dpre_out;
  float* g_out;
  double* partial;
  int relu_prev;
  // pixel chunks per image (grid z): enough blocks for small batches; a
  // dgrad writes one Fisher partial per (image, chunk)
  int hw_chunks = 1;
  // per-image max |value| of the stored output (mode 0) / dpre_out (mode 1)
  // for the next fp16-split GEMM (float bits; null = not recorded)
  uint32_t* out_amax = nullptr;
};
void launch_splitk_epilogue(const SplitEpi& e, cudaStream_t st);
// Pixel chunks of a split-K epilogue over n images of HW pixels x C channels
// (a function of the shape only, so plans and launches agree).
int splitk_hw_chunks(int64_t n, int HW, int C);
// Per-image max |x| of an NHWC tensor of N images x per_img floats into
// amax[n] (float bits, atomicMax: amax must start at 0 or a smaller value)
void launch_amax(const float* x, int64_t N, int64_t per_img, uint32_t* amax, cudaStream_t st);

// GAP + linear head + softmax-CE (+ backward, + last-layer Fisher partial,
// + the masked head gradient dpre of the last layer).
struct HeadArgs {
  const float* act;  // (N, HW, C) last layer output
  int N, HW, C, K;
  double grad_n;  // the batch size dz is divided by (the global N when sharded)
  const double* head_src;  // K x C source (z-stream or explicit)
  double head_scale;
  const int32_t* labels;
  double* probs;        // N x K
  double* ex_loss;      // N
  bool backward;
  bool relu_last;
  double* partial;      // N x C (sum_hw A*g), nullable
  float* dpre;          // (N, HW, C) masked gradient, nullable
  float* g_out;         // (N, HW, C) unmasked gradient, nullable
};
void launch_head(const HeadArgs& a, cudaStream_t st);
// Fisher reduction: per (layer, channel) delta = sum_n (sum_tiles partial)^2 / (2N).
struct FisherLayer {
  const double* partial;  // example n's tile partials at partial + n * nstride
  int C, tiles;
  int64_t out_off;
  int64_t nstride;
};
// s_out (nullable): s_nc stored at s_out[n * s_ld + out_off + c], the
// per-example sums an example-sharded evaluation gathers to its root.
void launch_fisher_reduce(const FisherLayer* layers_dev, int L, int max_c, int N,
                          double* per_channel, double* s_out, int64_t s_ld, cudaStream_t st);

}  // namespace nb

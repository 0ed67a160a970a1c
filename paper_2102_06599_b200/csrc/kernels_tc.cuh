// Host interface of the tcgen05 implicit-GEMM conv kernels (kernels_tc.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace nb {
namespace tc {

constexpr int kMaxPhases = 4;      // sub-pixel phases of a stride-2 dgrad
constexpr int kMaxPhaseTaps = 32;  // taps per phase (kernels up to 5x5 in one phase)

// One tap of a phase, packed: bits 0-11 = tap index kh*KW+kw into the B
// operand's K dimension, bits 12-21 / 22-31 = signed 10-bit offsets (h, w) of
// the A box relative to the tile origin (in A-tensor elements, before the
// element stride).
__host__ __device__ inline int32_t pack_tap(int kidx, int dh, int dw) {
  return int32_t(uint32_t(kidx & 0xFFF) | (uint32_t(dh & 0x3FF) << 12) |
                 (uint32_t(dw & 0x3FF) << 22));
}
__host__ __device__ inline int tap_kidx(int32_t t) { return int(uint32_t(t) & 0xFFF); }
__host__ __device__ inline int tap_dh(int32_t t) { return (int(uint32_t(t) << 10) >> 22); }
__host__ __device__ inline int tap_dw(int32_t t) { return int(t) >> 22; }

// One GEMM launch: an output-channel range (all its groups) of a conv layer,
// fprop (mode 0) or dgrad (mode 1).  See kernels_tc.cu.
//
// The GEMM's M dimension is a set of `nphase` pixel grids.  Phase p covers
// the output pixels (n, oy*PS + py[p], ox*PS + px[p]) for oy < OHp[p],
// ox < OWp[p]; fprop and stride-1 dgrad have one phase with PS = 1, a
// stride-2 dgrad has the four sub-pixel phases (PS = 2), each a stride-1
// correlation of dY with the taps whose parity matches the phase.
struct TcArgs {
  int mode;
  int nimg;
  // tile geometry shared by all phases (planned on the largest phase grid)
  int OH, OW;  // largest phase grid
  int BW, BH, BNI, tiles_w, tiles_h, tiles_n, m_tiles;
  int n_tiles, n_tiles_per_group;
  // split-K: the (tap, channel-chunk) K blocks of a tile are divided into
  // ksplit contiguous ranges, each accumulated by its own work unit into its
  // own copy of the output (ws + ks * ws_stride, same layout as out);
  // k_splitk_epilogue then sums the copies in order and runs the epilogue
  int ksplit;
  float* ws;
  int64_t ws_stride;
  int S;  // element stride of the A box (fprop stride; 1 for dgrad)
  // phases
  int nphase, PS;
  int OHp[kMaxPhases], OWp[kMaxPhases], py[kMaxPhases], px[kMaxPhases];
  int ntaps[kMaxPhases];
  int32_t taps[kMaxPhases][kMaxPhaseTaps];
  // A operand (4-D NHWC activation): 32-channel K chunks per tap, channel base
  int a_cblocks, a_c_base, a_c_per_group;
  // B operand (2-D K-major weights [rows][taps*K]): K per tap, row bases
  int b_k_per_tap, b_row_base, b_row_per_group;
  // fprop over a band of output rows [oh_base, oh_base + OHp[0]) of the
  // OutH-row output (the masked box executor, nb_conv_band); 0 otherwise
  int oh_base;
  // epilogue output (NHWC over OutH x OutW pixels, ld channels)
  float* out;
  int OutH, OutW;
  int out_ld, out_c_base, out_c_per_group;
  int relu;
  // dgrad fused epilogue
  const float* a_prev;
  float* dpre_out;
  float* g_out;
  double* partial;
  int relu_prev, part_tiles_per_img, part_ld;
  // kw-fused plan (KWF): +1 fprop, -1 dgrad, 0 off -- see Cfg in kernels_tc.cu
  int kwf_sgn;
  int kwf_w;  // image row width of a kw-fused plan (a lane segment per row)
  // 3xTF32 converters: both groups split every stage (channel halves) rather
  // than alternating stages (lower per-stage latency for shallow rings)
  int conv_halves;
  // 16-bit split (Cfg BF): 1 = fp16 halves (kind::f16 f16, scaled), 0 = bf16.
  // fp16 scaling: A row r of image n is multiplied by 2^(14 - e_n) before the
  // split, e_n the exponent of a_amax[n] (max |A| of image n, float bits;
  // null = no scaling), the weights were packed times b_scale; the epilogue
  // multiplies the accumulator by 2^-(14 - e_n) and b_inv = 1 / b_scale.
  // Powers of two: the scaled products and sums are the unscaled ones
  // exactly, outside fp16 subnormals.
  int h16_f16;
  // halo mode (split converters, single CTA, S == 1; kernels_tc.cu): the A
  // map's box is halo_w x halo_h pixels (x BNI images) at the tile origin
  // plus (halo_dw0, halo_dh0)[phase], the smallest tap offsets of the phase
  int halo, halo_w, halo_h;
  int halo_dh0[kMaxPhases], halo_dw0[kMaxPhases];
  const uint32_t* a_amax;
  float b_inv;
  // per-image max |value| of what this launch writes for the next GEMM
  // (fprop: the stored output; dgrad: dpre_out), atomicMax on float bits;
  // null = not recorded
  uint32_t* out_amax;
  // experiments only (NB_TC_DEBUG; every bit but the stage cap gives
  // garbage results): 2 = no MMAs, 4 = no A loads, 8 = no B loads, 16 = no
  // epilogue, 32 = no split conversion, 64 = no tiles at all, 128 = MMAs
  // read stage 0's TMEM columns only, 2048 = no A_prev loads, 4096 = no
  // Fisher reduction, 8192 = no dpre stores, 16384 = B prefetch before the
  // grid dependency (a correct variant, not garbage); bits 16..19 cap the ring depth
  // (0 = the configured stage count)
  int debug;
  // experiments only (NB_TC_TRACE): CTA 0 records clock64() stamps of its
  // first kTraceStages K blocks here (see kernels_tc.cu)
  long long* trace;
};
constexpr int kTraceStages = 256;
// trace roles per stage (see kernels_tc.cu trace()); CTA stamps follow them
constexpr int kTraceRoles = 10;

struct TcLaunch {
  CUtensorMap mapA, mapBh, mapBl;
  TcArgs args;
  int bn;       // N tile (of the pair, when pair)
  bool split3;  // 3xTF32
  bool pair;    // CTA pair (cluster of 2): M = 256 per tcgen05.mma.cta_group::2
  bool mc = false;  // multicast cluster of 2: B halves multicast, MMAs per CTA
  bool kwf = false;  // kw-fused 64-channel plan (MMA N = 192)
  bool bf = false;   // 16-bit split (with split3): 16-bit B_hi / B_lo, kind::f16 MMAs
                     // (args.h16_f16: fp16, else bf16)
  int num_sms;
};

// Fills the M-tile geometry of `a` for an OH x OW (largest phase) grid over
// nimg images; false if the TMA box would be illegal.
bool plan_tiles(int OH, int OW, int nimg, int S, TcArgs& a);
// Encodes the tensor maps (A: C x W x H x N activation, B: rows x K weights).
// (B_hi / B_lo are bf16 arrays when L.bf)
bool make_maps(TcLaunch& L, const float* A, int AC, int AW, int AH, int AN, const void* Bhi,
               const void* Blo, int BK, int Brows);
cudaError_t launch(const TcLaunch& L, cudaStream_t st);
// Halo buffer bytes the kernel configuration of L offers (0: no halo mode)
int halo_capacity(const TcLaunch& L);

}  // namespace tc
}  // namespace nb

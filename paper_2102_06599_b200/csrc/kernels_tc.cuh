// Host interface of the tcgen05 implicit-GEMM conv kernels (kernels_tc.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace nb {
namespace tc {

// One GEMM launch: an output-channel range (all its groups) of a conv layer,
// fprop (mode 0) or stride-1 dgrad (mode 1).  See kernels_tc.cu.
struct TcArgs {
  int mode;
  // GEMM output pixel space (fprop: OH x OW; dgrad: the layer input H x W)
  int nimg, OH, OW;
  // M tile = BNI images x BH rows x BW columns (<= 128 pixels)
  int BW, BH, BNI, tiles_w, tiles_h, tiles_n, m_tiles;
  int n_tiles, n_tiles_per_group;
  int taps_h, taps_w, S, P;
  // A operand (4-D NHWC activation): 32-channel K chunks per tap, channel base
  int a_cblocks, a_c_base, a_c_per_group;
  // B operand (2-D K-major weights [rows][taps*K]): K per tap, row bases
  int b_k_per_tap, b_row_base, b_row_per_group;
  // epilogue output (NHWC, ld channels)
  float* out;
  int out_ld, out_c_base, out_c_per_group;
  int relu;
  // dgrad fused epilogue
  const float* a_prev;
  float* dpre_out;
  float* g_out;
  double* partial;
  int relu_prev, part_tiles_per_img, part_ld;
};

struct TcLaunch {
  CUtensorMap mapA, mapBh, mapBl;
  TcArgs args;
  int bn;
  bool split3;
  int num_sms;
};

// Fills the M-tile geometry of `a` for an OH x OW output over nimg images;
// false if the TMA box would be illegal.
bool plan_tiles(int OH, int OW, int nimg, int S, TcArgs& a);
// Encodes the tensor maps (A: C x W x H x N activation, B: rows x K weights).
bool make_maps(TcLaunch& L, const float* A, int AC, int AW, int AH, int AN, const float* Bhi,
               const float* Blo, int BK, int Brows);
cudaError_t launch(const TcLaunch& L, cudaStream_t st);

}  // namespace tc
}  // namespace nb

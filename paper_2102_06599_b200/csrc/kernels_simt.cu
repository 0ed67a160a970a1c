// fp32 FFMA kernels of the nb200 hot path: layout conversion, weight packing,
// direct (grouped / depthwise / generic) conv fprop and the dgrad with the
// fused Fisher epilogue, the fp64 head, and the deterministic Fisher
// reduction.  Tensor-core-shaped ranges use kernels_tc.cu instead.
//
// Activations are NHWC fp32 in HBM (channels contiguous: coalesced across
// output channels for fprop and across input channels for dgrad).
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "kernels.cuh"

namespace nb {

namespace {

__global__ void k_nchw64_to_nhwc32(const double* __restrict__ src, float* __restrict__ dst,
                                   int64_t N, int C, int H, int W) {
  const int64_t total = N * C * H * W;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    // i indexes dst (n, h, w, c)
    const int c = int(i % C);
    int64_t p = i / C;
    const int w = int(p % W);
    p /= W;
    const int h = int(p % H);
    const int64_t n = p / H;
    dst[i] = float(src[((n * C + c) * H + h) * W + w]);
  }
}

__global__ void k_nhwc32_to_nchw64(const float* __restrict__ src, double* __restrict__ dst,
                                   int64_t N, int C, int H, int W) {
  const int64_t total = N * C * H * W;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    // i indexes dst (n, c, h, w)
    const int w = int(i % W);
    int64_t p = i / W;
    const int h = int(p % H);
    p /= H;
    const int c = int(p % C);
    const int64_t n = p / C;
    dst[i] = double(src[((n * H + h) * W + w) * C + c]);
  }
}

// Weights of one range, from the dense (Co_eff, Ci, Kh, Kw) fp64 tensor of
// the reference (I/nnet.hpp:65-67; grouped variants read only the diagonal
// blocks, I/nnet.hpp:111-127), scaled (z * 1/sqrt(fan-in), or 1 for explicit
// weights) in fp64 and rounded once to fp32, into two packings:
//   Wf[tap][j][co_local]  (fprop: coalesced over output channels)
//   Wd[tap][t][ci]        (dgrad: coalesced over input channels)
__global__ void k_pack_weights(const double* __restrict__ src, double scale, int Ci, int taps,
                               RangeDesc r, PackDst d) {
  const int64_t total = int64_t(r.len) * r.slice_ci * taps;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int co_local = int(e % r.len);
    const int64_t q = e / r.len;
    const int j = int(q % r.slice_ci);
    const int tap = int(q / r.slice_ci);
    const int g = co_local / r.slice_co;
    const int t = co_local - g * r.slice_co;
    const int ci = g * r.slice_ci + j;
    const int64_t co = r.b + co_local;
    const float v = float(src[(co * Ci + ci) * taps + tap] * scale);
    if (d.wf) d.wf[r.wf_off + e] = v;
    if (d.wd) d.wd[r.wd_off + (int64_t(tap) * r.slice_co + t) * Ci + ci] = v;
    uint32_t hb, lb;
    split_tf32(__float_as_uint(v), hb, lb);
    const float hi = __uint_as_float(hb), lo = __uint_as_float(lb);
    // 16-bit split pair of v' = v * h16_scale (a power of two): rn(v'), rn(v' - that)
    uint16_t bhi = 0, blo = 0;
    if (d.h16 == 1) {
      const __nv_bfloat16 bh = __float2bfloat16_rn(v);
      bhi = __bfloat16_as_ushort(bh);
      blo = __bfloat16_as_ushort(__float2bfloat16_rn(v - __bfloat162float(bh)));
    } else if (d.h16 == 2) {
      const float vs = v * d.h16_scale;
      const __half fh = __float2half_rn(vs);
      bhi = __half_as_ushort(fh);
      blo = __half_as_ushort(__float2half_rn(vs - __half2float(fh)));
    }
    const int kh = tap / d.KW, kw = tap - kh * d.KW, KH = taps / d.KW;
    if (d.tcf_hi) {
      const int kpf = d.kpf ? d.kpf : r.slice_ci;
      const int64_t i = d.col_f   ? int64_t(co_local) * 32 + tap * r.slice_ci + j
                        : d.kwf_f ? ((int64_t(kw) * r.len + co_local) * KH + kh) * r.slice_ci + j
                                  : (int64_t(co_local) * taps + tap) * kpf + (d.dense_f ? ci : j);
      if (d.h16) {
        reinterpret_cast<uint16_t*>(d.tcf_hi)[i] = bhi;
        reinterpret_cast<uint16_t*>(d.tcf_lo)[i] = blo;
      } else {
        d.tcf_hi[i] = hi;
        d.tcf_lo[i] = lo;
      }
    }
    if (d.tcd_hi) {
      const int kpd = d.kpd ? d.kpd : r.slice_co;
      const int64_t i = d.kwf_d ? ((int64_t(kw) * Ci + ci) * KH + kh) * r.slice_co + t
                                : (int64_t(ci) * taps + tap) * kpd + (d.dense_d ? co_local : t);
      if (d.h16) {
        reinterpret_cast<uint16_t*>(d.tcd_hi)[i] = bhi;
        reinterpret_cast<uint16_t*>(d.tcd_lo)[i] = blo;
      } else {
        d.tcd_hi[i] = hi;
        d.tcd_lo[i] = lo;
      }
    }
  }
}

// Direct conv fprop of one range, register-blocked: a block owns 128 output
// pixels x CO_T output channels of one group; the group's weights for those
// channels are staged in shared memory K-chunk by K-chunk (Wf[tap][j][co]),
// every thread keeps its pixel's CO_T accumulators in registers and each
// input value it loads feeds CO_T FMAs (weights are shared-memory
// broadcasts).  Padded taps are skipped (I/nnet.hpp:121-123).
constexpr int kFpPix = 128;
constexpr int kFpKChunk = 128;

template <int CO_T, int PX>
__global__ void __launch_bounds__(kFpPix) k_fprop_blocked(ConvGeom g, int ri,
                                                          const float* __restrict__ x,
                                                          const float* __restrict__ wbase,
                                                          float* __restrict__ y, bool relu) {
  // PX pixels per thread (pixels threadIdx.x + 128 i): each shared-memory
  // weight read feeds PX pixels
  __shared__ float ws[kFpKChunk * PX][CO_T];
  const RangeDesc r = g.r[ri];
  const float* __restrict__ wf = wbase + r.wf_off;
  const int co_chunks = (r.slice_co + CO_T - 1) / CO_T;
  const int grp = blockIdx.y / co_chunks;
  const int co0 = (blockIdx.y % co_chunks) * CO_T;  // within the group
  const int nco = min(CO_T, r.slice_co - co0);
  const int64_t npix = int64_t(g.N) * g.OH * g.OW;
  const int64_t pix0 = int64_t(blockIdx.x) * kFpPix * PX;
  bool valid[PX];
  int ow[PX], oh[PX];
  int64_t n[PX];
#pragma unroll
  for (int i = 0; i < PX; ++i) {
    const int64_t pix = pix0 + threadIdx.x + i * kFpPix;
    valid[i] = pix < npix;
    const int64_t pp = valid[i] ? pix : 0;
    ow[i] = int(pp % g.OW);
    oh[i] = int((pp / g.OW) % g.OH);
    n[i] = pp / (int64_t(g.OW) * g.OH);
  }
  float acc[PX][CO_T];
#pragma unroll
  for (int i = 0; i < PX; ++i)
#pragma unroll
    for (int t = 0; t < CO_T; ++t) acc[i][t] = 0.f;
  const int K = r.slice_ci * g.KH * g.KW;
  // float4 input path: a tap's slice_ci channels are contiguous and aligned,
  // and K chunks hold whole taps (summation order per output unchanged)
  const bool vec4 = r.slice_ci % 4 == 0 && kFpKChunk % r.slice_ci == 0 && g.Ci % 4 == 0;
  for (int k0 = 0; k0 < K; k0 += kFpKChunk) {
    const int kn = min(kFpKChunk, K - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < kn * CO_T; e += kFpPix) {
      const int kk = e / CO_T, t = e % CO_T;
      ws[kk][t] = t < nco ? wf[int64_t(k0 + kk) * r.len + grp * r.slice_co + co0 + t] : 0.f;
    }
    __syncthreads();
    if (vec4) {
      // whole taps of the chunk, the tap's slice_ci inputs as float4s
      for (int kk = 0; kk < kn; kk += r.slice_ci) {
        const int tap = (k0 + kk) / r.slice_ci;
        const int kh = tap / g.KW, kw = tap - kh * g.KW;
        const float4* xp[PX];
#pragma unroll
        for (int i = 0; i < PX; ++i) {
          const int ih = g.S * oh[i] - g.P + kh, iw = g.S * ow[i] - g.P + kw;
          xp[i] = (valid[i] && ih >= 0 && ih < g.H && iw >= 0 && iw < g.W)
                      ? reinterpret_cast<const float4*>(x + ((n[i] * g.H + ih) * g.W + iw) * g.Ci +
                                                        int64_t(grp) * r.slice_ci)
                      : nullptr;  // padded taps add nothing (I/nnet.hpp:121-123)
        }
        for (int j4 = 0; j4 < r.slice_ci / 4; ++j4) {
          float4 xv[PX];
#pragma unroll
          for (int i = 0; i < PX; ++i)
            xv[i] = xp[i] ? __ldg(xp[i] + j4) : make_float4(0.f, 0.f, 0.f, 0.f);
          const int b = kk + 4 * j4;
#pragma unroll
          for (int t = 0; t < CO_T; ++t) {
            const float w0 = ws[b][t], w1 = ws[b + 1][t], w2 = ws[b + 2][t], w3 = ws[b + 3][t];
#pragma unroll
            for (int i = 0; i < PX; ++i) {
              if (!xp[i]) continue;
              float a = acc[i][t];
              a = fmaf(xv[i].x, w0, a);
              a = fmaf(xv[i].y, w1, a);
              a = fmaf(xv[i].z, w2, a);
              acc[i][t] = fmaf(xv[i].w, w3, a);
            }
          }
        }
      }
    } else {
      for (int kk = 0; kk < kn; ++kk) {
        const int k = k0 + kk;
        const int tap = k / r.slice_ci, j = k - tap * r.slice_ci;
        const int kh = tap / g.KW, kw = tap - kh * g.KW;
#pragma unroll
        for (int i = 0; i < PX; ++i) {
          const int ih = g.S * oh[i] - g.P + kh, iw = g.S * ow[i] - g.P + kw;
          if (!valid[i] || ih < 0 || ih >= g.H || iw < 0 || iw >= g.W) continue;
          const float xv =
              __ldg(x + ((n[i] * g.H + ih) * g.W + iw) * g.Ci + int64_t(grp) * r.slice_ci + j);
#pragma unroll
          for (int t = 0; t < CO_T; ++t) acc[i][t] = fmaf(xv, ws[kk][t], acc[i][t]);
        }
      }
    }
  }
  // stage the block's pixels x CO_T outputs in ws (row p rotated by p so the
  // per-thread writes are bank-conflict free), then store them with
  // consecutive threads on consecutive 16-byte pieces of each pixel's run
  __syncthreads();
#pragma unroll
  for (int i = 0; i < PX; ++i) {
    if (!valid[i]) continue;
    const int p = threadIdx.x + i * kFpPix;
#pragma unroll
    for (int t = 0; t < CO_T; ++t)
      ws[p][(t + p) & (CO_T - 1)] = (relu && !(acc[i][t] > 0.f)) ? 0.f : acc[i][t];  // I/nnet.hpp:138-139
  }
  __syncthreads();
  const int cbase = r.b + grp * r.slice_co + co0;
  const bool vec = (cbase % 4 == 0) && (g.Co % 4 == 0) && (nco % 4 == 0);
  if (vec) {
    const int quads = nco / 4;
    for (int e = threadIdx.x; e < kFpPix * PX * quads; e += kFpPix) {
      const int p = e / quads, qd = e - p * quads;
      if (pix0 + p >= npix) break;
      float4 o;
      o.x = ws[p][(4 * qd + p) & (CO_T - 1)];
      o.y = ws[p][(4 * qd + 1 + p) & (CO_T - 1)];
      o.z = ws[p][(4 * qd + 2 + p) & (CO_T - 1)];
      o.w = ws[p][(4 * qd + 3 + p) & (CO_T - 1)];
      *reinterpret_cast<float4*>(y + (pix0 + p) * g.Co + cbase + 4 * qd) = o;
    }
  } else {
    for (int e = threadIdx.x; e < kFpPix * PX * nco; e += kFpPix) {
      const int p = e / nco, t = e - p * nco;
      if (pix0 + p >= npix) break;
      y[(pix0 + p) * g.Co + cbase + t] = ws[p][(t + p) & (CO_T - 1)];
    }
  }
}

// Grouped / depthwise fprop with a shared-memory halo tile (ranges whose
// groups are too narrow for the tensor cores).  A block owns a tile of
// kGTH x kGTW output pixels of one image and CC output channels (whole
// groups); it stages the input halo rows x cols x (the groups' input
// channels) with coalesced float4 loads, and every thread keeps one output
// channel's weights in registers and accumulates its pixels from smem.
constexpr int kGPix = 256, kGThreads = 256;

// Output tile of the grouped kernel: up to 32 columns, rows filling 256 pixels.
struct GTile {
  int tw, th;
};
inline __host__ __device__ GTile gtile(int OH, int OW) {
  GTile t;
  t.tw = OW < 32 ? OW : 32;
  t.th = kGPix / t.tw;
  if (t.th > OH) t.th = OH;
  return t;
}

template <int CC, int KMAX>
__global__ void __launch_bounds__(kGThreads, KMAX <= 9 ? 4 : KMAX <= 36 ? 2 : 1)
    k_fprop_grouped(ConvGeom g, int ri,
                                                             const float* __restrict__ x,
                                                             const float* __restrict__ wbase,
                                                             float* __restrict__ y, bool relu) {
  extern __shared__ float halo[];  // [IH][IW][CIc]
  const RangeDesc r = g.r[ri];
  const float* __restrict__ wf = wbase + r.wf_off;
  const GTile T = gtile(g.OH, g.OW);
  const int tiles_w = (g.OW + T.tw - 1) / T.tw;
  const int oh0 = (blockIdx.x / tiles_w) * T.th, ow0 = (blockIdx.x % tiles_w) * T.tw;
  const int64_t n = blockIdx.y;
  const int c0 = blockIdx.z * CC;                     // first output channel (range-local)
  const int nco = min(CC, r.len - c0);
  const int gsb = c0 / r.slice_co;                    // first group of the chunk
  const int ci0 = gsb * r.slice_ci;                   // its first input channel
  const int gse = (c0 + nco - 1) / r.slice_co;        // last group
  const int cic = (gse - gsb + 1) * r.slice_ci;       // input channels staged
  const int IH = (T.th - 1) * g.S + g.KH, IW = (T.tw - 1) * g.S + g.KW;
  const int ih0 = oh0 * g.S - g.P, iw0 = ow0 * g.S - g.P;
  // ---- stage the halo (zero outside the image: padded taps add nothing)
  const bool vec = (cic % 4 == 0) && (ci0 % 4 == 0) && (g.Ci % 4 == 0);
  if (vec) {
    const int q4 = cic / 4;
    for (int e = threadIdx.x; e < IH * IW * q4; e += kGThreads) {
      const int q = e % q4, pc = e / q4, iw = pc % IW, ih = pc / IW;
      const int gh = ih0 + ih, gw = iw0 + iw;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gh >= 0 && gh < g.H && gw >= 0 && gw < g.W)
        v = __ldg(reinterpret_cast<const float4*>(x + ((n * g.H + gh) * g.W + gw) * g.Ci + ci0) + q);
      reinterpret_cast<float4*>(halo)[(ih * IW + iw) * q4 + q] = v;
    }
  } else {
    for (int e = threadIdx.x; e < IH * IW * cic; e += kGThreads) {
      const int q = e % cic, pc = e / cic, iw = pc % IW, ih = pc / IW;
      const int gh = ih0 + ih, gw = iw0 + iw;
      halo[e] = (gh >= 0 && gh < g.H && gw >= 0 && gw < g.W)
                    ? __ldg(x + ((n * g.H + gh) * g.W + gw) * g.Ci + ci0 + q)
                    : 0.f;
    }
  }
  __syncthreads();
  const int col = threadIdx.x % CC, lane_p = threadIdx.x / CC;
  constexpr int PL = kGThreads / CC;  // pixel lanes
  if (col >= nco) return;
  const int co = c0 + col;                       // range-local output channel
  const int cil = (co / r.slice_co - gsb) * r.slice_ci;  // its group's first staged input
  const int K = r.slice_ci * g.KH * g.KW;
  // per K element: its weight and its smem offset relative to the pixel
  float wr[KMAX];
  int off[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    const int kc = k < K ? k : K - 1;
    const int tap = kc / r.slice_ci, j = kc - tap * r.slice_ci;
    const int kh = tap / g.KW, kw = tap - kh * g.KW;
    wr[k] = k < K ? __ldg(wf + int64_t(k) * r.len + co) : 0.f;  // Wf[tap][j][co]
    off[k] = (kh * IW + kw) * cic + cil + j;
  }
  for (int p = lane_p; p < T.th * T.tw; p += PL) {
    const int th = p / T.tw, tw = p % T.tw;
    const int oh = oh0 + th, ow = ow0 + tw;
    if (oh >= g.OH || ow >= g.OW) continue;
    const float* hp = halo + (th * g.S * IW + tw * g.S) * cic;
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) acc = fmaf(hp[off[k]], wr[k], acc);
    y[((n * g.OH + oh) * g.OW + ow) * g.Co + r.b + co] = (relu && !(acc > 0.f)) ? 0.f : acc;
  }
}

// 3x3 stride-1 grouped / depthwise fprop (groups of SLICE input channels):
// the halo is staged channel-major ([channel][row][col], plane stride = 1
// mod 32 so the 32 channels of a warp hit 32 banks), each thread owns one
// output channel with its 9*SLICE weights in registers and produces 4
// adjacent output pixels of a row per step: 6 shared loads per (input
// channel, tap row) feed 12 FMAs, with constant-offset addressing.
template <int SLICE>
__global__ void __launch_bounds__(kGThreads, SLICE <= 2 ? 4 : 2)
    k_fprop_grouped3(ConvGeom g, int ri, const float* __restrict__ x,
                     const float* __restrict__ wbase, float* __restrict__ y, bool relu) {
  extern __shared__ float halo[];  // [cic][IH][IW] with plane stride PS
  const RangeDesc r = g.r[ri];
  const float* __restrict__ wf = wbase + r.wf_off;
  const GTile T = gtile(g.OH, g.OW);
  const int tiles_w = (g.OW + T.tw - 1) / T.tw;
  const int oh0 = (blockIdx.x / tiles_w) * T.th, ow0 = (blockIdx.x % tiles_w) * T.tw;
  const int64_t n = blockIdx.y;
  const int c0 = blockIdx.z * 32;
  const int nco = min(32, r.len - c0);
  const int gsb = c0 / r.slice_co, gse = (c0 + nco - 1) / r.slice_co;
  const int ci0 = gsb * SLICE, cic = (gse - gsb + 1) * SLICE;
  const int IH = T.th + 2, IW = T.tw + 2 + 3;  // +3: the last quad may read past the tile
  const int PS = ((IH * IW + 31) / 32) * 32 + 1;
  const int ih0 = oh0 - g.P, iw0 = ow0 - g.P;
  if ((cic & 3) == 0 && (ci0 & 3) == 0 && (g.Ci & 3) == 0) {
    const int q4 = cic / 4;
    for (int e = threadIdx.x; e < IH * IW * q4; e += kGThreads) {
      const int q = e % q4, pc = e / q4, iw = pc % IW, ih = pc / IW;
      const int gh = ih0 + ih, gw = iw0 + iw;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gh >= 0 && gh < g.H && gw >= 0 && gw < g.W && iw < T.tw + 2)
        v = __ldg(reinterpret_cast<const float4*>(x + ((n * g.H + gh) * g.W + gw) * g.Ci + ci0) + q);
      float* d = halo + 4 * q * PS + pc;
      d[0] = v.x;
      d[PS] = v.y;
      d[2 * PS] = v.z;
      d[3 * PS] = v.w;
    }
  } else {
    for (int e = threadIdx.x; e < IH * IW * cic; e += kGThreads) {
      const int q = e % cic, pc = e / cic, iw = pc % IW, ih = pc / IW;
      const int gh = ih0 + ih, gw = iw0 + iw;
      halo[q * PS + pc] = (gh >= 0 && gh < g.H && gw >= 0 && gw < g.W && iw < T.tw + 2)
                              ? __ldg(x + ((n * g.H + gh) * g.W + gw) * g.Ci + ci0 + q)
                              : 0.f;
    }
  }
  __syncthreads();
  // weights: registers for narrow groups, else a [tap*SLICE + j][32] smem
  // block after the halo (column = the thread's output channel)
  constexpr bool kRegW = SLICE <= 4;
  float* wsm = halo + cic * PS;
  if (!kRegW) {
    for (int e = threadIdx.x; e < 9 * SLICE * 32; e += kGThreads) {
      const int cc = e & 31, k = e >> 5;
      wsm[e] = cc < nco ? __ldg(wf + int64_t(k) * r.len + c0 + cc) : 0.f;
    }
    __syncthreads();
  }
  const int col = threadIdx.x & 31, lane_p = threadIdx.x >> 5;
  constexpr int PL = kGThreads / 32;
  if (col >= nco) return;
  const int co = c0 + col;
  const int cil = (co / r.slice_co - gsb) * SLICE;
  float w3[kRegW ? SLICE : 1][9];
  if (kRegW) {
#pragma unroll
    for (int j = 0; j < (kRegW ? SLICE : 1); ++j)
#pragma unroll
      for (int t = 0; t < 9; ++t) w3[j][t] = __ldg(wf + int64_t(t * SLICE + j) * r.len + co);
  }
  auto wt = [&](int j, int t) {
    if constexpr (kRegW) return w3[j][t];
    else return wsm[(t * SLICE + j) * 32 + col];
  };
  const int quads_w = (T.tw + 3) / 4;
  float* yb = y + r.b + co;
  for (int qd = lane_p; qd < T.th * quads_w; qd += PL) {
    const int th = qd / quads_w, tw = (qd - th * quads_w) * 4;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll(kRegW ? SLICE : 1)
    for (int j = 0; j < SLICE; ++j) {
      const float* hp = halo + (cil + j) * PS + th * IW + tw;
#pragma unroll
      for (int kh = 0; kh < 3; ++kh) {
        float v[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) v[i] = hp[kh * IW + i];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int kw = 0; kw < 3; ++kw) acc[q] = fmaf(v[q + kw], wt(j, kh * 3 + kw), acc[q]);
      }
    }
    const int oh = oh0 + th;
    if (oh >= g.OH) continue;
    const int64_t rowb = (n * g.OH + oh) * int64_t(g.OW);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int ow = ow0 + tw + q;
      if (tw + q < T.tw && ow < g.OW)
        yb[(rowb + ow) * g.Co] = (relu && !(acc[q] > 0.f)) ? 0.f : acc[q];
    }
  }
}

// 3x3 stride-1 dgrad of a single-range grouped / depthwise layer (groups of
// SLICE = slice_co output channels), same structure as k_fprop_grouped3:
// g[ih,iw,ci] = sum_t sum_{kh,kw} Wd[kh,kw][t][ci] * dpre[ih+P-kh, iw+P-kw,
// co(t)] over the dpre halo (rows / cols past the cropped output are zero),
// with the fused epilogue of k_dgrad_direct: g_out, the ReLU-masked dpre of
// the previous layer and per-(image, tile, channel) partials of A*g summed in
// a fixed order (tile = the gtile() grid over H x W).
template <int SLICE>
__global__ void __launch_bounds__(kGThreads, SLICE <= 2 ? 4 : 2)
    k_dgrad_grouped3(ConvGeom g, const float* __restrict__ dpre, const float* __restrict__ wbase,
                     const float* __restrict__ a_prev, bool relu_prev, float* __restrict__ dpre_out,
                     float* __restrict__ g_out, double* __restrict__ partial) {
  extern __shared__ float halo[];  // [cst][IH][IW] plane stride PS, then weights
  __shared__ float red[kGThreads / 32][33];
  const RangeDesc r = g.r[0];
  const float* __restrict__ wd = wbase + r.wd_off;
  const GTile T = gtile(g.H, g.W);
  const int tiles_w = (g.W + T.tw - 1) / T.tw;
  const int tile = blockIdx.x;
  const int ih0t = (tile / tiles_w) * T.th, iw0t = (tile % tiles_w) * T.tw;
  const int64_t n = blockIdx.y;
  const int c0 = blockIdx.z * 32;              // first dgrad-output (input) channel
  const int nci = min(32, g.Ci - c0);
  const int gsb = c0 / r.slice_ci, gse = (c0 + nci - 1) / r.slice_ci;
  const int co0 = r.b + gsb * SLICE, cst = (gse - gsb + 1) * SLICE;  // staged dpre channels
  const int IH = T.th + 2, IW = T.tw + 2 + 3;
  const int PS = ((IH * IW + 31) / 32) * 32 + 1;
  const int oh0 = ih0t + g.P - 2, ow0 = iw0t + g.P - 2;  // first dpre row / col needed
  if ((cst & 3) == 0 && (co0 & 3) == 0 && (g.Co & 3) == 0) {
    const int q4 = cst / 4;
    for (int e = threadIdx.x; e < IH * IW * q4; e += kGThreads) {
      const int q = e % q4, pc = e / q4, iw = pc % IW, ih = pc / IW;
      const int gh = oh0 + ih, gw = ow0 + iw;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gh >= 0 && gh < g.OH && gw >= 0 && gw < g.OW && iw < T.tw + 2)
        v = __ldg(reinterpret_cast<const float4*>(dpre + ((n * g.OH + gh) * g.OW + gw) * g.Co + co0) + q);
      float* d = halo + 4 * q * PS + pc;
      d[0] = v.x;
      d[PS] = v.y;
      d[2 * PS] = v.z;
      d[3 * PS] = v.w;
    }
  } else {
    for (int e = threadIdx.x; e < IH * IW * cst; e += kGThreads) {
      const int q = e % cst, pc = e / cst, iw = pc % IW, ih = pc / IW;
      const int gh = oh0 + ih, gw = ow0 + iw;
      halo[q * PS + pc] = (gh >= 0 && gh < g.OH && gw >= 0 && gw < g.OW && iw < T.tw + 2)
                              ? __ldg(dpre + ((n * g.OH + gh) * g.OW + gw) * g.Co + co0 + q)
                              : 0.f;
    }
  }
  constexpr bool kRegW = SLICE <= 4;
  float* wsm = halo + cst * PS;
  if (!kRegW) {
    for (int e = threadIdx.x; e < 9 * SLICE * 32; e += kGThreads) {
      const int cc = e & 31, k = e >> 5;  // k = tap * SLICE + t
      wsm[e] = cc < nci ? __ldg(wd + int64_t(k) * g.Ci + c0 + cc) : 0.f;
    }
  }
  __syncthreads();
  const int col = threadIdx.x & 31, lane_p = threadIdx.x >> 5;
  constexpr int PL = kGThreads / 32;
  const bool act = col < nci;
  const int ci = c0 + col;
  const int tl = act ? (ci / r.slice_ci - gsb) * SLICE : 0;  // first staged dpre channel of its group
  float w3[kRegW ? SLICE : 1][9];
  if (kRegW && act) {
#pragma unroll
    for (int t = 0; t < (kRegW ? SLICE : 1); ++t)
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) w3[t][tap] = __ldg(wd + int64_t(tap * SLICE + t) * g.Ci + ci);
  }
  auto wt = [&](int t, int tap) {
    if constexpr (kRegW) return w3[t][tap];
    else return wsm[(tap * SLICE + t) * 32 + col];
  };
  const int quads_w = (T.tw + 3) / 4;
  float contrib = 0.f;
  if (act) {
    for (int qd = lane_p; qd < T.th * quads_w; qd += PL) {
      const int th = qd / quads_w, tw = (qd - th * quads_w) * 4;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll(kRegW ? SLICE : 1)
      for (int t = 0; t < SLICE; ++t) {
        const float* hp = halo + (tl + t) * PS + th * IW + tw;
#pragma unroll
        for (int rr = 0; rr < 3; ++rr) {  // staged row th + rr holds dpre row ih + P - (2 - rr)
          float v[6];
#pragma unroll
          for (int i = 0; i < 6; ++i) v[i] = hp[rr * IW + i];
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc)
              acc[q] = fmaf(v[q + cc], wt(t, (2 - rr) * 3 + (2 - cc)), acc[q]);
        }
      }
      const int ih = ih0t + th;
      if (ih >= g.H) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int iw = iw0t + tw + q;
        if (tw + q >= T.tw || iw >= g.W) continue;
        const int64_t idx = ((n * g.H + ih) * g.W + iw) * g.Ci + ci;
        if (g_out) g_out[idx] = acc[q];
        if (a_prev) {
          const float a = a_prev[idx];
          contrib = fmaf(a, acc[q], contrib);
          if (dpre_out) dpre_out[idx] = (relu_prev && !(a > 0.f)) ? 0.f : acc[q];  // I/nnet.hpp:229-233
        } else if (dpre_out) {
          dpre_out[idx] = acc[q];
        }
      }
    }
  }
  if (!partial) return;
  red[lane_p][col] = contrib;
  __syncthreads();
  if (lane_p == 0 && act) {
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < PL; ++k) sum += red[k][col];
    partial[(n * gridDim.x + tile) * g.Ci + ci] = double(sum);
  }
}

// Depthwise fprop (slice_ci = slice_co = 1): threads run over channels
// (coalesced NHWC loads and stores), each computing kDwRun consecutive
// output pixels of one row with its channel's taps held in registers.
constexpr int kDwRun = 4;

__global__ void __launch_bounds__(256) k_fprop_dw(ConvGeom g, int ri,
                                                  const float* __restrict__ x,
                                                  const float* __restrict__ wbase,
                                                  float* __restrict__ y, bool relu) {
  const RangeDesc r = g.r[ri];
  const int c = blockIdx.x * 32 + threadIdx.x;  // channel within the range
  if (c >= r.len) return;
  const int runs_w = (g.OW + kDwRun - 1) / kDwRun;
  const int64_t unit = int64_t(blockIdx.y) * 8 + threadIdx.y;  // (n, oh, run)
  if (unit >= int64_t(g.N) * g.OH * runs_w) return;
  const int run = int(unit % runs_w);
  const int oh = int((unit / runs_w) % g.OH);
  const int64_t n = unit / (int64_t(runs_w) * g.OH);
  const int ci = c * r.slice_ci / r.slice_co;  // == c for depthwise
  const float* __restrict__ wf = wbase + r.wf_off;
  float acc[kDwRun];
#pragma unroll
  for (int q = 0; q < kDwRun; ++q) acc[q] = 0.f;
  for (int kh = 0; kh < g.KH; ++kh) {
    const int ih = g.S * oh - g.P + kh;
    if (ih < 0 || ih >= g.H) continue;
    const float* __restrict__ xr = x + (n * g.H + ih) * int64_t(g.W) * g.Ci + r.b + ci;
    for (int kw = 0; kw < g.KW; ++kw) {
      const float wv = __ldg(wf + int64_t(kh * g.KW + kw) * r.len + c);
#pragma unroll
      for (int q = 0; q < kDwRun; ++q) {
        const int ow = run * kDwRun + q;
        const int iw = g.S * ow - g.P + kw;
        if (ow < g.OW && iw >= 0 && iw < g.W) acc[q] = fmaf(__ldg(xr + int64_t(iw) * g.Ci), wv, acc[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kDwRun; ++q) {
    const int ow = run * kDwRun + q;
    if (ow < g.OW)
      y[((n * g.OH + oh) * g.OW + ow) * g.Co + r.b + c] = (relu && !(acc[q] > 0.f)) ? 0.f : acc[q];
  }
}

// Direct dgrad (the dgrad MAC loop of I/nnet.hpp:235-243 as a gather):
// g[n,ih,iw,ci] = sum_r sum_t sum_{kh,kw} Wd_r[tap][t][ci] *
// dpre[n, oh, ow, b_r + (ci/slice_ci_r)*slice_co_r + t] with
// oh = (ih+p-kh)/s when integral and inside the (cropped) output.
// Block = 32 channels x 8 pixel lanes; grid = (ci tiles, pixel tiles, N).
// Fused epilogue: partial[n][tile][ci] = sum over the tile of A*g in a fixed
// order (deterministic), dpre_out = g masked by the previous layer's ReLU.
__global__ void __launch_bounds__(256) k_dgrad_direct(
    ConvGeom g, const float* __restrict__ dpre, const float* __restrict__ wbase,
    const float* __restrict__ a_prev, bool relu_prev, float* __restrict__ dpre_out,
    float* __restrict__ g_out, double* __restrict__ partial) {
  __shared__ float red[8][33];
  const int ci = blockIdx.x * 32 + threadIdx.x;
  const int tile = blockIdx.y;
  const int64_t n = blockIdx.z;
  const int HW = g.H * g.W;
  const int p0 = tile * kDgradTilePix;
  const int p1 = min(HW, p0 + kDgradTilePix);
  float contrib = 0.f;
  if (ci < g.Ci) {
    for (int p = p0 + threadIdx.y; p < p1; p += 8) {
      const int ih = p / g.W, iw = p - (p / g.W) * g.W;
      float acc = 0.f;
      for (int ri = 0; ri < g.nranges; ++ri) {
        const RangeDesc r = g.r[ri];
        const float* __restrict__ wd = wbase + r.wd_off;
        const int co0 = r.b + (ci / r.slice_ci) * r.slice_co;
        for (int kh = 0; kh < g.KH; ++kh) {
          const int th = ih + g.P - kh;
          if (th < 0) break;
          if (th % g.S) continue;
          const int oh = th / g.S;
          if (oh >= g.OH) continue;
          for (int kw = 0; kw < g.KW; ++kw) {
            const int tw = iw + g.P - kw;
            if (tw < 0) break;
            if (tw % g.S) continue;
            const int ow = tw / g.S;
            if (ow >= g.OW) continue;
            const float* __restrict__ dr = dpre + ((n * g.OH + oh) * g.OW + ow) * g.Co + co0;
            const float* __restrict__ wr =
                wd + int64_t(kh * g.KW + kw) * r.slice_co * g.Ci + ci;
#pragma unroll 4
            for (int t = 0; t < r.slice_co; ++t) acc = fmaf(wr[int64_t(t) * g.Ci], dr[t], acc);
          }
        }
      }
      const int64_t idx = (n * HW + p) * g.Ci + ci;
      if (g_out) g_out[idx] = acc;
      if (a_prev) {
        const float a = a_prev[idx];
        contrib = fmaf(a, acc, contrib);
        if (dpre_out) dpre_out[idx] = (relu_prev && !(a > 0.f)) ? 0.f : acc;  // I/nnet.hpp:229-233
      } else if (dpre_out) {
        dpre_out[idx] = acc;
      }
    }
  }
  if (!partial) return;
  red[threadIdx.y][threadIdx.x] = contrib;
  __syncthreads();
  if (threadIdx.y == 0 && ci < g.Ci) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    partial[(n * gridDim.y + tile) * g.Ci + ci] = double(s);
  }
}

// One block per example; fp64 throughout (head_logits/softmax/CE,
// I/nnet.hpp:152-194; dz/dpool/g[L-1], I/nnet.hpp:209-224).
__global__ void __launch_bounds__(512) k_head(HeadArgs a) {
  extern __shared__ double sm[];
  double* pooled = sm;            // C
  double* dpool = sm + a.C;       // C
  double* z = sm + 2 * a.C;       // K
  double* dz = z + a.K;           // K
  double* rsum = dz + a.K;        // blockDim: per-(row group, channel) partial sums
  const int n = blockIdx.x;
  const float* act = a.act + int64_t(n) * a.HW * a.C;
  // narrow layers (C < blockDim): R row groups per channel, combined in
  // group order, so a small batch still keeps every thread busy
  const int R = a.C < int(blockDim.x) ? int(blockDim.x) / a.C : 1;
  const int rg = int(threadIdx.x) / a.C, rc = int(threadIdx.x) % a.C;
  if (R > 1) {
    if (rg < R) {
      double s = 0.0;
      for (int j = rg; j < a.HW; j += R) s += double(act[int64_t(j) * a.C + rc]);
      rsum[rg * a.C + rc] = s;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < a.C; i += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < R; ++q) s += rsum[q * a.C + i];
      pooled[i] = s / double(a.HW);
    }
  } else {
    for (int i = threadIdx.x; i < a.C; i += blockDim.x) {
      double s = 0.0;
      for (int j = 0; j < a.HW; ++j) s += double(act[int64_t(j) * a.C + i]);
      pooled[i] = s / double(a.HW);
    }
  }
  __syncthreads();
  // logits: one warp per class, lanes stride the channels, fixed-order
  // xor-butterfly (fp64) -- the class loop no longer runs serially
  {
    const int wid = threadIdx.x / 32, ln = threadIdx.x % 32, nw = blockDim.x / 32;
    for (int k = wid; k < a.K; k += nw) {
      double s = 0.0;
      for (int i = ln; i < a.C; i += 32)
        s += (a.head_src[int64_t(k) * a.C + i] * a.head_scale) * pooled[i];
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (ln == 0) z[k] = s;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = z[0];
    for (int k = 0; k < a.K; ++k) m = fmax(m, z[k]);
    double sum = 0.0;
    for (int k = 0; k < a.K; ++k) sum += (dz[k] = exp(z[k] - m));
    for (int k = 0; k < a.K; ++k) dz[k] /= sum;
    const int y = a.labels[n];
    a.ex_loss[n] = -log(fmax(dz[y], 1e-300));
    for (int k = 0; k < a.K; ++k) a.probs[int64_t(n) * a.K + k] = dz[k];
    dz[y] -= 1.0;
    for (int k = 0; k < a.K; ++k) dz[k] /= a.grad_n;
  }
  __syncthreads();
  if (!a.backward) return;
  for (int i = threadIdx.x; i < a.C; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < a.K; ++k) s += (a.head_src[int64_t(k) * a.C + i] * a.head_scale) * dz[k];
    dpool[i] = s;
  }
  __syncthreads();
  if (R > 1) {
    if (rg < R) {
      const double gv = dpool[rc] / double(a.HW);
      const float gf = float(gv);
      double s = 0.0;
      for (int j = rg; j < a.HW; j += R) {
        const int64_t idx = (int64_t(n) * a.HW + j) * a.C + rc;
        const float av = a.act[idx];
        s += double(av) * gv;
        if (a.dpre) a.dpre[idx] = (a.relu_last && !(av > 0.f)) ? 0.f : gf;
        if (a.g_out) a.g_out[idx] = gf;
      }
      rsum[rg * a.C + rc] = s;
    }
    __syncthreads();
    if (a.partial)
      for (int i = threadIdx.x; i < a.C; i += blockDim.x) {
        double s = 0.0;
        for (int q = 0; q < R; ++q) s += rsum[q * a.C + i];
        a.partial[int64_t(n) * a.C + i] = s;
      }
    return;
  }
  for (int i = threadIdx.x; i < a.C; i += blockDim.x) {
    const double gv = dpool[i] / double(a.HW);
    const float gf = float(gv);
    double s = 0.0;
    for (int j = 0; j < a.HW; ++j) {
      const int64_t idx = (int64_t(n) * a.HW + j) * a.C + i;
      const float av = a.act[idx];
      s += double(av) * gv;
      if (a.dpre) a.dpre[idx] = (a.relu_last && !(av > 0.f)) ? 0.f : gf;
      if (a.g_out) a.g_out[idx] = gf;
    }
    if (a.partial) a.partial[int64_t(n) * a.C + i] = s;
  }
}

// delta[l][c] = (sum_n s_nc^2) / (2N), s_nc = -sum_tiles partial (fixed
// order), I/nnet.hpp:330-345.  Block = 32 channels x 16 example lanes; the
// 16 lane sums are combined in a fixed order (deterministic, fp64).
__global__ void __launch_bounds__(512) k_fisher_reduce(const FisherLayer* __restrict__ layers,
                                                       int N, double* __restrict__ per_channel,
                                                       double* __restrict__ s_out, int64_t s_ld) {
  __shared__ double red[16][33];
  const FisherLayer L = layers[blockIdx.y];
  const int c = blockIdx.x * 32 + threadIdx.x;
  if (blockIdx.x * 32 >= L.C) return;
  double acc = 0.0;
  if (c < L.C) {
    for (int n = threadIdx.y; n < N; n += 16) {
      const double* p = L.partial + int64_t(n) * L.nstride + c;
      double s = 0.0;
      for (int t = 0; t < L.tiles; ++t) s -= p[int64_t(t) * L.C];
      if (s_out) s_out[int64_t(n) * s_ld + L.out_off + c] = s;
      acc += s * s;
    }
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c < L.C) {
    double tot = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) tot += red[k][threadIdx.x];
    per_channel[L.out_off + c] = tot / (2.0 * double(N));
  }
}

// Split-K epilogue: block = 32 channels x 8 pixel lanes, grid = (channel
// tiles, N); each thread walks pixels p = lane, lane+8, ... of one image.
__global__ void __launch_bounds__(256) k_splitk_epilogue(SplitEpi e) {
  __shared__ float red[8][33];
  // launched with programmatic stream serialization: let the next conv
  // launch early, then wait for the split units this reduces
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int64_t n = blockIdx.y;
  const int cs = (e.HW + e.hw_chunks - 1) / e.hw_chunks, pend = min(e.HW, int(blockIdx.z + 1) * cs);
  float contrib = 0.f;
  float mx = 0.f;  // max |stored value| for the next fp16-split GEMM (image n)
  if (c < e.C) {
    for (int p = int(blockIdx.z) * cs + threadIdx.y; p < pend; p += 8) {
      const int64_t idx = (n * e.HW + p) * e.ld + e.c0 + c;
      float v = 0.f;
      for (int k = 0; k < e.ksplit; ++k) v += e.ws[k * e.ws_stride + idx];
      if (e.mode == 0) {
        const float o = (e.relu && !(v > 0.f)) ? 0.f : v;  // I/nnet.hpp:138-139
        e.out[idx] = o;
        mx = fmaxf(mx, fabsf(o));
      } else {
        if (e.g_out) e.g_out[idx] = v;
        if (e.a_prev) {
          const float a = e.a_prev[idx];
          contrib = fmaf(a, v, contrib);
          if (e.dpre_out) {
            const float o = (e.relu_prev && !(a > 0.f)) ? 0.f : v;
            e.dpre_out[idx] = o;
            mx = fmaxf(mx, fabsf(o));
          }
        } else if (e.dpre_out) {
          e.dpre_out[idx] = v;
          mx = fmaxf(mx, fabsf(v));
        }
      }
    }
  }
  if (e.out_amax) {  // one atomic per warp (the block is one image)
    const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
    if (threadIdx.x == 0 && m) atomicMax(e.out_amax + n, m);
  }
  if (e.mode == 0 || !e.partial) return;
  red[threadIdx.y][threadIdx.x] = contrib;
  __syncthreads();
  if (threadIdx.y == 0 && c < e.C) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    e.partial[(n * e.hw_chunks + blockIdx.z) * e.ld + e.c0 + c] = double(s);
  }
}

// k_splitk_epilogue with float4 channel quads (C, ld, c0 multiples of 4):
// thread (tx, ty) of block (cq, n) owns channels 4*(32*cq + tx) .. +3 and the
// pixels ty, ty + 8, ...; same fixed summation orders as the scalar kernel.
__global__ void __launch_bounds__(256) k_splitk_epilogue4(SplitEpi e) {
  __shared__ float red[8][129];
  // launched with programmatic stream serialization: let the next conv
  // launch early, then wait for the split units this reduces
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int c = (blockIdx.x * 32 + threadIdx.x) * 4;
  const int64_t n = blockIdx.y;
  const int cs = (e.HW + e.hw_chunks - 1) / e.hw_chunks, pend = min(e.HW, int(blockIdx.z + 1) * cs);
  float contrib[4] = {0.f, 0.f, 0.f, 0.f};
  float mx = 0.f;  // max |stored value| for the next fp16-split GEMM (image n)
  if (c < e.C) {
    // the partials and A_prev are read-only here: every load of a pixel is
    // issued (non-coherent path) before its sums, and two splits at a time
#pragma unroll 2
    for (int p = int(blockIdx.z) * cs + threadIdx.y; p < pend; p += 8) {
      const int64_t idx = (n * e.HW + p) * e.ld + e.c0 + c;
      const float4* wsp = reinterpret_cast<const float4*>(e.ws + idx);
      const int64_t wst = e.ws_stride / 4;
      const float4 w0 = __ldg(wsp);
      const float4 w1 = e.ksplit > 1 ? __ldg(wsp + wst) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 a = e.mode == 1 && e.a_prev ? __ldg(reinterpret_cast<const float4*>(e.a_prev + idx))
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      v.x += w0.x;
      v.y += w0.y;
      v.z += w0.z;
      v.w += w0.w;
      if (e.ksplit > 1) {
        v.x += w1.x;
        v.y += w1.y;
        v.z += w1.z;
        v.w += w1.w;
      }
      for (int k = 2; k < e.ksplit; ++k) {
        const float4 w = __ldg(wsp + k * wst);
        v.x += w.x;
        v.y += w.y;
        v.z += w.z;
        v.w += w.w;
      }
      if (e.mode == 0) {
        if (e.relu) {
          v.x = v.x > 0.f ? v.x : 0.f;
          v.y = v.y > 0.f ? v.y : 0.f;
          v.z = v.z > 0.f ? v.z : 0.f;
          v.w = v.w > 0.f ? v.w : 0.f;
        }
        *reinterpret_cast<float4*>(e.out + idx) = v;
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      } else {
        if (e.g_out) *reinterpret_cast<float4*>(e.g_out + idx) = v;
        if (e.a_prev) {
          contrib[0] = fmaf(a.x, v.x, contrib[0]);
          contrib[1] = fmaf(a.y, v.y, contrib[1]);
          contrib[2] = fmaf(a.z, v.z, contrib[2]);
          contrib[3] = fmaf(a.w, v.w, contrib[3]);
          if (e.dpre_out) {
            float4 d;
            d.x = (e.relu_prev && !(a.x > 0.f)) ? 0.f : v.x;
            d.y = (e.relu_prev && !(a.y > 0.f)) ? 0.f : v.y;
            d.z = (e.relu_prev && !(a.z > 0.f)) ? 0.f : v.z;
            d.w = (e.relu_prev && !(a.w > 0.f)) ? 0.f : v.w;
            *reinterpret_cast<float4*>(e.dpre_out + idx) = d;
            mx = fmaxf(mx, fmaxf(fmaxf(fabsf(d.x), fabsf(d.y)), fmaxf(fabsf(d.z), fabsf(d.w))));
          }
        } else if (e.dpre_out) {
          *reinterpret_cast<float4*>(e.dpre_out + idx) = v;
          mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
        }
      }
    }
  }
  if (e.out_amax) {  // one atomic per warp (the block is one image)
    const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
    if (threadIdx.x == 0 && m) atomicMax(e.out_amax + n, m);
  }
  if (e.mode == 0 || !e.partial) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) red[threadIdx.y][4 * threadIdx.x + i] = contrib[i];
  __syncthreads();
  const int t = threadIdx.y * 32 + threadIdx.x;
  if (t < 128 && blockIdx.x * 128 + t < e.C) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][t];
    e.partial[(n * e.hw_chunks + blockIdx.z) * e.ld + e.c0 + blockIdx.x * 128 + t] = double(s);
  }
}

int grid_for(int64_t total, int block) {
  int64_t g = (total + block - 1) / block;
  const int64_t cap = 148 * 32;
  return int(g < 1 ? 1 : (g > cap ? cap : g));
}

// per-image max |x| (blocks over (chunk, image); one atomic per warp)
__global__ void __launch_bounds__(256) k_amax(const float* __restrict__ x, int64_t per_img,
                                              uint32_t* __restrict__ amax) {
  const int64_t n = blockIdx.y;
  const float* p = x + n * per_img;
  float mx = 0.f;
  if (per_img % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const float4* q = reinterpret_cast<const float4*>(p);
    for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < per_img / 4; i += int64_t(gridDim.x) * 256) {
      const float4 v = q[i];
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
  } else {
    for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < per_img; i += int64_t(gridDim.x) * 256)
      mx = fmaxf(mx, fabsf(p[i]));
  }
  const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(mx));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(amax + n, m);
}

}  // namespace

void launch_nchw64_to_nhwc32(const double* src, float* dst, int64_t N, int C, int H, int W,
                             cudaStream_t st) {
  const int64_t total = N * C * H * W;
  k_nchw64_to_nhwc32<<<grid_for(total, 256), 256, 0, st>>>(src, dst, N, C, H, W);
}

void launch_nhwc32_to_nchw64(const float* src, double* dst, int64_t N, int C, int H, int W,
                             cudaStream_t st) {
  const int64_t total = N * C * H * W;
  k_nhwc32_to_nchw64<<<grid_for(total, 256), 256, 0, st>>>(src, dst, N, C, H, W);
}

void launch_pack_weights(const double* src, double scale, const ConvGeom& g, int range,
                         const PackDst& d, cudaStream_t st) {
  const RangeDesc& r = g.r[range];
  const int taps = g.KH * g.KW;
  const int64_t total = int64_t(r.len) * r.slice_ci * taps;
  k_pack_weights<<<grid_for(total, 256), 256, 0, st>>>(src, scale, g.Ci, taps, r, d);
}

// shared memory of k_fprop_grouped3 for a 32-channel output chunk
size_t grouped3_smem(const ConvGeom& g, const RangeDesc& r) {
  const GTile T = gtile(g.OH, g.OW);
  const int cic = ((32 + r.slice_co - 1) / r.slice_co + 1) * r.slice_ci;
  const int IH3 = T.th + 2, IW3 = T.tw + 5;
  return (size_t(cic) * (((IH3 * IW3 + 31) / 32) * 32 + 1) + 9 * size_t(r.slice_ci) * 32) * 4;
}

bool grouped3_ok(const ConvGeom& g, const RangeDesc& r) {
  return r.groups >= 2 && g.KH == 3 && g.KW == 3 && g.S == 1 &&
         (r.slice_ci == 1 || r.slice_ci == 2 || r.slice_ci == 4 || r.slice_ci == 8 ||
          r.slice_ci == 16) &&
         grouped3_smem(g, r) <= 200 * 1024;
}

bool grouped_smem_ok(const ConvGeom& g, const RangeDesc& r) {
  if (grouped3_ok(g, r)) return true;
  if (r.groups < 2 || g.S > 2) return false;
  const int K = r.slice_ci * g.KH * g.KW;
  if (K > 64) return false;
  // the staged input channels of a 32-channel output chunk
  const int groups_per_chunk = (32 + r.slice_co - 1) / r.slice_co + 1;
  const int cic = groups_per_chunk * r.slice_ci;
  const GTile T = gtile(g.OH, g.OW);
  const int IH = (T.th - 1) * g.S + g.KH, IW = (T.tw - 1) * g.S + g.KW;
  return size_t(IH) * IW * cic * 4 <= 96 * 1024;
}

// Depthwise 3x3 stride-1 pad-1 fprop as a register sliding window (NHWC).
// DRAM sees each input and output once (plus the strips' halo rows); with
// one output column per thread every input pixel also crossed L1 three times
// and the loop was load-instruction bound (47% of HBM on 64@56, N=256); eight
// columns per thread load each pixel once per column block: 65% (profiles/).
constexpr int kDwStrip = 16;

// V = channels per thread (1 or 2): vector type and its lanes
template <int V>
struct DwVec;
template <>
struct DwVec<1> {
  using T = float;
  __device__ static float zero() { return 0.f; }
  __device__ static float& at(float& v, int) { return v; }
};
template <>
struct DwVec<2> {
  using T = float2;
  __device__ static float2 zero() { return make_float2(0.f, 0.f); }
  __device__ static float& at(float2& v, int i) { return i ? v.y : v.x; }
};

// Thread = V adjacent channels x OWB adjacent output columns of a
// `strip`-row strip; a register window of 3
// input rows x (OWB + 2) columns slides down the strip (each input pixel is
// loaded once per thread column block, the next row is in flight while the
// current one computes).  A warp covers 32 channel groups of one column
// block: its loads and stores are contiguous channel runs.
template <int V, int OWB>
__global__ void __launch_bounds__(256, OWB == 1 ? (V == 1 ? 8 : 4) : (OWB == 2 ? 3 : 2))
    k_dw3_nhwc(ConvGeom g, int ri, const float* __restrict__ x, const float* __restrict__ wbase,
               float* __restrict__ y, bool relu, int strip) {
  using DV = DwVec<V>;
  using T = typename DV::T;
  constexpr int WW = OWB + 2;
  const RangeDesc r = g.r[ri];
  const int np = r.len / V;
  const int p = blockIdx.z * blockDim.x + threadIdx.x;  // channel group (range-local)
  const int ow0 = (blockIdx.x * blockDim.y + threadIdx.y) * OWB;
  const int strips = (g.OH + strip - 1) / strip;
  const int64_t n = blockIdx.y / strips;
  const int oh0 = int(blockIdx.y % strips) * strip, oh1 = min(g.OH, oh0 + strip);
  if (p >= np || ow0 >= g.OW) return;
  const int c = V * p;  // depthwise: input channel == range-local output channel
  const float* __restrict__ wf = wbase + r.wf_off;  // Wf[tap][0][co]
  T w[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) w[t] = __ldg(reinterpret_cast<const T*>(wf + int64_t(t) * r.len + c));
  const int64_t row = int64_t(g.W) * g.Ci;
  const float* __restrict__ xn = x + n * g.H * row + c;
  auto ld = [&](int ih, int iw) {
    return (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W)
               ? __ldg(reinterpret_cast<const T*>(xn + ih * row + int64_t(iw) * g.Ci))
               : DV::zero();
  };
  T win[3][WW];  // [input row - (oh - 1)][input column - (ow0 - 1)]
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < WW; ++j) win[i][j] = ld(oh0 - 1 + i, ow0 - 1 + j);
  float* __restrict__ yp = y + (n * g.OH * g.OW + ow0) * int64_t(g.Co) + r.b + c;
  for (int oh = oh0; oh < oh1; ++oh) {
    T nxt[WW];  // the next step's input row, in flight while this one computes
#pragma unroll
    for (int j = 0; j < WW; ++j) nxt[j] = oh + 1 < oh1 ? ld(oh + 2, ow0 - 1 + j) : DV::zero();
#pragma unroll
    for (int o = 0; o < OWB; ++o) {
      T a = DV::zero();
#pragma unroll
      for (int kh = 0; kh < 3; ++kh)
#pragma unroll
        for (int kw = 0; kw < 3; ++kw)
#pragma unroll
          for (int i = 0; i < V; ++i)
            DV::at(a, i) = fmaf(DV::at(win[kh][o + kw], i), DV::at(w[kh * 3 + kw], i), DV::at(a, i));
      if (relu)
#pragma unroll
        for (int i = 0; i < V; ++i) DV::at(a, i) = DV::at(a, i) > 0.f ? DV::at(a, i) : 0.f;
      if (OWB == 1 || ow0 + o < g.OW)
        *reinterpret_cast<T*>(yp + (int64_t(oh) * g.OW + o) * g.Co) = a;
    }
#pragma unroll
    for (int j = 0; j < WW; ++j) {
      win[0][j] = win[1][j];
      win[1][j] = win[2][j];
      win[2][j] = nxt[j];
    }
  }
}

// dgrad of a depthwise 3x3 stride-1 pad-1 layer on the same register window
// (thread = a channel pair x OWB input columns of a strip of input rows):
// g[ih, iw] = sum_{kh,kw} W[kh,kw] * dpre[ih + 1 - kh, iw + 1 - kw], with the
// fused epilogue of k_dgrad_grouped3 (g_out, the ReLU-masked dpre of the
// previous layer, A*g partials).  Partials: one per (image, tile, channel),
// tile = (strip, column-block group); the block's column blocks are summed
// in threadIdx.y order (deterministic).
template <int OWB>
__global__ void __launch_bounds__(256, 2)
    k_dgrad_dw3(ConvGeom g, const float* __restrict__ dpre, const float* __restrict__ wbase,
                const float* __restrict__ a_prev, bool relu_prev, float* __restrict__ dpre_out,
                float* __restrict__ g_out, double* __restrict__ partial, int strip) {
  constexpr int WW = OWB + 2;
  __shared__ float2 red[256];
  const RangeDesc r = g.r[0];
  const int np = g.Ci / 2;
  const int p = blockIdx.z * blockDim.x + threadIdx.x;  // channel pair
  const int iw0 = (blockIdx.x * blockDim.y + threadIdx.y) * OWB;
  const int strips = (g.H + strip - 1) / strip;
  const int64_t n = blockIdx.y / strips;
  const int sidx = int(blockIdx.y % strips);
  const int ih0 = sidx * strip, ih1 = min(g.H, ih0 + strip);
  const int c = 2 * p;
  float2 contrib = make_float2(0.f, 0.f);
  if (p < np && iw0 < g.W) {
    const float* __restrict__ wd = wbase + r.wd_off;  // Wd[tap][ci]
    float2 w[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) w[t] = __ldg(reinterpret_cast<const float2*>(wd + int64_t(t) * g.Ci + c));
    const int64_t drow = int64_t(g.OW) * g.Co;
    const float* __restrict__ dn = dpre + n * g.OH * drow + r.b + c;
    auto ld = [&](int oh, int ow) {
      return (oh >= 0 && oh < g.OH && ow >= 0 && ow < g.OW)
                 ? __ldg(reinterpret_cast<const float2*>(dn + oh * drow + int64_t(ow) * g.Co))
                 : make_float2(0.f, 0.f);
    };
    float2 win[3][WW];  // [dpre row - (ih - 1)][dpre column - (iw0 - 1)]
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < WW; ++j) win[i][j] = ld(ih0 - 1 + i, iw0 - 1 + j);
    for (int ih = ih0; ih < ih1; ++ih) {
      const int64_t rowi = ((n * g.H + ih) * g.W + iw0) * int64_t(g.Ci) + c;
      float2 nxt[WW], av[OWB];
#pragma unroll
      for (int j = 0; j < WW; ++j) nxt[j] = ih + 1 < ih1 ? ld(ih + 2, iw0 - 1 + j) : make_float2(0.f, 0.f);
#pragma unroll
      for (int o = 0; o < OWB; ++o)
        av[o] = a_prev && iw0 + o < g.W
                    ? __ldg(reinterpret_cast<const float2*>(a_prev + rowi + int64_t(o) * g.Ci))
                    : make_float2(0.f, 0.f);
#pragma unroll
      for (int o = 0; o < OWB; ++o) {
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const float2 wv = w[(2 - i) * 3 + (2 - j)];
            acc.x = fmaf(win[i][o + j].x, wv.x, acc.x);
            acc.y = fmaf(win[i][o + j].y, wv.y, acc.y);
          }
        if (iw0 + o >= g.W) continue;
        const int64_t idx = rowi + int64_t(o) * g.Ci;
        if (g_out) *reinterpret_cast<float2*>(g_out + idx) = acc;
        if (a_prev) {
          contrib.x = fmaf(av[o].x, acc.x, contrib.x);
          contrib.y = fmaf(av[o].y, acc.y, contrib.y);
          if (dpre_out)  // I/nnet.hpp:229-233
            *reinterpret_cast<float2*>(dpre_out + idx) =
                make_float2((relu_prev && !(av[o].x > 0.f)) ? 0.f : acc.x,
                            (relu_prev && !(av[o].y > 0.f)) ? 0.f : acc.y);
        } else if (dpre_out) {
          *reinterpret_cast<float2*>(dpre_out + idx) = acc;
        }
      }
#pragma unroll
      for (int j = 0; j < WW; ++j) {
        win[0][j] = win[1][j];
        win[1][j] = win[2][j];
        win[2][j] = nxt[j];
      }
    }
  }
  if (!partial) return;
  red[threadIdx.y * blockDim.x + threadIdx.x] = contrib;
  __syncthreads();
  if (threadIdx.y == 0 && p < np) {
    float2 sum = make_float2(0.f, 0.f);
    for (int k = 0; k < int(blockDim.y); ++k) {
      sum.x += red[k * blockDim.x + threadIdx.x].x;
      sum.y += red[k * blockDim.x + threadIdx.x].y;
    }
    const int64_t tile = int64_t(sidx) * gridDim.x + blockIdx.x;
    double* dst = partial + (n * int64_t(strips) * gridDim.x + tile) * g.Ci + c;
    dst[0] = double(sum.x);
    dst[1] = double(sum.y);
  }
}

// launch shape of the depthwise register-window kernels: channel-group
// threads x column-block threads, grid (column-block groups, N x strips,
// channel blocks)
struct DwShape {
  dim3 block, grid;
  int strip, strips, owb;
};
DwShape dw3_shape(int64_t N, int OH, int OW, int np, int owb) {
  DwShape d;
  const int ncb = (OW + owb - 1) / owb;  // column blocks
  const int tp = np < 32 ? np : 32;
  int tw = std::max(1, std::min(256 / tp, ncb));
  const int gx = (ncb + tw - 1) / tw;
  tw = (ncb + gx - 1) / gx;  // balance the column blocks over the grid
  // strip rows (shorter strips for small images measured slower: each
  // re-reads two halo rows and refills the window)
  d.strip = kDwStrip;
  d.strips = (OH + d.strip - 1) / d.strip;
  d.block = dim3(tp, tw);
  d.grid = dim3(unsigned(gx), unsigned(N * d.strips), unsigned((np + tp - 1) / tp));
  d.owb = owb;
  return d;
}

bool dw3_dgrad_ok(const ConvGeom& g) {
  static const bool on = [] {  // NB_DW3_DGRAD=0: the shared-memory halo kernel instead
    const char* e = std::getenv("NB_DW3_DGRAD");
    return !e || std::atoi(e) != 0;
  }();
  if (!on || g.nranges != 1) return false;
  const RangeDesc& r = g.r[0];
  return r.b == 0 && r.len == g.Co && g.Ci == g.Co && r.groups == r.len && r.slice_ci == 1 &&
         r.slice_co == 1 && g.KH == 3 && g.KW == 3 && g.S == 1 && g.P == 1 && g.Ci % 2 == 0 &&
         g.H == g.OH && g.W == g.OW;
}
constexpr int kDwDgradOwb = 4;

bool dw3_ok(const ConvGeom& g, const RangeDesc& r) {
  static const bool on = [] {  // NB_DW3=0: the shared-memory halo kernel instead
    const char* e = std::getenv("NB_DW3");
    return !e || std::atoi(e) != 0;
  }();
  return on && r.groups == r.len && r.slice_ci == 1 && r.slice_co == 1 && g.KH == 3 &&
         g.KW == 3 && g.S == 1 && g.P == 1 && r.len % 4 == 0 && r.b % 4 == 0 && g.Ci % 4 == 0 &&
         g.Co % 4 == 0 && (r.wf_off % 2) == 0;
}

void launch_fprop_direct(const ConvGeom& g, int range, const float* x, const float* wbase,
                         float* y, bool relu, cudaStream_t st) {
  const RangeDesc& r = g.r[range];
  if (dw3_ok(g, r)) {
    // NB_DW3_V: channels per thread (2 default; 1 = one channel per thread,
    // measured 2x slower: instruction-bound at 8 blocks / SM)
    static const int V = [] {
      const char* e = std::getenv("NB_DW3_V");
      return e && std::atoi(e) == 1 ? 1 : 2;
    }();
    // NB_DW3_OWB: output columns per thread (1, 2, 4 or 8 with V=2)
    // NB_DW3_OWB fixes it; by default the widest of 8, 4, 2, 1 whose grid
    // still has a wave of 512 threads per SM (small batches / images need the
    // parallelism more than the reuse)
    static const int OWB_ENV = [] {
      const char* e = std::getenv("NB_DW3_OWB");
      const int v = e ? std::atoi(e) : 0;
      return v == 1 || v == 2 || v == 4 || v == 8 ? v : 0;
    }();
    int OWB = OWB_ENV ? OWB_ENV : 8;
    DwShape d = dw3_shape(g.N, g.OH, g.OW, r.len / V, OWB);
    while (!OWB_ENV && OWB > 1 &&
           int64_t(d.grid.x) * d.grid.y * d.grid.z * d.block.x * d.block.y < int64_t(148) * 512) {
      OWB /= 2;
      d = dw3_shape(g.N, g.OH, g.OW, r.len / V, OWB);
    }
    auto go = [&](auto kern) { kern<<<d.grid, d.block, 0, st>>>(g, range, x, wbase, y, relu, d.strip); };
    if (V == 2) {
      if (OWB == 8) go(k_dw3_nhwc<2, 8>);
      else if (OWB == 4) go(k_dw3_nhwc<2, 4>);
      else if (OWB == 2) go(k_dw3_nhwc<2, 2>);
      else go(k_dw3_nhwc<2, 1>);
    } else {
      if (OWB == 4) go(k_dw3_nhwc<1, 4>);
      else if (OWB == 2) go(k_dw3_nhwc<1, 2>);
      else go(k_dw3_nhwc<1, 1>);
    }
    return;
  }
  if (grouped_smem_ok(g, r)) {
    const GTile T = gtile(g.OH, g.OW);
    const int tiles = ((g.OH + T.th - 1) / T.th) * ((g.OW + T.tw - 1) / T.tw);
    const int chunks = (r.len + 31) / 32;
    // worst-case staged channels of a chunk (see grouped_smem_ok)
    const int cic = ((32 + r.slice_co - 1) / r.slice_co + 1) * r.slice_ci;
    const int IH = (T.th - 1) * g.S + g.KH, IW = (T.tw - 1) * g.S + g.KW;
    const size_t smem = size_t(IH) * IW * cic * 4;
    const int K = r.slice_ci * g.KH * g.KW;
    dim3 grid(tiles, g.N, chunks);
    auto go = [&](auto kern, size_t bytes) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
      kern<<<grid, kGThreads, bytes, st>>>(g, range, x, wbase, y, relu);
    };
    if (grouped3_ok(g, r)) {
      const size_t smem3 = grouped3_smem(g, r);
      switch (r.slice_ci) {
        case 1: go(k_fprop_grouped3<1>, smem3); break;
        case 2: go(k_fprop_grouped3<2>, smem3); break;
        case 4: go(k_fprop_grouped3<4>, smem3); break;
        case 8: go(k_fprop_grouped3<8>, smem3); break;
        default: go(k_fprop_grouped3<16>, smem3); break;
      }
    } else if (K <= 9) {
      go(k_fprop_grouped<32, 9>, smem);
    } else if (K <= 18) {
      go(k_fprop_grouped<32, 18>, smem);
    } else if (K <= 36) {
      go(k_fprop_grouped<32, 36>, smem);
    } else {
      go(k_fprop_grouped<32, 64>, smem);
    }
    return;
  }
  if (r.slice_ci == 1 && r.slice_co == 1) {
    const int64_t units = int64_t(g.N) * g.OH * ((g.OW + kDwRun - 1) / kDwRun);
    dim3 grid((r.len + 31) / 32, unsigned((units + 7) / 8));
    k_fprop_dw<<<grid, dim3(32, 8), 0, st>>>(g, range, x, wbase, y, relu);
    return;
  }
  const int64_t npix = int64_t(g.N) * g.OH * g.OW;
  const unsigned gx = unsigned((npix + kFpPix - 1) / kFpPix);
  const unsigned gx2 = unsigned((npix + 2 * kFpPix - 1) / (2 * kFpPix));
  if (r.slice_co <= 16) {
    k_fprop_blocked<16, 2><<<dim3(gx2, r.groups), kFpPix, 0, st>>>(g, range, x, wbase, y, relu);
  } else if (r.slice_co <= 32) {
    k_fprop_blocked<32, 2><<<dim3(gx2, r.groups), kFpPix, 0, st>>>(g, range, x, wbase, y, relu);
  } else {
    const int chunks = (r.slice_co + 63) / 64;
    k_fprop_blocked<64, 1><<<dim3(gx, r.groups * chunks), kFpPix, 0, st>>>(g, range, x, wbase,
                                                                           y, relu);
  }
}

size_t dgrad_grouped3_smem(const ConvGeom& g) {
  const RangeDesc& r = g.r[0];
  const GTile T = gtile(g.H, g.W);
  const int cst = ((32 + r.slice_ci - 1) / r.slice_ci + 1) * r.slice_co;
  const int IH = T.th + 2, IW = T.tw + 5;
  return (size_t(cst) * (((IH * IW + 31) / 32) * 32 + 1) + 9 * size_t(r.slice_co) * 32) * 4;
}

bool dgrad_grouped3_ok(const ConvGeom& g) {
  if (g.nranges != 1) return false;
  const RangeDesc& r = g.r[0];
  return r.groups >= 2 && g.KH == 3 && g.KW == 3 && g.S == 1 &&
         (r.slice_co == 1 || r.slice_co == 2 || r.slice_co == 4 || r.slice_co == 8 ||
          r.slice_co == 16) &&
         dgrad_grouped3_smem(g) <= 200 * 1024;
}

int direct_dgrad_tiles(const ConvGeom& g) {
  if (dw3_dgrad_ok(g)) {
    const DwShape d = dw3_shape(g.N, g.H, g.W, g.Ci / 2, kDwDgradOwb);
    return d.strips * int(d.grid.x);
  }
  if (dgrad_grouped3_ok(g)) {
    const GTile T = gtile(g.H, g.W);
    return ((g.H + T.th - 1) / T.th) * ((g.W + T.tw - 1) / T.tw);
  }
  return dgrad_tiles(g.H, g.W);
}

void launch_dgrad_direct(const ConvGeom& g, const float* dpre, const float* wbase,
                         const float* a_prev, bool relu_prev, float* dpre_out, float* g_out,
                         double* partial, cudaStream_t st) {
  if (dw3_dgrad_ok(g)) {
    const DwShape d = dw3_shape(g.N, g.H, g.W, g.Ci / 2, kDwDgradOwb);
    k_dgrad_dw3<kDwDgradOwb><<<d.grid, d.block, 0, st>>>(g, dpre, wbase, a_prev, relu_prev,
                                                         dpre_out, g_out, partial, d.strip);
    return;
  }
  if (dgrad_grouped3_ok(g)) {
    const size_t smem = dgrad_grouped3_smem(g);
    dim3 grid(direct_dgrad_tiles(g), g.N, (g.Ci + 31) / 32);
    auto go = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      kern<<<grid, kGThreads, smem, st>>>(g, dpre, wbase, a_prev, relu_prev, dpre_out, g_out,
                                          partial);
    };
    switch (g.r[0].slice_co) {
      case 1: go(k_dgrad_grouped3<1>); break;
      case 2: go(k_dgrad_grouped3<2>); break;
      case 4: go(k_dgrad_grouped3<4>); break;
      case 8: go(k_dgrad_grouped3<8>); break;
      default: go(k_dgrad_grouped3<16>); break;
    }
    return;
  }
  dim3 grid((g.Ci + 31) / 32, dgrad_tiles(g.H, g.W), g.N);
  k_dgrad_direct<<<grid, dim3(32, 8), 0, st>>>(g, dpre, wbase, a_prev, relu_prev, dpre_out,
                                               g_out, partial);
}

void launch_splitk_epilogue(const SplitEpi& e, cudaStream_t st) {
  // programmatic dependent launch: its launch overlaps the conv's tail (the
  // kernel waits on griddepcontrol before reading the partials)
  static const bool pdl = [] {
    const char* v = std::getenv("NB_TC_PDL");
    return !v || std::atoi(v) != 0;
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(32, 8);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  if (e.C % 4 == 0 && e.ld % 4 == 0 && e.c0 % 4 == 0) {
    cfg.gridDim = dim3((e.C + 127) / 128, e.N, e.hw_chunks);
    cudaLaunchKernelEx(&cfg, k_splitk_epilogue4, e);
    return;
  }
  cfg.gridDim = dim3((e.C + 31) / 32, e.N, e.hw_chunks);
  cudaLaunchKernelEx(&cfg, k_splitk_epilogue, e);
}

__global__ void k_im2col32(const float* __restrict__ x, int64_t N, int H, int W, int Ci, int KH,
                           int KW, int S, int P, int OH, int OW, float* __restrict__ out) {
  const int64_t total = N * OH * OW * 32;
  const int K = Ci * KH * KW;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int k = int(e % 32);
    const int64_t pix = e / 32;
    const int ow = int(pix % OW), oh = int((pix / OW) % OH);
    const int64_t n = pix / (int64_t(OW) * OH);
    float v = 0.f;
    if (k < K) {
      const int tap = k / Ci, c = k - tap * Ci;
      const int ih = oh * S - P + tap / KW, iw = ow * S - P + tap % KW;
      if (ih >= 0 && ih < H && iw >= 0 && iw < W) v = x[((n * H + ih) * W + iw) * Ci + c];
    }
    out[e] = v;
  }
}

void launch_amax(const float* x, int64_t N, int64_t per_img, uint32_t* amax, cudaStream_t st) {
  if (N <= 0 || per_img <= 0) return;
  int64_t bx = (per_img / 4 + 255) / 256;
  const int64_t cap = (148 * 8 + N - 1) / N;
  bx = bx < 1 ? 1 : (bx > cap ? cap : bx);
  k_amax<<<dim3(unsigned(bx), unsigned(N)), 256, 0, st>>>(x, per_img, amax);
}

void launch_im2col32(const float* x, int64_t N, int H, int W, int Ci, int KH, int KW, int S,
                     int P, int OH, int OW, float* out, cudaStream_t st) {
  k_im2col32<<<grid_for(N * OH * OW * 32, 256), 256, 0, st>>>(x, N, H, W, Ci, KH, KW, S, P, OH,
                                                             OW, out);
}

int splitk_hw_chunks(int64_t n, int HW, int C) {
  // about two blocks per SM, at least 64 pixels per chunk
  const int64_t base = int64_t((C + 127) / 128) * n;
  int64_t ch = (2 * 148 + base - 1) / base;
  const int64_t cap = HW / 64 > 1 ? HW / 64 : 1;
  return int(ch < 1 ? 1 : (ch > cap ? cap : ch));
}

void launch_head(const HeadArgs& a, cudaStream_t st) {
  constexpr int kThreads = 512;
  const size_t smem = sizeof(double) * (2 * size_t(a.C) + 2 * size_t(a.K) + kThreads);
  k_head<<<a.N, kThreads, smem, st>>>(a);
}

void launch_fisher_reduce(const FisherLayer* layers_dev, int L, int max_c, int N,
                          double* per_channel, double* s_out, int64_t s_ld, cudaStream_t st) {
  dim3 grid((max_c + 31) / 32, L);
  k_fisher_reduce<<<grid, dim3(32, 16), 0, st>>>(layers_dev, N, per_channel, s_out, s_ld);
}

}  // namespace nb

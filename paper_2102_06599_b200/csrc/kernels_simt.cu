// fp32 FFMA kernels of the nb200 hot path: layout conversion, weight packing,
// direct (grouped / depthwise / generic) conv fprop and the dgrad with the
// fused Fisher epilogue, the fp64 head, and the deterministic Fisher
// reduction.  Tensor-core-shaped ranges use kernels_tc.cu instead.
//
// Activations are NHWC fp32 in HBM (channels contiguous: coalesced across
// output channels for fprop and across input channels for dgrad).
#include <cfloat>
#include <cmath>

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
    if (d.tcf_hi) {
      const int64_t i = (int64_t(co_local) * taps + tap) * r.slice_ci + j;
      d.tcf_hi[i] = hi;
      d.tcf_lo[i] = lo;
    }
    if (d.tcd_hi) {
      const int64_t i = (int64_t(ci) * taps + tap) * r.slice_co + t;
      d.tcd_hi[i] = hi;
      d.tcd_lo[i] = lo;
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

template <int CO_T>
__global__ void __launch_bounds__(kFpPix) k_fprop_blocked(ConvGeom g, int ri,
                                                          const float* __restrict__ x,
                                                          const float* __restrict__ wbase,
                                                          float* __restrict__ y, bool relu) {
  __shared__ float ws[kFpKChunk][CO_T];
  const RangeDesc r = g.r[ri];
  const float* __restrict__ wf = wbase + r.wf_off;
  const int co_chunks = (r.slice_co + CO_T - 1) / CO_T;
  const int grp = blockIdx.y / co_chunks;
  const int co0 = (blockIdx.y % co_chunks) * CO_T;  // within the group
  const int nco = min(CO_T, r.slice_co - co0);
  const int64_t npix = int64_t(g.N) * g.OH * g.OW;
  const int64_t pix = int64_t(blockIdx.x) * kFpPix + threadIdx.x;
  const bool valid = pix < npix;
  int ow = 0, oh = 0;
  int64_t n = 0;
  if (valid) {
    ow = int(pix % g.OW);
    oh = int((pix / g.OW) % g.OH);
    n = pix / (int64_t(g.OW) * g.OH);
  }
  float acc[CO_T];
#pragma unroll
  for (int t = 0; t < CO_T; ++t) acc[t] = 0.f;
  const int K = r.slice_ci * g.KH * g.KW;
  for (int k0 = 0; k0 < K; k0 += kFpKChunk) {
    const int kn = min(kFpKChunk, K - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < kn * CO_T; e += kFpPix) {
      const int kk = e / CO_T, t = e % CO_T;
      ws[kk][t] = t < nco ? wf[int64_t(k0 + kk) * r.len + grp * r.slice_co + co0 + t] : 0.f;
    }
    __syncthreads();
    if (valid) {
      for (int kk = 0; kk < kn; ++kk) {
        const int k = k0 + kk;
        const int tap = k / r.slice_ci, j = k - tap * r.slice_ci;
        const int kh = tap / g.KW, kw = tap - kh * g.KW;
        const int ih = g.S * oh - g.P + kh, iw = g.S * ow - g.P + kw;
        if (ih < 0 || ih >= g.H || iw < 0 || iw >= g.W) continue;
        const float xv =
            __ldg(x + ((n * g.H + ih) * g.W + iw) * g.Ci + int64_t(grp) * r.slice_ci + j);
#pragma unroll
        for (int t = 0; t < CO_T; ++t) acc[t] = fmaf(xv, ws[kk][t], acc[t]);
      }
    }
  }
  if (!valid) return;
  float* yo = y + pix * g.Co + r.b + grp * r.slice_co + co0;
#pragma unroll
  for (int t = 0; t < CO_T; ++t)
    if (t < nco) yo[t] = (relu && !(acc[t] > 0.f)) ? 0.f : acc[t];  // I/nnet.hpp:138-139
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
__global__ void k_head(HeadArgs a) {
  extern __shared__ double sm[];
  double* pooled = sm;            // C
  double* dpool = sm + a.C;       // C
  double* z = sm + 2 * a.C;       // K
  double* dz = z + a.K;           // K
  const int n = blockIdx.x;
  const float* act = a.act + int64_t(n) * a.HW * a.C;
  for (int i = threadIdx.x; i < a.C; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < a.HW; ++j) s += double(act[int64_t(j) * a.C + i]);
    pooled[i] = s / double(a.HW);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < a.K; k += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < a.C; ++i) s += (a.head_src[int64_t(k) * a.C + i] * a.head_scale) * pooled[i];
    z[k] = s;
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
    for (int k = 0; k < a.K; ++k) dz[k] /= double(a.N);
  }
  __syncthreads();
  if (!a.backward) return;
  for (int i = threadIdx.x; i < a.C; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < a.K; ++k) s += (a.head_src[int64_t(k) * a.C + i] * a.head_scale) * dz[k];
    dpool[i] = s;
  }
  __syncthreads();
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
                                                       int N, double* __restrict__ per_channel) {
  __shared__ double red[16][33];
  const FisherLayer L = layers[blockIdx.y];
  const int c = blockIdx.x * 32 + threadIdx.x;
  if (blockIdx.x * 32 >= L.C) return;
  double acc = 0.0;
  if (c < L.C) {
    for (int n = threadIdx.y; n < N; n += 16) {
      const double* p = L.partial + int64_t(n) * L.tiles * L.C + c;
      double s = 0.0;
      for (int t = 0; t < L.tiles; ++t) s -= p[int64_t(t) * L.C];
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
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int64_t n = blockIdx.y;
  float contrib = 0.f;
  if (c < e.C) {
    for (int p = threadIdx.y; p < e.HW; p += 8) {
      const int64_t idx = (n * e.HW + p) * e.ld + e.c0 + c;
      float v = 0.f;
      for (int k = 0; k < e.ksplit; ++k) v += e.ws[k * e.ws_stride + idx];
      if (e.mode == 0) {
        e.out[idx] = (e.relu && !(v > 0.f)) ? 0.f : v;  // I/nnet.hpp:138-139
      } else {
        if (e.g_out) e.g_out[idx] = v;
        if (e.a_prev) {
          const float a = e.a_prev[idx];
          contrib = fmaf(a, v, contrib);
          if (e.dpre_out) e.dpre_out[idx] = (e.relu_prev && !(a > 0.f)) ? 0.f : v;
        } else if (e.dpre_out) {
          e.dpre_out[idx] = v;
        }
      }
    }
  }
  if (e.mode == 0 || !e.partial) return;
  red[threadIdx.y][threadIdx.x] = contrib;
  __syncthreads();
  if (threadIdx.y == 0 && c < e.C) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][threadIdx.x];
    e.partial[n * e.ld + e.c0 + c] = double(s);
  }
}

int grid_for(int64_t total, int block) {
  int64_t g = (total + block - 1) / block;
  const int64_t cap = 148 * 32;
  return int(g < 1 ? 1 : (g > cap ? cap : g));
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

void launch_fprop_direct(const ConvGeom& g, int range, const float* x, const float* wbase,
                         float* y, bool relu, cudaStream_t st) {
  const RangeDesc& r = g.r[range];
  if (r.slice_ci == 1 && r.slice_co == 1) {
    const int64_t units = int64_t(g.N) * g.OH * ((g.OW + kDwRun - 1) / kDwRun);
    dim3 grid((r.len + 31) / 32, unsigned((units + 7) / 8));
    k_fprop_dw<<<grid, dim3(32, 8), 0, st>>>(g, range, x, wbase, y, relu);
    return;
  }
  const int64_t npix = int64_t(g.N) * g.OH * g.OW;
  const unsigned gx = unsigned((npix + kFpPix - 1) / kFpPix);
  if (r.slice_co <= 16) {
    k_fprop_blocked<16><<<dim3(gx, r.groups), kFpPix, 0, st>>>(g, range, x, wbase, y, relu);
  } else if (r.slice_co <= 32) {
    k_fprop_blocked<32><<<dim3(gx, r.groups), kFpPix, 0, st>>>(g, range, x, wbase, y, relu);
  } else {
    const int chunks = (r.slice_co + 63) / 64;
    k_fprop_blocked<64><<<dim3(gx, r.groups * chunks), kFpPix, 0, st>>>(g, range, x, wbase, y,
                                                                        relu);
  }
}

void launch_dgrad_direct(const ConvGeom& g, const float* dpre, const float* wbase,
                         const float* a_prev, bool relu_prev, float* dpre_out, float* g_out,
                         double* partial, cudaStream_t st) {
  dim3 grid((g.Ci + 31) / 32, dgrad_tiles(g.H, g.W), g.N);
  k_dgrad_direct<<<grid, dim3(32, 8), 0, st>>>(g, dpre, wbase, a_prev, relu_prev, dpre_out,
                                               g_out, partial);
}

void launch_splitk_epilogue(const SplitEpi& e, cudaStream_t st) {
  dim3 grid((e.C + 31) / 32, e.N);
  k_splitk_epilogue<<<grid, dim3(32, 8), 0, st>>>(e);
}

void launch_head(const HeadArgs& a, cudaStream_t st) {
  const size_t smem = sizeof(double) * (2 * size_t(a.C) + 2 * size_t(a.K));
  k_head<<<a.N, 256, smem, st>>>(a);
}

void launch_fisher_reduce(const FisherLayer* layers_dev, int L, int max_c, int N,
                          double* per_channel, cudaStream_t st) {
  dim3 grid((max_c + 31) / 32, L);
  k_fisher_reduce<<<grid, dim3(32, 16), 0, st>>>(layers_dev, N, per_channel);
}

}  // namespace nb

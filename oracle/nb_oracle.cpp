// TEST INFRASTRUCTURE ONLY -- the CPU oracle of the nb200 hot path.
//
// A restatement, in plain loops, of the reference's fp64 conv-net engine and
// Fisher Potential (nestopt, /root/reference/proj/include/nestopt = I/).  It
// is the checker the GPU parity tests compare against and the "port" CPU
// baseline; the product (paper_2102_06599_b200/) never links or calls it.
//
// Pinning: tests/test_oracle.py checks this restatement against the
// reference itself (oracle/_ref/libnestopt_ref.so, built from the reference
// headers by oracle/Makefile) and against the committed golden fixtures in
// tests/golden/ that oracle/gen_golden.py generated from the reference.
//
// Weights and batches use std::mt19937_64 + std::normal_distribution<double>
// / std::uniform_int_distribution<int> from the same libstdc++ the reference
// is compiled with, so they are bit-identical to the reference's draws.
// Conv sums run in a different loop order than the reference (fp64, so the
// results agree to ~1e-15 relative); head, softmax and the Fisher reduction
// follow the reference's summation order exactly.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "nb200.h"

namespace {

thread_local std::string g_err;

struct Spec {  // ConvSpec derived quantities, I/ir.hpp:45-57
  const nb_conv_spec* s;
  int64_t co_eff() const { return s->co / s->bottleneck_out; }
  int64_t raw_oh() const { return (s->h + 2 * s->pad - s->kh) / s->stride + 1; }
  int64_t raw_ow() const { return (s->w + 2 * s->pad - s->kw) / s->stride + 1; }
  int64_t oh() const { return raw_oh() / s->spatial_div_h; }
  int64_t ow() const { return raw_ow() / s->spatial_div_w; }
  std::vector<nb_channel_split> ranges() const {  // I/ir.hpp:54-57
    if (s->num_splits > 0) return {s->splits, s->splits + s->num_splits};
    return {{0, co_eff(), s->groups}};
  }
};

void validate(const nb_conv_spec* sp) {  // ConvSpec::validate, I/ir.hpp:59-86
  Spec S{sp};
  const nb_conv_spec& s = *sp;
  auto req = [](bool ok, const char* m) {
    if (!ok) throw std::invalid_argument(m);
  };
  req(s.ci >= 1 && s.co >= 1 && s.h >= 1 && s.w >= 1, "dims must be positive");
  req(s.kh >= 1 && s.kw >= 1 && s.stride >= 1 && s.pad >= 0, "bad kernel/stride/pad");
  req(s.groups >= 1 && s.co % s.groups == 0 && s.ci % s.groups == 0,
      "Co and Ci must be divisible by groups");
  req(s.bottleneck_out >= 1 && s.co % s.bottleneck_out == 0,
      "Co must be divisible by bottleneck factor");
  req(S.raw_oh() >= 1 && S.raw_ow() >= 1, "kernel larger than padded input");
  req(s.spatial_div_h >= 1 && S.raw_oh() % s.spatial_div_h == 0 &&
          s.spatial_div_w >= 1 && S.raw_ow() % s.spatial_div_w == 0,
      "spatial size must be divisible by spatial bottleneck factor");
  int64_t pos = 0;
  for (int64_t i = 0; i < s.num_splits; ++i) {
    const nb_channel_split& r = s.splits[i];
    req(r.begin == pos && r.end > r.begin && r.end <= S.co_eff(),
        "channel splits must be contiguous and disjoint");
    req(r.groups >= 1 && (r.end - r.begin) % r.groups == 0 && s.ci % r.groups == 0,
        "split range and Ci must be divisible by its group factor");
    pos = r.end;
  }
  if (s.num_splits > 0)
    req(pos == S.co_eff(), "channel splits must cover [0, Co)");
  else
    req(S.co_eff() % s.groups == 0, "effective Co must be divisible by groups");
}

// Network::init_weights, I/nnet.hpp:58-79.
void init_weights(const nb_network* net, std::vector<std::vector<double>>& W,
                  std::vector<double>& head) {
  const int64_t L = net->num_layers;
  W.assign(L, {});
  for (int64_t l = 0; l < L; ++l) {
    const nb_conv_spec& s = net->layers[l].spec;
    std::mt19937_64 rng(net->seed * 0x9e3779b97f4a7c15ull + l + 1);
    std::normal_distribution<double> dist(
        0.0, 1.0 / std::sqrt(double(s.ci * s.kh * s.kw)));
    W[l].resize(Spec{&s}.co_eff() * s.ci * s.kh * s.kw);
    for (double& v : W[l]) v = dist(rng);
  }
  const int64_t C = Spec{&net->layers[L - 1].spec}.co_eff();
  std::mt19937_64 rng(net->seed * 0x9e3779b97f4a7c15ull + L + 1);
  std::normal_distribution<double> dist(0.0, 1.0 / std::sqrt(double(C)));
  head.resize(net->num_classes * C);
  for (double& v : head) v = dist(rng);
}

// make_batch, I/nnet.hpp:87-101.
void make_batch(const nb_network* net, int64_t n, uint64_t seed, double* x,
                int32_t* labels) {
  const nb_conv_spec& s0 = net->layers[0].spec;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(0.0, 1.0);
  std::uniform_int_distribution<int> lab(0, int(net->num_classes) - 1);
  const int64_t per = s0.ci * s0.h * s0.w;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < per; ++j) x[i * per + j] = dist(rng);
    labels[i] = lab(rng);
  }
}

// Output columns whose tap iw = stride*ow - pad + kw lands inside [0, W):
// ow >= first_tap(pad - kw) and ow <= last_tap(W - 1 + pad - kw).  Skipping
// the others up front is the same MAC set (padded taps skipped,
// I/nnet.hpp:121-123) and the same per-output summation order.
inline int64_t first_tap(int64_t num, int64_t stride) {
  return num <= 0 ? 0 : (num + stride - 1) / stride;
}
inline int64_t last_tap(int64_t num, int64_t stride) {
  return num < 0 ? -1 : num / stride;
}

// Eq. 1-3 over the canonical MAC set of for_each_conv_mac (I/nnet.hpp:108-128)
// / reference_conv (I/interp.hpp:151-186): for each range/group, out[co] +=
// W[co, ci, kh, kw] * in[ci, s*oh-p+kh, s*ow-p+kw], padded taps skipped.
template <typename T>
void conv_image(const nb_conv_spec* sp, const T* in, const T* w, T* out) {
  Spec S{sp};
  const nb_conv_spec& s = *sp;
  const int64_t OH = S.oh(), OW = S.ow(), H = s.h, Wd = s.w;
  std::fill(out, out + S.co_eff() * OH * OW, T{});
  for (const auto& r : S.ranges()) {
    const int64_t slice_co = (r.end - r.begin) / r.groups, slice_ci = s.ci / r.groups;
    for (int64_t co = r.begin; co < r.end; ++co) {
      const int64_t g = (co - r.begin) / slice_co;
      T* o = out + co * OH * OW;
      for (int64_t ci = g * slice_ci; ci < (g + 1) * slice_ci; ++ci)
        for (int64_t kh = 0; kh < s.kh; ++kh)
          for (int64_t kw = 0; kw < s.kw; ++kw) {
            const T wv = w[((co * s.ci + ci) * s.kh + kh) * s.kw + kw];
            const T* ip = in + ci * H * Wd;
            const int64_t ow0 = first_tap(s.pad - kw, s.stride),
                          ow1 = std::min(OW, last_tap(Wd - 1 + s.pad - kw, s.stride) + 1);
            for (int64_t oh = 0; oh < OH; ++oh) {
              const int64_t ih = s.stride * oh - s.pad + kh;
              if (ih < 0 || ih >= H) continue;
              T* orow = o + oh * OW;
              const T* irow = ip + ih * Wd - s.pad + kw;
              for (int64_t ow = ow0; ow < ow1; ++ow) orow[ow] += wv * irow[s.stride * ow];
            }
          }
    }
  }
}

// The dgrad MAC loop of activation_gradients (I/nnet.hpp:235-243):
// dx[ci, ih, iw] += W[co, ci, kh, kw] * dy[co, oh, ow] over the same MAC set.
void dgrad_image(const nb_conv_spec* sp, const double* dy, const double* w, double* dx) {
  Spec S{sp};
  const nb_conv_spec& s = *sp;
  const int64_t OH = S.oh(), OW = S.ow(), H = s.h, Wd = s.w;
  std::fill(dx, dx + s.ci * H * Wd, 0.0);
  for (const auto& r : S.ranges()) {
    const int64_t slice_co = (r.end - r.begin) / r.groups, slice_ci = s.ci / r.groups;
    for (int64_t co = r.begin; co < r.end; ++co) {
      const int64_t g = (co - r.begin) / slice_co;
      const double* d = dy + co * OH * OW;
      for (int64_t ci = g * slice_ci; ci < (g + 1) * slice_ci; ++ci)
        for (int64_t kh = 0; kh < s.kh; ++kh)
          for (int64_t kw = 0; kw < s.kw; ++kw) {
            const double wv = w[((co * s.ci + ci) * s.kh + kh) * s.kw + kw];
            double* xp = dx + ci * H * Wd;
            const int64_t ow0 = first_tap(s.pad - kw, s.stride),
                          ow1 = std::min(OW, last_tap(Wd - 1 + s.pad - kw, s.stride) + 1);
            for (int64_t oh = 0; oh < OH; ++oh) {
              const int64_t ih = s.stride * oh - s.pad + kh;
              if (ih < 0 || ih >= H) continue;
              double* xrow = xp + ih * Wd - s.pad + kw;
              const double* drow = d + oh * OW;
              for (int64_t ow = ow0; ow < ow1; ++ow) xrow[s.stride * ow] += wv * drow[ow];
            }
          }
    }
  }
}

struct Net {
  const nb_network* net;
  std::vector<std::vector<double>> W;
  std::vector<double> head;
  std::vector<int64_t> C, OH, OW;  // per layer output dims
};

void load(Net& N, const nb_network* net, const nb_weights* w) {
  if (net->num_layers < 1) throw std::invalid_argument("network has no layers");
  N.net = net;
  for (int64_t l = 0; l < net->num_layers; ++l) {
    validate(&net->layers[l].spec);
    Spec S{&net->layers[l].spec};
    if (l > 0) {
      const nb_conv_spec& c = net->layers[l].spec;
      if (c.ci != N.C[l - 1] || c.h != N.OH[l - 1] || c.w != N.OW[l - 1])
        throw std::invalid_argument("layer input shape does not match");
    }
    N.C.push_back(S.co_eff());
    N.OH.push_back(S.oh());
    N.OW.push_back(S.ow());
  }
  init_weights(net, N.W, N.head);
  if (w && w->layer)
    for (int64_t l = 0; l < net->num_layers; ++l)
      std::memcpy(N.W[l].data(), w->layer[l], N.W[l].size() * 8);
  if (w && w->head) std::memcpy(N.head.data(), w->head, N.head.size() * 8);
}

// forward (I/nnet.hpp:180-197) + activation_gradients (:201-247) +
// fisher_potential (:321-352) for a whole batch.
void fisher(const Net& N, int64_t n, const double* x, const int32_t* labels,
            bool want_grads, double* per_channel, double* per_layer, double* total,
            double* loss, double* probs, double* acts_out, double* grads_out) {
  const nb_network* net = N.net;
  const int64_t L = net->num_layers, K = net->num_classes;
  const nb_conv_spec& s0 = net->layers[0].spec;
  const int64_t in_sz = s0.ci * s0.h * s0.w;
  std::vector<int64_t> sz(L);
  for (int64_t l = 0; l < L; ++l) sz[l] = N.C[l] * N.OH[l] * N.OW[l];
  // acts[n][l], grads[n][l]
  std::vector<std::vector<std::vector<double>>> A(n), G(n);
  std::vector<std::vector<double>> P(n);
  std::vector<double> ex_loss(n);
#pragma omp parallel for schedule(dynamic)
  for (int64_t e = 0; e < n; ++e) {
    A[e].resize(L);
    const double* cur = x + e * in_sz;
    for (int64_t l = 0; l < L; ++l) {
      A[e][l].resize(sz[l]);
      conv_image(&net->layers[l].spec, cur, N.W[l].data(), A[e][l].data());
      if (net->layers[l].relu)
        for (double& v : A[e][l]) v = v > 0.0 ? v : 0.0;
      cur = A[e][l].data();
    }
    // head_logits + softmax, I/nnet.hpp:152-176
    const int64_t c = N.C[L - 1], hw = N.OH[L - 1] * N.OW[L - 1];
    std::vector<double> pooled(c, 0.0), z(K, 0.0), p(K);
    for (int64_t i = 0; i < c; ++i) {
      for (int64_t j = 0; j < hw; ++j) pooled[i] += A[e][L - 1][i * hw + j];
      pooled[i] /= double(hw);
    }
    for (int64_t k = 0; k < K; ++k)
      for (int64_t i = 0; i < c; ++i) z[k] += N.head[k * c + i] * pooled[i];
    double m = z[0];
    for (double v : z) m = std::max(m, v);
    double sum = 0.0;
    for (int64_t k = 0; k < K; ++k) sum += (p[k] = std::exp(z[k] - m));
    for (double& v : p) v /= sum;
    ex_loss[e] = -std::log(std::max(p[labels[e]], 1e-300));
    P[e] = p;
    if (!want_grads) continue;
    // activation_gradients, I/nnet.hpp:209-243
    std::vector<double> dz(p);
    dz[labels[e]] -= 1.0;
    for (double& v : dz) v /= double(n);
    std::vector<double> dpool(c, 0.0);
    for (int64_t k = 0; k < K; ++k)
      for (int64_t i = 0; i < c; ++i) dpool[i] += N.head[k * c + i] * dz[k];
    G[e].resize(L);
    G[e][L - 1].resize(sz[L - 1]);
    for (int64_t i = 0; i < c; ++i)
      for (int64_t j = 0; j < hw; ++j) G[e][L - 1][i * hw + j] = dpool[i] / double(hw);
    for (int64_t l = L - 1; l >= 1; --l) {
      std::vector<double> dpre = G[e][l];
      if (net->layers[l].relu)
        for (int64_t i = 0; i < sz[l]; ++i)
          if (A[e][l][i] <= 0.0) dpre[i] = 0.0;
      G[e][l - 1].resize(sz[l - 1]);
      dgrad_image(&net->layers[l].spec, dpre.data(), N.W[l].data(), G[e][l - 1].data());
    }
  }
  double lsum = 0.0;
  for (int64_t e = 0; e < n; ++e) {
    lsum += ex_loss[e];
    if (probs) std::memcpy(probs + e * K, P[e].data(), K * 8);
  }
  if (loss) *loss = lsum / double(n);
  if (!want_grads) return;
  // fisher_potential reduction, I/nnet.hpp:330-350 (same summation order).
  double tot = 0.0;
  int64_t off = 0;
  for (int64_t l = 0; l < L; ++l) {
    const int64_t hw = N.OH[l] * N.OW[l];
    double layer = 0.0;
    for (int64_t ch = 0; ch < N.C[l]; ++ch) {
      double acc = 0.0;
      for (int64_t e = 0; e < n; ++e) {
        double s = 0.0;
        for (int64_t j = 0; j < hw; ++j)
          s -= A[e][l][ch * hw + j] * G[e][l][ch * hw + j];
        acc += s * s;
      }
      const double delta = acc / (2.0 * double(n));
      if (per_channel) per_channel[off + ch] = delta;
      layer += delta;
    }
    off += N.C[l];
    if (per_layer) per_layer[l] = layer;
    tot += layer;
  }
  if (total) *total = tot;
  if (acts_out || grads_out) {
    int64_t o = 0;
    for (int64_t l = 0; l < L; ++l)
      for (int64_t e = 0; e < n; ++e) {
        if (acts_out) std::memcpy(acts_out + o, A[e][l].data(), sz[l] * 8);
        if (grads_out) std::memcpy(grads_out + o, G[e][l].data(), sz[l] * 8);
        o += sz[l];
      }
  }
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

int orc_validate_spec(const nb_conv_spec* s) {
  return guard([&] { validate(s); });
}

int orc_init_weights(const nb_network* net, double* weights, double* head) {
  return guard([&] {
    std::vector<std::vector<double>> W;
    std::vector<double> h;
    init_weights(net, W, h);
    size_t off = 0;
    for (auto& w : W) {
      if (weights) std::memcpy(weights + off, w.data(), w.size() * 8);
      off += w.size();
    }
    if (head) std::memcpy(head, h.data(), h.size() * 8);
  });
}

int orc_make_batch(const nb_network* net, int64_t n, uint64_t seed, double* x,
                   int32_t* labels) {
  return guard([&] { make_batch(net, n, seed, x, labels); });
}

// reference_conv<T> on one image (is_int: int64, else fp64).
int orc_conv(const nb_conv_spec* s, int is_int, const void* in, const void* w, void* out) {
  return guard([&] {
    validate(s);
    if (is_int)
      conv_image<long long>(s, static_cast<const long long*>(in),
                            static_cast<const long long*>(w), static_cast<long long*>(out));
    else
      conv_image<double>(s, static_cast<const double*>(in), static_cast<const double*>(w),
                         static_cast<double*>(out));
  });
}

int orc_conv_dgrad(const nb_conv_spec* s, const double* dy, const double* w, double* dx) {
  return guard([&] {
    validate(s);
    dgrad_image(s, dy, w, dx);
  });
}

// fisher_potential with optional forward/gradient outputs (see fisher()).
int orc_fisher(const nb_network* net, const nb_weights* w, const nb_batch* b,
               nb_fisher_out* out, double* acts, double* grads) {
  return guard([&] {
    Net N;
    load(N, net, w);
    const nb_conv_spec& s0 = net->layers[0].spec;
    std::vector<double> x;
    std::vector<int32_t> lab;
    const double* xp = b->inputs;
    const int32_t* lp = b->labels;
    if (!xp) {
      x.resize(b->n * s0.ci * s0.h * s0.w);
      lab.resize(b->n);
      make_batch(net, b->n, b->seed, x.data(), lab.data());
      xp = x.data();
      lp = lab.data();
    }
    out->seed = b->seed;
    fisher(N, b->n, xp, lp, true, out->per_channel, out->per_layer, &out->total,
           &out->loss, out->probs, acts, grads);
  });
}

// forward only: probs and mean loss.
int orc_forward(const nb_network* net, const nb_weights* w, const nb_batch* b,
                double* probs, double* loss) {
  return guard([&] {
    Net N;
    load(N, net, w);
    const nb_conv_spec& s0 = net->layers[0].spec;
    std::vector<double> x;
    std::vector<int32_t> lab;
    const double* xp = b->inputs;
    const int32_t* lp = b->labels;
    if (!xp) {
      x.resize(b->n * s0.ci * s0.h * s0.w);
      lab.resize(b->n);
      make_batch(net, b->n, b->seed, x.data(), lab.data());
      xp = x.data();
      lp = lab.data();
    }
    fisher(N, b->n, xp, lp, false, nullptr, nullptr, nullptr, loss, probs, nullptr,
           nullptr);
  });
}

}  // extern "C"

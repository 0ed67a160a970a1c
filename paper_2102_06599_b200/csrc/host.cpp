// Host-side descriptors of the nb200 hot path: ConvSpec/Network validation,
// MAC counts, shape repair, the z-stream weight cache, make_batch and the
// LPT scheduler helper.  No device code here.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <random>
#include <thread>

#include "common.hpp"

namespace nb {

namespace {
thread_local std::string g_last_error;

uint64_t mix(uint64_t h, uint64_t v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  return h;
}
}  // namespace

void set_last_error(const std::string& m) { g_last_error = m; }

Spec Spec::from(const nb_conv_spec& s) {
  Spec o;
  o.ci = s.ci;
  o.co = s.co;
  o.h = s.h;
  o.w = s.w;
  o.kh = s.kh;
  o.kw = s.kw;
  o.stride = s.stride;
  o.pad = s.pad;
  o.groups = s.groups;
  o.bottleneck_out = s.bottleneck_out;
  o.sdh = s.spatial_div_h;
  o.sdw = s.spatial_div_w;
  if (s.num_splits < 0) fail(NB_ERR_INVALID_SPEC, "negative split count");
  if (s.num_splits > 0 && !s.splits) fail(NB_ERR_INVALID_SPEC, "null split array");
  o.splits.assign(s.splits, s.splits + s.num_splits);
  return o;
}

// ConvSpec::validate, I/ir.hpp:59-86 (same checks, same order, same messages).
void Spec::validate() const {
  auto req = [](bool ok, const char* msg) {
    if (!ok) fail(NB_ERR_INVALID_SPEC, msg);
  };
  req(ci >= 1 && co >= 1 && h >= 1 && w >= 1, "dims must be positive");
  req(kh >= 1 && kw >= 1 && stride >= 1 && pad >= 0, "bad kernel/stride/pad");
  req(groups >= 1 && co % groups == 0 && ci % groups == 0,
      "Co and Ci must be divisible by groups");
  req(bottleneck_out >= 1 && co % bottleneck_out == 0,
      "Co must be divisible by bottleneck factor");
  req(raw_oh() >= 1 && raw_ow() >= 1, "kernel larger than padded input");
  req(sdh >= 1 && raw_oh() % sdh == 0 && sdw >= 1 && raw_ow() % sdw == 0,
      "spatial size must be divisible by spatial bottleneck factor");
  int64_t pos = 0;
  for (const auto& s : splits) {
    req(s.begin == pos && s.end > s.begin && s.end <= co_eff(),
        "channel splits must be contiguous and disjoint");
    req(s.groups >= 1 && (s.end - s.begin) % s.groups == 0 && ci % s.groups == 0,
        "split range and Ci must be divisible by its group factor");
    pos = s.end;
  }
  if (!splits.empty())
    req(pos == co_eff(), "channel splits must cover [0, Co)");
  else
    req(co_eff() % groups == 0, "effective Co must be divisible by groups");
}

// count_macs(conv_nest(spec)) (I/interp.hpp:190-202 over I/ir.hpp:427-521):
// per range the S2 instance count len * oh * ow * (Ci/G) * Kh * Kw, padded
// taps included.
int64_t Spec::macs() const {
  int64_t t = 0;
  for (const auto& r : ranges())
    t += (r.end - r.begin) * oh() * ow() * (ci / r.groups) * kh * kw;
  return t;
}

bool Spec::operator==(const Spec& o) const {
  if (ci != o.ci || co != o.co || h != o.h || w != o.w || kh != o.kh || kw != o.kw ||
      stride != o.stride || pad != o.pad || bottleneck_out != o.bottleneck_out ||
      sdh != o.sdh || sdw != o.sdw)
    return false;
  // Numerically a spec is its range list: groups only matters without splits.
  auto a = ranges(), b = o.ranges();
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (a[i].begin != b[i].begin || a[i].end != b[i].end || a[i].groups != b[i].groups)
      return false;
  return true;
}

uint64_t Spec::hash() const {
  uint64_t h0 = 0;
  for (int64_t v : {ci, co, h, w, kh, kw, stride, pad, bottleneck_out, sdh, sdw})
    h0 = mix(h0, uint64_t(v));
  for (const auto& r : ranges()) {
    h0 = mix(h0, uint64_t(r.begin));
    h0 = mix(h0, uint64_t(r.end));
    h0 = mix(h0, uint64_t(r.groups));
  }
  return h0;
}

// Network::validate, I/nnet.hpp:40-55.
NetDesc NetDesc::from(const nb_network* net) {
  if (!net) fail(NB_ERR_CONFIG, "null network");
  NetDesc d;
  if (net->num_layers < 1 || !net->layers) fail(NB_ERR_CONFIG, "network has no layers");
  if (net->num_classes < 2) fail(NB_ERR_CONFIG, "need at least two classes");
  d.num_classes = net->num_classes;
  d.seed = net->seed;
  for (int64_t l = 0; l < net->num_layers; ++l) {
    Spec s = Spec::from(net->layers[l].spec);
    s.validate();
    if (l > 0) {
      const Spec& p = d.specs.back();
      if (s.ci != p.co_eff() || s.h != p.oh() || s.w != p.ow())
        fail(NB_ERR_CONFIG, "layer " + std::to_string(l) +
                                " input shape does not match layer " +
                                std::to_string(l - 1) + " output shape");
    }
    d.specs.push_back(std::move(s));
    d.relu.push_back(net->layers[l].relu != 0);
  }
  return d;
}

bool NetDesc::same_shape(const NetDesc& o) const {
  if (specs.size() != o.specs.size() || num_classes != o.num_classes || seed != o.seed)
    return false;
  for (size_t l = 0; l < specs.size(); ++l)
    if (!(specs[l] == o.specs[l]) || relu[l] != o.relu[l]) return false;
  return true;
}

uint64_t NetDesc::hash() const {
  uint64_t h0 = mix(uint64_t(num_classes), seed);
  for (size_t l = 0; l < specs.size(); ++l) {
    h0 = mix(h0, specs[l].hash());
    h0 = mix(h0, relu[l] ? 1 : 2);
  }
  return h0;
}

int64_t NetDesc::fprop_macs() const {
  int64_t t = 0;
  for (const auto& s : specs) t += s.macs();
  return t;
}

int64_t NetDesc::dgrad_macs() const {
  int64_t t = 0;
  for (size_t l = 1; l < specs.size(); ++l) t += specs[l].macs();
  return t;
}

// ---------------------------------------------------------------------------
// z-stream cache (the reference's init_weights draws, generated once per
// (seed, stream) and extended on demand).

namespace {
struct ZKey {
  uint64_t seed;
  int64_t stream;
  bool operator<(const ZKey& o) const {
    return seed != o.seed ? seed < o.seed : stream < o.stream;
  }
};
std::mutex g_z_mu;
std::map<ZKey, std::shared_ptr<std::vector<double>>> g_z;
}  // namespace

const std::vector<double>& z_stream(uint64_t seed, int64_t stream, int64_t count) {
  {
    std::lock_guard<std::mutex> lk(g_z_mu);
    auto& slot = g_z[{seed, stream}];
    if (slot && int64_t(slot->size()) >= count) return *slot;
  }
  // Generated outside the lock so z_prefetch can fill several layers'
  // streams at once; a racing thread producing the same stream produces
  // the same numbers, and the longer vector wins.
  // Same engine seeding and draw sequence as I/nnet.hpp:64-68 / :72-75.
  auto v = std::make_shared<std::vector<double>>(size_t(count));
  std::mt19937_64 rng(seed * 0x9e3779b97f4a7c15ull + uint64_t(stream) + 1);
  std::normal_distribution<double> dist(0.0, 1.0);
  for (double& x : *v) x = dist(rng);
  std::lock_guard<std::mutex> lk(g_z_mu);
  auto& slot = g_z[{seed, stream}];
  if (!slot || slot->size() < v->size()) {
    slot = v;  // older (shorter) vectors stay alive in holders' copies only
    static std::vector<std::shared_ptr<std::vector<double>>> keep;
    keep.push_back(v);  // references handed out must outlive extensions
  }
  return *slot;
}

void z_prefetch(uint64_t seed, const std::vector<std::pair<int64_t, int64_t>>& streams) {
  // Longest first, so the 2.4M-draw layers do not start last.
  std::vector<std::pair<int64_t, int64_t>> todo(streams);
  std::sort(todo.begin(), todo.end(),
            [](const auto& a, const auto& b) { return a.second > b.second; });
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nt = std::min<size_t>(todo.size(), std::min(hw, 16u));
  std::atomic<size_t> next{0};
  std::vector<std::thread> pool;
  for (size_t t = 0; t < nt; ++t)
    pool.emplace_back([&] {
      for (size_t i; (i = next.fetch_add(1)) < todo.size();)
        z_stream(seed, todo[i].first, todo[i].second);
    });
  for (auto& th : pool) th.join();
}

// make_batch, I/nnet.hpp:87-101: per example Ci*H*W normals, then one label.
void make_batch(const NetDesc& net, int64_t n, uint64_t seed, double* x, int32_t* labels) {
  const Spec& s0 = net.specs.front();
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(0.0, 1.0);
  std::uniform_int_distribution<int> lab(0, int(net.num_classes) - 1);
  const int64_t per = s0.ci * s0.h * s0.w;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < per; ++j) x[i * per + j] = dist(rng);
    labels[i] = lab(rng);
  }
}

}  // namespace nb

using namespace nb;

extern "C" {

const char* nb_version(void) { return "nb200 0.1 (sm_100a)"; }
int nb_abi_version(void) { return NB200_ABI_VERSION; }
const char* nb_last_error(void) { return g_last_error.c_str(); }

nb_status nb_validate_spec(const nb_conv_spec* spec) {
  return guard([&] {
    if (!spec) fail(NB_ERR_INVALID_SPEC, "null spec");
    Spec::from(*spec).validate();
  });
}

nb_status nb_validate_network(const nb_network* net) {
  return guard([&] { NetDesc::from(net); });
}

nb_status nb_conv_macs(const nb_conv_spec* spec, int64_t* macs) {
  return guard([&] {
    Spec s = Spec::from(*spec);
    s.validate();
    *macs = s.macs();
  });
}

nb_status nb_network_macs(const nb_network* net, int64_t* macs) {
  return guard([&] {
    // network_macs (I/search.hpp:84-88) validates each spec via conv_nest.
    if (!net || net->num_layers < 1) fail(NB_ERR_CONFIG, "network has no layers");
    int64_t t = 0;
    for (int64_t l = 0; l < net->num_layers; ++l) {
      Spec s = Spec::from(net->layers[l].spec);
      s.validate();
      t += s.macs();
    }
    *macs = t;
  });
}

// repair_network shape propagation, I/nnet.hpp:372-382, then validate.
nb_status nb_repair_network(int64_t num_layers, nb_layer* layers) {
  return guard([&] {
    for (int64_t l = 1; l < num_layers; ++l) {
      Spec p = Spec::from(layers[l - 1].spec);
      nb_conv_spec& c = layers[l].spec;
      c.ci = p.co_eff();
      c.h = p.oh();
      c.w = p.ow();
    }
    nb_network net{num_layers, layers, 2, 0};
    NetDesc::from(&net);
  });
}

nb_status nb_schedule_lpt(const double* cost, int64_t count, int32_t bins,
                          int32_t* assignment) {
  return guard([&] {
    if (bins < 1) fail(NB_ERR_CONFIG, "need at least one bin");
    std::vector<int64_t> order(static_cast<size_t>(count));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int64_t a, int64_t b) { return cost[a] > cost[b]; });
    std::vector<double> load(size_t(bins), 0.0);
    for (int64_t j : order) {
      int32_t best = 0;
      for (int32_t b = 1; b < bins; ++b)
        if (load[b] < load[best]) best = b;
      assignment[j] = best;
      load[best] += cost[j];
    }
  });
}

nb_status nb_fisher_flops(const nb_network* net, int64_t n, double* flops) {
  return guard([&] {
    NetDesc d = NetDesc::from(net);
    *flops = 2.0 * double(n) * double(d.fprop_macs() + d.dgrad_macs());
  });
}

nb_status nb_init_weights(const nb_network* net, double* weights, double* head) {
  return guard([&] {
    NetDesc d = NetDesc::from(net);
    std::vector<std::pair<int64_t, int64_t>> want;
    for (int64_t l = 0; l < d.L(); ++l) want.push_back({l, d.specs[l].weight_count()});
    want.push_back({d.L(), d.num_classes * d.c_last()});
    z_prefetch(d.seed, want);
    size_t off = 0;
    for (int64_t l = 0; l < d.L(); ++l) {
      const Spec& s = d.specs[l];
      const int64_t cnt = s.weight_count();
      const auto& z = z_stream(d.seed, l, cnt);
      const double sd = 1.0 / std::sqrt(double(s.ci * s.kh * s.kw));
      if (weights)
        for (int64_t k = 0; k < cnt; ++k) weights[off + k] = z[k] * sd + 0.0;
      off += size_t(cnt);
    }
    const int64_t hc = d.num_classes * d.c_last();
    const auto& z = z_stream(d.seed, d.L(), hc);
    const double sd = 1.0 / std::sqrt(double(d.c_last()));
    if (head)
      for (int64_t k = 0; k < hc; ++k) head[k] = z[k] * sd + 0.0;
  });
}

nb_status nb_make_batch(const nb_network* net, int64_t n, uint64_t seed, double* inputs,
                        int32_t* labels) {
  return guard([&] {
    NetDesc d = NetDesc::from(net);
    make_batch(d, n, seed, inputs, labels);
  });
}

int nb_fisher_accepts(const nb_fisher_out* original, const nb_fisher_out* candidate) {
  return candidate->total >= original->total;  // I/nnet.hpp:356-359
}

}  // extern "C"

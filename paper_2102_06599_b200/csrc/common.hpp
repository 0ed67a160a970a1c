// Shared host-side definitions of the nb200 library.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "nb200.h"

namespace nb {

// NVTX range over a scope (scheduler calls, evaluations, layers), for
// Nsight Systems / `ncu --nvtx` filtering; header-only NVTX3, a no-op when no
// tool is attached.
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
  Range(const Range&) = delete;
  Range& operator=(const Range&) = delete;
};

// Status-carrying exception; converted to nb_status at the C ABI.
struct Error : std::runtime_error {
  nb_status status;
  Error(nb_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(nb_status s, const std::string& m) { throw Error(s, m); }

void set_last_error(const std::string& m);

// Runs f, mapping exceptions onto nb_status (the ABI never throws).
template <typename F>
nb_status guard(F&& f) {
  try {
    f();
    return NB_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc& e) {
    set_last_error("host out of memory");
    return NB_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return NB_ERR_INTERNAL;
  }
}

// Value copy of one ConvSpec (I/ir.hpp:26-87) with its derived shapes.
struct Spec {
  int64_t ci = 1, co = 1, h = 1, w = 1, kh = 1, kw = 1, stride = 1, pad = 0,
          groups = 1, bottleneck_out = 1, sdh = 1, sdw = 1;
  std::vector<nb_channel_split> splits;

  static Spec from(const nb_conv_spec& s);
  int64_t co_eff() const { return co / bottleneck_out; }
  int64_t raw_oh() const { return (h + 2 * pad - kh) / stride + 1; }
  int64_t raw_ow() const { return (w + 2 * pad - kw) / stride + 1; }
  int64_t oh() const { return raw_oh() / sdh; }
  int64_t ow() const { return raw_ow() / sdw; }
  std::vector<nb_channel_split> ranges() const {  // I/ir.hpp:54-57
    if (!splits.empty()) return splits;
    return {{0, co_eff(), groups}};
  }
  void validate() const;     // ConvSpec::validate, I/ir.hpp:59-86
  int64_t macs() const;      // count_macs(conv_nest(spec)), padded taps included
  int64_t weight_count() const { return co_eff() * ci * kh * kw; }
  bool operator==(const Spec& o) const;
  uint64_t hash() const;
};

struct NetDesc {
  std::vector<Spec> specs;
  std::vector<bool> relu;
  int64_t num_classes = 10;
  uint64_t seed = 0;

  static NetDesc from(const nb_network* net);  // validates (Network::validate)
  int64_t L() const { return int64_t(specs.size()); }
  int64_t c_last() const { return specs.back().co_eff(); }
  bool same_shape(const NetDesc& o) const;
  uint64_t hash() const;
  int64_t fprop_macs() const;
  int64_t dgrad_macs() const;  // layers >= 1 (I/nnet.hpp:225)
};

// Per-(seed, layer) standard-normal stream z_l of Network::init_weights
// (I/nnet.hpp:64-68): weights of layer l are z_l[k] * (1/sqrt(Ci*Kh*Kw)), the
// head is z_L[k] * (1/sqrt(C_last)).  libstdc++'s normal_distribution
// returns z*stddev + mean, so scaling a cached prefix is bit-exact.
const std::vector<double>& z_stream(uint64_t seed, int64_t stream, int64_t count);
// Fills several (stream, count) z-streams in parallel host threads.
void z_prefetch(uint64_t seed, const std::vector<std::pair<int64_t, int64_t>>& streams);

void make_batch(const NetDesc& net, int64_t n, uint64_t seed, double* x, int32_t* labels);

}  // namespace nb

// Candidate scheduler: the B200 replacement of evaluate_all
// (I/search.hpp:315-334).  The reference runs `jobs` CPU threads that pull
// candidate indices from an atomic counter; here candidates are first
// de-duplicated (identical networks score bit-identically, so one run
// answers all copies -- this is what makes the reference's exact ties,
// I/nnet.hpp:358, reproducible), then assigned to GPUs longest-processing-
// time-first on their estimated FLOPs, and one host worker per GPU keeps
// one evaluation in flight on each of that GPU's sessions (streams).
// Results land in fixed slots, so the output does not depend on the number
// of GPUs or sessions.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>
#include <unordered_map>

#include "engine.hpp"

using namespace nb;

namespace {
struct Result {
  std::vector<double> per_channel, per_layer, probs;
  double total = 0, loss = 0;
};
}  // namespace

extern "C" nb_status nb_evaluate(nb_session* const* sessions, int32_t num_sessions,
                                 const nb_network* nets, int64_t count, nb_precision prec,
                                 nb_fisher_out* outs, nb_eval_stats* stats) {
  return guard([&] {
    if (num_sessions < 1 || !sessions) fail(NB_ERR_CONFIG, "need at least one session");
    if (num_sessions > 16) fail(NB_ERR_UNSUPPORTED, "at most 16 sessions per call");
    if (count < 0 || (count > 0 && (!nets || !outs))) fail(NB_ERR_CONFIG, "null candidates");
    const int64_t N = sessions[0]->n;
    std::vector<NetDesc> descs;
    descs.reserve(size_t(count));
    for (int64_t i = 0; i < count; ++i) descs.push_back(NetDesc::from(&nets[i]));

    // Dedupe: first occurrence of each distinct network is the one run.
    std::vector<int64_t> rep(static_cast<size_t>(count));
    std::vector<int64_t> uniq;
    std::unordered_multimap<uint64_t, int64_t> seen;
    for (int64_t i = 0; i < count; ++i) {
      const uint64_t h = descs[i].hash();
      int64_t found = -1;
      auto range = seen.equal_range(h);
      for (auto it = range.first; it != range.second; ++it)
        if (descs[it->second].same_shape(descs[i])) {
          found = it->second;
          break;
        }
      if (found < 0) {
        seen.emplace(h, i);
        uniq.push_back(i);
        rep[i] = i;
      } else {
        rep[i] = found;
      }
    }

    // LPT on estimated FLOPs (2*N*(fprop + dgrad MACs)).
    std::vector<double> cost(uniq.size());
    for (size_t u = 0; u < uniq.size(); ++u)
      cost[u] = 2.0 * double(N) *
                double(descs[uniq[u]].fprop_macs() + descs[uniq[u]].dgrad_macs());
    std::vector<int32_t> bin(uniq.size(), 0);
    if (!uniq.empty()) {
      nb_status st = nb_schedule_lpt(cost.data(), int64_t(uniq.size()), num_sessions, bin.data());
      if (st != NB_OK) fail(st, nb_last_error());
    }
    // within a worker, largest first (the LPT order)
    std::vector<size_t> order(uniq.size());
    for (size_t u = 0; u < order.size(); ++u) order[u] = u;
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t a, size_t b) { return cost[a] > cost[b]; });

    // One host worker per GPU drives all of that GPU's sessions round-robin:
    // it enqueues an evaluation on each session's stream and collects the
    // oldest only when its session comes round again, so up to
    // (sessions per GPU) evaluations are in flight without several host
    // threads contending for the same device.
    std::vector<Result> res(uniq.size());
    for (size_t u = 0; u < uniq.size(); ++u) {
      const NetDesc& d = descs[uniq[u]];
      int64_t ch = 0;
      for (const auto& sp : d.specs) ch += sp.co_eff();
      res[u].per_channel.resize(size_t(ch));
      res[u].per_layer.resize(size_t(d.L()));
      res[u].probs.resize(size_t(N * d.num_classes));
    }
    std::vector<int> devs;
    for (int32_t k = 0; k < num_sessions; ++k)
      if (std::find(devs.begin(), devs.end(), sessions[k]->ctx->device) == devs.end())
        devs.push_back(sessions[k]->ctx->device);
    std::vector<double> busy(size_t(num_sessions), 0.0), est(size_t(num_sessions), 0.0);
    std::exception_ptr err;
    std::mutex err_mu;
    auto worker = [&](int dev) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<int32_t> mine;  // this GPU's sessions
      for (int32_t k = 0; k < num_sessions; ++k)
        if (sessions[k]->ctx->device == dev) mine.push_back(k);
      // this GPU's networks, largest first, interleaved from its sessions' LPT bins
      std::vector<std::pair<size_t, int32_t>> work;
      for (size_t u : order)
        if (std::find(mine.begin(), mine.end(), bin[u]) != mine.end())
          work.emplace_back(u, bin[u]);
      std::vector<Pending> pend(mine.size());
      try {
        for (size_t i = 0; i < work.size(); ++i) {
          const size_t slot = i % mine.size();
          run_finish(pend[slot]);
          const size_t u = work[i].first;
          Result& r = res[u];
          RunOut ro;
          ro.per_channel = r.per_channel.data();
          ro.per_layer = r.per_layer.data();
          ro.total = &r.total;
          ro.loss = &r.loss;
          ro.probs = r.probs.data();
          run_enqueue(sessions[mine[slot]], descs[uniq[u]], nullptr, prec, true, ro, pend[slot]);
          est[size_t(mine[slot])] += cost[u];
        }
        for (auto& p : pend) run_finish(p);
      } catch (...) {
        std::lock_guard<std::mutex> lk(err_mu);
        if (!err) err = std::current_exception();
        for (auto& p : pend) {
          try {
            run_finish(p);
          } catch (...) {
          }
        }
      }
      const double ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      for (int32_t k : mine) busy[size_t(k)] = ms;
    };
    // NB_SCHED_THREADS=1: one host thread per session instead of per GPU
    // (launch submission in parallel; each thread keeps one evaluation of its
    // session in flight)
    static const bool per_session = [] {
      const char* e = std::getenv("NB_SCHED_THREADS");
      return e && std::atoi(e) == 1;
    }();
    auto session_worker = [&](int32_t k) {
      auto t0 = std::chrono::steady_clock::now();
      Pending pend;
      try {
        for (size_t u : order) {
          if (bin[u] != k) continue;
          Result& r = res[u];
          RunOut ro;
          ro.per_channel = r.per_channel.data();
          ro.per_layer = r.per_layer.data();
          ro.total = &r.total;
          ro.loss = &r.loss;
          ro.probs = r.probs.data();
          run_enqueue(sessions[k], descs[uniq[u]], nullptr, prec, true, ro, pend);
          est[size_t(k)] += cost[u];
          run_finish(pend);
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(err_mu);
        if (!err) err = std::current_exception();
        try {
          run_finish(pend);
        } catch (...) {
        }
      }
      busy[size_t(k)] =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    if (per_session && num_sessions > 1) {
      std::vector<std::thread> pool;
      for (int32_t k = 0; k < num_sessions; ++k) pool.emplace_back(session_worker, k);
      for (auto& t : pool) t.join();
    } else if (devs.size() == 1) {
      worker(devs[0]);
    } else {
      std::vector<std::thread> pool;
      for (int d : devs) pool.emplace_back(worker, d);
      for (auto& t : pool) t.join();
    }
    if (err) std::rethrow_exception(err);

    std::vector<size_t> slot_of(size_t(count), 0);
    for (size_t u = 0; u < uniq.size(); ++u) slot_of[size_t(uniq[u])] = u;
    for (int64_t i = 0; i < count; ++i) {
      const Result& r = res[slot_of[size_t(rep[i])]];
      nb_fisher_out& o = outs[i];
      if (o.per_channel) std::copy(r.per_channel.begin(), r.per_channel.end(), o.per_channel);
      if (o.per_layer) std::copy(r.per_layer.begin(), r.per_layer.end(), o.per_layer);
      if (o.probs) std::copy(r.probs.begin(), r.probs.end(), o.probs);
      o.total = r.total;
      o.loss = r.loss;
      o.seed = sessions[0]->seed;
    }
    if (stats) {
      stats->evaluated = int64_t(uniq.size());
      stats->deduplicated = count - int64_t(uniq.size());
      for (int k = 0; k < 16; ++k) {
        stats->est_flops[k] = k < num_sessions ? est[size_t(k)] : 0.0;
        stats->busy_ms[k] = k < num_sessions ? busy[size_t(k)] : 0.0;
      }
    }
  });
}

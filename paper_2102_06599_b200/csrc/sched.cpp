// Candidate scheduler: the B200 replacement of evaluate_all
// (I/search.hpp:315-334).  The reference runs `jobs` CPU threads that pull
// candidate indices from an atomic counter (dynamic self-scheduling); here:
//
//  * candidates are de-duplicated first -- identical networks score
//    bit-identically, so one run answers all copies (this is what makes the
//    reference's exact ties, I/nnet.hpp:358, reproducible);
//  * the distinct networks form ONE queue in longest-processing-time order
//    (estimated FLOPs 2*N*(fprop + dgrad MACs), ties by index), which every
//    session pulls from whenever its previous evaluation has completed on
//    the device -- list scheduling in LPT order, so a GPU whose candidates
//    run faster than estimated simply takes more of them;
//  * one host worker per GPU drives all of that GPU's sessions (a session =
//    a context with its own stream holding the batch): it enqueues an
//    evaluation asynchronously and polls its completion event, keeping one
//    evaluation in flight per session without several host threads
//    contending for the same device;
//  * a device failure (CUDA error, out of memory) on one session retires
//    that session and re-queues its candidate for the others; only when no
//    session is left does the call fail;
//  * results land in fixed per-candidate slots, so the output does not
//    depend on the number of GPUs or sessions, nor on which session ran
//    what (every session plans identically for the same batch).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <deque>
#include <exception>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <unordered_set>

#include "engine.hpp"

using namespace nb;

namespace {
struct Result {
  std::vector<double> per_channel, per_layer, probs;
  double total = 0, loss = 0;
};

bool device_failure(nb_status s) { return s == NB_ERR_CUDA || s == NB_ERR_OUT_OF_MEMORY; }

// NB_SCHED_FAULT=k: the k-th session's first evaluation fails as a device
// error (fault injection for the re-queue path; tests/test_sched.py).
int injected_fault_session() {
  const char* e = std::getenv("NB_SCHED_FAULT");
  return e && *e ? std::atoi(e) : -1;
}
}  // namespace

extern "C" nb_status nb_evaluate(nb_session* const* sessions, int32_t num_sessions,
                                 const nb_network* nets, int64_t count, nb_precision prec,
                                 nb_fisher_out* outs, nb_eval_stats* stats) {
  return guard([&] {
    Range range("nb_evaluate");
    if (num_sessions < 1 || !sessions) fail(NB_ERR_CONFIG, "need at least one session");
    if (count < 0 || (count > 0 && (!nets || !outs))) fail(NB_ERR_CONFIG, "null candidates");
    // every session holds the same batch on its own context: a context's
    // result staging and arenas serve one evaluation at a time
    std::unordered_set<const nb_ctx*> ctxs;
    for (int32_t k = 0; k < num_sessions; ++k) {
      const nb_session* s = sessions[k];
      if (!s || !s->ctx) fail(NB_ERR_CONFIG, "null session");
      if (!ctxs.insert(s->ctx).second)
        fail(NB_ERR_CONFIG, "two sessions share a context (one context per session)");
      const nb_session* s0 = sessions[0];
      if (s->n != s0->n || s->seed != s0->seed || s->ci != s0->ci || s->h != s0->h ||
          s->w != s0->w || s->num_classes != s0->num_classes)
        fail(NB_ERR_CONFIG, "sessions hold different batches");
    }
    const int64_t N = sessions[0]->n;
    std::vector<NetDesc> descs;
    descs.reserve(size_t(count));
    for (int64_t i = 0; i < count; ++i) descs.push_back(NetDesc::from(&nets[i]));

    // Dedupe: the first occurrence of each distinct network is the one run.
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

    // The LPT-ordered queue of distinct networks.
    std::vector<double> cost(uniq.size());
    for (size_t u = 0; u < uniq.size(); ++u)
      cost[u] = 2.0 * double(N) *
                double(descs[uniq[u]].fprop_macs() + descs[uniq[u]].dgrad_macs());
    std::vector<size_t> order(uniq.size());
    for (size_t u = 0; u < order.size(); ++u) order[u] = u;
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t a, size_t b) { return cost[a] > cost[b]; });
    std::deque<size_t> queue(order.begin(), order.end());

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

    // Every session's run buffers sized for the largest distinct network
    // before any evaluation starts: a buffer grown mid-call reallocates, and
    // a reallocation synchronizes the whole device (stalling every stream).
    {
      const int64_t L0 = uniq.empty() ? 0 : descs[uniq[0]].L();
      NetPlan need;
      int64_t maxL = L0, maxK = 1;
      bool h16 = false;
      for (size_t u = 0; u < uniq.size(); ++u) {
        const NetDesc& d = descs[uniq[u]];
        const NetPlan P = lower(d, N, prec, sessions[0]->ctx->num_sms, N, true);
        need.act_total = std::max(need.act_total, P.act_total);
        need.part_total = std::max(need.part_total, P.part_total);
        need.ws_floats = std::max(need.ws_floats, P.ws_floats);
        need.dpre_floats = std::max(need.dpre_floats, P.dpre_floats);
        need.ch_total = std::max(need.ch_total, P.ch_total);
        maxL = std::max(maxL, d.L());
        maxK = std::max(maxK, d.num_classes);
        h16 = h16 || P.h16 == 2;
      }
      need.h16 = h16 ? 2 : 0;
      if (!uniq.empty())
        for (int32_t k = 0; k < num_sessions; ++k) {
          nb_ctx* c = sessions[k]->ctx;
          std::lock_guard<std::recursive_mutex> lk(c->mu);
          ctx_activate(c);
          reserve_run(c, need, N, maxK, maxL, false, false);
        }
    }

    const size_t S = size_t(num_sessions);
    // NB_SCHED_LOG: per-evaluation enqueue / completion times (experiments)
    static const bool sched_log = std::getenv("NB_SCHED_LOG") != nullptr;
    const auto t_call = std::chrono::steady_clock::now();
    std::vector<double> busy(S, 0.0), est(S, 0.0);
    std::vector<int64_t> done(S, 0);
    std::mutex mu;  // guards queue, outstanding, alive, fatal, requeued
    int64_t outstanding = int64_t(uniq.size());
    int alive = num_sessions;
    int64_t requeued = 0;
    std::exception_ptr fatal, last_device_error;
    const int fault_at = injected_fault_session();

    auto worker = [&](int dev) {
      std::vector<int32_t> mine;
      for (int32_t k = 0; k < num_sessions; ++k)
        if (sessions[k]->ctx->device == dev) mine.push_back(k);
      std::vector<Pending> pend(mine.size());
      std::vector<size_t> cur(mine.size(), 0);
      std::vector<char> dead(mine.size(), 0), faulted(mine.size(), 0);
      // a failure of slot j on network u: device errors retire the session
      // and hand u back to the queue; anything else ends the call
      auto on_fail = [&](size_t j, size_t u) {
        std::lock_guard<std::mutex> lk(mu);
        try {
          throw;
        } catch (const Error& e) {
          if (device_failure(e.status)) {
            dead[j] = 1;
            --alive;
            queue.push_front(u);
            ++requeued;
            last_device_error = std::current_exception();
            if (alive == 0 && !fatal) fatal = last_device_error;
            return;
          }
          if (!fatal) fatal = std::current_exception();
        } catch (...) {
          if (!fatal) fatal = std::current_exception();
        }
      };
      for (;;) {
        bool progress = false, busy_slots = false;
        for (size_t j = 0; j < mine.size(); ++j) {
          if (dead[j]) continue;
          const int32_t k = mine[j];
          if (pend[j].active) {
            if (!run_ready(pend[j])) {
              busy_slots = true;
              continue;
            }
            try {
              run_finish(pend[j]);
              busy[size_t(k)] += run_device_ms(sessions[k]->ctx);
              if (sched_log)
                std::fprintf(stderr, "sched s%d done at %.3f ms (device %.3f ms)\n", k,
                             std::chrono::duration<double, std::milli>(
                                 std::chrono::steady_clock::now() - t_call).count(),
                             run_device_ms(sessions[k]->ctx));
              ++done[size_t(k)];
              std::lock_guard<std::mutex> lk(mu);
              --outstanding;
            } catch (...) {
              on_fail(j, cur[j]);
              continue;
            }
            progress = true;
          }
          size_t u;
          {
            std::lock_guard<std::mutex> lk(mu);
            if (fatal || queue.empty()) continue;
            u = queue.front();
            queue.pop_front();
          }
          cur[j] = u;
          try {
            if (k == fault_at && !faulted[j]) {
              faulted[j] = 1;
              fail(NB_ERR_CUDA, "injected device fault (NB_SCHED_FAULT)");
            }
            Result& r = res[u];
            RunOut ro;
            ro.per_channel = r.per_channel.data();
            ro.per_layer = r.per_layer.data();
            ro.total = &r.total;
            ro.loss = &r.loss;
            ro.probs = r.probs.data();
            const auto te0 = std::chrono::steady_clock::now();
            run_enqueue(sessions[k], descs[uniq[u]], nullptr, prec, true, ro, pend[j]);
            if (sched_log)
              std::fprintf(stderr, "sched s%d enq u%zu at %.3f ms (%.3f ms)\n", k, u,
                           std::chrono::duration<double, std::milli>(te0 - t_call).count(),
                           std::chrono::duration<double, std::milli>(
                               std::chrono::steady_clock::now() - te0).count());
            est[size_t(k)] += cost[u];
            busy_slots = true;
            progress = true;
          } catch (...) {
            on_fail(j, u);
          }
        }
        {
          std::lock_guard<std::mutex> lk(mu);
          const bool all_dead = std::all_of(dead.begin(), dead.end(), [](char d) { return d; });
          if ((fatal || outstanding == 0 || all_dead) && !busy_slots) break;
          if (all_dead) break;
        }
        if (!progress) std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
      // a failed call still drains its in-flight evaluations
      for (auto& p : pend) {
        try {
          run_finish(p);
        } catch (...) {
        }
      }
    };
    if (devs.size() == 1) {
      worker(devs[0]);
    } else {
      std::vector<std::thread> pool;
      for (int d : devs) pool.emplace_back(worker, d);
      for (auto& t : pool) t.join();
    }
    if (fatal) std::rethrow_exception(fatal);
    if (outstanding != 0) {
      if (last_device_error) std::rethrow_exception(last_device_error);
      fail(NB_ERR_INTERNAL, "scheduler finished with unevaluated candidates");
    }

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
      stats->requeued = requeued;
      stats->failed_sessions = num_sessions - alive;
      for (size_t k = 0; k < S; ++k) {
        if (stats->est_flops) stats->est_flops[k] = est[k];
        if (stats->busy_ms) stats->busy_ms[k] = busy[k];
        if (stats->evaluations) stats->evaluations[k] = done[k];
      }
    }
  });
}

// Semantic legality on the GPU: check_semantic_legality
// (I/transforms.hpp:598-663) over compute_dependences(original, cap, false)
// (I/ir.hpp:326-403), same verdicts and the same first reordered pair.
//
// The reference builds the dependence set on the host as vectors of
// vector<long long> (one heap object per instance and per touch), sorts them
// and binary-searches the transformed schedule -- about 4 s for a nest at the
// 1e6-instance cap.  Here every instance and touch is one 64-bit key:
//   instance key = sid | (domain coordinate - lo) packed per sid
//   touch key    = tensor | (cell - lo) packed per tensor | original rank
// so both sorts are CUB radix sorts over exactly the bits in use, and the
// sorted order is the reference's (sid, coord) / (tensor, cell, inst)
// lexicographic order.  Passes, one thread per instance / touch:
//   1 enumerate the transformed nest -> (key, schedule rank); radix sort;
//     adjacent equal keys = "duplicates an instance"
//   2 enumerate the original -> rankT[inst] (binary search of its key in the
//     sorted transformed keys; MISS = not an instance of the transformed
//     nest) and its touches of written tensors; radix sort
//   3 per touch j: scan the earlier touches i of its cell group in order,
//     form the reference's pairs (i, j) (a write among them, different
//     instances, not one accumulation chain) and test rankT order; the
//     first failing (i, j) in the reference's iteration order is an atomicMin
//     over (i << 32 | j)
// The verdict and message need only that pair: missing rank -> "instance sets
// differ", else "dependence ... is reordered" with both instances decoded.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "engine.hpp"
#include "nest_expr.cuh"

namespace nb {
namespace {

constexpr int kLDepth = 24, kLDom = 8, kLAcc = 4, kLRank = 8, kMaxSid = 16, kMaxTen = 8;
constexpr uint32_t kMiss = 0xffffffffu;
// bound on the pair-scan work (sum over cell groups of g*(g-1)/2); beyond it
// the call returns NB_ERR_UNSUPPORTED and the caller runs the host check
constexpr unsigned long long kScanBudget = 200ull * 1000 * 1000 * 1000;

struct LAcc {
  int tensor, mode, rank;
  int idx_off[kLRank];
};

struct LStmt {
  int depth, ndomain, naccess, sid, gid;
  int64_t count, ioff, toff;  // instances; first global instance / touch index
  int64_t rank_base;
  int64_t ext[kLDepth], stride[kLDepth];
  int coord_off[kLDom];
  LAcc acc[kLAcc];
};

struct Pack {
  int cbits;  // coordinate bits (max over sids); instance key = sid << cbits | coords
  int cellbits, ibits;  // touch key = ((tensor << cellbits) | cell) << ibits | inst
  int64_t slo[kMaxSid][kLDom];
  int sshift[kMaxSid][kLDom];
  int64_t tlo[kMaxTen][kLRank];
  int tshift[kMaxTen][kLRank];
};

struct Result {
  unsigned long long best;  // (i << 32 | j) of the first failing pair
  unsigned long long pairs;
  unsigned long long scan;  // pair-scan work
  int dup;
  int over_budget;
};

__device__ __forceinline__ int find_stmt(const LStmt* s, int ns, int64_t g) {
  int k = 0;
  while (k + 1 < ns && s[k + 1].ioff <= g) ++k;
  return k;
}

// decode the local instance index into loop values (any bijection works:
// the schedule rank comes from the rank formula, not from the index)
__device__ __forceinline__ int64_t loops_and_rank(const LStmt& s, int64_t local, int64_t* v) {
  int64_t r = local, rank = s.rank_base;
  for (int d = s.depth - 1; d >= 0; --d) {
    v[d] = r % s.ext[d];
    r /= s.ext[d];
    rank += v[d] * s.stride[d];
  }
  return rank;
}

__device__ __forceinline__ uint64_t inst_key(const Pack& p, const LStmt& s, const int64_t* dom) {
  uint64_t k = uint64_t(s.sid) << p.cbits;
  for (int i = 0; i < s.ndomain; ++i)
    k |= uint64_t(dom[i] - p.slo[s.sid][i]) << p.sshift[s.sid][i];
  return k;
}

__global__ void k_enum_transformed(const LStmt* __restrict__ stmts, int ns, int64_t n,
                                   const int64_t* __restrict__ code, const Pack p,
                                   uint64_t* __restrict__ keys, uint32_t* __restrict__ ranks) {
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n;
       g += int64_t(gridDim.x) * blockDim.x) {
    const LStmt& s = stmts[find_stmt(stmts, ns, g)];
    int64_t v[kLDepth], dom[kLDom];
    const int64_t rank = loops_and_rank(s, g - s.ioff, v);
    for (int i = 0; i < s.ndomain; ++i) dom[i] = nexpr::run(code, s.coord_off[i], v);
    keys[g] = inst_key(p, s, dom);
    ranks[g] = uint32_t(rank);
  }
}

__global__ void k_adjacent_dup(const uint64_t* __restrict__ keys, int64_t n, Result* res) {
  for (int64_t i = 1 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    if (keys[i] == keys[i - 1]) res->dup = 1;
}

__device__ __forceinline__ int64_t lower_bound(const uint64_t* a, int64_t n, uint64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_enum_original(const LStmt* __restrict__ stmts, int ns, int64_t n,
                                const int64_t* __restrict__ code, const Pack p,
                                const uint64_t* __restrict__ tkeys, const uint32_t* __restrict__ tranks,
                                int64_t n1, uint32_t* __restrict__ rank_t,
                                uint64_t* __restrict__ touch_key, uint32_t* __restrict__ touch_val) {
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n;
       g += int64_t(gridDim.x) * blockDim.x) {
    const LStmt& s = stmts[find_stmt(stmts, ns, g)];
    int64_t v[kLDepth], dom[kLDom];
    const int64_t local = g - s.ioff;
    const int64_t inst = loops_and_rank(s, local, v);  // index in the original schedule
    for (int i = 0; i < s.ndomain; ++i) dom[i] = nexpr::run(code, s.coord_off[i], v);
    const uint64_t key = inst_key(p, s, dom);
    const int64_t pos = lower_bound(tkeys, n1, key);
    rank_t[inst] = (pos < n1 && tkeys[pos] == key) ? tranks[pos] : kMiss;
    for (int a = 0; a < s.naccess; ++a) {
      const LAcc& acc = s.acc[a];
      uint64_t cell = uint64_t(acc.tensor);
      cell <<= p.cellbits;
      for (int k = 0; k < acc.rank; ++k)
        cell |= uint64_t(nexpr::run(code, acc.idx_off[k], dom) - p.tlo[acc.tensor][k])
                << p.tshift[acc.tensor][k];
      const int64_t t = s.toff + local * s.naccess + a;
      touch_key[t] = (cell << p.ibits) | uint64_t(inst);
      touch_val[t] = uint32_t(s.gid) << 2 | uint32_t(acc.mode);
    }
  }
}

// work of the pair scan: sum over cell groups of g*(g-1)/2
__global__ void k_scan_cost(const uint64_t* __restrict__ key, int64_t n, int ibits, Result* res) {
  unsigned long long w = 0;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t grp = key[j] >> ibits;
    if (j > 0 && (key[j - 1] >> ibits) == grp) continue;
    const int64_t end = lower_bound(key, n, (grp + 1) << ibits);
    const unsigned long long g = static_cast<unsigned long long>(end - j);
    w += g * (g - 1) / 2;
  }
  for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
  if ((threadIdx.x & 31) == 0 && w) atomicAdd(&res->scan, w);
}

__global__ void k_pairs(const uint64_t* __restrict__ key, const uint32_t* __restrict__ val,
                        int64_t n, int ibits, const uint32_t* __restrict__ rank_t, Result* res) {
  if (res->scan > kScanBudget) {
    if (blockIdx.x == 0 && threadIdx.x == 0) res->over_budget = 1;
    return;
  }
  const uint64_t imask = (uint64_t(1) << ibits) - 1;
  unsigned long long pairs = 0, first = ~0ull;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t kj = key[j];
    const int64_t start = lower_bound(key, j, (kj >> ibits) << ibits);
    const uint32_t vj = val[j];
    const uint32_t mj = vj & 3u, gj = vj >> 2;
    const uint64_t ij = kj & imask;
    const uint32_t rj = rank_t[ij];
    for (int64_t i = start; i < j; ++i) {
      const uint32_t vi = val[i];
      const uint32_t mi = vi & 3u;
      if (mi == 0 && mj == 0) continue;                 // two reads
      if (mi == 2 && mj == 2 && (vi >> 2) == gj) continue;  // one accumulation chain
      const uint64_t ii = key[i] & imask;
      if (ii == ij) continue;                           // same instance
      ++pairs;
      const uint32_t ri = rank_t[ii];
      if (ri == kMiss || rj == kMiss || ri >= rj) {
        first = min(first, (static_cast<unsigned long long>(i) << 32) |
                               static_cast<unsigned long long>(j));
        break;
      }
    }
  }
  // one atomic per warp: when every touch fails (e.g. all inits after their
  // accumulations) per-thread atomics on one word serialize
  for (int o = 16; o; o >>= 1) {
    pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
    first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (pairs) atomicAdd(&res->pairs, pairs);
    if (first != ~0ull) atomicMin(&res->best, first);
  }
}

struct Described {
  int stmt[2];
  int64_t coord[2][kLDom];
};

// statement entry and domain coordinate of two original instances
__global__ void k_describe(const LStmt* __restrict__ stmts, int ns, int64_t n,
                           const int64_t* __restrict__ code, int64_t a, int64_t b,
                           Described* out) {
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < n;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int si = find_stmt(stmts, ns, g);
    const LStmt& s = stmts[si];
    int64_t v[kLDepth];
    const int64_t inst = loops_and_rank(s, g - s.ioff, v);
    if (inst != a && inst != b) continue;
    const int w = inst == a ? 0 : 1;
    out->stmt[w] = si;
    for (int i = 0; i < s.ndomain; ++i) out->coord[w][i] = nexpr::run(code, s.coord_off[i], v);
    if (a == b) {
      out->stmt[1] = si;
      for (int i = 0; i < s.ndomain; ++i) out->coord[1][i] = out->coord[0][i];
    }
  }
}

int bits_for(uint64_t span) {  // bits to hold values 0..span
  int b = 0;
  while (b < 64 && (span >> b) != 0) ++b;
  return b;
}

struct Flat {
  std::vector<LStmt> stmts;
  int64_t n = 0, touches = 0;
};

}  // namespace
}  // namespace nb

using namespace nb;

extern "C" nb_status nb_semantic_legality(nb_ctx* ctx, const nb_legal_nest* original,
                                          const nb_legal_nest* transformed, nb_legal_out* out) {
  return guard([&] {
    Range range("nb_semantic_legality");
    if (!ctx || !original || !transformed || !out) fail(NB_ERR_CONFIG, "null argument");
    std::memset(out, 0, sizeof(*out));
    std::vector<int64_t> code;
    auto add = [&](const nb_nest_expr& e) {
      const int off = int(code.size() / 2);
      code.push_back(e.nops);
      code.push_back(0);
      int depth = 0, maxd = 0;
      for (int i = 0; i < e.nops; ++i) {
        const int64_t op = e.code[2 * i], arg = e.code[2 * i + 1];
        if (op < 0 || op > 5) fail(NB_ERR_CONFIG, "bad nest expression op");
        if ((op == 4 || op == 5) && arg == 0) fail(NB_ERR_CONFIG, "division by zero in a nest");
        depth += op <= 1 ? 1 : op == 2 ? 1 - int(arg) : 0;
        if (depth < 1) fail(NB_ERR_CONFIG, "malformed nest expression");
        maxd = std::max(maxd, depth);
        code.push_back(op);
        code.push_back(arg);
      }
      if (depth != 1 || maxd > nexpr::kStack) fail(NB_ERR_UNSUPPORTED, "nest expression too deep");
      return off;
    };
    // per-sid / per-tensor bounds (union over both nests) -> packing
    int64_t slo[kMaxSid][kLDom], shi[kMaxSid][kLDom], tlo[kMaxTen][kLRank], thi[kMaxTen][kLRank];
    int sdom[kMaxSid], trank[kMaxTen];
    std::fill(sdom, sdom + kMaxSid, -1);
    std::fill(trank, trank + kMaxTen, -1);
    auto flatten = [&](const nb_legal_nest* nest, bool orig) {
      Flat f;
      for (int64_t i = 0; i < nest->num_stmts; ++i) {
        const nb_legal_stmt& src = nest->stmts[i];
        if (src.depth > kLDepth || src.ndomain > kLDom || src.naccess > kLAcc || src.sid < 0 ||
            src.sid >= kMaxSid || src.gid < 0 || src.gid >= (1 << 29))
          fail(NB_ERR_UNSUPPORTED, "nest exceeds the legality kernel's limits");
        if (!orig && src.naccess) fail(NB_ERR_CONFIG, "transformed entries carry no accesses");
        LStmt d{};
        d.depth = src.depth;
        d.ndomain = src.ndomain;
        d.naccess = src.naccess;
        d.sid = src.sid;
        d.gid = src.gid;
        d.rank_base = src.rank_base;
        int64_t cnt = 1;
        for (int k = 0; k < src.depth; ++k) {
          if (src.extents[k] < 0) fail(NB_ERR_CONFIG, "negative extent");
          d.ext[k] = src.extents[k];
          d.stride[k] = src.rank_stride[k];
          cnt *= src.extents[k];
        }
        d.count = cnt;
        d.ioff = f.n;
        d.toff = f.touches;
        if (sdom[src.sid] >= 0 && sdom[src.sid] != src.ndomain)
          fail(NB_ERR_UNSUPPORTED, "statement id with two domain arities");
        if (sdom[src.sid] < 0) {
          sdom[src.sid] = src.ndomain;
          for (int k = 0; k < src.ndomain; ++k) slo[src.sid][k] = src.lo[k], shi[src.sid][k] = src.hi[k];
        }
        for (int k = 0; k < src.ndomain; ++k) {
          d.coord_off[k] = add(src.coord[k]);
          slo[src.sid][k] = std::min(slo[src.sid][k], src.lo[k]);
          shi[src.sid][k] = std::max(shi[src.sid][k], src.hi[k]);
        }
        for (int a = 0; a < src.naccess; ++a) {
          const nb_legal_access& sa = src.access[a];
          if (sa.tensor < 0 || sa.tensor >= kMaxTen || sa.rank > kLRank || sa.mode < 0 ||
              sa.mode > 2)
            fail(NB_ERR_UNSUPPORTED, "access exceeds the legality kernel's limits");
          if (trank[sa.tensor] >= 0 && trank[sa.tensor] != sa.rank)
            fail(NB_ERR_UNSUPPORTED, "tensor accessed with two arities");
          if (trank[sa.tensor] < 0) {
            trank[sa.tensor] = sa.rank;
            for (int k = 0; k < sa.rank; ++k) tlo[sa.tensor][k] = sa.lo[k], thi[sa.tensor][k] = sa.hi[k];
          }
          d.acc[a].tensor = sa.tensor;
          d.acc[a].mode = sa.mode;
          d.acc[a].rank = sa.rank;
          for (int k = 0; k < sa.rank; ++k) {
            d.acc[a].idx_off[k] = add(sa.idx[k]);
            tlo[sa.tensor][k] = std::min(tlo[sa.tensor][k], sa.lo[k]);
            thi[sa.tensor][k] = std::max(thi[sa.tensor][k], sa.hi[k]);
          }
        }
        f.n += cnt;
        f.touches += cnt * src.naccess;
        f.stmts.push_back(d);
      }
      return f;
    };
    Flat fo = flatten(original, true), ft = flatten(transformed, false);
    if (fo.n >= (int64_t(1) << 31) || ft.n >= (int64_t(1) << 31) || fo.touches >= (int64_t(1) << 31))
      fail(NB_ERR_UNSUPPORTED, "nest too large for the legality kernel");
    const int64_t code_ops = int64_t(code.size() / 2);
    (void)code_ops;

    Pack p{};
    int nsid = 0, nten = 0;
    for (int s = 0; s < kMaxSid; ++s) {
      if (sdom[s] < 0) continue;
      nsid = s + 1;
      int sh = 0;
      for (int k = sdom[s] - 1; k >= 0; --k) {  // last coordinate least significant
        if (shi[s][k] < slo[s][k]) fail(NB_ERR_CONFIG, "empty coordinate bounds");
        p.slo[s][k] = slo[s][k];
        p.sshift[s][k] = sh;
        sh += bits_for(uint64_t(shi[s][k] - slo[s][k]));
      }
      p.cbits = std::max(p.cbits, sh);
    }
    for (int t = 0; t < kMaxTen; ++t) {
      if (trank[t] < 0) continue;
      nten = t + 1;
      int sh = 0;
      for (int k = trank[t] - 1; k >= 0; --k) {
        if (thi[t][k] < tlo[t][k]) fail(NB_ERR_CONFIG, "empty cell bounds");
        p.tlo[t][k] = tlo[t][k];
        p.tshift[t][k] = sh;
        sh += bits_for(uint64_t(thi[t][k] - tlo[t][k]));
      }
      p.cellbits = std::max(p.cellbits, sh);
    }
    p.ibits = std::max(1, bits_for(uint64_t(std::max<int64_t>(fo.n, 1) - 1)));
    const int sid_bits = bits_for(uint64_t(std::max(nsid, 1) - 1));
    const int ten_bits = bits_for(uint64_t(std::max(nten, 1) - 1));
    const int key_bits = std::max(1, sid_bits + p.cbits);
    const int tkey_bits = std::max(1, ten_bits + p.cellbits + p.ibits);
    if (key_bits > 63 || tkey_bits > 63)
      fail(NB_ERR_UNSUPPORTED, "instance or touch keys do not fit 64 bits");

    const bool same_size = fo.n == ft.n;
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ctx_activate(ctx);
    cudaStream_t st = ctx->stream;
    // workspace layout (256-byte aligned slices of ctx->legal)
    size_t off = 0;
    auto slice = [&](size_t bytes) {
      const size_t o = off;
      off += (bytes + 255) & ~size_t(255);
      return o;
    };
    const int64_t n1 = std::max<int64_t>(ft.n, 1), n0 = std::max<int64_t>(fo.n, 1),
                  nt = std::max<int64_t>(fo.touches, 1);
    size_t sort1 = 0, sort2 = 0;
    NB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort1, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                            (uint32_t*)nullptr, (uint32_t*)nullptr, n1, 0,
                                            key_bits, st));
    NB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort2, (uint64_t*)nullptr, (uint64_t*)nullptr,
                                            (uint32_t*)nullptr, (uint32_t*)nullptr, nt, 0,
                                            tkey_bits, st));
    const size_t o_code = slice(code.size() * 8), o_so = slice(fo.stmts.size() * sizeof(LStmt)),
                 o_st = slice(ft.stmts.size() * sizeof(LStmt)), o_res = slice(sizeof(Result)),
                 o_desc = slice(sizeof(Described)), o_k1 = slice(n1 * 8), o_k1s = slice(n1 * 8),
                 o_r1 = slice(n1 * 4), o_r1s = slice(n1 * 4), o_rt = slice(n0 * 4),
                 o_tk = slice(nt * 8), o_tks = slice(nt * 8), o_tv = slice(nt * 4),
                 o_tvs = slice(nt * 4), o_tmp = slice(std::max(sort1, sort2));
    ctx->legal.ensure(off);
    char* base = static_cast<char*>(ctx->legal.p);
    auto at = [&](size_t o) { return static_cast<void*>(base + o); };
    int64_t* d_code = static_cast<int64_t*>(at(o_code));
    LStmt* d_so = static_cast<LStmt*>(at(o_so));
    LStmt* d_st = static_cast<LStmt*>(at(o_st));
    Result* d_res = static_cast<Result*>(at(o_res));
    Described* d_desc = static_cast<Described*>(at(o_desc));
    uint64_t *k1 = static_cast<uint64_t*>(at(o_k1)), *k1s = static_cast<uint64_t*>(at(o_k1s));
    uint32_t *r1 = static_cast<uint32_t*>(at(o_r1)), *r1s = static_cast<uint32_t*>(at(o_r1s));
    uint32_t* rt = static_cast<uint32_t*>(at(o_rt));
    uint64_t *tk = static_cast<uint64_t*>(at(o_tk)), *tks = static_cast<uint64_t*>(at(o_tks));
    uint32_t *tv = static_cast<uint32_t*>(at(o_tv)), *tvs = static_cast<uint32_t*>(at(o_tvs));
    void* tmp = at(o_tmp);

    if (!code.empty())
      NB_CUDA(cudaMemcpyAsync(d_code, code.data(), code.size() * 8, cudaMemcpyHostToDevice, st));
    if (!fo.stmts.empty())
      NB_CUDA(cudaMemcpyAsync(d_so, fo.stmts.data(), fo.stmts.size() * sizeof(LStmt),
                              cudaMemcpyHostToDevice, st));
    if (!ft.stmts.empty())
      NB_CUDA(cudaMemcpyAsync(d_st, ft.stmts.data(), ft.stmts.size() * sizeof(LStmt),
                              cudaMemcpyHostToDevice, st));
    Result init{~0ull, 0, 0, 0, 0};
    NB_CUDA(cudaMemcpyAsync(d_res, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    auto grid = [&](int64_t n) {
      return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(ctx->num_sms) * 16)));
    };
    if (ft.n > 0) {
      k_enum_transformed<<<grid(ft.n), 256, 0, st>>>(d_st, int(ft.stmts.size()), ft.n, d_code, p,
                                                    k1, r1);
      NB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, sort1, k1, k1s, r1, r1s, ft.n, 0, key_bits, st));
      k_adjacent_dup<<<grid(ft.n), 256, 0, st>>>(k1s, ft.n, d_res);
      ctx->launches += 2;
    }
    if (same_size && fo.n > 0) {
      k_enum_original<<<grid(fo.n), 256, 0, st>>>(d_so, int(fo.stmts.size()), fo.n, d_code, p,
                                                 k1s, r1s, ft.n, rt, tk, tv);
      ctx->launches++;
      if (fo.touches > 0) {
        NB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, sort2, tk, tks, tv, tvs, fo.touches, 0,
                                                tkey_bits, st));
        k_scan_cost<<<grid(fo.touches), 256, 0, st>>>(tks, fo.touches, p.ibits, d_res);
        k_pairs<<<grid(fo.touches), 256, 0, st>>>(tks, tvs, fo.touches, p.ibits, rt, d_res);
        ctx->launches += 2;
      }
    }
    NB_CUDA(cudaGetLastError());
    Result res{};
    NB_CUDA(cudaMemcpyAsync(&res, d_res, sizeof(res), cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaStreamSynchronize(st));
    out->pairs = int64_t(res.pairs);
    if (res.dup) {
      out->verdict = NB_ILLEGAL_DUPLICATE;
      return;
    }
    if (!same_size) {
      out->verdict = NB_NOT_APPLICABLE;
      return;
    }
    if (res.over_budget) fail(NB_ERR_UNSUPPORTED, "dependence scan above the kernel's budget");
    if (res.best == ~0ull) {
      out->verdict = NB_LEGAL;
      return;
    }
    const int64_t i = int64_t(res.best >> 32), j = int64_t(res.best & 0xffffffffull);
    uint64_t ki = 0, kj = 0;
    NB_CUDA(cudaMemcpyAsync(&ki, tks + i, 8, cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaMemcpyAsync(&kj, tks + j, 8, cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaStreamSynchronize(st));
    const uint64_t imask = (uint64_t(1) << p.ibits) - 1;
    const int64_t a = int64_t(ki & imask), b = int64_t(kj & imask);
    uint32_t ra = 0, rb = 0;
    NB_CUDA(cudaMemcpyAsync(&ra, rt + a, 4, cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaMemcpyAsync(&rb, rt + b, 4, cudaMemcpyDeviceToHost, st));
    k_describe<<<grid(fo.n), 256, 0, st>>>(d_so, int(fo.stmts.size()), fo.n, d_code, a, b, d_desc);
    ctx->launches++;
    Described desc{};
    NB_CUDA(cudaMemcpyAsync(&desc, d_desc, sizeof(desc), cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaGetLastError());
    NB_CUDA(cudaStreamSynchronize(st));
    if (ra == kMiss || rb == kMiss) {
      out->verdict = NB_NOT_APPLICABLE;
      return;
    }
    out->verdict = NB_ILLEGAL_REORDER;
    out->src_inst = a;
    out->dst_inst = b;
    out->src_stmt = desc.stmt[0];
    out->dst_stmt = desc.stmt[1];
    for (int k = 0; k < kLDom; ++k) {
      out->src_coord[k] = desc.coord[0][k];
      out->dst_coord[k] = desc.coord[1][k];
    }
  });
}

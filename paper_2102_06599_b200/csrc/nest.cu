// General loop-nest executor: execute<T> (I/interp.hpp:67-145) on the GPU
// for transformed nests with no ConvSpec (the paper's Sequence 1 and other
// non-channel groupings).  One thread per multiply-accumulate
// instance: the instance index is decoded into its loop values, the
// statement's coordinate programs give the original conv domain point, the
// access programs give the tensor cells, and the product is accumulated into
// the output (int64 exactly; fp64 by atomic add).
#include <vector>

#include "engine.hpp"
#include "nest_expr.cuh"

namespace nb {
namespace {

constexpr int kMaxDomain = 8, kMaxRank = 4, kMaxAcc = 4, kMaxDepth = 16;
using nexpr::kStack;
using nexpr::run;

struct DevAccess {
  int tensor, zero_pad, rank;
  int idx_off[kMaxRank];  // program offsets (in ops) into the code array
};

struct DevStmt {
  int depth;
  int64_t extents[kMaxDepth];
  int ndomain;
  int coord_off[kMaxDomain];
  int naccess;
  DevAccess acc[kMaxAcc];
};

template <typename T>
__global__ void k_nest_exec(DevStmt s, int64_t count, const int64_t* __restrict__ code,
                            const T* __restrict__ in, const T* __restrict__ w, T* __restrict__ out,
                            longlong4 shp_o, longlong4 shp_i, longlong4 shp_w, int* err) {
  for (int64_t inst = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; inst < count;
       inst += int64_t(gridDim.x) * blockDim.x) {
    int64_t loops[kMaxDepth];
    int64_t r = inst;
    for (int d = s.depth - 1; d >= 0; --d) {  // innermost loop varies fastest
      loops[d] = r % s.extents[d];
      r /= s.extents[d];
    }
    int64_t dom[kMaxDomain];
    for (int i = 0; i < s.ndomain; ++i) dom[i] = run(code, s.coord_off[i], loops);
    T prod = T(1);
    int64_t o_lin = -1;
    for (int a = 0; a < s.naccess; ++a) {
      const DevAccess& acc = s.acc[a];
      const long long* dims = acc.tensor == 0 ? &shp_o.x : acc.tensor == 1 ? &shp_i.x : &shp_w.x;
      int64_t lin = 0;
      bool inb = true;
      for (int k = 0; k < acc.rank; ++k) {
        const int64_t v = run(code, acc.idx_off[k], dom);
        if (v < 0 || v >= dims[k]) inb = false;
        lin = lin * dims[k] + v;
      }
      if (acc.tensor == 0) {
        if (!inb) atomicExch(err, 2);  // accumulate outside the output
        o_lin = inb ? lin : -1;
        continue;
      }
      if (!inb) {
        if (!acc.zero_pad) atomicExch(err, 1);  // read outside a tensor
        prod = T(0);
        continue;
      }
      prod *= (acc.tensor == 1 ? in : w)[lin];
    }
    if (o_lin < 0) continue;
    if constexpr (sizeof(T) == 8 && T(0.5) == T(0)) {
      atomicAdd(reinterpret_cast<unsigned long long*>(out + o_lin),
                static_cast<unsigned long long>(prod));  // two's complement: exact
    } else {
      atomicAdd(out + o_lin, prod);
    }
  }
}

// The masked box executor's cell pass: per output cell, the smallest and
// largest input channel (index 0 of the statement's "I" access) and the
// number of multiply-accumulate instances adding into it.
__global__ void k_nest_cells(DevStmt s, int64_t count, const int64_t* __restrict__ code,
                             longlong4 shp_o, longlong4 shp_i, longlong4 shp_w, int* ci_lo,
                             int* ci_hi, unsigned long long* cnt) {
  for (int64_t inst = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; inst < count;
       inst += int64_t(gridDim.x) * blockDim.x) {
    int64_t loops[kMaxDepth];
    int64_t r = inst;
    for (int d = s.depth - 1; d >= 0; --d) {
      loops[d] = r % s.extents[d];
      r /= s.extents[d];
    }
    int64_t dom[kMaxDomain];
    for (int i = 0; i < s.ndomain; ++i) dom[i] = run(code, s.coord_off[i], loops);
    int64_t o_lin = -1, ci = -1;
    for (int a = 0; a < s.naccess; ++a) {
      const DevAccess& acc = s.acc[a];
      if (acc.tensor == 2) continue;
      const long long* dims = acc.tensor == 0 ? &shp_o.x : &shp_i.x;
      if (acc.tensor == 1) {
        ci = run(code, acc.idx_off[0], dom);
        continue;
      }
      int64_t lin = 0;
      bool inb = true;
      for (int k = 0; k < acc.rank; ++k) {
        const int64_t v = run(code, acc.idx_off[k], dom);
        if (v < 0 || v >= dims[k]) inb = false;
        lin = lin * dims[k] + v;
      }
      o_lin = inb ? lin : -1;
    }
    if (o_lin < 0) continue;
    atomicMin(ci_lo + o_lin, int(ci));
    atomicMax(ci_hi + o_lin, int(ci));
    atomicAdd(cnt + o_lin, 1ull);
  }
}

int64_t numel(const int64_t* d, int rank) {
  int64_t n = 1;
  for (int i = 0; i < rank; ++i) n *= d[i];
  return n;
}

// The nest's statements as device descriptors over one flattened code
// array of postfix programs (each program starts with a (nops, 0) header).
void compile(const nb_nest* nest, std::vector<int64_t>& code, std::vector<DevStmt>& stmts,
             std::vector<int64_t>& counts) {
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
      if (depth != 1 || maxd > kStack) fail(NB_ERR_UNSUPPORTED, "nest expression too deep");
      return off;
    };
    for (int64_t i = 0; i < nest->num_stmts; ++i) {
      const nb_nest_stmt& src = nest->stmts[i];
      if (src.depth > kMaxDepth || src.ndomain > kMaxDomain || src.naccess > kMaxAcc)
        fail(NB_ERR_UNSUPPORTED, "nest statement exceeds the executor's limits");
      DevStmt d{};
      d.depth = src.depth;
      int64_t cnt = 1;
      for (int k = 0; k < src.depth; ++k) {
        d.extents[k] = src.extents[k];
        cnt *= src.extents[k];
      }
      d.ndomain = src.ndomain;
      for (int k = 0; k < src.ndomain; ++k) d.coord_off[k] = add(src.coord[k]);
      d.naccess = src.naccess;
      int writes = 0;
      for (int a = 0; a < src.naccess; ++a) {
        const nb_nest_access& sa = src.access[a];
        if (sa.rank > kMaxRank) fail(NB_ERR_UNSUPPORTED, "access rank above 4");
        const int want = sa.tensor == 0 ? nest->out_rank : sa.tensor == 1 ? nest->in_rank
                                                                          : nest->w_rank;
        if (sa.rank != want) fail(NB_ERR_SHAPE_MISMATCH, "access arity does not match tensor rank");
        writes += sa.tensor == 0;
        d.acc[a].tensor = sa.tensor;
        d.acc[a].zero_pad = sa.zero_pad;
        d.acc[a].rank = sa.rank;
        for (int k = 0; k < sa.rank; ++k) d.acc[a].idx_off[k] = add(sa.idx[k]);
      }
      if (writes != 1) fail(NB_ERR_GENERIC, "multiply-accumulate statement lacks an RMW access");
      stmts.push_back(d);
      counts.push_back(cnt);
    }
}

}  // namespace
}  // namespace nb

using namespace nb;

extern "C" nb_status nb_nest_execute(nb_ctx* ctx, const nb_nest* nest, int32_t is_int,
                                     const void* in, const void* w, void* out) {
  return guard([&] {
    Range range("nb_nest_execute");
    if (!ctx || !nest || !in || !w || !out) fail(NB_ERR_CONFIG, "null argument");
    if (nest->out_rank > kMaxRank || nest->in_rank > kMaxRank || nest->w_rank > kMaxRank)
      fail(NB_ERR_UNSUPPORTED, "tensor rank above 4");
    std::vector<int64_t> code;
    std::vector<DevStmt> stmts;
    std::vector<int64_t> counts;
    compile(nest, code, stmts, counts);
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ctx_activate(ctx);
    cudaStream_t st = ctx->stream;
    const int64_t no = numel(nest->out_shape, nest->out_rank),
                  ni = numel(nest->in_shape, nest->in_rank),
                  nw = numel(nest->w_shape, nest->w_rank);
    // io: [code | err | out | in | w], 8-byte elements
    const size_t code_b = (code.size() * 8 + 255) & ~size_t(255);
    ctx->io.ensure(code_b + 256 + size_t(no + ni + nw) * 8);
    char* base = static_cast<char*>(ctx->io.p);
    int64_t* d_code = reinterpret_cast<int64_t*>(base);
    int* d_err = reinterpret_cast<int*>(base + code_b);
    char* d_out = base + code_b + 256;
    char* d_in = d_out + no * 8;
    char* d_w = d_in + ni * 8;
    NB_CUDA(cudaMemcpyAsync(d_code, code.data(), code.size() * 8, cudaMemcpyHostToDevice, st));
    NB_CUDA(cudaMemsetAsync(d_err, 0, 4, st));
    NB_CUDA(cudaMemsetAsync(d_out, 0, size_t(no) * 8, st));
    NB_CUDA(cudaMemcpyAsync(d_in, in, size_t(ni) * 8, cudaMemcpyHostToDevice, st));
    NB_CUDA(cudaMemcpyAsync(d_w, w, size_t(nw) * 8, cudaMemcpyHostToDevice, st));
    auto shp = [](const int64_t* d) { return make_longlong4(d[0], d[1], d[2], d[3]); };
    for (size_t i = 0; i < stmts.size(); ++i) {
      if (counts[i] == 0) continue;
      const int64_t blocks = std::min<int64_t>((counts[i] + 255) / 256, int64_t(ctx->num_sms) * 64);
      if (is_int)
        k_nest_exec<long long><<<unsigned(blocks), 256, 0, st>>>(
            stmts[i], counts[i], d_code, reinterpret_cast<const long long*>(d_in),
            reinterpret_cast<const long long*>(d_w), reinterpret_cast<long long*>(d_out),
            shp(nest->out_shape), shp(nest->in_shape), shp(nest->w_shape), d_err);
      else
        k_nest_exec<double><<<unsigned(blocks), 256, 0, st>>>(
            stmts[i], counts[i], d_code, reinterpret_cast<const double*>(d_in),
            reinterpret_cast<const double*>(d_w), reinterpret_cast<double*>(d_out),
            shp(nest->out_shape), shp(nest->in_shape), shp(nest->w_shape), d_err);
      ctx->launches++;
    }
    int err = 0;
    NB_CUDA(cudaMemcpyAsync(&err, d_err, 4, cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaMemcpyAsync(out, d_out, size_t(no) * 8, cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaGetLastError());
    NB_CUDA(cudaStreamSynchronize(st));
    if (err == 1) fail(NB_ERR_GENERIC, "read outside a tensor");  // IndexOutOfRange
    if (err == 2) fail(NB_ERR_GENERIC, "accumulate outside the output");
  });
}

extern "C" nb_status nb_nest_cells(nb_ctx* ctx, const nb_nest* nest, int32_t* ci_lo,
                                   int32_t* ci_hi, int64_t* count) {
  return guard([&] {
    Range range("nb_nest_cells");
    if (!ctx || !nest || !ci_lo || !ci_hi || !count) fail(NB_ERR_CONFIG, "null argument");
    if (nest->out_rank > kMaxRank || nest->in_rank > kMaxRank || nest->w_rank > kMaxRank)
      fail(NB_ERR_UNSUPPORTED, "tensor rank above 4");
    std::vector<int64_t> code;
    std::vector<DevStmt> stmts;
    std::vector<int64_t> counts;
    compile(nest, code, stmts, counts);
    std::lock_guard<std::recursive_mutex> lk(ctx->mu);
    ctx_activate(ctx);
    cudaStream_t st = ctx->stream;
    const int64_t no = numel(nest->out_shape, nest->out_rank);
    // io: [code | ci_lo | ci_hi | count]
    const size_t code_b = (code.size() * 8 + 255) & ~size_t(255);
    const size_t cell_b = (size_t(no) * 4 + 255) & ~size_t(255);
    ctx->io.ensure(code_b + 2 * cell_b + size_t(no) * 8);
    char* base = static_cast<char*>(ctx->io.p);
    int64_t* d_code = reinterpret_cast<int64_t*>(base);
    int* d_lo = reinterpret_cast<int*>(base + code_b);
    int* d_hi = reinterpret_cast<int*>(base + code_b + cell_b);
    auto* d_cnt = reinterpret_cast<unsigned long long*>(base + code_b + 2 * cell_b);
    NB_CUDA(cudaMemcpyAsync(d_code, code.data(), code.size() * 8, cudaMemcpyHostToDevice, st));
    NB_CUDA(cudaMemsetAsync(d_lo, 0x7f, size_t(no) * 4, st));  // ~INT_MAX
    NB_CUDA(cudaMemsetAsync(d_hi, 0xff, size_t(no) * 4, st));  // -1
    NB_CUDA(cudaMemsetAsync(d_cnt, 0, size_t(no) * 8, st));
    auto shp = [](const int64_t* d) { return make_longlong4(d[0], d[1], d[2], d[3]); };
    for (size_t i = 0; i < stmts.size(); ++i) {
      if (counts[i] == 0) continue;
      const int64_t blocks = std::min<int64_t>((counts[i] + 255) / 256, int64_t(ctx->num_sms) * 64);
      k_nest_cells<<<unsigned(blocks), 256, 0, st>>>(stmts[i], counts[i], d_code,
                                                     shp(nest->out_shape), shp(nest->in_shape),
                                                     shp(nest->w_shape), d_lo, d_hi, d_cnt);
      ctx->launches++;
    }
    NB_CUDA(cudaMemcpyAsync(ci_lo, d_lo, size_t(no) * 4, cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaMemcpyAsync(ci_hi, d_hi, size_t(no) * 4, cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaMemcpyAsync(count, d_cnt, size_t(no) * 8, cudaMemcpyDeviceToHost, st));
    NB_CUDA(cudaGetLastError());
    NB_CUDA(cudaStreamSynchronize(st));
  });
}

/*
 * nb200 -- C ABI of the B200-native hot path of arXiv 2102.06599
 * ("NAS as program transformation exploration", reference library `nestopt`).
 *
 * The reference exposes no FFI: its operator API is the header-only C++
 * namespace `nestopt` (/root/reference/proj/include/nestopt).  This header is
 * the drop-in boundary a maintainer binds from that C++ host (see
 * INTEGRATION.md and integration/nestopt_b200.hpp): every entry point below
 * replaces one reference function, cited as I/<file>:<line> where
 * I/ = proj/include/nestopt/.
 *
 * Conventions (mirroring the reference's):
 *  - plain C types only; host buffers are caller-owned, fp64 and in the
 *    reference's layouts (per image (C,H,W) row-major, weights
 *    (Co_eff,Ci,Kh,Kw), head [num_classes][C_last]); they are never retained
 *    after a call returns.  Device memory is owned by the context.
 *  - errors: every call returns an nb_status whose values map 1:1 onto the
 *    nestopt exception classes (I/errors.hpp); nb_last_error() returns the
 *    message of the last failing call on the calling thread.
 *  - threading: calls on one context are serialized internally; different
 *    contexts (one per GPU) run concurrently.
 *  - there is no CPU fallback: without a usable CUDA device every compute
 *    entry point fails with NB_ERR_NO_DEVICE.
 */
#ifndef NB200_H
#define NB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NB200_ABI_VERSION 2

typedef enum nb_status {
  NB_OK = 0,
  NB_ERR_INVALID_SPEC = 1,    /* nestopt::InvalidSpec   I/errors.hpp:11 */
  NB_ERR_CONFIG = 2,          /* nestopt::ConfigError   I/errors.hpp:64 */
  NB_ERR_SHAPE_MISMATCH = 3,  /* nestopt::ShapeMismatch I/errors.hpp:60 */
  NB_ERR_CAP_EXCEEDED = 4,    /* nestopt::CapExceeded   I/errors.hpp:17 (host gate only) */
  NB_ERR_TRANSFORM = 5,       /* nestopt::TransformError I/errors.hpp:22 */
  NB_ERR_PARSE = 6,           /* nestopt::ParseError    I/errors.hpp:46 */
  NB_ERR_IO = 7,              /* nestopt::IoError       I/errors.hpp:67 */
  NB_ERR_GENERIC = 8,         /* nestopt::Error         I/errors.hpp:8  */
  NB_ERR_CUDA = 100,          /* CUDA runtime / launch failure */
  NB_ERR_NO_DEVICE = 101,     /* no usable sm_100 device: no CPU fallback exists */
  NB_ERR_OUT_OF_MEMORY = 102,
  NB_ERR_UNSUPPORTED = 103,
  NB_ERR_INTERNAL = 199
} nb_status;

/* Arithmetic mode of the conv kernels.  Head, softmax and the Fisher
 * reduction always run in fp64. */
typedef enum nb_precision {
  NB_PREC_FP32 = 0, /* fp32-accurate (default, used for legality decisions):
                       3xTF32 tcgen05 implicit GEMM for tensor-core-shaped
                       ranges, fp32 FFMA for the rest */
  NB_PREC_TF32 = 1, /* 1xTF32 tcgen05 throughput mode (looser tolerance) */
  NB_PREC_SIMT = 2  /* fp32 FFMA kernels only (parity baseline) */
} nb_precision;

/* ChannelSplit, I/ir.hpp:20-24 */
typedef struct nb_channel_split {
  int64_t begin, end, groups;
} nb_channel_split;

/* ConvSpec, I/ir.hpp:26-87 (field for field). */
typedef struct nb_conv_spec {
  int64_t ci, co, h, w, kh, kw, stride, pad, groups, bottleneck_out,
      spatial_div_h, spatial_div_w;
  int64_t num_splits;             /* 0 = single range {0, co_eff, groups} */
  const nb_channel_split* splits; /* num_splits entries */
} nb_conv_spec;

/* Layer, I/nnet.hpp:23-26 */
typedef struct nb_layer {
  nb_conv_spec spec;
  int32_t relu;
  int32_t reserved;
} nb_layer;

/* Network, I/nnet.hpp:28-79, without its weight tensors: weights are either
 * drawn exactly as Network::init_weights does (I/nnet.hpp:58-79, from
 * `seed`), or passed explicitly through nb_weights. */
typedef struct nb_network {
  int64_t num_layers;
  const nb_layer* layers;
  int64_t num_classes;
  uint64_t seed;
} nb_network;

/* Explicit Network::weights / Network::head.  NULL (or NULL members) =
 * init_weights(seed). */
typedef struct nb_weights {
  const double* const* layer; /* num_layers pointers, (Co_eff,Ci,Kh,Kw) each */
  const double* head;         /* [num_classes][C_last] */
} nb_weights;

/* Batch, I/nnet.hpp:81-85.  inputs == NULL => make_batch(net, n, seed)
 * (I/nnet.hpp:87-101), drawn bit-identically on the host. */
typedef struct nb_batch {
  int64_t n;
  const double* inputs;  /* n x (Ci,H,W) of layer 0, or NULL */
  const int32_t* labels; /* n, or NULL when inputs == NULL */
  uint64_t seed;
} nb_batch;

/* FisherReport, I/nnet.hpp:272-277, plus the forward loss. */
typedef struct nb_fisher_out {
  double* per_channel; /* sum_l Co_eff(l) doubles (layer-major), or NULL */
  double* per_layer;   /* num_layers doubles, or NULL */
  double total;
  uint64_t seed;       /* batch seed the scores were computed under */
  double loss;         /* mean cross-entropy of the forward pass */
  double* probs;       /* n x num_classes softmax, or NULL */
} nb_fisher_out;

typedef struct nb_ctx nb_ctx;         /* one per GPU: stream, arena, caches */
typedef struct nb_session nb_session; /* a context + one HBM-resident batch */

/* Per-kernel-family device time, recorded with CUDA events on the launching
 * stream while profiling is enabled (nb_ctx_set_profiling). */
typedef struct nb_kernel_stat {
  char name[48];
  int64_t launches;
  double ms;          /* summed event time */
  double flops;       /* algorithmic FLOPs (2 x count_macs-style MACs) */
  double bytes;       /* algorithmic HBM bytes (read once + write once) */
} nb_kernel_stat;

/* Scheduler statistics of one nb_evaluate call.  The per-session arrays are
 * caller-owned (num_sessions entries each) and may be NULL. */
typedef struct nb_eval_stats {
  int64_t evaluated;       /* distinct networks run on a device */
  int64_t deduplicated;    /* candidates answered from an identical network */
  int64_t requeued;        /* evaluations handed back after a device failure */
  int32_t failed_sessions; /* sessions retired by a device failure */
  int32_t reserved;
  double* est_flops;       /* per session: estimated FLOPs of what it ran */
  double* busy_ms;         /* per session: device time of its evaluations */
  int64_t* evaluations;    /* per session: networks it evaluated */
} nb_eval_stats;

/* ---- library ---------------------------------------------------------- */
const char* nb_version(void);
int nb_abi_version(void);
int nb_device_count(void);
const char* nb_last_error(void);

/* ---- host-side descriptors (no device needed) ------------------------- */
/* ConvSpec::validate, I/ir.hpp:59-86 */
nb_status nb_validate_spec(const nb_conv_spec* spec);
/* Network::validate, I/nnet.hpp:40-55 */
nb_status nb_validate_network(const nb_network* net);
/* count_macs(conv_nest(spec)), I/interp.hpp:190-202 + I/ir.hpp:427 */
nb_status nb_conv_macs(const nb_conv_spec* spec, int64_t* macs);
/* network_macs, I/search.hpp:84-88 */
nb_status nb_network_macs(const nb_network* net, int64_t* macs);
/* repair_network shape propagation, I/nnet.hpp:372-382 (in place on a
 * caller-owned layer array; weights are redrawn lazily on the device). */
nb_status nb_repair_network(int64_t num_layers, nb_layer* layers);
/* Longest-processing-time-first assignment of `count` jobs of estimated
 * cost to `bins` workers (ties broken by index); deterministic. */
nb_status nb_schedule_lpt(const double* cost, int64_t count, int32_t bins,
                          int32_t* assignment);
/* Estimated FLOPs of one Fisher evaluation: 2*N*(fprop MACs + dgrad MACs). */
nb_status nb_fisher_flops(const nb_network* net, int64_t n, double* flops);
/* Network::init_weights, I/nnet.hpp:58-79 (host, bit-identical draws):
 * weights = concatenation of the per-layer (Co_eff,Ci,Kh,Kw) tensors. */
nb_status nb_init_weights(const nb_network* net, double* weights, double* head);
/* make_batch, I/nnet.hpp:87-101 (host, bit-identical draws). */
nb_status nb_make_batch(const nb_network* net, int64_t n, uint64_t seed,
                        double* inputs, int32_t* labels);

/* ---- contexts ------------------------------------------------------------ */
nb_status nb_ctx_create(int device, nb_ctx** out);
/* CUDA device ordinal of a context (-1 for NULL). */
int nb_ctx_device(const nb_ctx* ctx);
nb_status nb_ctx_destroy(nb_ctx* ctx);
/* The CUDA stream (cudaStream_t) all of the context's kernels run on. */
void* nb_ctx_stream(nb_ctx* ctx);
/* enable = 0: off; k >= 1: CUDA events around every launch of every k-th
 * evaluation (sampling keeps the event overhead out of long runs). */
nb_status nb_ctx_set_profiling(nb_ctx* ctx, int enable);
/* Copies up to `cap` stats, returns the number of families in *count. */
nb_status nb_ctx_kernel_stats(nb_ctx* ctx, nb_kernel_stat* stats, int32_t cap,
                              int32_t* count);
nb_status nb_ctx_reset_stats(nb_ctx* ctx);
/* Drops the context's packed-weight and z-stream caches (device memory). */
nb_status nb_ctx_clear_caches(nb_ctx* ctx);
/* Number of nb200 kernel launches issued by this context so far. */
int64_t nb_ctx_launch_count(nb_ctx* ctx);

/* ---- single conv layer (reference_conv / layer_forward) ------------------ */
/* reference_conv<double> (I/interp.hpp:151-186) / layer_forward
 * (I/nnet.hpp:130-141) over n images: x n x (Ci,H,W), w (Co_eff,Ci,Kh,Kw),
 * y n x (Co_eff,out_h,out_w); relu != 0 applies the layer's ReLU. */
nb_status nb_conv_forward(nb_ctx* ctx, const nb_conv_spec* spec, int64_t n,
                          const double* x, const double* w, double* y,
                          int32_t relu, nb_precision prec);
/* The dgrad step of activation_gradients (I/nnet.hpp:235-243): dx n x
 * (Ci,H,W) = sum over for_each_conv_mac of W * dy, dy n x (Co_eff,oh,ow). */
nb_status nb_conv_dgrad(nb_ctx* ctx, const nb_conv_spec* spec, int64_t n,
                        const double* dy, const double* w, double* dx,
                        nb_precision prec);
/* reference_conv restricted to the output rows [oh_lo, oh_hi) (the other
 * rows of y are left undefined): one box of the masked box executor of
 * nests with no ConvSpec (integration/nestopt_b200.hpp execute_boxes), the
 * tensor-core tiles covering only the band.  No ReLU. */
nb_status nb_conv_band(nb_ctx* ctx, const nb_conv_spec* spec, int64_t n, const double* x,
                       const double* w, int32_t oh_lo, int32_t oh_hi, double* y,
                       nb_precision prec);

/* ---- general loop nests (execute, I/interp.hpp:67-145) -------------------- */
/* A transformed conv loop nest in executable form, for nests with no
 * ConvSpec (derived_spec == nullopt, e.g. the paper's Sequence 1,
 * I/transforms.hpp:531-550).  Built from the reference's LoopNest by the
 * bridge (integration/nestopt_b200.hpp nb200::execute): one entry per
 * multiply-accumulate statement of each block of compute_blocks
 * (I/ir.hpp:163-218); Init statements are not passed (the output starts at
 * zero, as execute's provenance-allocated tensor does).
 * Expressions are postfix programs of (op, arg) int64 pairs:
 *   0 const arg | 1 slot arg | 2 add the top arg values | 3 mul by arg |
 *   4 floor-div by arg | 5 floor-mod by arg   (AffineExpr, I/affine.hpp:17-111)
 */
typedef struct nb_nest_expr {
  int32_t nops;
  const int64_t* code; /* 2 * nops */
} nb_nest_expr;

typedef struct nb_nest_access {
  int32_t tensor;   /* 0 = the written tensor O (read-modify-write), 1 = I, 2 = K */
  int32_t zero_pad; /* out-of-range reads yield zero (else an error) */
  int32_t rank;
  const nb_nest_expr* idx; /* rank expressions over the statement's domain values */
} nb_nest_access;

typedef struct nb_nest_stmt {
  int32_t depth;           /* loops enclosing the statement */
  const int64_t* extents;  /* depth trip counts, outermost first */
  int32_t ndomain;
  const nb_nest_expr* coord; /* ndomain expressions over the loop values */
  int32_t naccess;
  const nb_nest_access* access;
} nb_nest_stmt;

typedef struct nb_nest {
  int64_t num_stmts;
  const nb_nest_stmt* stmts;
  int64_t out_shape[4], in_shape[4], w_shape[4]; /* unused trailing dims = 1 */
  int32_t out_rank, in_rank, w_rank;
} nb_nest;

/* execute<T> (I/interp.hpp:67-145) on the GPU: every MAC instance of the
 * nest adds prod(reads) into the output cell it addresses (int64 exactly,
 * or fp64).  is_int != 0: in/w/out are int64, else double. */
nb_status nb_nest_execute(nb_ctx* ctx, const nb_nest* nest, int32_t is_int, const void* in,
                          const void* w, void* out);
/* The masked box executor's cell pass over the same nest: per output cell
 * (out_shape order), the smallest / largest input channel (index 0 of the
 * statement's "I" access; INT32_MAX-ish / -1 when nothing adds into it) and
 * the number of multiply-accumulate instances that add into it. */
nb_status nb_nest_cells(nb_ctx* ctx, const nb_nest* nest, int32_t* ci_lo, int32_t* ci_hi,
                        int64_t* count);

/* ---- semantic legality (check_semantic_legality, I/transforms.hpp:598-663) */
/* The brute-force dependence-preservation check of a semantic run (split /
 * interchange / unroll steps) on the GPU.  Both nests are passed as
 * statement entries of their compute_blocks (I/ir.hpp:163-218), Init
 * statements included, in block order:
 *  - schedule rank of an instance (its index in for_each_instance order,
 *    I/ir.hpp:262-300) = rank_base + sum_k v_k * rank_stride[k];
 *  - sid interns Statement::id across both nests (instance identity is the
 *    (sid, domain coordinate) pair); gid is compute_dependences' per-nest
 *    interning (I/ir.hpp:343-346) and only matters for the original;
 *  - accesses (original only; transformed entries pass naccess = 0) are the
 *    ones to tensors some statement of the original writes, tensor ids in
 *    the reference's interning order -- touches of read-only tensors can
 *    never form a dependence pair.
 * lo/hi bound every domain value / cell index (any superset box is fine;
 * the bridge uses interval arithmetic over the affine programs).  Instance
 * caps (CapExceeded) stay with the caller; NB_ERR_UNSUPPORTED means the keys
 * do not fit 64 bits and the caller must run the host check. */
typedef struct nb_legal_access {
  int32_t tensor;
  int32_t mode; /* 0 Read, 1 Write, 2 ReadModifyWrite (AccessMode) */
  int32_t rank;
  const nb_nest_expr* idx; /* over the statement's domain values */
  const int64_t* lo;       /* rank bounds of each index */
  const int64_t* hi;
} nb_legal_access;

typedef struct nb_legal_stmt {
  int32_t sid, gid;
  int32_t depth;
  const int64_t* extents;     /* depth trip counts, outermost first */
  int64_t rank_base;
  const int64_t* rank_stride; /* depth entries */
  int32_t ndomain;
  const nb_nest_expr* coord;  /* ndomain expressions over the loop values */
  const int64_t* lo;          /* ndomain bounds of each coordinate */
  const int64_t* hi;
  int32_t naccess;
  const nb_legal_access* access;
} nb_legal_stmt;

typedef struct nb_legal_nest {
  int64_t num_stmts;
  const nb_legal_stmt* stmts;
} nb_legal_nest;

typedef enum nb_legal_verdict {
  NB_LEGAL = 0,
  NB_ILLEGAL_DUPLICATE = 1, /* "transformed schedule duplicates an instance" */
  NB_NOT_APPLICABLE = 2,    /* "instance sets differ (...)" */
  NB_ILLEGAL_REORDER = 3    /* "dependence S(..) -> S(..) is reordered" */
} nb_legal_verdict;

typedef struct nb_legal_out {
  int32_t verdict;
  /* NB_ILLEGAL_REORDER: the first reordered pair in the reference's order,
   * as original-schedule instance indices, entries of original->stmts and
   * domain coordinates */
  int64_t src_inst, dst_inst;
  int32_t src_stmt, dst_stmt;
  int64_t src_coord[8], dst_coord[8];
  int64_t pairs; /* dependence pairs checked (reduction pairs excluded) */
} nb_legal_out;

nb_status nb_semantic_legality(nb_ctx* ctx, const nb_legal_nest* original,
                               const nb_legal_nest* transformed, nb_legal_out* out);

/* ---- network-level entry points ----------------------------------------- */
/* forward, I/nnet.hpp:180-197: probs n x classes, example_loss n, loss. */
nb_status nb_forward(nb_ctx* ctx, const nb_network* net, const nb_weights* w,
                     const nb_batch* batch, nb_precision prec, double* probs,
                     double* example_loss, double* loss);
/* forward + activation_gradients, I/nnet.hpp:180-247: acts/grads laid out
 * for l in [0,L): for n: (C,H,W) of layer l's post-activation output. */
nb_status nb_activation_gradients(nb_ctx* ctx, const nb_network* net,
                                  const nb_weights* w, const nb_batch* batch,
                                  nb_precision prec, double* acts,
                                  double* grads);
/* fisher_potential, I/nnet.hpp:321-352. */
nb_status nb_fisher_potential(nb_ctx* ctx, const nb_network* net,
                              const nb_weights* w, const nb_batch* batch,
                              nb_precision prec, nb_fisher_out* out);
/* fisher_accepts, I/nnet.hpp:356-359 (candidate.total >= original.total). */
int nb_fisher_accepts(const nb_fisher_out* original,
                      const nb_fisher_out* candidate);

/* ---- sessions: a batch kept resident in HBM ------------------------------ */
nb_status nb_session_create(nb_ctx* ctx, const nb_network* shape_net,
                            const nb_batch* batch, nb_session** out);
nb_status nb_session_destroy(nb_session* s);
nb_ctx* nb_session_ctx(nb_session* s);
nb_status nb_session_fisher(nb_session* s, const nb_network* net,
                            const nb_weights* w, nb_precision prec,
                            nb_fisher_out* out);
/* fisher_potential (I/nnet.hpp:321-350) of one network with the batch split
 * into example shards (the secondary axis for fewer networks
 * than GPUs): shards[i] holds examples [n_0+..+n_{i-1}, +n_i) of one batch,
 * normally one session per GPU, each on its own context.  Every shard
 * divides dz by the whole batch's N and plans its launches for it; the
 * per-example sums s_nc are gathered into shards[0]'s GPU (peer copies) and
 * reduced there in the unsharded kernel's fixed order, so the report
 * (per_channel, per_layer, total, loss, probs) is bitwise that of one
 * session holding the whole batch.  NB_ERR_CONFIG for repeated contexts or
 * shards of different batch seeds. */
nb_status nb_fisher_sharded(nb_session* const* shards, int32_t count,
                            const nb_network* net, const nb_weights* w,
                            nb_precision prec, nb_fisher_out* out);
/* forward only (transformed-net inference): probs n x classes, loss. */
nb_status nb_session_forward(nb_session* s, const nb_network* net,
                             const nb_weights* w, nb_precision prec,
                             double* probs, double* loss);

/* ---- candidate scheduler (evaluate_all, I/search.hpp:315-334) ------------ */
/* Scores `count` candidate networks (all drawn with init_weights) on the
 * given sessions -- each on its own context (normally one or a few per GPU),
 * all holding the same batch (NB_ERR_CONFIG otherwise).  Identical networks
 * are evaluated once; the rest form one queue in longest-processing-time
 * order (nb_fisher_flops) that every session pulls from as soon as its
 * previous evaluation completes (the reference's self-scheduling,
 * next.fetch_add(1)), one host worker thread per GPU.  A session that hits
 * a device error is retired and its candidate re-queued for the others; the
 * call fails only when no session is left.  Results land in outs[i]
 * regardless of which session ran them, so the output is independent of the
 * number of sessions and GPUs (the reference's jobs=k == jobs=1 guarantee,
 * T/test_search.cpp:83-94). */
nb_status nb_evaluate(nb_session* const* sessions, int32_t num_sessions,
                      const nb_network* nets, int64_t count, nb_precision prec,
                      nb_fisher_out* outs, nb_eval_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* NB200_H */

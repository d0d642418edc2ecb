// bt_reduce.cuh -- argument block of the deterministic gradient reducer (C-ABI visible).
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BT_MAX_TABLE 64 /* per-EST pointer table entries (peer or local slots) */
#define BT_MAX_REPLICA_OUT 8

enum { BT_DTYPE_F64 = 0, BT_DTYPE_F32 = 1 };
enum { BT_REDUCE_UPDATE = 0, BT_REDUCE_MEAN_ONLY = 1, BT_REDUCE_SUM_ONLY = 2, BT_REDUCE_ADAM = 3,
       BT_REDUCE_MEAN_CHECK = 4, /* MEAN_ONLY + the non-finite flag (pass 1 of a guarded update) */
       BT_REDUCE_APPLY_SGD = 5,  /* pass 2 alone: momentum SGD from `stage`, gated (multi-rank guard) */
       BT_REDUCE_APPLY_ADAM = 6  /* pass 2 alone: Adam from `stage`, gated */ };

/* out[p] = reduce_sum(g[(rot[p]+k) % E][p] for k in 0..E-1, fanin) / E   (buckets.py:115-123)
 * then, in BT_REDUCE_UPDATE mode, v' = mu*v + out; p' = p - lr*v'      (model.py:206-212);
 * in BT_REDUCE_ADAM mode (the north star's "or Adam"): m' = mu*m + (1-mu)*out (m = vel),
 * s' = beta2*s + (1-beta2)*out*out (s = vel2), p' = p - lr*(m'*bc1) / (sqrt(s'*bc2) + eps), with the
 * bias corrections bc1 = 1/(1-mu^t), bc2 = 1/(1-beta2^t) supplied by the caller.
 * BT_REDUCE_SUM_ONLY writes the raw fold (no division): the per-GPU subtree of
 * the hierarchical RankTree(2) path, whose top level is then folded over the G
 * partials in rank order with divisor = E.
 * Contributions are addressed by EST rank k: either a table of E base pointers
 * (each may be a local slot or a peer GPU's slot mapped by CUDA IPC) or one
 * strided buffer (grads_ld > 0: base grads[0], EST k at grads[0] + k*grads_ld
 * elements).  The order of every addition depends only on (E, fanin, rot):
 * never on the GPU, CTA or thread count. */
typedef struct bt_reduce_args {
  int32_t dtype;  /* BT_DTYPE_F64 | BT_DTYPE_F32 */
  int32_t mode;   /* BT_REDUCE_UPDATE | BT_REDUCE_MEAN_ONLY */
  int32_t E;      /* contributions per element (EST count) */
  int32_t fanin;  /* 0 = Sequential, >= 2 = Tree(fanin) */
  int32_t nout;   /* extra replica outputs (P2P stores = fused parameter all-gather) */
  int32_t divisor;   /* 0: divide by E; > 0: divide by this (hierarchical top level: the job's E) */
  int64_t n;         /* elements in this shard */
  int64_t grads_ld;  /* > 0: strided mode */
  const void *grads[BT_MAX_TABLE];
  const int32_t *rot; /* [n] rotation start (Tree parity with the bucket map) or NULL */
  const void *param, *vel;       /* inputs (unused in MEAN_ONLY) */
  void *param_out, *vel_out;     /* outputs; may alias the inputs */
  void *extra_param_out[BT_MAX_REPLICA_OUT];
  void *extra_vel_out[BT_MAX_REPLICA_OUT];
  double lr, mu;
  int32_t *flags; /* [4] device status; NUMERIC + first bad index */
  /* BT_REDUCE_ADAM only (appended: earlier fields keep their offsets) */
  const void *vel2;   /* second-moment input */
  void *vel2_out;     /* second-moment output; may alias vel2 */
  void *extra_vel2_out[BT_MAX_REPLICA_OUT];
  double beta2, eps, bc1, bc2;
  /* Guarded update (UPDATE / ADAM): when `stage` [n] is non-NULL nothing is written unless every
   * synchronized gradient of the update is finite -- the reference's sgd_step raises before it
   * mutates anything (model.py:207-209).  Pass 1 folds, divides and checks into `stage`; pass 2
   * applies the update only if flags[0] == 0 and every gate[i] (i < ngate) is 0 (gate: the
   * status words other ranks published for their shards of the same update; NULL when the whole
   * update is local).  A gated-off pass 2 marks flags NUMERIC so every rank raises. */
  void *stage;
  const int32_t *gate;
  int32_t ngate;
  int32_t pad_;
} bt_reduce_args;

#ifdef __cplusplus
}
#endif

// bt_mlp.cuh -- argument block of the fused MLP step kernel (C-ABI visible).
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

// Model shape pinned by the reference (model.py:27-34).
#define BT_INPUT_DIM 8
#define BT_HIDDEN 16
#define BT_W1 0
#define BT_B1 (BT_INPUT_DIM * BT_HIDDEN)
#define BT_W2 (BT_B1 + BT_HIDDEN)
#define BT_B2 (BT_W2 + BT_HIDDEN)
#define BT_P (BT_B2 + 1) /* 161 */
#define BT_ROW (BT_INPUT_DIM + 1) /* dataset row: 8 x-values then y (sampling.py:24-35) */
#define BT_MAX_XDEV 8 /* devices of one multi-device exchange group */
#define BT_XSP 162    /* inbox slot stride in doubles (161 rounded to 16 bytes) */

/* One launch runs K consecutive mini-batches of the data-parallel step
 * (engine.py:271-329) for the ESTs [est_base, est_base+E) of an E_total-EST job.
 * All pointers are caller-owned DEVICE memory. */
typedef struct bt_mlp_args {
  int32_t E;           /* ESTs handled by this launch */
  int32_t est_base;    /* global virtual rank of local EST 0 */
  int32_t E_total;     /* ESTs in the job (allreduce divisor, rotation, row deal) */
  int32_t B;           /* micro-batch rows per EST */
  int32_t X;           /* executor replicas held here (replica agreement check) */
  int32_t K;           /* mini-batches in this launch */
  int32_t fuse_reduce; /* 1: allreduce + sgd in-kernel (E must equal E_total); 0: grads only */
  int32_t est_per_cta; /* ESTs per CTA (grid = ceil(E / est_per_cta)) */
  int32_t comm_fanin;  /* executor 0's variant for the allreduce (engine.py:309); 0 = Sequential */
  int32_t est_fanin_uniform; /* 0: per-EST est_fanin only; f+1: every est_fanin[] is f (a hint that lets
                                the launcher pick a specialised kernel; a wrong hint is reported as InputError) */
  int64_t rank_override; /* >= 0: TrackedStat rank of EST 0 (pure forward_backward seam) */
  double rate, lr, mu, jitter;
  /* state */
  double *replicas;        /* [X][2][P]: params then velocity, one block per executor */
  const int32_t *est_fanin;/* [E] batch-reduction fanin of each local EST's executor (0 = Sequential) */
  uint64_t *rng;           /* [E] dropout stream state (WorkerContext.dropout_rng) */
  double *stat_mean;       /* [E] TrackedStat.running_mean */
  uint64_t *stat_count;    /* [E] TrackedStat.update_count */
  double *grads;           /* fuse_reduce: [2][E][P] step-parity double buffer; else [E][P] */
  double *losses;          /* [K][E] */
  const int32_t *rot;      /* [P] allreduce rotation start per parameter (Tree only) or NULL */
  /* data: explicit global batch (split_by_rank) OR the device sampler */
  const double *rows;      /* [K][B*E_total][9] or NULL */
  const double *dataset;   /* [n][9] resident dataset (sampler mode) */
  const int32_t *lists;    /* [n_epochs][E_total][spe*B] epoch index lists (sampler mode) */
  uint64_t seed;           /* job seed (worker_rng, sampling.py:99-101) */
  int64_t step0;           /* global step of the first mini-batch in this launch */
  int64_t spe;             /* steps per epoch */
  int64_t epoch_base;      /* epoch of lists[0] */
  /* control */
  int32_t *flags;          /* [4] sticky device status (bt::Flag) */
  uint32_t *bar;           /* grid barrier counter, zeroed by the launcher */
  double *param_trace;     /* [K][P] parameters after each mini-batch (RunLog fingerprints) or NULL */
  int64_t dataset_rows;    /* rows in `dataset` (sampler mode); lets the kernel stage it in shared memory */
  /* Multi-device exchange (n_dev > 1): this launch holds ESTs [est_base, est_base + E) of E_total,
   * est_base = dev_index * E, and runs K mini-batches in lock step with the other n_dev - 1 devices'
   * launches: every mini-batch each of its EST gradient values is stored into every other device's
   * inbox (peer memory, NVLink) as two 8-byte words {32 data bits, 32-bit mini-batch tag}, and each
   * device polls its own inbox until the tags match -- no fence, counter or host step; every device
   * folds all E_total slots in the canonical rank order itself (bit-identical on every device).
   * rng / stat_mean / stat_count / est_fanin / replicas are this device's (EST pointers offset to
   * est_base); losses is [K][E_total] and only this device's columns are written. */
  int32_t n_dev;           /* 1: every EST of the job is local */
  int32_t dev_index;       /* this device's position in the exchange group */
  double *xin[BT_MAX_XDEV];     /* every device's inbox, 16 bytes per value: [2][E_total][BT_XSP][2] u64
                                   (peer-mapped; zero-initialised; step parity x EST x parameter) */
  const double *xrep[BT_MAX_XDEV]; /* every device's first replica (peer-mapped) for the launch-start
                                      agreement check (engine.py:246-258), or all NULL to skip it --
                                      only valid when no device is still writing its replicas */
} bt_mlp_args;

#ifdef __cplusplus
}
#endif

/* srl.h -- C ABI of the B200-native SRL trainer hot path (libsrl.so, sm_100a).
 *
 * The method: one PPO update of SRL's trainer worker on a batch of trajectories
 * (arXiv 2306.16688, §3.2.2 "Trainer workers": aggregate a batch, load it
 * to the GPU, compute a gradient step; multi-trainer SPMD with gradient synchronisation at
 * the end of every iteration; L885 §5: the algorithm is PPO).  PAPER.md does not write the
 * PPO/GAE equations; the readings used here are DESIGN.md §3 (from SPEC.md S:L593-611 and
 * BASELINE.json north_star).  The calls follow SPEC.md's statement of the problem:
 *   gae -> srl_gae;  advantage normalisation -> srl_adv_norm;
 *   backward/ppo_step -> srl_ppo_step;  reduce_gradients ->
 *   srl_allreduce_grads.  srl_ppo_step mirrors Algorithm.step(sample) -> {'loss': ...}
 *   plus inc_version() of PAPER.md Code 1 (L649-654).
 *
 * Conventions (all entry points):
 *  - Pointers named *_dev / documented "device" are CUDA device pointers on the context's
 *    device (or the current device for ctx-less calls).  All work is enqueued on `stream`
 *    (stream-ordered, no host synchronisation); the caller keeps every buffer alive until
 *    that work completes.  The caller owns every batch buffer and the stream; a context owns
 *    its parameters, optimiser state, gradient bucket, workspace and communicator.
 *  - Argument validation (null pointers, shapes, strides, alignment, capacity) is done on
 *    the host before any launch; failure returns SRL_EINVAL and nothing is enqueued.
 *    srl_last_error() returns a thread-local message for the last non-OK status.
 *  - There is no CPU fallback: without a CUDA device every compute call returns SRL_ECUDA.
 *  - A context is single-owner: no concurrent calls on one context.
 */
#ifndef SRL_H
#define SRL_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* srl_stream_t;     /* == cudaStream_t; NULL = legacy default stream */
typedef struct srl_ctx srl_ctx;

typedef enum srl_status {
  SRL_OK = 0,
  SRL_EINVAL = 1,        /* bad argument: null pointer, shape, stride, alignment, n > max_local_n */
  SRL_ECUDA = 2,         /* CUDA runtime / launch failure, or no device */
  SRL_ENCCL = 3,         /* cross-rank exchange failure: NCCL error, or a peer-memory wait that
                            exceeded SRL_COMM_TIMEOUT_S (default 30 s, SPEC.md S:L532
                            ReduceTimeout); the context is then failed and must be destroyed */
  SRL_ENOMEM = 4,        /* device allocation failed */
  SRL_EUNSUPPORTED = 5,  /* valid request this build does not implement */
  SRL_ESTATE = 6         /* call not valid in the context's state */
} srl_status;

const char* srl_last_error(void);
int srl_abi_version(void);                    /* 3: round-2 ABI (comm_error, srl_debug_exchange) */

/* ---------------------------------------------------------------- a1: GAE
 * Generalised advantage estimation over time-major columns (SPEC.md S:L593-601,
 * BASELINE.json north_star, readings C-A1/C-A3).  For each column b and
 * t = T-1 .. 0, with m_t = 1 - d_t:
 *     delta_t = r_t + gamma * v_{t+1} * m_t - v_t,   A_t = delta_t + gamma*lambda*m_t*A_{t+1},
 *     A_T = 0,   R_t = A_t + v_t.
 * d_t = 1 means the episode ended AT transition t: it cuts v_{t+1} and A_{t+1}.
 *   rewards  device f32 [T][ld]          values device f32 [T+1][ld] (row T = bootstrap)
 *   dones    device u8  [T][ld] flags: 0 = continue, nonzero = episode ended at t ((flag & 3) == 2,
 *            i.e. bit 1 set and bit 0 clear, = time limit, see trunc_values)
 *   adv_out  device f32 [T][ld]          ret_out f32 [T][ld] or NULL
 *   trunc_values device f32 [T][ld] or NULL (NEXT-3, DESIGN.md §3.5 reading R-T, SURVEY C-A2):
 *             a dones byte with (flag & 3) == 2 marks a time-limit truncation at t:
 *             the recursion is still cut but delta_t = r_t + gamma * trunc_values_t - v_t.
 *             NULL: every nonzero dones byte is terminal.
 *   valid    device u8 [T][ld] or NULL (NEXT-3 reading R-P, SURVEY C-A17): entries with 0 are
 *             padding and are left out of stats_out (adv/ret are still written).  The caller
 *             cuts each padded column's chain with a dones flag on its last real step.
 *   stats_out device f64 [3] or NULL: {n, mean, M2} of adv over the T*B entries (M2 = sum of
 *             squared deviations), the input srl_adv_norm takes as local_stats.
 * Layout: element (t, b) at t*ld + b; ld >= B.  With ld == B the outputs are the dense
 * sample-major vectors srl_ppo_step consumes (sample i = t*B + b).  T >= 1, B >= 1.
 * Columns are independent: a rank passes its own block of columns. */
srl_status srl_gae(int T, int B, int ld, const float* rewards, const float* values,
                   const uint8_t* dones, const float* trunc_values, const uint8_t* valid,
                   float gamma, float lambda, float* adv_out, float* ret_out,
                   double* stats_out, srl_stream_t stream);

/* ---------------------------------------------------------------- a2: normalisation
 * Batch-wide advantage normalisation (C-A4):
 *     mu, sigma over ALL samples of ALL ranks of ctx (ctx == NULL: this buffer only);
 *     sigma = sqrt(M2 / N) (unbiased = 0, default) or sqrt(M2 / (N-1)) (unbiased = 1);
 *     A_hat_i = (A_i - mu) / (sigma + eps).
 *   adv         device f32 [n]; normalised in place iff apply != 0.
 *   local_stats device f64 [3] {n, mean, M2} of this rank's adv (from srl_gae), or NULL to
 *               compute them here (warp-shuffle + block reduction over adv).
 *   mean_std_out device f64 [2] {mu, sigma} or NULL.
 * With ctx != NULL and world > 1 the ranks' {n, mean, M2} are all-gathered (over NVLink peer
 * memory when the context mapped its peers, else NCCL) and merged in rank order (Chan et al.),
 * so mu and sigma are bit-identical on all ranks.  Every rank of ctx must make the call. */
srl_status srl_adv_norm(srl_ctx* ctx, float* adv, int64_t n, const double* local_stats,
                        float eps, int unbiased, int apply, double* mean_std_out,
                        srl_stream_t stream);

/* ---------------------------------------------------------------- a3-a7: model context */
typedef enum srl_precision {
  SRL_PREC_F16_SCALED = 0   /* fp16 GEMM operands, fp32 accumulate (TMEM), per-sample dZ */
} srl_precision;

typedef struct srl_ppo_config {
  int obs_dim;              /* observation width (>= 1) */
  int ld_obs;               /* fp16 row stride of obs, >= obs_dim, % 8 == 0 (16-B rows) */
  int n_hidden;             /* L >= 1 tanh layers */
  const int* hidden;        /* [L] widths, each a multiple of 64 in [64, 1024] */
  int n_heads;              /* H >= 1 categorical heads (C-A8) */
  const int* head_sizes;    /* [H]; sum + 1 (value column) <= 64 */
  float clip_eps, value_coef, entropy_coef;   /* 0.2, 0.5, 0.01 (C-A5) */
  float lr, beta1, beta2, adam_eps;           /* 3e-4, 0.9, 0.999, 1e-8 (C-A13) */
  float adv_eps;            /* 1e-8: A_hat = (A - mu) / (sigma + adv_eps) inside the loss */
  float gamma, gae_lambda;  /* 0.99, 0.95: GAE of srl_ppo_train_step */
  int adv_unbiased;         /* 0: population sigma (default, C-A4); 1: N-1 */
  int64_t max_local_n;      /* workspace sizing: largest n_local passed to srl_ppo_step, <= 2^31 - 1 */
  int precision;            /* srl_precision */
  /* NEXT-3 PPO variants (SURVEY.md C-A5 names them as the next extension):
   *   value_clip > 0: value loss max((V-R)^2, (V_c-R)^2), V_c = v_old + clip(V - v_old, +-value_clip)
   *     (reading R-V; srl_ppo_step then needs v_old).  0: plain (V-R)^2.
   *   max_grad_norm > 0: after the allreduce, g *= min(1, max_norm / (||g||_2 + 1e-6)) before
   *     Adam (reading R-G, PyTorch clip_grad_norm_).  0: off.
   *   epochs, minibatches (<= 0 read as 1): srl_ppo_train_step runs epochs x minibatches Adam
   *     updates; local minibatch k = sample rows [k*n/M, (k+1)*n/M) (reading R-M), every rank
   *     must then hold the same T*B.  Normalisation statistics are taken once per batch. */
  float value_clip;
  float max_grad_norm;
  int epochs, minibatches;
  /* NEXT-3 separate actor and critic trunks (DESIGN.md §3.5 reading R-AC):
   *   0: one shared tanh trunk, head [logits..., value] (C-A9).
   *   1: an actor trunk and a critic trunk of the same widths on the same obs; the policy head
   *      (A logits) on the actor's last layer, the value head on the critic's.  Flat layout:
   *      actor trunk (W_l, b_l), W_pi[A][h_L], b_pi[A], critic trunk, w_v[1][h_L], b_v[1]. */
  int separate_critic;
} srl_ppo_config;

/* Device-resident statistics written by srl_ppo_step (global means over n_global). */
typedef struct srl_ppo_stats {
  double policy_loss;       /* mean -min(rho A, clip(rho) A) */
  double value_loss;        /* mean (V - R)^2 (before value_coef) */
  double entropy;           /* mean sum-over-heads entropy */
  double clip_fraction;     /* mean 1[|rho - 1| > eps] */
  double approx_kl;         /* mean (logp_old - logpi) */
  double loss;              /* policy_loss + value_coef*value_loss - entropy_coef*entropy */
  double adv_mean, adv_std; /* the normalisation used */
  int64_t n_global;
  int64_t nonfinite;        /* non-finite per-sample losses + gradient entries (all ranks) */
  int64_t fp16_saturated;   /* fp16 stores clamped to +-65504 (all ranks) */
  int64_t step;             /* Adam step t after this call = policy version (Code 1 inc_version) */
  double grad_norm;         /* NEXT-3: global gradient norm before clipping (0 if max_grad_norm == 0) */
  int64_t comm_error;       /* 1: an exchange wait of this context timed out; Adam was skipped */
} srl_ppo_stats;

/* 128-byte NCCL unique id, produced on rank 0 and broadcast by the caller. */
srl_status srl_nccl_unique_id(uint8_t out[128]);

/* Create a context on CUDA device `device` for rank `rank` of `world`.  nccl_id must be the
 * same 128 bytes on every rank (NULL iff world == 1).  Parameters are zero until
 * srl_ppo_load_params.  Layout of the flat parameter vector (C-A10): for
 * l = 1..L+1, W_l[out][in] row-major then b_l[out]; head rows head 0 .. head H-1, value last. */
srl_status srl_ppo_create(const srl_ppo_config* cfg, int rank, int world,
                          const uint8_t* nccl_id, int device, srl_ctx** out);
srl_status srl_ppo_destroy(srl_ctx* ctx);

/* Context-owned device buffers: params f32 [P] (fp32 master), grads f32 [P + 8] (the
 * gradient bucket: P gradient entries then 8 reduced statistics), Adam m and v f32 [P].
 * layout_digest = FNV-1a-64 over the int32 dims and head sizes. */
srl_status srl_ppo_params(srl_ctx* ctx, float** params_dev, float** grads_dev, int64_t* P,
                          uint64_t* layout_digest);
srl_status srl_ppo_adam_state(srl_ctx* ctx, float** m_dev, float** v_dev, int64_t* step);

/* Copy P f32 parameters (device pointer) into the context, reset Adam (m = v = 0, t = 0)
 * and refresh the fp16 weight shadows the GEMMs read. */
srl_status srl_ppo_load_params(srl_ctx* ctx, const float* params_dev, srl_stream_t stream);

/* One PPO update on this rank's samples (rows a3 -> a4 -> a5 -> a6 -> a7 of DESIGN.md §2):
 * forward, clipped-surrogate + value + entropy loss, backward,
 * gradient allreduce over the ctx's ranks, Adam.  Mean loss over n_global samples.
 *   obs       device f16 bits [n_local][ld_obs]      actions device i32 [n_local][H]
 *   logp_old  device f32 [n_local]                     adv device f32 [n_local] (raw A)
 *   ret       device f32 [n_local] (R = A + v)
 *   v_old     device f32 [n_local]: the rollout values V_old (NEXT-3 value clipping); required
 *             iff cfg.value_clip > 0, ignored otherwise (may be NULL)
 *   valid     device u8 [n_local] or NULL (NEXT-3 R-P): rows with 0 are padding -- zero
 *             gradient, no statistics; n_global then counts the valid rows of all ranks.
 *             Padding rows must still hold finite observations (0 * inf in the dW GEMM).
 *   adv_mean_std device f64 [2] {mu, sigma} from srl_adv_norm (advantages normalised inside
 *             the loss kernel), or NULL if adv is already normalised.
 *   apply     1: full update.  0: stop after the backward pass: grads_dev holds this rank's
 *             gradient of (sum of its per-sample losses) / n_global, no communication, no
 *             Adam (SPEC backward).
 *   stats_out device srl_ppo_stats* or NULL.
 * n_local <= max_local_n, n_local >= 1, n_global >= n_local. */
srl_status srl_ppo_step(srl_ctx* ctx, int64_t n_local, int64_t n_global,
                        const uint16_t* obs, const int32_t* actions, const float* logp_old,
                        const float* adv, const float* ret, const float* v_old,
                        const uint8_t* valid, const double* adv_mean_std, int apply,
                        srl_ppo_stats* stats_out, srl_stream_t stream);

/* One whole trainer step on this rank's shard of a time-major batch (rows a1 -> a7):
 * srl_gae into context-owned adv/ret (cfg gamma, gae_lambda), global normalisation moments
 * (NCCL all-gather of {n, mean, M2} when world > 1), then srl_ppo_step(apply = 1) once per
 * minibatch per epoch (cfg.epochs x cfg.minibatches, NEXT-3), v_old = values rows 0..T-1.
 * stats_out holds the last update's statistics.
 * This is Algorithm.step(sample) (PAPER.md Code 1, L649-654) for PPO.
 *   rewards f32 [T][B], values f32 [T+1][B], dones u8 [T][B] (dense, ld = B)
 *   trunc_values f32 [T][B] or NULL, valid u8 [T][B] or NULL: as srl_gae (NEXT-3); with valid,
 *   n_global = the number of valid samples of all ranks, and minibatches must be 1
 *   (SRL_EUNSUPPORTED otherwise).
 *   obs f16 bits [T*B][ld_obs], actions i32 [T*B][H], logp_old f32 [T*B] (sample i = t*B + b)
 *   n_global = sum over ranks of T*B.  T*B <= max_local_n. */
srl_status srl_ppo_train_step(srl_ctx* ctx, int T, int B, int64_t n_global,
                              const float* rewards, const float* values, const uint8_t* dones,
                              const float* trunc_values, const uint8_t* valid,
                              const uint16_t* obs, const int32_t* actions, const float* logp_old,
                              srl_ppo_stats* stats_out, srl_stream_t stream);

/* NEXT-2: policy-worker batched inference (§3.2.1: policy workers "flush
 * requests, run a batched forward and respond"; SPEC.md S:L443 counter-based RNG keyed by
 * (seed, client_id, request_id); DESIGN.md §3.6 reading R-S).  With the context's current
 * parameters: forward (a3's kernels), then the head GEMM with a sampling epilogue:
 *   u(h) = top 24 bits of sm64(sm64(seed ^ key) + h) / 2^24, sm64 = SplitMix64 finaliser;
 *   a_h = min { j : u(h) < sum_{k<=j} softmax(z^h)_k }  (deterministic != 0: argmax, lowest
 *   index on ties);  logp = sum_h log softmax(z^h)[a_h];  value = V.
 *   obs       device f16 bits [n][ld_obs] (16-byte aligned)
 *   keys      device u64 [n] request keys (e.g. client_id << 32 | request_id), NULL: key = row
 *   actions_out device i32 [n][H]; logp_out, value_out device f32 [n].
 * 1 <= n <= max_local_n.  Overwrites the context's activation workspace (not the gradients). */
srl_status srl_policy_rollout(srl_ctx* ctx, int64_t n, const uint16_t* obs, const uint64_t* keys,
                              uint64_t seed, int deterministic, int32_t* actions_out,
                              float* logp_out, float* value_out, srl_stream_t stream);

/* NEXT-1: trainer data pre-fetching (§4.1: "we reserve GPU memory for two
 * batches of training samples ... while the GPU computes the gradient on this sample batch,
 * another sample batch is pre-fetched into the other memory block").  The context owns two
 * device batch slots (allocated on first use, sized for max_local_n).
 *   srl_batch_upload copies one host batch (same layouts as srl_ppo_train_step; pinned host
 *   memory makes the copies asynchronous) into slot 0 or 1 on the context's own copy stream,
 *   after the last step that read that slot has finished with it.  It returns immediately.
 *   trunc_values / valid: optional host arrays (NULL: none for this batch), NEXT-3.
 *   srl_ppo_train_step_slot makes `stream` wait for that upload, runs srl_ppo_train_step on the
 *   slot, and releases the slot for the next upload.
 * Alternating slots overlaps the H2D copy of batch k+1 with the step on batch k. */
srl_status srl_batch_upload(srl_ctx* ctx, int slot, int T, int B, const float* rewards,
                            const float* values, const uint8_t* dones, const uint16_t* obs,
                            const int32_t* actions, const float* logp_old,
                            const float* trunc_values, const uint8_t* valid);
srl_status srl_ppo_train_step_slot(srl_ctx* ctx, int slot, int64_t n_global,
                                   srl_ppo_stats* stats_out, srl_stream_t stream);

/* How srl_ppo_step reduces the gradient bucket across ranks (a6): 0 = world 1 (none),
 * 1 = NCCL allreduce, 2 = two-shot allreduce over NVLink peer memory (CUDA IPC-mapped buckets:
 * each rank sums its 1/world chunk of all ranks' buckets in rank order, then gathers the other
 * chunks; the default when every rank could map every peer; SRL_P2P_AR=0 selects NCCL).  On
 * the peer path the exchange runs inside the step's update launch, between the split-K
 * finalise and Adam (SRL_XFUSED=0: as its own launch; bit-identical results).
 * -1 on a null ctx. */
int srl_ppo_comm_path(srl_ctx* ctx);

/* a6: in-place allreduce over the ctx's ranks of a device f32 buffer (SPEC reduce_gradients
 * S:L505-513): op 0 = sum, op 1 = mean (the sum times 1/world in fp32).  world == 1: identity.
 * With the peer path and count <= P + 8 it is the step's own two-shot rank-order exchange
 * (bit-identical on all ranks); otherwise NCCL.  Every rank must make the call with the same
 * count. */
srl_status srl_allreduce_grads(srl_ctx* ctx, float* buf, int64_t count, int op,
                               srl_stream_t stream);

/* ---------------------------------------------------------------- profiling
 * With profiling on, srl_ppo_step records a CUDA event pair on its stream around every
 * kernel (or collective) it launches, with that launch's algorithmic FLOPs and HBM bytes
 * (DESIGN.md §5).  srl_prof_read(i) waits for record i and returns its name (static string),
 * duration in ms and the two algorithmic counts.  srl_prof_reset drops all records. */
srl_status srl_prof_enable(srl_ctx* ctx, int on);
srl_status srl_prof_reset(srl_ctx* ctx);
int srl_prof_count(srl_ctx* ctx);
srl_status srl_prof_read(srl_ctx* ctx, int i, const char** name, float* ms, double* flops,
                         double* bytes);

/* ---------------------------------------------------------------- test hook
 * D[M][N] (device f32, dense) = sum_k A(m,k) * B(n,k) through the tcgen05 GEMM core with
 * its split-K epilogue (the dW path of a5).  A: a_mn == 0 -> fp16 [M][lda] (K contiguous),
 * a_mn == 1 -> fp16 [K][lda] (M contiguous); B likewise with N.  lda, ldb % 8 == 0.
 * bn in {64, 128, 256} is the N tile; splits >= 1 the K split count; cg = 1 (one SM per
 * 128-row tile) or 2 (CTA pair, tcgen05 cta_group::2, 256-row tiles; bn >= 128).
 * Used by tests only. */
srl_status srl_debug_gemm(int M, int N, int K, const uint16_t* A, int a_mn, int lda,
                          const uint16_t* B, int b_mn, int ldb, int bn, int splits, int cg,
                          float* D, srl_stream_t stream);

/* ---------------------------------------------------------------- test hook
 * The a2/a6 peer-memory exchange kernels for `world` VIRTUAL ranks on one GPU (no real peer):
 *   x        device f32 [world][ld]: rank r's bucket at x + r*ld (count entries); rank r's
 *            chunk of x[r] is overwritten with the reduced values (as on real ranks)
 *   out      device f32 [world][ld]: rank r's result = scale * (sum over ranks 0..world-1 of
 *            x, in rank order) in every entry < count
 *   tri      device f64 [world][3] {n, mean, M2} per rank, or NULL; mean_std device f64
 *            [world][2] rank r's merged {mu, sigma} (sigma population or, unbiased, N-1)
 * Every flag a rank waits for is pre-published and the phases run in the order the flags
 * would enforce (all ranks' phase 1, then all ranks' phase 2).  Synchronous.  Tests only. */
srl_status srl_debug_exchange(int world, int64_t count, int64_t ld, float* x, float* out,
                              float scale, const double* tri, double* mean_std, int unbiased,
                              srl_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif

/* oracle.h -- TEST INFRASTRUCTURE ONLY (not part of the product path).
 *
 * Plain, slow, obviously-correct CPU reference of SRL's trainer hot path
 * (arXiv 2306.16688; §3.2.2 trainer workers, L885 §5 "we employ PPO").
 * PAPER.md names PPO but states none of its equations; each function below follows the
 * reading written in DESIGN.md §3, which takes the
 * formulas from SPEC.md's `learning` module and the standard PPO/GAE algorithm.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load liboracle.so.  It shares no code, header, table or helper with the CUDA library.
 * All arithmetic is double (long double for the batch moments); inputs arrive in the
 * exact values the GPU path receives (fp32 arrays, fp16 observations widened exactly).
 *
 * Network (C-A9, C-A10): obs -> L tanh layers -> head of A+1 outputs (A = sum of the
 * categorical head sizes, value last).  Flat parameter layout: for each layer l = 1..L+1,
 * W_l[out][in] row-major, then b_l[out]; head rows ordered head 0 .. head H-1, value last.
 */
#ifndef SRL_ORACLE_H
#define SRL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* C-1  GAE by the backward recursion (BASELINE.json north_star):
 *   m_t = 1 - d_t;  delta_t = r_t + gamma * v_{t+1} * m_t - v_t;
 *   A_t = delta_t + gamma * lambda * m_t * A_{t+1},  A_T = 0;   R_t = A_t + v_t  (C-A1, C-A3).
 * r, d: [T][ld], v: [T+1][ld] (row T = bootstrap value).  adv, ret: dense [T][B].
 * d is a flag byte: nonzero ends the episode at t (m_t = 0).  NEXT-3 reading R-T (SURVEY C-A2):
 * with trunc_values [T][ld] non-null, a flag with (flag & 3) == 2 (bit 1 set, bit 0 clear) is a time-limit
 * truncation: the recursion is still cut, but delta_t bootstraps from the truncated state,
 *   delta_t = r_t + gamma * trunc_values_t - v_t.
 * trunc_values NULL: every nonzero flag is terminal (the core's reading). */
void oracle_gae(int T, int B, int ld, const float* r, const float* v, const uint8_t* d,
                const float* trunc_values, double gamma, double lambda, double* adv, double* ret);

/* C-2  batch moments, two-pass in long double: mean, and M2 = sum (a - mean)^2. */
void oracle_moments(const double* a, int64_t n, double* mean, double* m2);

/* C-2  advantage normalisation (C-A4): sigma = sqrt(M2 / n) (population,
 * unbiased=0) or sqrt(M2 / (n-1)) (unbiased=1);  out_i = (a_i - mean) / (sigma + eps). */
void oracle_adv_norm(const double* a, int64_t n, double eps, int unbiased,
                     double* out, double* mean_out, double* std_out);

/* number of parameters of the network */
int64_t oracle_param_count(int obs_dim, int L, const int* hidden, int H, const int* heads);

/* C-3  forward: per sample, naive dense layers in double.
 * obs: [n][obs_dim] (dense).  out: [n][A+1] = (logits..., value). */
void oracle_forward(int obs_dim, int L, const int* hidden, int H, const int* heads,
                    const double* params, int64_t n, const double* obs, double* out);

/* C-4  PPO loss and its exact gradient (C-A5..C-A7):
 *   per head h: l^h = logsoftmax(z^h) (max-subtracted), p^h = exp(l^h);
 *   logpi = sum_h l^h[a_h];  H = sum_h -sum_j p^h_j l^h_j;  rho = exp(logpi - logp_old);
 *   loss_i = -min(rho*A, clip(rho, 1-eps, 1+eps)*A) + c_v (V - R)^2 - c_e H.
 * The mean loss of the batch is sum_i loss_i / N with N = the GLOBAL sample count; the
 * gradient of that mean w.r.t. every parameter, restricted to these n samples, is ADDED to
 * grad[P] with grad_scale = 1/N (so K shards summed in rank order give the K=1 gradient).
 * Per-sample logit gradient (derivative of loss_i):
 *   d/dz^h_j = -mask*A*rho*(1[j=a_h] - p^h_j) + c_e p^h_j (l^h_j + H^h),
 *   mask = (A >= 0 ? rho <= 1+eps : rho >= 1-eps) (inclusive, C-A6);  d/dV = 2 c_v (V - R).
 * sums[5] += { sum loss_pg, sum (V-R)^2, sum H, sum 1[|rho-1| > eps], sum (logp_old - logpi) }.
 * adv_hat: advantages already normalised.  per_sample (nullable): [n] loss_i.
 * NEXT-3 value clipping (DESIGN.md §3.5 reading R-V; value_clip > 0 and v_old non-null):
 *   V_c = v_old + clip(V - v_old, -value_clip, +value_clip);
 *   l_v = max((V - R)^2, (V_c - R)^2);  dl_v/dV = 2 (V - R) if (V - R)^2 >= (V_c - R)^2, else
 *   2 (V_c - R) * 1[|V - v_old| <= value_clip].  value_clip <= 0 or v_old NULL: l_v = (V - R)^2. */
void oracle_loss_and_grad(int obs_dim, int L, const int* hidden, int H, const int* heads,
                          const double* params, int64_t n, const double* obs,
                          const int32_t* actions, const double* logp_old,
                          const double* adv_hat, const double* ret,
                          double clip_eps, double value_coef, double entropy_coef,
                          double grad_scale, double* grad, double* sums, double* per_sample,
                          const double* v_old, double value_clip);

/* NEXT-3 separate actor and critic trunks (
 * DESIGN.md §3.5 reading R-AC): the same obs feeds an actor trunk (L tanh layers, widths
 * hidden) with a linear policy head (A logits) and a critic trunk (same widths) with a linear
 * value head (1 output).  Flat layout: actor trunk W_l[out][in], b_l for l = 1..L; W_pi[A][h_L],
 * b_pi[A]; critic trunk likewise; w_v[1][h_L], b_v[1].  out / loss / gradient exactly as the
 * shared-trunk functions (logits..., V), the policy and entropy terms reaching the actor only
 * and the value term the critic only. */
int64_t oracle_param_count_ac(int obs_dim, int L, const int* hidden, int H, const int* heads);
void oracle_forward_ac(int obs_dim, int L, const int* hidden, int H, const int* heads,
                       const double* params, int64_t n, const double* obs, double* out);
void oracle_loss_and_grad_ac(int obs_dim, int L, const int* hidden, int H, const int* heads,
                             const double* params, int64_t n, const double* obs,
                             const int32_t* actions, const double* logp_old,
                             const double* adv_hat, const double* ret,
                             double clip_eps, double value_coef, double entropy_coef,
                             double grad_scale, double* grad, double* sums, double* per_sample,
                             const double* v_old, double value_clip);

/* NEXT-3 global gradient-norm clipping (PyTorch clip_grad_norm_ semantics, C-A5 extension):
 *   norm = sqrt(sum g_i^2);  if max_norm / (norm + 1e-6) < 1: g *= max_norm / (norm + 1e-6).
 * Returns the pre-clip norm.  max_norm <= 0: no-op (norm still returned). */
double oracle_clip_grad_norm(int64_t P, double* g, double max_norm);

/* NEXT-2 policy-worker inference (§3.2.1; SPEC.md policy worker S:L443:
 * "actions sampled from the policy distribution using a per-worker counter-based RNG keyed by
 * (seed, client_id, request_id)"; DESIGN.md §3.6 reading R-S).
 * Counter RNG: sm64(x) = SplitMix64 finaliser of x + 0x9E3779B97F4A7C15;
 *   u(seed, key, h) = (sm64(sm64(seed ^ key) + h) >> 40) * 2^-24   in [0, 1), exact in f32.
 * Per request i (key = keys[i], or i if keys is NULL) and head h: forward, log-softmax l^h,
 * p^h = exp(l^h); sampled action a_h = min { j : u < sum_{k<=j} p^h_k } (A_h - 1 if rounding
 * leaves none); deterministic != 0: a_h = argmax_j z^h_j (lowest index on ties).
 * Outputs: actions [n][H], logp [n] = sum_h l^h[a_h], value [n] = V.
 * margin (nullable) [n][H]: distance of u from the nearest CDF boundary (sampling) or the gap
 * between the two largest logits (deterministic) -- for the tests' decision-margin filter. */
double oracle_uniform(uint64_t seed, uint64_t key, int h);
void oracle_rollout(int obs_dim, int L, const int* hidden, int H, const int* heads,
                    const double* params, int64_t n, const double* obs, const uint64_t* keys,
                    uint64_t seed, int deterministic, int32_t* actions, double* logp,
                    double* value, double* margin);

/* C-6  Adam (C-A13), PyTorch semantics, step t >= 1:
 *   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;
 *   p -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps). */
void oracle_adam(int64_t P, double* p, double* m, double* v, const double* g, int64_t t,
                 double lr, double b1, double b2, double eps);

/* Timing driver for bench.py's all-core cpu_baseline: splits the n
 * samples into `threads` contiguous blocks, runs oracle_loss_and_grad on each block in its
 * own OpenMP thread into its own zeroed grad / sums buffers, then adds the buffers in block
 * order (fixed, deterministic).  The per-sample arithmetic is exactly oracle_loss_and_grad's;
 * only the order of the final sums differs (pinned against the 1-thread call to 1e-12).
 * ac != 0: the separate-trunk network (oracle_loss_and_grad_ac). */
void oracle_loss_and_grad_mt(int obs_dim, int L, const int* hidden, int H, const int* heads,
                             const double* params, int64_t n, const double* obs,
                             const int32_t* actions, const double* logp_old,
                             const double* adv_hat, const double* ret,
                             double clip_eps, double value_coef, double entropy_coef,
                             double grad_scale, double* grad, double* sums,
                             const double* v_old, double value_clip, int threads, int ac);

#ifdef __cplusplus
}
#endif
#endif

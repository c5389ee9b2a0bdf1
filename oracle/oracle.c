/* oracle.c -- TEST INFRASTRUCTURE ONLY.  See oracle.h for the contract and citations.
 *
 * Plain C99 in double.  Every function is a direct transcription of a definition in
 * DESIGN.md §3; there is no blocking, fusion or reordering beyond the
 * definition, so it can be checked against the formulas by eye.  Pins: tests/test_oracle_*.py.
 * Parity status per function: all pinned except the conventions listed
 * there as "parity unpinned" (hyper-parameter defaults, sigma convention, head sizes, init).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- C-1 GAE */
void oracle_gae(int T, int B, int ld, const float* r, const float* v, const uint8_t* d,
                const float* trunc_values, double gamma, double lambda, double* adv, double* ret) {
  for (int b = 0; b < B; ++b) {
    double A_next = 0.0;                         /* A_T = 0 */
    for (int t = T - 1; t >= 0; --t) {
      const uint8_t f = d[(int64_t)t * ld + b];
      double m = 1.0 - (double)(f != 0);                           /* m_t = 1 - d_t */
      double r_t = r[(int64_t)t * ld + b];
      double v_t = v[(int64_t)t * ld + b];
      double v_n = v[(int64_t)(t + 1) * ld + b];
      double boot = v_n * m;                                       /* v_{t+1} m_t */
      if (trunc_values && (f & 3) == 2)                            /* NEXT-3 R-T: time limit */
        boot = trunc_values[(int64_t)t * ld + b];
      double delta = r_t + gamma * boot - v_t;                     /* delta_t */
      double A = delta + gamma * lambda * m * A_next;              /* A_t */
      adv[(int64_t)t * B + b] = A;
      ret[(int64_t)t * B + b] = A + v_t;                           /* R_t = A_t + v_t */
      A_next = A;
    }
  }
}

/* ---------------------------------------------------------------- C-2 normalisation */
void oracle_moments(const double* a, int64_t n, double* mean, double* m2) {
  long double s = 0.0L;
  for (int64_t i = 0; i < n; ++i) s += a[i];
  long double mu = n > 0 ? s / (long double)n : 0.0L;
  long double q = 0.0L;
  for (int64_t i = 0; i < n; ++i) {
    long double e = (long double)a[i] - mu;
    q += e * e;
  }
  *mean = (double)mu;
  *m2 = (double)q;
}

void oracle_adv_norm(const double* a, int64_t n, double eps, int unbiased,
                     double* out, double* mean_out, double* std_out) {
  double mu, m2;
  oracle_moments(a, n, &mu, &m2);
  double denom = unbiased ? (double)(n - 1) : (double)n;
  double sigma = denom > 0 ? sqrt(m2 / denom) : 0.0;
  for (int64_t i = 0; i < n; ++i) out[i] = (a[i] - mu) / (sigma + eps);
  if (mean_out) *mean_out = mu;
  if (std_out) *std_out = sigma;
}

/* ---------------------------------------------------------------- network helpers */
static int n_actions(int H, const int* heads) {
  int A = 0;
  for (int h = 0; h < H; ++h) A += heads[h];
  return A;
}

/* d[0] = obs_dim, d[1..L] = hidden, d[L+1] = A + 1 */
static void layer_dims(int obs_dim, int L, const int* hidden, int H, const int* heads, int* d) {
  d[0] = obs_dim;
  for (int l = 0; l < L; ++l) d[l + 1] = hidden[l];
  d[L + 1] = n_actions(H, heads) + 1;
}

int64_t oracle_param_count(int obs_dim, int L, const int* hidden, int H, const int* heads) {
  int d[64];
  layer_dims(obs_dim, L, hidden, H, heads, d);
  int64_t P = 0;
  for (int l = 0; l <= L; ++l) P += (int64_t)d[l + 1] * d[l] + d[l + 1];
  return P;
}

/* y[l] for l = 0..L (y[0] = obs row), z = head output.  ys: (L+1) x maxw, z: A+1 */
static void forward_one(int L, const int* d, const double* params, const double* x,
                        double* ys, int maxw, double* z) {
  memcpy(ys, x, sizeof(double) * d[0]);
  int64_t off = 0;
  for (int l = 0; l <= L; ++l) {
    const double* W = params + off;                       /* W_l[out][in] */
    const double* bias = W + (int64_t)d[l + 1] * d[l];    /* b_l[out] */
    const double* in = ys + (int64_t)l * maxw;
    double* outp = (l < L) ? ys + (int64_t)(l + 1) * maxw : z;
    for (int o = 0; o < d[l + 1]; ++o) {
      double acc = bias[o];
      for (int i = 0; i < d[l]; ++i) acc += W[(int64_t)o * d[l] + i] * in[i];
      outp[o] = (l < L) ? tanh(acc) : acc;                 /* tanh trunk, linear head */
    }
    off += (int64_t)d[l + 1] * d[l] + d[l + 1];
  }
}

/* ---------------------------------------------------------------- C-3 forward */
void oracle_forward(int obs_dim, int L, const int* hidden, int H, const int* heads,
                    const double* params, int64_t n, const double* obs, double* out) {
  int d[64];
  layer_dims(obs_dim, L, hidden, H, heads, d);
  int maxw = 0;
  for (int l = 0; l <= L + 1; ++l) maxw = d[l] > maxw ? d[l] : maxw;
  double* ys = (double*)malloc(sizeof(double) * (size_t)(L + 1) * maxw);
  for (int64_t i = 0; i < n; ++i)
    forward_one(L, d, params, obs + i * obs_dim, ys, maxw, out + i * d[L + 1]);
  free(ys);
}

/* ---------------------------------------------------------------- C-4 loss and gradient */
/* one sample's PPO loss terms from its head outputs z[A+1] (logits..., V), and the gradient
 * of loss_i w.r.t. z, times grad_scale, into delta[A+1].  lsm, p: [A+1] scratch; Hh: [H]. */
static void sample_loss(int H, const int* heads, int A, const double* z, const int32_t* act,
                        double logp_old, double Ah, double R, const double* v_old_i,
                        double value_clip, double clip_eps, double value_coef,
                        double entropy_coef, double grad_scale, double* lsm, double* p,
                        double* Hh, double* delta, double* sums, double* loss_out) {
  /* per-head log-softmax (max-subtracted), probabilities, log-prob, entropy */
  double logpi = 0.0, ent = 0.0;
  int s = 0;
  for (int h = 0; h < H; ++h) {
    double mx = z[s];
    for (int j = 1; j < heads[h]; ++j) mx = z[s + j] > mx ? z[s + j] : mx;
    double se = 0.0;
    for (int j = 0; j < heads[h]; ++j) se += exp(z[s + j] - mx);
    double lse = mx + log(se);
    double hh = 0.0;
    for (int j = 0; j < heads[h]; ++j) {
      lsm[s + j] = z[s + j] - lse;
      p[s + j] = exp(lsm[s + j]);
      hh -= p[s + j] * lsm[s + j];
    }
    Hh[h] = hh;
    ent += hh;
    logpi += lsm[s + act[h]];
    s += heads[h];
  }
  const double rho = exp(logpi - logp_old);
  const double rho_c = rho < 1.0 - clip_eps ? 1.0 - clip_eps
                     : (rho > 1.0 + clip_eps ? 1.0 + clip_eps : rho);
  const double s1 = rho * Ah, s2 = rho_c * Ah;
  const double l_pg = -(s1 < s2 ? s1 : s2);
  const double V = z[A];
  double l_v = (V - R) * (V - R);
  double dV = 2.0 * (V - R);                                    /* d l_v / dV */
  if (value_clip > 0.0 && v_old_i) {                            /* NEXT-3 value clipping */
    const double dlt = V - *v_old_i;
    const double Vc = *v_old_i + (dlt < -value_clip ? -value_clip : (dlt > value_clip ? value_clip : dlt));
    const double l_c = (Vc - R) * (Vc - R);
    if (l_c > l_v) {
      l_v = l_c;
      dV = (fabs(dlt) <= value_clip) ? 2.0 * (Vc - R) : 0.0;
    }
  }
  *loss_out = l_pg + value_coef * l_v - entropy_coef * ent;
  sums[0] += l_pg;
  sums[1] += l_v;
  sums[2] += ent;
  sums[3] += fabs(rho - 1.0) > clip_eps ? 1.0 : 0.0;
  sums[4] += logp_old - logpi;

  /* per-sample logit gradient (closed form, see header), times grad_scale = 1/N */
  const double mask = (Ah >= 0.0) ? (rho <= 1.0 + clip_eps ? 1.0 : 0.0)
                                  : (rho >= 1.0 - clip_eps ? 1.0 : 0.0);
  s = 0;
  for (int h = 0; h < H; ++h) {
    for (int j = 0; j < heads[h]; ++j) {
      double onehot = (j == act[h]) ? 1.0 : 0.0;
      double g = -mask * Ah * rho * (onehot - p[s + j])
                 + entropy_coef * p[s + j] * (lsm[s + j] + Hh[h]);
      delta[s + j] = grad_scale * g;
    }
    s += heads[h];
  }
  delta[A] = grad_scale * value_coef * dV;
}

void oracle_loss_and_grad(int obs_dim, int L, const int* hidden, int H, const int* heads,
                          const double* params, int64_t n, const double* obs,
                          const int32_t* actions, const double* logp_old,
                          const double* adv_hat, const double* ret,
                          double clip_eps, double value_coef, double entropy_coef,
                          double grad_scale, double* grad, double* sums, double* per_sample,
                          const double* v_old, double value_clip) {
  int d[64];
  layer_dims(obs_dim, L, hidden, H, heads, d);
  const int A = d[L + 1] - 1;
  int maxw = 0;
  for (int l = 0; l <= L + 1; ++l) maxw = d[l] > maxw ? d[l] : maxw;
  int64_t offs[64];
  offs[0] = 0;
  for (int l = 0; l <= L; ++l) offs[l + 1] = offs[l] + (int64_t)d[l + 1] * d[l] + d[l + 1];

  double* ys = (double*)malloc(sizeof(double) * (size_t)(L + 1) * maxw);
  double* z = (double*)malloc(sizeof(double) * (size_t)(A + 1));
  double* lsm = (double*)malloc(sizeof(double) * (size_t)(A + 1));   /* log-softmax */
  double* p = (double*)malloc(sizeof(double) * (size_t)(A + 1));
  double* Hh = (double*)malloc(sizeof(double) * (size_t)(H > 0 ? H : 1));
  double* delta = (double*)malloc(sizeof(double) * (size_t)maxw);
  double* dy = (double*)malloc(sizeof(double) * (size_t)maxw);

  for (int64_t i = 0; i < n; ++i) {
    forward_one(L, d, params, obs + i * obs_dim, ys, maxw, z);
    double loss_i;
    sample_loss(H, heads, A, z, actions + i * H, logp_old[i], adv_hat[i], ret[i],
                (value_clip > 0.0 && v_old) ? v_old + i : NULL, value_clip, clip_eps,
                value_coef, entropy_coef, grad_scale, lsm, p, Hh, delta, sums, &loss_i);
    if (per_sample) per_sample[i] = loss_i;

    /* backprop through the layers, l = L (head) down to 0 */
    for (int l = L; l >= 0; --l) {
      const double* W = params + offs[l];
      double* gW = grad + offs[l];
      double* gb = gW + (int64_t)d[l + 1] * d[l];
      const double* in = ys + (int64_t)l * maxw;                /* y_l, input of layer l */
      for (int o = 0; o < d[l + 1]; ++o) {
        for (int k = 0; k < d[l]; ++k) gW[(int64_t)o * d[l] + k] += delta[o] * in[k];
        gb[o] += delta[o];
      }
      if (l == 0) break;
      for (int k = 0; k < d[l]; ++k) {
        double acc = 0.0;
        for (int o = 0; o < d[l + 1]; ++o) acc += delta[o] * W[(int64_t)o * d[l] + k];
        dy[k] = acc;
      }
      for (int k = 0; k < d[l]; ++k) delta[k] = dy[k] * (1.0 - in[k] * in[k]);  /* tanh' */
    }
  }
  free(ys); free(z); free(lsm); free(p); free(Hh); free(delta); free(dy);
}

/* ---------------------------------------------------------------- NEXT-3 separate trunks */
/* Layout (DESIGN.md §3.5 reading R-AC): actor trunk (L tanh layers W_l[out][in], b_l), actor
 * head W_pi[A][h_L], b_pi[A], then critic trunk (same widths), critic head w_v[1][h_L], b_v. */
static int64_t trunk_count(int L, const int* d) {       /* d[0..L]: obs, hidden widths */
  int64_t P = 0;
  for (int l = 0; l < L; ++l) P += (int64_t)d[l + 1] * d[l] + d[l + 1];
  return P;
}

int64_t oracle_param_count_ac(int obs_dim, int L, const int* hidden, int H, const int* heads) {
  int d[64];
  layer_dims(obs_dim, L, hidden, H, heads, d);
  const int A = d[L + 1] - 1;
  return 2 * trunk_count(L, d) + (int64_t)A * d[L] + A + d[L] + 1;
}

/* one trunk: ys row l (l = 0..L) = y_l, y_0 = x;  y_l = tanh(W_l y_{l-1} + b_l) */
static void trunk_fwd(int L, const int* d, const double* p, const double* x, double* ys, int maxw) {
  memcpy(ys, x, sizeof(double) * d[0]);
  int64_t off = 0;
  for (int l = 0; l < L; ++l) {
    const double* W = p + off;
    const double* b = W + (int64_t)d[l + 1] * d[l];
    const double* in = ys + (int64_t)l * maxw;
    double* out = ys + (int64_t)(l + 1) * maxw;
    for (int o = 0; o < d[l + 1]; ++o) {
      double acc = b[o];
      for (int i = 0; i < d[l]; ++i) acc += W[(int64_t)o * d[l] + i] * in[i];
      out[o] = tanh(acc);
    }
    off += (int64_t)d[l + 1] * d[l] + d[l + 1];
  }
}

/* a linear head on y: out[r] = b[r] + sum_k W[r][k] y[k], r < rows */
static void head_fwd(int rows, int in, const double* W, const double* y, double* out) {
  const double* b = W + (int64_t)rows * in;
  for (int r = 0; r < rows; ++r) {
    double acc = b[r];
    for (int k = 0; k < in; ++k) acc += W[(int64_t)r * in + k] * y[k];
    out[r] = acc;
  }
}

/* backprop of a head + trunk: dlt[rows] = dloss/d(head out) (scaled); adds the head's and the
 * trunk's gradients.  delta, dy: [maxw] scratch. */
static void head_trunk_bwd(int L, const int* d, int rows, const double* p_trunk,
                           const double* W_head, const double* ys, int maxw, const double* dlt,
                           double* g_trunk, double* g_head, double* delta, double* dy) {
  const int in = d[L];
  const double* yL = ys + (int64_t)L * maxw;
  for (int r = 0; r < rows; ++r) {
    for (int k = 0; k < in; ++k) g_head[(int64_t)r * in + k] += dlt[r] * yL[k];
    g_head[(int64_t)rows * in + r] += dlt[r];
  }
  for (int k = 0; k < in; ++k) {
    double acc = 0.0;
    for (int r = 0; r < rows; ++r) acc += dlt[r] * W_head[(int64_t)r * in + k];
    delta[k] = acc * (1.0 - yL[k] * yL[k]);                      /* tanh' of layer L */
  }
  int64_t offs[64];
  offs[0] = 0;
  for (int l = 0; l < L; ++l) offs[l + 1] = offs[l] + (int64_t)d[l + 1] * d[l] + d[l + 1];
  for (int l = L - 1; l >= 0; --l) {                             /* trunk layer l: d[l] -> d[l+1] */
    const double* W = p_trunk + offs[l];
    double* gW = g_trunk + offs[l];
    double* gb = gW + (int64_t)d[l + 1] * d[l];
    const double* inl = ys + (int64_t)l * maxw;
    for (int o = 0; o < d[l + 1]; ++o) {
      for (int k = 0; k < d[l]; ++k) gW[(int64_t)o * d[l] + k] += delta[o] * inl[k];
      gb[o] += delta[o];
    }
    if (l == 0) break;
    for (int k = 0; k < d[l]; ++k) {
      double acc = 0.0;
      for (int o = 0; o < d[l + 1]; ++o) acc += delta[o] * W[(int64_t)o * d[l] + k];
      dy[k] = acc;
    }
    for (int k = 0; k < d[l]; ++k) delta[k] = dy[k] * (1.0 - inl[k] * inl[k]);
  }
}

void oracle_forward_ac(int obs_dim, int L, const int* hidden, int H, const int* heads,
                       const double* params, int64_t n, const double* obs, double* out) {
  int d[64];
  layer_dims(obs_dim, L, hidden, H, heads, d);
  const int A = d[L + 1] - 1;
  int maxw = 0;
  for (int l = 0; l <= L; ++l) maxw = d[l] > maxw ? d[l] : maxw;
  const int64_t T = trunk_count(L, d);
  const double* pa = params;                                  /* actor trunk */
  const double* wpi = pa + T;                                 /* actor head [A][h_L] + [A] */
  const double* pc = wpi + (int64_t)A * d[L] + A;             /* critic trunk */
  const double* wv = pc + T;                                  /* critic head [1][h_L] + [1] */
  double* ya = (double*)malloc(sizeof(double) * (size_t)(L + 1) * maxw);
  double* yc = (double*)malloc(sizeof(double) * (size_t)(L + 1) * maxw);
  for (int64_t i = 0; i < n; ++i) {
    trunk_fwd(L, d, pa, obs + i * obs_dim, ya, maxw);
    trunk_fwd(L, d, pc, obs + i * obs_dim, yc, maxw);
    head_fwd(A, d[L], wpi, ya + (int64_t)L * maxw, out + i * (A + 1));
    head_fwd(1, d[L], wv, yc + (int64_t)L * maxw, out + i * (A + 1) + A);
  }
  free(ya);
  free(yc);
}

void oracle_loss_and_grad_ac(int obs_dim, int L, const int* hidden, int H, const int* heads,
                             const double* params, int64_t n, const double* obs,
                             const int32_t* actions, const double* logp_old,
                             const double* adv_hat, const double* ret,
                             double clip_eps, double value_coef, double entropy_coef,
                             double grad_scale, double* grad, double* sums, double* per_sample,
                             const double* v_old, double value_clip) {
  int d[64];
  layer_dims(obs_dim, L, hidden, H, heads, d);
  const int A = d[L + 1] - 1;
  int maxw = 0;
  for (int l = 0; l <= L + 1; ++l) maxw = d[l] > maxw ? d[l] : maxw;
  const int64_t T = trunk_count(L, d);
  const int64_t o_pi = T, o_c = T + (int64_t)A * d[L] + A, o_v = o_c + T;
  double* ya = (double*)malloc(sizeof(double) * (size_t)(L + 1) * maxw);
  double* yc = (double*)malloc(sizeof(double) * (size_t)(L + 1) * maxw);
  double* z = (double*)malloc(sizeof(double) * (size_t)(A + 1));
  double* lsm = (double*)malloc(sizeof(double) * (size_t)(A + 1));
  double* p = (double*)malloc(sizeof(double) * (size_t)(A + 1));
  double* Hh = (double*)malloc(sizeof(double) * (size_t)(H > 0 ? H : 1));
  double* dz = (double*)malloc(sizeof(double) * (size_t)(A + 1));
  double* delta = (double*)malloc(sizeof(double) * (size_t)maxw);
  double* dy = (double*)malloc(sizeof(double) * (size_t)maxw);
  for (int64_t i = 0; i < n; ++i) {
    trunk_fwd(L, d, params, obs + i * obs_dim, ya, maxw);
    trunk_fwd(L, d, params + o_c, obs + i * obs_dim, yc, maxw);
    head_fwd(A, d[L], params + o_pi, ya + (int64_t)L * maxw, z);
    head_fwd(1, d[L], params + o_v, yc + (int64_t)L * maxw, z + A);
    double loss_i;
    sample_loss(H, heads, A, z, actions + i * H, logp_old[i], adv_hat[i], ret[i],
                (value_clip > 0.0 && v_old) ? v_old + i : NULL, value_clip, clip_eps,
                value_coef, entropy_coef, grad_scale, lsm, p, Hh, dz, sums, &loss_i);
    if (per_sample) per_sample[i] = loss_i;
    /* logits -> actor head + trunk; V -> critic head + trunk */
    head_trunk_bwd(L, d, A, params, params + o_pi, ya, maxw, dz, grad, grad + o_pi, delta, dy);
    head_trunk_bwd(L, d, 1, params + o_c, params + o_v, yc, maxw, dz + A, grad + o_c, grad + o_v,
                   delta, dy);
  }
  free(ya); free(yc); free(z); free(lsm); free(p); free(Hh); free(dz); free(delta); free(dy);
}

/* ---------------------------------------------------------------- NEXT-2 rollout */
static uint64_t sm64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double oracle_uniform(uint64_t seed, uint64_t key, int h) {
  return (double)(sm64(sm64(seed ^ key) + (uint64_t)h) >> 40) * (1.0 / 16777216.0);
}

void oracle_rollout(int obs_dim, int L, const int* hidden, int H, const int* heads,
                    const double* params, int64_t n, const double* obs, const uint64_t* keys,
                    uint64_t seed, int deterministic, int32_t* actions, double* logp,
                    double* value, double* margin) {
  int d[64];
  layer_dims(obs_dim, L, hidden, H, heads, d);
  const int A = d[L + 1] - 1;
  double* z = (double*)malloc(sizeof(double) * (size_t)(A + 1));
  double* out = (double*)malloc(sizeof(double) * (size_t)(A + 1));
  for (int64_t i = 0; i < n; ++i) {
    oracle_forward(obs_dim, L, hidden, H, heads, params, 1, obs + i * obs_dim, z);
    const uint64_t key = keys ? keys[i] : (uint64_t)i;
    double lp = 0.0;
    int s = 0;
    for (int h = 0; h < H; ++h) {
      const int a_n = heads[h];
      double mx = z[s];
      for (int j = 1; j < a_n; ++j) mx = z[s + j] > mx ? z[s + j] : mx;
      double se = 0.0;
      for (int j = 0; j < a_n; ++j) se += exp(z[s + j] - mx);
      const double lse = mx + log(se);
      for (int j = 0; j < a_n; ++j) out[j] = z[s + j] - lse;     /* log-softmax */
      int a = a_n - 1;
      double mg = 1.0;
      if (deterministic) {
        a = 0;
        for (int j = 1; j < a_n; ++j) if (z[s + j] > z[s + a]) a = j;
        for (int j = 0; j < a_n; ++j)
          if (j != a && z[s + a] - z[s + j] < mg) mg = z[s + a] - z[s + j];
      } else {
        const double u = oracle_uniform(seed, key, h);
        double cdf = 0.0;
        for (int j = 0; j < a_n; ++j) {         /* inverse CDF: first j with u < cdf_j */
          cdf += exp(out[j]);
          if (j < a_n - 1 && fabs(u - cdf) < mg) mg = fabs(u - cdf);
          if (u < cdf) { a = j; break; }
        }
      }
      actions[i * H + h] = a;
      lp += out[a];
      if (margin) margin[i * H + h] = mg;
      s += a_n;
    }
    logp[i] = lp;
    value[i] = z[A];
  }
  free(z);
  free(out);
}

/* ---------------------------------------------------------------- NEXT-3 grad-norm clip */
double oracle_clip_grad_norm(int64_t P, double* g, double max_norm) {
  long double ss = 0.0L;
  for (int64_t i = 0; i < P; ++i) ss += (long double)g[i] * g[i];
  const double norm = sqrt((double)ss);
  if (max_norm > 0.0) {
    const double coef = max_norm / (norm + 1e-6);
    if (coef < 1.0)
      for (int64_t i = 0; i < P; ++i) g[i] *= coef;
  }
  return norm;
}

/* ---------------------------------------------------------------- C-6 Adam */
void oracle_adam(int64_t P, double* p, double* m, double* v, const double* g, int64_t t,
                 double lr, double b1, double b2, double eps) {
  const double bc1 = 1.0 - pow(b1, (double)t);
  const double bc2 = 1.0 - pow(b2, (double)t);
  for (int64_t i = 0; i < P; ++i) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    double mhat = m[i] / bc1;
    double vhat = v[i] / bc2;
    p[i] -= lr * mhat / (sqrt(vhat) + eps);
  }
}

/* ---------------------------------------------------------------- all-core timing driver */
void oracle_loss_and_grad_mt(int obs_dim, int L, const int* hidden, int H, const int* heads,
                             const double* params, int64_t n, const double* obs,
                             const int32_t* actions, const double* logp_old,
                             const double* adv_hat, const double* ret,
                             double clip_eps, double value_coef, double entropy_coef,
                             double grad_scale, double* grad, double* sums,
                             const double* v_old, double value_clip, int threads, int ac) {
  if (threads < 1) threads = 1;
  const int64_t P = ac ? oracle_param_count_ac(obs_dim, L, hidden, H, heads)
                       : oracle_param_count(obs_dim, L, hidden, H, heads);
  double* g = (double*)calloc((size_t)threads * (size_t)P, sizeof(double));
  double* s = (double*)calloc((size_t)threads * 5, sizeof(double));
  #pragma omp parallel for num_threads(threads) schedule(static, 1)
  for (int k = 0; k < threads; ++k) {
    const int64_t lo = n * k / threads, hi = n * (k + 1) / threads;
    const int H_ = H;
    const int od = obs_dim;
    if (hi > lo)
      (ac ? oracle_loss_and_grad_ac : oracle_loss_and_grad)(
          obs_dim, L, hidden, H, heads, params, hi - lo, obs + lo * od, actions + lo * H_,
          logp_old + lo, adv_hat + lo, ret + lo, clip_eps, value_coef, entropy_coef, grad_scale,
          g + (int64_t)k * P, s + 5 * k, NULL, v_old ? v_old + lo : NULL, value_clip);
  }
  for (int k = 0; k < threads; ++k) {            /* block order */
    for (int64_t i = 0; i < P; ++i) grad[i] += g[(int64_t)k * P + i];
    for (int j = 0; j < 5; ++j) sums[j] += s[5 * k + j];
  }
  free(g);
  free(s);
}

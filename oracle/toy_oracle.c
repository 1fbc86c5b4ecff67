/* TEST INFRASTRUCTURE ONLY -- see toy_oracle.h for scope and the reference
 * file:line each function restates.  Written in plain C so that it can never be
 * mistaken for (or linked into) the product library. */
#include "toy_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- mt19937_64 (std::mersenne_twister_engine 64-bit parameters) ------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* libstdc++ std::generate_canonical<double,53>(mt19937_64) then
 * uniform_real_distribution: u * (b - a) + a. */
static double uniform(mt64* g, double a, double b) {
  double u = (double)mt64_next(g) / 18446744073709551616.0;
  if (u >= 1.0) u = nextafter(1.0, 0.0);
  return u * (b - a) + a;
}

/* oracle.cpp:94-111 */
int toy_make_model(const int* dims, int n_dims, uint64_t seed, double* params) {
  if (n_dims < 2) return 2;
  mt64 g;
  mt64_seed(&g, seed);
  size_t off = 0;
  for (int s = 0; s + 1 < n_dims; ++s) {
    const int in = dims[s], out = dims[s + 1];
    const double scale = 1.0 / sqrt((double)in);
    for (long i = 0; i < (long)out * in; ++i) params[off++] = uniform(&g, -0.5, 0.5) * scale;
    for (int i = 0; i < out; ++i) params[off++] = uniform(&g, -0.5, 0.5) * 0.1;
  }
  return 0;
}

/* oracle.cpp:113-123 */
int toy_make_batch(const int* dims, int n_dims, int size, uint64_t seed, double* inputs,
                   double* targets) {
  mt64 g;
  mt64_seed(&g, seed ^ 0x9e3779b97f4a7c15ULL);
  for (long i = 0; i < (long)size * dims[0]; ++i) inputs[i] = uniform(&g, -1.0, 1.0);
  for (long i = 0; i < (long)size * dims[n_dims - 1]; ++i)
    targets[i] = uniform(&g, -1.0, 1.0) * 0.5;
  return 0;
}

/* ---- dense task index: (is_backward, pipeline, micro, stage) -> flat task id ---- */
typedef struct {
  int P, M, S;
  int* slot; /* -1 = absent */
} task_index;

static int ti_key(const task_index* ix, int b, int p, int m, int s) {
  if (p < 0 || m < 0 || s < 0 || p >= ix->P || m >= ix->M || s >= ix->S) return -1;
  return ((b * ix->P + p) * ix->M + m) * ix->S + s;
}

static void ti_build(task_index* ix, int total, const int* tasks) {
  ix->P = ix->M = ix->S = 1;
  for (int t = 0; t < total; ++t) {
    const int* k = tasks + 6 * t;
    if (k[1] + 1 > ix->P) ix->P = k[1] + 1;
    if (k[2] + 1 > ix->M) ix->M = k[2] + 1;
    if (k[3] + 2 > ix->S) ix->S = k[3] + 2;
  }
  const int n = 2 * ix->P * ix->M * ix->S;
  ix->slot = (int*)malloc(sizeof(int) * n);
  for (int i = 0; i < n; ++i) ix->slot[i] = -1;
  for (int t = 0; t < total; ++t) {
    const int* k = tasks + 6 * t;
    if (k[0] != 0 && k[0] != 1) continue;
    const int key = ti_key(ix, k[0], k[1], k[2], k[3]);
    if (ix->slot[key] < 0) ix->slot[key] = t; /* first occurrence wins (map::emplace) */
  }
}

static int ti_find(const task_index* ix, int b, int p, int m, int s) {
  const int key = ti_key(ix, b, p, m, s);
  return key < 0 ? -1 : ix->slot[key];
}

/* listsched.hpp:52-163 restated over flat arrays; returns 3 on a dependency cycle. */
int toy_list_schedule(int workers, const int* counts, const int* tasks, double f_dur,
                      double b_dur, double p2p_fwd, double p2p_bwd, int relaxed,
                      double* starts, double* ends, double* makespan) {
  const double kInf = INFINITY, kEps = 1e-12;
  int total = 0;
  int* base = (int*)malloc(sizeof(int) * (workers + 1));
  for (int w = 0; w < workers; ++w) {
    base[w] = total;
    total += counts[w];
  }
  base[workers] = total;
  int* owner = (int*)malloc(sizeof(int) * (total ? total : 1));
  for (int w = 0; w < workers; ++w)
    for (int i = base[w]; i < base[w + 1]; ++i) owner[i] = w;
  task_index ix;
  ti_build(&ix, total, tasks);
  char* done = (char*)calloc((size_t)(total > 0 ? total : 1), 1);
  double* free_at = (double*)calloc(workers, sizeof(double));
  int* head = (int*)calloc(workers, sizeof(int));
  for (int t = 0; t < total; ++t) starts[t] = ends[t] = -1;
  *makespan = 0;
  int rc = 0;

  for (int remaining = total; remaining > 0; --remaining) {
    int best = -1;
    double best_est = kInf;
    for (int w = 0; w < workers; ++w) {
      const int n = counts[w];
      while (head[w] < n && done[base[w] + head[w]]) ++head[w];
      if (head[w] >= n) continue;
      int cand = -1;
      double cand_est = kInf;
      int fwd_pending = 0;
      for (int i = head[w]; i < n; ++i) {
        const int t = base[w] + i;
        if (done[t]) continue;
        const int* k = tasks + 6 * t;
        const int eligible = i == head[w] || (relaxed && k[0] == 0 && !fwd_pending);
        if (eligible) {
          double est = free_at[w];
          int blocked = 0;
          /* predecessor list: (is_backward, stage, edge cost) */
          int pb[2], ps[2], np = 0;
          double pc[2];
          if (k[0] == 0 && k[3] > 0) {
            pb[np] = 0; ps[np] = k[3] - 1; pc[np++] = p2p_fwd;
          } else if (k[0] == 1) {
            pb[np] = 1; ps[np] = k[3] + 1; pc[np++] = p2p_bwd;
            pb[np] = 0; ps[np] = k[3]; pc[np++] = 0.0;
          }
          for (int q = 0; q < np && !blocked; ++q) {
            const int d = ti_find(&ix, pb[q], k[1], k[2], ps[q]);
            if (d < 0 || d == t) continue;
            if (!done[d]) { blocked = 1; break; }
            const double e = ends[d] + (owner[d] == w ? 0.0 : pc[q]);
            if (e > est) est = e;
          }
          if (blocked) est = kInf;
          if (est < cand_est - kEps) { cand = t; cand_est = est; }
        }
        if (k[0] == 0) fwd_pending = 1;
        if (!relaxed) break;
        if (fwd_pending && i > head[w]) break;
      }
      if (cand >= 0 && cand_est < best_est - kEps) { best = cand; best_est = cand_est; }
    }
    if (best < 0) { rc = 3; break; }
    const int kind = tasks[6 * best];
    const double dur = kind == 1 ? b_dur : kind == 0 ? f_dur : 0.0;
    starts[best] = best_est;
    ends[best] = best_est + dur;
    done[best] = 1;
    free_at[owner[best]] = best_est + dur;
    if (best_est + dur > *makespan) *makespan = best_est + dur;
  }
  free(base); free(owner); free(ix.slot); free(done); free(free_at); free(head);
  return rc;
}

/* ---- ToyModel numerics (oracle.cpp:34-76) ------------------------------------- */
typedef struct { double* v; double* c; } kahan;

static void kahan_add(kahan* k, long i, double x) {
  const double y = x - k->c[i];
  const double t = k->v[i] + y;
  k->c[i] = (t - k->v[i]) - y;
  k->v[i] = t;
}

static void stage_forward(const double* w, const double* b, const double* x, double* y,
                          int out, int in) {
  for (int o = 0; o < out; ++o) {
    double acc = b[o];
    for (int i = 0; i < in; ++i) acc += w[(long)o * in + i] * x[i];
    y[o] = tanh(acc);
  }
}

static void stage_backward(const double* w, const double* x, const double* y,
                           const double* g_y, int out, int in, double scale, kahan* gw,
                           kahan* gb, double* g_x) {
  for (int i = 0; i < in; ++i) g_x[i] = 0.0;
  for (int o = 0; o < out; ++o) {
    const double gz = g_y[o] * (1.0 - y[o] * y[o]);
    kahan_add(gb, o, gz * scale);
    for (int i = 0; i < in; ++i) {
      kahan_add(gw, (long)o * in + i, gz * x[i] * scale);
      g_x[i] += w[(long)o * in + i] * gz;
    }
  }
}

typedef struct {
  int D;
  const int* dims;
  long* w_off; /* offset of W_s in the flat params */
  long* b_off;
  long n_params;
} layout;

static void layout_build(layout* L, const int* dims, int n_dims) {
  L->D = n_dims - 1;
  L->dims = dims;
  L->w_off = (long*)malloc(sizeof(long) * L->D);
  L->b_off = (long*)malloc(sizeof(long) * L->D);
  long off = 0;
  for (int s = 0; s < L->D; ++s) {
    L->w_off[s] = off;
    off += (long)dims[s] * dims[s + 1];
    L->b_off[s] = off;
    off += dims[s + 1];
  }
  L->n_params = off;
}

static void layout_free(layout* L) { free(L->w_off); free(L->b_off); }

/* Per-(replica, pipeline) gradient accumulators over the whole flat parameter
 * vector: grads[(r * P + p)] is a kahan over n_params entries. */
static kahan* grads_new(int copies, long n) {
  kahan* g = (kahan*)malloc(sizeof(kahan) * copies);
  for (int i = 0; i < copies; ++i) {
    g[i].v = (double*)calloc(n, sizeof(double));
    g[i].c = (double*)calloc(n, sizeof(double));
  }
  return g;
}

static void grads_free(kahan* g, int copies) {
  for (int i = 0; i < copies; ++i) { free(g[i].v); free(g[i].c); }
  free(g);
}

static kahan view(const kahan* k, long off) {
  kahan v = {k->v + off, k->c + off};
  return v;
}

/* oracle.cpp:125-151 */
int toy_sequential_sgd(const int* dims, int n_dims, const double* params,
                       const double* inputs, const double* targets, int batch, double lr,
                       double* params_out) {
  layout L;
  layout_build(&L, dims, n_dims);
  kahan* g = grads_new(1, L.n_params);
  int maxd = 0;
  for (int s = 0; s < n_dims; ++s) if (dims[s] > maxd) maxd = dims[s];
  double* acts = (double*)malloc(sizeof(double) * n_dims * maxd);
  double* gy = (double*)malloc(sizeof(double) * maxd);
  double* gx = (double*)malloc(sizeof(double) * maxd);
  const double scale = 1.0 / batch;
  for (int n = 0; n < batch; ++n) {
    memcpy(acts, inputs + (long)n * dims[0], sizeof(double) * dims[0]);
    for (int s = 0; s < L.D; ++s)
      stage_forward(params + L.w_off[s], params + L.b_off[s], acts + s * maxd,
                    acts + (s + 1) * maxd, dims[s + 1], dims[s]);
    const int od = dims[L.D];
    for (int o = 0; o < od; ++o)
      gy[o] = acts[L.D * maxd + o] - targets[(long)n * od + o];
    for (int s = L.D - 1; s >= 0; --s) {
      kahan gw = view(&g[0], L.w_off[s]), gb = view(&g[0], L.b_off[s]);
      stage_backward(params + L.w_off[s], acts + s * maxd, acts + (s + 1) * maxd, gy,
                     dims[s + 1], dims[s], scale, &gw, &gb, gx);
      memcpy(gy, gx, sizeof(double) * dims[s]);
    }
  }
  for (long i = 0; i < L.n_params; ++i) params_out[i] = params[i] - lr * g[0].v[i];
  grads_free(g, 1);
  free(acts); free(gy); free(gx);
  layout_free(&L);
  return 0;
}

/* oracle.cpp:162-300 (Engine) + 304-351 (replay).  All 2f*W model copies stay
 * bit-identical (every copy receives the same summed update, oracle.cpp:294-298),
 * so one parameter vector stands for all of them; gradient sums stay per copy so
 * that the final summation order matches oracle.cpp:288-293. */
int toy_run_iteration(int D, int W, int N, int B, int halved, int workers, const int* counts,
                      const int* tasks, const int* dims, int n_dims, const double* params,
                      const double* inputs, const double* targets, int batch, double lr,
                      double* params_out, int* peak_stash) {
  if (n_dims - 1 != D) return 2;
  if (batch != B * N * W) return 2;
  int total = 0;
  for (int w = 0; w < workers; ++w) total += counts[w];
  int* owner = (int*)malloc(sizeof(int) * (total ? total : 1));
  int* local = (int*)malloc(sizeof(int) * (total ? total : 1));
  for (int w = 0, t = 0; w < workers; ++w)
    for (int i = 0; i < counts[w]; ++i, ++t) { owner[t] = w; local[t] = i; }

  /* replay order: tick_schedule with the unit profile (backward_ratio 2 ->
   * f = 1 tick, b = 2; halved: f = 2, b = 2), sorted by (start, worker, index). */
  double* st = (double*)malloc(sizeof(double) * (total ? total : 1));
  double* en = (double*)malloc(sizeof(double) * (total ? total : 1));
  double mk;
  int rc = toy_list_schedule(workers, counts, tasks, halved ? 2.0 : 1.0, 2.0, 0.0, 0.0, 0,
                             st, en, &mk);
  if (rc) { free(owner); free(local); free(st); free(en); return rc; }
  int* order = (int*)malloc(sizeof(int) * (total ? total : 1));
  for (int t = 0; t < total; ++t) order[t] = t;
  /* insertion sort by (start, worker, index): t is already (worker, index)-ordered */
  for (int a = 1; a < total; ++a) {
    const int x = order[a];
    int b = a - 1;
    while (b >= 0 && (st[order[b]] > st[x] || (st[order[b]] == st[x] && order[b] > x))) {
      order[b + 1] = order[b];
      --b;
    }
    order[b + 1] = x;
  }

  int P = 1;
  for (int t = 0; t < total; ++t) if (tasks[6 * t + 1] + 1 > P) P = tasks[6 * t + 1] + 1;
  layout L;
  layout_build(&L, dims, n_dims);
  kahan* g = grads_new(W * P, L.n_params);
  int maxd = 0;
  for (int s = 0; s < n_dims; ++s) if (dims[s] > maxd) maxd = dims[s];

  /* stash[(r,p,m,s)] -> B inputs and B outputs (maxd each); grad_in likewise */
  const int M = N > 0 ? N : 1;
  const long nkeys = (long)W * P * M * D;
  double** st_in = (double**)calloc(nkeys, sizeof(double*));
  double** st_out = (double**)calloc(nkeys, sizeof(double*));
  double** gin = (double**)calloc(nkeys, sizeof(double*));
  int* live = (int*)calloc(workers, sizeof(int));
  for (int w = 0; w < workers; ++w) peak_stash[w] = 0;
  double* gy = (double*)malloc(sizeof(double) * maxd);
  const double scale = 1.0 / (double)batch;
#define KEY(r, p, m, s) ((((long)(r) * P + (p)) * M + (m)) * D + (s))

  for (int oi = 0; oi < total && rc == 0; ++oi) {
    const int t = order[oi];
    const int* k = tasks + 6 * t;
    const int kind = k[0], p = k[1], m = k[2], s = k[3], wk = k[4];
    if (kind != 0 && kind != 1) continue;
    if (m >= M || s >= D) { rc = 2; break; }
    for (int r = 0; r < W && rc == 0; ++r) {
      const long key = KEY(r, p, m, s);
      const int in = dims[s], out = dims[s + 1];
      const double* w = params + L.w_off[s];
      if (kind == 0) { /* Engine::forward, oracle.cpp:202-242 */
        double* xi = (double*)malloc(sizeof(double) * B * maxd);
        double* yo = (double*)malloc(sizeof(double) * B * maxd);
        for (int i = 0; i < B; ++i) {
          const double* x;
          if (s == 0) {
            x = inputs + (long)((r * N + m) * B + i) * dims[0];
          } else {
            const double* up = st_out[KEY(r, p, m, s - 1)];
            if (!up) { rc = 3; break; }
            x = up + (long)i * maxd;
          }
          memcpy(xi + (long)i * maxd, x, sizeof(double) * in);
          stage_forward(w, params + L.b_off[s], x, yo + (long)i * maxd, out, in);
        }
        st_in[key] = xi;
        st_out[key] = yo;
        if (r == 0 && ++live[wk] > peak_stash[wk]) peak_stash[wk] = live[wk];
      } else { /* Engine::backward, oracle.cpp:244-280 */
        double* xi = st_in[key];
        double* yo = st_out[key];
        if (!xi) { rc = 3; break; }
        st_in[key] = st_out[key] = NULL;
        if (r == 0) --live[wk];
        double* down = (double*)malloc(sizeof(double) * B * maxd);
        kahan* acc = &g[r * P + p];
        kahan gw = view(acc, L.w_off[s]), gb = view(acc, L.b_off[s]);
        for (int i = 0; i < B; ++i) {
          if (s == D - 1) {
            const double* tg = targets + (long)((r * N + m) * B + i) * out;
            for (int o = 0; o < out; ++o) gy[o] = yo[(long)i * maxd + o] - tg[o];
          } else {
            if (!gin[key]) { rc = 3; break; }
            memcpy(gy, gin[key] + (long)i * maxd, sizeof(double) * out);
          }
          stage_backward(w, xi + (long)i * maxd, yo + (long)i * maxd, gy, out, in, scale, &gw,
                         &gb, down + (long)i * maxd);
        }
        free(gin[key]);
        gin[key] = NULL;
        if (s > 0) {
          free(gin[KEY(r, p, m, s - 1)]);
          gin[KEY(r, p, m, s - 1)] = down;
        } else {
          free(down);
        }
        free(xi);
        free(yo);
      }
    }
  }
#undef KEY
  if (rc == 0) {
    /* apply_stage_update for every stage (oracle.cpp:283-299,344-345) */
    for (int s = 0; s < D; ++s) {
      const long lo = L.w_off[s], hi = L.b_off[s] + dims[s + 1];
      for (long i = lo; i < hi; ++i) {
        double tot = 0.0;
        for (int r = 0; r < W; ++r)
          for (int p = 0; p < P; ++p) tot += g[r * P + p].v[i];
        params_out[i] = params[i] - lr * tot;
      }
    }
  }
  for (long i = 0; i < nkeys; ++i) { free(st_in[i]); free(st_out[i]); free(gin[i]); }
  free(st_in); free(st_out); free(gin); free(live); free(gy);
  grads_free(g, W * P);
  layout_free(&L);
  free(owner); free(local); free(st); free(en); free(order);
  return rc;
}

/* oracle.cpp:412-425 */
double toy_max_relative_diff(const int* dims, int n_dims, const double* a, const double* b) {
  long n = 0;
  for (int s = 0; s + 1 < n_dims; ++s) n += (long)dims[s] * dims[s + 1] + dims[s + 1];
  double worst = 0;
  for (long i = 0; i < n; ++i) {
    double den = fabs(a[i]);
    if (fabs(b[i]) > den) den = fabs(b[i]);
    if (den < 1e-9) den = 1e-9;
    const double r = fabs(a[i] - b[i]) / den;
    if (r > worst) worst = r;
  }
  return worst;
}

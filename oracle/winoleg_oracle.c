/* TEST INFRASTRUCTURE ONLY — CPU oracle for the quantized Winograd F(o,k) layer.
 *
 * A plain-C, fp64 restatement of the reference hot path, operation for operation, so that its
 * results are bit-identical to the reference's default (numba) backend:
 *
 *   fake_quant / compute_scale      reference quantize.py:103-126 (max-abs scale, rint = half-even,
 *                                   clip to +-qmax, +-qmax codes snap to +-max_abs)
 *   cast hook + StageStat           quantize.py:129-148, STAGE_BITS quantize.py:80-90
 *   run_pipeline stage order        pipeline.py:106-158 (crop before the final cast, :156-158)
 *   _extract_tiles / _scatter_tiles pipeline.py:79-99
 *   sandwich                        _kernels.py:69-92  tmp = X.R (l ascending), out = L.tmp (l ascending)
 *   hadamard_accumulate             _kernels.py:94-105 out += u*v, c ascending, from 0.0
 *
 * Compiled with -ffp-contract=off so no multiply-add is fused (numba's loops are unfused).
 * Extension beyond the reference (documented in DESIGN.md): a batch of n images whose stage
 * scales are shared by `images_per_group` consecutive images (1 == the reference's per-call
 * semantics applied per image).  Groups are independent and run on `nthreads` pthreads.
 *
 * Only tests/, bench.py's cpu-baseline leg and __graft_entry__.smoke may load this library.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { B_INPUT = 0, B_WEIGHTS, B_INPUT_T, B_WEIGHT_T, B_BASE, B_HADAMARD, B_OUTPUT };

typedef struct {
  int o, k, m;
  const double *G, *BT, *AT, *Pinv, *G_P, *BPT, *APT; /* row-major fp64 */
} plan_t;

static void unpack_plan(plan_t* p, const double* mats, int o, int k) {
  int m = o + k - 1;
  p->o = o;
  p->k = k;
  p->m = m;
  p->G = mats;
  p->BT = p->G + m * k;
  p->AT = p->BT + m * m;
  p->Pinv = p->AT + o * m;
  p->G_P = p->Pinv + m * m;
  p->BPT = p->G_P + m * k;
  p->APT = p->BPT + m * m;
}

/* quantize.py:103-126, applied in place; returns max_abs and writes scale/codes. */
static double fake_quant_inplace(double* a, size_t n, int bits, double* scale_out, int32_t* codes) {
  double mx = 0.0;
  for (size_t i = 0; i < n; ++i) {
    double v = fabs(a[i]);
    if (v > mx) mx = v;
  }
  const double q = (double)((1 << (bits - 1)) - 1);
  if (mx == 0.0) { /* all-zero: unchanged, scale 1.0 (quantize.py:108, :115-117) */
    *scale_out = 1.0;
    if (codes)
      for (size_t i = 0; i < n; ++i) codes[i] = 0;
    return 0.0;
  }
  const double s = mx / q;
  *scale_out = s;
  for (size_t i = 0; i < n; ++i) {
    double c = nearbyint(a[i] / s);
    if (c > q) c = q;
    if (c < -q) c = -q;
    if (codes) codes[i] = (int32_t)c;
    if (c == q)
      a[i] = mx;
    else if (c == -q)
      a[i] = -mx;
    else
      a[i] = c * s;
  }
  return mx;
}

/* _kernels.py:69-92 for one tile: out[a x d] = L[a x b] . X[b x c] . R[c x d], R given as R[c][d]. */
static void sandwich1(const double* L, int a, int b, const double* X, int c, const double* R, int d, double* tmp,
                      double* out) {
  for (int i = 0; i < b; ++i) {
    for (int j = 0; j < d; ++j) tmp[i * d + j] = 0.0;
    for (int l = 0; l < c; ++l) {
      const double v = X[i * c + l];
      for (int j = 0; j < d; ++j) tmp[i * d + j] += v * R[l * d + j];
    }
  }
  for (int i = 0; i < a; ++i) {
    for (int j = 0; j < d; ++j) out[i * d + j] = 0.0;
    for (int l = 0; l < b; ++l) {
      const double v = L[i * b + l];
      for (int j = 0; j < d; ++j) out[i * d + j] += v * tmp[l * d + j];
    }
  }
}

static void transpose(const double* M, int r, int c, double* Mt) {
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) Mt[j * r + i] = M[i * c + j];
}

/* sandwich over a batch of tiles with L and R = L^T (every stage of pipeline.py has that form) */
static void sandwich_batch(const double* L, int a, int b, const double* X, size_t ntiles, double* out) {
  double R[64 * 64], tmp[64 * 64];
  transpose(L, a, b, R); /* R is [b][a] */
  for (size_t t = 0; t < ntiles; ++t) sandwich1(L, a, b, X + t * b * b, b, R, a, tmp, out + t * a * a);
}

typedef struct {
  /* inputs */
  const double *x, *w;
  int n, cin, h, wd, cout, legendre;
  const int* bits;
  plan_t plan;
  /* precomputed weight side, shared by groups */
  const double* u;  /* [cout][cin][m][m] fake-quantized weight transform */
  /* per-group work */
  int g0, g1, ipg;
  double* y;
  double* stats; /* [ngroups][9][3] */
  int32_t** capture;
  int nstages;
  const double* wstats; /* weight stage stats: [nw][3] */
  int nw;
} job_t;

static void put_stat(double* st, int bits, double mx, double s) {
  st[0] = bits;
  st[1] = mx;
  st[2] = s;
}

/* Input half of run_pipeline for one group (pipeline.py:119, :121-123, :129-158). */
static void run_group(job_t* J, int g) {
  const plan_t* P = &J->plan;
  const int m = P->m, o = P->o, k = P->k, mm = m * m;
  const int n0 = g * J->ipg, ng = J->ipg;
  const int cin = J->cin, cout = J->cout, H = J->h, W = J->wd;
  const int oh = H - k + 1, ow = W - k + 1;
  const int th = (oh + o - 1) / o, tw = (ow + o - 1) / o, T = th * tw;
  const int hp = (th - 1) * o + m, wp = (tw - 1) * o + m;
  double* st = J->stats + (size_t)g * 9 * 3;
  int si = 0;
  double s;
  const int leg = J->legendre;
  const int* bits = J->bits;
  int32_t** cap = J->capture;

  /* cast("input") over the whole group tensor */
  size_t nx = (size_t)ng * cin * H * W;
  double* xq = (double*)malloc(nx * sizeof(double));
  memcpy(xq, J->x + (size_t)n0 * cin * H * W, nx * sizeof(double));
  int32_t* c_in = cap ? cap[0] + (size_t)n0 * cin * H * W : NULL;
  double mx = fake_quant_inplace(xq, nx, bits[B_INPUT], &s, c_in);
  put_stat(st + 3 * si++, bits[B_INPUT], mx, s);
  /* weight stats (identical for every group; computed once) */
  for (int i = 0; i < J->nw; ++i) memcpy(st + 3 * si++, J->wstats + 3 * i, 3 * sizeof(double));

  /* _extract_tiles: zero pad to hp x wp, m x m windows at stride o, tile index = ty*tw + tx */
  size_t ntile = (size_t)ng * cin * T;
  double* v = (double*)calloc(ntile * mm, sizeof(double));
  for (int im = 0; im < ng; ++im)
    for (int c = 0; c < cin; ++c) {
      const double* xs = xq + ((size_t)im * cin + c) * H * W;
      for (int ty = 0; ty < th; ++ty)
        for (int tx = 0; tx < tw; ++tx) {
          double* tl = v + (((size_t)im * cin + c) * T + ty * tw + tx) * mm;
          for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) {
              int r = ty * o + i, cc = tx * o + j;
              tl[i * m + j] = (r < H && cc < W) ? xs[(size_t)r * W + cc] : 0.0;
            }
        }
    }
  (void)hp;
  (void)wp;
  double* v2 = (double*)malloc(ntile * mm * sizeof(double));
  int stage_ix = leg ? 4 : 3; /* capture index of the next input-side stage */
  if (!leg) {
    sandwich_batch(P->BT, m, m, v, ntile, v2);
    mx = fake_quant_inplace(v2, ntile * mm, bits[B_INPUT_T], &s,
                            cap ? cap[stage_ix] + (size_t)n0 * cin * T * mm : NULL);
    put_stat(st + 3 * si++, bits[B_INPUT_T], mx, s);
  } else {
    double Pit[64];
    transpose(P->Pinv, m, m, Pit);
    sandwich_batch(Pit, m, m, v, ntile, v2); /* P^-T . X . P^-1 */
    mx = fake_quant_inplace(v2, ntile * mm, bits[B_BASE], &s, cap ? cap[4] + (size_t)n0 * cin * T * mm : NULL);
    put_stat(st + 3 * si++, bits[B_BASE], mx, s);
    sandwich_batch(P->BPT, m, m, v2, ntile, v); /* B_P^T . V . B_P */
    mx = fake_quant_inplace(v, ntile * mm, bits[B_INPUT_T], &s, cap ? cap[5] + (size_t)n0 * cin * T * mm : NULL);
    put_stat(st + 3 * si++, bits[B_INPUT_T], mx, s);
    double* t_ = v;
    v = v2;
    v2 = t_; /* quantized input transform now in v2 */
  }
  /* hadamard_accumulate: acc[im][o][t][ij] = sum_c u[o][c][ij] * v[im][c][t][ij], c ascending */
  size_t nacc = (size_t)ng * cout * T * mm;
  double* acc = (double*)calloc(nacc, sizeof(double));
  for (int im = 0; im < ng; ++im)
    for (int oc = 0; oc < cout; ++oc) {
      double* ao = acc + ((size_t)im * cout + oc) * T * mm;
      for (int c = 0; c < cin; ++c) {
        const double* uo = J->u + ((size_t)oc * cin + c) * mm;
        const double* vc = v2 + ((size_t)im * cin + c) * T * mm;
        for (int t = 0; t < T; ++t)
          for (int e = 0; e < mm; ++e) ao[(size_t)t * mm + e] += uo[e] * vc[(size_t)t * mm + e];
      }
    }
  int hix = leg ? 6 : 4;
  mx = fake_quant_inplace(acc, nacc, bits[B_HADAMARD], &s, cap ? cap[hix] + (size_t)n0 * cout * T * mm : NULL);
  put_stat(st + 3 * si++, bits[B_HADAMARD], mx, s);

  /* output transform */
  size_t nyt = (size_t)ng * cout * T * o * o;
  double* yt = (double*)malloc(nyt * sizeof(double));
  size_t nacc_t = (size_t)ng * cout * T;
  if (!leg) {
    sandwich_batch(P->AT, o, m, acc, nacc_t, yt);
  } else {
    double Pit[64];
    transpose(P->Pinv, m, m, Pit);
    double* mid = (double*)malloc(nacc * sizeof(double));
    sandwich_batch(Pit, m, m, acc, nacc_t, mid);
    mx = fake_quant_inplace(mid, nacc, bits[B_BASE], &s, cap ? cap[7] + (size_t)n0 * cout * T * mm : NULL);
    put_stat(st + 3 * si++, bits[B_BASE], mx, s);
    sandwich_batch(P->APT, o, m, mid, nacc_t, yt);
    free(mid);
  }
  /* _scatter_tiles + crop, then cast("output") */
  size_t ny = (size_t)ng * cout * oh * ow;
  double* y = J->y + (size_t)n0 * cout * oh * ow;
  for (int im = 0; im < ng; ++im)
    for (int oc = 0; oc < cout; ++oc)
      for (int r = 0; r < oh; ++r)
        for (int c = 0; c < ow; ++c) {
          int ty = r / o, tx = c / o;
          const double* tl = yt + (((size_t)im * cout + oc) * T + ty * tw + tx) * o * o;
          y[(((size_t)im * cout + oc) * oh + r) * ow + c] = tl[(r % o) * o + (c % o)];
        }
  int oix = leg ? 8 : 5;
  mx = fake_quant_inplace(y, ny, bits[B_OUTPUT], &s, cap ? cap[oix] + (size_t)n0 * cout * oh * ow : NULL);
  put_stat(st + 3 * si++, bits[B_OUTPUT], mx, s);
  free(xq);
  free(v);
  free(v2);
  free(acc);
  free(yt);
}

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  for (int g = J->g0; g < J->g1; ++g) run_group(J, g);
  return NULL;
}

/* Quantized Winograd correlation of x [n][cin][h][w] (already zero padded by the caller) with
 * w [cout][cin][k][k]; y [n][cout][h-k+1][w-k+1]; stats [n/ipg][9][3] = (bits, max_abs, scale)
 * in the reference's stage order (6 rows canonical, 9 Legendre).  `capture`, if non-NULL, holds
 * one int32 code buffer per stage index (see oracle.py for the layouts).  Returns 0 on success. */
int wlo_quant_conv(const double* x, int n, int cin, int h, int w, const double* wt, int cout, const double* mats,
                   int o, int k, int legendre, const int* bits, int images_per_group, double* y, double* stats,
                   int32_t** capture, int nthreads) {
  plan_t P;
  unpack_plan(&P, mats, o, k);
  const int m = P.m, mm = m * m;
  if (images_per_group <= 0 || n % images_per_group) return -1;
  if (h < k || w < k) return -2;
  /* weights side (pipeline.py:120, :124-137), computed once — identical for every group */
  size_t nw = (size_t)cout * cin * k * k;
  double* wq = (double*)malloc(nw * sizeof(double));
  memcpy(wq, wt, nw * sizeof(double));
  double wstats[3 * 3];
  int nws = 0;
  double s, mx;
  mx = fake_quant_inplace(wq, nw, bits[B_WEIGHTS], &s, capture ? capture[1] : NULL);
  put_stat(wstats + 3 * nws++, bits[B_WEIGHTS], mx, s);
  size_t nu = (size_t)cout * cin * mm;
  double* u = (double*)malloc(nu * sizeof(double));
  const double* Gl = legendre ? P.G_P : P.G;
  sandwich_batch(Gl, m, k, wq, (size_t)cout * cin, u);
  mx = fake_quant_inplace(u, nu, bits[B_WEIGHT_T], &s, capture ? capture[2] : NULL);
  put_stat(wstats + 3 * nws++, bits[B_WEIGHT_T], mx, s);
  if (legendre) {
    double* u2 = (double*)malloc(nu * sizeof(double));
    sandwich_batch(P.Pinv, m, m, u, (size_t)cout * cin, u2); /* P^-1 . U . P^-T */
    mx = fake_quant_inplace(u2, nu, bits[B_BASE], &s, capture ? capture[3] : NULL);
    put_stat(wstats + 3 * nws++, bits[B_BASE], mx, s);
    free(u);
    u = u2;
  }
  free(wq);
  /* The reference casts "input" before "weights" but the two are independent, so computing the
   * weight side first changes nothing but the order the stats are written (done per group). */
  const int ngroups = n / images_per_group;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > ngroups) nthreads = ngroups;
  job_t* jobs = (job_t*)calloc(nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc(nthreads, sizeof(pthread_t));
  for (int t = 0; t < nthreads; ++t) {
    job_t* J = &jobs[t];
    J->x = x;
    J->w = wt;
    J->n = n;
    J->cin = cin;
    J->h = h;
    J->wd = w;
    J->cout = cout;
    J->legendre = legendre;
    J->bits = bits;
    J->plan = P;
    J->u = u;
    J->ipg = images_per_group;
    J->g0 = (int)((long)ngroups * t / nthreads);
    J->g1 = (int)((long)ngroups * (t + 1) / nthreads);
    J->y = y;
    J->stats = stats;
    J->capture = capture;
    J->wstats = wstats;
    J->nw = nws;
  }
  /* the stats row order must follow the reference: input, weights, weight_transform, ... so the
     weight rows are placed after "input" inside run_group. */
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, &jobs[t]);
  worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(jobs);
  free(th);
  free(u);
  return 0;
}

/* fake_quant on a flat array (quantize.py:112-126); returns max_abs, writes scale. */
double wlo_fake_quant(double* a, long n, int bits, double* scale, int32_t* codes) {
  return fake_quant_inplace(a, (size_t)n, bits, scale, codes);
}

/* Float (identity-cast) pipeline for one image: pipeline.py:161-164 (used by tests of the
 * float path).  Implemented as the quantized path with casts disabled is not possible in this
 * file's structure, so it is left to the Python oracle; exported symbol kept minimal. */

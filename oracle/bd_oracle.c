/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the blockwise-distillation step.
 * See bd_oracle.h for what it restates and DESIGN.md §3 for the numerics
 * contract shared with the GPU path.  Deterministic for any OpenMP thread
 * count: every parallel loop owns its outputs; every reduction is accumulated
 * in double in a fixed order.
 */
#include "bd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static const int T_CH[5] = {3, 64, 128, 256, 512};
static const int T_HW[5] = {32, 32, 16, 8, 4};
static const float BN_EPS = 1e-5f;

int bdo_in_channels(int k) { return T_CH[k]; }
int bdo_out_channels(int k) { return T_CH[k + 1]; }
int bdo_in_hw(int k) { return T_HW[k]; }
int bdo_out_hw(int k) { return T_HW[k + 1]; }

int bdo_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------ bf16 / philox */
float bdo_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) { /* inf / nan */
    if (u & 0x007FFFFFu) u |= 0x00400000u;
    u &= 0xFFFF0000u;
  } else {
    const uint32_t lsb = (u >> 16) & 1u;
    u = (u + 0x7FFFu + lsb) & 0xFFFF0000u;
  }
  float r;
  memcpy(&r, &u, 4);
  return r;
}

static inline float rnd(float x, int bf16) { return bf16 ? bdo_bf16(x) : x; }

void bdo_philox(const uint32_t c_in[4], const uint32_t k_in[2], uint32_t out[4]) {
  uint32_t c0 = c_in[0], c1 = c_in[1], c2 = c_in[2], c3 = c_in[3];
  uint32_t k0 = k_in[0], k1 = k_in[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* uniform in [-1, 1): (u >> 8) * 2^-24 * 2 - 1, exact in fp32 */
static inline float sym_unit(uint32_t u) { return 2.0f * ((float)(u >> 8) * (1.0f / 16777216.0f)) - 1.0f; }

void bdo_input(int n, int64_t first, uint32_t seed, float* out, int bf16) {
  const int64_t per = 32 * 32 * 3;
  const uint32_t key[2] = {seed, 0xDA7A0000u};
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    for (int64_t e = 0; e < per; ++e) {
      const uint64_t idx = (uint64_t)(first + i) * (uint64_t)per + (uint64_t)e;
      const uint32_t ctr[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), 0u, 0u};
      uint32_t o[4];
      bdo_philox(ctr, key, o);
      out[(int64_t)i * per + e] = rnd(sym_unit(o[0]), bf16);
    }
  }
}

static void fill_uniform(float* dst, size_t count, uint32_t seed, uint32_t tensor_id, float bound, int bf16) {
  const uint32_t key[2] = {seed, 0xB200B200u};
  for (size_t i = 0; i < count; ++i) {
    const uint32_t ctr[4] = {(uint32_t)i, tensor_id, 0u, 0u};
    uint32_t o[4];
    bdo_philox(ctr, key, o);
    dst[i] = rnd(sym_unit(o[0]) * bound, bf16);
  }
}

static float kaiming_bound(int fan_in, float gain) { return sqrtf(6.0f / (float)fan_in) * gain; }

/* ------------------------------------------------------------------ teacher program */
typedef struct {
  int cin, cout, r, stride, pad, in_hw, out_hw;
  float gain;
} conv_spec;

/* Convs of teacher block k in program order: [stem], per BasicBlock: conv1, conv2, [proj]. */
static int teacher_convs(int k, conv_spec* cs) {
  int n = 0;
  int cin = T_CH[k];
  int hw = T_HW[k];
  if (k == 0) {
    cs[n++] = (conv_spec){3, 64, 3, 1, 1, 32, 32, 1.0f};
    cin = 64;
  }
  const int cout = T_CH[k + 1];
  const int s = T_HW[k] / T_HW[k + 1];
  for (int b = 0; b < 2; ++b) {
    const int st = b == 0 ? s : 1;
    const int ci = b == 0 ? cin : cout;
    const int ohw = hw / st;
    cs[n++] = (conv_spec){ci, cout, 3, st, 1, hw, ohw, 1.0f};
    cs[n++] = (conv_spec){cout, cout, 3, 1, 1, ohw, ohw, 0.5f};
    if (st != 1 || ci != cout) cs[n++] = (conv_spec){ci, cout, 1, st, 0, hw, ohw, 1.0f};
    hw = ohw;
  }
  return n;
}

static size_t conv_params(const conv_spec* c) { return (size_t)c->cout * c->r * c->r * c->cin + (size_t)c->cout; }

size_t bdo_teacher_param_count(int k) {
  conv_spec cs[8];
  const int n = teacher_convs(k, cs);
  size_t t = 0;
  for (int i = 0; i < n; ++i) t += conv_params(&cs[i]);
  return t;
}

void bdo_teacher_init(int k, uint32_t seed, float* p, int bf16) {
  conv_spec cs[8];
  const int n = teacher_convs(k, cs);
  for (int j = 0; j < n; ++j) {
    const size_t wn = (size_t)cs[j].cout * cs[j].r * cs[j].r * cs[j].cin;
    fill_uniform(p, wn, seed, (uint32_t)(1000 * k + 10 * j), kaiming_bound(cs[j].cin * cs[j].r * cs[j].r, cs[j].gain),
                 bf16);
    p += wn;
    /* biases stay fp32 on the GPU (epilogue operand) */
    fill_uniform(p, (size_t)cs[j].cout, seed, (uint32_t)(1000 * k + 10 * j + 1), 0.1f, 0);
    p += cs[j].cout;
  }
}

/* ------------------------------------------------------------------ conv kernels (NHWC, W[K][R][S][C]) */
static inline float dot(const float* a, const float* b, int n) {
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int i = 0;
  for (; i + 8 <= n; i += 8)
    for (int l = 0; l < 8; ++l) acc[l] += a[i + l] * b[i + l];
  float s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  for (; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* y[n,p,q,k] = sum_{r,s,c} x[n, p*st+r-pad, q*st+s-pad, c] w[k,r,s,c] */
static void conv_fwd(const float* x, int N, int H, int W, int C, const float* w, int K, int R, int st, int pad,
                     int P, int Q, float* y) {
#pragma omp parallel for schedule(static)
  for (int np = 0; np < N * P; ++np) {
    const int n = np / P, p = np % P;
    for (int q = 0; q < Q; ++q) {
      float* out = y + (((size_t)n * P + p) * Q + q) * K;
      for (int k = 0; k < K; ++k) {
        float acc = 0.0f;
        for (int r = 0; r < R; ++r) {
          const int h = p * st + r - pad;
          if (h < 0 || h >= H) continue;
          for (int s = 0; s < R; ++s) {
            const int ww = q * st + s - pad;
            if (ww < 0 || ww >= W) continue;
            acc += dot(x + (((size_t)n * H + h) * W + ww) * C, w + (((size_t)k * R + r) * R + s) * C, C);
          }
        }
        out[k] = acc;
      }
    }
  }
}

/* dw[k,r,s,c] = sum_{n,p,q} dy[n,p,q,k] x[n, p*st+r-pad, q*st+s-pad, c]   (double accumulation) */
static void conv_wgrad(const float* x, int N, int H, int W, int C, const float* dy, int K, int R, int st, int pad,
                       int P, int Q, float* dw) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int k = 0; k < K; ++k) {
    double* acc = (double*)calloc((size_t)R * R * C, sizeof(double));
    for (int n = 0; n < N; ++n)
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < Q; ++q) {
          const double g = dy[(((size_t)n * P + p) * Q + q) * K + k];
          if (g == 0.0) continue;
          for (int r = 0; r < R; ++r) {
            const int h = p * st + r - pad;
            if (h < 0 || h >= H) continue;
            for (int s = 0; s < R; ++s) {
              const int ww = q * st + s - pad;
              if (ww < 0 || ww >= W) continue;
              const float* xs = x + (((size_t)n * H + h) * W + ww) * C;
              double* a = acc + ((size_t)r * R + s) * C;
              for (int c = 0; c < C; ++c) a[c] += g * xs[c];
            }
          }
        }
    for (size_t i = 0; i < (size_t)R * R * C; ++i) dw[(size_t)k * R * R * C + i] = (float)acc[i];
    free(acc);
  }
}

/* dx[n,h,w,c] = sum_{k,r,s} dy[n,h-r+pad,w-s+pad,k] w[k,r,s,c]   (stride 1 only) */
static void conv_dgrad_s1(const float* dy, int N, int H, int W, int K, const float* w, int C, int R, int pad,
                          float* dx) {
  float* wt = (float*)malloc(sizeof(float) * (size_t)R * R * C * K); /* wt[r][s][c][k] */
  for (int k = 0; k < K; ++k)
    for (int r = 0; r < R; ++r)
      for (int s = 0; s < R; ++s)
        for (int c = 0; c < C; ++c) wt[(((size_t)r * R + s) * C + c) * K + k] = w[(((size_t)k * R + r) * R + s) * C + c];
#pragma omp parallel for schedule(static)
  for (int nh = 0; nh < N * H; ++nh) {
    const int n = nh / H, h = nh % H;
    for (int ww = 0; ww < W; ++ww) {
      float* out = dx + (((size_t)n * H + h) * W + ww) * C;
      for (int c = 0; c < C; ++c) {
        float acc = 0.0f;
        for (int r = 0; r < R; ++r) {
          const int p = h - r + pad;
          if (p < 0 || p >= H) continue;
          for (int s = 0; s < R; ++s) {
            const int q = ww - s + pad;
            if (q < 0 || q >= W) continue;
            acc += dot(dy + (((size_t)n * H + p) * W + q) * K, wt + (((size_t)r * R + s) * C + c) * K, K);
          }
        }
        out[c] = acc;
      }
    }
  }
  free(wt);
}

/* ------------------------------------------------------------------ teacher forward */
static void bias_act(float* y, size_t m, int K, const float* b, const float* res, int relu, int bf16) {
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)m; ++i) {
    for (int k = 0; k < K; ++k) {
      float v = y[(size_t)i * K + k] + b[k];
      if (res) v += res[(size_t)i * K + k];
      if (relu) v = v > 0.0f ? v : 0.0f;
      y[(size_t)i * K + k] = rnd(v, bf16);
    }
  }
}

int bdo_teacher_fwd(int k, const float* tp, int n, const float* in, float* out, int bf16) {
  conv_spec cs[8];
  const int nc = teacher_convs(k, cs);
  size_t maxel = (size_t)n * 32 * 32 * 64 * 2;
  float* a = (float*)malloc(sizeof(float) * maxel);
  float* h = (float*)malloc(sizeof(float) * maxel);
  float* sc = (float*)malloc(sizeof(float) * maxel);
  float* o = (float*)malloc(sizeof(float) * maxel);
  int j = 0;
  int hw = T_HW[k];
  int C = T_CH[k];
  memcpy(a, in, sizeof(float) * (size_t)n * hw * hw * C);
  if (k == 0) {
    const conv_spec* c = &cs[j];
    conv_fwd(a, n, 32, 32, 3, tp, 64, 3, 1, 1, 32, 32, h);
    bias_act(h, (size_t)n * 32 * 32, 64, tp + (size_t)64 * 27, NULL, 1, bf16);
    tp += conv_params(c);
    ++j;
    memcpy(a, h, sizeof(float) * (size_t)n * 32 * 32 * 64);
    C = 64;
  }
  for (int b = 0; b < 2; ++b) {
    const conv_spec* c1 = &cs[j++];
    const conv_spec* c2 = &cs[j++];
    const int proj = (c1->stride != 1 || c1->cin != c1->cout);
    const conv_spec* cp = proj ? &cs[j++] : NULL;
    const int P = c1->out_hw;
    const size_t m = (size_t)n * P * P;
    const float* w1 = tp;
    const float* b1 = w1 + (size_t)c1->cout * 9 * c1->cin;
    const float* w2 = tp + conv_params(c1);
    const float* b2 = w2 + (size_t)c2->cout * 9 * c2->cin;
    const float* wp = proj ? w2 + conv_params(c2) : NULL;
    const float* bp = proj ? wp + (size_t)cp->cout * cp->cin : NULL;
    conv_fwd(a, n, hw, hw, C, w1, c1->cout, 3, c1->stride, 1, P, P, h);
    bias_act(h, m, c1->cout, b1, NULL, 1, bf16);
    const float* res = a;
    if (proj) {
      conv_fwd(a, n, hw, hw, C, wp, cp->cout, 1, cp->stride, 0, P, P, sc);
      bias_act(sc, m, cp->cout, bp, NULL, 0, bf16);
      res = sc;
    }
    conv_fwd(h, n, P, P, c1->cout, w2, c2->cout, 3, 1, 1, P, P, o);
    bias_act(o, m, c2->cout, b2, res, 1, bf16);
    tp += conv_params(c1) + conv_params(c2) + (proj ? conv_params(cp) : 0);
    memcpy(a, o, sizeof(float) * m * c2->cout);
    hw = P;
    C = c2->cout;
  }
  memcpy(out, a, sizeof(float) * (size_t)n * hw * hw * C);
  free(a);
  free(h);
  free(sc);
  free(o);
  (void)nc;
  return 0;
}

/* ------------------------------------------------------------------ student */
typedef struct {
  int cin, cout, mid, stride, hin, hout;
  size_t w1, w2, wsc, g1, b1, g2, b2, gsc, bsc, total; /* offsets */
} student_geom;

static student_geom sgeom(int k) {
  student_geom g;
  g.cin = T_CH[k];
  g.cout = T_CH[k + 1];
  g.mid = g.cout / 2;
  g.hin = T_HW[k];
  g.hout = T_HW[k + 1];
  g.stride = g.hin / g.hout;
  size_t o = 0;
  g.w1 = o;
  o += (size_t)g.mid * 9 * g.cin;
  g.w2 = o;
  o += (size_t)g.cout * 9 * g.mid;
  g.wsc = o;
  o += (size_t)g.cout * g.cin;
  g.g1 = o;
  o += g.mid;
  g.b1 = o;
  o += g.mid;
  g.g2 = o;
  o += g.cout;
  g.b2 = o;
  o += g.cout;
  g.gsc = o;
  o += g.cout;
  g.bsc = o;
  o += g.cout;
  g.total = o;
  return g;
}

size_t bdo_student_param_count(int k) { return sgeom(k).total; }

void bdo_student_init(int k, uint32_t seed, float* p) {
  const student_geom g = sgeom(k);
  fill_uniform(p + g.w1, (size_t)g.mid * 9 * g.cin, seed, (uint32_t)(10 * k + 0), kaiming_bound(9 * g.cin, 1.0f), 0);
  fill_uniform(p + g.w2, (size_t)g.cout * 9 * g.mid, seed, (uint32_t)(10 * k + 1), kaiming_bound(9 * g.mid, 1.0f), 0);
  fill_uniform(p + g.wsc, (size_t)g.cout * g.cin, seed, (uint32_t)(10 * k + 2), kaiming_bound(g.cin, 1.0f), 0);
  for (int i = 0; i < g.mid; ++i) {
    p[g.g1 + i] = 1.0f;
    p[g.b1 + i] = 0.0f;
  }
  for (int i = 0; i < g.cout; ++i) {
    p[g.g2 + i] = 1.0f;
    p[g.b2 + i] = 0.0f;
    p[g.gsc + i] = 1.0f;
    p[g.bsc + i] = 0.0f;
  }
}

/* per-channel batch statistics: mean and biased variance (double sums). */
static void bn_stats(const float* y, size_t m, int C, float* mean, float* rstd) {
#pragma omp parallel for schedule(static)
  for (int c = 0; c < C; ++c) {
    double s1 = 0.0, s2 = 0.0;
    for (size_t i = 0; i < m; ++i) {
      const double v = y[i * C + c];
      s1 += v;
      s2 += v * v;
    }
    const double mu = s1 / (double)m;
    const double var = s2 / (double)m - mu * mu;
    mean[c] = (float)mu;
    rstd[c] = 1.0f / sqrtf((float)var + BN_EPS);
  }
}

/* shadow copy of a master weight in the GEMM operand precision */
static float* shadow(const float* w, size_t n, int bf16) {
  float* s = (float*)malloc(sizeof(float) * n);
  for (size_t i = 0; i < n; ++i) s[i] = rnd(w[i], bf16);
  return s;
}

int bdo_student_fwd_bwd(int k, const float* sp, int n, const float* in, const float* t_out, double norm, int bf16,
                        float* grads, double* loss_out) {
  const student_geom g = sgeom(k);
  const int P = g.hout;
  const size_t m = (size_t)n * P * P;
  float* w1 = shadow(sp + g.w1, (size_t)g.mid * 9 * g.cin, bf16);
  float* w2 = shadow(sp + g.w2, (size_t)g.cout * 9 * g.mid, bf16);
  float* wsc = shadow(sp + g.wsc, (size_t)g.cout * g.cin, bf16);
  float* y1 = (float*)malloc(sizeof(float) * m * g.mid);
  float* a1 = (float*)malloc(sizeof(float) * m * g.mid);
  float* y2 = (float*)malloc(sizeof(float) * m * g.cout);
  float* ys = (float*)malloc(sizeof(float) * m * g.cout);
  float* dy2 = (float*)malloc(sizeof(float) * m * g.cout);
  float* dys = (float*)malloc(sizeof(float) * m * g.cout);
  float* g1 = (float*)malloc(sizeof(float) * m * g.mid);
  float *mu1 = malloc(sizeof(float) * g.mid), *r1 = malloc(sizeof(float) * g.mid);
  float *mu2 = malloc(sizeof(float) * g.cout), *r2 = malloc(sizeof(float) * g.cout);
  float *mus = malloc(sizeof(float) * g.cout), *rs = malloc(sizeof(float) * g.cout);

  /* forward */
  conv_fwd(in, n, g.hin, g.hin, g.cin, w1, g.mid, 3, g.stride, 1, P, P, y1);
  for (size_t i = 0; i < m * g.mid; ++i) y1[i] = rnd(y1[i], bf16);
  bn_stats(y1, m, g.mid, mu1, r1);
  const float* G1 = sp + g.g1;
  const float* B1 = sp + g.b1;
  /* BN as a per-channel affine map: A = gamma*rstd, B = beta - A*mean */
  float* A1 = (float*)malloc(sizeof(float) * g.mid);
  float* C1 = (float*)malloc(sizeof(float) * g.mid);
  for (int c = 0; c < g.mid; ++c) {
    A1[c] = G1[c] * r1[c];
    C1[c] = fmaf(-A1[c], mu1[c], B1[c]);
  }
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)m; ++i)
    for (int c = 0; c < g.mid; ++c) {
      const float z = fmaf(A1[c], y1[i * g.mid + c], C1[c]);
      a1[i * g.mid + c] = rnd(z > 0.0f ? z : 0.0f, bf16);
    }
  conv_fwd(a1, n, P, P, g.mid, w2, g.cout, 3, 1, 1, P, P, y2);
  conv_fwd(in, n, g.hin, g.hin, g.cin, wsc, g.cout, 1, g.stride, 0, P, P, ys);
  for (size_t i = 0; i < m * g.cout; ++i) {
    y2[i] = rnd(y2[i], bf16);
    ys[i] = rnd(ys[i], bf16);
  }
  bn_stats(y2, m, g.cout, mu2, r2);
  bn_stats(ys, m, g.cout, mus, rs);

  /* loss + relu backward + BN2/BNsc backward.  Both BNs are per-channel affine maps
   * z = A2*y2 + As*ysc + (B2 + Bsc); the backward needs sum g, sum g*y2, sum g*ysc, from which
   * sum g*xhat = rstd * (sum g*y - mean * sum g), and dy = A*g + Q*y + R. */
  const float* G2 = sp + g.g2;
  const float* B2 = sp + g.b2;
  const float* Gs = sp + g.gsc;
  const float* Bs = sp + g.bsc;
  float *A2 = malloc(sizeof(float) * g.cout), *As = malloc(sizeof(float) * g.cout), *Bz = malloc(sizeof(float) * g.cout);
  for (int c = 0; c < g.cout; ++c) {
    A2[c] = G2[c] * r2[c];
    As[c] = Gs[c] * rs[c];
    Bz[c] = fmaf(-A2[c], mu2[c], B2[c]) + fmaf(-As[c], mus[c], Bs[c]);
  }
  const float gscale = (float)(2.0 / norm);
  double* part = (double*)calloc((size_t)n * (1 + 3 * (size_t)g.cout), sizeof(double));
#pragma omp parallel for schedule(static)
  for (int s = 0; s < n; ++s) {
    double* ps = part + (size_t)s * (1 + 3 * (size_t)g.cout);
    for (int pq = 0; pq < P * P; ++pq) {
      const size_t i = (size_t)s * P * P + pq;
      for (int c = 0; c < g.cout; ++c) {
        const float v2 = y2[i * g.cout + c], vs = ys[i * g.cout + c];
        const float z = fmaf(A2[c], v2, fmaf(As[c], vs, Bz[c]));
        const float sv = z > 0.0f ? z : 0.0f;
        const float d = sv - t_out[i * g.cout + c];
        ps[0] += (double)d * (double)d;
        const float gg = z > 0.0f ? d * gscale : 0.0f;
        ps[1 + c] += gg;
        ps[1 + g.cout + c] += (double)gg * v2;
        ps[1 + 2 * g.cout + c] += (double)gg * vs;
      }
    }
  }
  double loss = 0.0;
  double* red = (double*)calloc(3 * (size_t)g.cout, sizeof(double));
  for (int s = 0; s < n; ++s) {
    const double* ps = part + (size_t)s * (1 + 3 * (size_t)g.cout);
    loss += ps[0];
    for (int c = 0; c < 3 * g.cout; ++c) red[c] += ps[1 + c];
  }
  *loss_out = loss / norm;
  float* gr = grads;
  memset(gr, 0, sizeof(float) * g.total);
  float *Q2 = malloc(sizeof(float) * g.cout), *R2 = malloc(sizeof(float) * g.cout);
  float *Qs = malloc(sizeof(float) * g.cout), *Rs = malloc(sizeof(float) * g.cout);
  for (int c = 0; c < g.cout; ++c) {
    const double sgv = red[c];
    const double sgx2 = (double)r2[c] * (red[g.cout + c] - (double)mu2[c] * sgv);
    const double sgxs = (double)rs[c] * (red[2 * g.cout + c] - (double)mus[c] * sgv);
    gr[g.b2 + c] = (float)sgv;
    gr[g.bsc + c] = (float)sgv;
    gr[g.g2 + c] = (float)sgx2;
    gr[g.gsc + c] = (float)sgxs;
    const double c2 = (double)A2[c] / (double)m, cs = (double)As[c] / (double)m;
    Q2[c] = (float)(-c2 * sgx2 * (double)r2[c]);
    R2[c] = (float)(-c2 * (sgv - sgx2 * (double)r2[c] * (double)mu2[c]));
    Qs[c] = (float)(-cs * sgxs * (double)rs[c]);
    Rs[c] = (float)(-cs * (sgv - sgxs * (double)rs[c] * (double)mus[c]));
  }
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)m; ++i)
    for (int c = 0; c < g.cout; ++c) {
      const float v2 = y2[i * g.cout + c], vs = ys[i * g.cout + c];
      const float z = fmaf(A2[c], v2, fmaf(As[c], vs, Bz[c]));
      const float sv = z > 0.0f ? z : 0.0f;
      const float d = sv - t_out[i * g.cout + c];
      const float gg = z > 0.0f ? d * gscale : 0.0f;
      dy2[i * g.cout + c] = rnd(fmaf(A2[c], gg, fmaf(Q2[c], v2, R2[c])), bf16);
      dys[i * g.cout + c] = rnd(fmaf(As[c], gg, fmaf(Qs[c], vs, Rs[c])), bf16);
    }
  free(A2);
  free(As);
  free(Bz);
  free(Q2);
  free(R2);
  free(Qs);
  free(Rs);

  /* conv2 / shortcut weight gradients, conv2 dgrad with the relu mask of a1 */
  conv_wgrad(a1, n, P, P, g.mid, dy2, g.cout, 3, 1, 1, P, P, gr + g.w2);
  conv_wgrad(in, n, g.hin, g.hin, g.cin, dys, g.cout, 1, g.stride, 0, P, P, gr + g.wsc);
  conv_dgrad_s1(dy2, n, P, P, g.cout, w2, g.mid, 3, 1, g1);
  for (size_t i = 0; i < m * g.mid; ++i) g1[i] = rnd(a1[i] > 0.0f ? g1[i] : 0.0f, bf16);

  /* BN1 backward: sums of g1 and g1*y1, then dy1 = A1*g1 + Q1*y1 + R1 */
  double* red1 = (double*)calloc(2 * (size_t)g.mid, sizeof(double));
#pragma omp parallel for schedule(static)
  for (int c = 0; c < g.mid; ++c) {
    double sg = 0.0, sgy = 0.0;
    for (size_t i = 0; i < m; ++i) {
      const double gv = g1[i * g.mid + c];
      sg += gv;
      sgy += gv * y1[i * g.mid + c];
    }
    red1[c] = sg;
    red1[g.mid + c] = sgy;
  }
  float *Q1 = malloc(sizeof(float) * g.mid), *R1 = malloc(sizeof(float) * g.mid);
  for (int c = 0; c < g.mid; ++c) {
    const double sgv = red1[c];
    const double sgx = (double)r1[c] * (red1[g.mid + c] - (double)mu1[c] * sgv);
    gr[g.b1 + c] = (float)sgv;
    gr[g.g1 + c] = (float)sgx;
    const double c1 = (double)A1[c] / (double)m;
    Q1[c] = (float)(-c1 * sgx * (double)r1[c]);
    R1[c] = (float)(-c1 * (sgv - sgx * (double)r1[c] * (double)mu1[c]));
  }
  float* dy1 = a1; /* reuse */
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)m; ++i)
    for (int c = 0; c < g.mid; ++c)
      dy1[i * g.mid + c] = rnd(fmaf(A1[c], g1[i * g.mid + c], fmaf(Q1[c], y1[i * g.mid + c], R1[c])), bf16);
  free(Q1);
  free(R1);
  free(A1);
  free(C1);
  conv_wgrad(in, n, g.hin, g.hin, g.cin, dy1, g.mid, 3, g.stride, 1, P, P, gr + g.w1);

  free(w1);
  free(w2);
  free(wsc);
  free(y1);
  free(a1);
  free(y2);
  free(ys);
  free(dy2);
  free(dys);
  free(g1);
  free(mu1);
  free(r1);
  free(mu2);
  free(r2);
  free(mus);
  free(rs);
  free(part);
  free(red);
  free(red1);
  return 0;
}

void bdo_sgd(size_t count, float* w, float* v, const float* g, float lr, float mu) {
  for (size_t i = 0; i < count; ++i) {
    v[i] = fmaf(mu, v[i], g[i]);
    w[i] = fmaf(-lr, v[i], w[i]);
  }
}

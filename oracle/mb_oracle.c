/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle of the MobileNetV2 -> ProxylessNAS blockwise-distillation
 * step (mb_oracle.h; numerics contract DESIGN.md §10).  Deterministic for any OpenMP thread count:
 * every parallel loop owns its outputs; every reduction runs in double in a fixed order.
 */
#include "mb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "bd_oracle.h" /* bdo_philox, bdo_bf16 */

static const float BN_EPS = 1e-5f;

static inline float rnd(float x, int bf16) { return bf16 ? bdo_bf16(x) : x; }
static inline float sym_unit(uint32_t u) { return 2.0f * ((float)(u >> 8) * (1.0f / 16777216.0f)) - 1.0f; }
static inline float relu6(float z) { return z > 0.0f ? (z < 6.0f ? z : 6.0f) : 0.0f; }
static inline int mask6(float a) { return a > 0.0f && a < 6.0f; }

/* ------------------------------------------------------------------ architecture */
typedef struct {
  int t, k, cin, cout, stride; /* teacher: expansion t (1 = no expand conv), kernel k; stored widths */
  int cin_t, cout_t;           /* the architecture's true widths (<= stored; the rest are zero channels) */
} mb_layer;

/* teacher families: 0 = MobileNetV2 (ReLU6), 1 = EfficientNet-B0 (swish + squeeze-excite) */
static int FAM = 0;
/* boundary widths: stored (tensor-tile granularity) and true (MobileNetV2-1.0 / EfficientNet-B0).
 * Channels beyond the true width are stored but identically zero: their weights are initialised to
 * zero and receive zero gradients, so the model computed is exactly the true-width network
 * (DESIGN.md §10). */
static const int CHF[2][7] = {{3, 32, 32, 64, 128, 192, 320}, {3, 32, 64, 128, 128, 192, 320}};
static const int CTF[2][7] = {{3, 24, 32, 64, 96, 160, 320}, {3, 24, 40, 80, 112, 192, 320}};
static const int NLF[2][6] = {{3, 3, 4, 3, 3, 1}, {3, 2, 3, 3, 4, 1}}; /* teacher MBConv layers per block */
static const int KF[2][6] = {{3, 3, 3, 3, 3, 3}, {3, 5, 3, 5, 5, 3}};  /* teacher kernel per block */
#define CH (CHF[FAM])
#define CT (CTF[FAM])
#define NL (NLF[FAM])
static const int DIV[7] = {1, 4, 8, 16, 16, 32, 32};

void mbo_set_family(int f) { FAM = (f == 1) ? 1 : 0; }
int mbo_family(void) { return FAM; }

static int teacher_layer(int b, int l, mb_layer* o) {
  static const mb_layer B0[3] = {{1, 3, 32, 16, 1, 32, 16}, {6, 3, 16, 32, 2, 16, 24}, {6, 3, 32, 32, 1, 24, 24}};
  if (l < 0 || l >= NL[b]) return 0;
  if (b == 0) {
    *o = B0[l];
    return 1;
  }
  const int cin = CH[b], cout = CH[b + 1];
  const int s = DIV[b + 1] / DIV[b];
  const int k = KF[FAM][b];
  *o = l == 0 ? (mb_layer){6, k, cin, cout, s, CT[b], CT[b + 1]} : (mb_layer){6, k, cout, cout, 1, CT[b + 1], CT[b + 1]};
  return 1;
}

/* squeeze-excite width of an EfficientNet layer (0.25 x the layer's input channels): stored / true */
static int se_ch(const mb_layer* m) { return FAM == 1 ? (m->cin / 4 > 0 ? m->cin / 4 : 1) : 0; }
static int se_ch_t(const mb_layer* m) { return FAM == 1 ? (m->cin_t / 4 > 0 ? m->cin_t / 4 : 1) : 0; }
/* a residual joins input and output when the stride is 1 and the TRUE widths agree */
static int has_res(const mb_layer* m) { return m->stride == 1 && m->cin_t == m->cout_t; }
static inline float swishf(float z) { return z / (1.0f + expf(-z)); }
static inline float sigmoidf(float z) { return 1.0f / (1.0f + expf(-z)); }
/* the teacher's activation: ReLU6 (MobileNetV2) or swish (EfficientNet-B0) */
static inline float tact(float z) {
  if (FAM == 1) return swishf(z);
  return z > 0.0f ? (z < 6.0f ? z : 6.0f) : 0.0f;
}

static int round_ch(int c) { return c <= 16 ? 16 : c <= 32 ? 32 : (c + 63) / 64 * 64; }
static int expand_ch(int cin, int t) { return t == 1 ? cin : round_ch(cin * t); }
static int expand_ch_t(int cin_t, int t) { return t == 1 ? cin_t : cin_t * t; }

int mbo_channels(int b) { return CH[b]; }
int mbo_true_channels(int b) { return CT[b]; }
int mbo_hw(int b, int S) { return S / DIV[b]; }

/* student layers: block 0 = [stem, MBConv1 (fixed), searchable...]; others all searchable */
int mbo_student_layers(int b) { return NL[b] + (b == 0 ? 1 : 0); }
int mbo_layer_candidates(int b, int l) { return (b == 0 && l < 2) ? 1 : MBO_CANDIDATES; }

static void cand_ke(int b, int l, int c, int* k, int* e) {
  if (b == 0 && l < 2) {
    *k = 3;
    *e = 1;
    return;
  }
  static const int KS[3] = {3, 5, 7}, ES[2] = {3, 6};
  *k = KS[c % 3];
  *e = ES[c / 3];
}

/* student MB layer l (block 0: l >= 1) geometry */
static mb_layer student_mb(int b, int l) {
  mb_layer t;
  teacher_layer(b, b == 0 ? l - 1 : l, &t);
  return t;
}

typedef struct {
  size_t we, wd, wp, g1, b1, g2, b2, g3, b3, total;
  int E, k, e;
  int Et; /* true expanded width */
} cand_layout;

static cand_layout cand_lay(int b, int l, int c) {
  cand_layout L;
  memset(&L, 0, sizeof(L));
  if (b == 0 && l == 0) { /* stem: w[32][3][3][16 stored], g, b */
    L.wd = 0;
    L.g2 = 32 * 9 * 16;
    L.b2 = L.g2 + 32;
    L.total = L.b2 + 32;
    L.E = 32;
    L.Et = 32;
    L.k = 3;
    L.e = 0;
    return L;
  }
  const mb_layer m = student_mb(b, l);
  cand_ke(b, l, c, &L.k, &L.e);
  L.E = expand_ch(m.cin, L.e);
  L.Et = expand_ch_t(m.cin_t, L.e);
  size_t o = 0;
  if (L.e != 1) {
    L.we = o;
    o += (size_t)L.E * m.cin;
  }
  L.wd = o;
  o += (size_t)L.E * L.k * L.k;
  L.wp = o;
  o += (size_t)m.cout * L.E;
  if (L.e != 1) {
    L.g1 = o;
    o += L.E;
    L.b1 = o;
    o += L.E;
  }
  L.g2 = o;
  o += L.E;
  L.b2 = o;
  o += L.E;
  L.g3 = o;
  o += m.cout;
  L.b3 = o;
  o += m.cout;
  L.total = o;
  return L;
}

size_t mbo_candidate_offset(int b, int l, int cand, size_t* count) {
  size_t off = 0;
  for (int i = 0; i < mbo_student_layers(b); ++i)
    for (int c = 0; c < mbo_layer_candidates(b, i); ++c) {
      const cand_layout L = cand_lay(b, i, c);
      if (i == l && c == cand) {
        if (count) *count = L.total;
        return off;
      }
      off += L.total;
    }
  if (count) *count = 0;
  return off;
}

size_t mbo_student_param_count(int b) {
  return mbo_candidate_offset(b, mbo_student_layers(b), 0, NULL);
}

/* teacher flat params: [stem W[32][3][3][16] + bias] then per layer [expand W + b] [dw W + b] [proj W + b] */
size_t mbo_teacher_param_count(int b) {
  size_t t = b == 0 ? 32 * 9 * 16 + 32 : 0;
  for (int l = 0; l < NL[b]; ++l) {
    mb_layer m;
    teacher_layer(b, l, &m);
    const int E = expand_ch(m.cin, m.t);
    const int cs = se_ch(&m);
    if (m.t != 1) t += (size_t)E * m.cin + E;
    t += (size_t)E * m.k * m.k + E;
    if (cs) t += (size_t)cs * E + cs + (size_t)E * cs + E;
    t += (size_t)m.cout * E + m.cout;
  }
  return t;
}

/* ------------------------------------------------------------------ data / init */
void mbo_input(int n, int64_t first, int S, uint32_t seed, float* out, int bf16) {
  const int64_t per = (int64_t)S * S * 3;
  const uint32_t key[2] = {seed, 0xDA7A0000u};
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i)
    for (int64_t e = 0; e < per; ++e) {
      const uint64_t idx = (uint64_t)(first + i) * (uint64_t)per + (uint64_t)e;
      const uint32_t ctr[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), 0u, 0u};
      uint32_t o[4];
      bdo_philox(ctr, key, o);
      out[(int64_t)i * per + e] = rnd(sym_unit(o[0]), bf16);
    }
}

/* dst[k][r][s][cs] = (k < kt && c < ct) ? U(-1,1)*bound : 0, Philox counter (flat index of the true
 * [kt][r][s][ct] tensor, tensor id) — the product's pbdk_init_uniform */
static void fill(float* dst, int K, int kt, int R, int cs, int ct, uint32_t seed, uint32_t tid, float bound,
                 int bf16) {
  const uint32_t key[2] = {seed, 0xB200B200u};
  for (int k = 0; k < K; ++k)
    for (int rs = 0; rs < R * R; ++rs)
      for (int c = 0; c < cs; ++c) {
        float v = 0.0f;
        if (k < kt && c < ct) {
          const uint32_t i = (uint32_t)(((size_t)k * R * R + rs) * ct + c);
          const uint32_t ctr[4] = {i, tid, 0u, 0u};
          uint32_t o[4];
          bdo_philox(ctr, key, o);
          v = rnd(sym_unit(o[0]) * bound, bf16);
        }
        dst[((size_t)k * R * R + rs) * cs + c] = v;
      }
}

static float kaiming(int fan_in, float gain) { return sqrtf(6.0f / (float)fan_in) * gain; }

/* teacher tensor ids: 20000 + 1000*block + 10*conv (+1 bias), convs in program order */
void mbo_teacher_init(int b, uint32_t seed, float* p, int bf16) {
  int j = 0;
  if (b == 0) {
    fill(p, 32, 32, 3, 16, 3, seed, 20000u + 10u * j, kaiming(27, 1.0f), bf16);
    p += 32 * 9 * 16;
    fill(p, 32, 32, 1, 1, 1, seed, 20000u + 10u * j + 1u, 0.1f, 0);
    p += 32;
    ++j;
  }
  for (int l = 0; l < NL[b]; ++l) {
    mb_layer m;
    teacher_layer(b, l, &m);
    const int E = expand_ch(m.cin, m.t), Et = expand_ch_t(m.cin_t, m.t);
    const uint32_t base = 20000u + 1000u * (uint32_t)b;
    if (m.t != 1) {
      fill(p, E, Et, 1, m.cin, m.cin_t, seed, base + 10u * j, kaiming(m.cin_t, 1.0f), bf16);
      p += (size_t)E * m.cin;
      fill(p, E, Et, 1, 1, 1, seed, base + 10u * j + 1u, 0.1f, 0);
      p += E;
      ++j;
    }
    fill(p, E, Et, m.k, 1, 1, seed, base + 10u * j, kaiming(m.k * m.k, 1.0f), bf16);
    p += (size_t)E * m.k * m.k;
    fill(p, E, Et, 1, 1, 1, seed, base + 10u * j + 1u, 0.1f, 0);
    p += E;
    ++j;
    const int cs = se_ch(&m), cst = se_ch_t(&m);
    if (cs) { /* squeeze-excite: W1 [cs][E] + b1, W2 [E][cs] + b2 */
      fill(p, cs, cst, 1, E, Et, seed, base + 10u * j, kaiming(Et, 1.0f), bf16);
      p += (size_t)cs * E;
      fill(p, cs, cst, 1, 1, 1, seed, base + 10u * j + 1u, 0.1f, 0);
      p += cs;
      ++j;
      fill(p, E, Et, 1, cs, cst, seed, base + 10u * j, kaiming(cst, 1.0f), bf16);
      p += (size_t)E * cs;
      fill(p, E, Et, 1, 1, 1, seed, base + 10u * j + 1u, 0.1f, 0);
      p += E;
      ++j;
    }
    const int res = has_res(&m);
    fill(p, m.cout, m.cout_t, 1, E, Et, seed, base + 10u * j, kaiming(Et, res ? 0.5f : 1.0f), bf16);
    p += (size_t)m.cout * E;
    fill(p, m.cout, m.cout_t, 1, 1, 1, seed, base + 10u * j + 1u, 0.1f, 0);
    p += m.cout;
    ++j;
  }
}

/* student tensor ids: 40000 + 1000*block + 100*layer + 10*cand + {0 expand, 1 dw, 2 project} */
void mbo_student_init(int b, uint32_t seed, float* p) {
  for (int l = 0; l < mbo_student_layers(b); ++l)
    for (int c = 0; c < mbo_layer_candidates(b, l); ++c) {
      const cand_layout L = cand_lay(b, l, c);
      float* q = p + mbo_candidate_offset(b, l, c, NULL);
      const uint32_t tid = 40000u + 1000u * (uint32_t)b + 100u * (uint32_t)l + 10u * (uint32_t)c;
      if (b == 0 && l == 0) {
        fill(q, 32, 32, 3, 16, 3, seed, tid, kaiming(27, 1.0f), 0);
        for (int i = 0; i < 32; ++i) {
          q[L.g2 + i] = 1.0f;
          q[L.b2 + i] = 0.0f;
        }
        continue;
      }
      const mb_layer m = student_mb(b, l);
      if (L.e != 1) fill(q + L.we, L.E, L.Et, 1, m.cin, m.cin_t, seed, tid, kaiming(m.cin_t, 1.0f), 0);
      fill(q + L.wd, L.E, L.Et, L.k, 1, 1, seed, tid + 1u, kaiming(L.k * L.k, 1.0f), 0);
      fill(q + L.wp, m.cout, m.cout_t, 1, L.E, L.Et, seed, tid + 2u, kaiming(L.Et, 1.0f), 0);
      for (int i = 0; i < L.E; ++i) {
        if (L.e != 1) {
          q[L.g1 + i] = 1.0f;
          q[L.b1 + i] = 0.0f;
        }
        q[L.g2 + i] = 1.0f;
        q[L.b2 + i] = 0.0f;
      }
      for (int i = 0; i < m.cout; ++i) {
        q[L.g3 + i] = 1.0f;
        q[L.b3 + i] = 0.0f;
      }
    }
}

/* path[l] = Philox(counter {draw lo, draw hi, layer, block}, key {seed, 0x5EA4C400}) mod candidates */
void mbo_sample_path(int b, uint32_t seed, int64_t draw, int* path) {
  const uint32_t key[2] = {seed, 0x5EA4C400u};
  for (int l = 0; l < mbo_student_layers(b); ++l) {
    const int nc = mbo_layer_candidates(b, l);
    if (nc == 1) {
      path[l] = 0;
      continue;
    }
    const uint32_t ctr[4] = {(uint32_t)draw, (uint32_t)((uint64_t)draw >> 32), (uint32_t)l, (uint32_t)b};
    uint32_t o[4];
    bdo_philox(ctr, key, o);
    path[l] = (int)(o[0] % (uint32_t)nc);
  }
}

/* ------------------------------------------------------------------ ops (NHWC) */
static inline float dot(const float* a, const float* b, int n) {
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int i = 0;
  for (; i + 8 <= n; i += 8)
    for (int l = 0; l < 8; ++l) acc[l] += a[i + l] * b[i + l];
  float s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  for (; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* y[m][k] = sum_c x[m][c] w[k][c] (tensor cores on the GPU: only the accumulation order differs) */
static void conv1x1(const float* x, size_t m, int C, const float* w, int K, float* y) {
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)m; ++i)
    for (int k = 0; k < K; ++k) y[(size_t)i * K + k] = dot(x + (size_t)i * C, w + (size_t)k * C, C);
}

/* dx[m][c] = sum_k dy[m][k] w[k][c] */
static void conv1x1_dgrad(const float* dy, size_t m, int K, const float* w, int C, float* dx) {
  float* wt = (float*)malloc(sizeof(float) * (size_t)K * C);
  for (int k = 0; k < K; ++k)
    for (int c = 0; c < C; ++c) wt[(size_t)c * K + k] = w[(size_t)k * C + c];
  conv1x1(dy, m, K, wt, C, dx);
  free(wt);
}

/* dw[k][c] = sum_m dy[m][k] x[m][c]  (double) */
static void conv1x1_wgrad(const float* x, size_t m, int C, const float* dy, int K, float* dw) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int k = 0; k < K; ++k) {
    double* acc = (double*)calloc((size_t)C, sizeof(double));
    for (size_t i = 0; i < m; ++i) {
      const double g = dy[i * K + k];
      if (g == 0.0) continue;
      const float* xs = x + i * C;
      for (int c = 0; c < C; ++c) acc[c] += g * xs[c];
    }
    for (int c = 0; c < C; ++c) dw[(size_t)k * C + c] = (float)acc[c];
    free(acc);
  }
}

/* depthwise: y[n,p,q,c] = fmaf chain over (r, s) ascending of x[n, p*st+r-pad, q*st+s-pad, c] w[c][r][s] */
static void dw_fwd(const float* x, int N, int H, int W, int C, const float* w, int k, int st, int P, int Q, float* y) {
  const int pad = k / 2;
#pragma omp parallel for schedule(static)
  for (int np = 0; np < N * P; ++np) {
    const int n = np / P, p = np % P;
    for (int q = 0; q < Q; ++q)
      for (int c = 0; c < C; ++c) {
        float acc = 0.0f;
        for (int r = 0; r < k; ++r) {
          const int h = p * st + r - pad;
          if (h < 0 || h >= H) continue;
          for (int s = 0; s < k; ++s) {
            const int ww = q * st + s - pad;
            if (ww < 0 || ww >= W) continue;
            acc = fmaf(x[(((size_t)n * H + h) * W + ww) * C + c], w[((size_t)c * k + r) * k + s], acc);
          }
        }
        y[(((size_t)n * P + p) * Q + q) * C + c] = acc;
      }
  }
}

/* dx[n,h,w,c] = fmaf chain over (r, s) ascending of dy[n,(h+pad-r)/st,(w+pad-s)/st,c] w[c][r][s] */
static void dw_dgrad(const float* dy, int N, int P, int Q, int C, const float* w, int k, int st, int H, int W,
                     float* dx) {
  const int pad = k / 2;
#pragma omp parallel for schedule(static)
  for (int nh = 0; nh < N * H; ++nh) {
    const int n = nh / H, h = nh % H;
    for (int ww = 0; ww < W; ++ww)
      for (int c = 0; c < C; ++c) {
        float acc = 0.0f;
        for (int r = 0; r < k; ++r) {
          const int pn = h + pad - r;
          if (pn < 0 || pn % st != 0 || pn / st >= P) continue;
          for (int s = 0; s < k; ++s) {
            const int qn = ww + pad - s;
            if (qn < 0 || qn % st != 0 || qn / st >= Q) continue;
            acc = fmaf(dy[(((size_t)n * P + pn / st) * Q + qn / st) * C + c], w[((size_t)c * k + r) * k + s], acc);
          }
        }
        dx[(((size_t)n * H + h) * W + ww) * C + c] = acc;
      }
  }
}

/* dw[c][r][s] = sum_{n,p,q} dy[n,p,q,c] x[n, p*st+r-pad, q*st+s-pad, c]  (double) */
static void dw_wgrad(const float* x, int N, int H, int W, int C, const float* dy, int k, int st, int P, int Q,
                     float* dw) {
  const int pad = k / 2;
#pragma omp parallel for schedule(static)
  for (int c = 0; c < C; ++c)
    for (int r = 0; r < k; ++r)
      for (int s = 0; s < k; ++s) {
        double acc = 0.0;
        for (int n = 0; n < N; ++n)
          for (int p = 0; p < P; ++p) {
            const int h = p * st + r - pad;
            if (h < 0 || h >= H) continue;
            for (int q = 0; q < Q; ++q) {
              const int ww = q * st + s - pad;
              if (ww < 0 || ww >= W) continue;
              acc += (double)dy[(((size_t)n * P + p) * Q + q) * C + c] * x[(((size_t)n * H + h) * W + ww) * C + c];
            }
          }
        dw[((size_t)c * k + r) * k + s] = (float)acc;
      }
}

/* stem: y[n,p,q,k] = fmaf chain over (r, s, c<3) of x[n,2p+r-1,2q+s-1,c] w[k][r][s][c] (w stored with 16 ch) */
static void stem_fwd(const float* x, int N, int S, const float* w, float* y) {
  const int P = S / 2;
#pragma omp parallel for schedule(static)
  for (int np = 0; np < N * P; ++np) {
    const int n = np / P, p = np % P;
    for (int q = 0; q < P; ++q)
      for (int k = 0; k < 32; ++k) {
        float acc = 0.0f;
        for (int r = 0; r < 3; ++r) {
          const int h = 2 * p + r - 1;
          if (h < 0 || h >= S) continue;
          for (int s = 0; s < 3; ++s) {
            const int ww = 2 * q + s - 1;
            if (ww < 0 || ww >= S) continue;
            for (int c = 0; c < 3; ++c)
              acc = fmaf(x[(((size_t)n * S + h) * S + ww) * 3 + c], w[((size_t)k * 9 + r * 3 + s) * 16 + c], acc);
          }
        }
        y[(((size_t)n * P + p) * P + q) * 32 + k] = acc;
      }
  }
}

static void stem_wgrad(const float* x, int N, int S, const float* dy, float* dw) {
  const int P = S / 2;
  memset(dw, 0, sizeof(float) * 32 * 9 * 16);
#pragma omp parallel for schedule(static)
  for (int k = 0; k < 32; ++k)
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s)
        for (int c = 0; c < 3; ++c) {
          double acc = 0.0;
          for (int n = 0; n < N; ++n)
            for (int p = 0; p < P; ++p) {
              const int h = 2 * p + r - 1;
              if (h < 0 || h >= S) continue;
              for (int q = 0; q < P; ++q) {
                const int ww = 2 * q + s - 1;
                if (ww < 0 || ww >= S) continue;
                acc += (double)dy[(((size_t)n * P + p) * P + q) * 32 + k] * x[(((size_t)n * S + h) * S + ww) * 3 + c];
              }
            }
          dw[((size_t)k * 9 + r * 3 + s) * 16 + c] = (float)acc;
        }
}

static void round_all(float* y, size_t n, int bf16) {
  if (!bf16) return;
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)n; ++i) y[i] = bdo_bf16(y[i]);
}

/* teacher epilogue: y = rnd(act(y + b [+ res])) ; act 0 none, 6 relu6 */
static void bias_act(float* y, size_t m, int K, const float* b, const float* res, int act, int bf16) {
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)m; ++i)
    for (int k = 0; k < K; ++k) {
      float v = y[(size_t)i * K + k] + b[k];
      if (res) v += res[(size_t)i * K + k];
      if (act == 6) v = relu6(v);
      if (act == 7) v = tact(v);
      y[(size_t)i * K + k] = rnd(v, bf16);
    }
}

/* squeeze-excite on y [n][hw][E] in place: pooled = mean_hw y (double sum), h = swish(W1 pooled + b1),
 * gate = sigmoid(W2 h + b2), y = rnd(y * gate).  p = [W1 [cs][E], b1 [cs], W2 [E][cs], b2 [E]]. */
static void se_apply(float* y, int n, int hw, int E, int cs, const float* p, int bf16) {
  const float* W1 = p;
  const float* b1 = W1 + (size_t)cs * E;
  const float* W2 = b1 + cs;
  const float* b2 = W2 + (size_t)E * cs;
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) {
    float* pooled = (float*)malloc(sizeof(float) * E);
    float* h = (float*)malloc(sizeof(float) * cs);
    float* gate = (float*)malloc(sizeof(float) * E);
    float* yi = y + (size_t)i * hw * E;
    for (int c = 0; c < E; ++c) {
      double acc = 0.0;
      for (int q = 0; q < hw; ++q) acc += yi[(size_t)q * E + c];
      pooled[c] = (float)(acc / hw);
    }
    for (int j = 0; j < cs; ++j) {
      float acc = b1[j];
      for (int c = 0; c < E; ++c) acc = fmaf(W1[(size_t)j * E + c], pooled[c], acc);
      h[j] = swishf(acc);
    }
    for (int c = 0; c < E; ++c) {
      float acc = b2[c];
      for (int j = 0; j < cs; ++j) acc = fmaf(W2[(size_t)c * cs + j], h[j], acc);
      gate[c] = sigmoidf(acc);
    }
    for (int q = 0; q < hw; ++q)
      for (int c = 0; c < E; ++c) yi[(size_t)q * E + c] = rnd(yi[(size_t)q * E + c] * gate[c], bf16);
    free(pooled);
    free(h);
    free(gate);
  }
}

/* ------------------------------------------------------------------ teacher forward */
int mbo_teacher_fwd(int b, const float* tp, int n, int S, const float* in, float* out, int bf16) {
  int H = mbo_hw(b, S);
  int C = CH[b];
  size_t cap = (size_t)n * (S / 2) * (S / 2) * 32;
  for (int l = 0; l < NL[b]; ++l) {
    mb_layer m;
    teacher_layer(b, l, &m);
    const size_t e = (size_t)n * H * H * expand_ch(m.cin, m.t);
    if (e > cap) cap = e;
  }
  float* x = (float*)malloc(sizeof(float) * cap);
  float* e1 = (float*)malloc(sizeof(float) * cap);
  float* e2 = (float*)malloc(sizeof(float) * cap);
  float* o = (float*)malloc(sizeof(float) * cap);
  if (b == 0) {
    stem_fwd(in, n, S, tp, x);
    bias_act(x, (size_t)n * (S / 2) * (S / 2), 32, tp + 32 * 9 * 16, NULL, 7, bf16);
    tp += 32 * 9 * 16 + 32;
    H = S / 2;
  } else {
    memcpy(x, in, sizeof(float) * (size_t)n * H * H * C);
  }
  for (int l = 0; l < NL[b]; ++l) {
    mb_layer m;
    teacher_layer(b, l, &m);
    const int E = expand_ch(m.cin, m.t);
    const int P = (H + 2 * (m.k / 2) - m.k) / m.stride + 1;
    const float* a = x;
    if (m.t != 1) {
      conv1x1(x, (size_t)n * H * H, m.cin, tp, E, e1);
      bias_act(e1, (size_t)n * H * H, E, tp + (size_t)E * m.cin, NULL, 7, bf16);
      tp += (size_t)E * m.cin + E;
      a = e1;
    }
    dw_fwd(a, n, H, H, E, tp, m.k, m.stride, P, P, e2);
    bias_act(e2, (size_t)n * P * P, E, tp + (size_t)E * m.k * m.k, NULL, 7, bf16);
    tp += (size_t)E * m.k * m.k + E;
    const int cs = se_ch(&m);
    if (cs) se_apply(e2, n, P * P, E, cs, tp, bf16);
    if (cs) tp += (size_t)cs * E + cs + (size_t)E * cs + E;
    conv1x1(e2, (size_t)n * P * P, E, tp, m.cout, o);
    const int res = has_res(&m);
    bias_act(o, (size_t)n * P * P, m.cout, tp + (size_t)m.cout * E, res ? x : NULL, 0, bf16);
    tp += (size_t)m.cout * E + m.cout;
    memcpy(x, o, sizeof(float) * (size_t)n * P * P * m.cout);
    H = P;
    C = m.cout;
  }
  memcpy(out, x, sizeof(float) * (size_t)n * H * H * C);
  free(x);
  free(e1);
  free(e2);
  free(o);
  return 0;
}

/* ------------------------------------------------------------------ student: training-mode BN */
typedef struct {
  float *mean, *rstd, *A, *B;
} bn_t;

static bn_t bn_forward(const float* y, size_t m, int C, const float* gamma, const float* beta) {
  bn_t s;
  s.mean = (float*)malloc(sizeof(float) * C);
  s.rstd = (float*)malloc(sizeof(float) * C);
  s.A = (float*)malloc(sizeof(float) * C);
  s.B = (float*)malloc(sizeof(float) * C);
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
    s.mean[c] = (float)mu;
    s.rstd[c] = 1.0f / sqrtf((float)var + BN_EPS);
    s.A[c] = gamma[c] * s.rstd[c];
    s.B[c] = fmaf(-s.A[c], s.mean[c], beta[c]);
  }
  return s;
}

static void bn_free(bn_t* s) {
  free(s->mean);
  free(s->rstd);
  free(s->A);
  free(s->B);
}

/* a = rnd(act(A*y + B)) */
static void bn_apply(const float* y, size_t m, int C, const bn_t* s, int act, int bf16, float* a) {
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)m; ++i)
    for (int c = 0; c < C; ++c) {
      float z = fmaf(s->A[c], y[(size_t)i * C + c], s->B[c]);
      if (act == 6) z = relu6(z);
      a[(size_t)i * C + c] = rnd(z, bf16);
    }
}

/* BN backward from the upstream gradient g: dbeta = sum g, dgamma = sum g*xhat,
 * dy = rnd(fmaf(A, g, fmaf(Q, y, R))) */
static void bn_backward(const float* g, const float* y, size_t m, int C, const bn_t* s, int bf16, float* dgamma,
                        float* dbeta, float* dy) {
  float* Q = (float*)malloc(sizeof(float) * C);
  float* R = (float*)malloc(sizeof(float) * C);
#pragma omp parallel for schedule(static)
  for (int c = 0; c < C; ++c) {
    double sg = 0.0, sgy = 0.0;
    for (size_t i = 0; i < m; ++i) {
      const double gv = g[i * C + c];
      sg += gv;
      sgy += gv * y[i * C + c];
    }
    const double sgx = (double)s->rstd[c] * (sgy - (double)s->mean[c] * sg);
    dbeta[c] = (float)sg;
    dgamma[c] = (float)sgx;
    const double c1 = (double)s->A[c] / (double)m;
    Q[c] = (float)(-c1 * sgx * (double)s->rstd[c]);
    R[c] = (float)(-c1 * (sg - sgx * (double)s->rstd[c] * (double)s->mean[c]));
  }
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)m; ++i)
    for (int c = 0; c < C; ++c) {
      const size_t j = (size_t)i * C + c;
      dy[j] = rnd(fmaf(s->A[c], g[j], fmaf(Q[c], y[j], R[c])), bf16);
    }
  free(Q);
  free(R);
}

static float* shadow(const float* w, size_t n, int bf16) {
  float* s = (float*)malloc(sizeof(float) * (n ? n : 1));
  for (size_t i = 0; i < n; ++i) s[i] = rnd(w[i], bf16);
  return s;
}

typedef struct {
  int H, P, cin, cout, E, k, e, stride, res;
  cand_layout L;
  const float* p; /* candidate params */
  float* gr;      /* candidate grads */
  float *we, *wd, *wp;
  float *x, *y1, *a1, *y2, *a2, *y3; /* x = layer input (owned by the previous layer / caller) */
  bn_t bn1, bn2, bn3;
} layer_state;

int mbo_student_fwd_bwd(int b, const float* sp, const int* path, int n, int S, const float* in, const float* t_out,
                        double norm, int bf16, float* grads, double* loss_out) {
  const int NLs = mbo_student_layers(b);
  memset(grads, 0, sizeof(float) * mbo_student_param_count(b));
  layer_state* st = (layer_state*)calloc((size_t)NLs, sizeof(layer_state));
  int H = mbo_hw(b, S);
  const float* x = in;
  /* ---- stem (block 0) */
  float *stem_y = NULL, *stem_a = NULL;
  bn_t stem_bn;
  const float* stem_p = NULL;
  float* stem_w = NULL;
  int l0 = 0;
  if (b == 0) {
    const cand_layout L = cand_lay(0, 0, 0);
    stem_p = sp;
    const size_t m = (size_t)n * (S / 2) * (S / 2);
    stem_w = shadow(sp, 32 * 9 * 16, bf16);
    stem_y = (float*)malloc(sizeof(float) * m * 32);
    stem_a = (float*)malloc(sizeof(float) * m * 32);
    stem_fwd(in, n, S, stem_w, stem_y);
    round_all(stem_y, m * 32, bf16);
    stem_bn = bn_forward(stem_y, m, 32, sp + L.g2, sp + L.b2);
    bn_apply(stem_y, m, 32, &stem_bn, 6, bf16, stem_a);
    x = stem_a;
    H = S / 2;
    l0 = 1;
  }
  /* ---- forward through the MBConv layers */
  for (int l = l0; l < NLs; ++l) {
    layer_state* s = &st[l];
    const mb_layer m = student_mb(b, l);
    s->L = cand_lay(b, l, path[l]);
    s->H = H;
    s->cin = m.cin;
    s->cout = m.cout;
    s->stride = m.stride;
    s->E = s->L.E;
    s->k = s->L.k;
    s->e = s->L.e;
    s->P = (H + 2 * (s->k / 2) - s->k) / s->stride + 1;
    s->res = has_res(&m);
    const size_t off = mbo_candidate_offset(b, l, path[l], NULL);
    s->p = sp + off;
    s->gr = grads + off;
    const size_t mi = (size_t)n * H * H, mo = (size_t)n * s->P * s->P;
    s->x = (float*)x;
    const float* a = x;
    if (s->e != 1) {
      s->we = shadow(s->p + s->L.we, (size_t)s->E * s->cin, bf16);
      s->y1 = (float*)malloc(sizeof(float) * mi * s->E);
      s->a1 = (float*)malloc(sizeof(float) * mi * s->E);
      conv1x1(x, mi, s->cin, s->we, s->E, s->y1);
      round_all(s->y1, mi * s->E, bf16);
      s->bn1 = bn_forward(s->y1, mi, s->E, s->p + s->L.g1, s->p + s->L.b1);
      bn_apply(s->y1, mi, s->E, &s->bn1, 6, bf16, s->a1);
      a = s->a1;
    }
    s->wd = shadow(s->p + s->L.wd, (size_t)s->E * s->k * s->k, bf16);
    s->wp = shadow(s->p + s->L.wp, (size_t)s->cout * s->E, bf16);
    s->y2 = (float*)malloc(sizeof(float) * mo * s->E);
    s->a2 = (float*)malloc(sizeof(float) * mo * s->E);
    s->y3 = (float*)malloc(sizeof(float) * mo * s->cout);
    dw_fwd(a, n, H, H, s->E, s->wd, s->k, s->stride, s->P, s->P, s->y2);
    round_all(s->y2, mo * s->E, bf16);
    s->bn2 = bn_forward(s->y2, mo, s->E, s->p + s->L.g2, s->p + s->L.b2);
    bn_apply(s->y2, mo, s->E, &s->bn2, 6, bf16, s->a2);
    conv1x1(s->a2, mo, s->E, s->wp, s->cout, s->y3);
    round_all(s->y3, mo * s->cout, bf16);
    s->bn3 = bn_forward(s->y3, mo, s->cout, s->p + s->L.g3, s->p + s->L.b3);
    if (l + 1 < NLs) { /* the next layer's input z = rnd(A3*y3 + B3 [+ x]) */
      float* z = (float*)malloc(sizeof(float) * mo * s->cout);
#pragma omp parallel for schedule(static)
      for (long long i = 0; i < (long long)mo; ++i)
        for (int c = 0; c < s->cout; ++c) {
          const size_t j = (size_t)i * s->cout + c;
          float v = fmaf(s->bn3.A[c], s->y3[j], s->bn3.B[c]);
          if (s->res) v += x[j];
          z[j] = rnd(v, bf16);
        }
      x = z;
    }
    H = s->P;
  }
  /* ---- loss on the last layer: z = A3*y3 + B3 [+ x] (fp32), g = rnd((z - t) * 2/norm) */
  layer_state* last = &st[NLs - 1];
  const size_t mo = (size_t)n * last->P * last->P;
  const int Co = last->cout;
  float* dz = (float*)malloc(sizeof(float) * mo * Co);
  const float gscale = (float)(2.0 / norm);
  double* part = (double*)calloc((size_t)n, sizeof(double));
  const size_t per = (size_t)last->P * last->P;
#pragma omp parallel for schedule(static)
  for (int smp = 0; smp < n; ++smp)
    for (size_t i = (size_t)smp * per; i < (size_t)(smp + 1) * per; ++i)
      for (int c = 0; c < Co; ++c) {
        const size_t j = i * Co + c;
        float v = fmaf(last->bn3.A[c], last->y3[j], last->bn3.B[c]);
        if (last->res) v += last->x[j];
        const float d = v - t_out[j];
        part[smp] += (double)d * (double)d;
        dz[j] = rnd(d * gscale, bf16);
      }
  double loss = 0.0;
  for (int smp = 0; smp < n; ++smp) loss += part[smp];
  *loss_out = loss / norm;
  free(part);
  /* ---- backward */
  for (int l = NLs - 1; l >= l0; --l) {
    layer_state* s = &st[l];
    const size_t mi = (size_t)n * s->H * s->H, mo2 = (size_t)n * s->P * s->P;
    float* dy3 = (float*)malloc(sizeof(float) * mo2 * s->cout);
    bn_backward(dz, s->y3, mo2, s->cout, &s->bn3, bf16, s->gr + s->L.g3, s->gr + s->L.b3, dy3);
    conv1x1_wgrad(s->a2, mo2, s->E, dy3, s->cout, s->gr + s->L.wp);
    float* g2 = (float*)malloc(sizeof(float) * mo2 * s->E);
    conv1x1_dgrad(dy3, mo2, s->cout, s->wp, s->E, g2);
    for (size_t i = 0; i < mo2 * s->E; ++i) g2[i] = rnd(mask6(s->a2[i]) ? g2[i] : 0.0f, bf16);
    float* dy2 = (float*)malloc(sizeof(float) * mo2 * s->E);
    bn_backward(g2, s->y2, mo2, s->E, &s->bn2, bf16, s->gr + s->L.g2, s->gr + s->L.b2, dy2);
    const float* a_in = s->e != 1 ? s->a1 : s->x;
    dw_wgrad(a_in, n, s->H, s->H, s->E, dy2, s->k, s->stride, s->P, s->P, s->gr + s->L.wd);
    float* dnext = NULL; /* gradient w.r.t. the layer input x */
    const int need_dx = l > 0;  /* block input (teacher output) needs no gradient */
    if (s->e != 1) {
      float* g1 = (float*)malloc(sizeof(float) * mi * s->E);
      dw_dgrad(dy2, n, s->P, s->P, s->E, s->wd, s->k, s->stride, s->H, s->H, g1);
      for (size_t i = 0; i < mi * s->E; ++i) g1[i] = rnd(mask6(s->a1[i]) ? g1[i] : 0.0f, bf16);
      float* dy1 = (float*)malloc(sizeof(float) * mi * s->E);
      bn_backward(g1, s->y1, mi, s->E, &s->bn1, bf16, s->gr + s->L.g1, s->gr + s->L.b1, dy1);
      conv1x1_wgrad(s->x, mi, s->cin, dy1, s->E, s->gr + s->L.we);
      if (need_dx) {
        dnext = (float*)malloc(sizeof(float) * mi * s->cin);
        conv1x1_dgrad(dy1, mi, s->E, s->we, s->cin, dnext);
        for (size_t i = 0; i < mi * s->cin; ++i) dnext[i] = rnd(dnext[i] + (s->res ? dz[i] : 0.0f), bf16);
      }
      free(g1);
      free(dy1);
    } else if (need_dx) { /* MBConv1: the layer input feeds the depthwise conv directly */
      dnext = (float*)malloc(sizeof(float) * mi * s->cin);
      dw_dgrad(dy2, n, s->P, s->P, s->E, s->wd, s->k, s->stride, s->H, s->H, dnext);
      if (l == 1 && b == 0) { /* input = stem activation: relu6 mask */
        for (size_t i = 0; i < mi * s->cin; ++i) dnext[i] = rnd(mask6(s->x[i]) ? dnext[i] : 0.0f, bf16);
      } else {
        for (size_t i = 0; i < mi * s->cin; ++i) dnext[i] = rnd(dnext[i] + (s->res ? dz[i] : 0.0f), bf16);
      }
    }
    free(dy3);
    free(g2);
    free(dy2);
    free(dz);
    dz = dnext;
  }
  if (b == 0) { /* stem backward: dz = relu6-masked gradient of the stem activation */
    const cand_layout L = cand_lay(0, 0, 0);
    const size_t m = (size_t)n * (S / 2) * (S / 2);
    float* dys = (float*)malloc(sizeof(float) * m * 32);
    bn_backward(dz, stem_y, m, 32, &stem_bn, bf16, grads + L.g2, grads + L.b2, dys);
    stem_wgrad(in, n, S, dys, grads);
    free(dys);
    free(dz);
    free(stem_y);
    free(stem_w);
    bn_free(&stem_bn);
  }
  (void)stem_p;
  /* ---- cleanup */
  for (int l = l0; l < NLs; ++l) {
    layer_state* s = &st[l];
    if (l > l0) free(s->x); /* z of the previous layer */
    if (s->e != 1) {
      free(s->we);
      free(s->y1);
      free(s->a1);
      bn_free(&s->bn1);
    }
    free(s->wd);
    free(s->wp);
    free(s->y2);
    free(s->a2);
    free(s->y3);
    bn_free(&s->bn2);
    bn_free(&s->bn3);
  }
  if (b == 0) free(stem_a);
  free(st);
  return 0;
}

void mbo_sgd_path(int b, const int* path, float* w, float* v, const float* g, float lr, float mu) {
  for (int l = 0; l < mbo_student_layers(b); ++l) {
    size_t cnt = 0;
    const size_t off = mbo_candidate_offset(b, l, path[l], &cnt);
    for (size_t i = off; i < off + cnt; ++i) {
      v[i] = fmaf(mu, v[i], g[i]);
      w[i] = fmaf(-lr, v[i], w[i]);
    }
  }
}

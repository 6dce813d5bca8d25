/* ORACLE — test infrastructure only (see cpu_member.h for the contract and the
 * reference file:line each function restates). */
#include "cpu_member.h"

#include <math.h>
#if defined(__AVX2__)
#include <immintrin.h>
#endif
#include <stdlib.h>
#include <string.h>

/* splitmix64 finaliser, as /root/reference/proj/src/runtime/backend.cpp:12-17. */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

float orc_round_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) { /* inf / nan: truncate, keep quiet */
    if (u & 0x007fffffu) u |= 0x00400000u;
    u &= 0xffff0000u;
  } else {
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    u &= 0xffff0000u;
  }
  float y;
  memcpy(&y, &u, 4);
  return y;
}

static uint64_t stream_key(uint64_t seed, int layer, int is_bias) {
  return orc_splitmix64(seed * 0x100000001b3ULL + (uint64_t)(2 * layer + is_bias + 1));
}

static float unit24(uint64_t key, uint64_t idx) {
  uint64_t h = orc_splitmix64(key ^ (idx * 0x9e3779b97f4a7c15ULL));
  return (float)(h >> 40) / 16777216.0f;
}

float orc_weight(uint64_t seed, int layer, uint64_t idx, int fan_in, int fan_out) {
  float limit = (float)sqrt(6.0 / (double)(fan_in + fan_out));
  float u = unit24(stream_key(seed, layer, 0), idx);
  return (2.0f * u - 1.0f) * limit;
}

float orc_bias(uint64_t seed, int layer, uint64_t idx) {
  float u = unit24(stream_key(seed, layer, 1), idx);
  return (2.0f * u - 1.0f) * 0.01f;
}

float orc_feature(uint64_t seed, uint64_t idx) {
  uint64_t h = orc_splitmix64(seed * 0x2545f4914f6cdd1dULL + idx);
  return (float)(h >> 40) / 16777216.0f;
}

void orc_fill_features(uint64_t seed, size_t rows, size_t width, float* x) {
  size_t n = rows * width;
  for (size_t i = 0; i < n; ++i) x[i] = orc_feature(seed, i);
}

struct orc_mlp {
  int n_layers;
  int widths[ORC_MAX_LAYERS + 1];
  int padded_out[ORC_MAX_LAYERS];
  int quantize;
  float* w[ORC_MAX_LAYERS];  /* [fan_out][fan_in], quantised if bf16 mode */
  float* wt[ORC_MAX_LAYERS]; /* [fan_in][padded_out], zero padded */
  float* b[ORC_MAX_LAYERS];  /* [padded_out], fp32 */
};

orc_mlp* orc_mlp_create(int n_layers, const int* widths, uint64_t seed,
                        int quantize_bf16) {
  if (n_layers < 1 || n_layers > ORC_MAX_LAYERS) return NULL;
  orc_mlp* m = (orc_mlp*)calloc(1, sizeof(orc_mlp));
  m->n_layers = n_layers;
  m->quantize = quantize_bf16;
  for (int l = 0; l <= n_layers; ++l) m->widths[l] = widths[l];
  for (int l = 0; l < n_layers; ++l) {
    int fi = widths[l], fo = widths[l + 1];
    int po = (fo + 15) / 16 * 16;
    m->padded_out[l] = po;
    m->w[l] = (float*)malloc(sizeof(float) * (size_t)fi * fo);
    m->wt[l] = (float*)calloc((size_t)fi * po, sizeof(float));
    m->b[l] = (float*)calloc((size_t)po, sizeof(float));
    for (int o = 0; o < fo; ++o) {
      for (int i = 0; i < fi; ++i) {
        uint64_t idx = (uint64_t)o * fi + i;
        float v = orc_weight(seed, l, idx, fi, fo);
        if (quantize_bf16) v = orc_round_bf16(v);
        m->w[l][idx] = v;
        m->wt[l][(size_t)i * po + o] = v;
      }
      m->b[l][o] = orc_bias(seed, l, (uint64_t)o);
    }
  }
  return m;
}

void orc_mlp_destroy(orc_mlp* m) {
  if (!m) return;
  for (int l = 0; l < m->n_layers; ++l) {
    free(m->w[l]);
    free(m->wt[l]);
    free(m->b[l]);
  }
  free(m);
}

int orc_mlp_classes(const orc_mlp* m) { return m->widths[m->n_layers]; }

void orc_mlp_layer(const orc_mlp* m, int l, float* w, float* b) {
  int fi = m->widths[l], fo = m->widths[l + 1];
  if (w) memcpy(w, m->w[l], sizeof(float) * (size_t)fi * fo);
  if (b) memcpy(b, m->b[l], sizeof(float) * (size_t)fo);
}

#define RB 4  /* rows per register block */
#define JB 16 /* outputs per register block */

/* y[RB][po] = act(x[RB][fi] . wt + b): accumulation strictly in k order per
 * output, fp32; the j loop vectorises without reassociation. */
static void dense_block(const float* x, int fi, const float* wt, const float* b,
                        int po, int relu_q, int quantize, float* y) {
  for (int j0 = 0; j0 < po; j0 += JB) {
    float acc[RB][JB];
#if defined(__AVX2__) && defined(__FMA__)
    /* 4 rows x 16 outputs in 8 ymm registers; acc[r][j] += x[r][k] * w[k][j]
     * with one fused multiply-add per k, k ascending. */
    __m256 a00 = _mm256_setzero_ps(), a01 = _mm256_setzero_ps();
    __m256 a10 = _mm256_setzero_ps(), a11 = _mm256_setzero_ps();
    __m256 a20 = _mm256_setzero_ps(), a21 = _mm256_setzero_ps();
    __m256 a30 = _mm256_setzero_ps(), a31 = _mm256_setzero_ps();
    for (int k = 0; k < fi; ++k) {
      const float* wrow = wt + (size_t)k * po + j0;
      __m256 w0 = _mm256_loadu_ps(wrow), w1 = _mm256_loadu_ps(wrow + 8);
      __m256 x0 = _mm256_broadcast_ss(x + k);
      __m256 x1 = _mm256_broadcast_ss(x + (size_t)fi + k);
      __m256 x2 = _mm256_broadcast_ss(x + 2 * (size_t)fi + k);
      __m256 x3 = _mm256_broadcast_ss(x + 3 * (size_t)fi + k);
      a00 = _mm256_fmadd_ps(x0, w0, a00);
      a01 = _mm256_fmadd_ps(x0, w1, a01);
      a10 = _mm256_fmadd_ps(x1, w0, a10);
      a11 = _mm256_fmadd_ps(x1, w1, a11);
      a20 = _mm256_fmadd_ps(x2, w0, a20);
      a21 = _mm256_fmadd_ps(x2, w1, a21);
      a30 = _mm256_fmadd_ps(x3, w0, a30);
      a31 = _mm256_fmadd_ps(x3, w1, a31);
    }
    _mm256_storeu_ps(acc[0], a00);
    _mm256_storeu_ps(acc[0] + 8, a01);
    _mm256_storeu_ps(acc[1], a10);
    _mm256_storeu_ps(acc[1] + 8, a11);
    _mm256_storeu_ps(acc[2], a20);
    _mm256_storeu_ps(acc[2] + 8, a21);
    _mm256_storeu_ps(acc[3], a30);
    _mm256_storeu_ps(acc[3] + 8, a31);
#else
    memset(acc, 0, sizeof(acc));
    for (int k = 0; k < fi; ++k) {
      const float* wrow = wt + (size_t)k * po + j0;
      for (int r = 0; r < RB; ++r) {
        float xv = x[(size_t)r * fi + k];
        for (int j = 0; j < JB; ++j) acc[r][j] += xv * wrow[j];
      }
    }
#endif
    for (int r = 0; r < RB; ++r) {
      for (int j = 0; j < JB; ++j) {
        float v = acc[r][j] + b[j0 + j];
        if (relu_q) {
          v = v > 0.0f ? v : 0.0f;
          if (quantize) v = orc_round_bf16(v);
        }
        y[(size_t)r * po + j0 + j] = v;
      }
    }
  }
}

void orc_mlp_forward(const orc_mlp* m, const float* x, size_t rows, float* out) {
  int maxw = m->widths[0];
  for (int l = 0; l < m->n_layers; ++l)
    if (m->padded_out[l] > maxw) maxw = m->padded_out[l];
  float* a = (float*)calloc((size_t)RB * maxw, sizeof(float));
  float* c = (float*)calloc((size_t)RB * maxw, sizeof(float));
  int C = m->widths[m->n_layers];
  int fi0 = m->widths[0];
  for (size_t r0 = 0; r0 < rows; r0 += RB) {
    size_t nr = rows - r0 < RB ? rows - r0 : RB;
    memset(a, 0, sizeof(float) * (size_t)RB * maxw);
    for (size_t r = 0; r < nr; ++r)
      for (int k = 0; k < fi0; ++k) {
        float v = x[(r0 + r) * (size_t)fi0 + k];
        a[r * (size_t)fi0 + k] = m->quantize ? orc_round_bf16(v) : v;
      }
    int fi = fi0;
    for (int l = 0; l < m->n_layers; ++l) {
      int po = m->padded_out[l];
      int last = l == m->n_layers - 1;
      dense_block(a, fi, m->wt[l], m->b[l], po, !last, m->quantize, c);
      /* next layer reads exactly widths[l+1] features per row */
      int fo = m->widths[l + 1];
      for (int r = 0; r < RB; ++r)
        memmove(a + (size_t)r * fo, c + (size_t)r * po, sizeof(float) * (size_t)fo);
      fi = fo;
    }
    for (size_t r = 0; r < nr; ++r)
      memcpy(out + (r0 + r) * (size_t)C, a + r * (size_t)C, sizeof(float) * (size_t)C);
  }
  free(a);
  free(c);
}

/* ---------------------------------------------------------------- CNN */
typedef struct {
  int fi, fo, po;
  float* w;  /* [fo][fi] */
  float* wt; /* [fi][po] */
  float* b;  /* [po] */
} orc_layer;

static void layer_init(orc_layer* L, uint64_t seed, int l, int fi, int fo, int quantize) {
  L->fi = fi;
  L->fo = fo;
  L->po = (fo + 15) / 16 * 16;
  L->w = (float*)malloc(sizeof(float) * (size_t)fi * fo);
  L->wt = (float*)calloc((size_t)fi * L->po, sizeof(float));
  L->b = (float*)calloc((size_t)L->po, sizeof(float));
  for (int o = 0; o < fo; ++o) {
    for (int i = 0; i < fi; ++i) {
      uint64_t idx = (uint64_t)o * fi + i;
      float v = orc_weight(seed, l, idx, fi, fo);
      if (quantize) v = orc_round_bf16(v);
      L->w[idx] = v;
      L->wt[(size_t)i * L->po + o] = v;
    }
    L->b[o] = orc_bias(seed, l, (uint64_t)o);
  }
}

static void layer_free(orc_layer* L) {
  free(L->w);
  free(L->wt);
  free(L->b);
}

/* y[rows][po] for rows a multiple of RB (x rows of stride fi). */
static void layer_apply(const orc_layer* L, const float* x, size_t rows, int relu_q, int quantize,
                        float* y) {
  for (size_t r = 0; r < rows; r += RB)
    dense_block(x + r * (size_t)L->fi, L->fi, L->wt, L->b, L->po, relu_q, quantize,
                y + r * (size_t)L->po);
}

struct orc_cnn {
  int S, P, G, c1, c2, hidden, C, quantize;
  orc_layer L[4];
};

orc_cnn* orc_cnn_create(int S, int P, int c1, int c2, int hidden, int C, uint64_t seed,
                        int quantize_bf16) {
  if (P < 1 || S < P || S % P != 0 || c1 < 1 || c2 < 1 || hidden < 1 || C < 1) return NULL;
  orc_cnn* m = (orc_cnn*)calloc(1, sizeof(orc_cnn));
  m->S = S;
  m->P = P;
  m->G = S / P;
  m->c1 = c1;
  m->c2 = c2;
  m->hidden = hidden;
  m->C = C;
  m->quantize = quantize_bf16;
  layer_init(&m->L[0], seed, 0, P * P, c1, quantize_bf16);
  layer_init(&m->L[1], seed, 1, 9 * c1, c2, quantize_bf16);
  layer_init(&m->L[2], seed, 2, m->G * m->G * c2, hidden, quantize_bf16);
  layer_init(&m->L[3], seed, 3, hidden, C, quantize_bf16);
  return m;
}

void orc_cnn_destroy(orc_cnn* m) {
  if (!m) return;
  for (int l = 0; l < 4; ++l) layer_free(&m->L[l]);
  free(m);
}

int orc_cnn_classes(const orc_cnn* m) { return m->C; }

void orc_cnn_layer(const orc_cnn* m, int l, float* w, float* b) {
  const orc_layer* L = &m->L[l];
  if (w) memcpy(w, L->w, sizeof(float) * (size_t)L->fi * L->fo);
  if (b) memcpy(b, L->b, sizeof(float) * (size_t)L->fo);
}

/* Logits and/or hidden activations, RB samples at a time. */
static void cnn_run(const orc_cnn* m, const float* x, size_t rows, float* logits, float* hid) {
  const int S = m->S, P = m->P, G = m->G, G2 = G * G, c1 = m->c1, c2 = m->c2;
  const size_t gp = (size_t)(G2 + RB - 1) / RB * RB; /* pixel rows, padded to RB */
  const int po1 = m->L[0].po, po2 = m->L[1].po, poh = m->L[2].po, poc = m->L[3].po;
  const int feat = G2 * c2;
  float* x1 = (float*)calloc(gp * (size_t)(P * P), sizeof(float));
  float* y1 = (float*)calloc(gp * (size_t)po1, sizeof(float));
  float* x2 = (float*)calloc(gp * (size_t)(9 * c1), sizeof(float));
  float* y2 = (float*)calloc(gp * (size_t)po2, sizeof(float));
  float* f = (float*)calloc((size_t)RB * feat, sizeof(float));
  float* h = (float*)calloc((size_t)RB * poh, sizeof(float));
  float* hc = (float*)calloc((size_t)RB * m->hidden, sizeof(float));
  float* z = (float*)calloc((size_t)RB * poc, sizeof(float));
  for (size_t r0 = 0; r0 < rows; r0 += RB) {
    const size_t nr = rows - r0 < RB ? rows - r0 : RB;
    memset(f, 0, sizeof(float) * (size_t)RB * feat);
    for (size_t s = 0; s < nr; ++s) {
      const float* img = x + (r0 + s) * (size_t)(S * S);
      for (int p = 0; p < G2; ++p) {
        const int i = p / G, j = p % G;
        for (int a = 0; a < P; ++a)
          for (int b = 0; b < P; ++b) {
            float v = img[(P * i + a) * S + P * j + b];
            x1[(size_t)p * (P * P) + a * P + b] = m->quantize ? orc_round_bf16(v) : v;
          }
      }
      layer_apply(&m->L[0], x1, gp, 1, m->quantize, y1);
      for (int p = 0; p < G2; ++p) {
        const int i = p / G, j = p % G;
        for (int t = 0; t < 9; ++t) {
          const int ii = i + t / 3 - 1, jj = j + t % 3 - 1;
          float* dst = x2 + (size_t)p * (9 * c1) + (size_t)t * c1;
          if (ii < 0 || ii >= G || jj < 0 || jj >= G)
            memset(dst, 0, sizeof(float) * (size_t)c1);
          else
            memcpy(dst, y1 + (size_t)(ii * G + jj) * po1, sizeof(float) * (size_t)c1);
        }
      }
      layer_apply(&m->L[1], x2, gp, 1, m->quantize, y2);
      for (int p = 0; p < G2; ++p)
        memcpy(f + s * (size_t)feat + (size_t)p * c2, y2 + (size_t)p * po2, sizeof(float) * (size_t)c2);
    }
    dense_block(f, feat, m->L[2].wt, m->L[2].b, poh, 1, m->quantize, h);
    for (int r = 0; r < RB; ++r)
      memcpy(hc + (size_t)r * m->hidden, h + (size_t)r * poh, sizeof(float) * (size_t)m->hidden);
    if (hid)
      for (size_t r = 0; r < nr; ++r)
        memcpy(hid + (r0 + r) * (size_t)m->hidden, hc + r * (size_t)m->hidden,
               sizeof(float) * (size_t)m->hidden);
    if (logits) {
      dense_block(hc, m->hidden, m->L[3].wt, m->L[3].b, poc, 0, m->quantize, z);
      for (size_t r = 0; r < nr; ++r)
        memcpy(logits + (r0 + r) * (size_t)m->C, z + r * (size_t)poc, sizeof(float) * (size_t)m->C);
    }
  }
  free(x1);
  free(y1);
  free(x2);
  free(y2);
  free(f);
  free(h);
  free(hc);
  free(z);
}

void orc_cnn_forward(const orc_cnn* m, const float* x, size_t rows, float* out) {
  cnn_run(m, x, rows, out, NULL);
}

void orc_cnn_hidden(const orc_cnn* m, const float* x, size_t rows, float* out) {
  cnn_run(m, x, rows, NULL, out);
}

void orc_softmax_rows(const float* z, size_t rows, int C, float* p) {
  for (size_t r = 0; r < rows; ++r) {
    const float* zr = z + r * (size_t)C;
    float* pr = p + r * (size_t)C;
    float mx = zr[0];
    for (int c = 1; c < C; ++c) mx = zr[c] > mx ? zr[c] : mx;
    float s = 0.0f;
    for (int c = 0; c < C; ++c) {
      pr[c] = expf(zr[c] - mx);
      s += pr[c];
    }
    float inv = 1.0f / s;
    for (int c = 0; c < C; ++c) pr[c] = pr[c] * inv;
  }
}

void orc_argmax_rows(const float* y, size_t rows, int C, int32_t* out) {
  for (size_t r = 0; r < rows; ++r) {
    const float* yr = y + r * (size_t)C;
    int best = 0;
    for (int c = 1; c < C; ++c)
      if (yr[c] > yr[best]) best = c;
    out[r] = best;
  }
}

/* combine.cpp:99-135, applied to all rows at once (the per-segment staging of
 * combine.cpp:60-91 does not change the arithmetic: each y element is folded
 * in model-id order starting from +0.0f). */
void orc_fold(int rule, int M, size_t rows, int C, const float* const* blocks,
              const double* weights, float* y, int32_t* winners) {
  size_t n = rows * (size_t)C;
  memset(y, 0, sizeof(float) * n);
  if (rule == 0 || rule == 2) {
    float inv = 1.0f / (float)M;
    for (int m = 0; m < M; ++m) {
      float w = rule == 0 ? inv : (float)weights[m];
      const volatile float* bm = blocks[m];
      for (size_t i = 0; i < n; ++i) {
        float prod = bm[i] * w; /* separate rounding: no FMA contraction */
        volatile float keep = prod;
        y[i] += keep;
      }
    }
    if (winners) orc_argmax_rows(y, rows, C, winners);
    return;
  }
  for (int m = 0; m < M; ++m) {
    const float* bm = blocks[m];
    for (size_t r = 0; r < rows; ++r) {
      int best = 0;
      for (int c = 1; c < C; ++c)
        if (bm[r * (size_t)C + c] > bm[r * (size_t)C + best]) best = c;
      y[r * (size_t)C + best] += 1.0f;
    }
  }
  if (winners) orc_argmax_rows(y, rows, C, winners);
}

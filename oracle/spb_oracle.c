/* TEST INFRASTRUCTURE ONLY -- see spb_oracle.h. Restates the reference SPB
 * path in C, operation for operation, citing the reference file:line each
 * function follows (paths relative to /root/reference/proj). */
#include "spb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { ST_OK = 0, ST_ARGUMENT = 1, ST_PROTOCOL = 2 };

/* ---- Rng: include/jigsaw/rng.hpp:13-58 ---------------------------------- */

/* rng.hpp:47-53 */
uint64_t orc_mix(uint64_t a, uint64_t b) {
  uint64_t z = a ^ (b + 0x9E3779B97F4A7C15ULL + (a << 6) + (a >> 2));
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

orc_rng orc_rng_new(uint64_t key) {
  orc_rng r = {key, 0};
  return r;
}

/* rng.hpp:18 -- a split child starts a fresh counter */
orc_rng orc_rng_split(const orc_rng* r, uint64_t tag) { return orc_rng_new(orc_mix(r->key, tag)); }

/* rng.hpp:20 */
uint64_t orc_next_u64(orc_rng* r) { return orc_mix(r->key, ++r->counter); }

/* rng.hpp:26-29: Lemire multiply-shift on a 128-bit product */
uint64_t orc_next_below(orc_rng* r, uint64_t n) {
  return (uint64_t)(((unsigned __int128)orc_next_u64(r) * n) >> 64);
}

/* rng.hpp:23 */
double orc_next_unit(orc_rng* r) { return (double)(orc_next_u64(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:40-45 (Box-Muller) */
double orc_next_gaussian(orc_rng* r) {
  double u1 = orc_next_unit(r);
  double u2 = orc_next_unit(r);
  if (u1 <= 0.0) u1 = 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

void orc_rng_stream(uint64_t key, const uint64_t* tags, int ntags, int kind, uint64_t bound, int n,
                    uint64_t* out) {
  orc_rng r = orc_rng_new(key);
  for (int i = 0; i < ntags; ++i) r = orc_rng_split(&r, tags[i]);
  for (int i = 0; i < n; ++i) {
    if (kind == 0) {
      out[i] = orc_next_u64(&r);
    } else if (kind == 1) {
      out[i] = orc_next_below(&r, bound);
    } else {
      double d = kind == 2 ? orc_next_unit(&r) : orc_next_gaussian(&r);
      memcpy(&out[i], &d, sizeof d);
    }
  }
}

/* draw_batch spb.cpp:127-131 on stream Rng(seed).split(s).split(j)
 * (spb.cpp:176,187,141). */
void orc_draw_batch(uint64_t seed, int step, int worker, int count, int dataset_size, int* out) {
  orc_rng root = orc_rng_new(seed);
  orc_rng st = orc_rng_split(&root, (uint64_t)step);
  orc_rng w = orc_rng_split(&st, (uint64_t)worker);
  for (int i = 0; i < count; ++i) out[i] = (int)orc_next_below(&w, (uint64_t)dataset_size);
}

/* ---- bookkeeping: spb.cpp:16-49 ----------------------------------------- */

/* spb.cpp:16-21 */
int orc_suffix_layers(int j, int k, int L, int* out) {
  if (k < 1 || L < 1) return ST_ARGUMENT;
  if (j < 1 || j > k) return ST_ARGUMENT;
  *out = (int)(((long long)j * L + k - 1) / k);
  return ST_OK;
}

/* spb.cpp:23-29 */
int orc_chunk_coverage(int m, int k, int* out) {
  if (k < 1) return ST_ARGUMENT;
  if (m < 1 || m > k) return ST_ARGUMENT;
  for (int i = 0; i < m; ++i) out[i] = k - m + 1 + i;
  return ST_OK;
}

/* spb.cpp:31-41; out[2(m-1)], out[2(m-1)+1] = first, last of chunk m */
int orc_chunk_layout(int k, int L, int* out) {
  if (k < 1 || L < 1) return ST_ARGUMENT;
  for (int m = 1; m <= k; ++m) {
    int s_hi, s_lo = 0;
    orc_suffix_layers(k - m + 1, k, L, &s_hi);
    if (m != k) orc_suffix_layers(k - m, k, L, &s_lo);
    out[2 * (m - 1)] = L - s_hi + 1;
    out[2 * (m - 1) + 1] = (m == k) ? L : L - s_lo;
  }
  return ST_OK;
}

/* spb.cpp:43-49 */
int orc_layer_chunks(int k, int L, int* out) {
  if (k < 1 || L < 1) return ST_ARGUMENT;
  int* spans = (int*)malloc(sizeof(int) * 2 * (size_t)k);
  orc_chunk_layout(k, L, spans);
  for (int l = 0; l < L; ++l) out[l] = 0;
  for (int m = 1; m <= k; ++m)
    for (int l = spans[2 * (m - 1)]; l <= spans[2 * (m - 1) + 1]; ++l) out[l - 1] = m;
  free(spans);
  return ST_OK;
}

/* ---- ChainMlp: model.cpp:86-186, 208-231 -------------------------------- */

static long block_len(const int* widths, int l /* 0-based */) {
  return (long)widths[l + 1] * widths[l] + widths[l + 1];
}

/* make_random_chain_mlp model.cpp:208-231 (stream Rng(seed).split(0x313a)) */
void orc_gen_chain_mlp(const int* widths, int nw, int samples, uint64_t seed, double* X, double* Y,
                       double* const* W) {
  orc_rng root = orc_rng_new(seed);
  orc_rng rng = orc_rng_split(&root, 0x313aULL);
  int L = nw - 1;
  for (int l = 0; l < L; ++l) {
    long n = block_len(widths, l);
    double scale = 1.0 / sqrt((double)widths[l]);
    for (long i = 0; i < n; ++i) W[l][i] = scale * (2.0 * orc_next_unit(&rng) - 1.0);
  }
  for (int s = 0; s < samples; ++s) {
    double t = 0.0;
    for (int i = 0; i < widths[0]; ++i) {
      double v = orc_next_gaussian(&rng);
      X[(size_t)s * widths[0] + i] = v;
      t += v;
    }
    Y[s] = tanh(t) + 0.1 * orc_next_gaussian(&rng);
  }
}

/* mlp_forward model.cpp:108-128. acts[l] has widths[l] entries; acts[0] is
 * the input. The last layer is affine, the others tanh. */
static void forward(const int* widths, int L, const double* const* x, const double* input,
                    double** acts) {
  memcpy(acts[0], input, sizeof(double) * (size_t)widths[0]);
  for (int l = 1; l <= L; ++l) {
    int out_w = widths[l], in_w = widths[l - 1];
    const double* Wm = x[l - 1];
    const double* bias = Wm + (long)out_w * in_w;
    const double* prev = acts[l - 1];
    for (int o = 0; o < out_w; ++o) {
      double z = bias[o];
      const double* wrow = Wm + (long)o * in_w;
      for (int i = 0; i < in_w; ++i) z += wrow[i] * prev[i];
      acts[l][o] = (l == L) ? z : tanh(z);
    }
  }
}

static double** alloc_acts(const int* widths, int L) {
  double** acts = (double**)malloc(sizeof(double*) * (size_t)(L + 1));
  for (int l = 0; l <= L; ++l) acts[l] = (double*)malloc(sizeof(double) * (size_t)widths[l]);
  return acts;
}

static void free_acts(double** acts, int L) {
  for (int l = 0; l <= L; ++l) free(acts[l]);
  free(acts);
}

/* model.cpp:131-137; the 0.5*||out-y||^2 generalisation to n_L > 1 is the
 * throughput variant (parity unpinned: the reference rejects n_L != 1,
 * model.cpp:93). */
double orc_sample_loss(const int* widths, int L, const double* const* x, const double* input,
                       const double* target) {
  double** acts = alloc_acts(widths, L);
  forward(widths, L, x, input, acts);
  double loss = 0.0;
  for (int o = 0; o < widths[L]; ++o) {
    double d = acts[L][o] - target[o];
    loss += 0.5 * d * d;
  }
  free_acts(acts, L);
  return loss;
}

/* ChainMlp::loss model.cpp:139-143 */
double orc_loss(const int* widths, int L, const double* const* x, const double* X, const double* Y,
                int N) {
  double total = 0.0;
  for (int s = 0; s < N; ++s)
    total += orc_sample_loss(widths, L, x, X + (size_t)s * widths[0], Y + (size_t)s * widths[L]);
  return total / N;
}

/* ChainMlp::add_sample_gradient model.cpp:145-186 */
int orc_add_sample_gradient(const int* widths, int L, const double* const* x, const double* input,
                            const double* target, int suffix, double* const* acc,
                            long long* layer_ops) {
  if (suffix < 1 || suffix > L) return ST_ARGUMENT;
  double** acts = alloc_acts(widths, L);
  forward(widths, L, x, input, acts);
  int maxw = 0;
  for (int l = 0; l <= L; ++l)
    if (widths[l] > maxw) maxw = widths[l];
  double* delta = (double*)malloc(sizeof(double) * (size_t)maxw);
  double* next = (double*)malloc(sizeof(double) * (size_t)maxw);
  int stop = L - suffix + 1;
  for (int o = 0; o < widths[L]; ++o) delta[o] = acts[L][o] - target[o]; /* model.cpp:156 */
  for (int l = L; l >= stop; --l) {
    int out_w = widths[l], in_w = widths[l - 1];
    const double* Wm = x[l - 1];
    double* gW = acc[l - 1];
    double* gb = gW + (long)out_w * in_w;
    const double* prev = acts[l - 1];
    long long ops = 0;
    for (int o = 0; o < out_w; ++o) { /* wgrad model.cpp:165-171 */
      double d = delta[o];
      double* grow = gW + (long)o * in_w;
      for (int i = 0; i < in_w; ++i) grow[i] += d * prev[i];
      gb[o] += d;
      ops += in_w + 1;
    }
    if (l > stop) { /* dgrad model.cpp:172-183 */
      for (int i = 0; i < in_w; ++i) next[i] = 0.0;
      for (int o = 0; o < out_w; ++o) {
        double d = delta[o];
        const double* wrow = Wm + (long)o * in_w;
        for (int i = 0; i < in_w; ++i) next[i] += d * wrow[i];
      }
      for (int i = 0; i < in_w; ++i) next[i] *= 1.0 - prev[i] * prev[i];
      ops += (long long)out_w * in_w + in_w;
      double* t = delta;
      delta = next;
      next = t;
    }
    if (layer_ops) layer_ops[l - 1] += ops;
  }
  free(delta);
  free(next);
  free_acts(acts, L);
  return ST_OK;
}

/* partial_backprop spb.cpp:51-68. Covered blocks out_blocks[l-1] (l >=
 * covered_from) are overwritten with the batch mean; absent ones are not
 * touched (the reference leaves them empty). */
int orc_partial_backprop(const int* widths, int L, const double* X, const double* Y, int N,
                         const double* const* x, const int* batch, int len, int suffix,
                         double* const* out_blocks, long long* layer_ops, int* covered_from) {
  if (suffix < 1 || suffix > L) return ST_ARGUMENT;
  if (len <= 0) return ST_ARGUMENT;
  for (int i = 0; i < len; ++i)
    if (batch[i] < 0 || batch[i] >= N) return ST_ARGUMENT; /* model.cpp:150 */
  int from = L - suffix + 1;
  if (covered_from) *covered_from = from;
  for (int l = from; l <= L; ++l) memset(out_blocks[l - 1], 0, sizeof(double) * (size_t)block_len(widths, l - 1));
  for (int i = 0; i < len; ++i) {
    int s = batch[i];
    orc_add_sample_gradient(widths, L, x, X + (size_t)s * widths[0], Y + (size_t)s * widths[L],
                            suffix, out_blocks, layer_ops);
  }
  double inv = 1.0 / (double)len;
  for (int l = from; l <= L; ++l) {
    long n = block_len(widths, l - 1);
    for (long c = 0; c < n; ++c) out_blocks[l - 1][c] *= inv;
  }
  return ST_OK;
}

/* aggregate spb.cpp:70-106. blocks[j*L + l] = worker j+1's block l+1 (NULL
 * when absent), dims the matching lengths. */
int orc_aggregate(int k, int L, const double* const* blocks, const int* dims,
                  const int* covered_from, double* const* out) {
  if (k < 1) return ST_ARGUMENT;
  for (int j = 1; j <= k; ++j) { /* spb.cpp:74-87 */
    int s;
    orc_suffix_layers(j, k, L, &s);
    if (covered_from[j - 1] != L - s + 1) return ST_PROTOCOL;
    for (int l = 1; l <= L; ++l) {
      int present = blocks[(j - 1) * L + (l - 1)] != NULL && dims[(j - 1) * L + (l - 1)] > 0;
      if (present != (l >= covered_from[j - 1])) return ST_PROTOCOL;
    }
  }
  int* chunk_of = (int*)malloc(sizeof(int) * (size_t)L);
  orc_layer_chunks(k, L, chunk_of);
  int st = ST_OK;
  for (int l = 1; l <= L && st == ST_OK; ++l) { /* spb.cpp:91-104 */
    int m = chunk_of[l - 1];
    int first = k - m + 1;
    int dim = dims[(first - 1) * L + (l - 1)];
    double* dst = out[l - 1];
    for (int c = 0; c < dim; ++c) dst[c] = 0.0;
    for (int w = first; w <= k; ++w) {
      const double* src = blocks[(w - 1) * L + (l - 1)];
      if (dims[(w - 1) * L + (l - 1)] != dim) {
        st = ST_PROTOCOL;
        break;
      }
      for (int c = 0; c < dim; ++c) dst[c] += src[c];
    }
    double inv = 1.0 / (double)m;
    for (int c = 0; c < dim; ++c) dst[c] *= inv;
  }
  free(chunk_of);
  return st;
}

/* One SPB-SGD iteration, the body of spb_sgd_run spb.cpp:187-196 (Constant
 * schedule; spb_estimate :135-145 or baseline_estimate :149-160 when full),
 * without the diagnostic loss(xbar) of :202. x is updated in place. */
int orc_spb_step(const int* widths, int L, const double* X, const double* Y, int N,
                 double* const* x, int k, int B, double lr, uint64_t seed, int s, int full) {
  if (k < 1 || B < 1 || B % k != 0) return ST_ARGUMENT; /* spb.cpp:11-14 */
  int per = B / k;
  double** grads = (double**)calloc((size_t)k * L, sizeof(double*));
  int* dims = (int*)calloc((size_t)k * L, sizeof(int));
  int* cov = (int*)malloc(sizeof(int) * (size_t)k);
  int* batch = (int*)malloc(sizeof(int) * (size_t)per);
  int st = ST_OK;
  for (int j = 1; j <= k && st == ST_OK; ++j) {
    int suffix = L;
    if (!full) orc_suffix_layers(j, k, L, &suffix);
    orc_draw_batch(seed, s, j, per, N, batch);
    for (int l = L - suffix + 1; l <= L; ++l) {
      dims[(j - 1) * L + l - 1] = (int)block_len(widths, l - 1);
      grads[(j - 1) * L + l - 1] = (double*)malloc(sizeof(double) * (size_t)block_len(widths, l - 1));
    }
    st = orc_partial_backprop(widths, L, X, Y, N, (const double* const*)x, batch, per, suffix,
                              grads + (size_t)(j - 1) * L, NULL, &cov[j - 1]);
  }
  if (st == ST_OK) {
    double** g = (double**)malloc(sizeof(double*) * (size_t)L);
    for (int l = 0; l < L; ++l) g[l] = (double*)calloc((size_t)block_len(widths, l), sizeof(double));
    if (full) { /* axpy(mean, 1.0/k, g_j) spb.cpp:157 */
      for (int j = 0; j < k; ++j)
        for (int l = 0; l < L; ++l) {
          long n = block_len(widths, l);
          for (long c = 0; c < n; ++c) g[l][c] += (1.0 / k) * grads[j * L + l][c];
        }
    } else {
      st = orc_aggregate(k, L, (const double* const*)grads, dims, cov, g);
    }
    if (st == ST_OK) /* axpy(x, -gamma, g) spb.cpp:196, spb.cpp:120-123 */
      for (int l = 0; l < L; ++l) {
        long n = block_len(widths, l);
        for (long c = 0; c < n; ++c) x[l][c] += -lr * g[l][c];
      }
    for (int l = 0; l < L; ++l) free(g[l]);
    free(g);
  }
  for (long i = 0; i < (long)k * L; ++i) free(grads[i]);
  free(grads);
  free(dims);
  free(cov);
  free(batch);
  return st;
}

/* Momentum SGD + weight decay as the paper's experiments use it
 * (PAPER.md:9-10). NOT in the reference (spb.cpp:196 is plain SGD): restated
 * with PyTorch SGD semantics (no dampening, no Nesterov; the first step sets
 * buf = g'). Parity unpinned by the reference. */
void orc_sgd_momentum(long n, double* w, const double* g, double* buf, double lr, double momentum,
                      double weight_decay, int first_step) {
  for (long i = 0; i < n; ++i) {
    double gi = g[i] + weight_decay * w[i];
    double step = gi;
    if (momentum != 0.0) {
      buf[i] = first_step ? gi : momentum * buf[i] + gi;
      step = buf[i];
    }
    w[i] -= lr * step;
  }
}

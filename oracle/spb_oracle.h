/* TEST INFRASTRUCTURE ONLY -- the CPU oracle for the SPB hot path.
 *
 * A plain-C, fp64 restatement of the reference's SPB training step
 * (/root/reference/proj/src/spb/{spb,model}.cpp, include/jigsaw/rng.hpp).
 * Every function cites the reference lines it follows and keeps the same
 * floating-point operation order, so compiled with -O2 -ffp-contract=off it
 * is bit-identical to the reference (pinned in tests/test_oracle.py against
 * oracle/_ref/libjigsaw_ref.so and tests/golden/). Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU legs may load it; the product
 * (paper_2111_10672_b200/) never does.
 *
 * Layout conventions (the reference's Params, model.hpp:11,93-94): params are
 * L blocks; block l (0-based) holds W_{l+1} row-major [n_{l+1} x n_l] followed
 * by b_{l+1} [n_{l+1}]. Datasets are row-major X [N x n_0], Y [N x n_L].
 *
 * Status codes follow include/spb_b200.h: 0 ok, 1 ArgumentError,
 * 2 ProtocolError, 3 ConfigError.
 */
#ifndef SPB_ORACLE_H
#define SPB_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t key;
  uint64_t counter;
} orc_rng;

uint64_t orc_mix(uint64_t a, uint64_t b);
orc_rng orc_rng_new(uint64_t key);
orc_rng orc_rng_split(const orc_rng* r, uint64_t tag);
uint64_t orc_next_u64(orc_rng* r);
uint64_t orc_next_below(orc_rng* r, uint64_t n);
double orc_next_unit(orc_rng* r);
double orc_next_gaussian(orc_rng* r);
void orc_rng_stream(uint64_t key, const uint64_t* tags, int ntags, int kind, uint64_t bound, int n,
                    uint64_t* out);
void orc_draw_batch(uint64_t seed, int step, int worker, int count, int dataset_size, int* out);

int orc_suffix_layers(int j, int k, int L, int* out);
int orc_chunk_coverage(int m, int k, int* out);
int orc_chunk_layout(int k, int L, int* out);
int orc_layer_chunks(int k, int L, int* out);

void orc_gen_chain_mlp(const int* widths, int nw, int samples, uint64_t seed, double* X, double* Y,
                       double* const* W);

int orc_add_sample_gradient(const int* widths, int L, const double* const* x, const double* input,
                            const double* target, int suffix, double* const* acc,
                            long long* layer_ops);
double orc_sample_loss(const int* widths, int L, const double* const* x, const double* input,
                       const double* target);
double orc_loss(const int* widths, int L, const double* const* x, const double* X, const double* Y,
                int N);
int orc_partial_backprop(const int* widths, int L, const double* X, const double* Y, int N,
                         const double* const* x, const int* batch, int len, int suffix,
                         double* const* out_blocks, long long* layer_ops, int* covered_from);
int orc_aggregate(int k, int L, const double* const* blocks, const int* dims,
                  const int* covered_from, double* const* out);
int orc_spb_step(const int* widths, int L, const double* X, const double* Y, int N,
                 double* const* x, int k, int B, double lr, uint64_t seed, int s, int full);
void orc_sgd_momentum(long n, double* w, const double* g, double* buf, double lr, double momentum,
                      double weight_decay, int first_step);

#ifdef __cplusplus
}
#endif
#endif

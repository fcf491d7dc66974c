/*
 * spb_b200.h -- C ABI of the B200-native Structured Partial Backpropagation
 * (SPB) training step (arXiv 2111.10672). libspb_b200.so exports exactly the
 * functions below; everything is plain pointers and sizes, no torch or C++
 * types. Each entry point names the reference interface it replaces
 * (/root/reference/proj, file:line).
 *
 * Conventions
 *  - Status codes: every call returns spb_status. The reference throws
 *    jigsaw::ArgumentError / ProtocolError / ConfigError
 *    (include/jigsaw/errors.hpp:9-25); exceptions cannot cross a C ABI, so the
 *    same conditions return SPB_E_ARGUMENT / SPB_E_PROTOCOL / SPB_E_CONFIG and
 *    spb_last_error() holds the message. CUDA / NCCL failures are
 *    SPB_E_CUDA / SPB_E_NCCL. The C++ adapter (include/spb_b200/jigsaw_spb.hpp)
 *    rethrows the reference exception types.
 *  - Layer numbering is the reference's: layers 1..L, input side first;
 *    workers 1..k; chunks 1..k (spb.hpp:13-18).
 *  - Parameter blocks use the reference Params layout (model.hpp:93-94):
 *    block l (0-based pointer index l-1) = W_l row-major [n_l x n_{l-1}]
 *    followed by b_l [n_l], i.e. n_l*n_{l-1} + n_l floats. Values are fp32.
 *  - Datasets: X row-major [N x n_0], Y row-major [N x n_L].
 *  - A context (spb_ctx) owns device state on one GPU and one CUDA stream.
 *    It is not thread-safe (the reference's const/thread-safe model methods,
 *    model.hpp:21-25, are mirrored by one context per thread).
 */
#ifndef SPB_B200_H
#define SPB_B200_H
#include <stddef.h>
#include <stdint.h>

#if defined(SPB_BUILD_LIB)
#define SPB_API __attribute__((visibility("default")))
#else
#define SPB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPB_OK = 0,
  SPB_E_ARGUMENT = 1, /* jigsaw::ArgumentError */
  SPB_E_PROTOCOL = 2, /* jigsaw::ProtocolError */
  SPB_E_CONFIG = 3,   /* jigsaw::ConfigError */
  SPB_E_CUDA = 4,
  SPB_E_NCCL = 5
} spb_status;

typedef struct spb_ctx spb_ctx;

/* Message of the last failing call on this thread (context-free calls) or
 * on ctx (context calls; ctx may be NULL). Never NULL. */
SPB_API const char* spb_last_error(const spb_ctx* ctx);

/* ---- SPB bookkeeping: integer-exact host code -------------------------------
 * Replaces suffix_layers spb.hpp:39 (spb.cpp:16-21). Worker j of k on an
 * L-layer model backpropagates ceil(j*L/k) layers. */
SPB_API spb_status spb_suffix_layers(int j, int k, int L, int* out);
/* chunk_coverage spb.hpp:42 (spb.cpp:23-29): workers {k-m+1..k} into out[0..m). */
SPB_API spb_status spb_chunk_coverage(int m, int k, int* out);
/* chunk_layout spb.hpp:46 (spb.cpp:31-41): out[2(m-1)], out[2(m-1)+1] =
 * first, last layer of chunk m (first > last when the chunk is empty). */
SPB_API spb_status spb_chunk_layout(int k, int L, int* out);
/* layer_chunks spb.hpp:49 (spb.cpp:43-49): out[l-1] = chunk of layer l =
 * number of contributing workers of layer l. */
SPB_API spb_status spb_layer_chunks(int k, int L, int* out);
/* draw_batch (spb.cpp:127-131) on the stream Rng(seed).split(step).split(worker)
 * (spb.cpp:176,187,141): count sample indices in [0, dataset_size). */
SPB_API spb_status spb_draw_batch(uint64_t seed, int step, int worker, int count, int dataset_size, int* out);
/* Worker placement for multi-GPU runs: the workers (1-based, ascending) that
 * rank `rank` of `nranks` hosts: one each when nranks == k; below 4 ranks
 * balanced pairs (j, k+1-j), so every rank carries the same backward work;
 * from 4 ranks contiguous blocks (fewer contributing ranks per layer, fewer
 * exchange bytes; measured faster there). SPB_PLACEMENT=balanced|contiguous
 * overrides. Writes *count entries to out (size >= k). */
SPB_API spb_status spb_rank_workers(int k, int L, int rank, int nranks, int* out, int* count);

/* make_random_chain_mlp (model.hpp:240-241, model.cpp:208-231): the
 * reference's synthetic instance (stream Rng(seed).split(0x313a)), generated
 * in fp64 exactly as the reference does and rounded to fp32. X [samples x n_0],
 * Y [samples x n_L] (the scalar target repeated when n_L > 1), W[l] = block l+1. */
SPB_API spb_status spb_make_random_chain_mlp(const int* widths, int n_widths, int samples, uint64_t seed, float* X,
                                             float* Y, float* const* W);

/* ---- Context: the ChainMlp "layer" (model.hpp:95-111) on one B200 ---------
 * widths[0..n_widths): [n_0, ..., n_L]; n_L <= 16 (the reference requires
 * n_L == 1, model.cpp:93; wider heads are the 0.5*||out-y||^2 throughput
 * variant). k workers of per_worker_batch samples each may run per step.
 * device < 0: the calling thread's current CUDA device. */
SPB_API spb_status spb_create(const int* widths, int n_widths, int k, int per_worker_batch, int device,
                      spb_ctx** out);
/* ConvNet (BASELINE configs[3]: CIFAR10-shaped, ResNet18
 * widths): layers 1..nconv are 3x3 convolutions (padding 1) with tanh,
 * lowered to the same tcgen05 GEMMs via im2col; layer nconv+1 is the affine
 * head (nout <= 16) on the globally average-pooled features; per-sample loss
 * 0.5 ||out - y||^2, the ChainMlp's. geom = {in_h, in_w, in_c, then
 * (c_out, stride in {1, 2}) per convolution}. Parameter block l is W_l
 * [c_out x 9 c_in] row-major with columns (ky * 3 + kx) * c_in + ci, then b_l;
 * samples are NHWC images (in_h * in_w * in_c floats). Every other entry
 * point (dataset, params, train_steps, partial_backprop, multi-GPU, profile)
 * takes the context as for a ChainMlp; rows count samples. No reference
 * counterpart: the reference has no convolutional model (parity unpinned). */
SPB_API spb_status spb_create_conv(const int* geom, int nconv, int nout, int k, int per_worker_batch, int device,
                                   spb_ctx** out);
SPB_API spb_status spb_destroy(spb_ctx* ctx);
/* ChainMlp's dataset (model.cpp:86-101), uploaded to HBM. */
SPB_API spb_status spb_set_dataset(spb_ctx* ctx, const float* X, const float* Y, int N);
/* Params in / out (LayeredModel::initial_params, spb_sgd_run's iterate x). */
SPB_API spb_status spb_set_params(spb_ctx* ctx, const float* const* blocks);
SPB_API spb_status spb_get_params(spb_ctx* ctx, float* const* blocks);
/* Where single-GPU steps apply the optimizer:
 *   0: aggregate every layer into the gradient buffer (readable with
 *      spb_get_grads), then one update kernel per layer beside the backward;
 *   1: inside every wgrad GEMM epilogue (W updated in place; the aggregated
 *      gradient is not materialised);
 *   2 (default): inside the epilogue of the layers whose wgrad covers <= 512
 *      contributor rows (where that is cheaper), per-layer kernels otherwise.
 * spb_get_grads after a step is complete only in mode 0. Multi-GPU steps and
 * the ConvNet always use per-layer updates. */
SPB_API spb_status spb_set_fused_update(spb_ctx* ctx, int fused);
/* Cross-step pipelining for spb_train_steps / spb_time_train_steps: up to
 * `steps` (1..16; env SPB_CHAIN; default 1: longer chains measured slower
 * on most configurations) consecutive SPB iterations are
 * captured into ONE CUDA graph in which iteration t+1's forward of layer l
 * waits only for W_l of iteration t (its update and, multi-GPU, its exchange)
 * instead of for the whole iteration, so the exchange / update tail of one
 * iteration overlaps the next forward. Results are identical for every value
 * (the same kernels in the same data order); 1 = one graph per iteration. */
SPB_API spb_status spb_set_chain(spb_ctx* ctx, int steps);
/* Timeline of `steps` (1..16) chained SPB iterations, as replayed from ONE
 * graph (diagnostic; no reference counterpart): a %globaltimer stamp kernel
 * on the op's stream before and after every op (GEMMs, reductions, updates,
 * exchanges, p2p flag waits). Per op (up to cap): begin / end ns, class
 * (0 fwd, 1 wgrad, 2 dgrad, 3 head, 4 colreduce (unused since the bias joined
 * the wgrad GEMM), 5 update, 6 gather, 7 comm,
 * 100 wait), stream (0 main, 1 wgrad, 2 update, 3 split, 4 collectives,
 * 10+p / 20+p gradient / weight pulls from peer p), step index in the chain.
 * Parameters advance by `steps` iterations twice (warm-up replay + traced). */
SPB_API spb_status spb_trace_steps(spb_ctx* ctx, uint64_t seed, int step0, int steps, int full_backprop, int cap,
                                   long long* t_begin, long long* t_end, int* cls, int* stream, int* sub, int* n_out);
/* Optimizer: x -= lr * g (spb.cpp:196) when momentum = weight_decay = 0;
 * otherwise momentum SGD + weight decay (PyTorch semantics). */
SPB_API spb_status spb_set_optimizer(spb_ctx* ctx, float lr, float momentum, float weight_decay);

/* ---- Worker: partial_backprop spb.hpp:54-56 (spb.cpp:51-68) ------------------
 * Mean over `batch` (dataset indices, len > 0) of the per-sample gradients of
 * the last `suffix` layers at the context's current params. out_blocks[l-1]
 * receives block l for covered layers l >= L-suffix+1 and is not touched for
 * absent ones (may be NULL). layer_ops (nullable, L entries) is accumulated
 * with the reference's per-layer op counts (model.cpp:165-184). */
SPB_API spb_status spb_partial_backprop(spb_ctx* ctx, const int* batch, int len, int suffix, float* const* out_blocks,
                                long long* layer_ops, int* covered_from);

/* ---- Gradient aggregator: aggregate spb.hpp:61 (spb.cpp:70-106) ---------------
 * blocks[j*L + l] = worker j+1's block l+1 (host fp32, NULL when absent),
 * dims[j*L + l] its length (0 when absent), covered_from[j] its first covered
 * layer. Validates the protocol exactly like the reference, then averages
 * each layer over its contributors on the GPU. out[l] receives layer l+1. */
SPB_API spb_status spb_aggregate(spb_ctx* ctx, int k, int L, const float* const* blocks, const int* dims,
                         const int* covered_from, float* const* out);
/* The same in fp64 (the reference's Params precision), context-free, on
 * `device` (< 0: the calling thread's current CUDA device): per element the
 * contributors are summed in ascending worker order and the sum multiplied by
 * 1.0 / m, exactly the reference's operations (spb.cpp:97-103) with
 * round-to-nearest and no contraction -- bit-identical to the CPU code. */
SPB_API spb_status spb_aggregate64(int device, int k, int L, const double* const* blocks, const int* dims,
                                   const int* covered_from, double* const* out);

/* ---- Training step: one SPB-SGD iteration (spb.cpp:187-196) -------------------
 * Every worker j hosted by this context draws per_worker_batch samples from
 * Rng(seed).split(step).split(j) (on the GPU, bit-exact), runs its forward pass
 * and the backward pass truncated at layer L - ceil(jL/k) + 1, each layer's
 * gradient is averaged over its contributors (x 1/(m_l * per_worker_batch)),
 * and the optimizer updates the params. full_backprop != 0 runs the DP
 * baseline (every worker backpropagates all L layers, plain mean;
 * baseline_estimate spb.cpp:149-160) on the same kernels. The step is
 * captured once as a CUDA graph and replayed `steps` times for steps
 * step0, step0+1, ...; losses (nullable, host) receives each step's mini-batch
 * loss (mean of 0.5*||out-y||^2 over this context's rows). */
SPB_API spb_status spb_train_steps(spb_ctx* ctx, uint64_t seed, int step0, int steps, int full_backprop,
                           float* losses);
/* Same step, but the mini-batch rows come from HOST memory (the reference's
 * model owns a host dataset): X_rows [rows x n_0], Y_rows [rows x n_L] in
 * hosted-worker order, rows = hosted workers * per_worker_batch. Copies in,
 * steps, and copies the loss out (synchronous). */
SPB_API spb_status spb_step_host(spb_ctx* ctx, const float* X_rows, const float* Y_rows, int full_backprop,
                         float* loss_out);
/* spb_step_host without the synchronisation (a training loop's input
 * pipeline): the host rows go to a double-buffered device staging area on
 * the context's copy stream, so the next step's host-to-device copy runs
 * while this step computes; the loss goes to a pinned ring and is written to
 * *loss_out by the next spb_synchronize. X_rows / Y_rows (pinned memory for
 * an asynchronous copy) and loss_out must stay valid and unchanged until
 * then. Same results as spb_step_host. */
SPB_API spb_status spb_step_host_async(spb_ctx* ctx, const float* X_rows, const float* Y_rows, int full_backprop,
                                       float* loss_out);
/* The aggregated per-layer gradient the last unfused step applied
 * (aggregate's output, spb.cpp:70-106, in the Params block layout), or for
 * spb_partial_backprop the covered blocks of the last call. */
SPB_API spb_status spb_get_grads(spb_ctx* ctx, float* const* blocks);
/* ChainMlp::loss (model.cpp:139-143) over the whole uploaded dataset. */
SPB_API spb_status spb_loss(spb_ctx* ctx, double* out);
/* ChainMlp::sample_loss / loss (model.cpp:130-143) in fp64 on the GPU, at the
 * fp64 parameters `blocks` (reference Params layout, L blocks): *out = the sum
 * over samples[0..count) (samples == NULL: the whole dataset) of
 * 0.5 * ||out - y||^2. The reference's precision, for callers that difference
 * losses (the verify suite's finite-difference check, verify.cpp:217-248);
 * the training step itself stays fp32. ChainMlp contexts only. */
SPB_API spb_status spb_loss64(spb_ctx* ctx, const double* const* blocks, const int* samples, int count, double* out);
/* Waits for all work queued on the context's stream. */
SPB_API spb_status spb_synchronize(spb_ctx* ctx);
/* The context's CUDA stream (cudaStream_t), for event timing by callers. */
SPB_API void* spb_stream(spb_ctx* ctx);

/* ---- Multi-GPU: one context per rank, one SPB worker set per GPU --------------
 * unique_id: 128 bytes from spb_comm_unique_id() on rank 0, broadcast by the
 * caller. After this call spb_train_steps runs only this rank's workers
 * (spb_rank_workers) and aggregates each layer over its contributors. The
 * aggregation mode comes from the environment variable SPB_COMM:
 *  - "p2p" (default for 2 ranks): each layer's parameters are sharded over the ranks;
 *    the rank owning a shard pulls the contributors' gradients of it over
 *    NVLink with the copy engines (CUDA IPC), applies the optimizer and the
 *    other ranks pull the updated fp32 shard back, synchronised by
 *    epoch-stamped device flags (no NCCL in the step);
 *  - "sub" (default for a ConvNet over a non-power-of-two rank count, and
 *    above 8 ranks):
 *    NCCL over contributor sub-communicators (ncclCommSplit, one per distinct
 *    contributor-rank set): a layer's gradient is reduce-scattered among the
 *    ranks hosting one of its contributing workers ONLY, each of them updates
 *    its shard, and every member broadcasts its updated fp32 shard to all
 *    ranks (a sole contributor updates the whole layer);
 *  - "rh" (power-of-two rank counts; the ConvNet's default at 4 and 8 ranks): the p2p protocol's buffers with
 *    Rabenseifner's schedule -- recursive-halving reduce-scatter, the owner's
 *    update, recursive-doubling all-gather of the fp32 weights -- so every
 *    copy-engine pull is from ONE peer (single-peer NVLink copies run at
 *    ~760 GB/s, all-to-all pulls at ~450 GB/s);
 *  - "push" (MLP; default from 3 to 8 ranks, e.g. 8 = one SPB worker per GPU):
 *    the wgrad GEMM epilogue stores each
 *    gradient row straight into the owning rank's staging slot (NVLink
 *    stores through CUDA IPC, staged through shared memory into 128-byte row
 *    segments); the owner sums its rows and applies the optimizer; the peers
 *    pull the new fp32 rows (copy engines) and split them into (hi, lo);
 * Ranks of one node only. The placement of workers on ranks: spb_rank_workers. */
SPB_API spb_status spb_comm_unique_id(void* out128);
SPB_API spb_status spb_comm_init(spb_ctx* ctx, const void* unique_id128, int rank, int nranks);
/* Tuning aid (process-wide): k-blocks of K (32 each) the tensor cores
 * accumulate per TMEM chunk before the epilogue folds the chunk into fp32
 * registers, for GEMM kind 0 (forward), 1 (dgrad), 2 (wgrad); kblocks < 1
 * restores the default (4 / 2 / 4). Smaller chunks: less of the tensor
 * core's round-toward-zero accumulation bias, more TMEM drain traffic. Takes
 * effect for graphs captured afterwards (new contexts). */
SPB_API spb_status spb_set_gemm_chunk(int kind, int kblocks);
/* sub mode's shard of a layer segment of `count` floats over `parts` ranks:
 * member i of a layer's contributor set owns [i * shard, min(count, (i + 1) *
 * shard)); shard is a multiple of 4 floats and parts * shard >= count. */
SPB_API spb_status spb_layer_shard(long long count, int parts, long long* shard);
/* Active aggregation mode: 2 p2p, 3 sub, 4 push, 5 rh (-1 before spb_comm_init, 0 one rank). */
SPB_API spb_status spb_comm_mode(spb_ctx* ctx, int* mode);
/* The per-layer contributor plan spb_comm_init sets up (host-only, no GPU):
 * for layer l (index l-1) rank_mask has bit r set when rank r hosts a
 * worker that backpropagates into l (the layer's contributing ranks); kind
 * is 1 (root = that rank) when exactly one rank contributes, else 0. */
SPB_API spb_status spb_bucket_plan(int k, int L, int nranks, int full_backprop, int* kind, int* root,
                                   int* rank_mask);

/* ---- Gradient-noise estimator (spb.hpp:84-101) -----------------------------------
 * empirical_variance (spb.cpp:212-265) at the context's current parameters,
 * on the GPU, with the reference's sampling protocol sample for sample:
 * out = {spb, spb_se, baseline, baseline_se, p_hat[0..k), p_se[0..k)}.
 * cfg.k / cfg.B must match the context (k, k * per_worker_batch); one GPU. */
SPB_API spb_status spb_empirical_variance(spb_ctx* ctx, int k, int B, int trials, uint64_t seed, double* out);

/* ---- Task profiles for the Jigsaw simulator (profile.hpp:20-40) -----------------
 * One worker task on this GPU: forward + head over `rows` samples, then the
 * truncated backward of the top `suffix` layers (partial_backprop,
 * spb.cpp:51-68), each captured as a graph and replayed `reps` times.
 * forward_ms: forward + head; backward_ms: the additional time of the
 * backward; peak_mem_gb: the task's device working set (parameters as hi/lo,
 * covered gradient blocks, activations, Delta buffers), in 1e9 bytes. These
 * fill one ProfileEntry knot at fraction suffix / L (profile.cpp:118-171). */
SPB_API spb_status spb_profile_task(spb_ctx* ctx, int rows, int suffix, int reps, float* forward_ms, float* backward_ms,
                                    double* peak_mem_gb);

/* ---- Introspection for tests and the bench ----------------------------------- */
/* Batch indices the last device-drawn step used (rows in hosted-worker order). */
SPB_API spb_status spb_last_batch(spb_ctx* ctx, int* out, int rows);
/* Number of this library's kernel launches per step of the last
 * spb_train_steps / spb_step_host call (the captured graph's kernel nodes). */
SPB_API spb_status spb_launches_per_step(spb_ctx* ctx, int* out);

/* One SPB step run eagerly (not from the graph) with CUDA events around every
 * launch. Per kernel class c (0 forward GEMM, 1 wgrad GEMM, 2 dgrad GEMM,
 * 3 head, 4 bias/head-gradient reductions, 5 optimizer update, 6 gather,
 * 7 collectives): ms[c] summed launch time, work[c] algorithmic work (GEMM
 * FLOPs 2*M*N*K; update HBM bytes), launches[c]; step_ms the whole step. */
SPB_API spb_status spb_profile_step(spb_ctx* ctx, uint64_t seed, int step, int full_backprop, int ncls, float* ms,
                                    double* work, int* launches, float* step_ms);
/* spb_train_steps timed with CUDA events on the context's stream (ms total). */
SPB_API spb_status spb_time_train_steps(spb_ctx* ctx, uint64_t seed, int step0, int steps, int full_backprop,
                                        float* ms);

#ifdef __cplusplus
}
#endif
#endif /* SPB_B200_H */

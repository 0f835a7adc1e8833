/*
 * scmoe.h -- C ABI of the B200-native ScMoE layer (LongCat-Flash shortcut-
 * connected MoE with zero-computation experts).
 *
 * This is the drop-in boundary for the reference's hot path (moelab,
 * /root/reference/proj/include/moelab).  Every entry point names the
 * reference function it replaces.  Plain C: opaque handles, plain pointers
 * and sizes, int status codes; no C++ or torch types.
 *
 * Two tiers:
 *   - device tier: pointers are device pointers, calls are stream-ordered on
 *     the context's stream and return as soon as the work is enqueued;
 *   - host tier (suffix _host): pointers are host pointers, the call copies
 *     inputs in, runs the device tier and copies results out before it
 *     returns.  This is what the C++ compat headers (include/moelab_b200/)
 *     and the reference-facing bindings use.
 *
 * Errors: a C ABI cannot throw, so the reference's exception taxonomy
 * (common.hpp:11-33) is returned as a status code; scmoe_last_error(ctx)
 * gives the message.  Host-checkable errors (ConfigError, DimensionError)
 * are returned by the call itself.  Data-dependent errors found on the
 * device by device-tier calls (StateError for an expert index out of range,
 * blocks.hpp:375-377) are latched in the context and returned by the next
 * scmoe_synchronize(ctx); host-tier calls always synchronize and return them
 * directly.
 *
 * Thread safety: no global mutable state; one context per calling thread.
 */
#ifndef SCMOE_H
#define SCMOE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SCMOE_OK = 0,
    SCMOE_ERR_CONFIG = 1,    /* moelab::ConfigError    (common.hpp:21) */
    SCMOE_ERR_DIMENSION = 2, /* moelab::DimensionError (common.hpp:13) */
    SCMOE_ERR_STATE = 3,     /* moelab::StateError     (common.hpp:25) */
    SCMOE_ERR_PARAMETER = 4, /* moelab::ParameterError (common.hpp:17) */
    SCMOE_ERR_CUDA = 5,      /* device / driver failure (no reference equivalent) */
    SCMOE_ERR_INTERNAL = 6
} scmoe_status;

/* Expert-bank storage precision. */
typedef enum {
    SCMOE_PREC_F32_EXACT = 0, /* fp32 weights in the reference layout; sequential-k SIMT
                                 kernels, bitwise equal to moe_forward<float> */
    SCMOE_PREC_BF16 = 1,      /* bf16 weights, transposed K-major for the tcgen05 grouped
                                 GEMM (fp32 accumulate); rel-L2 <= 2e-2 vs the oracle */
    SCMOE_PREC_F64_EXACT = 2  /* fp64 weights in the reference layout (ExpertBank<double>);
                                 bitwise equal to moe_forward<double>; scmoe_*_f64 calls */
} scmoe_precision;

/* GammaMode (blocks.hpp:185): FfnOnly / All / Off. */
typedef enum { SCMOE_GAMMA_FFN_ONLY = 0, SCMOE_GAMMA_ALL = 1, SCMOE_GAMMA_OFF = 2 } scmoe_gamma_mode;

typedef struct scmoe_ctx scmoe_ctx;
typedef struct scmoe_router scmoe_router;
typedef struct scmoe_bank scmoe_bank;

/* ---- context ------------------------------------------------------------ */
int scmoe_ctx_create(int device, scmoe_ctx** out);
int scmoe_ctx_destroy(scmoe_ctx* ctx);
const char* scmoe_last_error(const scmoe_ctx* ctx);
/* Use a caller-owned cudaStream_t (NULL restores the context's own stream). */
int scmoe_set_stream(scmoe_ctx* ctx, void* cuda_stream);
void* scmoe_get_stream(const scmoe_ctx* ctx);
/* Waits for the stream; returns (and clears) any latched device-side error. */
int scmoe_synchronize(scmoe_ctx* ctx);
/* SM budget of this context's persistent kernels (CTAs of the exact router /
 * the grouped GEMM; 0 = every SM).  A context whose GEMMs run beside NCCL
 * collectives (e.g. the dense branch under the EP all-to-all) leaves SMs
 * free for the communication kernels this way. */
int scmoe_ctx_set_sm_budget(scmoe_ctx* ctx, int router_sms, int gemm_sms);
/* Schedule hint for callers that pipeline batches themselves (e.g. expert
 * parallelism): on = this context's router launches use the small kernel that
 * co-resides with a grouped GEMM running on another stream. */
int scmoe_ctx_set_overlapped(scmoe_ctx* ctx, int on);
/* Number of kernels this context has launched (instrumentation). */
uint64_t scmoe_kernel_launches(const scmoe_ctx* ctx);
const char* scmoe_version(void);

/* Device memory helpers for callers without their own allocator. */
int scmoe_device_alloc(scmoe_ctx* ctx, size_t bytes, void** out);
int scmoe_device_free(scmoe_ctx* ctx, void* p);
int scmoe_copy_h2d(scmoe_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes);
int scmoe_copy_d2h(scmoe_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes);

/* ---- router: RouterState<float> (router.hpp:20-62) ------------------------ */
/* Constructor + validate(); ConfigError exactly where RouterState throws. */
int scmoe_router_create(scmoe_ctx* ctx, size_t d_model, size_t n_ffn, size_t n_zero,
                        size_t top_k, size_t k_expected, double mu, double mu_decay,
                        scmoe_router** out);
int scmoe_router_destroy(scmoe_ctx* ctx, scmoe_router* r);
/* w: [d_model, n_ffn+n_zero] row-major fp32 (RouterState::w). */
int scmoe_router_set_weights_host(scmoe_ctx* ctx, scmoe_router* r, const float* w);
int scmoe_router_set_weights(scmoe_ctx* ctx, scmoe_router* r, const float* w_dev);
/* b: [E] doubles; ConfigError if a zero-expert bias is non-zero (router.hpp:59-60). */
int scmoe_router_set_bias_host(scmoe_ctx* ctx, scmoe_router* r, const double* b);
int scmoe_router_get_bias_host(scmoe_ctx* ctx, scmoe_router* r, double* b);
int scmoe_router_set_mu(scmoe_ctx* ctx, scmoe_router* r, double mu, double mu_decay);
int scmoe_router_get_mu(scmoe_ctx* ctx, scmoe_router* r, double* mu, double* mu_decay);
/* tokens_routed [E] u64 and tokens_seen (router.hpp:30-31). */
int scmoe_router_get_counters_host(scmoe_ctx* ctx, scmoe_router* r, uint64_t* tokens_routed,
                                   uint64_t* tokens_seen);
int scmoe_router_set_counters_host(scmoe_ctx* ctx, scmoe_router* r, const uint64_t* tokens_routed,
                                   uint64_t tokens_seen);
/* Device pointer to the router's [E] u64 counters (for EP all-reduce). */
uint64_t* scmoe_router_counters_dev(scmoe_router* r);
const double* scmoe_router_bias_dev(scmoe_router* r);

/* route_topk (router.hpp:133-141): logits = x W (fp32, sequential k, no FMA),
 * softmax_rows (tensor.hpp:174-192, glibc-expf port), biased top-K with
 * lowest-index ties (router.hpp:90-104), unbiased gates.
 *   x [T, d] fp32; indices [T*K] u32; gates [T*K] f64; ffn_count [T] u32;
 *   probs [T, E] fp32 or NULL (router.hpp:139 probs_out). */
int scmoe_route_topk(scmoe_ctx* ctx, scmoe_router* r, const float* x, size_t tokens,
                     uint32_t* indices, double* gates, uint32_t* ffn_count, float* probs);
int scmoe_route_topk_host(scmoe_ctx* ctx, scmoe_router* r, const float* x, size_t tokens,
                          uint32_t* indices, double* gates, uint32_t* ffn_count, float* probs);
/* route_from_probs (router.hpp:107-130) on given probabilities [T, E]. */
int scmoe_route_from_probs_f32(scmoe_ctx* ctx, scmoe_router* r, const float* probs, size_t tokens,
                               uint32_t* indices, double* gates, uint32_t* ffn_count);
int scmoe_route_from_probs_f64(scmoe_ctx* ctx, scmoe_router* r, const double* probs, size_t tokens,
                               uint32_t* indices, double* gates, uint32_t* ffn_count);
int scmoe_route_from_probs_f32_host(scmoe_ctx* ctx, scmoe_router* r, const float* probs,
                                    size_t tokens, uint32_t* indices, double* gates,
                                    uint32_t* ffn_count);
int scmoe_route_from_probs_f64_host(scmoe_ctx* ctx, scmoe_router* r, const double* probs,
                                    size_t tokens, uint32_t* indices, double* gates,
                                    uint32_t* ffn_count);
/* Routing statistics of one decision, from a device
 * histogram of the slots: mean / std of activated FFN experts per token
 * (RoutingDecision::mean_ffn / std_ffn, router.hpp:73-86), per-expert slot
 * load (stats.hpp:64-67; [n_ffn + n_zero], NULL to skip) and the slot-counted
 * LB group frequencies (lb_group_frequencies, router.hpp:193-216; lb_groups +
 * (n_zero > 0) entries, NULL to skip; ConfigError unless lb_groups divides
 * n_ffn).  indices / ffn_count are device pointers; results land in host
 * memory when the call returns.  Bitwise equal to the reference. */
int scmoe_routing_stats(scmoe_ctx* ctx, const uint32_t* indices, const uint32_t* ffn_count,
                        size_t tokens, size_t top_k, size_t n_ffn, size_t n_zero,
                        size_t k_expected, size_t lb_groups, double* mean_ffn, double* std_ffn,
                        double* per_expert_load, double* lb_freq);
int scmoe_routing_stats_host(scmoe_ctx* ctx, const uint32_t* indices, const uint32_t* ffn_count,
                             size_t tokens, size_t top_k, size_t n_ffn, size_t n_zero,
                             size_t k_expected, size_t lb_groups, double* mean_ffn,
                             double* std_ffn, double* per_expert_load, double* lb_freq);
/* route_topk for RouterState<double> (router.hpp:133-141 with S = double):
 * the projection in double (sequential DMUL/DADD per output), softmax with
 * the glibc exp(double) restatement, same selection.  The router supplies the
 * configuration and bias; its weights in double are passed as w [d, E].
 * Bit-exact with the reference (not on the fp32 hot path). */
int scmoe_route_topk_f64(scmoe_ctx* ctx, scmoe_router* r, const double* x, size_t tokens,
                         const double* w, uint32_t* indices, double* gates, uint32_t* ffn_count,
                         double* probs /* nullable */);
int scmoe_route_topk_f64_host(scmoe_ctx* ctx, scmoe_router* r, const double* x, size_t tokens,
                              const double* w, uint32_t* indices, double* gates,
                              uint32_t* ffn_count, double* probs);
/* Device glibc exp(double) restatement on n inputs (verification hook). */
int scmoe_debug_exp(scmoe_ctx* ctx, const double* in_dev, double* out_dev, size_t n);
/* accumulate_counters (router.hpp:144-150): slot-counted, zero experts included. */
int scmoe_accumulate_counters(scmoe_ctx* ctx, scmoe_router* r, const uint32_t* indices,
                              size_t tokens);
int scmoe_accumulate_counters_host(scmoe_ctx* ctx, scmoe_router* r, const uint32_t* indices,
                                   size_t tokens);
/* bias_update (router.hpp:155-176).  StateError on an empty batch or counters
 * that do not cover K slots per token.  delta [E] (host) may be NULL. */
int scmoe_bias_update(scmoe_ctx* ctx, scmoe_router* r, double* delta);

/* ---- expert bank: ExpertBank<float> (blocks.hpp:203-213) ------------------ */
int scmoe_bank_create(scmoe_ctx* ctx, size_t n_ffn, size_t d_model, size_t inter,
                      int precision, size_t segmentation_m, int gamma_mode, scmoe_bank** out);
int scmoe_bank_destroy(scmoe_ctx* ctx, scmoe_bank* b);
/* w_in [d, inter], w_out [inter, d] row-major fp32 (Parameter::value). */
int scmoe_bank_set_expert_host(scmoe_ctx* ctx, scmoe_bank* b, size_t e, const float* w_in,
                               const float* w_out);
int scmoe_bank_set_expert(scmoe_ctx* ctx, scmoe_bank* b, size_t e, const float* w_in_dev,
                          const float* w_out_dev);
/* Synthetic weights generated on the device, bitwise equal to
 * seeded_init<float>({d,inter}, Uniform, variance, CounterRng(seed).stream(stream0 + 2e))
 * and stream(stream0 + 2e + 1) for w_out (rng.hpp:82-94). */
int scmoe_bank_init_uniform(scmoe_ctx* ctx, scmoe_bank* b, uint64_t seed, uint64_t stream0,
                            double variance);
/* Same for the expert shard [first, first + n) of a larger bank: local expert
 * i gets global expert (first + i)'s streams. */
int scmoe_bank_init_uniform_shard(scmoe_ctx* ctx, scmoe_bank* b, uint64_t seed, uint64_t stream0,
                                  double variance, size_t first_expert);
double scmoe_bank_gamma_ffn(const scmoe_bank* b);
double scmoe_bank_gamma_zero(const scmoe_bank* b);
size_t scmoe_bank_device_bytes(const scmoe_bank* b);

/* moe_forward (blocks.hpp:372-394), optionally renormalised (moe_block
 * renormalize=true, blocks.hpp:240-247) and with a fused residual
 * out = residual + moe(x) (model.hpp:400).  x [T, d] fp32; indices/gates
 * [T*K]; residual [T, d] or NULL; out [T, d] fp32. */
int scmoe_moe_forward(scmoe_ctx* ctx, scmoe_bank* b, const float* x, size_t tokens,
                      const uint32_t* indices, const double* gates, size_t top_k, size_t n_zero,
                      int renormalize, const float* residual, float* out);
int scmoe_moe_forward_host(scmoe_ctx* ctx, scmoe_bank* b, const float* x, size_t tokens,
                           const uint32_t* indices, const double* gates, size_t top_k,
                           size_t n_zero, int renormalize, const float* residual, float* out);

/* Graph::rmsnorm forward (graph.hpp:322-335), fp32, eps as given (1e-6 default). */
/* ExpertBank<double> / moe_forward<double> (blocks.hpp:372-394, S = double):
 * a SCMOE_PREC_F64_EXACT bank, weights set in double; the expert FFN in
 * double (sequential DMUL/DADD, sign-branched logistic on the glibc exp
 * restatement) and the combine in double, bitwise equal to the reference. */
int scmoe_bank_set_expert_f64(scmoe_ctx* ctx, scmoe_bank* b, size_t expert, const double* w_in,
                              const double* w_out);
int scmoe_bank_set_expert_f64_host(scmoe_ctx* ctx, scmoe_bank* b, size_t expert,
                                   const double* w_in, const double* w_out);
int scmoe_moe_forward_f64(scmoe_ctx* ctx, scmoe_bank* b, const double* x, size_t tokens,
                          const uint32_t* indices, const double* gates, size_t top_k,
                          size_t n_zero, int renormalize, const double* residual, double* out);
int scmoe_moe_forward_f64_host(scmoe_ctx* ctx, scmoe_bank* b, const double* x, size_t tokens,
                               const uint32_t* indices, const double* gates, size_t top_k,
                               size_t n_zero, int renormalize, const double* residual,
                               double* out);
int scmoe_rmsnorm(scmoe_ctx* ctx, const float* x, const float* gain, size_t rows, size_t d,
                  float eps, float* out);

/* ScMoE layer, MoE branch of Model::build_layer (model.hpp:394-400):
 *   hmoe = rmsnorm(a1, gain); probs = softmax(hmoe W_r); d = route_from_probs;
 *   out = a3 + moe_block(hmoe, probs, d, bank, renormalize).
 * gain may be NULL (unit gain).  indices/gates/ffn_count receive the routing. */
int scmoe_layer_forward(scmoe_ctx* ctx, scmoe_router* r, scmoe_bank* b, const float* a1,
                        const float* a3, const float* gain, size_t tokens, int renormalize,
                        uint32_t* indices, double* gates, uint32_t* ffn_count, float* out);
/* Pipelined form for a stream of micro-batches (serving / the paper's
 * two-batch overlap): batch i+1's front half (rmsnorm, exact router, top-K,
 * permutation) runs on the tensor-core-idle FP32 pipes while batch i's
 * expert GEMMs stream weights from HBM.  Results are identical to n calls of
 * scmoe_layer_forward; arrays hold one device pointer per batch (a3 may be
 * NULL).  Stream-ordered on the context's stream. */
int scmoe_layer_forward_batches(scmoe_ctx* ctx, scmoe_router* r, scmoe_bank* b, size_t n_batches,
                                const float* const* a1, const float* const* a3, const float* gain,
                                size_t tokens, int renormalize, uint32_t* const* indices,
                                double* const* gates, uint32_t* const* ffn_count,
                                float* const* out);
int scmoe_layer_forward_host(scmoe_ctx* ctx, scmoe_router* r, scmoe_bank* b, const float* a1,
                             const float* a3, const float* gain, size_t tokens, int renormalize,
                             uint32_t* indices, double* gates, uint32_t* ffn_count, float* out);
/* Host tier for a stream of batches (one call per serving window): batch i's
 * inputs are copied in while batch i-1 computes and batch i-2's outputs are
 * copied out (two copy streams + the compute stream, device buffers double
 * buffered).  Results are identical to n calls of scmoe_layer_forward_host;
 * arrays hold one host pointer per batch (pinned memory for real overlap;
 * a3 and the routing outputs may be NULL arrays).  Returns after the last
 * output has landed. */
int scmoe_layer_forward_host_batches(scmoe_ctx* ctx, scmoe_router* r, scmoe_bank* b,
                                     size_t n_batches, const float* const* a1,
                                     const float* const* a3, const float* gain, size_t tokens,
                                     int renormalize, uint32_t* const* indices,
                                     double* const* gates, uint32_t* const* ffn_count,
                                     float* const* out);

/* Dense shortcut-path FFN of the ScMoE layer:
 *   out = a1 + ffn_block(rmsnorm(a1, gain))        (model.hpp:390-391)
 *   ffn_block(x) = silu(x W_in) W_out               (blocks.hpp:397-402)
 * `dense` is a one-expert bf16 bank (scmoe_bank_create(ctx, 1, d, inter,
 * SCMOE_PREC_BF16, ...)); the two GEMMs run on the same tcgen05 grouped-GEMM
 * kernel as the experts (all tokens form one expert's tiles).  Uses its own
 * workspace buffers, so it may run on another context's stream beside the
 * MoE branch (the ScMoE overlap window).  Device pointers, stream-ordered. */
int scmoe_dense_ffn(scmoe_ctx* ctx, scmoe_bank* dense, const float* a1, const float* gain,
                    size_t tokens, float* out);

/* ---- expert parallelism ------------------------------------
 * Experts are block-partitioned over G ranks (rank g owns FFN experts
 * [g*N/G, (g+1)*N/G)); router and bias are replicated, tokens sharded, zero
 * experts stay local.  One layer = route -> plan -> pack -> all-to-all ->
 * scmoe_moe_rows -> all-to-all back -> scmoe_combine_rows; the transport
 * (NCCL all_to_all) is the caller's.  Expert rows are returned per slot and
 * combined at the source in rank order, so the G-rank output is bitwise equal
 * to the single-GPU output. */

/* Front half of the layer (model.hpp:394-397): hmoe = rmsnorm(a1, gain) (fp32
 * and bf16 copies), exact router, top-K.  hmoe_bf16 may be NULL. */
int scmoe_rmsnorm_route(scmoe_ctx* ctx, scmoe_router* r, const float* a1, const float* gain,
                        size_t tokens, float* hmoe, void* hmoe_bf16, uint32_t* indices,
                        double* gates, uint32_t* ffn_count);
/* Dispatch plan: FFN slots grouped by owning rank, (token, slot) ascending
 * within a rank.  send_counts [G] (device), slot_send_pos [T*K] (-1: zero
 * expert), send_token [T*K] / send_expert [T*K] (global expert id) per send
 * row.  All device pointers. */
int scmoe_ep_plan(scmoe_ctx* ctx, const uint32_t* indices, size_t tokens, size_t top_k,
                  size_t n_ffn, size_t n_zero, int world, int* send_counts, int* slot_send_pos,
                  int* send_token, int* send_expert);
/* The permutation of moe_block (blocks.hpp:349-359) as the device computes it
 * (the same kernels as the layer path): expert_count [n_ffn + n_zero] = slots
 * per expert (zero experts included), slot_row [T*K] = position of token t in
 * expert e's ascending token list, -1 for a zero expert.  Device pointers
 * (either output may be NULL); StateError (latched) for an index >= E. */
int scmoe_permutation(scmoe_ctx* ctx, const uint32_t* indices, size_t tokens, size_t top_k,
                      size_t n_ffn, size_t n_zero, int* expert_count, int* slot_row);
/* dst[i] = src[rows[i]] for i < n_rows (bf16 rows of width d). */
int scmoe_gather_rows_bf16(scmoe_ctx* ctx, const void* src, size_t d, const int* rows,
                           size_t n_rows, void* dst);
/* Expert FFN (blocks.hpp:361-365) on rows that each carry one expert:
 * y[r] = silu(x[r] W_in[e_r - expert_offset]) W_out[e_r - expert_offset],
 * bf16 in / bf16 out, rows in the given order.  bf16 banks only. */
int scmoe_moe_rows(scmoe_ctx* ctx, scmoe_bank* b, const void* x_bf16, const int* row_expert,
                   int expert_offset, size_t rows, void* y_bf16);
/* moe_combine (blocks.hpp:226-274) + residual from per-slot expert rows:
 * slot (t,s) with an FFN expert reads y_rows[slot_row[t*K+s]]. */
/* Peer-memory transport (NVLink, symmetric buffers mapped in every rank; the
 * caller owns the mapping, e.g. torch symmetric memory):
 * scmoe_ep_put_rows -- the dispatch: send row j (scmoe_ep_plan order, grouped
 *   by destination: rows [send_start[g], send_start[g+1]) go to rank g) is
 *   stored into peer_rows[g] at row dst_offset[g] + j - send_start[g], its
 *   expert id into peer_expert[g]; all arrays are device arrays, peer_* hold
 *   device addresses.  A cross-rank barrier must follow before the rows are read.
 * scmoe_moe_rows_to -- scmoe_moe_rows whose GEMM2 epilogue writes the output
 *   row of received row r straight to row_dst[r] (an address, typically the
 *   source rank's receive-back buffer over NVLink): the return all-to-all is
 *   fused into the GEMM, overlapping its tiles.  Barrier before the combine. */
int scmoe_ep_put_rows(scmoe_ctx* ctx, const void* src_bf16, size_t d, const int* send_token,
                      const int* send_expert, size_t n_send, const int* send_start,
                      const int64_t* dst_offset, const uint64_t* peer_rows,
                      const uint64_t* peer_expert, int world);
int scmoe_moe_rows_to(scmoe_ctx* ctx, scmoe_bank* b, const void* x_bf16, const int* row_expert,
                      int expert_offset, size_t rows, const uint64_t* row_dst);
int scmoe_combine_rows(scmoe_ctx* ctx, scmoe_bank* b, const float* x, const void* y_rows_bf16,
                       const int* slot_row, const uint32_t* indices, const double* gates,
                       size_t tokens, size_t top_k, size_t n_ffn_total, int renormalize,
                       const float* residual, float* out);

/* ---- expert-parallel layer, device-resident orchestration ------------------
 * One process (or thread) per GPU; the whole layer runs stream-ordered on the
 * device with no host synchronisation per call: route, dispatch plan, an
 * on-device exchange of the [G][G] slot-count matrix (each rank stores its row
 * into every peer's buffer + an epoch flag), dispatch of the bf16 rows by peer
 * stores over NVLink into the owners' receive buffers, grouped GEMMs on the
 * received rows (count read on the device) whose GEMM2 epilogue writes every
 * output row into the source rank's return buffer, an epoch barrier, and the
 * rank-order combine at the source.  Output bitwise equal to the single-GPU
 * layer (scmoe_layer_forward) on the same tokens.  NCCL supplies the
 * communicator, the one-time exchange of the buffers' CUDA IPC handles and
 * the controller's counter all-reduce (router.hpp:158-169). */
typedef struct scmoe_ep scmoe_ep;
/* ncclUniqueId for rank 0 to hand to the other ranks out of band. */
size_t scmoe_ep_unique_id_bytes(void);
int scmoe_ep_unique_id(void* out);
/* Collective over the `world` ranks.  rank g owns FFN experts
 * [g*n_ffn/world, (g+1)*n_ffn/world); max_tokens bounds the tokens per rank and
 * call; max_recv_rows = 0 sizes the receive buffers for the worst case
 * (world * max_tokens * min(top_k, n_ffn/world) rows: no routing can overflow). */
int scmoe_ep_create(scmoe_ctx* ctx, int world, int rank, const void* nccl_unique_id,
                    size_t d_model, size_t n_ffn, size_t n_zero, size_t top_k, size_t max_tokens,
                    size_t max_recv_rows, scmoe_ep** out);
int scmoe_ep_destroy(scmoe_ep* ep); /* collective */
size_t scmoe_ep_capacity_rows(const scmoe_ep* ep);
/* Kernels launched by the layer's contexts (the caller's + internal ones). */
uint64_t scmoe_ep_kernel_launches(const scmoe_ep* ep);
/* Timing reference for the exposed-communication share: on = 0 replaces the
 * row transfers by no-ops (received rows left as they are, spread over the
 * local experts; GEMM2 rows stay local).  Results are garbage while off. */
int scmoe_ep_set_comm(scmoe_ep* ep, int on);
/* SMs the dense branch's GEMMs leave free (default 16). */
int scmoe_ep_set_dense_reserve(scmoe_ep* ep, int reserve_sms);
/* One layer on this rank's T tokens (Model::build_layer MoE branch,
 * model.hpp:394-400): out = residual + moe(rmsnorm(a1)), residual = a3, or,
 * with a one-expert bf16 `dense` bank, dd = a1 + ffn_block(rmsnorm(a1))
 * computed on a second stream beside routing / dispatch / experts / return
 * (the ScMoE overlap window; model.hpp:390-391).  bank = this rank's experts.
 * Device pointers, stream-ordered on ctx's stream. */
int scmoe_ep_layer_forward(scmoe_ep* ep, scmoe_router* r, scmoe_bank* bank, scmoe_bank* dense,
                           const float* a1, const float* a3, const float* gain, size_t tokens,
                           int renormalize, uint32_t* indices, double* gates,
                           uint32_t* ffn_count, float* out);
/* A stream of batches, pipelined: batch i+1's front half (route, plan,
 * exchange, dispatch) on one stream beside batch i's back half (expert GEMMs
 * with the fused return, combine) on another; two buffer sets alternate.
 * corun_router selects the router kernel that co-resides with the GEMM.
 * Identical to n_batches scmoe_ep_layer_forward calls. */
int scmoe_ep_layer_forward_batches(scmoe_ep* ep, scmoe_router* r, scmoe_bank* bank,
                                   size_t n_batches, const float* const* a1,
                                   const float* const* a3, const float* gain, size_t tokens,
                                   int renormalize, int corun_router, uint32_t* const* indices,
                                   double* const* gates, uint32_t* const* ffn_count,
                                   float* const* out);
/* accumulate_counters of this rank's routing (router.hpp:144-150) and, with
 * update, bias_update over the GLOBAL batch (router.hpp:155-176): the [E]
 * counters and tokens_seen are summed over the ranks on the device
 * (ncclAllReduce, exact integers), so every rank applies the same update.
 * delta [E] (host, nullable) receives the deltas (synchronises).  StateError
 * from the device check latches (next scmoe_synchronize). */
int scmoe_ep_controller_step(scmoe_ep* ep, scmoe_router* r, const uint32_t* indices,
                             size_t tokens, int update, double* delta);
/* [world][world] slot counts of the most recent call (synchronises). */
int scmoe_ep_count_matrix_host(scmoe_ep* ep, int* matrix);

/* ---- Multi-head latent attention, forward value, S = float (f2 row) --------
 * MlaParams<float> (blocks.hpp:38-58); mla_block forward (blocks.hpp:73-102)
 * over packed sequences; MlaCache + mla_infer_step (blocks.hpp:106-181).
 * Bitwise equal to the reference (sequential-k fp32 projections, exact rope,
 * causal attention with the glibc-expf restatement and in-order sums).
 * Weights are row-major Parameter values: w_dq [d,dq], w_uq [dq,H*dhc],
 * w_qr [dq,H*dhr], w_dkv [d,dkv], w_uk [dkv,H*dhc], w_uv [dkv,H*dhc],
 * w_kr [d,dhr], w_o [H*dhc,d].  Errors: ParameterError for zero d/dq/dkv
 * (mla_scale_factors, blocks.hpp:21-22); DimensionError for H = 0 or odd dhr
 * (tensor.hpp:202-204) and rows not packing whole sequences (graph.hpp:404);
 * StateError when the cache length differs from the position (blocks.hpp:135-137). */
typedef struct scmoe_mla scmoe_mla;
typedef struct scmoe_mla_cache scmoe_mla_cache;
enum {
    SCMOE_MLA_W_DQ = 0, SCMOE_MLA_W_UQ = 1, SCMOE_MLA_W_QR = 2, SCMOE_MLA_W_DKV = 3,
    SCMOE_MLA_W_UK = 4, SCMOE_MLA_W_UV = 5, SCMOE_MLA_W_KR = 6, SCMOE_MLA_W_O = 7
};
int scmoe_mla_create(scmoe_ctx* ctx, size_t d_model, size_t d_q, size_t d_kv, size_t n_heads,
                     size_t d_head_c, size_t d_head_r, double rope_base,
                     int variance_alignment, scmoe_mla** out);
int scmoe_mla_destroy(scmoe_ctx* ctx, scmoe_mla* m);
/* which = SCMOE_MLA_W_*; w is that matrix, row-major, host / device. */
int scmoe_mla_set_weight_host(scmoe_ctx* ctx, scmoe_mla* m, int which, const float* w);
int scmoe_mla_set_weight(scmoe_ctx* ctx, scmoe_mla* m, int which, const float* w_dev);
/* Forward precision of scmoe_mla_forward (and the full layer's MLAs):
 * SCMOE_PREC_F32_EXACT (default; bitwise equal to the reference) or
 * SCMOE_PREC_BF16: every contraction (projections, scores, P.V) on the
 * tcgen05 grouped GEMM with bf16 operands and fp32 accumulation, causal
 * softmax in fp32 (rel-L2 <= 2e-2 vs the reference).  ConfigError unless d,
 * d_q, d_kv and H*d_head_c are multiples of 64 and d_head_c <= 256.  The
 * cached decode step (mla_infer_step) stays exact. */
int scmoe_mla_set_precision(scmoe_ctx* ctx, scmoe_mla* m, int precision);
/* out [rows, d] = mla_block(h [rows, d], seq_len) value (stream-ordered). */
int scmoe_mla_forward(scmoe_ctx* ctx, scmoe_mla* m, const float* h_dev, size_t rows,
                      size_t seq_len, float* out_dev);
int scmoe_mla_forward_host(scmoe_ctx* ctx, scmoe_mla* m, const float* h, size_t rows,
                           size_t seq_len, float* out);
int scmoe_mla_cache_create(scmoe_ctx* ctx, scmoe_mla* m, size_t capacity_hint,
                           scmoe_mla_cache** out);
int scmoe_mla_cache_destroy(scmoe_ctx* ctx, scmoe_mla_cache* cache);
int scmoe_mla_cache_length(scmoe_ctx* ctx, scmoe_mla_cache* cache, size_t* length);
/* c_kv [len, d_kv] and the rotated k_r [len, d_head_r] (either may be NULL). */
int scmoe_mla_cache_read_host(scmoe_ctx* ctx, scmoe_mla* m, scmoe_mla_cache* cache, float* c_kv,
                              float* k_r);
/* out [1, d] = mla_infer_step(h_t [1, d], position); appends to the cache. */
int scmoe_mla_infer_step(scmoe_ctx* ctx, scmoe_mla* m, scmoe_mla_cache* cache,
                         const float* h_t_dev, size_t position, float* out_dev);
int scmoe_mla_infer_step_host(scmoe_ctx* ctx, scmoe_mla* m, scmoe_mla_cache* cache,
                              const float* h_t, size_t position, float* out);

/* ---- The full ScMoE layer (Model::build_layer, model.hpp:355-409) ----------
 *   a1 = x + MLA1(rmsnorm(x, norm1));  dd = a1 + FFN(rmsnorm(a1, norm_ffn));
 *   a3 = dd + MLA2(rmsnorm(dd, norm2)); out = a3 + moe(rmsnorm(a1, norm_moe)).
 * MLA exact fp32, dense FFN (one-expert bf16 bank) and MoE (bank precision)
 * as in the calls above.  overlap = 1 runs the MoE branch on a second stream
 * beside the dense FFN and MLA2 (results identical).  a1_out / a3_out are
 * optional [T, d] outputs; the routing outputs are as scmoe_layer_forward's. */
int scmoe_layer_full_forward(scmoe_ctx* ctx, scmoe_mla* mla1, scmoe_mla* mla2, scmoe_bank* dense,
                             scmoe_router* r, scmoe_bank* bank, const float* norm1,
                             const float* norm_ffn, const float* norm2, const float* norm_moe,
                             const float* x, size_t T, size_t seq_len, int renormalize,
                             int overlap, uint32_t* indices, double* gates, uint32_t* ffn_count,
                             float* a1_out, float* a3_out, float* out);

/* ---- CounterRng (rng.hpp:15-64), host side, for synthetic inputs --------- */
uint64_t scmoe_rng_stream_seed(uint64_t seed, uint64_t id);
/* out[i] = (float) CounterRng(seed).normal_at(first + i)  (router.hpp:357-360) */
void scmoe_rng_fill_normal_host(uint64_t seed, uint64_t first, size_t n, float* out, int threads);
/* out[i] = seeded_init Uniform element first+i (rng.hpp:89-94), on the device. */
int scmoe_rng_fill_uniform(scmoe_ctx* ctx, uint64_t seed, uint64_t first, size_t n,
                           double variance, float* out_dev);

/* ---- diagnostics ---------------------------------------------------------- */
/* Per-stage timing with CUDA events on the context's stream (off by default).
 * flush() waits for the stream and aggregates by stage name; entry(i) reads
 * one aggregate (name valid until the next flush). */
int scmoe_profile_enable(scmoe_ctx* ctx, int on);
int scmoe_profile_flush(scmoe_ctx* ctx, int* n_entries);
int scmoe_profile_entry(scmoe_ctx* ctx, int i, const char** name, double* total_ms,
                        uint64_t* launches);
/* Record i of the last flush in issue order: its stage name and device
 * start / end time in ms relative to the flush's first record (a timeline
 * across streams). */
int scmoe_profile_span(scmoe_ctx* ctx, int i, const char** name, double* start_ms,
                       double* end_ms);
/* out[i] = device instantiation of the glibc-expf restatement used by the
 * softmax and SiLU kernels (bit-exactness check against host libm). */
int scmoe_debug_expf(scmoe_ctx* ctx, const float* in_dev, float* out_dev, size_t n);
/* Same over the consecutive bit patterns first_bits, first_bits+1, ... */
int scmoe_debug_expf_range(scmoe_ctx* ctx, uint32_t first_bits, float* out_dev, size_t n);

#ifdef __cplusplus
}
#endif
#endif /* SCMOE_H */

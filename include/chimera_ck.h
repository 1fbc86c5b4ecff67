/* chimera_ck.h -- the C-ABI boundary of the Chimera-B200 build (libchimera.so).
 *
 * The reference (`pipesim`, /root/reference/proj) is a C++ library with no FFI; its
 * public surface is the headers in proj/include/pipesim/.  This build keeps those
 * C++ headers verbatim in include/pipesim/ (drop-in) and puts a thin extern "C"
 * layer under them so that any host language (and our Python mirror) can bind
 * plain pointers and sizes.  Each entry point names the reference interface it
 * replaces.  See INTEGRATION.md for the bindings a reference user adds.
 *
 * Conventions:
 *   - status: 0 ok, 2 invalid input (InvalidConfigError), 3 internal error
 *     (CUDA/NCCL failure, missing activation, deadlock timeout);
 *   - ck_last_error() returns the message of the calling thread's last failure;
 *   - strings returned through `char**` are malloc'd: release with ck_free();
 *   - the caller owns host buffers; a context (ck_toy_*, ck_gpt_*) owns all device
 *     memory; one host thread drives a context (calls are not thread-safe).
 *   - no torch types cross this boundary.
 */
#ifndef CHIMERA_CK_H
#define CHIMERA_CK_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CK_API __attribute__((visibility("default")))
#else
#define CK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ common */
CK_API const char* ck_last_error(void);
CK_API void ck_free(void* p);

/* ------------------------------------------------- host schedule layer (C++) */
/* schedgen::generate (proj/include/pipesim/schedgen.hpp:92) + to_json(.., indent)
 * (proj/include/pipesim/core.hpp:182).  JSON is the reference wire format. */
CK_API int pipesim_generate(const char* config_json, const char* profile_json, int indent,
                     char** out_json);
/* validate_config (core.hpp:173); violations joined by '\n' (empty = valid). */
CK_API int pipesim_validate_config(const char* config_json, const char* profile_json, char** out);
/* analysis::validate_dependencies (analysis.hpp:41). */
CK_API int pipesim_validate_dependencies(const char* schedule_json, char** out);
/* analysis::bubble_ratio_per_worker (analysis.hpp:53) on the zero-comm timing. */
CK_API int pipesim_bubble_ratio_per_worker(const char* schedule_json, const char* profile_json,
                                    int64_t* num, int64_t* den, int cap);
/* analysis::memory_profile (analysis.hpp:59). */
CK_API int pipesim_memory_profile(const char* schedule_json, const char* profile_json, int* act_counts,
                           int* weight_counts, double* act_bytes, double* weight_bytes,
                           int* peak_worker, double* peak_bytes, int cap);
/* dessim::simulate (dessim.hpp:58) + memory_trace peaks; policy 0 end-of-iteration,
 * 1 eager-sync, 2 eager-sync-opt. */
CK_API int pipesim_simulate(const char* schedule_json, const char* profile_json, int policy,
                     int zero_comm, double eager_overhead, char** out_json);
/* The `pipesim simulate -o <prefix>` outputs (proj/tools/main.cpp:134-170,367-370):
 * the timeline JSON document (indent 2 + newline) and the Gantt chart of the same
 * simulation (gantt::render_svg / render_ascii, proj/src/gantt.cpp:35-125). */
CK_API int pipesim_simulate_timeline(const char* schedule_json, const char* profile_json, int policy,
                                     double eager_overhead, char** out_json);
CK_API int pipesim_gantt(const char* schedule_json, const char* profile_json, int policy,
                         double eager_overhead, int svg, char** out);
/* Gantt chart of a timeline document in that schema -- e.g. a measured GPU iteration
 * (gpt.measured_timeline); time unit = the profile's F_t for the ASCII columns. */
CK_API int pipesim_gantt_timeline(const char* timeline_json, const char* profile_json, int svg, char** out);
/* perfmodel::replicas_per_stage / critical_path / predict_T (perfmodel.hpp:61-75). */
CK_API int pipesim_replicas_per_stage(const char* config_json);
CK_API int pipesim_critical_path(const char* schedule_json, const char* profile_json, int* C_f,
                          int* C_b);
CK_API int pipesim_predict_T(const char* config_json, const char* profile_json, double* T);
/* analysis::validate_dependencies / bubble_ratio_per_worker / steady_state_idle /
 * memory_profile (proj/include/pipesim/analysis.hpp:41-60) and perfmodel::free_regions /
 * critical_path (proj/include/pipesim/perfmodel.hpp:63-70) in one JSON document
 * {"violations", "bubble", "steady_state_idle", "memory", "free_regions", "critical_path"}. */
CK_API int pipesim_analysis_report(const char* schedule_json, const char* profile_json, char** out_json);
/* perfmodel::plan (proj/include/pipesim/perfmodel.hpp:78-83): JSON list of
 * {"W","D","B","N","scaling","recompute","T_predicted"}, fastest first. */
CK_API int pipesim_plan(int P, long long B_hat, const char* profile_json, const char* scheme, char** out_json);
/* Issue order used by the executors: (worker, index) sorted by unit-tick start,
 * the reference oracle's replay order (proj/src/oracle.cpp:312-327). */
CK_API int pipesim_replay_order(const char* schedule_json, int* worker, int* index, int cap);

/* ------------------------------------------ ToyModel executor (sm_100a, fp64) */
/* oracle::run_iteration_traced (proj/include/pipesim/oracle.hpp:72): one iteration of
 * the schedule on the current GPU; params are flat per stage [W_s (out x in), b_s];
 * peak_stash[w] = peak live activation stashes of worker w (replica 0). */
CK_API int ck_toy_run_iteration(const char* schedule_json, const int* dims, int n_dims,
                                const double* params_in, const double* inputs,
                                const double* targets, int batch, double lr, double* params_out,
                                int* peak_stash, int cap);
/* oracle::make_model / make_batch (oracle.hpp:44-45), host-side, bit-identical. */
CK_API int ck_toy_make_model(const int* dims, int n_dims, uint64_t seed, double* params);
CK_API int ck_toy_make_batch(const int* dims, int n_dims, int size, uint64_t seed,
                             double* inputs, double* targets);
/* oracle::check_gradients (proj/include/pipesim/oracle.hpp:77, oracle.cpp:358-410):
 * central finite differences (fp64, one CTA per parameter and sign) vs the analytic
 * gradient, both on the GPU; *max_rel_err = max |fd - g| / max(1, |fd|, |g|). */
CK_API int ck_toy_check_gradients(const int* dims, int n_dims, const double* params, const double* inputs,
                                  const double* targets, int batch, double step, double* max_rel_err);
/* oracle::sequential_sgd (oracle.hpp:56): plain mini-batch SGD on the GPU. */
CK_API int ck_toy_sequential_sgd(const int* dims, int n_dims, const double* params_in,
                                 const double* inputs, const double* targets, int batch,
                                 double lr, double* params_out);

/* ------------------------------------------------------ kernel launchers (device ptrs) */
/* tcgen05/TMA GEMM with fused epilogue (cuda/gemm.cu).  epi: 0 bf16 store (+bias),
 * 1 bias+GELU (out=U, out2=gelu(U)), 2 bias+residual(aux), 3 x gelu'(aux), 4 fp32 +=,
 * 5 fp32 store.  a_mn/b_mn select MN-major operands (see cuda/gemm.cuh). */
/* Split-K variant for the bf16 epilogues: ws = fp32 workspace (zero-filled, >= M*N,
 * left zeroed); K-slices reduce-add into it, one finalize pass applies the epilogue.
 * ksplit > 1 forces the slice count, 0 lets the wave model decide (it may not split);
 * tile >= 0 forces the tile (0 CTA pair 256x256, 256 / 128 / 64: single CTA 128 x tile). */
CK_API int ck_gemm_bf16_split(int epi, int a_mn, int b_mn, int M, int N, int K, const void* A, long long lda,
                              const void* B, long long ldb, void* out, long long ldo, const void* bias,
                              const void* aux, long long ld_aux, void* out2, long long ld_out2, float* colsum,
                              float* ws, long long ws_elems, int ksplit, int tile, void* stream);
CK_API int ck_gemm_bf16(int epi, int a_mn, int b_mn, int M, int N, int K, const void* A,
                        long long lda, const void* B, long long ldb, void* out, long long ldo,
                        const void* bias, const void* aux, long long ld_aux, void* out2,
                        long long ld_out2, void* stream);
/* ck_gemm_bf16 plus, for epi 3, colsum[N] += column sums of the bf16 output (the fused bias
   gradient of the layer whose pre-activation gradient this GEMM produces). */
CK_API int ck_gemm_bf16_ex(int epi, int a_mn, int b_mn, int M, int N, int K, const void* A,
                           long long lda, const void* B, long long ldb, void* out, long long ldo,
                           const void* bias, const void* aux, long long ld_aux, void* out2,
                           long long ld_out2, float* colsum, void* stream);

/* LayerNorm (eps 1e-5), rows of h (h % 256 == 0); stats fp32. */
CK_API int ck_layernorm_fwd(const void* x, const void* g, const void* b, void* y, float* mean,
                            float* rstd, int M, int h, void* stream);
CK_API int ck_layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd,
                            const void* g, const void* dres, void* dx, float* dgamma,
                            float* dbeta, int M, int h, void* stream);
/* ck_layernorm_bwd that also accumulates dsum[h] += sum over rows of the (bf16) dx: the
   bias gradient of the linear layer that produced the residual stream (fused bias grad,
   replaces a ck_bias_grad pass over dx). */
CK_API int ck_layernorm_bwd_dsum(const void* dy, const void* x, const float* mean, const float* rstd,
                                 const void* g, const void* dres, void* dx, float* dgamma,
                                 float* dbeta, float* dsum, int M, int h, void* stream);
/* token + position embedding and its scatter-add backward (fp32 grads). */
CK_API int ck_embed_fwd(const int32_t* tok, const void* wte, const void* wpe, void* x, int M,
                        int seq, int h, void* stream);
CK_API int ck_embed_bwd(const int32_t* tok, const void* dx, float* dwte, float* dwpe, int M,
                        int seq, int h, void* stream);
/* in-place softmax cross-entropy forward+backward over the first V of Vp columns. */
CK_API int ck_xent_fwd_bwd(void* logits, long long ld, const int32_t* labels, int M, int V, int Vp,
                           float grad_scale, float loss_scale, float* loss_sum, void* stream);
CK_API int ck_bias_grad(const void* dy, float* db, int M, int N, void* stream);
CK_API int ck_sgd_update(float* w32, void* w16, float* const* grads, int copies, long long n,
                         float lr, void* stream);
/* flash attention, head dim 64, over packed qkv [B*seq, 3*H*64]. */
CK_API int ck_attn_fwd(const void* qkv, void* out, float* lse, int B, int seq, int H, int causal,
                       void* stream);
/* tcgen05/TMEM flash attention forward (S and O accumulate in tensor memory). */
CK_API int ck_attn_fwd_tc(const void* qkv, void* out, float* lse, int B, int seq, int H,
                          int causal, void* stream);
CK_API int ck_attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse,
                       void* dqkv, float* scratch, int B, int seq, int H, int causal, void* stream);
CK_API long long ck_attn_bwd_scratch_floats(int B, int seq, int H);
/* tcgen05/TMEM flash attention backward (same contract / scratch as ck_attn_bwd). */
CK_API int ck_attn_bwd_tc(const void* qkv, const void* out, const void* dout, const float* lse,
                          void* dqkv, float* scratch, int B, int seq, int H, int causal, void* stream);
/* ck_attn_bwd_tc that also accumulates dbias[3 H 64] += column sums of the bf16 dqkv it
   writes: the QKV bias gradient, summed in the dQ conversion and the dK / dV epilogue. */
CK_API int ck_attn_bwd_tc_dbias(const void* qkv, const void* out, const void* dout, const float* lse,
                                void* dqkv, float* scratch, float* dbias, int B, int seq, int H, int causal,
                                void* stream);

/* ------------------------------------------------------- GPT-2 stage executor */
/* Transformer shape (head dim 64; vocab padded to a multiple of 8, e.g. 50304). */
typedef struct ck_gpt_model {
  int n_layer, hidden, heads, ffn, seq, vocab, vocab_padded, causal;
  const int* stage_layers;  /* optional layers per stage (D entries summing to n_layer) */
  int n_stage_layers;       /* 0 = even split */
} ck_gpt_model;
typedef struct ck_gpt ck_gpt;
/* A trainer for logical ranks [first_rank, first_rank + n_ranks) of the schedule
 * (rank = replica * D + worker), on the current device.  Replaces the reference
 * oracle::run_iteration's Engine (proj/src/oracle.cpp:162-356) for a real model. */
CK_API int ck_gpt_create(const ck_gpt_model* model, const char* schedule_json, float lr,
                         int first_rank, int n_ranks, ck_gpt** out);
CK_API int ck_gpt_destroy(ck_gpt* h);
/* JSON: per held stage {stage, numel, tensors:[{name, offset, rows, cols, init}]}. */
CK_API int ck_gpt_layout(ck_gpt* h, char** out_json);
/* JSON: peak_stash_per_rank, device_bytes, launches_per_step, graph, steps. */
CK_API int ck_gpt_stats(ck_gpt* h, char** out_json);
CK_API int ck_gpt_stage_numel(ck_gpt* h, int stage, long long* n);
CK_API int ck_gpt_set_params(ck_gpt* h, int stage, const float* host);
CK_API int ck_gpt_get_params(ck_gpt* h, int stage, float* host);
/* tokens / labels: int32 [W*N*B*seq], sample (r*N + m)*B + i (oracle.cpp:200). */
CK_API int ck_gpt_set_batch(ck_gpt* h, const int32_t* tokens, const int32_t* labels,
                            int from_host);
/* one iteration (all micro-batches, gradient sync, SGD); *loss = mean token loss. */
CK_API int ck_gpt_step(ck_gpt* h, float* loss);
/* one eager iteration with CUDA-event timestamps around every task on its rank's
 * stream: JSON {iteration_ms, tasks:[{rank, kind, pipeline, micro, stage, start_ms,
 * end_ms}]} relative to the iteration start on this process. */
CK_API int ck_gpt_profile_step(ck_gpt* h, char** out_json);
/* Engine-style driving of one iteration (replaces oracle::Engine's loop,
 * proj/src/oracle.cpp:304-356): begin, then one call per task of the schedule in a
 * dependency-respecting order -- task = int32[6] {kind, pipeline_id, micro_batch, stage,
 * worker, replica_group} (pipesim::Task field order, core.hpp:57-64), run for every
 * local replica -- then end (gradient sync + SGD, *loss = mean token loss).  A task
 * whose input activation / gradient was not produced yet returns 3 (the reference's
 * MissingActivationError) with nothing enqueued; foreign or repeated tasks return 2. */
CK_API int ck_gpt_begin_iteration(ck_gpt* h);
CK_API int ck_gpt_run_task(ck_gpt* h, const int32_t* task);
CK_API int ck_gpt_end_iteration(ck_gpt* h, float* loss);
/* enqueue one iteration on the trainer stream without waiting (graph replay). */
CK_API int ck_gpt_launch(ck_gpt* h);
CK_API int ck_gpt_set_graph(ck_gpt* h, int on);
/* dessim::SyncPolicy of the stage gradient allreduce (proj/src/dessim.cpp:101-135):
 * 0 end-of-iteration, 1 eager-sync (default: each stage's allreduce + SGD launched on a
 * comm stream as soon as its last local backward is issued), 2 eager-sync-opt (eager
 * iff the reference's interior-slack rule marks every holder eager). */
CK_API int ck_gpt_set_sync_policy(ck_gpt* h, int policy);
/* The CostProfile (pipesim JSON) the gradient-sync plan is computed on: dessim::simulate
 * (proj/src/dessim.cpp:60-135) decides eager-sync-opt per stage and orders the stage
 * collectives.  Every process of a run must pass identical values (the collective order
 * must agree).  Drops the captured iteration graph. */
CK_API int ck_gpt_set_cost_profile(ck_gpt* h, const char* profile_json);
/* {"policy", "profile", "order": [{"stage", "eager", "planned_start"}...]} */
CK_API int ck_gpt_sync_plan(ck_gpt* h, char** out_json);
/* Stage optimizer (beyond the reference's SGD): kind 0 SGD (default,
 * proj/src/oracle.cpp:283-299), 1 AdamW (decoupled weight decay; lr = the trainer's).
 * zero != 0: ZeRO-1 -- each process holding a stage keeps 1/R of the AdamW moments and
 * updates that share (reduce-scatter + fp32 all-gather over the stage communicator).
 * Multi-process: call after connect. */
CK_API int ck_gpt_set_optimizer(ck_gpt* h, int kind, float beta1, float beta2, float eps, float weight_decay,
                                int zero);
CK_API void* ck_gpt_stream(ck_gpt* h);
/* Multi-process (one process per GPU): export this process's 128 bytes of CUDA-IPC
 * handles, all-gather them (host side, e.g. torch.distributed), then connect with all
 * processes' handles in process order and the NCCL ids (ck_nccl_unique_id): either one
 * (a world communicator split per stage) or D, one per stage (each stage communicator
 * initialised on its own: no world communicator, so several processes may share a GPU
 * as long as every stage's holders are on distinct GPUs). */
CK_API int ck_gpt_ipc_handles(ck_gpt* h, char* out, int cap);
CK_API int ck_gpt_connect(ck_gpt* h, const char* all_handles, int n_bytes, const char* nccl_id,
                          int id_bytes);
CK_API int ck_nccl_unique_id(char* out, int cap);
/* Host-only: the cross-process message plan (producer/consumer ranks, every process's
 * inbox/outbox layout, stage allreduce groups) for `ranks_per_proc` ranks per process. */
CK_API int ck_link_plan(const char* schedule_json, int ranks_per_proc, long long msg_bytes,
                        char** out_json);

#ifdef __cplusplus
}
#endif
#endif /* CHIMERA_CK_H */

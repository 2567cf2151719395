/*
 * go_b200.h — C-ABI of libgo_b200.so, the B200-native (sm_100a) policy-evaluation
 * path of GO (arXiv 2010.12438): embed -> policy -> sample -> simulate.
 *
 * The reference (/root/reference/pkg/src/graphopt) is pure Python + numpy and has
 * no FFI; its boundary is its Python function signatures.  Each
 * entry point below states the reference function it replaces.  The Python mirror in
 * paper_2010_12438_b200/ binds these with ctypes (INTEGRATION.md shows the stub).
 *
 * Conventions
 *   - Every function returns int status: GO_OK (0) or an error code; go_last_error()
 *     returns a thread-local message.  The Python layer maps codes to the reference's
 *     exception types (ValueError, FloatingPointError, AssertionError, ...).
 *   - "dev" pointers are CUDA device pointers owned by the caller (torch allocations
 *     in the Python layer); "host" pointers are host memory.  The library never frees
 *     caller memory.  `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Handles (go_ctx_t, go_graph_t) own library workspaces / uploaded static graph
 *     data.  A handle is not thread-safe: use one context per stream.
 *   - No CPU fallback: a missing/failed CUDA device is an error (GO_ERR_CUDA).
 */
#ifndef GO_B200_H
#define GO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GO_OK = 0,
  GO_ERR_VALUE = 1,      /* bad argument / shape / range  -> ValueError          */
  GO_ERR_CUDA = 2,       /* CUDA runtime failure                                  */
  GO_ERR_CYCLE = 3,      /* graph has a cycle               -> GraphError          */
  GO_ERR_NONFINITE = 4,  /* non-finite embeddings           -> FloatingPointError  */
  GO_ERR_DEADLOCK = 5,   /* DES deadlock                     -> AssertionError      */
  GO_ERR_UNSUPPORTED = 6 /* configuration outside the kernels' limits               */
};

typedef struct go_ctx* go_ctx_t;
typedef struct go_graph* go_graph_t;

const char* go_last_error(void);
int go_version(void);

/* ---------------------------------------------------------------- context ---- */
int go_ctx_create(int device, go_ctx_t* out);
int go_ctx_destroy(go_ctx_t ctx);
/* bytes of device workspace currently held by the context */
int go_ctx_workspace_bytes(go_ctx_t ctx, int64_t* out);
/* Number of CUDA kernels this library has launched (process-wide counter). */
long long go_launch_count(void);
/* Per-kernel-class CUDA-event timing on the launching stream (enable resets the
 * statistics).  Classes: 0 heads attention, 1 trunk attention, 2 segment max,
 * 3 gemm, 4 DES, 5 sampler, 6 neighbour sampling, 7 other.  total_work is the
 * algorithmic FLOPs (attention, gemm) or bytes (segment max) or placement-nodes
 * (DES) of the timed launches. */
int go_ctx_set_timing(go_ctx_t ctx, int enable);
int go_ctx_kernel_stats(go_ctx_t ctx, int32_t cls, int64_t* count, double* total_ms,
                        double* total_work);

/* ------------------------------------------------------- host graph ingest ---- */
/* Topological order, ascending-id tie-break (replaces graph.py:173-201
 * _partial_topo/_topo_order).  Returns GO_ERR_CYCLE on a cycle. */
int go_topo_order(int32_t n, int64_t e, const int32_t* src, const int32_t* dst,
                  int32_t* order_out /*host n*/);

/* Greedy balanced contiguous placement (replaces baselines.py:75-118
 * greedy_placement; same earliest-split tie-break, O(D N log N)).
 * flops_topo: flops in topo order.  cuts_out: host d+1. */
int go_greedy_cuts(int32_t n, const double* flops_topo, int32_t d, int64_t* cuts_out);

/* Greedy fusion pass (replaces simulator.py:199-277 apply_fusion; same visit order,
 * candidate choice, max_group and cycle rule).  op: op index per node (graph.py:16-30);
 * label_out host [n]: group root per node (canonicalised by go_graph_set_fusion). */
int go_apply_fusion(int32_t n, int64_t e, const int32_t* src, const int32_t* dst,
                    const int32_t* op, const int64_t* priorities, int32_t max_group,
                    int64_t* label_out);

/* Upload a graph (host arrays, node-id indexed; edges in graph.edges order) and
 * build its static device tables: topo order, undirected sorted neighbour CSR in
 * topo-row space (graph.py:131-133), features (graph.py:297-301), and the
 * singleton FusedGraph DES tables (simulator.py:86-172, costmodel.py:149-187).
 * coloc: colocation-group id per node or -1.  Replaces ComputationGraph +
 * singleton_fused construction. */
int go_graph_create(go_ctx_t ctx, int32_t n, int64_t e, const int32_t* op,
                    const double* flops, const double* out_bytes, const int32_t* coloc,
                    const int32_t* src, const int32_t* dst, const double* ebytes,
                    go_graph_t* out);
int go_graph_destroy(go_graph_t g);
/* host copies of the derived tables: order (n), neighbour CSR offsets (n+1) */
int go_graph_topo(go_graph_t g, int32_t* order_out);
int go_graph_num_neighbors(go_graph_t g, int64_t* total_out);

/* Rebuild the graph's DES tables for an arbitrary fused grouping (group label per
 * node; simulator.py:86-172 FusedGraph).  is_acyclic_out = 0 reproduces
 * topo_index None ("cycle_after_fusion"). */
int go_graph_set_fusion(go_graph_t g, const int64_t* group_label /*host n*/,
                        int32_t* num_groups_out, int32_t* is_acyclic_out);

/* ----------------------------------------------------------- policy config ---- */
typedef struct {
  int32_t gs_layers, gs_dim, gs_knn;                    /* EmbedConfig  (embedding.py:17-21) */
  int32_t trf_layers, d_model, n_head, d_head, d_inner; /* PolicyConfig (policy.py:21-33)    */
  int32_t segment_len;
  int32_t num_tasks;      /* 1..3, canonical order (policy.py:18)           */
  int32_t task_sizes[3];  /* actions per task in that order                 */
} go_config_t;

/* Parameter blob: float32 device buffer; param_offsets (host, int64) gives the
 * element offset of every tensor in the canonical slot order documented in
 * paper_2010_12438_b200/params.py (go_param_slots); row-major [in, out] like the
 * reference ParamStore (tensor.py:391). */
int go_param_count(const go_config_t* cfg, int32_t* num_slots_out);

/* One batch of forwards ("super-positioned" ragged batch: forwards may use different
 * graphs).  Rows of forward f are [row_off[f], row_off[f+1]) in topo order.
 *   graphs       host [F] graph handle per forward, or NULL for a graph-less batch
 *                (trunk/heads stages only) described by row_counts
 *   row_counts   host [F] rows per forward when graphs == NULL
 *   embed_seeds  host [F] neighbour-sampling seed per forward (policy.py:289)
 *   prev_actions dev  [T][total_rows] int32, node-indexed within each forward's row
 *                span (prev_actions[t][row_off[f] + node]); NULL = iteration 1.
 * Outputs (dev, any may be NULL except logits):
 *   node_embed [rows, gs_dim], graph_embed [F, gs_dim]   (embedding.py:73-98)
 *   hid        [rows, d_model]                            (policy.py:135-177)
 *   logits     [T][rows, a_t] packed per task             (policy.py:187-217)
 *   value      [F]
 *   reps (in the batch struct) [T][rows, d_model] action representations or NULL
 * stage_mask: bit0 embed, bit1 trunk, bit2 heads (a stage not run takes its input
 * from the corresponding output pointer: node_embed/graph_embed for the trunk,
 * hid for the heads).  mod_override: dev [F, d_model] or NULL (policy.py:137).
 * ablate_mask: bit t = zero action input of task t (policy.py:189). */
typedef struct {
  int32_t num_forwards;
  const go_graph_t* graphs;
  const int64_t* row_counts;
  const int64_t* embed_seeds;
  const int32_t* prev_actions;
  int32_t stage_mask;
  int32_t ablate_mask;
  const float* mod_override;
  /* optional dev [total_rows, feature_dim] float32 feature matrix; NULL = build the
   * rows in-kernel from the graph statics + prev_actions (graph.py:268-313) */
  const float* features;
  int32_t feature_dim;
  float* reps;
  /* optional trunk cache hook (policy.py:137,170-172 cache_perturb, diagnostics): when
   * set, before layer l's attention the library copies that layer's inputs xm
   * (host float32 [rows, d_model]) and calls cache_hook(user, l, xm, prefix, rows,
   * d_model); prefix (host, pre-filled with xm) receives, for every segment s >= 1,
   * the values its queries use as the previous segment's cached keys/values in place
   * of xm's rows of segment s-1.  Single forward, segment_len <= 64; the layer then
   * runs on the fp32 SIMT attention kernel. */
  void (*cache_hook)(void* user, int32_t layer, const float* xm, float* prefix,
                     int64_t rows, int32_t d_model);
  void* cache_hook_user;
} go_batch_t;

int go_forward(go_ctx_t ctx, const go_config_t* cfg, const float* params,
               const int64_t* param_offsets, const go_batch_t* batch,
               float* node_embed, float* graph_embed, float* hid, float* logits,
               float* value, void* stream);
/* Same, plus a device status word (int32, OR-ed): bit0 = non-finite node embeddings
 * (embedding.py:96-97 raises FloatingPointError on it).  The Python layer checks it
 * when it next synchronises, so a batch is not stalled per forward. */
int go_forward_status(go_ctx_t ctx, const go_config_t* cfg, const float* params,
                      const int64_t* param_offsets, const go_batch_t* batch,
                      float* node_embed, float* graph_embed, float* hid, float* logits,
                      float* value, int32_t* status_dev, void* stream);

/* Neighbour sample of one graph (embedding.py:47-70 _neighbor_arrays): the gather
 * list in topo-row space, segment r = rows [seg_off[r], seg_off[r+1]), neighbours
 * sorted by node id.  seg_off_out host int64 [n+1]; gather_dev dev int32 [seg_off[n]]
 * (query the size with gather_dev = NULL). */
int go_neighbor_arrays(go_ctx_t ctx, go_graph_t g, int64_t seed, int32_t k,
                       int64_t* seg_off_out, int32_t* gather_dev, void* stream);

/* Per-row categorical sampling in float64 (policy.py:220-237), bit-compatible with
 * numpy given the same logits and uniforms.  pcg_states host [F][4] = (state_hi,
 * state_lo, inc_hi, inc_lo) of each forward's numpy PCG64 generator *before* this
 * call; row r of task t consumes draw t*n_f + r (policy.py:235, 299-306: rng.random
 * per task in canonical order).  The caller advances its generators by T*n_f draws.
 * logits dev [T][rows, a_t] float32 or float64 (logits_flags bit 0); with bit 1 set
 * every forward reads the SAME logits block, [T][rows of forward 0, a_t] (mode S: many
 * placements sampled from one forward).  actions_out dev
 * int32 [T][rows]: node-indexed within each forward's span (row order when graphs is
 * NULL); logp_out dev float64 [T][rows], topo-row indexed. */
int go_sample(go_ctx_t ctx, const go_config_t* cfg, int32_t num_forwards,
              const go_graph_t* graphs, const int64_t* row_counts,
              const uint64_t* pcg_states, const void* logits, int32_t logits_flags,
              double temperature, int32_t* actions_out, double* logp_out, void* stream);

/* PPO loss and parameter gradient of one minibatch (replaces training.py:146-227:
 * _sample_loss per sample + mean + Tensor.backward).  The samples are the forwards of
 * `batch` with their last-iteration inputs (prev_actions, embed_seeds = the bundle's
 * embed seed).  actions: dev int32 [T][rows], the sampled actions, node-indexed per
 * span; old_logp: dev float64 [T][rows], topo-row indexed; fparams: host [F][4] =
 * (advantage, temperature, reward, 0).  grads: dev float32 with the parameter-blob
 * layout, ACCUMULATED (caller zeroes per minibatch); the loss is the sum over the F
 * samples divided by loss_denominator (<= 0: F), so ranks holding parts of one
 * minibatch produce gradients that all-reduce(sum) to the minibatch mean.  stats_out: host float64 [14*F]: [F][3][4] (sum surr, sum entropy, sum
 * ratio, clipped count) per task slot, then [F] (value - reward)^2, then [F] value.
 * Kernels: attention forward (with log-sum-exp) and dq / dk,dv backward on split-fp16
 * mma.sync tensor cores (fp32-class, csrc/attn_bwd_mma.cu), forward and dX GEMMs on the
 * tcgen05 split-precision GEMM; fp32 SIMT re-runs gated on the fp16 range flags.
 * Environment: GO_TRAIN_ATTN=simt|mma16, GO_TRAIN_FWD=simt, GO_TRAIN_GEMM=simt select
 * the fp32 SIMT / single-fp16 variants (testing and A/B timing only). */
int go_ppo_grad(go_ctx_t ctx, const go_config_t* cfg, const float* params,
                const int64_t* param_offsets, const go_batch_t* batch, const int32_t* actions,
                const double* old_logp, const double* fparams, double clip_eps,
                double entropy_coef, double value_coef, int32_t loss_denominator, float* grads,
                double* stats_out, void* stream);

/* Fused bias-corrected Adam over a flat float32 blob (replaces tensor.py:428-441
 * ParamStore.adam_step; every element steps, zero gradient where none flowed). */
int go_adam(go_ctx_t ctx, float* params, const float* grads, float* m, float* v, int64_t count,
            int64_t step, double lr, double beta1, double beta2, double eps, void* stream);

/* Float64-master Adam (tensor.py:428-441 ParamStore.adam_step, same float64
 * operations in the same order): params / m / v are float64 device arrays kept across
 * the update, params32 receives the float32 copy the forward/backward kernels read. */
int go_adam64(go_ctx_t ctx, double* params, float* params32, const float* grads, double* m,
              double* v, int64_t count, int64_t step, double lr, double beta1, double beta2,
              double eps, void* stream);

/* Batched exact discrete-event simulation (simulator.py:280-441) of K placements of
 * one graph (its current fused tables) + reward (training.py:37-44).
 *   placement  dev int32 [K][n] node-indexed device per node
 *   priorities dev int32 [K][n] or [n] (prio_per_placement = 0)
 *   topology   host: peak[d], mem_bw[d], cap[d], link_bw[d*d]
 *   policy     0 = priority, 1 = fifo
 *   baseline   reward normaliser (> 0) or 0 to skip the reward
 * Outputs dev: step_time f64[K], valid u8[K], violation i8[K] (0 none, 1 colocation,
 * 2 oom, 3 cycle_after_fusion), busy f64[K][d], peak f64[K][d], reward f64[K]. */
int go_simulate(go_ctx_t ctx, go_graph_t g, int32_t num_placements, const int32_t* placement,
                const int32_t* priorities, int32_t prio_per_placement, int32_t d,
                const double* peak, const double* mem_bw, const double* cap,
                const double* link_bw, int32_t policy, double baseline,
                double* step_time, uint8_t* valid, int8_t* violation, double* busy,
                double* peak_mem, double* reward, void* stream);

/* One started compute or transfer of a traced simulation (simulator.py:61-67
 * TraceEvent): kind 0 = compute on device `src_or_device`, kind 1 = transfer on link
 * src_or_device -> dst; group_id = the computing group / the receiving group. */
typedef struct {
  double t_start, t_end;
  int32_t kind, src_or_device, dst, group_id;
} go_trace_event_t;

/* simulate(..., record_trace=True) for ONE placement (simulator.py:280-441 with the
 * trace appends of :360-373): same results as go_simulate (priorities per node,
 * device pointers) plus the device event log in start order; trace_count receives the
 * number of events (at most groups + cross-device edges; events past trace_capacity are
 * counted but not written).  The caller sorts them as simulator.py:432-433 does. */
int go_simulate_trace(go_ctx_t ctx, go_graph_t g, const int32_t* placement,
                      const int32_t* priorities, int32_t d, const double* peak,
                      const double* mem_bw, const double* cap, const double* link_bw,
                      int32_t policy, double* step_time, uint8_t* valid, int8_t* violation,
                      double* busy, double* peak_mem, go_trace_event_t* trace,
                      int64_t trace_capacity, int64_t* trace_count, void* stream);

/* Simulated annealing (baselines.py:146-206) of `chains` independent chains on the
 * device DES, one chain per 32-thread block.  rng_words (host) holds each chain's numpy
 * PCG64 state (state_hi, state_lo, inc_hi, inc_lo of default_rng(seed)); the chain
 * consumes it draw for draw like the reference (task index, node, value per move,
 * a uniform for an uphill move).  state / best: dev int32 [chains][2][n] (placement,
 * priorities), both set to the start assignment by the caller; best receives each
 * chain's best state and best_time (dev f64 [chains]) its step time (inf: none
 * valid).  Annealed tasks: task_slots[t] 0 = placement, 1 = schedule_priority, in the
 * caller's task order, with task_sizes[t] actions.  initial_temperature NaN = 10% of
 * the initial step time (1.0 if infinite). */
int go_anneal(go_ctx_t ctx, go_graph_t g, int32_t chains, const uint64_t* rng_words,
              int32_t* state, int32_t* best, int32_t d, const double* peak, const double* mem_bw,
              const double* cap, const double* link_bw, int32_t policy, int32_t iterations,
              int32_t moves_per_step, double initial_temperature, double cooling_rate,
              int32_t num_tasks, const int32_t* task_slots, const int32_t* task_sizes,
              double* best_time, void* stream);

#ifdef __cplusplus
}
#endif
#endif

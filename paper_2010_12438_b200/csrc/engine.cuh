// Internal structures of libgo_b200: context, graph handle, kernel launchers.
#pragma once
#include <cstddef>
#include <vector>

#include "common.cuh"

// Device view of one graph's static tables (topo-row space unless noted).
struct GraphView {
  int32_t n;
  const int32_t* order;    // topo row -> node id
  const int32_t* op_row;   // op index per topo row
  const float* static4;    // [n][4]: log1p(flops), log1p(out_bytes), indeg, outdeg
  const int64_t* nbr_off;  // [n+1] undirected neighbours, CSR by topo row
  const int32_t* nbr_row;  // neighbour topo rows, sorted by neighbour node id
  const int64_t* samp_off; // [n+1] prefix of min(deg, k) for the configured k
};

// One group's static DES fields packed in a 64-B record, so the event loop reaches all
// it needs about a group with one L2 round trip (the separate arrays below cost one
// dependent load each).  Offsets fit int32 (checked when the view is built).
struct __align__(64) DesGroupRec {
  double cost_flops, cost_bytes;
  int32_t topo, rep, pending0, nsucc;  // one 16-B load for the per-placement state fill
  int32_t out_off, out_cnt;     // external out edges [out_off, out_off + out_cnt)
  int32_t pred_off, pred_cnt;   // distinct predecessor groups (16-B aligned: one load)
  double resident;
  int32_t pad[2];
};
static_assert(sizeof(DesGroupRec) == 64 && offsetof(DesGroupRec, topo) % 16 == 0 &&
                  offsetof(DesGroupRec, out_off) % 16 == 0,
              "DesGroupRec vector loads need 16-B aligned fields");

// Device DES tables of the current (fused) grouping: simulator.py:86-172.
struct DesView {
  const DesGroupRec* grec;     // [G] packed per-group record (the event loop reads these)
  const int32_t* src_grp;      // groups without external in-edges, ascending
  int32_t num_src;
  int32_t n, G;
  const int32_t* grp_rep;      // [G] lowest member node id
  const int32_t* pending0;     // [G] #external in-edges
  const int64_t* out_off;      // [G+1] external out edges sorted (src, dst), stable
  const int32_t* out_grp;      // destination group per out edge
  const double* out_bytes;     // bytes per out edge
  const double* cost_flops;    // [G]
  const double* cost_bytes;    // [G]
  const int32_t* topo_index;   // [G]
  const double* resident;      // [G]
  const int32_t* nsucc;        // [G] distinct successor groups
  const int64_t* pred_off;     // [G+1] distinct predecessor groups
  const int32_t* pred_grp;
  const int64_t* coloc_off;    // [C+1] colocation groups -> member groups
  const int32_t* coloc_grp;
  int32_t num_coloc;
  int32_t mem_int_exact;       // all resident bytes integral and sum < 2**53
  int64_t max_out_deg;
  int64_t num_edges;            // external out edges in total
};

// Kernel classes timed with CUDA events on the launching stream (go_ctx_set_timing).
enum KernelClass { K_HEADS_ATTN = 0, K_TRUNK_ATTN, K_SEGMAX, K_GEMM, K_DES, K_SAMPLE,
                   K_NEIGHBOR, K_OTHER, K_NUM_CLASSES };

struct TimedLaunch {
  int cls;
  cudaEvent_t a, b;
  double work;  // algorithmic units (flops or bytes) of this launch, set by the caller
};

struct go_ctx {
  int device = 0;
  bool timing = false;
  std::vector<TimedLaunch> timed;
  std::vector<cudaEvent_t> event_pool;
  double stat_ms[K_NUM_CLASSES] = {0};
  double stat_work[K_NUM_CLASSES] = {0};
  long long stat_count[K_NUM_CLASSES] = {0};
  cudaEvent_t get_event();
  void resolve_timing();
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* ws_small = nullptr;  // metadata uploads (row offsets, tiles, graph views)
  size_t ws_small_bytes = 0;
  void* pinned = nullptr;    // pinned staging for metadata
  size_t pinned_bytes = 0;
  cudaEvent_t staged = nullptr;  // last metadata upload done
  void* des_ws = nullptr;
  size_t des_ws_bytes = 0;
  void* ensure(size_t bytes);
  void* ensure_small(size_t bytes);
  void* ensure_pinned(size_t bytes);
  void* ensure_des(size_t bytes);
  ~go_ctx();
};

struct go_graph {
  go_ctx* ctx = nullptr;
  int32_t n = 0;
  int64_t e = 0;
  std::vector<int32_t> order, pos, op, src, dst, coloc;
  std::vector<double> flops, out_bytes, ebytes;
  std::vector<int64_t> nbr_off;
  std::vector<int32_t> nbr_row;
  // device
  int32_t* d_order = nullptr;
  int32_t* d_op_row = nullptr;
  float* d_static4 = nullptr;
  int64_t* d_nbr_off = nullptr;
  int32_t* d_nbr_row = nullptr;
  int64_t* d_samp_off = nullptr;
  int32_t samp_k = -1;
  int64_t samp_total = 0;
  // DES
  DesView des{};
  std::vector<void*> des_allocs;
  bool acyclic = true;
  void set_fusion(const std::vector<int64_t>& label);
  void ensure_samp(int32_t k);
  GraphView view() const;
  ~go_graph();
};

namespace go {

// RAII: records start/stop events around the launches in its scope when timing is on.
struct KTimer {
  go_ctx* ctx;
  int cls;
  cudaStream_t st;
  double work;
  cudaEvent_t a = nullptr;
  KTimer(go_ctx* c, int k, cudaStream_t s, double w) : ctx(c), cls(k), st(s), work(w) {
    if (ctx && ctx->timing) {
      a = ctx->get_event();
      cudaEventRecord(a, st);
    }
  }
  ~KTimer() {
    if (ctx && ctx->timing && a) {
      cudaEvent_t b = ctx->get_event();
      cudaEventRecord(b, st);
      ctx->timed.push_back({cls, a, b, work});
    }
  }
};

// ---- kernels: dense.cu
void gemm(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
          const float* W, int64_t ldw, const float* bias, float* C, int64_t ldc, int64_t M,
          int N, int act, cudaStream_t st);
void add_layernorm(const float* a, int64_t lda, const float* b, int64_t ldb, const float* g,
                   const float* beta, float* out, int64_t ldo, int64_t M, int D, cudaStream_t st);
void mul_rowvec(const float* x, int64_t ldx, const float* vec, int64_t ldv,
                const int32_t* row_fwd, float* out, int64_t ldo, int64_t M, int D,
                cudaStream_t st);
constexpr int MEAN_CHUNK = 256;
void mean_rows(const float* x, int64_t ldx, const int64_t* row_off_dev, int F,
               const int64_t* chunk_tab, int64_t nc, int D, float* out, int64_t ldo,
               float* part, cudaStream_t st,
               int32_t* finite_flag = nullptr);
void check_finite(const float* x, int64_t ld, int64_t M, int D, int32_t* flag, cudaStream_t st);
void row_fwd_fill(const int64_t* row_off_dev, int F, int64_t R, int32_t* row_fwd,
                  cudaStream_t st);
// one length-1 transformer block + 2*sigmoid per forward (policy.py:122-132)
struct BlockW {
  const float *v_w, *v_b, *o_w, *o_b, *ln1_g, *ln1_b, *w1, *b1, *w2, *b2, *ln2_g, *ln2_b;
};
void modulate(const float* graph_embed, int64_t ldg, int F, int gs_dim, const float* in_w,
              const float* in_b, const BlockW& w, int d_model, int d_head_total, int d_inner,
              float* mod_out, cudaStream_t st);
void value_head(const float* mean, int F, int D, const float* w, const float* b, float* out,
                cudaStream_t st);

// ---- kernels: embed.cu
void neighbor_sample(const GraphView* views_dev, const int64_t* row_off_dev,
                     const int64_t* gbase_dev, const int64_t* seeds_dev, int F,
                     int64_t total_rows, const int32_t* row_fwd, int k, int32_t* gidx,
                     int32_t* segoff, cudaStream_t st);
void features_inproj(const GraphView* views_dev, const int64_t* row_off_dev,
                     const int32_t* row_fwd, int64_t R, const int32_t* prev_actions,
                     int num_tasks, const int32_t* task_col, const float* in_w,
                     const float* in_b, int D, float* h, int64_t ldh, cudaStream_t st);
// segoff[R+1]: flat segment bounds into gidx, written by neighbor_sample
// sigmoid_of_max: t holds pre-activations; out = sigmoid(max) (= max of sigmoid)
void segment_max(const float* t, int64_t ldt, const int32_t* segoff, const int32_t* gidx,
                 int64_t R, int D, float* out, int64_t ldo, cudaStream_t st,
                 int32_t* argmax = nullptr, bool sigmoid_of_max = false);

void row_node_fill(const GraphView* views_dev, const int64_t* row_off_dev,
                   const int32_t* row_fwd, int64_t R, int32_t* row_node, cudaStream_t st);

// ---- kernels: attention.cu
struct AttnTile {
  int64_t q0, q1, k0, k1;
};
// gate (optional): run only if *gate != 0 (the re-run behind the tensor-core trunk kernel)
void attention(const float* q, const float* k, const float* v, int64_t ld, int n_head,
               int d_head, const AttnTile* tiles_dev, int64_t num_tiles, float* out,
               int64_t ldo, cudaStream_t st, float* lse = nullptr,
               const int32_t* gate = nullptr, const float* kalt = nullptr,
               const float* valt = nullptr);

// ---- kernels: tc_attention16.cu (fp16 operands, fixed-offset softmax; flags the launch
// over to the tf32 / online kernels when a bound exceeds the fp16-exact range)
struct TcWork;
void attention_f16_tc(const float* q, const float* k, const float* v, int64_t ld, int n_head,
                      int d_head, int64_t R, int64_t Ttot, const TcWork* works_dev,
                      int64_t num_works, const int64_t* tile_row0_dev, const int32_t* tile_n_dev,
                      void* qh, void* kb, void* vb, float* out, int64_t ldo,
                      const int32_t* row_fwd, unsigned* kmax, int32_t* flag, int32_t* wflag,
                      float qscale, cudaStream_t st);

// ---- kernels: trunk_mma.cu (banded trunk attention on mma.sync m16n8k16, d_head <= 16);
// *flag (zeroed here) is set if some operand left the fp16 range -- the caller then
// re-runs attention() gated on it
bool trunk_mma_supported(int d_head);
void trunk_attention_mma(const float* q, const float* k, const float* v, int64_t ld, int n_head,
                         int d_head, const AttnTile* tiles_dev, int64_t num_tiles, float* out,
                         int64_t ldo, int32_t* flag, cudaStream_t st, float* lse = nullptr,
                         bool split = false);

// ---- kernels: tc_attention.cu (tcgen05 / TMEM full attention, d_head <= 16)
struct TcWork {
  int32_t f, q0, n, tiles;
  int64_t row0, tile0;
};
bool tc_attention_supported(int d_head);
// works: 384-query items (one CTA each in the fp16 and tf32 kernels)
void tc_build_tables(const std::vector<int64_t>& row_off, std::vector<TcWork>& works,
                     std::vector<int64_t>& tile_row0, std::vector<int32_t>& tile_n);
// int32 scratch attention_full_tc needs: launch flag, max |k| per (forward, head),
// fallback marks per (head, work item)
int64_t tc_attention_scratch_ints(int F, int n_head, int64_t num_works);
void attention_full_tc(const float* q, const float* k, const float* v, int64_t ld, int n_head,
                       int d_head, int64_t R, int64_t Ttot, const TcWork* works_dev,
                       int64_t num_works, const int64_t* tile_row0_dev,
                       const int32_t* tile_n_dev, float* qh, float* kb, float* vb, float* out,
                       int64_t ldo, const int32_t* row_fwd, int F, int32_t* scratch,
                       cudaStream_t st);

// per-call batch metadata (engine.cu make_meta): row offsets, graph views, tiles
struct BatchMeta {
  int F = 0;
  int64_t R = 0;
  std::vector<int64_t> row_off, gbase;
  int64_t gtotal = 0;
  // device
  const int64_t* d_row_off = nullptr;
  const int64_t* d_seeds = nullptr;
  const int64_t* d_gbase = nullptr;
  const GraphView* d_views = nullptr;
  const AttnTile* d_trunk_tiles = nullptr;
  int64_t n_trunk_tiles = 0;
  const AttnTile* d_head_tiles = nullptr;
  int64_t n_head_tiles = 0;
  const int64_t* d_chunks = nullptr;
  int64_t n_chunks = 0;
  double trunk_pairs = 0, head_pairs = 0;  // sum of (query, key) pairs per head
  // tensor-core heads attention tables
  const TcWork* d_tc_works = nullptr;
  int64_t n_tc_works = 0;
  const int64_t* d_tile_row0 = nullptr;
  const int32_t* d_tile_n = nullptr;
  int64_t n_tiles = 0;
};
BatchMeta make_meta(go_ctx* ctx, const go_config_t& cfg, const go_batch_t& b, bool need_embed,
                    bool need_trunk, bool need_heads, cudaStream_t st, const void* extra = nullptr,
                    size_t extra_bytes = 0, const void** extra_dev = nullptr);

// ---- kernels: tc_gemm.cu (tcgen05 3-pass split-precision dense layers)
// Prepacked weight: tf32 hi/lo (w32) and fp16 hi/lo of W * 2^8 (w16, optional) plus the
// fp16 pass's range flag (ovf, zero-initialised; optional).
struct TcW {
  const float* w32 = nullptr;
  const void* w16 = nullptr;
  int32_t* ovf = nullptr;
  const int32_t* gate = nullptr;  // set: tf32 pass only, run only if *gate != 0
};
int tc_gemm_bn(int N);
size_t tc_gemm_packed_floats(int K, int N);
void tc_gemm_pack(const float* W0, const float* W1, const float* W2, int Nsub, int64_t ldw, int K,
                  int N, float* out, cudaStream_t st);
void tc_gemm_pack16(const float* W0, const float* W1, const float* W2, int Nsub, int64_t ldw,
                    int K, int N, void* out, cudaStream_t st,
                    int32_t* ovf = nullptr);
void tc_gemm(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
             const TcW& W, const float* bias, float* C, int64_t ldc, int64_t M, int N, int act,
             cudaStream_t st);
// C2 = act(A1 @ W + bias) * rowscale[row_fwd[r]] (rowscale: [F, N]); C (unscaled) optional
void tc_gemm_scaled(const float* A1, int64_t lda1, int K1, const TcW& Wpk, const float* bias,
                    float* C, int64_t ldc, const float* rowscale, const int32_t* row_fwd,
                    float* C2, int64_t ldc2, int64_t M, int N, int act, cudaStream_t st);
void tc_gemm_pack16_bn(const float* W, int64_t ldw, int K, int N, int BN, void* out,
                       cudaStream_t st, int32_t* ovf);
// fused trunk FFN: C = LN(X + relu(X W1 + b1) W2 + b2) * g + beta, C2 = C * rowscale
// (d_model 128, d_inner 512); *ovf set if X / H leave the fp16 range (caller re-runs)
void tc_ffn(const float* X, int64_t ldx, const void* W1_16, const void* W2_16, const float* b1,
            const float* b2, const float* g, const float* beta, float* C, int64_t ldc,
            const float* rowscale, const int32_t* row_fwd, float* C2, int64_t ldc2, int64_t M,
            int32_t* ovf, cudaStream_t st, bool layernorm = true);
void tc_gemm_ln(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
                const TcW& W, const float* bias, const float* resid, int64_t ldr,
                const float* g, const float* beta, float* C, int64_t ldc, const float* rowscale,
                const int32_t* row_fwd, float* C2, int64_t ldc2, int64_t M, int N,
                cudaStream_t st);

// ---- kernels: sample.cu
void sample_rows(const void* logits, int logits_f64, int64_t ldl, int a, int64_t R,
                 const int64_t* row_off_dev, const int32_t* row_fwd, const int32_t* order_of_row,
                 const uint64_t* pcg_dev, int64_t task, double temperature,
                 int32_t* actions, double* logp, cudaStream_t st, bool shared = false);

// ---- kernels: des.cu
// device simulated annealing, C chains (des.cu anneal_kernel); cur / best: dev
// [C][2][n] (placement | priorities), both initialised to the start state by the caller
int anneal_chains(const DesView& v, int C, const uint64_t* rng_words_host, int32_t* cur,
                  int32_t* best, int d, const double* peak, const double* mem_bw,
                  const double* cap, const double* link_bw, int policy, int iterations,
                  int moves, double t_init, double cooling, int ntasks, const int* slots,
                  const int* sizes, double* best_time, go_ctx* ctx, cudaStream_t st);
struct DesTraceRec {  // one started compute / transfer of a traced simulation
  double t0, t1;
  int32_t kind, a, b, grp;
};
int simulate_batch(const DesView& v, int K, const int32_t* placement, int64_t pstride,
                   const int32_t* prio, int64_t prio_stride, int d, const double* peak,
                   const double* mem_bw, const double* cap, const double* link_bw, int policy,
                   double baseline, double* step_time, uint8_t* valid, int8_t* violation,
                   double* busy, double* peak_mem, double* reward, go_ctx* ctx,
                   cudaStream_t st, DesTraceRec* trace = nullptr, int64_t trace_cap = 0,
                   int64_t* trace_count = nullptr);

}  // namespace go

// libgo_b200 engine: context/workspace management, the batched policy forward
// (embed -> trunk -> heads, embedding.py:73-98 + policy.py:135-217), sampling and
// simulation entry points of the C-ABI (include/go_b200.h).
#include <algorithm>
#include <cstring>
#include <mutex>

#include "engine.cuh"

namespace go {

std::atomic<long long> g_launch_count{0};
static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

int num_sms() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// ---------------------------------------------------------------------------------
// Parameter slots (canonical order; mirrored by paper_2010_12438_b200/params.py).
struct Slots {
  int gs_layers, trf_layers, T;
  int e_in_w() const { return 0; }
  int e_in_b() const { return 1; }
  int e_layer(int l, int w) const { return 2 + 4 * l + w; }  // agg_w, agg_b, fc_w, fc_b
  int pbase() const { return 2 + 4 * gs_layers; }
  int p_in_w() const { return pbase(); }
  int p_in_b() const { return pbase() + 1; }
  // block b in [0, trf_layers]; b == trf_layers is policy/mod/
  int blk(int b, int w) const { return pbase() + 2 + 16 * b + w; }
  int ta(int w) const { return pbase() + 2 + 16 * (trf_layers + 1) + w; }
  int task(int t, int w) const { return ta(8) + 10 * t + w; }
  int value_w() const { return ta(8) + 10 * T; }
  int value_b() const { return value_w() + 1; }
  int count() const { return value_b() + 1; }
};
enum { Q_W = 0, Q_B, K_W, K_B, V_W, V_B, O_W, O_B, LN1_G, LN1_B, FF_W1, FF_B1, FF_W2, FF_B2,
       LN2_G, LN2_B };
enum { CAT_W = 0, CAT_B, LN_G, LN_B, FC_W1, FC_B1, FC_W2, FC_B2, OUT_W, OUT_B };

static Slots slots_of(const go_config_t& c) { return Slots{c.gs_layers, c.trf_layers, c.num_tasks}; }

static void validate(const go_config_t& c) {
  GO_CHECK(c.gs_layers >= 0 && c.gs_dim > 0 && c.gs_knn >= 1, "bad EmbedConfig");
  GO_CHECK(c.trf_layers >= 0 && c.d_model > 0 && c.n_head > 0 && c.d_head > 0 && c.d_inner > 0 &&
               c.segment_len > 0,
           "bad PolicyConfig");
  GO_CHECK(c.num_tasks >= 1 && c.num_tasks <= 3, "at least one task required");
  for (int t = 0; t < c.num_tasks; ++t) GO_CHECK(c.task_sizes[t] >= 1, "empty action space");
}

// ---------------------------------------------------------------------------------
// Metadata staging: host tables packed into one pinned buffer, one H2D copy.
struct Stager {
  std::vector<char> buf;
  size_t add(const void* p, size_t bytes) {
    size_t off = round_up((int64_t)buf.size(), 256);
    buf.resize(off + bytes);
    if (bytes) std::memcpy(buf.data() + off, p, bytes);
    return off;
  }
  template <class T>
  size_t add(const std::vector<T>& v) {
    return add(v.data(), v.size() * sizeof(T));
  }
  char* upload(go_ctx* ctx, cudaStream_t st) {
    char* dev = reinterpret_cast<char*>(ctx->ensure_small(std::max<size_t>(buf.size(), 256)));
    char* pin = reinterpret_cast<char*>(ctx->ensure_pinned(std::max<size_t>(buf.size(), 256)));
    std::memcpy(pin, buf.data(), buf.size());
    CUDA_CHECK(cudaMemcpyAsync(dev, pin, buf.size(), cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaEventRecord(ctx->staged, st));
    return dev;
  }
};



static void build_tiles(const std::vector<int64_t>& row_off, int64_t S, bool banded,
                        std::vector<AttnTile>& out) {
  const int64_t QT = 64;
  for (size_t f = 0; f + 1 < row_off.size(); ++f) {
    int64_t f0 = row_off[f], f1 = row_off[f + 1];
    if (!banded) {
      for (int64_t q = f0; q < f1; q += QT) out.push_back({q, std::min(q + QT, f1), f0, f1});
      continue;
    }
    for (int64_t s0 = f0; s0 < f1; s0 += S) {
      int64_t s1 = std::min(s0 + S, f1);
      int64_t k0 = std::max(f0, s0 - S);
      for (int64_t q = s0; q < s1; q += QT) out.push_back({q, std::min(q + QT, s1), k0, s1});
    }
  }
}

BatchMeta make_meta(go_ctx* ctx, const go_config_t& cfg, const go_batch_t& b,
                     bool need_embed, bool need_trunk, bool need_heads, cudaStream_t st,
                     const void* extra, size_t extra_bytes, const void** extra_dev) {
  BatchMeta m;
  m.F = b.num_forwards;
  GO_CHECK(m.F >= 1, "empty batch");
  m.row_off.assign(m.F + 1, 0);
  m.gbase.assign(m.F, 0);
  std::vector<GraphView> views(m.F);
  std::vector<int64_t> seeds(m.F, 0);
  GO_CHECK(b.graphs || (b.row_counts && !need_embed), "graph handles required");
  for (int f = 0; f < m.F; ++f) {
    m.gbase[f] = m.gtotal;
    seeds[f] = b.embed_seeds ? b.embed_seeds[f] : 0;
    GO_CHECK(seeds[f] >= 0, "seed must be non-negative");
    if (!b.graphs) {
      GO_CHECK(b.row_counts[f] >= 0, "negative row count");
      m.row_off[f + 1] = m.row_off[f] + b.row_counts[f];
      views[f] = GraphView{};
      views[f].n = (int32_t)b.row_counts[f];
      continue;
    }
    go_graph* g = b.graphs[f];
    GO_CHECK(g != nullptr, "null graph handle");
    if (need_embed) g->ensure_samp(cfg.gs_knn);
    m.row_off[f + 1] = m.row_off[f] + g->n;
    m.gtotal += need_embed ? g->samp_total : 0;
    views[f] = g->view();
  }
  m.R = m.row_off[m.F];
  Stager s;
  size_t o_row = s.add(m.row_off), o_seed = s.add(seeds), o_gb = s.add(m.gbase),
         o_views = s.add(views);
  std::vector<AttnTile> tt, ht;
  if (need_trunk) build_tiles(m.row_off, cfg.segment_len, true, tt);
  if (need_heads) build_tiles(m.row_off, 0, false, ht);
  for (auto& t : tt) m.trunk_pairs += (double)(t.q1 - t.q0) * (double)(t.k1 - t.k0);
  for (auto& t : ht) m.head_pairs += (double)(t.q1 - t.q0) * (double)(t.k1 - t.k0);
  size_t o_tt = s.add(tt), o_ht = s.add(ht);
  std::vector<TcWork> tcw;
  std::vector<int64_t> trow0;
  std::vector<int32_t> tn;
  if (need_heads) tc_build_tables(m.row_off, tcw, trow0, tn);
  size_t o_tcw = s.add(tcw), o_tr = s.add(trow0), o_tn = s.add(tn);
  // mean chunks: [nc] r0, [nc] r1, [F] first, [F] end
  std::vector<int64_t> c0, c1, f0(m.F), f1(m.F);
  for (int f = 0; f < m.F; ++f) {
    f0[f] = (int64_t)c0.size();
    for (int64_t r = m.row_off[f]; r < m.row_off[f + 1]; r += MEAN_CHUNK) {
      c0.push_back(r);
      c1.push_back(std::min<int64_t>(r + MEAN_CHUNK, m.row_off[f + 1]));
    }
    f1[f] = (int64_t)c0.size();
  }
  m.n_chunks = (int64_t)c0.size();
  std::vector<int64_t> ch;
  ch.insert(ch.end(), c0.begin(), c0.end());
  ch.insert(ch.end(), c1.begin(), c1.end());
  ch.insert(ch.end(), f0.begin(), f0.end());
  ch.insert(ch.end(), f1.begin(), f1.end());
  size_t o_ch = s.add(ch);
  size_t o_ex = s.add(extra, extra_bytes);
  char* dev = s.upload(ctx, st);
  if (extra_dev) *extra_dev = dev + o_ex;
  m.d_row_off = reinterpret_cast<const int64_t*>(dev + o_row);
  m.d_seeds = reinterpret_cast<const int64_t*>(dev + o_seed);
  m.d_gbase = reinterpret_cast<const int64_t*>(dev + o_gb);
  m.d_views = reinterpret_cast<const GraphView*>(dev + o_views);
  m.d_trunk_tiles = reinterpret_cast<const AttnTile*>(dev + o_tt);
  m.n_trunk_tiles = (int64_t)tt.size();
  m.d_head_tiles = reinterpret_cast<const AttnTile*>(dev + o_ht);
  m.n_head_tiles = (int64_t)ht.size();
  m.d_chunks = reinterpret_cast<const int64_t*>(dev + o_ch);
  m.d_tc_works = reinterpret_cast<const TcWork*>(dev + o_tcw);
  m.n_tc_works = (int64_t)tcw.size();
  m.d_tile_row0 = reinterpret_cast<const int64_t*>(dev + o_tr);
  m.d_tile_n = reinterpret_cast<const int32_t*>(dev + o_tn);
  m.n_tiles = (int64_t)trow0.size();
  return m;
}

// Simple bump allocator over the context workspace.
struct Arena {
  char* base;
  size_t off = 0, cap;
  template <class T>
  T* take(int64_t count) {
    size_t bytes = round_up(std::max<int64_t>(count, 1) * (int64_t)sizeof(T), 256);
    GO_CHECK(off + bytes <= cap, "workspace overflow");
    T* p = reinterpret_cast<T*>(base + off);
    off += bytes;
    return p;
  }
};

static inline int64_t ldp(int w) { return round_up(w, 4); }

static size_t forward_ws_bytes(const go_config_t& c, int64_t R, int64_t gtotal, int F,
                               int64_t nchunks) {
  int64_t wmax = std::max(c.gs_dim, c.d_model);
  int64_t W = (int64_t)c.n_head * c.d_head;
  int64_t per_row = 6 * ldp((int)wmax) + 4 * ldp((int)W) + ldp(c.d_inner);
  // + tensor-core attention operands: qh [H][R][16], kb/vb [H][tiles*64][16]
  per_row += 3 * (int64_t)c.n_head * 16 + 2;
  size_t b = (size_t)R * per_row * 4 + (size_t)R * 12 + (size_t)gtotal * 4 + 512 +
             (size_t)F * 2 * c.n_head * 64 * 16 * 4 +
             (size_t)(F + 4) * (ldp(c.d_model) + ldp(c.gs_dim)) * 8 +
             (size_t)(nchunks + 4) * wmax * 4 + 64 * 256;
  return b + (1 << 20);
}

}  // namespace go

using namespace go;

// ---------------------------------------------------------------------------------
void* go_ctx::ensure(size_t bytes) {
  if (bytes > ws_bytes) {
    if (ws) CUDA_CHECK(cudaFree(ws));
    ws = nullptr;
    size_t nb = std::max(bytes, ws_bytes + ws_bytes / 4);
    CUDA_CHECK(cudaMalloc(&ws, nb));
    ws_bytes = nb;
  }
  return ws;
}
void* go_ctx::ensure_small(size_t bytes) {
  if (bytes > ws_small_bytes) {
    if (staged) CUDA_CHECK(cudaEventSynchronize(staged));
    if (ws_small) CUDA_CHECK(cudaFree(ws_small));
    ws_small = nullptr;
    size_t nb = std::max(bytes, (size_t)1 << 20);
    CUDA_CHECK(cudaMalloc(&ws_small, nb));
    ws_small_bytes = nb;
  } else if (staged) {
    // the previous call's kernels may still read the small buffer
    CUDA_CHECK(cudaEventSynchronize(staged));
  }
  return ws_small;
}
void* go_ctx::ensure_pinned(size_t bytes) {
  if (bytes > pinned_bytes) {
    if (pinned) CUDA_CHECK(cudaFreeHost(pinned));
    pinned = nullptr;
    size_t nb = std::max(bytes, (size_t)1 << 20);
    CUDA_CHECK(cudaMallocHost(&pinned, nb));
    pinned_bytes = nb;
  }
  return pinned;
}
void* go_ctx::ensure_des(size_t bytes) {
  if (bytes > des_ws_bytes) {
    if (des_ws) CUDA_CHECK(cudaFree(des_ws));
    des_ws = nullptr;
    CUDA_CHECK(cudaMalloc(&des_ws, bytes));
    des_ws_bytes = bytes;
  }
  return des_ws;
}
cudaEvent_t go_ctx::get_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CUDA_CHECK(cudaEventCreate(&e));
  return e;
}

void go_ctx::resolve_timing() {
  for (auto& t : timed) {
    CUDA_CHECK(cudaEventSynchronize(t.b));
    float ms = 0.f;
    CUDA_CHECK(cudaEventElapsedTime(&ms, t.a, t.b));
    stat_ms[t.cls] += ms;
    stat_work[t.cls] += t.work;
    stat_count[t.cls] += 1;
    event_pool.push_back(t.a);
    event_pool.push_back(t.b);
  }
  timed.clear();
}

go_ctx::~go_ctx() {
  for (auto& t : timed) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto e : event_pool) cudaEventDestroy(e);
  if (staged) cudaEventSynchronize(staged);
  cudaDeviceSynchronize();
  if (ws) cudaFree(ws);
  if (ws_small) cudaFree(ws_small);
  if (pinned) cudaFreeHost(pinned);
  if (des_ws) cudaFree(des_ws);
  if (staged) cudaEventDestroy(staged);
}

// ---------------------------------------------------------------------------------
// The forward.  Stage order and math follow the reference exactly; every dense op
// is one launch over all rows of all forwards in the batch.
static void run_forward(go_ctx* ctx, const go_config_t& cfg, const float* P,
                        const int64_t* off, const go_batch_t& b, float* node_embed,
                        float* graph_embed, float* hid, float* logits, float* value,
                        int32_t* status_dev, cudaStream_t st) {
  validate(cfg);
  const bool do_e = b.stage_mask & 1, do_t = b.stage_mask & 2, do_h = b.stage_mask & 4;
  BatchMeta m = make_meta(ctx, cfg, b, do_e, do_t, do_h, st);
  const int64_t R = m.R;
  const int F = m.F;
  Slots S = slots_of(cfg);
  auto W_ = [&](int slot) { return P + off[slot]; };
  const int gs = cfg.gs_dim, dm = cfg.d_model, W = cfg.n_head * cfg.d_head, di = cfg.d_inner;
  const int64_t wmax = std::max(gs, dm);
  const int64_t LW = ldp((int)wmax), LA = ldp(W), LI = ldp(di);
  const size_t hook_bytes =
      b.cache_hook ? (size_t)cfg.trf_layers * R * (ldp(cfg.d_model) + 2 * LA + 192) * 4 : 0;
  Arena A{reinterpret_cast<char*>(
              ctx->ensure(forward_ws_bytes(cfg, R, m.gtotal, F, m.n_chunks) + hook_bytes)),
          0, ctx->ws_bytes};
  float* X[6];
  for (int i = 0; i < 6; ++i) X[i] = A.take<float>(R * LW);
  float* Qb = A.take<float>(R * LA);
  float* Kb = A.take<float>(R * LA);
  float* Vb = A.take<float>(R * LA);
  float* Ab = A.take<float>(R * LA);
  float* F1 = A.take<float>(R * LI);
  int32_t* row_fwd = A.take<int32_t>(R);
  GO_CHECK(m.gtotal + R < ((int64_t)1 << 31), "neighbour list exceeds 2^31 entries");
  int32_t* gidx = A.take<int32_t>(m.gtotal);
  int32_t* segoff = A.take<int32_t>(R + 1);
  float* mod = A.take<float>((int64_t)F * dm);
  float* meanb = A.take<float>((int64_t)F * dm);
  float* part = A.take<float>((m.n_chunks + 1) * wmax);
  row_fwd_fill(m.d_row_off, F, R, row_fwd, st);

  // ---- embed (embedding.py:73-98)
  if (do_e) {
    GO_CHECK(node_embed && graph_embed, "embed outputs required");
    int32_t tcol[3] = {0, 0, 0};
    int c = 16;
    for (int t = 0; t < cfg.num_tasks; ++t) {
      tcol[t] = c;
      c += cfg.task_sizes[t];
    }
    neighbor_sample(m.d_views, m.d_row_off, m.d_gbase, m.d_seeds, F, R, row_fwd, cfg.gs_knn,
                    gidx, segoff, st);
    float* h = cfg.gs_layers == 0 ? node_embed : X[0];
    if (b.features)  // explicit feature matrix (embed() called with features)
      gemm(b.features, b.feature_dim, b.feature_dim, nullptr, 0, 0, W_(S.e_in_w()), gs,
           W_(S.e_in_b()), h, cfg.gs_layers == 0 ? gs : LW, R, gs, 0, st);
    else
      features_inproj(m.d_views, m.d_row_off, row_fwd, R, b.prev_actions, cfg.num_tasks, tcol,
                      W_(S.e_in_w()), W_(S.e_in_b()), gs, h, cfg.gs_layers == 0 ? gs : LW, st);
    int64_t ldh = LW;
    for (int l = 0; l < cfg.gs_layers; ++l) {
      float* t = X[1];
      float* pooled = X[2];
      gemm(h, ldh, gs, nullptr, 0, 0, W_(S.e_layer(l, 0)), gs, W_(S.e_layer(l, 1)), t, LW, R, gs,
           2, st);
      {
        // algorithmic bytes: gathered rows + output rows (fp32) + indices (int32) +
        // segment offsets (int64) + row->forward map (int32)
        double bytes = (double)(m.gtotal + R) * gs * 4 + (double)m.gtotal * 4 +
                       (double)(R + 1) * 8 + (double)R * 4;
        KTimer kt(ctx, K_SEGMAX, st, bytes);
        segment_max(t, LW, segoff, gidx, R, gs, pooled, LW,
                    st);
      }
      bool last = l == cfg.gs_layers - 1;
      float* hn = last ? node_embed : (h == X[0] ? X[3] : X[0]);
      int64_t ldn = last ? gs : LW;
      gemm(h, ldh, gs, pooled, LW, gs, W_(S.e_layer(l, 2)), gs, W_(S.e_layer(l, 3)), hn, ldn, R,
           gs, 1, st);
      h = hn;
      ldh = ldn;
    }
    // non-finite check fused into the mean's pass over node_embed
    mean_rows(node_embed, gs, m.d_row_off, F, m.d_chunks, m.n_chunks, gs, graph_embed, gs, part,
              st, status_dev);
  }

  // ---- trunk (policy.py:122-177), layer-major block-banded attention
  if (do_t) {
    GO_CHECK(!b.cache_hook || (F == 1 && cfg.segment_len <= 64),
             "the trunk cache hook needs one forward and segment_len <= 64");
    GO_CHECK(node_embed && graph_embed && hid, "trunk inputs/outputs required");
    const float* modp = b.mod_override;
    if (!modp) {
      int mb = cfg.trf_layers;
      BlockW bw{W_(S.blk(mb, V_W)),  W_(S.blk(mb, V_B)),  W_(S.blk(mb, O_W)),  W_(S.blk(mb, O_B)),
                W_(S.blk(mb, LN1_G)), W_(S.blk(mb, LN1_B)), W_(S.blk(mb, FF_W1)),
                W_(S.blk(mb, FF_B1)), W_(S.blk(mb, FF_W2)), W_(S.blk(mb, FF_B2)),
                W_(S.blk(mb, LN2_G)), W_(S.blk(mb, LN2_B))};
      modulate(graph_embed, gs, F, gs, W_(S.p_in_w()), W_(S.p_in_b()), bw, dm, W, di, mod, st);
      modp = mod;
    }
    float* x = cfg.trf_layers == 0 ? hid : X[0];
    int64_t ldx = cfg.trf_layers == 0 ? dm : LW;
    gemm(node_embed, gs, gs, nullptr, 0, 0, W_(S.p_in_w()), dm, W_(S.p_in_b()), x, ldx, R, dm, 0,
         st);
    for (int l = 0; l < cfg.trf_layers; ++l) {
      float* xm = X[1];
      mul_rowvec(x, ldx, modp, dm, row_fwd, xm, LW, R, dm, st);
      gemm(xm, LW, dm, nullptr, 0, 0, W_(S.blk(l, Q_W)), W, W_(S.blk(l, Q_B)), Qb, LA, R, W, 0, st);
      gemm(xm, LW, dm, nullptr, 0, 0, W_(S.blk(l, K_W)), W, W_(S.blk(l, K_B)), Kb, LA, R, W, 0, st);
      gemm(xm, LW, dm, nullptr, 0, 0, W_(S.blk(l, V_W)), W, W_(S.blk(l, V_B)), Vb, LA, R, W, 0, st);
      if (b.cache_hook) {  // cache_perturb (policy.py:170-172), see run_forward_tc
        std::vector<float> hx((size_t)R * dm);
        CUDA_CHECK(cudaMemcpy2DAsync(hx.data(), dm * 4, xm, LW * 4, dm * 4, R,
                                     cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        std::vector<float> hp = hx;
        b.cache_hook(b.cache_hook_user, l, hx.data(), hp.data(), R, dm);
        float* pfx = A.take<float>(R * dm);
        float* kp = A.take<float>(R * LA);
        float* vp = A.take<float>(R * LA);
        CUDA_CHECK(cudaMemcpyAsync(pfx, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice, st));
        gemm(pfx, dm, dm, nullptr, 0, 0, W_(S.blk(l, K_W)), W, W_(S.blk(l, K_B)), kp, LA, R, W, 0,
             st);
        gemm(pfx, dm, dm, nullptr, 0, 0, W_(S.blk(l, V_W)), W, W_(S.blk(l, V_B)), vp, LA, R, W, 0,
             st);
        attention(Qb, Kb, Vb, LA, cfg.n_head, cfg.d_head, m.d_trunk_tiles, m.n_trunk_tiles, Ab,
                  LA, st, nullptr, nullptr, kp, vp);
        CUDA_CHECK(cudaStreamSynchronize(st));
      } else {
        KTimer kt(ctx, K_TRUNK_ATTN, st, 4.0 * m.trunk_pairs * W);
        attention(Qb, Kb, Vb, LA, cfg.n_head, cfg.d_head, m.d_trunk_tiles, m.n_trunk_tiles, Ab,
                  LA, st);
      }
      float* o = X[2];
      gemm(Ab, LA, W, nullptr, 0, 0, W_(S.blk(l, O_W)), dm, W_(S.blk(l, O_B)), o, LW, R, dm, 0, st);
      float* h1 = X[3];
      add_layernorm(xm, LW, o, LW, W_(S.blk(l, LN1_G)), W_(S.blk(l, LN1_B)), h1, LW, R, dm, st);
      gemm(h1, LW, dm, nullptr, 0, 0, W_(S.blk(l, FF_W1)), di, W_(S.blk(l, FF_B1)), F1, LI, R, di, 1,
           st);
      float* f2 = X[4];
      gemm(F1, LI, di, nullptr, 0, 0, W_(S.blk(l, FF_W2)), dm, W_(S.blk(l, FF_B2)), f2, LW, R, dm, 0,
           st);
      bool last = l == cfg.trf_layers - 1;
      float* xn = last ? hid : (x == X[0] ? X[5] : X[0]);
      int64_t ldn = last ? dm : LW;
      add_layernorm(h1, LW, f2, LW, W_(S.blk(l, LN2_G)), W_(S.blk(l, LN2_B)), xn, ldn, R, dm, st);
      x = xn;
      ldx = ldn;
    }
  }

  // ---- task heads (policy.py:187-217), full N x N attention per forward
  if (do_h) {
    GO_CHECK(hid && logits, "heads inputs/outputs required");
    const char* force = getenv("GO_ATTN");
    const bool use_tc = tc_attention_supported(cfg.d_head) && !(force && !strcmp(force, "simt"));
    float *tc_q = nullptr, *tc_k = nullptr, *tc_v = nullptr;
    int32_t* tc_scratch = nullptr;
    if (use_tc) {
      tc_q = A.take<float>((int64_t)cfg.n_head * R * 16);
      tc_k = A.take<float>((int64_t)cfg.n_head * m.n_tiles * 64 * 16);
      tc_v = A.take<float>((int64_t)cfg.n_head * m.n_tiles * 64 * 16);
      tc_scratch = A.take<int32_t>(tc_attention_scratch_ints(F, cfg.n_head, m.n_tc_works));
    }
    float* a_prev = nullptr;
    int64_t ld_prev = LW;
    float* rep_bufs[2] = {X[4], X[5]};
    int64_t lcol = 0;
    for (int t = 0; t < cfg.num_tasks; ++t) {
      bool zero_in = (a_prev == nullptr) || (b.ablate_mask >> t & 1);
      float* c = X[0];
      if (zero_in)  // [0 | hid] @ cat_w == hid @ cat_w[d:]
        gemm(hid, dm, dm, nullptr, 0, 0, W_(S.task(t, CAT_W)) + (int64_t)dm * dm, dm,
             W_(S.task(t, CAT_B)), c, LW, R, dm, 0, st);
      else
        gemm(a_prev, ld_prev, dm, hid, dm, dm, W_(S.task(t, CAT_W)), dm, W_(S.task(t, CAT_B)), c, LW,
             R, dm, 0, st);
      float* hh = X[1];
      add_layernorm(c, LW, nullptr, 0, W_(S.task(t, LN_G)), W_(S.task(t, LN_B)), hh, LW, R, dm, st);
      gemm(hh, LW, dm, nullptr, 0, 0, W_(S.ta(Q_W)), W, W_(S.ta(Q_B)), Qb, LA, R, W, 0, st);
      gemm(hh, LW, dm, nullptr, 0, 0, W_(S.ta(K_W)), W, W_(S.ta(K_B)), Kb, LA, R, W, 0, st);
      gemm(hh, LW, dm, nullptr, 0, 0, W_(S.ta(V_W)), W, W_(S.ta(V_B)), Vb, LA, R, W, 0, st);
      {
        KTimer kt(ctx, K_HEADS_ATTN, st, 4.0 * m.head_pairs * W);
        if (use_tc)
          attention_full_tc(Qb, Kb, Vb, LA, cfg.n_head, cfg.d_head, R, m.n_tiles, m.d_tc_works,
                            m.n_tc_works, m.d_tile_row0, m.d_tile_n, tc_q, tc_k, tc_v, Ab, LA,
                            row_fwd, F, tc_scratch, st);
        else
          attention(Qb, Kb, Vb, LA, cfg.n_head, cfg.d_head, m.d_head_tiles, m.n_head_tiles, Ab,
                    LA, st);
      }
      float* o = X[2];
      gemm(Ab, LA, W, nullptr, 0, 0, W_(S.ta(O_W)), dm, W_(S.ta(O_B)), o, LW, R, dm, 0, st);
      gemm(o, LW, dm, nullptr, 0, 0, W_(S.task(t, FC_W1)), di, W_(S.task(t, FC_B1)), F1, LI, R, di,
           1, st);
      float* rep = b.reps ? b.reps + (int64_t)t * R * dm : rep_bufs[t & 1];
      const int64_t ldr = b.reps ? dm : LW;
      gemm(F1, LI, di, nullptr, 0, 0, W_(S.task(t, FC_W2)), dm, W_(S.task(t, FC_B2)), rep, ldr, R,
           dm, 0, st);
      int a = cfg.task_sizes[t];
      gemm(rep, ldr, dm, nullptr, 0, 0, W_(S.task(t, OUT_W)), a, W_(S.task(t, OUT_B)), logits + lcol,
           a, R, a, 0, st);
      lcol += R * a;
      a_prev = rep;
      ld_prev = ldr;
    }
    if (value) {
      mean_rows(a_prev, ld_prev, m.d_row_off, F, m.d_chunks, m.n_chunks, dm, meanb, dm, part, st);
      value_head(meanb, F, dm, W_(S.value_w()), W_(S.value_b()), value, st);
    }
  }
}

// Tensor-core forward for 128-wide configs (the reference defaults): every dense layer
// is a tcgen05 3xTF32 GEMM with its bias/activation or residual+LayerNorm fused in
// the epilogue (tc_gemm.cu); Q/K/V are one merged GEMM; the trunk's modulation
// x*m is fused into the previous layer's LN2 epilogue.  Same math as run_forward.
static bool tc_forward_ok(const go_config_t& c, const go_batch_t& b) {
  const char* f = getenv("GO_GEMM");
  if (f && !strcmp(f, "simt")) return false;
  return c.gs_dim == 128 && c.d_model == 128 && c.n_head * c.d_head <= 144 && !b.features;
}

static void run_forward_tc(go_ctx* ctx, const go_config_t& cfg, const float* P,
                           const int64_t* off, const go_batch_t& b, float* node_embed,
                           float* graph_embed, float* hid, float* logits, float* value,
                           int32_t* status_dev, cudaStream_t st) {
  validate(cfg);
  const bool do_e = b.stage_mask & 1, do_t = b.stage_mask & 2, do_h = b.stage_mask & 4;
  BatchMeta m = make_meta(ctx, cfg, b, do_e, do_t, do_h, st);
  const int64_t R = m.R;
  const int F = m.F;
  Slots S = slots_of(cfg);
  auto W_ = [&](int slot) { return P + off[slot]; };
  const int gs = 128, dm = 128, H = cfg.n_head, dh = cfg.d_head, W = H * dh, di = cfg.d_inner;
  const int64_t LW = 128, LQ = 144, LA = ldp(W), LI = ldp(di);
  // workspace: activations + packed weights
  const int Lg = cfg.gs_layers, Lt = cfg.trf_layers, T = cfg.num_tasks;
  size_t pk = 0;
  pk += (size_t)Lg * (tc_gemm_packed_floats(gs, gs) + tc_gemm_packed_floats(2 * gs, gs));
  pk += tc_gemm_packed_floats(gs, dm);
  pk += (size_t)(Lt + 1) * (tc_gemm_packed_floats(dm, 3 * W) + tc_gemm_packed_floats(W, dm));
  pk += (size_t)Lt * (tc_gemm_packed_floats(dm, di) + tc_gemm_packed_floats(di, dm));
  for (int t = 0; t < T; ++t)
    pk += tc_gemm_packed_floats(2 * dm, dm) + tc_gemm_packed_floats(dm, dm) +
          tc_gemm_packed_floats(dm, di) + tc_gemm_packed_floats(di, dm) +
          tc_gemm_packed_floats(dm, cfg.task_sizes[t]);
  size_t bytes = forward_ws_bytes(cfg, R, m.gtotal, F, m.n_chunks) + (size_t)R * (LQ + 16) * 4 +
                 pk * 6 + (size_t)(Lt + 2) * 4 * 160 + (4u << 20) +
                 (b.cache_hook ? (size_t)Lt * R * (dm + LQ + 128) * 4 : 0);
  Arena A{reinterpret_cast<char*>(ctx->ensure(bytes)), 0, ctx->ws_bytes};
  float* X[6];
  for (int i = 0; i < 6; ++i) X[i] = A.take<float>(R * LW);
  float* QKV = A.take<float>(R * LQ);
  float* Ab = A.take<float>(R * LA);
  float* F1 = A.take<float>(R * LI);
  int32_t* row_fwd = A.take<int32_t>(R);
  GO_CHECK(m.gtotal + R < ((int64_t)1 << 31), "neighbour list exceeds 2^31 entries");
  int32_t* gidx = A.take<int32_t>(m.gtotal);
  int32_t* segoff = A.take<int32_t>(R + 1);
  float* mod = A.take<float>((int64_t)F * dm);
  float* meanb = A.take<float>((int64_t)F * dm);
  float* part = A.take<float>((m.n_chunks + 1) * 128);
  row_fwd_fill(m.d_row_off, F, R, row_fwd, st);
  // fused FFN for the 128 -> 512 -> 128 blocks of the trunk and the task heads
  // (tc_ffn.cuh; GO_FFN=0: two GEMMs each)
  const char* ffn_env = getenv("GO_FFN");
  const bool use_ffn = dm == 128 && di == 512 && !(ffn_env && ffn_env[0] == '0') &&
                       !(getenv("GO_GEMM_F16") && getenv("GO_GEMM_F16")[0] == '0');
  // every packed weight gets tf32 and fp16 copies and its own fp16 range flag
  constexpr int MAX_PACKS = 96;
  int32_t* ovf_flags = A.take<int32_t>(MAX_PACKS);
  CUDA_CHECK(cudaMemsetAsync(ovf_flags, 0, MAX_PACKS * sizeof(int32_t), st));
  int n_packs = 0;
  auto pack = [&](const float* w0, const float* w1, const float* w2, int Nsub, int64_t ldw, int K,
                  int N) {
    GO_CHECK(n_packs < MAX_PACKS, "too many packed weights");
    const int64_t nf = (int64_t)tc_gemm_packed_floats(K, N);
    float* out = A.take<float>(nf);
    void* out16 = A.take<float>((nf + 1) / 2);
    tc_gemm_pack(w0, w1, w2, Nsub, ldw, K, N, out, st);
    TcW w;
    w.w32 = out;
    w.w16 = out16;
    w.ovf = ovf_flags + n_packs++;
    tc_gemm_pack16(w0, w1, w2, Nsub, ldw, K, N, out16, st, w.ovf);
    return w;
  };
  auto pack1 = [&](const float* w, int K, int N) { return pack(w, nullptr, nullptr, N, N, K, N); };
  auto qkv_bias = [&](const float* bq, const float* bk, const float* bv) {
    float* bb = A.take<float>(160);
    CUDA_CHECK(cudaMemcpyAsync(bb, bq, W * 4, cudaMemcpyDeviceToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(bb + W, bk, W * 4, cudaMemcpyDeviceToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(bb + 2 * W, bv, W * 4, cudaMemcpyDeviceToDevice, st));
    return bb;
  };

  if (do_e) {
    GO_CHECK(node_embed && graph_embed, "embed outputs required");
    int32_t tcol[3] = {0, 0, 0};
    int c = 16;
    for (int t = 0; t < T; ++t) {
      tcol[t] = c;
      c += cfg.task_sizes[t];
    }
    neighbor_sample(m.d_views, m.d_row_off, m.d_gbase, m.d_seeds, F, R, row_fwd, cfg.gs_knn,
                    gidx, segoff, st);
    float* h = Lg == 0 ? node_embed : X[0];
    features_inproj(m.d_views, m.d_row_off, row_fwd, R, b.prev_actions, T, tcol, W_(S.e_in_w()),
                    W_(S.e_in_b()), gs, h, gs, st);
    for (int l = 0; l < Lg; ++l) {
      float* t = X[1];
      float* pooled = X[2];
      {
        KTimer kt(ctx, K_GEMM, st, 2.0 * R * gs * gs);
        // pre-activations: the sigmoid is applied to the pooled max instead (monotone)
        tc_gemm(h, gs, gs, nullptr, 0, 0, pack1(W_(S.e_layer(l, 0)), gs, gs), W_(S.e_layer(l, 1)),
                t, LW, R, gs, 0, st);
      }
      {
        double bytes = (double)(m.gtotal + R) * gs * 4 + (double)m.gtotal * 4 +
                       (double)(R + 1) * 8 + (double)R * 4;
        KTimer kt(ctx, K_SEGMAX, st, bytes);
        segment_max(t, LW, segoff, gidx, R, gs, pooled, LW, st, nullptr, true);
      }
      bool last = l == Lg - 1;
      float* hn = last ? node_embed : (h == X[0] ? X[3] : X[0]);
      {
        KTimer kt(ctx, K_GEMM, st, 2.0 * R * 2 * gs * gs);
        tc_gemm(h, gs, gs, pooled, LW, gs, pack1(W_(S.e_layer(l, 2)), 2 * gs, gs),
                W_(S.e_layer(l, 3)), hn, gs, R, gs, 1, st);
      }
      h = hn;
    }
    // non-finite check fused into the mean's pass over node_embed
    mean_rows(node_embed, gs, m.d_row_off, F, m.d_chunks, m.n_chunks, gs, graph_embed, gs, part,
              st, status_dev);
  }

  if (do_t) {
    GO_CHECK(!b.cache_hook || (F == 1 && cfg.segment_len <= 64),
             "the trunk cache hook needs one forward and segment_len <= 64");
    GO_CHECK(node_embed && graph_embed && hid, "trunk inputs/outputs required");
    const float* modp = b.mod_override;
    if (!modp) {
      int mb = Lt;
      BlockW bw{W_(S.blk(mb, V_W)),  W_(S.blk(mb, V_B)),  W_(S.blk(mb, O_W)),  W_(S.blk(mb, O_B)),
                W_(S.blk(mb, LN1_G)), W_(S.blk(mb, LN1_B)), W_(S.blk(mb, FF_W1)),
                W_(S.blk(mb, FF_B1)), W_(S.blk(mb, FF_W2)), W_(S.blk(mb, FF_B2)),
                W_(S.blk(mb, LN2_G)), W_(S.blk(mb, LN2_B))};
      modulate(graph_embed, gs, F, gs, W_(S.p_in_w()), W_(S.p_in_b()), bw, dm, W, di, mod, st);
      modp = mod;
    }
    float* x0 = Lt == 0 ? hid : X[0];
    // Warp-level MMA banded attention (trunk_mma.cu), with the SIMT kernel re-running a
    // layer whose operands left the fp16 range (gated on the layer's flag).  A tcgen05
    // version (2 CTAs/SM by TMEM, 0.61-0.66 ms per cfg4 forward vs 0.17 ms here) was
    // measured in round 1 and removed.  GO_TRUNK=simt forces the fp32 SIMT kernel
    // (A/B testing).
    const char* trunk_env = getenv("GO_TRUNK");
    const bool trunk_mma = trunk_mma_supported(dh) && !(trunk_env && !strcmp(trunk_env, "simt"));

    int32_t* trunk_flags = A.take<int32_t>(Lt + 1);
    {
      KTimer kt(ctx, K_GEMM, st, 2.0 * R * gs * dm);
      if (Lt > 0)  // xm = (node_embed @ in_w + b) * m(forward), modulation in the epilogue
        tc_gemm_scaled(node_embed, gs, gs, pack1(W_(S.p_in_w()), gs, dm), W_(S.p_in_b()),
                       nullptr, 0, modp, row_fwd, X[1], LW, R, dm, 0, st);
      else
        tc_gemm(node_embed, gs, gs, nullptr, 0, 0, pack1(W_(S.p_in_w()), gs, dm),
                W_(S.p_in_b()), x0, dm, R, dm, 0, st);
    }
    float* xm = X[1];
    for (int l = 0; l < Lt; ++l) {
      const float* bq = qkv_bias(W_(S.blk(l, Q_B)), W_(S.blk(l, K_B)), W_(S.blk(l, V_B)));
      const TcW wqkv = pack(W_(S.blk(l, Q_W)), W_(S.blk(l, K_W)), W_(S.blk(l, V_W)), W, W, dm, 3 * W);
      {
        KTimer kt(ctx, K_GEMM, st, 2.0 * R * dm * 3 * W);
        tc_gemm(xm, LW, dm, nullptr, 0, 0, wqkv, bq, QKV, LQ, R, 3 * W, 0, st);
      }
      if (b.cache_hook) {
        // cache_perturb (policy.py:170-172): the host hook rewrites the previous-segment
        // keys/values of every segment; their K/V projections go to QKVp and the SIMT
        // kernel reads rows before each tile's first query from there
        std::vector<float> hx((size_t)R * dm), hp;
        CUDA_CHECK(cudaMemcpy2DAsync(hx.data(), dm * 4, xm, LW * 4, dm * 4, R,
                                     cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        hp = hx;
        b.cache_hook(b.cache_hook_user, l, hx.data(), hp.data(), R, dm);
        float* pfx = A.take<float>(R * dm);
        float* qkvp = A.take<float>(R * LQ);
        CUDA_CHECK(cudaMemcpyAsync(pfx, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice, st));
        tc_gemm(pfx, dm, dm, nullptr, 0, 0, wqkv, bq, qkvp, LQ, R, 3 * W, 0, st);
        attention(QKV, QKV + W, QKV + 2 * W, LQ, H, dh, m.d_trunk_tiles, m.n_trunk_tiles, Ab, LA,
                  st, nullptr, nullptr, qkvp + W, qkvp + 2 * W);
        CUDA_CHECK(cudaStreamSynchronize(st));  // the host buffers above go out of scope
      } else {
        KTimer kt(ctx, K_TRUNK_ATTN, st, 4.0 * m.trunk_pairs * W);
        if (trunk_mma) {
          // split fp16 operands (3 MMAs per product): single fp16 Q/K/V put the trunk
          // output 1.03e-4 (normwise) from float64 at cfg3, where the random-init rows are
          // nearly parallel and the operand roundings do not average out
          trunk_attention_mma(QKV, QKV + W, QKV + 2 * W, LQ, H, dh, m.d_trunk_tiles,
                              m.n_trunk_tiles, Ab, LA, trunk_flags + l, st, nullptr, true);
          attention(QKV, QKV + W, QKV + 2 * W, LQ, H, dh, m.d_trunk_tiles, m.n_trunk_tiles, Ab,
                    LA, st, nullptr, trunk_flags + l);
        } else {
          attention(QKV, QKV + W, QKV + 2 * W, LQ, H, dh, m.d_trunk_tiles, m.n_trunk_tiles, Ab,
                    LA, st);
        }
      }
      float* h1 = X[2];
      {
        KTimer kt(ctx, K_GEMM, st, 2.0 * R * W * dm);
        tc_gemm_ln(Ab, LA, W, nullptr, 0, 0, pack1(W_(S.blk(l, O_W)), W, dm), W_(S.blk(l, O_B)), xm,
                   LW, W_(S.blk(l, LN1_G)), W_(S.blk(l, LN1_B)), h1, LW, nullptr, nullptr, nullptr,
                   0, R, dm, st);
      }
      bool last = l == Lt - 1;
      float* xm_next = (xm == X[1]) ? X[3] : X[1];
      if (use_ffn) {
        // fused FF1 -> relu -> FF2 -> +h1 -> LN (tc_ffn.cuh); the unfused tf32 GEMMs re-run
        // the layer only if an operand left the fp16 range (gated on fflag)
        KTimer kt(ctx, K_GEMM, st, 4.0 * R * dm * di);
        GO_CHECK(n_packs < MAX_PACKS, "too many packed weights");
        int32_t* fflag = ovf_flags + n_packs++;
        void* w1h = A.take<float>((int64_t)cdiv(di, 128) * cdiv(dm, 32) * 128 * 32);
        void* w2h = A.take<float>((int64_t)cdiv(dm, 128) * cdiv(di, 32) * 128 * 32);
        tc_gemm_pack16_bn(W_(S.blk(l, FF_W1)), di, dm, di, 128, w1h, st, fflag);
        tc_gemm_pack16_bn(W_(S.blk(l, FF_W2)), dm, di, dm, 128, w2h, st, fflag);
        tc_ffn(h1, LW, w1h, w2h, W_(S.blk(l, FF_B1)), W_(S.blk(l, FF_B2)), W_(S.blk(l, LN2_G)),
               W_(S.blk(l, LN2_B)), last ? hid : nullptr, dm, last ? nullptr : modp, row_fwd,
               last ? nullptr : xm_next, LW, R, fflag, st);
        TcW f1 = pack1(W_(S.blk(l, FF_W1)), dm, di), f2 = pack1(W_(S.blk(l, FF_W2)), di, dm);
        f1.gate = fflag;
        f2.gate = fflag;
        tc_gemm(h1, LW, dm, nullptr, 0, 0, f1, W_(S.blk(l, FF_B1)), F1, LI, R, di, 1, st);
        tc_gemm_ln(F1, LI, di, nullptr, 0, 0, f2, W_(S.blk(l, FF_B2)), h1, LW,
                   W_(S.blk(l, LN2_G)), W_(S.blk(l, LN2_B)), last ? hid : nullptr, dm,
                   last ? nullptr : modp, row_fwd, last ? nullptr : xm_next, LW, R, dm, st);
      } else {
        {
          KTimer kt(ctx, K_GEMM, st, 2.0 * R * dm * di);
          tc_gemm(h1, LW, dm, nullptr, 0, 0, pack1(W_(S.blk(l, FF_W1)), dm, di),
                  W_(S.blk(l, FF_B1)), F1, LI, R, di, 1, st);
        }
        KTimer kt(ctx, K_GEMM, st, 2.0 * R * di * dm);
        tc_gemm_ln(F1, LI, di, nullptr, 0, 0, pack1(W_(S.blk(l, FF_W2)), di, dm),
                   W_(S.blk(l, FF_B2)), h1, LW, W_(S.blk(l, LN2_G)), W_(S.blk(l, LN2_B)),
                   last ? hid : nullptr, dm, last ? nullptr : modp, row_fwd,
                   last ? nullptr : xm_next, LW, R, dm, st);
      }
      xm = xm_next;
    }
  }

  if (do_h) {
    GO_CHECK(hid && logits, "heads inputs/outputs required");
    const char* force = getenv("GO_ATTN");
    const bool use_tc = tc_attention_supported(dh) && !(force && !strcmp(force, "simt"));
    float *tc_q = nullptr, *tc_k = nullptr, *tc_v = nullptr;
    int32_t* tc_scratch = nullptr;
    if (use_tc) {
      tc_q = A.take<float>((int64_t)H * R * 16);
      tc_k = A.take<float>((int64_t)H * m.n_tiles * 64 * 16);
      tc_v = A.take<float>((int64_t)H * m.n_tiles * 64 * 16);
      tc_scratch = A.take<int32_t>(tc_attention_scratch_ints(F, H, m.n_tc_works));
    }
    const TcW ta_qkv = pack(W_(S.ta(Q_W)), W_(S.ta(K_W)), W_(S.ta(V_W)), W, W, dm, 3 * W);
    const float* ta_b = qkv_bias(W_(S.ta(Q_B)), W_(S.ta(K_B)), W_(S.ta(V_B)));
    const TcW ta_o = pack1(W_(S.ta(O_W)), W, dm);
    float* a_prev = nullptr;
    int64_t ld_prev = LW;
    float* rep_bufs[2] = {X[4], X[5]};
    int64_t lcol = 0;
    for (int t = 0; t < T; ++t) {
      bool zero_in = (a_prev == nullptr) || (b.ablate_mask >> t & 1);
      float* hh = X[1];
      {
        KTimer kt(ctx, K_GEMM, st, 2.0 * R * (zero_in ? 1 : 2) * dm * dm);
        if (zero_in)  // [0 | hid] @ cat_w == hid @ cat_w[d:]
          tc_gemm_ln(hid, dm, dm, nullptr, 0, 0, pack1(W_(S.task(t, CAT_W)) + (int64_t)dm * dm, dm, dm),
                     W_(S.task(t, CAT_B)), nullptr, 0, W_(S.task(t, LN_G)), W_(S.task(t, LN_B)), hh,
                     LW, nullptr, nullptr, nullptr, 0, R, dm, st);
        else
          tc_gemm_ln(a_prev, ld_prev, dm, hid, dm, dm, pack1(W_(S.task(t, CAT_W)), 2 * dm, dm),
                     W_(S.task(t, CAT_B)), nullptr, 0, W_(S.task(t, LN_G)), W_(S.task(t, LN_B)), hh,
                     LW, nullptr, nullptr, nullptr, 0, R, dm, st);
      }
      {
        KTimer kt(ctx, K_GEMM, st, 2.0 * R * dm * 3 * W);
        tc_gemm(hh, LW, dm, nullptr, 0, 0, ta_qkv, ta_b, QKV, LQ, R, 3 * W, 0, st);
      }
      {
        KTimer kt(ctx, K_HEADS_ATTN, st, 4.0 * m.head_pairs * W);
        if (use_tc)
          attention_full_tc(QKV, QKV + W, QKV + 2 * W, LQ, H, dh, R, m.n_tiles, m.d_tc_works,
                            m.n_tc_works, m.d_tile_row0, m.d_tile_n, tc_q, tc_k, tc_v, Ab, LA,
                            row_fwd, F, tc_scratch, st);
        else
          attention(QKV, QKV + W, QKV + 2 * W, LQ, H, dh, m.d_head_tiles, m.n_head_tiles, Ab, LA,
                    st);
      }
      float* o = X[2];
      float* rep = b.reps ? b.reps + (int64_t)t * R * dm : rep_bufs[t & 1];
      const int64_t ldr = b.reps ? dm : LW;
      int a = cfg.task_sizes[t];
      {
        KTimer kt(ctx, K_GEMM, st, 2.0 * R * W * dm);
        tc_gemm(Ab, LA, W, nullptr, 0, 0, ta_o, W_(S.ta(O_B)), o, LW, R, dm, 0, st);
      }
      if (use_ffn) {
        // rep = relu(o @ fc_w1 + b1) @ fc_w2 + b2 fused (tc_ffn.cuh, no LayerNorm); the
        // unfused tf32 GEMMs re-run only if an operand left the fp16 range
        KTimer kt(ctx, K_GEMM, st, 4.0 * R * dm * di);
        GO_CHECK(n_packs < MAX_PACKS, "too many packed weights");
        int32_t* fflag = ovf_flags + n_packs++;
        void* w1h = A.take<float>((int64_t)cdiv(di, 128) * cdiv(dm, 32) * 128 * 32);
        void* w2h = A.take<float>((int64_t)cdiv(dm, 128) * cdiv(di, 32) * 128 * 32);
        tc_gemm_pack16_bn(W_(S.task(t, FC_W1)), di, dm, di, 128, w1h, st, fflag);
        tc_gemm_pack16_bn(W_(S.task(t, FC_W2)), dm, di, dm, 128, w2h, st, fflag);
        tc_ffn(o, LW, w1h, w2h, W_(S.task(t, FC_B1)), W_(S.task(t, FC_B2)), nullptr, nullptr,
               rep, ldr, nullptr, nullptr, nullptr, 0, R, fflag, st, false);
        TcW f1 = pack1(W_(S.task(t, FC_W1)), dm, di), f2 = pack1(W_(S.task(t, FC_W2)), di, dm);
        f1.gate = fflag;
        f2.gate = fflag;
        tc_gemm(o, LW, dm, nullptr, 0, 0, f1, W_(S.task(t, FC_B1)), F1, LI, R, di, 1, st);
        tc_gemm(F1, LI, di, nullptr, 0, 0, f2, W_(S.task(t, FC_B2)), rep, ldr, R, dm, 0, st);
      } else {
        KTimer kt(ctx, K_GEMM, st, 4.0 * R * dm * di);
        tc_gemm(o, LW, dm, nullptr, 0, 0, pack1(W_(S.task(t, FC_W1)), dm, di), W_(S.task(t, FC_B1)),
                F1, LI, R, di, 1, st);
        tc_gemm(F1, LI, di, nullptr, 0, 0, pack1(W_(S.task(t, FC_W2)), di, dm), W_(S.task(t, FC_B2)),
                rep, ldr, R, dm, 0, st);
      }
      {
        KTimer kt(ctx, K_GEMM, st, 2.0 * R * dm * a);
        tc_gemm(rep, ldr, dm, nullptr, 0, 0, pack1(W_(S.task(t, OUT_W)), dm, a), W_(S.task(t, OUT_B)),
                logits + lcol, a, R, a, 0, st);
      }
      lcol += R * a;
      a_prev = rep;
      ld_prev = ldr;
    }
    if (value) {
      mean_rows(a_prev, ld_prev, m.d_row_off, F, m.d_chunks, m.n_chunks, dm, meanb, dm, part, st);
      value_head(meanb, F, dm, W_(S.value_w()), W_(S.value_b()), value, st);
    }
  }
}

extern "C" {

const char* go_last_error(void) { return g_last_error.c_str(); }
int go_version(void) { return 1; }

long long go_launch_count(void) { return go::g_launch_count.load(); }

int go_ctx_set_timing(go_ctx_t ctx, int enable) {
  return guarded([&] {
    ctx->resolve_timing();
    for (int i = 0; i < K_NUM_CLASSES; ++i) {
      ctx->stat_ms[i] = 0;
      ctx->stat_work[i] = 0;
      ctx->stat_count[i] = 0;
    }
    ctx->timing = enable != 0;
  });
}

int go_ctx_kernel_stats(go_ctx_t ctx, int32_t cls, int64_t* count, double* total_ms,
                        double* total_work) {
  return guarded([&] {
    GO_CHECK(cls >= 0 && cls < K_NUM_CLASSES, "bad kernel class");
    ctx->resolve_timing();
    *count = ctx->stat_count[cls];
    *total_ms = ctx->stat_ms[cls];
    *total_work = ctx->stat_work[cls];
  });
}

int go_ctx_create(int device, go_ctx_t* out) {
  return guarded([&] {
    int n = 0;
    CUDA_CHECK(cudaGetDeviceCount(&n));
    GO_CHECK(device >= 0 && device < n, "no CUDA device %d (found %d)", device, n);
    CUDA_CHECK(cudaSetDevice(device));
    auto* c = new go_ctx();
    c->device = device;
    CUDA_CHECK(cudaEventCreateWithFlags(&c->staged, cudaEventDisableTiming));
    *out = c;
  });
}

int go_ctx_destroy(go_ctx_t ctx) {
  return guarded([&] { delete ctx; });
}

int go_ctx_workspace_bytes(go_ctx_t ctx, int64_t* out) {
  return guarded([&] { *out = (int64_t)(ctx->ws_bytes + ctx->ws_small_bytes + ctx->des_ws_bytes); });
}

int go_param_count(const go_config_t* cfg, int32_t* num_slots_out) {
  return guarded([&] {
    validate(*cfg);
    *num_slots_out = slots_of(*cfg).count();
  });
}

int go_forward(go_ctx_t ctx, const go_config_t* cfg, const float* params,
               const int64_t* param_offsets, const go_batch_t* batch, float* node_embed,
               float* graph_embed, float* hid, float* logits, float* value, void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    if (tc_forward_ok(*cfg, *batch))
      run_forward_tc(ctx, *cfg, params, param_offsets, *batch, node_embed, graph_embed, hid,
                     logits, value, nullptr, (cudaStream_t)stream);
    else
      run_forward(ctx, *cfg, params, param_offsets, *batch, node_embed, graph_embed, hid, logits,
                  value, nullptr, (cudaStream_t)stream);
  });
}

// variant with a device status word (bit0: non-finite embeddings)
int go_forward_status(go_ctx_t ctx, const go_config_t* cfg, const float* params,
                      const int64_t* param_offsets, const go_batch_t* batch, float* node_embed,
                      float* graph_embed, float* hid, float* logits, float* value,
                      int32_t* status_dev, void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    if (tc_forward_ok(*cfg, *batch))
      run_forward_tc(ctx, *cfg, params, param_offsets, *batch, node_embed, graph_embed, hid,
                     logits, value, status_dev, (cudaStream_t)stream);
    else
      run_forward(ctx, *cfg, params, param_offsets, *batch, node_embed, graph_embed, hid, logits,
                  value, status_dev, (cudaStream_t)stream);
  });
}

int go_neighbor_arrays(go_ctx_t ctx, go_graph_t g, int64_t seed, int32_t k, int64_t* seg_off_out,
                       int32_t* gather_dev, void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    GO_CHECK(k >= 1, "k must be >= 1");
    GO_CHECK(seed >= 0, "seed must be non-negative");
    g->ensure_samp(k);
    std::vector<int64_t> so(g->n + 1, 0);
    for (int r = 0; r < g->n; ++r)
      so[r + 1] = so[r] + std::min<int64_t>(g->nbr_off[r + 1] - g->nbr_off[r], k);
    std::copy(so.begin(), so.end(), seg_off_out);
    if (!gather_dev) return;
    cudaStream_t st = (cudaStream_t)stream;
    go_config_t cfg{};
    cfg.gs_knn = k;
    go_graph_t gs[1] = {g};
    int64_t seeds[1] = {seed};
    go_batch_t b{};
    b.num_forwards = 1;
    b.graphs = gs;
    b.embed_seeds = seeds;
    BatchMeta m = make_meta(ctx, cfg, b, true, false, false, st);
    Arena A{reinterpret_cast<char*>(ctx->ensure((size_t)m.R * 4 + 4096)), 0, ctx->ws_bytes};
    int32_t* row_fwd = A.take<int32_t>(m.R);
    row_fwd_fill(m.d_row_off, 1, m.R, row_fwd, st);
    neighbor_sample(m.d_views, m.d_row_off, m.d_gbase, m.d_seeds, 1, m.R, row_fwd, k, gather_dev,
                    nullptr, st);
  });
}

int go_sample(go_ctx_t ctx, const go_config_t* cfg, int32_t num_forwards, const go_graph_t* graphs,
              const int64_t* row_counts, const uint64_t* pcg_states, const void* logits,
              int32_t logits_flags, double temperature, int32_t* actions_out, double* logp_out,
              void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    validate(*cfg);
    GO_CHECK(temperature >= 0.0, "temperature must be >= 0");
    GO_CHECK(pcg_states != nullptr, "generator states required");
    cudaStream_t st = (cudaStream_t)stream;
    go_batch_t b{};
    b.num_forwards = num_forwards;
    b.graphs = graphs;
    b.row_counts = row_counts;
    const void* dstate_v = nullptr;
    BatchMeta m = make_meta(ctx, *cfg, b, false, false, false, st, pcg_states,
                            (size_t)num_forwards * 32, &dstate_v);
    const uint64_t* dstate = reinterpret_cast<const uint64_t*>(dstate_v);
    Arena A{reinterpret_cast<char*>(ctx->ensure((size_t)m.R * 8 + 8192)), 0, ctx->ws_bytes};
    int32_t* row_fwd = A.take<int32_t>(m.R);
    int32_t* row_node = A.take<int32_t>(m.R);
    row_fwd_fill(m.d_row_off, m.F, m.R, row_fwd, st);
    row_node_fill(m.d_views, m.d_row_off, row_fwd, m.R, row_node, st);
    int64_t col = 0;
    const int T = cfg->num_tasks;
    const int logits_f64 = logits_flags & 1;
    const bool shared = (logits_flags & 2) != 0;  // all forwards read forward 0's block
    const int64_t lrows = shared ? m.row_off[1] - m.row_off[0] : m.R;
    GO_CHECK(!shared || [&] {
      for (int f = 1; f < m.F; ++f)
        if (m.row_off[f + 1] - m.row_off[f] != lrows) return false;
      return true;
    }(), "shared logits need forwards of equal row count");
    double bytes = 0;  // logits in, int32 action + float64 log-prob out, per row and task
    for (int t = 0; t < T; ++t)
      bytes += (double)m.R * ((logits_f64 ? 8.0 : 4.0) * cfg->task_sizes[t] + 12.0);
    KTimer kt(ctx, K_SAMPLE, st, bytes);
    for (int t = 0; t < T; ++t) {
      int a = cfg->task_sizes[t];
      const char* lp = reinterpret_cast<const char*>(logits) + col * (logits_f64 ? 8 : 4);
      sample_rows(lp, logits_f64, a, a, m.R, m.d_row_off, row_fwd, row_node, dstate, t,
                  temperature, actions_out + (int64_t)t * m.R, logp_out + (int64_t)t * m.R, st,
                  shared);
      col += lrows * a;
    }
  });
}

int go_simulate(go_ctx_t ctx, go_graph_t g, int32_t K, const int32_t* placement,
                const int32_t* priorities, int32_t prio_per_placement, int32_t d,
                const double* peak, const double* mem_bw, const double* cap,
                const double* link_bw, int32_t policy, double baseline, double* step_time,
                uint8_t* valid, int8_t* violation, double* busy, double* peak_mem, double* reward,
                void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    GO_CHECK(policy == 0 || policy == 1, "unknown policy");
    GO_CHECK(d >= 1, "need at least one device");
    cudaStream_t st = (cudaStream_t)stream;
    if (!g->acyclic) {
      // simulator.py:317-319: cycle_after_fusion -> (0, invalid, zeros)
      std::vector<double> z((size_t)K * d, 0.0), zk(K, 0.0), rk(K, -10.0);
      std::vector<uint8_t> v(K, 0);
      std::vector<int8_t> vi(K, 3);
      CUDA_CHECK(cudaMemcpyAsync(step_time, zk.data(), K * 8, cudaMemcpyHostToDevice, st));
      CUDA_CHECK(cudaMemcpyAsync(valid, v.data(), K, cudaMemcpyHostToDevice, st));
      CUDA_CHECK(cudaMemcpyAsync(violation, vi.data(), K, cudaMemcpyHostToDevice, st));
      if (busy) CUDA_CHECK(cudaMemcpyAsync(busy, z.data(), z.size() * 8, cudaMemcpyHostToDevice, st));
      if (peak_mem)
        CUDA_CHECK(cudaMemcpyAsync(peak_mem, z.data(), z.size() * 8, cudaMemcpyHostToDevice, st));
      if (reward && baseline > 0)
        CUDA_CHECK(cudaMemcpyAsync(reward, rk.data(), K * 8, cudaMemcpyHostToDevice, st));
      CUDA_CHECK(cudaStreamSynchronize(st));
      return;
    }
    KTimer kt(ctx, K_DES, st, (double)K * g->n);
    simulate_batch(g->des, K, placement, g->n, priorities, prio_per_placement ? g->n : 0, d, peak,
                   mem_bw, cap, link_bw, policy, baseline, step_time, valid, violation, busy,
                   peak_mem, reward, ctx, st);
  });
}

int go_simulate_trace(go_ctx_t ctx, go_graph_t g, const int32_t* placement,
                      const int32_t* priorities, int32_t d, const double* peak,
                      const double* mem_bw, const double* cap, const double* link_bw,
                      int32_t policy, double* step_time, uint8_t* valid, int8_t* violation,
                      double* busy, double* peak_mem, go_trace_event_t* trace,
                      int64_t trace_capacity, int64_t* trace_count, void* stream) {
  return guarded([&] {
    static_assert(sizeof(go_trace_event_t) == sizeof(DesTraceRec), "trace record layout");
    CUDA_CHECK(cudaSetDevice(ctx->device));
    GO_CHECK(policy == 0 || policy == 1, "unknown policy");
    GO_CHECK(d >= 1, "need at least one device");
    GO_CHECK(trace && trace_count && trace_capacity >= 0, "trace buffers required");
    cudaStream_t st = (cudaStream_t)stream;
    if (!g->acyclic) {  // simulator.py:317-319: no events, (0, invalid, zeros)
      std::vector<double> z((size_t)d, 0.0), zk(1, 0.0);
      uint8_t v = 0;
      int8_t vi = 3;
      int64_t zero = 0;
      CUDA_CHECK(cudaMemcpyAsync(step_time, zk.data(), 8, cudaMemcpyHostToDevice, st));
      CUDA_CHECK(cudaMemcpyAsync(valid, &v, 1, cudaMemcpyHostToDevice, st));
      CUDA_CHECK(cudaMemcpyAsync(violation, &vi, 1, cudaMemcpyHostToDevice, st));
      CUDA_CHECK(cudaMemcpyAsync(busy, z.data(), z.size() * 8, cudaMemcpyHostToDevice, st));
      CUDA_CHECK(cudaMemcpyAsync(peak_mem, z.data(), z.size() * 8, cudaMemcpyHostToDevice, st));
      CUDA_CHECK(cudaMemcpyAsync(trace_count, &zero, 8, cudaMemcpyHostToDevice, st));
      CUDA_CHECK(cudaStreamSynchronize(st));
      return;
    }
    simulate_batch(g->des, 1, placement, g->n, priorities, 0, d, peak, mem_bw, cap, link_bw,
                   policy, 0.0, step_time, valid, violation, busy, peak_mem, nullptr, ctx, st,
                   reinterpret_cast<DesTraceRec*>(trace), trace_capacity, trace_count);
  });
}

int go_anneal(go_ctx_t ctx, go_graph_t g, int32_t chains, const uint64_t* rng_words,
              int32_t* state, int32_t* best, int32_t d, const double* peak, const double* mem_bw,
              const double* cap, const double* link_bw, int32_t policy, int32_t iterations,
              int32_t moves_per_step, double initial_temperature, double cooling_rate,
              int32_t num_tasks, const int32_t* task_slots, const int32_t* task_sizes,
              double* best_time, void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    GO_CHECK(policy == 0 || policy == 1, "unknown policy");
    GO_CHECK(iterations >= 1, "iterations must be >= 1");
    GO_CHECK(cooling_rate > 0.0 && cooling_rate < 1.0, "cooling_rate must be in (0,1)");
    GO_CHECK(g->acyclic, "the annealed grouping has a cycle");
    GO_CHECK(num_tasks >= 1 && num_tasks <= 2, "1 or 2 annealed tasks");
    int slots[2] = {0, 0}, sizes[2] = {1, 1};
    for (int t = 0; t < num_tasks; ++t) {
      GO_CHECK(task_slots[t] == 0 || task_slots[t] == 1, "task slot must be 0 or 1");
      GO_CHECK(task_sizes[t] >= 1, "empty action space");
      slots[t] = task_slots[t];
      sizes[t] = task_sizes[t];
    }
    GO_CHECK(g->n >= 1, "empty graph");
    anneal_chains(g->des, chains, rng_words, state, best, d, peak, mem_bw, cap, link_bw, policy,
                  iterations, moves_per_step, initial_temperature, cooling_rate, num_tasks, slots,
                  sizes, best_time, ctx, (cudaStream_t)stream);
  });
}

}  // extern "C"

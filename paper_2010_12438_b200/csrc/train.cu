// PPO loss + gradient on device (training.py:146-233): a training forward that keeps
// every intermediate the backward needs, the clipped-surrogate / entropy / value loss
// with dL/dlogits, and the reverse sweep through heads, trunk, modulation and the
// GraphSAGE embedding, accumulating parameter gradients into a float32 blob with the
// parameter layout.  One call handles a whole minibatch as a ragged batch.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "train.cuh"

namespace go {

// parameter slot helpers (must match engine.cu / params.py)
namespace {
struct S2 {
  int gl, tl, T;
  int e_in_w() const { return 0; }
  int e_in_b() const { return 1; }
  int e_layer(int l, int w) const { return 2 + 4 * l + w; }
  int pbase() const { return 2 + 4 * gl; }
  int blk(int b, int w) const { return pbase() + 2 + 16 * b + w; }
  int ta(int w) const { return pbase() + 2 + 16 * (tl + 1) + w; }
  int task(int t, int w) const { return ta(8) + 10 * t + w; }
  int value_w() const { return ta(8) + 10 * T; }
};
enum { Q_W = 0, Q_B, K_W, K_B, V_W, V_B, O_W, O_B, LN1_G, LN1_B, FF_W1, FF_B1, FF_W2, FF_B2,
       LN2_G, LN2_B };
enum { CAT_W = 0, CAT_B, LN_G, LN_B, FC_W1, FC_B1, FC_W2, FC_B2, OUT_W, OUT_B };

struct Arena2 {
  char* base;
  size_t off = 0, cap;
  template <class T>
  T* take(int64_t count) {
    size_t bytes = round_up(std::max<int64_t>(count, 1) * (int64_t)sizeof(T), 256);
    GO_CHECK(off + bytes <= cap, "training workspace overflow");
    T* p = reinterpret_cast<T*>(base + off);
    off += bytes;
    return p;
  }
};

void build_kv_tiles(const std::vector<int64_t>& row_off, int64_t S, bool banded,
                    std::vector<KvTile>& out) {
  const int64_t KTL = 64;
  for (size_t f = 0; f + 1 < row_off.size(); ++f) {
    int64_t f0 = row_off[f], f1 = row_off[f + 1];
    if (!banded) {
      for (int64_t k = f0; k < f1; k += KTL) out.push_back({k, std::min(k + KTL, f1), f0, f1, 0, 0});
      continue;
    }
    for (int64_t s0 = f0; s0 < f1; s0 += S) {
      int64_t s1 = std::min(s0 + S, f1);
      int64_t n0 = s1, n1 = std::min(s1 + S, f1);  // next segment (attends to us via its cache)
      for (int64_t k = s0; k < s1; k += KTL)
        out.push_back({k, std::min(k + KTL, s1), s0, s1, n0, n1});
    }
  }
}

void build_q_tiles(const std::vector<int64_t>& row_off, int64_t S, bool banded,
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
}  // namespace

void run_ppo_grad(go_ctx* ctx, const go_config_t& cfg, const float* P, const int64_t* off,
                  const go_batch_t& b, const int32_t* actions, const double* old_logp,
                  const double* fparams_host, double clip_eps, double ent_coef, double value_coef,
                  int32_t denom, float* G, double* stats_host, cudaStream_t st) {
  const int F = b.num_forwards;
  const int C = denom > 0 ? denom : F;  // minibatch size the loss is averaged over
  GO_CHECK(F >= 1 && b.graphs, "ppo_grad needs graph handles");
  const int T = cfg.num_tasks;
  const int gs = cfg.gs_dim, dm = cfg.d_model, H = cfg.n_head, dh = cfg.d_head;
  const int W = H * dh, di = cfg.d_inner, Lg = cfg.gs_layers, Lt = cfg.trf_layers;
  S2 S{Lg, Lt, T};
  auto Pw = [&](int slot) { return P + off[slot]; };
  auto Gw = [&](int slot) { return G + off[slot]; };

  // ---- metadata (row offsets, graph views, per-forward scalars, attention tiles)
  go_batch_t bb = b;
  std::vector<int64_t> row_off(F + 1, 0);
  for (int f = 0; f < F; ++f) row_off[f + 1] = row_off[f] + b.graphs[f]->n;
  std::vector<AttnTile> tq, hq;
  std::vector<KvTile> tk, hk;
  build_q_tiles(row_off, cfg.segment_len, true, tq);
  build_q_tiles(row_off, 0, false, hq);
  build_kv_tiles(row_off, cfg.segment_len, true, tk);
  build_kv_tiles(row_off, 0, false, hk);
  // tcgen05 tape head attention (tc_tape.cu): 384-query work items and 64-row tiles
  std::vector<TcWork> tcw;
  std::vector<int64_t> trow0;
  std::vector<int32_t> tn;
  tc_build_tables(row_off, tcw, trow0, tn);
  std::vector<TcWork> qw;   // (forward, 256 queries) items of the tcgen05 dq kernel
  for (size_t i = 0; i < tcw.size(); ++i)
    if (tcw[i].q0 == 0)
      for (int32_t q0 = 0; q0 < tcw[i].n; q0 += 256) {
        TcWork x = tcw[i];
        x.q0 = q0;
        qw.push_back(x);
      }
  std::vector<TcWork> kvw;  // (forward, 128 keys) items of the tcgen05 dk / dv kernel
  for (size_t i = 0; i < tcw.size(); ++i)
    if (tcw[i].q0 == 0)
      for (int32_t k0 = 0; k0 < tcw[i].n; k0 += 128) {
        TcWork x = tcw[i];
        x.q0 = k0;
        kvw.push_back(x);
      }
  std::vector<char> extra;
  auto put = [&](const void* p, size_t n) {
    size_t o = round_up((int64_t)extra.size(), 256);
    extra.resize(o + n);
    if (n) std::memcpy(extra.data() + o, p, n);
    return o;
  };
  size_t o_fp = put(fparams_host, (size_t)F * 4 * 8);
  size_t o_tq = put(tq.data(), tq.size() * sizeof(AttnTile));
  size_t o_hq = put(hq.data(), hq.size() * sizeof(AttnTile));
  size_t o_tk = put(tk.data(), tk.size() * sizeof(KvTile));
  size_t o_hk = put(hk.data(), hk.size() * sizeof(KvTile));
  size_t o_tcw = put(tcw.data(), tcw.size() * sizeof(TcWork));
  size_t o_tr0 = put(trow0.data(), trow0.size() * sizeof(int64_t));
  size_t o_tn = put(tn.data(), tn.size() * sizeof(int32_t));
  size_t o_kvw = put(kvw.data(), kvw.size() * sizeof(TcWork));
  size_t o_qw = put(qw.data(), qw.size() * sizeof(TcWork));
  const void* exd = nullptr;
  BatchMeta m = make_meta(ctx, cfg, bb, true, false, false, st, extra.data(), extra.size(), &exd);
  const char* ex = reinterpret_cast<const char*>(exd);
  const double* d_fp = reinterpret_cast<const double*>(ex + o_fp);
  const AttnTile* d_tq = reinterpret_cast<const AttnTile*>(ex + o_tq);
  const AttnTile* d_hq = reinterpret_cast<const AttnTile*>(ex + o_hq);
  const KvTile* d_tk = reinterpret_cast<const KvTile*>(ex + o_tk);
  const KvTile* d_hk = reinterpret_cast<const KvTile*>(ex + o_hk);
  const TcWork* d_tcw = reinterpret_cast<const TcWork*>(ex + o_tcw);
  const int64_t* d_tr0 = reinterpret_cast<const int64_t*>(ex + o_tr0);
  const int32_t* d_tn = reinterpret_cast<const int32_t*>(ex + o_tn);
  const int64_t Ttot = (int64_t)trow0.size();
  const TcWork* d_kvw = reinterpret_cast<const TcWork*>(ex + o_kvw);
  const TcWork* d_qw = reinterpret_cast<const TcWork*>(ex + o_qw);
  const int64_t R = m.R;

  // ---- workspace
  size_t per_row = (size_t)(Lg + 1) * gs + (size_t)Lg * gs * 3 +
                   (size_t)Lt * (dm * 6 + W * 4 + H + di) + (size_t)dm +
                   (size_t)T * (dm * 4 + W * 4 + H + di) + 64 +
                   /* backward scratch */ (size_t)(8 * std::max(gs, dm) + 8 * W + 2 * di + 2 * H);
  size_t bytes = (size_t)R * per_row * 4 + (size_t)R * 16 + (size_t)m.gtotal * 4 +
                 (size_t)F * (4 * dm + 2 * gs + 64) * 8 + (size_t)(m.n_chunks + 4) * 512 * 4 +
                 (size_t)R * T * 64 + (8u << 20) + attention_backward_mma_scratch(R, H) +
                 /* backward dX scratch */ (size_t)R * std::max(dm, gs) * 4 +
                 /* packed tape weights (forward + transposed backward) */ 2 * (size_t)(2 * Lg + 6 * Lt + 8 * T + 4) *
                     (size_t)tc_gemm_packed_floats(std::max(2 * gs, di), std::max(dm, di)) * 6 + (16u << 20) +
                 tape_attention_tc_scratch(R, F, H);
  Arena2 A{reinterpret_cast<char*>(ctx->ensure(bytes)), 0, ctx->ws_bytes};
  int32_t* row_fwd = A.take<int32_t>(R);
  int32_t* row_node = A.take<int32_t>(R);
  GO_CHECK(m.gtotal + R < ((int64_t)1 << 31), "neighbour list exceeds 2^31 entries");
  int32_t* gidx = A.take<int32_t>(m.gtotal);
  int32_t* segoff = A.take<int32_t>(R + 1);
  // attention on mma.sync tensor cores (split-fp16 operands, three MMAs per product:
  // fp32-class results) with a gated fp32 SIMT re-run on range overflow;
  // GO_TRAIN_ATTN=simt keeps the fp32 SIMT kernels only (the tests' comparison path)
  const char* ta_env = getenv("GO_TRAIN_ATTN");
  const bool attn_mma = trunk_mma_supported(dh) && !(ta_env && !strcmp(ta_env, "simt"));
  int32_t* aflag = A.take<int32_t>(64);
  void* abw = A.take<char>((int64_t)attention_backward_mma_scratch(R, H));
  // the N x N head attention's tape forward on tcgen05 (split fp16, tc_tape.cu) unless
  // GO_TRAIN_ATTN selects another variant; falls back to the mma.sync forward when a score
  // bound exceeds the fp16 limit
  const bool tape_tc = attn_mma && dh <= 15 && !(ta_env && !strcmp(ta_env, "mma"));
  void* tape_ws = A.take<char>((int64_t)tape_attention_tc_scratch(R, F, H));
  auto attn_fwd = [&](const float* q, const float* k, const float* v, const AttnTile* tiles,
                      int64_t nt, float* out, float* lse, const int32_t* gate = nullptr) {
    if (attn_mma) {
      if (dh <= 15)
        attention_forward_mma(q, k, v, W, H, dh, tiles, nt, R, out, W, lse, abw, aflag, st,
                              gate);
      else
        trunk_attention_mma(q, k, v, W, H, dh, tiles, nt, out, W, aflag, st, lse, true);
      attention(q, k, v, W, H, dh, tiles, nt, out, W, st, lse, aflag);
    } else {
      attention(q, k, v, W, H, dh, tiles, nt, out, W, st, lse);
    }
  };
  // tape forward GEMMs on the tcgen05 split-precision GEMM (tc_gemm: fp16 3-pass with
  // the tf32 re-run on range overflow, as the inference forward); operands whose rows are
  // not 16-B aligned (the attention output, ld = H*d_head) stay on the fp32 SIMT GEMM.
  // GO_TRAIN_GEMM=simt keeps every tape GEMM on SIMT.
  const char* tg_env = getenv("GO_TRAIN_GEMM");
  const bool tc_fwd = !(tg_env && !strcmp(tg_env, "simt"));
  auto fgemm = [&](const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
                   const float* Wt, int64_t ldw, const float* bias, float* C, int64_t ldc,
                   int64_t M, int N, int act, cudaStream_t s_) {
    const auto al = [](const float* p, int64_t ld) {
      return p == nullptr || ((uintptr_t)p % 16 == 0 && ld % 4 == 0);
    };
    const bool ok = tc_fwd && al(A1, lda1) && al(A2, lda2) && (A2 == nullptr || K1 % 32 == 0);
    if (!ok) {
      gemm(A1, lda1, K1, A2, lda2, K2, Wt, ldw, bias, C, ldc, M, N, act, s_);
      return;
    }
    const int K = K1 + (A2 ? K2 : 0);
    const int64_t nf = (int64_t)tc_gemm_packed_floats(K, N);
    TcW w;
    float* w32 = A.take<float>(nf);
    void* w16 = A.take<float>((nf + 1) / 2);
    int32_t* ovf = A.take<int32_t>(1);
    CUDA_CHECK(cudaMemsetAsync(ovf, 0, sizeof(int32_t), s_));
    tc_gemm_pack(Wt, nullptr, nullptr, N, ldw, K, N, w32, s_);
    tc_gemm_pack16(Wt, nullptr, nullptr, N, ldw, K, N, w16, s_, ovf);
    w.w32 = w32;
    w.w16 = w16;
    w.ovf = ovf;
    tc_gemm(A1, lda1, K1, A2, lda2, K2, w, bias, C, ldc, M, N, act, s_);
  };
  // backward dX = dY W^T on the tcgen05 tf32 3-pass GEMM (fp32-class; gradients keep
  // fp32's exponent range, so no fp16 pass) for 16-B-aligned dY rows; accumulating calls
  // go through a scratch tile and an add.  Others stay on the SIMT dgemm_nt.
  float* dtmp = nullptr;
  const int tmp_cols = std::max(dm, gs);
  auto dgemm = [&](const float* dY, int64_t ldd, const float* Wt, int64_t ldw, float* dX,
                   int64_t ldx, int64_t M, int Kin, int Nout, bool accumulate) {
    const bool ok = tc_fwd && (uintptr_t)dY % 16 == 0 && ldd % 4 == 0 &&
                    (!accumulate || Kin <= tmp_cols);
    if (!ok) {
      dgemm_nt(dY, ldd, Wt, ldw, dX, ldx, M, Kin, Nout, accumulate, st);
      return;
    }
    float* wt = A.take<float>((int64_t)Nout * Kin);
    transpose(Wt, ldw, Kin, Nout, wt, st);
    TcW w;
    float* w32 = A.take<float>((int64_t)tc_gemm_packed_floats(Nout, Kin));
    tc_gemm_pack(wt, nullptr, nullptr, Kin, Kin, Nout, Kin, w32, st);
    w.w32 = w32;
    if (!accumulate) {
      tc_gemm(dY, ldd, Nout, nullptr, 0, 0, w, nullptr, dX, ldx, M, Kin, 0, st);
    } else {
      if (!dtmp) dtmp = A.take<float>(M * tmp_cols);
      tc_gemm(dY, ldd, Nout, nullptr, 0, 0, w, nullptr, dtmp, Kin, M, Kin, 0, st);
      add_into(dX, ldx, dtmp, Kin, M, Kin, st);
    }
  };
  auto attn_bwd = [&](const float* q, const float* k, const float* v, const float* O,
                      const float* dO_, const float* lse, const AttnTile* qt, int64_t nq,
                      const KvTile* kt, int64_t nk, float* Db, float* dq_, float* dk_a,
                      float* dv_a, float* dk_b, float* dv_b, const int32_t* gate = nullptr) {
    if (attn_mma)
      attention_backward_mma(q, k, v, O, dO_, W, lse, H, dh, qt, nq, kt, nk, Db, R, dq_, dk_a,
                             dv_a, dk_b, dv_b, abw, aflag, st, gate);
    else
      attention_backward(q, k, v, O, dO_, W, lse, H, dh, qt, nq, kt, nk, Db, R, dq_, dk_a, dv_a,
                         dk_b, dv_b, st);
  };
  row_fwd_fill(m.d_row_off, F, R, row_fwd, st);
  row_node_fill(m.d_views, m.d_row_off, row_fwd, R, row_node, st);

  // ================================================================ forward (tape)
  std::vector<float*> eh(Lg + 1), et(Lg), ep(Lg);
  std::vector<int32_t*> ea(Lg);
  for (int l = 0; l <= Lg; ++l) eh[l] = A.take<float>(R * gs);
  for (int l = 0; l < Lg; ++l) {
    et[l] = A.take<float>(R * gs);
    ep[l] = A.take<float>(R * gs);
    ea[l] = A.take<int32_t>(R * gs);
  }
  float* ge = A.take<float>((int64_t)F * gs);
  float* part = A.take<float>((m.n_chunks + 4) * std::max(gs, dm));
  int32_t tcol[3] = {0, 0, 0};
  {
    int c = 16;
    for (int t = 0; t < T; ++t) {
      tcol[t] = c;
      c += cfg.task_sizes[t];
    }
  }
  const int Fdim = 16 + [&] { int s = 0; for (int t = 0; t < T; ++t) s += cfg.task_sizes[t]; return s; }();
  neighbor_sample(m.d_views, m.d_row_off, m.d_gbase, m.d_seeds, F, R, row_fwd, cfg.gs_knn, gidx, segoff, st);
  features_inproj(m.d_views, m.d_row_off, row_fwd, R, b.prev_actions, T, tcol, Pw(S.e_in_w()),
                  Pw(S.e_in_b()), gs, eh[0], gs, st);
  for (int l = 0; l < Lg; ++l) {
    fgemm(eh[l], gs, gs, nullptr, 0, 0, Pw(S.e_layer(l, 0)), gs, Pw(S.e_layer(l, 1)), et[l], gs, R,
         gs, 2, st);
    segment_max(et[l], gs, segoff, gidx, R, gs, ep[l], gs, st,
                ea[l]);
    fgemm(eh[l], gs, gs, ep[l], gs, gs, Pw(S.e_layer(l, 2)), gs, Pw(S.e_layer(l, 3)), eh[l + 1], gs,
         R, gs, 1, st);
  }
  mean_rows(eh[Lg], gs, m.d_row_off, F, m.d_chunks, m.n_chunks, gs, ge, gs, part, st);
  const float* node_embed = eh[Lg];
  // modulation
  float* mod = A.take<float>((int64_t)F * dm);
  const int mb = Lt;
  BlockW bw{Pw(S.blk(mb, V_W)),  Pw(S.blk(mb, V_B)),  Pw(S.blk(mb, O_W)),  Pw(S.blk(mb, O_B)),
            Pw(S.blk(mb, LN1_G)), Pw(S.blk(mb, LN1_B)), Pw(S.blk(mb, FF_W1)), Pw(S.blk(mb, FF_B1)),
            Pw(S.blk(mb, FF_W2)), Pw(S.blk(mb, FF_B2)), Pw(S.blk(mb, LN2_G)), Pw(S.blk(mb, LN2_B))};
  modulate(ge, gs, F, gs, Pw(S.pbase()), Pw(S.pbase() + 1), bw, dm, W, di, mod, st);
  // trunk
  std::vector<float*> tx(Lt + 1), txm(Lt), tqv(Lt), tkv(Lt), tvv(Lt), tat(Lt), tls(Lt), tu1(Lt),
      th1(Lt), tf1(Lt), tu2(Lt);
  for (int l = 0; l <= Lt; ++l) tx[l] = A.take<float>(R * dm);
  for (int l = 0; l < Lt; ++l) {
    txm[l] = A.take<float>(R * dm);
    tqv[l] = A.take<float>(R * W);
    tkv[l] = A.take<float>(R * W);
    tvv[l] = A.take<float>(R * W);
    tat[l] = A.take<float>(R * W);
    tls[l] = A.take<float>(R * H);
    tu1[l] = A.take<float>(R * dm);
    th1[l] = A.take<float>(R * dm);
    tf1[l] = A.take<float>(R * di);
    tu2[l] = A.take<float>(R * dm);
  }
  fgemm(node_embed, gs, gs, nullptr, 0, 0, Pw(S.pbase()), dm, Pw(S.pbase() + 1), tx[0], dm, R, dm, 0,
       st);
  for (int l = 0; l < Lt; ++l) {
    mul_rowvec(tx[l], dm, mod, dm, row_fwd, txm[l], dm, R, dm, st);
    fgemm(txm[l], dm, dm, nullptr, 0, 0, Pw(S.blk(l, Q_W)), W, Pw(S.blk(l, Q_B)), tqv[l], W, R, W, 0, st);
    fgemm(txm[l], dm, dm, nullptr, 0, 0, Pw(S.blk(l, K_W)), W, Pw(S.blk(l, K_B)), tkv[l], W, R, W, 0, st);
    fgemm(txm[l], dm, dm, nullptr, 0, 0, Pw(S.blk(l, V_W)), W, Pw(S.blk(l, V_B)), tvv[l], W, R, W, 0, st);
    attn_fwd(tqv[l], tkv[l], tvv[l], d_tq, (int64_t)tq.size(), tat[l], tls[l]);
    fgemm(tat[l], W, W, nullptr, 0, 0, Pw(S.blk(l, O_W)), dm, Pw(S.blk(l, O_B)), tu1[l], dm, R, dm, 0, st);
    add_into(tu1[l], dm, txm[l], dm, R, dm, st);  // u1 = xm + o  (kept for LN1 backward)
    add_layernorm(tu1[l], dm, nullptr, 0, Pw(S.blk(l, LN1_G)), Pw(S.blk(l, LN1_B)), th1[l], dm, R, dm, st);
    fgemm(th1[l], dm, dm, nullptr, 0, 0, Pw(S.blk(l, FF_W1)), di, Pw(S.blk(l, FF_B1)), tf1[l], di, R,
         di, 1, st);
    fgemm(tf1[l], di, di, nullptr, 0, 0, Pw(S.blk(l, FF_W2)), dm, Pw(S.blk(l, FF_B2)), tu2[l], dm, R,
         dm, 0, st);
    add_into(tu2[l], dm, th1[l], dm, R, dm, st);  // u2 = h1 + ff
    add_layernorm(tu2[l], dm, nullptr, 0, Pw(S.blk(l, LN2_G)), Pw(S.blk(l, LN2_B)), tx[l + 1], dm, R,
                  dm, st);
  }
  const float* hid = tx[Lt];
  // heads
  std::vector<float*> hc(T), hh(T), hqv(T), hkv(T), hvv(T), hat(T), hls(T), ho(T), hf1(T), hrep(T),
      hlog(T);
  for (int t = 0; t < T; ++t) {
    hc[t] = A.take<float>(R * dm);
    hh[t] = A.take<float>(R * dm);
    hqv[t] = A.take<float>(R * W);
    hkv[t] = A.take<float>(R * W);
    hvv[t] = A.take<float>(R * W);
    hat[t] = A.take<float>(R * W);
    hls[t] = A.take<float>(R * H);
    ho[t] = A.take<float>(R * dm);
    hf1[t] = A.take<float>(R * di);
    hrep[t] = A.take<float>(R * dm);
    hlog[t] = A.take<float>(R * cfg.task_sizes[t]);
  }
  float* meanrep = A.take<float>((int64_t)F * dm);
  float* value = A.take<float>(F);
  std::vector<bool> zero_in(T);
  for (int t = 0; t < T; ++t) {
    zero_in[t] = (t == 0) || (b.ablate_mask >> t & 1);
    if (zero_in[t])
      fgemm(hid, dm, dm, nullptr, 0, 0, Pw(S.task(t, CAT_W)) + (int64_t)dm * dm, dm, Pw(S.task(t, CAT_B)),
           hc[t], dm, R, dm, 0, st);
    else
      fgemm(hrep[t - 1], dm, dm, hid, dm, dm, Pw(S.task(t, CAT_W)), dm, Pw(S.task(t, CAT_B)), hc[t], dm, R,
           dm, 0, st);
    add_layernorm(hc[t], dm, nullptr, 0, Pw(S.task(t, LN_G)), Pw(S.task(t, LN_B)), hh[t], dm, R, dm, st);
    fgemm(hh[t], dm, dm, nullptr, 0, 0, Pw(S.ta(Q_W)), W, Pw(S.ta(Q_B)), hqv[t], W, R, W, 0, st);
    fgemm(hh[t], dm, dm, nullptr, 0, 0, Pw(S.ta(K_W)), W, Pw(S.ta(K_B)), hkv[t], W, R, W, 0, st);
    fgemm(hh[t], dm, dm, nullptr, 0, 0, Pw(S.ta(V_W)), W, Pw(S.ta(V_B)), hvv[t], W, R, W, 0, st);
    // tcgen05 first; the mma.sync kernels are gated on its flag (they run only if the
    // split-fp16 tcgen05 path could not take the call) -- no host synchronisation
    const int32_t* fgate =
        tape_tc ? tape_attention_fwd_tc(hqv[t], hkv[t], hvv[t], W, H, dh, R, F, d_tcw,
                                        (int64_t)tcw.size(), d_tr0, d_tn, Ttot, row_fwd, hat[t],
                                        W, hls[t], tape_ws, st)
                : nullptr;
    attn_fwd(hqv[t], hkv[t], hvv[t], d_hq, (int64_t)hq.size(), hat[t], hls[t], fgate);
    fgemm(hat[t], W, W, nullptr, 0, 0, Pw(S.ta(O_W)), dm, Pw(S.ta(O_B)), ho[t], dm, R, dm, 0, st);
    fgemm(ho[t], dm, dm, nullptr, 0, 0, Pw(S.task(t, FC_W1)), di, Pw(S.task(t, FC_B1)), hf1[t], di, R,
         di, 1, st);
    fgemm(hf1[t], di, di, nullptr, 0, 0, Pw(S.task(t, FC_W2)), dm, Pw(S.task(t, FC_B2)), hrep[t], dm, R,
         dm, 0, st);
    int a = cfg.task_sizes[t];
    fgemm(hrep[t], dm, dm, nullptr, 0, 0, Pw(S.task(t, OUT_W)), a, Pw(S.task(t, OUT_B)), hlog[t], a, R,
         a, 0, st);
  }
  mean_rows(hrep[T - 1], dm, m.d_row_off, F, m.d_chunks, m.n_chunks, dm, meanrep, dm, part, st);
  value_head(meanrep, F, dm, Pw(S.value_w()), Pw(S.value_w() + 1), value, st);

  // ================================================================ loss
  double* stats = A.take<double>((int64_t)F * 3 * 4 + F);
  CUDA_CHECK(cudaMemsetAsync(stats, 0, ((size_t)F * 3 * 4 + F) * 8, st));
  std::vector<float*> dlog(T);
  for (int t = 0; t < T; ++t) {
    int a = cfg.task_sizes[t];
    dlog[t] = A.take<float>(R * a);
    ppo_loss(hlog[t], a, R, actions + (int64_t)t * R, row_node, old_logp + (int64_t)t * R, row_fwd,
             m.d_row_off, d_fp, clip_eps, ent_coef, T, C, t, dlog[t], stats, st);
  }
  // value loss: fparams[f][2] holds the reward
  float* dvalue = A.take<float>(F);
  double* rewards = A.take<double>(F);
  {
    std::vector<double> rw(F);
    for (int f = 0; f < F; ++f) rw[f] = fparams_host[4 * f + 2];
    CUDA_CHECK(cudaMemcpyAsync(rewards, rw.data(), F * 8, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
  }

  // ================================================================ backward
  float* d1 = A.take<float>(R * std::max(gs, dm));
  float* d2 = A.take<float>(R * std::max(gs, dm));
  float* d3 = A.take<float>(R * std::max(gs, dm));
  float* dhid = A.take<float>(R * dm);
  float* dF1 = A.take<float>(R * di);
  float* dQ = A.take<float>(R * W);
  float* dK = A.take<float>(R * W);
  float* dV = A.take<float>(R * W);
  float* dK2 = A.take<float>(R * W);
  float* dV2 = A.take<float>(R * W);
  float* dAt = A.take<float>(R * W);
  float* Dbuf = A.take<float>(R * H);
  float* dmod = A.take<float>((int64_t)F * dm);
  float* dge = A.take<float>((int64_t)F * gs);
  float* dprev = A.take<float>(R * dm);
  float* dxB = A.take<float>(R * dm);
  CUDA_CHECK(cudaMemsetAsync(dhid, 0, (size_t)R * dm * 4, st));
  CUDA_CHECK(cudaMemsetAsync(dmod, 0, (size_t)F * dm * 4, st));

  // ---- heads, last task first
  bool have_dprev = false;
  for (int t = T - 1; t >= 0; --t) {
    int a = cfg.task_sizes[t];
    float* drep = d1;
    // logits = rep out_w + out_b
    dgemm(dlog[t], a, Pw(S.task(t, OUT_W)), a, drep, dm, R, dm, a, false);
    wgrad(hrep[t], dm, dm, nullptr, 0, 0, dlog[t], a, R, a, Gw(S.task(t, OUT_W)), Gw(S.task(t, OUT_B)), st);
    if (t == T - 1)
      value_backward(value, meanrep, rewards, F, dm, value_coef, C, Pw(S.value_w()), dvalue,
                     Gw(S.value_w()), Gw(S.value_w() + 1), stats + (int64_t)F * 12, drep, dm,
                     m.d_row_off, row_fwd, R, st);
    if (have_dprev) add_into(drep, dm, dprev, dm, R, dm, st);
    // rep = f1 W2 + b2 ; f1 = relu(o W1 + b1)
    dgemm(drep, dm, Pw(S.task(t, FC_W2)), dm, dF1, di, R, di, dm, false);
    wgrad(hf1[t], di, di, nullptr, 0, 0, drep, dm, R, dm, Gw(S.task(t, FC_W2)), Gw(S.task(t, FC_B2)), st);
    act_backward(dF1, di, hf1[t], di, R, di, 1, st);
    float* dO = d2;
    dgemm(dF1, di, Pw(S.task(t, FC_W1)), di, dO, dm, R, dm, di, false);
    wgrad(ho[t], dm, dm, nullptr, 0, 0, dF1, di, R, di, Gw(S.task(t, FC_W1)), Gw(S.task(t, FC_B1)), st);
    // o = att Wo + bo
    dgemm(dO, dm, Pw(S.ta(O_W)), dm, dAt, W, R, W, dm, false);
    wgrad(hat[t], W, W, nullptr, 0, 0, dO, dm, R, dm, Gw(S.ta(O_W)), Gw(S.ta(O_B)), st);
    // dq, dk, dv on tcgen05 (tc_tape.cu) when the operands fit the split-fp16 path,
    // otherwise on the mma.sync kernels
    const int32_t* bgate =
        tape_tc ? tape_attention_bwd_tc(hqv[t], hkv[t], hvv[t], hat[t], dAt, W, H, dh, R, F,
                                        hls[t], d_kvw, (int64_t)kvw.size(), d_qw,
                                        (int64_t)qw.size(), d_tr0, d_tn, Ttot, Dbuf, dQ, dK, dV,
                                        tape_ws, st)
                : nullptr;
    attn_bwd(hqv[t], hkv[t], hvv[t], hat[t], dAt, hls[t], d_hq, (int64_t)hq.size(), d_hk,
             (int64_t)hk.size(), Dbuf, dQ, dK, dV, nullptr, nullptr, bgate);
    float* dHH = d3;
    dgemm(dQ, W, Pw(S.ta(Q_W)), W, dHH, dm, R, dm, W, false);
    dgemm(dK, W, Pw(S.ta(K_W)), W, dHH, dm, R, dm, W, true);
    dgemm(dV, W, Pw(S.ta(V_W)), W, dHH, dm, R, dm, W, true);
    wgrad(hh[t], dm, dm, nullptr, 0, 0, dQ, W, R, W, Gw(S.ta(Q_W)), Gw(S.ta(Q_B)), st);
    wgrad(hh[t], dm, dm, nullptr, 0, 0, dK, W, R, W, Gw(S.ta(K_W)), Gw(S.ta(K_B)), st);
    wgrad(hh[t], dm, dm, nullptr, 0, 0, dV, W, R, W, Gw(S.ta(V_W)), Gw(S.ta(V_B)), st);
    float* dC = d1;
    ln_backward(hc[t], dm, Pw(S.task(t, LN_G)), dHH, dm, dC, dm, false, R, dm, Gw(S.task(t, LN_G)),
                Gw(S.task(t, LN_B)), st);
    // c = [a_in | hid] cat_w + cat_b
    if (zero_in[t]) {
      wgrad(hid, dm, dm, nullptr, 0, 0, dC, dm, R, dm, Gw(S.task(t, CAT_W)) + (int64_t)dm * dm,
            Gw(S.task(t, CAT_B)), st);
      dgemm(dC, dm, Pw(S.task(t, CAT_W)) + (int64_t)dm * dm, dm, dhid, dm, R, dm, dm, true);
      have_dprev = false;
    } else {
      wgrad(hrep[t - 1], dm, dm, hid, dm, dm, dC, dm, R, dm, Gw(S.task(t, CAT_W)), Gw(S.task(t, CAT_B)),
            st);
      dgemm(dC, dm, Pw(S.task(t, CAT_W)) + (int64_t)dm * dm, dm, dhid, dm, R, dm, dm, true);
      dgemm(dC, dm, Pw(S.task(t, CAT_W)), dm, dprev, dm, R, dm, dm, false);
      have_dprev = true;
    }
  }

  // ---- trunk, last layer first
  float* dx = dhid;  // gradient w.r.t. x_{l+1}
  for (int l = Lt - 1; l >= 0; --l) {
    float* du2 = d1;
    ln_backward(tu2[l], dm, Pw(S.blk(l, LN2_G)), dx, dm, du2, dm, false, R, dm, Gw(S.blk(l, LN2_G)),
                Gw(S.blk(l, LN2_B)), st);
    // u2 = h1 + f1 W2 + b2
    dgemm(du2, dm, Pw(S.blk(l, FF_W2)), dm, dF1, di, R, di, dm, false);
    wgrad(tf1[l], di, di, nullptr, 0, 0, du2, dm, R, dm, Gw(S.blk(l, FF_W2)), Gw(S.blk(l, FF_B2)), st);
    act_backward(dF1, di, tf1[l], di, R, di, 1, st);
    float* dh1 = d2;
    cudaMemcpyAsync(dh1, du2, (size_t)R * dm * 4, cudaMemcpyDeviceToDevice, st);
    dgemm(dF1, di, Pw(S.blk(l, FF_W1)), di, dh1, dm, R, dm, di, true);
    wgrad(th1[l], dm, dm, nullptr, 0, 0, dF1, di, R, di, Gw(S.blk(l, FF_W1)), Gw(S.blk(l, FF_B1)), st);
    float* du1 = d3;
    ln_backward(tu1[l], dm, Pw(S.blk(l, LN1_G)), dh1, dm, du1, dm, false, R, dm, Gw(S.blk(l, LN1_G)),
                Gw(S.blk(l, LN1_B)), st);
    // u1 = xm + att Wo + bo
    dgemm(du1, dm, Pw(S.blk(l, O_W)), dm, dAt, W, R, W, dm, false);
    wgrad(tat[l], W, W, nullptr, 0, 0, du1, dm, R, dm, Gw(S.blk(l, O_W)), Gw(S.blk(l, O_B)), st);
    attn_bwd(tqv[l], tkv[l], tvv[l], tat[l], dAt, tls[l], d_tq, (int64_t)tq.size(), d_tk,
             (int64_t)tk.size(), Dbuf, dQ, dK, dV, dK2, dV2);
    // dxm = du1 + (dq Wq^T + dk_self Wk^T + dv_self Wv^T); weights see self + cache parts
    float* dxm = du1;
    dgemm(dQ, W, Pw(S.blk(l, Q_W)), W, dxm, dm, R, dm, W, true);
    dgemm(dK, W, Pw(S.blk(l, K_W)), W, dxm, dm, R, dm, W, true);
    dgemm(dV, W, Pw(S.blk(l, V_W)), W, dxm, dm, R, dm, W, true);
    add_into(dK, W, dK2, W, R, W, st);
    add_into(dV, W, dV2, W, R, W, st);
    wgrad(txm[l], dm, dm, nullptr, 0, 0, dQ, W, R, W, Gw(S.blk(l, Q_W)), Gw(S.blk(l, Q_B)), st);
    wgrad(txm[l], dm, dm, nullptr, 0, 0, dK, W, R, W, Gw(S.blk(l, K_W)), Gw(S.blk(l, K_B)), st);
    wgrad(txm[l], dm, dm, nullptr, 0, 0, dV, W, R, W, Gw(S.blk(l, V_W)), Gw(S.blk(l, V_B)), st);
    // xm = x * mod
    float* dxl = (dx == dhid) ? dxB : dhid;
    rowvec_backward(dxm, dm, tx[l], dm, mod, row_fwd, dxl, dm, dmod, R, dm, st);
    dx = dxl;
  }
  // x0 = node_embed in_w + in_b (policy/in_w)
  float* dne = A.take<float>(R * gs);
  float* dhB = A.take<float>(R * gs);
  float* dP = A.take<float>(R * gs);
  float* dt = A.take<float>(R * gs);
  dgemm(dx, dm, Pw(S.pbase()), dm, dne, gs, R, gs, dm, false);
  wgrad(node_embed, gs, gs, nullptr, 0, 0, dx, dm, R, dm, Gw(S.pbase()), Gw(S.pbase() + 1), st);
  // modulation: mod = 2 sigma(block(ge in_w + in_b))
  BlockG bg{Gw(S.blk(mb, V_W)),  Gw(S.blk(mb, V_B)),  Gw(S.blk(mb, O_W)),  Gw(S.blk(mb, O_B)),
            Gw(S.blk(mb, LN1_G)), Gw(S.blk(mb, LN1_B)), Gw(S.blk(mb, FF_W1)), Gw(S.blk(mb, FF_B1)),
            Gw(S.blk(mb, FF_W2)), Gw(S.blk(mb, FF_B2)), Gw(S.blk(mb, LN2_G)), Gw(S.blk(mb, LN2_B))};
  modulate_backward(ge, F, gs, Pw(S.pbase()), Pw(S.pbase() + 1), bw, dm, W, di, dmod, dge, bg,
                    Gw(S.pbase()), Gw(S.pbase() + 1), st);
  // ge = mean_rows(node_embed)
  mean_backward(dne, gs, dge, m.d_row_off, row_fwd, R, gs, st);

  // ---- embed, last layer first
  float* dcur = dne;
  float* other = dhB;
  for (int l = Lg - 1; l >= 0; --l) {
    // h_{l+1} = relu([h_l | pool] fc_w + fc_b)
    act_backward(dcur, gs, eh[l + 1], gs, R, gs, 1, st);
    wgrad(eh[l], gs, gs, ep[l], gs, gs, dcur, gs, R, gs, Gw(S.e_layer(l, 2)), Gw(S.e_layer(l, 3)), st);
    dgemm(dcur, gs, Pw(S.e_layer(l, 2)) + (int64_t)gs * gs, gs, dP, gs, R, gs, gs, false);
    dgemm(dcur, gs, Pw(S.e_layer(l, 2)), gs, other, gs, R, gs, gs, false);
    // pool = segmax(t) ; t = sigmoid(h agg_w + agg_b)
    CUDA_CHECK(cudaMemsetAsync(dt, 0, (size_t)R * gs * 4, st));
    segmax_backward(dP, gs, ea[l], R, gs, dt, gs, st);
    act_backward(dt, gs, et[l], gs, R, gs, 2, st);
    wgrad(eh[l], gs, gs, nullptr, 0, 0, dt, gs, R, gs, Gw(S.e_layer(l, 0)), Gw(S.e_layer(l, 1)), st);
    dgemm(dt, gs, Pw(S.e_layer(l, 0)), gs, other, gs, R, gs, gs, true);
    std::swap(dcur, other);
  }
  // h0 = feats in_w + in_b
  inproj_wgrad(m.d_views, m.d_row_off, row_fwd, R, b.prev_actions, T, tcol, dcur, gs, gs, Fdim,
               Gw(S.e_in_w()), Gw(S.e_in_b()), st);

  // ---- stats to host: [F][3][4] surr, ent, ratio, clipped ; [F] value err^2 ; [F] value
  std::vector<float> hv(F);
  CUDA_CHECK(cudaMemcpyAsync(stats_host, stats, ((size_t)F * 12 + F) * 8, cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaMemcpyAsync(hv.data(), value, F * 4, cudaMemcpyDeviceToHost, st));
  CUDA_CHECK(cudaStreamSynchronize(st));
  for (int f = 0; f < F; ++f) stats_host[(size_t)F * 13 + f] = hv[f];
}

}  // namespace go

using namespace go;

extern "C" {

int go_ppo_grad(go_ctx_t ctx, const go_config_t* cfg, const float* params,
                const int64_t* param_offsets, const go_batch_t* batch, const int32_t* actions,
                const double* old_logp, const double* fparams, double clip_eps, double ent_coef,
                double value_coef, int32_t loss_denominator, float* grads, double* stats_out,
                void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    run_ppo_grad(ctx, *cfg, params, param_offsets, *batch, actions, old_logp, fparams, clip_eps,
                 ent_coef, value_coef, loss_denominator, grads, stats_out, (cudaStream_t)stream);
  });
}

int go_adam(go_ctx_t ctx, float* params, const float* grads, float* m, float* v, int64_t count,
            int64_t step, double lr, double beta1, double beta2, double eps, void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    GO_CHECK(step >= 1, "adam step must be >= 1");
    adam(params, grads, m, v, count, lr, beta1, beta2, eps, step, (cudaStream_t)stream);
  });
}

int go_adam64(go_ctx_t ctx, double* params, float* params32, const float* grads, double* m,
              double* v, int64_t count, int64_t step, double lr, double beta1, double beta2,
              double eps, void* stream) {
  return guarded([&] {
    CUDA_CHECK(cudaSetDevice(ctx->device));
    GO_CHECK(step >= 1, "adam step must be >= 1");
    adam64(params, params32, grads, m, v, count, lr, beta1, beta2, eps, step,
           (cudaStream_t)stream);
  });
}

}  // extern "C"

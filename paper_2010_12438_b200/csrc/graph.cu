// Native graph ingest (host C++): topological order, neighbour CSR, feature
// statics, FusedGraph DES tables, greedy balanced placement.  Replaces the
// reference's Python construction paths (graph.py:78-201, simulator.py:86-172,
// costmodel.py:149-187, baselines.py:75-118) with O(N log N) host code; the
// result is uploaded once per graph and reused by every forward / simulation.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <queue>
#include <set>

#include "engine.cuh"

namespace go {

// CPython 3.12 builtin sum() over floats starting from int 0 (the reference's
// fused_cost sums, costmodel.py:181-187): the first term is taken exactly
// (0 + x), the rest use Neumaier's compensated summation, and the compensation is
// added at the end when non-zero and finite (Python/bltinmodule.c builtin_sum_impl).
struct PySum {
  double f = 0.0, c = 0.0;
  bool any = false;
  void add(double x) {
    if (!any) {
      f = x;
      any = true;
      return;
    }
    double t = f + x;
    if (std::fabs(f) >= std::fabs(x)) c += (f - t) + x;
    else c += (x - t) + f;
    f = t;
  }
  double value() const {
    if (!any) return 0.0;
    return (c != 0.0 && std::isfinite(c)) ? f + c : f;
  }
};

// Kahn with a min-heap on node id (graph.py:173-201).  Self-loops count toward the
// in-degree but add no successor, exactly like _partial_topo, so they are cycles.
std::vector<int32_t> topo_order(int32_t n, int64_t e, const int32_t* src, const int32_t* dst) {
  std::vector<int32_t> indeg(n, 0);
  std::vector<int64_t> off(n + 1, 0);
  for (int64_t j = 0; j < e; ++j) {
    GO_CHECK(src[j] >= 0 && src[j] < n && dst[j] >= 0 && dst[j] < n, "dangling edge %d->%d",
             src[j], dst[j]);
    indeg[dst[j]]++;
    if (src[j] != dst[j]) off[src[j] + 1]++;
  }
  for (int i = 0; i < n; ++i) off[i + 1] += off[i];
  std::vector<int32_t> succ(off[n]);
  std::vector<int64_t> fill(off.begin(), off.end() - 1);
  for (int64_t j = 0; j < e; ++j)
    if (src[j] != dst[j]) succ[fill[src[j]]++] = dst[j];
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> heap;
  for (int i = 0; i < n; ++i)
    if (indeg[i] == 0) heap.push(i);
  std::vector<int32_t> order;
  order.reserve(n);
  while (!heap.empty()) {
    int v = heap.top();
    heap.pop();
    order.push_back(v);
    for (int64_t j = off[v]; j < off[v + 1]; ++j)
      if (--indeg[succ[j]] == 0) heap.push(succ[j]);
  }
  if ((int32_t)order.size() != n) GO_THROW(GO_ERR_CYCLE, "cycle detected");
  return order;
}

// greedy_placement DP (baselines.py:75-118) with the same float64 values and the
// same first-argmin tie-break, in O(D N log N): for fixed (k, i) the candidate
// max(dp[j], P[i]-P[j]) is max of a non-decreasing and a non-increasing sequence
// in j (both hold in IEEE arithmetic), so the first argmin is found by binary search.
void greedy_cuts(int32_t n, const double* flops_topo, int32_t d, int64_t* cuts_out) {
  GO_CHECK(d >= 1, "need at least one device");
  std::vector<double> P(n + 1, 0.0);
  // np.cumsum: sequential left-to-right
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    acc = (i == 0) ? flops_topo[0] : acc + flops_topo[i];
    P[i + 1] = acc;
  }
  std::vector<double> dp(n + 1, INFINITY), nxt(n + 1);
  dp[0] = 0.0;
  std::vector<std::vector<int32_t>> choice(d + 1, std::vector<int32_t>(n + 1, 0));
  for (int k = 1; k <= d; ++k) {
    for (int i = 0; i <= n; ++i) {
      auto B = [&](int j) { return P[i] - P[j]; };
      // j* = first j in [0, i] with dp[j] >= B(j)
      int lo = 0, hi = i;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (dp[mid] >= B(mid)) hi = mid;
        else lo = mid + 1;
      }
      int js = lo;
      int best = js;
      double val = std::max(dp[js], B(js));
      if (js > 0) {
        double bv = B(js - 1);  // = cand[js-1] since dp < B there
        if (bv <= val) {
          // first j with B(j) <= bv (B non-increasing) -> start of the plateau
          int a = 0, b = js - 1;
          while (a < b) {
            int mid = (a + b) >> 1;
            if (B(mid) <= bv) b = mid;
            else a = mid + 1;
          }
          best = a;
          val = bv;
        }
      }
      nxt[i] = val;
      choice[k][i] = best;
    }
    std::swap(dp, nxt);
  }
  std::vector<int64_t> cuts;
  cuts.push_back(n);
  int i = n;
  for (int k = d; k >= 1; --k) {
    i = choice[k][i];
    cuts.push_back(i);
  }
  std::reverse(cuts.begin(), cuts.end());
  for (int k = 0; k <= d; ++k) cuts_out[k] = cuts[k];
}

// Greedy fusion pass (simulator.py:199-277): visit nodes by (-priority, id); a
// fusible node with non-zero priority merges its group with the group of its best
// visited fusible neighbour ((-priority, id) minimum) unless the union exceeds
// max_group or closes a cycle through a third group (simulator.py:180-196 DFS).
// The union keeps the larger root (ties: the visiting node's root).
void fuse_groups(int32_t n, int64_t e, const int32_t* src, const int32_t* dst,
                 const int32_t* op, const int64_t* pri, int32_t max_group, int64_t* label) {
  static const bool fusible_op[12] = {false, false, true, true, true, true,
                                      true,  true,  true, true, false, false};
  std::vector<int32_t> parent(n), size(n, 1);
  std::iota(parent.begin(), parent.end(), 0);
  bool any = false;
  for (int v = 0; v < n; ++v) any |= (pri[v] > 0 && fusible_op[op[v]]);
  if (!any) {
    for (int v = 0; v < n; ++v) label[v] = v;
    return;
  }
  auto find = [&](int v) {
    while (parent[v] != v) {
      parent[v] = parent[parent[v]];
      v = parent[v];
    }
    return v;
  };
  std::vector<std::set<int32_t>> succ(n), pred(n);
  std::vector<std::vector<int32_t>> nb(n);
  for (int64_t j = 0; j < e; ++j) {
    succ[src[j]].insert(dst[j]);
    pred[dst[j]].insert(src[j]);
    nb[src[j]].push_back(dst[j]);
    nb[dst[j]].push_back(src[j]);
  }
  for (auto& l : nb) {
    std::sort(l.begin(), l.end());
    l.erase(std::unique(l.begin(), l.end()), l.end());
  }
  std::vector<int32_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return pri[a] != pri[b] ? pri[a] > pri[b] : a < b; });
  std::vector<char> visited(n, 0);
  // Exact, windowed cycle check.  The group graph stays a DAG, and the two candidate
  // groups are joined by an edge a -> b, so b ~> a is impossible and only a path
  // a ~> b through a third group can close a cycle (the reference's two DFS runs
  // return the same answer).  A topological order of the *group* graph is maintained
  // (pos / at): every group on such a path lies strictly between pos[a] and pos[b], so
  // the search is confined to that window instead of all of a's descendants.  After a
  // merge the window is re-laid out as [groups not reachable from a] [a+b] [groups
  // reachable from a], which is again a valid order.  Cost per attempt: O(window).
  const std::vector<int32_t> topo = topo_order(n, e, src, dst);
  std::vector<int32_t> pos(n), at(n);
  for (int i = 0; i < n; ++i) {
    at[i] = topo[i];
    pos[topo[i]] = i;
  }
  std::vector<int32_t> stack, nonf, fw;
  std::vector<int32_t> mark(n, -1);
  int stamp = 0;
  auto third_path = [&](int x, int y) {  // edge x -> y exists
    const int lim = pos[y];
    ++stamp;
    stack.clear();
    for (int s : succ[x])
      if (s != y && pos[s] < lim && mark[s] != stamp) {
        mark[s] = stamp;
        stack.push_back(s);
      }
    while (!stack.empty()) {
      const int s = stack.back();
      stack.pop_back();
      for (int t : succ[s]) {
        if (t == y) return true;
        if (pos[t] < lim && mark[t] != stamp) {
          mark[t] = stamp;
          stack.push_back(t);
        }
      }
    }
    return false;
  };
  // re-lay the window [pos[x], pos[y]] after x and y merged into `root`
  auto relayout = [&](int x, int y, int root) {
    const int px = pos[x], py = pos[y];
    ++stamp;
    stack.clear();
    for (int s : succ[x])
      if (s != y && pos[s] < py && mark[s] != stamp) {
        mark[s] = stamp;
        stack.push_back(s);
      }
    while (!stack.empty()) {
      const int s = stack.back();
      stack.pop_back();
      for (int t : succ[s])
        if (pos[t] < py && mark[t] != stamp) {
          mark[t] = stamp;
          stack.push_back(t);
        }
    }
    nonf.clear();
    fw.clear();
    for (int p = px + 1; p < py; ++p) {
      const int g = at[p];
      if (g < 0) continue;
      (mark[g] == stamp ? fw : nonf).push_back(g);
    }
    int p = px;
    for (int g : nonf) {
      at[p] = g;
      pos[g] = p++;
    }
    at[p] = root;
    pos[root] = p++;
    for (int g : fw) {
      at[p] = g;
      pos[g] = p++;
    }
    for (; p <= py; ++p) at[p] = -1;
  };
  for (int v : order) {
    if (pri[v] > 0 && fusible_op[op[v]]) {
      int best = -1;
      for (int u : nb[v]) {
        if (!visited[u] || pri[u] <= 0 || !fusible_op[op[u]]) continue;
        if (best < 0 || pri[u] > pri[best] || (pri[u] == pri[best] && u < best)) best = u;
      }
      if (best >= 0) {
        int rv = find(v), ru = find(best);
        if (rv != ru && size[rv] + size[ru] <= max_group) {
          // orient the joining edge (original neighbours: one direction exists)
          const bool fwd_edge = succ[rv].count(ru) > 0;
          const int x = fwd_edge ? rv : ru, y = fwd_edge ? ru : rv;
          if (!third_path(x, y)) {
            // the group-graph edits must see the pre-merge adjacency: relayout first
            if (size[rv] < size[ru]) std::swap(rv, ru);
            parent[ru] = rv;
            size[rv] += size[ru];
            // relayout uses succ[x] before the fold (reachability from x within the
            // window is unchanged by the fold: it only renames x, y to rv)
            relayout(x, y, rv);
            std::set<int32_t> ns, np;
            for (int s : succ[rv]) ns.insert(s);
            for (int s : succ[ru]) ns.insert(s);
            for (int s : pred[rv]) np.insert(s);
            for (int s : pred[ru]) np.insert(s);
            ns.erase(rv);
            ns.erase(ru);
            np.erase(rv);
            np.erase(ru);
            for (int s : succ[ru]) pred[s].erase(ru);
            for (int s : pred[ru]) succ[s].erase(ru);
            for (int s : succ[rv]) pred[s].erase(rv);
            for (int s : pred[rv]) succ[s].erase(rv);
            succ[rv] = ns;
            pred[rv] = np;
            for (int s : ns) pred[s].insert(rv);
            for (int s : np) succ[s].insert(rv);
            succ[ru].clear();
            pred[ru].clear();
          }
        }
      }
    }
    visited[v] = 1;
  }
  for (int v = 0; v < n; ++v) label[v] = find(v);
}

}  // namespace go

using namespace go;

// -----------------------------------------------------------------------------------
template <class T>
static T* upload(const std::vector<T>& h, std::vector<void*>* track = nullptr) {
  T* d = nullptr;
  size_t bytes = std::max<size_t>(h.size(), 1) * sizeof(T);
  CUDA_CHECK(cudaMalloc(&d, bytes));
  if (!h.empty()) CUDA_CHECK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  if (track) track->push_back(d);
  return d;
}

GraphView go_graph::view() const {
  GraphView v;
  v.n = n;
  v.order = d_order;
  v.op_row = d_op_row;
  v.static4 = d_static4;
  v.nbr_off = d_nbr_off;
  v.nbr_row = d_nbr_row;
  v.samp_off = d_samp_off;
  return v;
}

void go_graph::ensure_samp(int32_t k) {
  if (samp_k == k) return;
  std::vector<int64_t> so(n + 1, 0);
  for (int r = 0; r < n; ++r) so[r + 1] = so[r] + std::min<int64_t>(nbr_off[r + 1] - nbr_off[r], k);
  if (d_samp_off) cudaFree(d_samp_off);
  d_samp_off = upload(so);
  samp_k = k;
  samp_total = so[n];
}

go_graph::~go_graph() {
  for (void* p : {(void*)d_order, (void*)d_op_row, (void*)d_static4, (void*)d_nbr_off,
                  (void*)d_nbr_row, (void*)d_samp_off})
    if (p) cudaFree(p);
  for (void* p : des_allocs) cudaFree(p);
}

// FusedGraph tables for a grouping (simulator.py:86-172): groups renumbered by
// ascending lowest member; external out edges sorted (src, dst) stably; costs per
// costmodel.py:149-187 with the reference's summation orders; resident bytes
// (simulator.py:125-133); distinct succ/pred group sets; heap-Kahn topo index.
void go_graph::set_fusion(const std::vector<int64_t>& label) {
  for (void* p : des_allocs) cudaFree(p);
  des_allocs.clear();
  // canonical group ids
  std::vector<int64_t> roots(label.begin(), label.end());
  std::sort(roots.begin(), roots.end());
  roots.erase(std::unique(roots.begin(), roots.end()), roots.end());
  int G = (int)roots.size();
  std::vector<int32_t> gm(n);
  for (int v = 0; v < n; ++v)
    gm[v] = (int32_t)(std::lower_bound(roots.begin(), roots.end(), label[v]) - roots.begin());
  std::vector<int32_t> first(G, INT32_MAX);
  for (int v = 0; v < n; ++v) first[gm[v]] = std::min(first[gm[v]], v);
  std::vector<int32_t> ord(G);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return first[a] < first[b]; });
  std::vector<int32_t> pos(G);
  for (int i = 0; i < G; ++i) pos[ord[i]] = i;
  for (int v = 0; v < n; ++v) gm[v] = pos[gm[v]];
  std::vector<int32_t> rep(G, INT32_MAX);
  std::vector<int64_t> gsize(G, 0);
  for (int v = 0; v < n; ++v) {
    rep[gm[v]] = std::min(rep[gm[v]], v);
    gsize[gm[v]]++;
  }
  // edges
  std::vector<int32_t> pend(G, 0);
  std::vector<std::vector<int64_t>> ext_out(G), ext_in(G);
  std::vector<char> has_out(n, 0), leaves(n, 0), any_out(n, 0);
  for (int64_t j = 0; j < e; ++j) {
    int gs = gm[src[j]], gd = gm[dst[j]];
    any_out[src[j]] = 1;
    has_out[src[j]] = 1;  // internal or external consumer (costmodel.py:183)
    if (gs != gd) {
      ext_out[gs].push_back(j);
      ext_in[gd].push_back(j);
      leaves[src[j]] = 1;
    }
  }
  int64_t num_out = 0, max_deg = 0;
  std::vector<int64_t> out_off(G + 1, 0);
  for (int i = 0; i < G; ++i) {
    std::stable_sort(ext_out[i].begin(), ext_out[i].end(), [&](int64_t a, int64_t b) {
      return src[a] != src[b] ? src[a] < src[b] : dst[a] < dst[b];
    });
    out_off[i + 1] = out_off[i] + (int64_t)ext_out[i].size();
    max_deg = std::max<int64_t>(max_deg, (int64_t)ext_out[i].size());
    pend[i] = (int32_t)ext_in[i].size();
  }
  num_out = out_off[G];
  std::vector<int32_t> out_grp(num_out);
  std::vector<double> out_b(num_out);
  for (int i = 0; i < G; ++i)
    for (size_t t = 0; t < ext_out[i].size(); ++t) {
      int64_t j = ext_out[i][t];
      out_grp[out_off[i] + t] = gm[dst[j]];
      out_b[out_off[i] + t] = ebytes[j];
    }
  // members sorted by id
  std::vector<std::vector<int32_t>> members(G);
  for (int v = 0; v < n; ++v) members[gm[v]].push_back(v);
  std::vector<double> cf(G), cb(G), res(G);
  bool int_exact = true;
  double res_total = 0.0;
  for (int i = 0; i < G; ++i) {
    PySum fl, reads, writes;
    for (int v : members[i]) fl.add(flops[v]);
    for (int64_t j : ext_in[i]) reads.add(ebytes[j]);
    // writers = {srcs of external_out} | (members - has_out), summed in id order
    for (int v : members[i])
      if (leaves[v] || !has_out[v]) writes.add(out_bytes[v]);
    cf[i] = fl.value();
    cb[i] = reads.value() + writes.value();
    // resident: members with no consumers or any consumer outside the group
    double tot = 0.0;
    for (int v : members[i])
      if (!any_out[v] || leaves[v]) tot += out_bytes[v];
    res[i] = tot;
    if (tot != std::floor(tot)) int_exact = false;
    res_total += tot;
  }
  if (res_total >= 9007199254740992.0) int_exact = false;
  // distinct group succ / pred
  std::vector<std::vector<int32_t>> gsucc(G), gpred(G);
  for (int i = 0; i < G; ++i) {
    std::vector<int32_t> s;
    for (int64_t t = out_off[i]; t < out_off[i + 1]; ++t) s.push_back(out_grp[t]);
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    gsucc[i] = s;
    for (int32_t t : s) gpred[t].push_back(i);
  }
  std::vector<int32_t> nsucc(G);
  std::vector<int64_t> pred_off(G + 1, 0);
  for (int i = 0; i < G; ++i) {
    nsucc[i] = (int32_t)gsucc[i].size();
    pred_off[i + 1] = pred_off[i] + (int64_t)gpred[i].size();
  }
  std::vector<int32_t> pred_grp;
  pred_grp.reserve(pred_off[G]);
  for (int i = 0; i < G; ++i) pred_grp.insert(pred_grp.end(), gpred[i].begin(), gpred[i].end());
  // heap-Kahn topo index over the group DAG (simulator.py:155-172)
  std::vector<int32_t> indeg(G), tindex(G, 0);
  for (int i = 0; i < G; ++i) indeg[i] = (int32_t)gpred[i].size();
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> heap;
  for (int i = 0; i < G; ++i)
    if (indeg[i] == 0) heap.push(i);
  int seen = 0;
  while (!heap.empty()) {
    int i = heap.top();
    heap.pop();
    tindex[i] = seen++;
    for (int32_t t : gsucc[i])
      if (--indeg[t] == 0) heap.push(t);
  }
  acyclic = (seen == G);
  // colocation groups -> member groups
  std::vector<int64_t> coff(1, 0);
  std::vector<int32_t> cgrp;
  int32_t maxc = -1;
  for (int v = 0; v < n; ++v) maxc = std::max(maxc, coloc[v]);
  if (maxc >= 0) {
    std::vector<std::vector<int32_t>> cm(maxc + 1);
    for (int v = 0; v < n; ++v)
      if (coloc[v] >= 0) cm[coloc[v]].push_back(gm[v]);
    for (auto& l : cm) {
      if (l.empty()) continue;
      cgrp.insert(cgrp.end(), l.begin(), l.end());
      coff.push_back((int64_t)cgrp.size());
    }
  }
  GO_CHECK(num_out < ((int64_t)1 << 31) && pred_off[G] < ((int64_t)1 << 31),
           "DES edge tables exceed 2^31 entries");
  std::vector<DesGroupRec> grec(G);
  for (int i = 0; i < G; ++i) {
    DesGroupRec& r = grec[i];
    r = DesGroupRec{};
    r.cost_flops = cf[i];
    r.cost_bytes = cb[i];
    r.resident = res[i];
    r.topo = tindex[i];
    r.rep = rep[i];
    r.out_off = (int32_t)out_off[i];
    r.out_cnt = (int32_t)(out_off[i + 1] - out_off[i]);
    r.pred_off = (int32_t)pred_off[i];
    r.pred_cnt = (int32_t)(pred_off[i + 1] - pred_off[i]);
    r.pending0 = pend[i];
    r.nsucc = nsucc[i];
  }
  DesView v{};
  v.n = n;
  v.G = G;
  v.grec = upload(grec, &des_allocs);
  std::vector<int32_t> srcs;
  for (int i = 0; i < G; ++i)
    if (pend[i] == 0) srcs.push_back(i);
  v.src_grp = upload(srcs, &des_allocs);
  v.num_src = (int32_t)srcs.size();
  v.grp_rep = upload(rep, &des_allocs);
  v.pending0 = upload(pend, &des_allocs);
  v.out_off = upload(out_off, &des_allocs);
  v.out_grp = upload(out_grp, &des_allocs);
  v.out_bytes = upload(out_b, &des_allocs);
  v.cost_flops = upload(cf, &des_allocs);
  v.cost_bytes = upload(cb, &des_allocs);
  v.topo_index = upload(tindex, &des_allocs);
  v.resident = upload(res, &des_allocs);
  v.nsucc = upload(nsucc, &des_allocs);
  v.pred_off = upload(pred_off, &des_allocs);
  v.pred_grp = upload(pred_grp, &des_allocs);
  v.coloc_off = upload(coff, &des_allocs);
  v.coloc_grp = upload(cgrp, &des_allocs);
  v.num_coloc = (int32_t)coff.size() - 1;
  v.mem_int_exact = int_exact ? 1 : 0;
  v.max_out_deg = max_deg;
  v.num_edges = num_out;
  des = v;
}

// -----------------------------------------------------------------------------------
extern "C" {

int go_topo_order(int32_t n, int64_t e, const int32_t* src, const int32_t* dst,
                  int32_t* order_out) {
  return guarded([&] {
    auto o = go::topo_order(n, e, src, dst);
    std::copy(o.begin(), o.end(), order_out);
  });
}

int go_greedy_cuts(int32_t n, const double* flops_topo, int32_t d, int64_t* cuts_out) {
  return guarded([&] { go::greedy_cuts(n, flops_topo, d, cuts_out); });
}

int go_apply_fusion(int32_t n, int64_t e, const int32_t* src, const int32_t* dst,
                    const int32_t* op, const int64_t* priorities, int32_t max_group,
                    int64_t* label_out) {
  return guarded([&] {
    for (int v = 0; v < n; ++v) GO_CHECK(op[v] >= 0 && op[v] < 12, "bad op index");
    go::fuse_groups(n, e, src, dst, op, priorities, max_group, label_out);
  });
}

int go_graph_create(go_ctx_t ctx, int32_t n, int64_t e, const int32_t* op, const double* flops,
                    const double* out_bytes, const int32_t* coloc, const int32_t* src,
                    const int32_t* dst, const double* ebytes, go_graph_t* out) {
  return guarded([&] {
    GO_CHECK(ctx && out, "null handle");
    GO_CHECK(n >= 0 && e >= 0, "negative sizes");
    CUDA_CHECK(cudaSetDevice(ctx->device));
    auto* g = new go_graph();
    try {
      g->ctx = ctx;
      g->n = n;
      g->e = e;
      g->op.assign(op, op + n);
      g->flops.assign(flops, flops + n);
      g->out_bytes.assign(out_bytes, out_bytes + n);
      if (coloc) g->coloc.assign(coloc, coloc + n);
      else g->coloc.assign(n, -1);
      g->src.assign(src, src + e);
      g->dst.assign(dst, dst + e);
      g->ebytes.assign(ebytes, ebytes + e);
      for (int v = 0; v < n; ++v) GO_CHECK(op[v] >= 0 && op[v] < 12, "bad op index %d", op[v]);
      g->order = go::topo_order(n, e, src, dst);
      g->pos.assign(n, 0);
      for (int r = 0; r < n; ++r) g->pos[g->order[r]] = r;
      // undirected sorted-unique neighbour sets (graph.py:131-133), by topo row
      std::vector<std::vector<int32_t>> nb(n);
      for (int64_t j = 0; j < e; ++j) {
        nb[dst[j]].push_back(src[j]);
        nb[src[j]].push_back(dst[j]);
      }
      g->nbr_off.assign(n + 1, 0);
      std::vector<int32_t> indeg(n, 0), outdeg(n, 0);
      for (int64_t j = 0; j < e; ++j) {
        indeg[dst[j]]++;
        outdeg[src[j]]++;
      }
      for (int v = 0; v < n; ++v) {
        auto& l = nb[v];
        std::sort(l.begin(), l.end());
        l.erase(std::unique(l.begin(), l.end()), l.end());
      }
      for (int r = 0; r < n; ++r) g->nbr_off[r + 1] = g->nbr_off[r] + (int64_t)nb[g->order[r]].size();
      g->nbr_row.resize(g->nbr_off[n]);
      std::vector<int32_t> op_row(n);
      std::vector<float> st4((size_t)n * 4);
      for (int r = 0; r < n; ++r) {
        int v = g->order[r];
        int64_t o = g->nbr_off[r];
        for (size_t t = 0; t < nb[v].size(); ++t) g->nbr_row[o + t] = g->pos[nb[v][t]];
        op_row[r] = op[v];
        st4[4 * r + 0] = (float)std::log1p(flops[v]);
        st4[4 * r + 1] = (float)std::log1p(out_bytes[v]);
        st4[4 * r + 2] = (float)indeg[v];
        st4[4 * r + 3] = (float)outdeg[v];
      }
      g->d_order = upload(g->order);
      g->d_op_row = upload(op_row);
      g->d_static4 = upload(st4);
      g->d_nbr_off = upload(g->nbr_off);
      g->d_nbr_row = upload(g->nbr_row);
      std::vector<int64_t> lab(n);
      std::iota(lab.begin(), lab.end(), 0);
      g->set_fusion(lab);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int go_graph_destroy(go_graph_t g) {
  return guarded([&] { delete g; });
}

int go_graph_topo(go_graph_t g, int32_t* order_out) {
  return guarded([&] { std::copy(g->order.begin(), g->order.end(), order_out); });
}

int go_graph_num_neighbors(go_graph_t g, int64_t* total_out) {
  return guarded([&] { *total_out = g->nbr_off[g->n]; });
}

int go_graph_set_fusion(go_graph_t g, const int64_t* label, int32_t* num_groups_out,
                        int32_t* is_acyclic_out) {
  return guarded([&] {
    std::vector<int64_t> lab(label, label + g->n);
    CUDA_CHECK(cudaSetDevice(g->ctx->device));
    g->set_fusion(lab);
    if (num_groups_out) *num_groups_out = g->des.G;
    if (is_acyclic_out) *is_acyclic_out = g->acyclic ? 1 : 0;
  });
}

}  // extern "C"

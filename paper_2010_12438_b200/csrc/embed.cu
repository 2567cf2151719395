// GraphSAGE embedding kernels (embedding.py:47-98, graph.py:268-313).
#include "engine.cuh"
#include "rng.cuh"

namespace go {

// ---------------------------------------------------------------------------------
// Neighbour sampling (embedding.py:47-70).  One thread per (forward, topo row).
// deg <= k: every undirected neighbour (sorted by node id).  deg > k: numpy-exact
// default_rng([seed, node]).choice(deg, k, replace=False) via Floyd's algorithm,
// mapped to neighbours and sorted by node id (== sorted by CSR position).
// Output gidx: per forward f, segment list starting at gbase[f] + samp_off[row],
// holding *batch* row indices (row_off[f] + neighbour topo row).
__global__ void neighbor_sample_kernel(const GraphView* __restrict__ views,
                                       const int64_t* __restrict__ row_off,
                                       const int64_t* __restrict__ gbase,
                                       const int64_t* __restrict__ seeds,
                                       const int32_t* __restrict__ row_fwd, int64_t R, int k,
                                       int32_t* __restrict__ gidx) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  int f = row_fwd[r];
  const GraphView& G = views[f];
  int64_t base = row_off[f];
  int64_t lr = r - base;
  int64_t o0 = G.nbr_off[lr], o1 = G.nbr_off[lr + 1];
  int64_t deg = o1 - o0;
  int32_t* out = gidx + gbase[f] + G.samp_off[lr];
  if (deg <= k) {
    for (int64_t j = 0; j < deg; ++j) out[j] = (int32_t)(base + G.nbr_row[o0 + j]);
    return;
  }
  // Floyd over PCG64(SeedSequence([seed, node])); keep the chosen set sorted in
  // registers (k is small: insertion into a sorted list).
  constexpr int KMAX = 32;
  uint32_t chosen[KMAX];
  int cnt = 0;
  Pcg64 g;
  g.seed2((uint64_t)seeds[f], (uint64_t)G.order[lr]);
  for (int64_t j = deg - k; j < deg; ++j) {
    uint32_t val = g.bounded((uint32_t)j);
    bool dup = false;
    for (int i = 0; i < cnt; ++i) dup |= (chosen[i] == val);
    uint32_t ins = dup ? (uint32_t)j : val;
    int p = cnt++;
    while (p > 0 && chosen[p - 1] > ins) {
      chosen[p] = chosen[p - 1];
      --p;
    }
    chosen[p] = ins;
  }
  for (int i = 0; i < k; ++i) out[i] = (int32_t)(base + G.nbr_row[o0 + chosen[i]]);
}

void neighbor_sample(const GraphView* views_dev, const int64_t* row_off_dev,
                     const int64_t* gbase_dev, const int64_t* seeds_dev, int F,
                     int64_t total_rows, const int32_t* row_fwd, int k, int32_t* gidx,
                     cudaStream_t st) {
  (void)F;
  if (total_rows <= 0) return;
  if (k > 32) GO_THROW(GO_ERR_UNSUPPORTED, "gs_knn %d > 32", k);
  neighbor_sample_kernel<<<(unsigned)cdiv(total_rows, 128), 128, 0, st>>>(
      views_dev, row_off_dev, gbase_dev, seeds_dev, row_fwd, total_rows, k, gidx);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// h0 = node_features @ embed/in_w + in_b (graph.py:268-313 + embedding.py:86).
// The feature row is sparse: one-hot op (12), log1p(flops), log1p(bytes), in/out
// degree, and one prev-action one-hot per task; the affine is a sum of <= 5+T
// weight rows.  task_col[t] = feature column of task t's action block.
__global__ void features_inproj_kernel(const GraphView* __restrict__ views,
                                       const int64_t* __restrict__ row_off,
                                       const int32_t* __restrict__ row_fwd, int64_t R,
                                       const int32_t* __restrict__ prev, int T,
                                       int tc0, int tc1, int tc2,
                                       const float* __restrict__ W, const float* __restrict__ b,
                                       int D, float* __restrict__ h, int64_t ldh) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= R * D) return;
  int64_t r = i / D;
  int c = (int)(i - r * D);
  int f = row_fwd[r];
  const GraphView& G = views[f];
  int64_t lr = r - row_off[f];
  const float* s4 = G.static4 + lr * 4;
  float acc = W[(int64_t)G.op_row[lr] * D + c];
  acc = fmaf(s4[0], W[(int64_t)12 * D + c], acc);
  acc = fmaf(s4[1], W[(int64_t)13 * D + c], acc);
  acc = fmaf(s4[2], W[(int64_t)14 * D + c], acc);
  acc = fmaf(s4[3], W[(int64_t)15 * D + c], acc);
  if (prev) {
    int node = G.order[lr];
    int tcs[3] = {tc0, tc1, tc2};
    for (int t = 0; t < T; ++t) {
      int a = prev[(int64_t)t * R + row_off[f] + node];
      acc += W[(int64_t)(tcs[t] + a) * D + c];
    }
  }
  h[r * ldh + c] = acc + b[c];
}

void features_inproj(const GraphView* views_dev, const int64_t* row_off_dev,
                     const int32_t* row_fwd, int64_t R, const int32_t* prev_actions,
                     int num_tasks, const int32_t* task_col, const float* in_w,
                     const float* in_b, int D, float* h, int64_t ldh, cudaStream_t st) {
  if (R <= 0) return;
  features_inproj_kernel<<<(unsigned)cdiv(R * D, 256), 256, 0, st>>>(
      views_dev, row_off_dev, row_fwd, R, prev_actions, num_tasks, task_col[0], task_col[1],
      task_col[2], in_w, in_b, D, h, ldh);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// pooled[r] = max over sampled neighbours j of t[j] (tensor.py:199-263 gather_rows +
// segment_max; empty segment -> 0).  One warp per row, float4 columns.  This is the
// HBM-bound GraphSAGE aggregation.
__global__ void segment_max_kernel(const float* __restrict__ t, int64_t ldt,
                                   const GraphView* __restrict__ views,
                                   const int64_t* __restrict__ row_off,
                                   const int64_t* __restrict__ gbase,
                                   const int32_t* __restrict__ row_fwd,
                                   const int32_t* __restrict__ gidx, int64_t R, int D,
                                   float* __restrict__ out, int64_t ldo,
                                   int32_t* __restrict__ argmax) {
  int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (r >= R) return;
  int f = row_fwd[r];
  const GraphView& G = views[f];
  int64_t lr = r - row_off[f];
  int64_t s0 = gbase[f] + G.samp_off[lr], s1 = gbase[f] + G.samp_off[lr + 1];
  if (argmax) {
    // training forward: also record the first maximal row per column (tensor.py:240-251)
    for (int c = lane; c < D; c += 32) {
      float m = 0.f;
      int32_t am = -1;
      if (s1 > s0) {
        m = -INFINITY;
        for (int64_t j = s0; j < s1; ++j) {
          float v = t[(int64_t)gidx[j] * ldt + c];
          if (v > m || am < 0) {
            m = v;
            am = gidx[j];
          }
        }
      }
      out[r * ldo + c] = m;
      argmax[r * D + c] = am;
    }
    return;
  }
  if (D == 128 && (ldt & 3) == 0 && (ldo & 3) == 0 && s1 - s0 <= 32) {
    // fast path: one float4 column slice per lane; the segment's neighbour indices
    // are loaded once (one lane each) and broadcast by shuffle, and the gathered rows
    // are fetched 4 at a time so each lane keeps 4 independent 16-B loads in flight.
    const int cnt = (int)(s1 - s0);
    const int myidx = lane < cnt ? gidx[s0 + lane] : 0;
    const float4* tb = reinterpret_cast<const float4*>(t) + lane;
    const int64_t ld4 = ldt >> 2;
    float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
    if (cnt > 0) {
      m = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      for (int j = 0; j < cnt; j += 4) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int jj = j + u < cnt ? j + u : j;  // duplicate a valid row: max is idempotent
          const int src = __shfl_sync(0xffffffffu, myidx, jj);
          v[u] = __ldg(tb + (int64_t)src * ld4);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          m.x = fmaxf(m.x, v[u].x);
          m.y = fmaxf(m.y, v[u].y);
          m.z = fmaxf(m.z, v[u].z);
          m.w = fmaxf(m.w, v[u].w);
        }
      }
    }
    reinterpret_cast<float4*>(out + r * ldo)[lane] = m;
  } else if ((D & 3) == 0 && (ldt & 3) == 0 && (ldo & 3) == 0) {
    int D4 = D >> 2;
    for (int c4 = lane; c4 < D4; c4 += 32) {
      float4 m = make_float4(0.f, 0.f, 0.f, 0.f);
      if (s1 > s0) {
        m = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        for (int64_t j = s0; j < s1; ++j) {
          float4 v = __ldg(reinterpret_cast<const float4*>(t + (int64_t)gidx[j] * ldt) + c4);
          m.x = fmaxf(m.x, v.x);
          m.y = fmaxf(m.y, v.y);
          m.z = fmaxf(m.z, v.z);
          m.w = fmaxf(m.w, v.w);
        }
      }
      reinterpret_cast<float4*>(out + r * ldo)[c4] = m;
    }
  } else {
    for (int c = lane; c < D; c += 32) {
      float m = 0.f;
      if (s1 > s0) {
        m = -INFINITY;
        for (int64_t j = s0; j < s1; ++j) m = fmaxf(m, t[(int64_t)gidx[j] * ldt + c]);
      }
      out[r * ldo + c] = m;
    }
  }
}

void segment_max(const float* t, int64_t ldt, const GraphView* views_dev,
                 const int64_t* row_off_dev, const int64_t* gbase_dev, const int32_t* row_fwd,
                 const int32_t* gidx, int64_t R, int D, float* out, int64_t ldo,
                 cudaStream_t st, int32_t* argmax) {
  if (R <= 0) return;
  segment_max_kernel<<<(unsigned)cdiv(R, 8), 256, 0, st>>>(t, ldt, views_dev, row_off_dev,
                                                           gbase_dev, row_fwd, gidx, R, D, out,
                                                           ldo, argmax);
  LAUNCH_CHECK();
}

// node id of every batch row (for node-indexed action scatter)
__global__ void row_node_kernel(const GraphView* __restrict__ views,
                                const int64_t* __restrict__ row_off,
                                const int32_t* __restrict__ row_fwd, int64_t R,
                                int32_t* __restrict__ row_node) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  int f = row_fwd[r];
  const int32_t* ord = views[f].order;
  row_node[r] = ord ? ord[r - row_off[f]] : (int32_t)(r - row_off[f]);
}

void row_node_fill(const GraphView* views_dev, const int64_t* row_off_dev,
                   const int32_t* row_fwd, int64_t R, int32_t* row_node, cudaStream_t st) {
  if (R <= 0) return;
  row_node_kernel<<<(unsigned)cdiv(R, 256), 256, 0, st>>>(views_dev, row_off_dev, row_fwd, R,
                                                          row_node);
  LAUNCH_CHECK();
}

}  // namespace go

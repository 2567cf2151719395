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
                                       int32_t* __restrict__ gidx, int32_t* __restrict__ segoff) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  int f = row_fwd[r];
  const GraphView& G = views[f];
  int64_t base = row_off[f];
  int64_t lr = r - base;
  if (segoff) {  // flat segment bounds (forwards are contiguous in gidx)
    if (r == 0) segoff[0] = 0;
    segoff[r + 1] = (int32_t)(gbase[f] + G.samp_off[lr + 1]);
  }
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
                     int32_t* segoff, cudaStream_t st) {
  (void)F;
  if (total_rows <= 0) return;
  if (k > 32) GO_THROW(GO_ERR_UNSUPPORTED, "gs_knn %d > 32", k);
  neighbor_sample_kernel<<<(unsigned)cdiv(total_rows, 128), 128, 0, st>>>(
      views_dev, row_off_dev, gbase_dev, seeds_dev, row_fwd, total_rows, k, gidx, segoff);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// h0 = node_features @ embed/in_w + in_b (graph.py:268-313 + embedding.py:86).
// The feature row is sparse: one-hot op (12), log1p(flops), log1p(bytes), in/out
// degree, and one prev-action one-hot per task; the affine is a sum of <= 5+T
// weight rows.  task_col[t] = feature column of task t's action block.
// One warp per feature row: the row's metadata (forward, op, the 4 static features, the
// previous actions) is loaded once per warp and each lane produces 4 output columns as
// a float4 (D % 4 == 0, D <= 128 * k handled by the column loop); W rows are L1-resident.
// Four rows per warp (8 lanes per row, each lane a column quad every 8): the row's chain
// of dependent metadata loads (forward -> view -> static features / op / node -> previous
// actions) is shared by 4x more output, which is what bounded the warp-per-row form.
__global__ void features_inproj_kernel(const GraphView* __restrict__ views,
                                       const int64_t* __restrict__ row_off,
                                       const int32_t* __restrict__ row_fwd, int64_t R,
                                       const int32_t* __restrict__ prev, int T,
                                       int tc0, int tc1, int tc2,
                                       const float* __restrict__ W, const float* __restrict__ b,
                                       int D, float* __restrict__ h, int64_t ldh) {
  const int lane = threadIdx.x & 31, q = lane & 7;
  const int64_t r = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 4 + (lane >> 3);
  if (r >= R) return;
  const int f = row_fwd[r];
  const GraphView& G = views[f];
  const int64_t lr = r - row_off[f];
  const float4 s4 = *reinterpret_cast<const float4*>(G.static4 + lr * 4);
  const int op = G.op_row[lr];
  int arow[3] = {0, 0, 0};
  const int TP = prev ? T : 0;  // no previous actions on the first iteration
  if (prev) {
    const int node = G.order[lr];
    const int tcs[3] = {tc0, tc1, tc2};
    for (int t = 0; t < T; ++t) arow[t] = tcs[t] + prev[(int64_t)t * R + row_off[f] + node];
  }
  const int D4 = D >> 2;
  const float4* W4 = reinterpret_cast<const float4*>(W);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  float4* h4 = reinterpret_cast<float4*>(h + r * ldh);
  for (int c = q; c < D4; c += 8) {
    float4 acc = W4[(int64_t)op * D4 + c];
    const float4 w12 = W4[(int64_t)12 * D4 + c], w13 = W4[(int64_t)13 * D4 + c];
    const float4 w14 = W4[(int64_t)14 * D4 + c], w15 = W4[(int64_t)15 * D4 + c];
    acc.x = fmaf(s4.x, w12.x, acc.x); acc.y = fmaf(s4.x, w12.y, acc.y);
    acc.z = fmaf(s4.x, w12.z, acc.z); acc.w = fmaf(s4.x, w12.w, acc.w);
    acc.x = fmaf(s4.y, w13.x, acc.x); acc.y = fmaf(s4.y, w13.y, acc.y);
    acc.z = fmaf(s4.y, w13.z, acc.z); acc.w = fmaf(s4.y, w13.w, acc.w);
    acc.x = fmaf(s4.z, w14.x, acc.x); acc.y = fmaf(s4.z, w14.y, acc.y);
    acc.z = fmaf(s4.z, w14.z, acc.z); acc.w = fmaf(s4.z, w14.w, acc.w);
    acc.x = fmaf(s4.w, w15.x, acc.x); acc.y = fmaf(s4.w, w15.y, acc.y);
    acc.z = fmaf(s4.w, w15.z, acc.z); acc.w = fmaf(s4.w, w15.w, acc.w);
    for (int t = 0; t < TP; ++t) {
      const float4 wa = W4[(int64_t)arow[t] * D4 + c];
      acc.x += wa.x; acc.y += wa.y; acc.z += wa.z; acc.w += wa.w;
    }
    const float4 bb = b4[c];
    h4[c] = make_float4(acc.x + bb.x, acc.y + bb.y, acc.z + bb.z, acc.w + bb.w);
  }
}

// Scalar form (one thread per output element) for widths that are not multiples of 4.
__global__ void features_inproj_scalar_kernel(const GraphView* __restrict__ views,
                                              const int64_t* __restrict__ row_off,
                                              const int32_t* __restrict__ row_fwd, int64_t R,
                                              const int32_t* __restrict__ prev, int T,
                                              int tc0, int tc1, int tc2,
                                              const float* __restrict__ W,
                                              const float* __restrict__ b, int D,
                                              float* __restrict__ h, int64_t ldh) {
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
  const bool vec = D % 4 == 0 && ldh % 4 == 0 && ((uintptr_t)in_w & 15) == 0 &&
                   ((uintptr_t)in_b & 15) == 0 && ((uintptr_t)h & 15) == 0;
  if (!vec) {
    features_inproj_scalar_kernel<<<(unsigned)cdiv(R * D, 256), 256, 0, st>>>(
        views_dev, row_off_dev, row_fwd, R, prev_actions, num_tasks, task_col[0], task_col[1],
        task_col[2], in_w, in_b, D, h, ldh);
    LAUNCH_CHECK();
    return;
  }
  features_inproj_kernel<<<(unsigned)cdiv(R, 32), 256, 0, st>>>(
      views_dev, row_off_dev, row_fwd, R, prev_actions, num_tasks, task_col[0], task_col[1],
      task_col[2], in_w, in_b, D, h, ldh);
  LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------------
// pooled[r] = max over sampled neighbours j of t[j] (tensor.py:199-263 gather_rows +
// segment_max; empty segment -> 0).  This is the HBM-bound GraphSAGE aggregation
// (SURVEY.md §8 A6).  segoff[R+1] holds the flat segment bounds into gidx.
//
// D == 128 fast path: 8 lanes per row (4 rows per warp), each lane owning 4 float4
// columns, so one load instruction of an 8-lane group reads a full 128-B line; the
// neighbour indices are fetched once and shuffled, and 4 neighbours x 4 column
// slices = 16 independent 16-B loads are in flight per lane.
// SIGMOID: the gathered rows are pre-activations and the output is sigmoid(max) --
// equal to max(sigmoid) because sigmoid is monotone (embedding.py:90-91), but applied
// to N pooled rows here instead of inside the producing GEMM's epilogue.
template <bool SIGMOID>
__global__ void segment_max128_kernel(const float* __restrict__ t, int64_t ldt,
                                      const int32_t* __restrict__ segoff,
                                      const int32_t* __restrict__ gidx, int64_t R,
                                      float* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane & 24;
  const int64_t r = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 4 + (lane >> 3);
  const bool live = r < R;
  const int s0 = live ? segoff[r] : 0, s1 = live ? segoff[r + 1] : 0;
  const int cnt = s1 - s0;
  const float4* tb = reinterpret_cast<const float4*>(t) + sub;
  const int64_t ld4 = ldt >> 2;
  float4 m[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) m[q] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
  for (int j0 = 0; __any_sync(0xffffffffu, j0 < cnt); j0 += 8) {
    const int myidx = (j0 + sub < cnt) ? gidx[s0 + j0 + sub] : -1;
#pragma unroll
    for (int jb = 0; jb < 8; jb += 4) {
      float4 v[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int src = __shfl_sync(0xffffffffu, myidx, grp + jb + u);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          v[u][q] = src >= 0 ? __ldg(tb + (int64_t)src * ld4 + 8 * q)
                             : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          m[q].x = fmaxf(m[q].x, v[u][q].x);
          m[q].y = fmaxf(m[q].y, v[u][q].y);
          m[q].z = fmaxf(m[q].z, v[u][q].z);
          m[q].w = fmaxf(m[q].w, v[u][q].w);
        }
    }
  }
  if (!live) return;
  if (SIGMOID) {
    auto sg = [](float x) { return 1.f / (1.f + expf(-x)); };
#pragma unroll
    for (int q = 0; q < 4; ++q) m[q] = make_float4(sg(m[q].x), sg(m[q].y), sg(m[q].z), sg(m[q].w));
  }
  float4* o = reinterpret_cast<float4*>(out + r * ldo) + sub;
#pragma unroll
  for (int q = 0; q < 4; ++q) o[8 * q] = cnt > 0 ? m[q] : make_float4(0.f, 0.f, 0.f, 0.f);
}

// General D (and the training forward, which also records the first maximal row per
// column, tensor.py:240-251): one warp per row.
__global__ void segment_max_kernel(const float* __restrict__ t, int64_t ldt,
                                   const int32_t* __restrict__ segoff,
                                   const int32_t* __restrict__ gidx, int64_t R, int D,
                                   float* __restrict__ out, int64_t ldo,
                                   int32_t* __restrict__ argmax) {
  int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (r >= R) return;
  const int64_t s0 = segoff[r], s1 = segoff[r + 1];
  if (argmax) {
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
  if ((D & 3) == 0 && (ldt & 3) == 0 && (ldo & 3) == 0) {
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

void segment_max(const float* t, int64_t ldt, const int32_t* segoff, const int32_t* gidx,
                 int64_t R, int D, float* out, int64_t ldo, cudaStream_t st, int32_t* argmax,
                 bool sigmoid_of_max) {
  if (R <= 0) return;
  const bool aligned = ((uintptr_t)t % 16 == 0) && ((uintptr_t)out % 16 == 0) &&
                       (ldt & 3) == 0 && (ldo & 3) == 0;
  if (sigmoid_of_max) {
    GO_CHECK(!argmax && D == 128 && aligned, "sigmoid-of-max needs the D=128 fast path");
    segment_max128_kernel<true><<<(unsigned)cdiv(R, 32), 256, 0, st>>>(t, ldt, segoff, gidx, R,
                                                                       out, ldo);
  } else if (!argmax && D == 128 && aligned) {
    segment_max128_kernel<false><<<(unsigned)cdiv(R, 32), 256, 0, st>>>(t, ldt, segoff, gidx, R,
                                                                        out, ldo);
  } else {
    segment_max_kernel<<<(unsigned)cdiv(R, 8), 256, 0, st>>>(t, ldt, segoff, gidx, R, D, out,
                                                             ldo, argmax);
  }
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

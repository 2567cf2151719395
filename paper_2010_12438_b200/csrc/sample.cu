// Per-row categorical sampling (policy.py:220-237) in float64 with numpy's exact
// operation order, fed by the reference's PCG64 uniform stream (policy.py:288,
// 299-306: one rng per iterate_decisions call, draws consumed (iteration, task,
// row)-major).  Compiled with -fmad=false so no a*b+c is contracted.
#include "engine.cuh"
#include "rng.cuh"

namespace go {

constexpr int SMAX = 32;  // max actions per task

// numpy pairwise_sum for n <= 128 (loops_utils.h.src): < 8 sequential from 0.0,
// else 8 accumulators + ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) + sequential tail.
__device__ inline double np_sum(const double* x, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, x[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = x[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], x[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, x[i]);
  return res;
}

__global__ void sample_kernel(const void* __restrict__ logits, int f64, int64_t ldl, int a,
                              int64_t R, const int64_t* __restrict__ row_off,
                              const int32_t* __restrict__ row_fwd,
                              const int32_t* __restrict__ row_node,
                              const uint64_t* __restrict__ pcg, int64_t task,
                              double temperature, int32_t* __restrict__ actions,
                              double* __restrict__ logp_out, bool shared) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  int f = row_fwd[r];
  int64_t base = row_off[f];
  int64_t lr = r - base, nf = row_off[f + 1] - base;
  double z[SMAX];
  const int64_t lrow = shared ? lr : r;  // shared: every forward reads forward 0's rows
  for (int j = 0; j < a; ++j)
    z[j] = f64 ? ((const double*)logits)[lrow * ldl + j]
               : (double)((const float*)logits)[lrow * ldl + j];
  int act = 0;
  double lp = 0.0;
  if (temperature == 0.0) {
    // np.argmax: first maximal index (policy.py:228-230)
    double best = z[0];
    for (int j = 1; j < a; ++j)
      if (z[j] > best) {
        best = z[j];
        act = j;
      }
  } else {
    double mx = -INFINITY;
    for (int j = 0; j < a; ++j) {
      z[j] = __ddiv_rn(z[j], temperature);
      mx = j == 0 ? z[j] : fmax(mx, z[j]);
    }
    double e[SMAX];
    for (int j = 0; j < a; ++j) {
      z[j] = __dsub_rn(z[j], mx);
      e[j] = exp(z[j]);
    }
    double lse = log(np_sum(e, a));
    double cum[SMAX];
    double c = 0.0;
    for (int j = 0; j < a; ++j) {
      z[j] = __dsub_rn(z[j], lse);  // logp
      c = (j == 0) ? exp(z[j]) : __dadd_rn(c, exp(z[j]));
      cum[j] = c;
    }
    Pcg64 g;
    const uint64_t* ps = pcg + 4 * (int64_t)f;
    g.state = ((u128)ps[0] << 64) | ps[1];
    g.inc = ((u128)ps[2] << 64) | ps[3];
    g.has32 = false;
    g.advance((uint64_t)(task * nf + lr));
    double u = __dmul_rn(g.random(), cum[a - 1]);
    for (int j = 0; j < a; ++j) act += (u > cum[j]) ? 1 : 0;
    lp = z[act];
  }
  actions[base + row_node[r]] = act;
  logp_out[r] = lp;
}

void sample_rows(const void* logits, int logits_f64, int64_t ldl, int a, int64_t R,
                 const int64_t* row_off_dev, const int32_t* row_fwd, const int32_t* row_node,
                 const uint64_t* pcg_dev, int64_t task, double temperature,
                 int32_t* actions, double* logp, cudaStream_t st, bool shared) {
  if (R <= 0) return;
  if (a < 1 || a > SMAX) GO_THROW(GO_ERR_UNSUPPORTED, "action space %d outside [1, %d]", a, SMAX);
  sample_kernel<<<(unsigned)cdiv(R, 128), 128, 0, st>>>(logits, logits_f64, ldl, a, R,
                                                        row_off_dev, row_fwd, row_node,
                                                        pcg_dev, task, temperature,
                                                        actions, logp, shared);
  LAUNCH_CHECK();
}

}  // namespace go

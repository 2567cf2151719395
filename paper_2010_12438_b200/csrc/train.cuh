// Declarations shared by the PPO backward (train.cu, train_kernels.cu).
#pragma once
#include "engine.cuh"

namespace go {

// key tile for the attention backward: keys [k0,k1) receive gradient from queries in
// [qa0,qa1) ("self") and [qb0,qb1) ("cache": the next trunk segment, whose K/V rows
// are gradient-stopped inputs, policy.py:169-174 -- weights only).
struct KvTile {
  int64_t k0, k1, qa0, qa1, qb0, qb1;
};

// gradient pointers of one transformer block (policy/mod/ here)
struct BlockG {
  float *v_w, *v_b, *o_w, *o_b, *ln1_g, *ln1_b, *w1, *b1, *w2, *b2, *ln2_g, *ln2_b;
};

void dgemm_nt(const float* dY, int64_t ldd, const float* W, int64_t ldw, float* dX, int64_t ldx,
              int64_t M, int Kin, int Nout, bool accumulate, cudaStream_t st);
void transpose(const float* W, int64_t ldw, int rows, int cols, float* out, cudaStream_t st);
void wgrad(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
           const float* dY, int64_t ldd, int64_t M, int N, float* dW, float* db, cudaStream_t st);
void wgrad_tc(const float* A1, int64_t lda1, int K1, const float* A2, int64_t lda2, int K2,
              const float* dY, int64_t ldd, int64_t M, int N, float* dW, float* db,
              cudaStream_t st);
void ln_backward(const float* u, int64_t ldu, const float* g, const float* dout, int64_t ldd,
                 float* dx, int64_t ldx, bool accumulate, int64_t M, int D, float* dg, float* db,
                 cudaStream_t st);
void act_backward(float* d, int64_t ldd, const float* y, int64_t ldy, int64_t M, int D, int act,
                  cudaStream_t st);
void add_into(float* a, int64_t lda, const float* b, int64_t ldb, int64_t M, int D,
              cudaStream_t st);
void segmax_backward(const float* dpool, int64_t ldp, const int32_t* arg, int64_t M, int D,
                     float* dt, int64_t ldt, cudaStream_t st);
void rowvec_backward(const float* dxm, int64_t ldd, const float* x, int64_t ldx, const float* mod,
                     const int32_t* row_fwd, float* dx, int64_t ldo, float* dmod, int64_t M, int D,
                     cudaStream_t st);
void mean_backward(float* dh, int64_t ldh, const float* dG, const int64_t* row_off,
                   const int32_t* row_fwd, int64_t M, int D, cudaStream_t st);
void attention_backward(const float* q, const float* k, const float* v, const float* O,
                        const float* dO, int64_t ld, const float* lse, int n_head, int d_head,
                        const AttnTile* qtiles, int64_t nq, const KvTile* ktiles, int64_t nk,
                        float* Dbuf, int64_t M, float* dq, float* dk_a, float* dv_a, float* dk_b,
                        float* dv_b, cudaStream_t st);
void attention_backward_D(const float* dO, const float* O, int64_t ld, int n_head, int d_head,
                          int64_t M, float* Dbuf, cudaStream_t st);
// the fp32 SIMT dq / dk,dv kernels alone (D already in Dbuf); gate: run only if *gate != 0
void attention_backward_simt(const float* q, const float* k, const float* v, const float* dO,
                             int64_t ld, const float* lse, int n_head, int d_head,
                             const AttnTile* qtiles, int64_t nq, const KvTile* ktiles, int64_t nk,
                             const float* Dbuf, float* dq, float* dk_a, float* dv_a, float* dk_b,
                             float* dv_b, const int32_t* gate, cudaStream_t st);
// tensor-core (split-fp16 mma.sync) forward with lse over packed operands (rows 0..M-1,
// d_head <= 15); scratch as for attention_backward_mma; *flag set on fp16 range overflow
void attention_forward_mma(const float* q, const float* k, const float* v, int64_t ld,
                           int n_head, int d_head, const AttnTile* tiles, int64_t nt, int64_t M,
                           float* out, int64_t ldo, float* lse, void* scratch, int32_t* flag,
                           cudaStream_t st, const int32_t* gate = nullptr);
// tensor-core (mma.sync fp16) backward, d_head <= 16, with the gated SIMT re-run
// (csrc/attn_bwd_mma.cu); scratch >= attention_backward_mma_scratch(M, n_head) bytes
size_t attention_backward_mma_scratch(int64_t M, int n_head);
// PPO tape head attention on tcgen05 (tc_tape.cu): forward with log2-sum-exp.  No host
// synchronisation: returns a device flag that is non-zero when the fp16 split path could not
// take the call (bound or range; the tcgen05 kernels then write nothing) -- pass it as the
// `gate` of the mma.sync path, whose kernels run only then.
size_t tape_attention_tc_scratch(int64_t R, int F, int n_head);
const int32_t* tape_attention_fwd_tc(const float* q, const float* k, const float* v, int64_t ld,
                           int n_head, int d_head, int64_t R, int F, const TcWork* works_dev,
                           int64_t num_works, const int64_t* tile_row0_dev,
                           const int32_t* tile_n_dev, int64_t Ttot, const int32_t* row_fwd,
                           float* out, int64_t ldo, float* lse, void* scratch,
                           cudaStream_t st);
// backward (dq, dk, dv; D into Dbuf); device flag as for the forward
const int32_t* tape_attention_bwd_tc(const float* q, const float* k, const float* v, const float* O,
                           const float* dO, int64_t ld, int n_head, int d_head, int64_t R,
                           int F, const float* lse, const TcWork* kv_works_dev,
                           int64_t num_kv_works, const TcWork* q_works_dev,
                           int64_t num_q_works, const int64_t* tile_row0_dev,
                           const int32_t* tile_n_dev, int64_t Ttot, float* Dbuf, float* dq,
                           float* dk, float* dv, void* scratch, cudaStream_t st);
void attention_backward_mma(const float* q, const float* k, const float* v, const float* O,
                            const float* dO, int64_t ld, const float* lse, int n_head,
                            int d_head, const AttnTile* qtiles, int64_t nq, const KvTile* ktiles,
                            int64_t nk, float* Dbuf, int64_t M, float* dq, float* dk_a,
                            float* dv_a, float* dk_b, float* dv_b, void* scratch,
                            int32_t* flag, cudaStream_t st, const int32_t* gate = nullptr);
void ppo_loss(const float* logits, int a, int64_t R, const int32_t* actions,
              const int32_t* row_node, const double* old_logp, const int32_t* row_fwd,
              const int64_t* row_off, const double* fparams, double eps, double c_ent, int T,
              int C, int t_index, float* dlogits, double* stats, cudaStream_t st);
void value_backward(const float* value, const float* mean, const double* rewards, int F, int D,
                    double c_v, int C, const float* vw, float* dvalue, float* dvw, float* dvb,
                    double* vstats, float* drep, int64_t ldr, const int64_t* row_off,
                    const int32_t* row_fwd, int64_t M, cudaStream_t st);
void inproj_wgrad(const GraphView* views, const int64_t* row_off, const int32_t* row_fwd,
                  int64_t R, const int32_t* prev, int T, const int32_t* tcol, const float* dh,
                  int64_t ldh, int D, int Fdim, float* dW, float* db, cudaStream_t st);
void modulate_backward(const float* ge, int F, int gs, const float* in_w, const float* in_b,
                       const BlockW& w, int dm, int wd, int di, const float* dmod, float* dge,
                       const BlockG& gr, float* d_in_w, float* d_in_b, cudaStream_t st);
void adam64(double* p, float* p32, const float* g, double* m, double* v, int64_t n, double lr,
            double b1, double b2, double eps, int64_t step, cudaStream_t st);
void adam(float* p, const float* g, float* m, float* v, int64_t n, double lr, double b1,
          double b2, double eps, int64_t step, cudaStream_t st);

}  // namespace go

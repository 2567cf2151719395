// Exact batched discrete-event simulation (simulator.py:280-441) + reward
// (training.py:37-44).  One thread simulates one placement; K placements run in
// parallel.  Compiled with -fmad=false; all float64 arithmetic is explicit IEEE
// round-to-nearest (__dadd_rn / __ddiv_rn), so makespans, busy times and memory
// peaks are bit-identical to the reference.
//
// Reference semantics reproduced:
//  * in-flight events: at most one compute per device and one transfer per link, so
//    the event heap's (time, kind, dev|src, i|dst, seq) order reduces to
//    (time, slot) with slot = dev for computes and D + src*D + dst for transfers;
//    all events at the minimum time form one batch, processed in slot order;
//    zero-duration events created by schedule() form the next batch.
//  * ready queue per device: min-heap on (-priority, ready_time, topo_index) or
//    (ready_time, topo_index) for FIFO (topo_index is unique).
//  * schedule(t): links in sorted (src, dst) order pop FIFO if idle, then devices
//    0..D-1 pop their queue if idle; busy[dev] += kernel_time.
//  * memory: (finish, +b) and (last-consumer finish, -b) events swept in
//    (time, kind, delta) order; processed online per time group (allocs before
//    frees; exact sorted order when byte values are not all integral).
#include <algorithm>
#include <cstring>

#include "engine.cuh"
#include "rng.cuh"

namespace go {

constexpr int DES_MAXD = 16;
constexpr double DINF = __builtin_huge_val();

struct HeapEnt {
  double rt;
  int32_t topo;
  int32_t grp;
  int32_t npri;  // -priority (0 for FIFO)
  int32_t pad;
};

__device__ __forceinline__ bool heap_less(const HeapEnt& a, const HeapEnt& b) {
  if (a.npri != b.npri) return a.npri < b.npri;
  if (a.rt != b.rt) return a.rt < b.rt;
  return a.topo < b.topo;
}

struct LinkEnt {
  int32_t edge;
  int32_t grp;
};

// Per-placement dynamic state of one group: pending in-edges, remaining consumers (<< 5)
// with the group's device in the low 5 bits, -priority (0 for FIFO) and the topo index --
// everything mark_ready / deliver / the memory sweep need, in one 16-B load.
struct DesNodeState {
  int32_t pend;
  int32_t remdev;
  int32_t npri;
  int32_t topo;
};

struct DesCaps {
  int64_t cq;  // ready-heap capacity per device
  int64_t cl;  // FIFO capacity per link
  int64_t cm;  // exact-mode memory list capacity per device
  // group states, ready heaps, link FIFOs, memory lists
  __host__ __device__ int64_t heap_offset(int G) const { return round_up((int64_t)G * 16, 16); }
  int64_t per_placement_bytes(int G, int d) const {
    int64_t b = heap_offset(G) + (int64_t)d * cq * sizeof(HeapEnt);
    b += (int64_t)d * d * cl * sizeof(LinkEnt);
    b += 2 * (int64_t)d * cm * sizeof(double);
    return round_up(b, 256);
  }
};

// group states for one placement (simulator.py:320-330 initial pending counts / devices /
// priorities); lane `l0` of `nl` cooperating threads
__device__ __forceinline__ void des_init_states(const DesView& V, const int32_t* __restrict__ pl,
                                                const int32_t* __restrict__ pr, int policy,
                                                DesNodeState* st, int l0, int nl) {
  for (int g = l0; g < V.G; g += nl) {
    const int4 r = *reinterpret_cast<const int4*>(&V.grec[g].topo);  // topo, rep, pend0, nsucc
    DesNodeState x;
    x.pend = r.z;
    x.remdev = (r.w << 5) | pl[r.y];
    x.npri = policy == 0 ? -pr[r.y] : 0;
    x.topo = r.x;
    st[g] = x;
  }
}

enum { ST_OK = 0, ST_OVERFLOW = 1, ST_DEADLOCK = 2, ST_MEMLIST = 3 };

// Optional event log (simulate(record_trace=True), simulator.py:61-67, 360-373): one
// record per started compute (kind 0, a = device) and per started transfer (kind 1,
// a -> b the link), in the order schedule() starts them; the host sorts them the way
// the reference does (simulator.py:432-433).
struct DesTraceLog {
  DesTraceRec* rec;  // capacity cap; nullptr: no trace
  int64_t cap;
  int64_t* count;
};

template <int M>
struct DesState {
  double dev_t[M];
  double busy[M], cur[M], pk[M], acc_a[M], acc_f[M];
  double link_t[M * M];
  int32_t dev_g[M], hs[M], na[M], nf[M];
  int32_t link_g[M * M], lq_h[M * M], lq_n[M * M];
  uint64_t lmask[(M * M + 63) / 64];
  uint64_t amask[(M * M + 63) / 64];  // links with a transfer in flight
};

// One placement's simulation: the reference's event loop (simulator.py:320-441) run by
// one thread.  S (the per-placement device / link state) lives in shared memory when
// the block is one placement (warp mode) -- local memory is interleaved across the
// warp's 32 threads, so a single active lane pulled a whole 128-B line per word and
// the warps' frames thrashed L1; `base` is this placement's global scratch (pending
// counts, ready heaps, link FIFOs, memory lists).  Returns the status; step time and
// violation (0 none, 1 colocation, 2 oom) through the references, busy / peak in S.
// MAXD: compile-time bound on the device count (4 / 8 / 16): sizing the link arrays
// for 8 devices (64 links instead of 256) took 4,096 random cfg4 placements from 2.14
// to 1.45 s before the state moved to shared memory (0.56 s).
template <int MAXD>
__device__ int des_run(const DesView& V, const int32_t* __restrict__ pl,
                       const int32_t* __restrict__ pr, int d, const double* __restrict__ peakf,
                       const double* __restrict__ mbw, const double* __restrict__ cap,
                       const double* __restrict__ lbw, int policy, DesCaps caps, char* base,
                       DesState<MAXD>& S, DesTraceLog tr, double& step, int8_t& viol_out,
                       bool states_ready = false, const double* __restrict__ ctab = nullptr,
                       const double* __restrict__ etab = nullptr) {
  const int G = V.G;
  DesNodeState* gst = reinterpret_cast<DesNodeState*>(base);
  HeapEnt* heaps = reinterpret_cast<HeapEnt*>(base + caps.heap_offset(G));
  LinkEnt* lq = reinterpret_cast<LinkEnt*>(heaps + (int64_t)d * caps.cq);
  double* mlist = reinterpret_cast<double*>(lq + (int64_t)d * d * caps.cl);
  // the caller's warp may have filled the states already (des_kernel)
  if (!states_ready) des_init_states(V, pl, pr, policy, gst, 0, 1);
  auto gdev = [&](int g) { return gst[g].remdev & 31; };
  int64_t n_trace = 0;  // events logged (the single-placement trace launch only)
  auto log_event = [&](double t0, double t1, int kind, int a, int b, int g) {
    if (tr.rec && n_trace < tr.cap) tr.rec[n_trace] = DesTraceRec{t0, t1, kind, a, b, g};
    ++n_trace;
  };

  // colocation (simulator.py:308-315): checked on group devices, simulation continues
  int8_t viol = 0;
  for (int c = 0; c < V.num_coloc && !viol; ++c) {
    int d0 = gdev(V.coloc_grp[V.coloc_off[c]]);
    for (int64_t j = V.coloc_off[c] + 1; j < V.coloc_off[c + 1]; ++j)
      if (gdev(V.coloc_grp[j]) != d0) {
        viol = 1;
        break;
      }
  }

  auto& dev_t = S.dev_t;
  auto& dev_g = S.dev_g;
  auto& hs = S.hs;
  auto& busy = S.busy;
  auto& cur = S.cur;
  auto& pk = S.pk;
  auto& acc_a = S.acc_a;
  auto& acc_f = S.acc_f;
  auto& na = S.na;
  auto& nf = S.nf;
  auto& link_t = S.link_t;
  auto& link_g = S.link_g;
  auto& lq_h = S.lq_h;
  auto& lq_n = S.lq_n;
  auto& lmask = S.lmask;
  auto& amask = S.amask;
  for (int i = 0; i < d; ++i) {
    dev_t[i] = DINF;
    dev_g[i] = -1;
    hs[i] = 0;
    busy[i] = 0.0;
    cur[i] = 0.0;
    pk[i] = 0.0;
    acc_a[i] = 0.0;
    acc_f[i] = 0.0;
    na[i] = nf[i] = 0;
  }
  const int L = d * d;
  for (int s = 0; s < L; ++s) {
    link_t[s] = DINF;
    link_g[s] = -1;
    lq_h[s] = 0;
    lq_n[s] = 0;
  }
  for (int w = 0; w < (L + 63) / 64; ++w) lmask[w] = amask[w] = 0;
  uint32_t dmask = 0;  // devices with a non-empty ready heap
  int status = ST_OK;

  auto heap_push = [&](int dev, const HeapEnt& e) {
    if (hs[dev] >= caps.cq) {
      status = ST_OVERFLOW;
      return;
    }
    HeapEnt* h = heaps + (int64_t)dev * caps.cq;
    int p = hs[dev]++;
    while (p > 0) {
      int q = (p - 1) >> 1;
      if (!heap_less(e, h[q])) break;
      h[p] = h[q];
      p = q;
    }
    h[p] = e;
    dmask |= 1u << dev;
  };
  auto heap_pop = [&](int dev) {
    HeapEnt* h = heaps + (int64_t)dev * caps.cq;
    HeapEnt top = h[0];
    int n = --hs[dev];
    if (n > 0) {
      HeapEnt last = h[n];
      int p = 0;
      while (true) {
        int c = 2 * p + 1;
        if (c >= n) break;
        if (c + 1 < n && heap_less(h[c + 1], h[c])) ++c;
        if (!heap_less(h[c], last)) break;
        h[p] = h[c];
        p = c;
      }
      h[p] = last;
    } else {
      dmask &= ~(1u << dev);
    }
    return top;
  };
  auto deliver = [&](int g, double t) {
    DesNodeState x = gst[g];
    gst[g].pend = --x.pend;
    if (x.pend == 0) {
      HeapEnt e;
      e.rt = t;
      e.topo = x.topo;
      e.grp = g;
      e.npri = x.npri;
      e.pad = 0;
      heap_push(x.remdev & 31, e);
    }
  };
  const bool exact_int = V.mem_int_exact != 0;
  uint32_t mdirty = 0;  // devices with allocs / frees queued in the current time group
  auto mem_add = [&](int dev, double b, bool alloc) {
    mdirty |= 1u << dev;
    if (exact_int) {
      if (alloc) acc_a[dev] = __dadd_rn(acc_a[dev], b);
      else acc_f[dev] = __dadd_rn(acc_f[dev], b);
      if (alloc) na[dev]++;
      else nf[dev]++;
      return;
    }
    double* lst = mlist + ((int64_t)dev * 2 + (alloc ? 0 : 1)) * caps.cm;
    int32_t& n = alloc ? na[dev] : nf[dev];
    if (n >= caps.cm) {
      status = ST_MEMLIST;
      return;
    }
    // keep sorted by delta ascending: allocs ascending b, frees descending b
    int p = n++;
    while (p > 0 && (alloc ? lst[p - 1] > b : lst[p - 1] < b)) {
      lst[p] = lst[p - 1];
      --p;
    }
    lst[p] = b;
  };
  auto mem_flush = [&]() {
    for (uint32_t m = mdirty; m; m &= m - 1) {  // ascending device order
      const int dev = __ffs(m) - 1;
      if (na[dev] == 0 && nf[dev] == 0) continue;
      if (exact_int) {
        double c = __dadd_rn(cur[dev], acc_a[dev]);
        if (na[dev]) pk[dev] = fmax(pk[dev], c);
        cur[dev] = __dsub_rn(c, acc_f[dev]);
        acc_a[dev] = acc_f[dev] = 0.0;
      } else {
        double* la = mlist + ((int64_t)dev * 2) * caps.cm;
        double* lf = la + caps.cm;
        for (int i = 0; i < na[dev]; ++i) {
          cur[dev] = __dadd_rn(cur[dev], la[i]);
          pk[dev] = fmax(pk[dev], cur[dev]);
        }
        for (int i = 0; i < nf[dev]; ++i) cur[dev] = __dadd_rn(cur[dev], -lf[i]);
      }
      na[dev] = nf[dev] = 0;
    }
    mdirty = 0;
  };

  // groups without external in-edges (host-built list, index order) start ready
  for (int i = 0; i < V.num_src && status == ST_OK; ++i) {
    const int g = V.src_grp[i];
    const DesNodeState x = gst[g];
    HeapEnt e;
    e.rt = 0.0;
    e.topo = x.topo;
    e.grp = g;
    e.npri = x.npri;
    e.pad = 0;
    heap_push(x.remdev & 31, e);
  }

  auto schedule = [&](double t) {
    for (int w = 0; w < (L + 63) / 64; ++w) {
      uint64_t m = lmask[w];
      while (m) {
        int b = __ffsll((long long)m) - 1;
        m &= m - 1;
        int s = w * 64 + b;
        if (link_t[s] != DINF) continue;
        LinkEnt* q = lq + (int64_t)s * caps.cl;
        LinkEnt e = q[lq_h[s]];
        const int32_t nh = lq_h[s] + 1;  // ring wrap without an integer division
        lq_h[s] = nh == (int32_t)caps.cl ? 0 : nh;
        if (--lq_n[s] == 0) lmask[w] &= ~(1ull << b);
        // etab (uniform link bandwidth): the same division, once per edge and launch
        double dt = etab ? etab[e.edge] : __ddiv_rn(V.out_bytes[e.edge], lbw[s]);
        link_t[s] = __dadd_rn(t, dt);
        link_g[s] = e.grp;
        if (tr.rec) log_event(t, link_t[s], 1, s / d, s % d, e.grp);
        amask[w] |= 1ull << b;
      }
    }
    uint32_t m = dmask;
    while (m) {
      int dev = __ffs(m) - 1;
      m &= m - 1;
      if (dev_t[dev] != DINF) continue;
      HeapEnt e = heap_pop(dev);
      int g = e.grp;
      double dt;
      if (ctab) {
        dt = ctab[(int64_t)g * d + dev];  // des_ctab_kernel: the same two divisions
      } else {
        const double2 fb = *reinterpret_cast<const double2*>(&V.grec[g].cost_flops);
        dt = fmax(__ddiv_rn(fb.x, peakf[dev]), __ddiv_rn(fb.y, mbw[dev]));
      }
      // Python max(a, b) returns a unless b > a; fmax agrees for non-NaN inputs
      busy[dev] = __dadd_rn(busy[dev], dt);
      dev_t[dev] = __dadd_rn(t, dt);
      dev_g[dev] = g;
      if (tr.rec) log_event(t, dev_t[dev], 0, dev, -1, g);
    }
  };

  schedule(0.0);
  int done = 0;
  double step_t = 0.0;
  double mem_time = -1.0;
  constexpr int LW = (MAXD * MAXD + 63) / 64;
  while (status == ST_OK) {
    // next event time, with the devices / links that finish exactly then (one pass; the
    // reference pops every event of the minimum time in (time, kind, slot) order)
    double dnow = DINF;
    uint32_t dset = 0;
#pragma unroll
    for (int i = 0; i < MAXD; ++i) {
      if (i < d) {
        const double t = dev_t[i];
        if (t < dnow) {
          dnow = t;
          dset = 1u << i;
        } else if (t == dnow) {
          dset |= 1u << i;
        }
      }
    }
    double lnow = DINF;
    uint64_t lset[LW];
#pragma unroll
    for (int w = 0; w < LW; ++w) {
      lset[w] = 0;
      if (w * 64 < L) {
        for (uint64_t mm = amask[w]; mm; mm &= mm - 1) {
          const int b = __ffsll((long long)mm) - 1;
          const double t = link_t[w * 64 + b];
          if (t < lnow) {
#pragma unroll
            for (int w2 = 0; w2 < LW; ++w2) lset[w2] = 0;
            lnow = t;
            lset[w] = 1ull << b;
          } else if (t == lnow) {
            lset[w] |= 1ull << b;
          }
        }
      }
    }
    const double now = fmin(dnow, lnow);
    if (now == DINF) break;
    if (dnow != now) dset = 0;
    if (lnow != now) {
#pragma unroll
      for (int w = 0; w < LW; ++w) lset[w] = 0;
    }
    if (now != mem_time) {
      mem_flush();
      mem_time = now;
    }
    // computes (kind 0) in device order
    for (uint32_t m = dset; m; m &= m - 1) {
      const int dev = __ffs(m) - 1;
      int g = dev_g[dev];
      dev_t[dev] = DINF;
      dev_g[dev] = -1;
      ++done;
      step_t = now;
      const DesGroupRec& rg = V.grec[g];
      const int4 oc = *reinterpret_cast<const int4*>(&rg.out_off);  // out_off/cnt, pred_off/cnt
      const double b = rg.resident;
      for (int64_t e = oc.x; e < (int64_t)oc.x + oc.y; ++e) {
        int gd = V.out_grp[e];
        int dd = gdev(gd);
        if (dd == dev) {
          deliver(gd, now);
        } else {
          int s = dev * d + dd;
          if (lq_n[s] >= caps.cl) {
            status = ST_OVERFLOW;
            break;
          }
          LinkEnt* q = lq + (int64_t)s * caps.cl;
          int32_t qi = lq_h[s] + lq_n[s];
          if (qi >= (int32_t)caps.cl) qi -= (int32_t)caps.cl;
          q[qi] = LinkEnt{(int32_t)e, gd};
          ++lq_n[s];
          lmask[s >> 6] |= 1ull << (s & 63);
        }
      }
      if (b != 0.0) mem_add(dev, b, true);
      for (int64_t j = oc.z; j < (int64_t)oc.z + oc.w; ++j) {
        int p = V.pred_grp[j];
        const int rd = gst[p].remdev - 32;
        gst[p].remdev = rd;
        if (rd < 32) {
          const double rp = V.grec[p].resident;
          if (rp != 0.0) mem_add(rd & 31, rp, false);
        }
      }
      if (oc.y == 0 && b != 0.0) mem_add(dev, b, false);  // no successors: nsucc == 0
    }
    // transfers (kind 1) in (src, dst) order
#pragma unroll
    for (int w = 0; w < LW; ++w) {
      for (uint64_t mm = lset[w]; mm; mm &= mm - 1) {
        const int b = __ffsll((long long)mm) - 1;
        const int s = w * 64 + b;
        int g = link_g[s];
        link_t[s] = DINF;
        link_g[s] = -1;
        amask[w] &= ~(1ull << b);
        deliver(g, now);
      }
    }
    if (status != ST_OK) break;
    schedule(now);
  }
  if (status == ST_OK) {
    mem_flush();
    if (done != G) status = ST_DEADLOCK;
  }
  if (tr.rec) *tr.count = n_trace;
  step = 0.0;
  viol_out = viol;
  if (status != ST_OK) return status;
  step = step_t;
  if (!viol)
    for (int dev = 0; dev < d; ++dev)
      if (pk[dev] > cap[dev]) {
        viol_out = 2;
        break;
      }
  return status;
}

// compute time of every group on every device, max(flops / peak, bytes / bw)
// (simulator.py kernel_time), once per launch instead of two float64 divisions per event
__global__ void des_ctab_kernel(DesView V, int d, const double* __restrict__ peakf,
                                const double* __restrict__ mbw, double* __restrict__ ctab) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)V.G * d) return;
  const int g = (int)(i / d), dev = (int)(i % d);
  ctab[i] = fmax(__ddiv_rn(V.grec[g].cost_flops, peakf[dev]),
                 __ddiv_rn(V.grec[g].cost_bytes, mbw[dev]));
}

// One placement per 32-thread block (measured 4.2x faster than one placement per lane on
// the cfg4 graph): the warp fills the group states, lane 0 runs the event loop with the
// device / link state in shared memory.
// transfer time of every external edge when all links share one bandwidth
__global__ void des_etab_kernel(DesView V, double lbw0, double* __restrict__ etab) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < V.num_edges) etab[i] = __ddiv_rn(V.out_bytes[i], lbw0);
}

template <int MAXD>
__global__ void des_kernel(DesView V, int K, const int32_t* __restrict__ placement,
                           int64_t pstride, const int32_t* __restrict__ prio, int64_t prio_stride,
                           int d, const double* __restrict__ peakf, const double* __restrict__ mbw,
                           const double* __restrict__ cap, const double* __restrict__ lbw,
                           int policy, double baseline, DesCaps caps, char* __restrict__ scratch,
                           int64_t scratch_stride, const int32_t* __restrict__ which,
                           double* __restrict__ o_step, uint8_t* __restrict__ o_valid,
                           int8_t* __restrict__ o_viol, double* __restrict__ o_busy,
                           double* __restrict__ o_peak, double* __restrict__ o_reward,
                           int32_t* __restrict__ o_status, DesTraceLog tr,
                           const double* __restrict__ ctab, const double* __restrict__ etab) {
  const int tid = blockIdx.x;
  if (tid >= K) return;
  const int kk = which ? which[tid] : tid;
  const int32_t* pl = placement + (int64_t)kk * pstride;
  char* base = scratch + (int64_t)tid * scratch_stride;
  const int32_t* pr = prio + (int64_t)kk * prio_stride;
  des_init_states(V, pl, pr, policy, reinterpret_cast<DesNodeState*>(base), threadIdx.x, 32);
  __syncwarp();
  if (threadIdx.x) return;
  __shared__ DesState<MAXD> S;
  double step;
  int8_t viol;
  const int status = des_run<MAXD>(V, pl, pr, d, peakf, mbw, cap, lbw, policy, caps, base, S, tr,
                                   step, viol, true, ctab, etab);
  o_status[tid] = status;
  if (status != ST_OK) return;
  o_step[kk] = step;
  o_valid[kk] = viol == 0;
  o_viol[kk] = viol;
  for (int dev = 0; dev < d; ++dev) {
    if (o_busy) o_busy[(int64_t)kk * d + dev] = S.busy[dev];
    if (o_peak) o_peak[(int64_t)kk * d + dev] = S.pk[dev];
  }
  if (o_reward && baseline > 0.0)
    o_reward[kk] = viol == 0 ? -sqrt(__ddiv_rn(step, baseline)) : -10.0;
}

int simulate_batch(const DesView& v, int K, const int32_t* placement, int64_t pstride,
                   const int32_t* prio, int64_t prio_stride, int d, const double* peak,
                   const double* mem_bw, const double* cap, const double* link_bw, int policy,
                   double baseline, double* step_time, uint8_t* valid, int8_t* violation,
                   double* busy, double* peak_mem, double* reward, go_ctx* ctx,
                   cudaStream_t st, DesTraceRec* trace, int64_t trace_cap, int64_t* trace_count) {
  GO_CHECK(!trace || K == 1, "event traces are recorded for one placement per call");
  if (K <= 0) return GO_OK;
  if (d > DES_MAXD) GO_THROW(GO_ERR_UNSUPPORTED, "%d devices > %d", d, DES_MAXD);
  // topology -> device (small; part of the DES workspace head)
  std::vector<double> topo(3 * d + d * d);
  for (int i = 0; i < d; ++i) {
    topo[i] = peak[i];
    topo[d + i] = mem_bw[i];
    topo[2 * d + i] = cap[i];
  }
  for (int i = 0; i < d * d; ++i) topo[3 * d + i] = link_bw[i];
  DesCaps caps{64, 64, 64};
  const int G = v.G;
  // one bandwidth on every link (src != dst): transfer times precomputed per edge
  bool uniform_links = d > 1;
  const double lbw0 = d > 1 ? link_bw[1] : 0.0;
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b)
      if (a != b && link_bw[a * d + b] != lbw0) uniform_links = false;
  auto run = [&](int count, const int32_t* which, DesCaps c) {
    int64_t stride = c.per_placement_bytes(G, d);
    const int64_t h_ctab = round_up((int64_t)topo.size() * 8, 256) +
                           round_up((int64_t)count * 4, 256) + round_up((int64_t)K * 4, 256);
    const int64_t h_etab = h_ctab + round_up((int64_t)G * d * 8, 256);
    const int64_t head = h_etab + round_up(std::max<int64_t>(v.num_edges, 1) * 8, 256);
    char* ws = reinterpret_cast<char*>(ctx->ensure_des(head + stride * count));
    double* dtopo = reinterpret_cast<double*>(ws);
    int32_t* dstatus = reinterpret_cast<int32_t*>(ws + round_up((int64_t)topo.size() * 8, 256));
    int32_t* dwhich = dstatus + round_up(count, 64);
    double* dctab = reinterpret_cast<double*>(ws + h_ctab);
    double* detab = reinterpret_cast<double*>(ws + h_etab);
    CUDA_CHECK(cudaMemcpyAsync(dtopo, topo.data(), topo.size() * 8, cudaMemcpyHostToDevice, st));
    if (which)
      CUDA_CHECK(cudaMemcpyAsync(dwhich, which, (size_t)count * 4, cudaMemcpyHostToDevice, st));
    auto kern = d <= 4 ? des_kernel<4> : d <= 8 ? des_kernel<8> : des_kernel<DES_MAXD>;
    const int64_t nct = (int64_t)G * d;
    des_ctab_kernel<<<(unsigned)cdiv(nct, 256), 256, 0, st>>>(v, d, dtopo, dtopo + d, dctab);
    LAUNCH_CHECK();
    if (uniform_links && v.num_edges > 0) {
      des_etab_kernel<<<(unsigned)cdiv(v.num_edges, 256), 256, 0, st>>>(v, lbw0, detab);
      LAUNCH_CHECK();
    }
    kern<<<(unsigned)count, 32, 0, st>>>(
        v, count, placement, pstride, prio, prio_stride, d, dtopo, dtopo + d, dtopo + 2 * d,
        dtopo + 3 * d, policy, baseline, c, ws + head, stride, which ? dwhich : nullptr,
        step_time, valid, violation, busy, peak_mem, reward, dstatus,
        DesTraceLog{trace, trace_cap, trace_count}, dctab, uniform_links ? detab : nullptr);
    LAUNCH_CHECK();
    std::vector<int32_t> hstat(count);
    CUDA_CHECK(cudaMemcpyAsync(hstat.data(), dstatus, (size_t)count * 4, cudaMemcpyDeviceToHost,
                               st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    return hstat;
  };
  std::vector<int32_t> stat = run(K, nullptr, caps);
  std::vector<int32_t> redo;
  for (int i = 0; i < K; ++i) {
    if (stat[i] == ST_DEADLOCK) GO_THROW(GO_ERR_DEADLOCK, "simulation deadlocked");
    if (stat[i] != ST_OK) redo.push_back(i);
  }
  if (!redo.empty()) {
    // rerun overflowing placements with capacities that cannot overflow
    DesCaps big{std::max<int64_t>(G, 1), std::max<int64_t>(v.num_edges, 1),
                std::max<int64_t>(G, 1)};
    for (size_t i0 = 0; i0 < redo.size(); i0 += 8) {
      int cnt = (int)std::min<size_t>(8, redo.size() - i0);
      std::vector<int32_t> s2 = run(cnt, redo.data() + i0, big);
      for (int j = 0; j < cnt; ++j)
        if (s2[j] != ST_OK)
          GO_THROW(s2[j] == ST_DEADLOCK ? GO_ERR_DEADLOCK : GO_ERR_UNSUPPORTED,
                   "simulation failed (status %d)", s2[j]);
    }
  }
  return GO_OK;
}


// ---------------------------------------------------------------------------------------
// Simulated annealing on the device DES (baselines.py:146-206), many chains at once.
//
// One chain per 32-thread block: lane 0 runs the chain's numpy stream (PCG64 with the
// Generator's buffered next_uint32 and Lemire bounded draws, rng.cuh), proposes the
// move(s), simulates the candidate with des_run and applies the Metropolis test; the
// warp copies the state into the best-so-far arrays on an improvement.  Every draw,
// the float64 acceptance arithmetic and the geometric cooling follow the reference
// line for line, so a chain seeded like SAConfig.seed walks exactly the reference's
// chain (the step times it compares are bit-exact); the other chains are independent
// restarts.  Moves are applied in place and undone on rejection.  Tasks annealed here:
// placement and schedule_priority over a fixed grouping (fusion priorities change the
// grouping, whose tables are built on the host).
namespace {
constexpr int SA_MAX_TASKS = 2;
constexpr int SA_MAX_MOVES = 16;
}

template <int MAXD>
__global__ void anneal_kernel(DesView V, int C, const uint64_t* __restrict__ rng_words,
                              int32_t* __restrict__ cur, int32_t* __restrict__ best, int d,
                              const double* __restrict__ peakf, const double* __restrict__ mbw,
                              const double* __restrict__ cap, const double* __restrict__ lbw,
                              int policy, int iterations, int moves, double t_init,
                              double cooling, int ntasks, int task_slot0, int task_slot1,
                              int size0, int size1, DesCaps caps, char* __restrict__ scratch,
                              int64_t scratch_stride, double* __restrict__ o_best,
                              int32_t* __restrict__ o_status) {
  const int c = blockIdx.x;
  if (c >= C) return;
  const int lane = threadIdx.x;
  const int n = V.n;
  // arrays per chain: [placement | priorities], current and best
  int32_t* cs = cur + (int64_t)c * 2 * n;
  int32_t* bs = best + (int64_t)c * 2 * n;
  __shared__ DesState<MAXD> S;
  __shared__ int sh_flag;  // 1 = copy current -> best, -1 = stop (DES failure)
  const int slot[SA_MAX_TASKS] = {task_slot0, task_slot1};
  const int size[SA_MAX_TASKS] = {size0, size1};
  Pcg64 rng;
  char* base = scratch + (int64_t)c * scratch_stride;
  double cur_time = 0.0, best_time = 0.0, temp = 0.0;
  auto evaluate = [&](double& t) -> int {
    double step;
    int8_t viol;
    const int stt = des_run<MAXD>(V, cs, cs + n, d, peakf, mbw, cap, lbw, policy, caps, base, S,
                                  DesTraceLog{nullptr, 0, nullptr}, step, viol);
    t = viol == 0 ? step : DINF;
    return stt;
  };
  if (lane == 0) {
    rng.state = ((u128)rng_words[4 * c] << 64) | rng_words[4 * c + 1];
    rng.inc = ((u128)rng_words[4 * c + 2] << 64) | rng_words[4 * c + 3];
    rng.has32 = false;
    rng.buf32 = 0;
    const int stt = evaluate(cur_time);
    best_time = cur_time;
    temp = t_init == t_init ? t_init : (isfinite(cur_time) ? 0.1 * cur_time : 1.0);
    sh_flag = stt == ST_OK ? 0 : -1;
    o_status[c] = stt;
  }
  __syncwarp();
  if (sh_flag < 0) return;
  int mv_slot[SA_MAX_MOVES], mv_node[SA_MAX_MOVES], mv_old[SA_MAX_MOVES];
  for (int it = 0; it < iterations; ++it) {
    if (lane == 0) {
      for (int m = 0; m < moves; ++m) {
        const int t = (int)rng.bounded((uint32_t)(ntasks - 1));  // rng.integers(len(tasks))
        const int v = (int)rng.bounded((uint32_t)(n - 1));       // rng.integers(n)
        const int val = (int)rng.bounded((uint32_t)(size[t] - 1));
        int32_t* arr = cs + (int64_t)slot[t] * n;
        mv_slot[m] = slot[t];
        mv_node[m] = v;
        mv_old[m] = arr[v];
        arr[v] = val;
      }
      double cand;
      const int stt = evaluate(cand);
      int flag = 0;
      if (stt != ST_OK) {
        o_status[c] = stt;
        flag = -1;
      } else {
        const double delta = cand - cur_time;
        bool accept = delta <= 0.0;
        if (!accept && temp > 0.0 && isfinite(delta))
          accept = rng.random() < exp(__ddiv_rn(-delta, temp));
        if (accept) {
          cur_time = cand;
          if (cur_time < best_time) {
            best_time = cur_time;
            flag = 1;
          }
        } else {
          for (int m = moves - 1; m >= 0; --m) cs[(int64_t)mv_slot[m] * n + mv_node[m]] = mv_old[m];
        }
        temp = __dmul_rn(temp, cooling);
      }
      sh_flag = flag;
    }
    __syncwarp();
    const int flag = sh_flag;
    if (flag < 0) return;
    if (flag == 1) {
      for (int64_t i = lane; i < 2 * (int64_t)n; i += 32) bs[i] = cs[i];
    }
    __syncwarp();
  }
  if (lane == 0) o_best[c] = best_time;
}

int anneal_chains(const DesView& v, int C, const uint64_t* rng_words_host, int32_t* cur,
                  int32_t* best, int d, const double* peak, const double* mem_bw,
                  const double* cap, const double* link_bw, int policy, int iterations,
                  int moves, double t_init, double cooling, int ntasks, const int* slots,
                  const int* sizes, double* best_time, go_ctx* ctx, cudaStream_t st) {
  GO_CHECK(C >= 1 && ntasks >= 1 && ntasks <= SA_MAX_TASKS, "bad annealing configuration");
  GO_CHECK(moves >= 1 && moves <= SA_MAX_MOVES, "moves_per_step must be in [1, %d]", SA_MAX_MOVES);
  if (d > DES_MAXD) GO_THROW(GO_ERR_UNSUPPORTED, "%d devices > %d", d, DES_MAXD);
  std::vector<double> topo(3 * d + d * d);
  for (int i = 0; i < d; ++i) {
    topo[i] = peak[i];
    topo[d + i] = mem_bw[i];
    topo[2 * d + i] = cap[i];
  }
  for (int i = 0; i < d * d; ++i) topo[3 * d + i] = link_bw[i];
  const int G = v.G;
  auto run = [&](DesCaps caps) {
    const int64_t stride = caps.per_placement_bytes(G, d);
    const int64_t head = round_up((int64_t)topo.size() * 8, 256) + round_up((int64_t)C * 32, 256) +
                         round_up((int64_t)C * 4, 256);
    char* ws = reinterpret_cast<char*>(ctx->ensure_des(head + stride * C));
    double* dtopo = reinterpret_cast<double*>(ws);
    uint64_t* dwords = reinterpret_cast<uint64_t*>(ws + round_up((int64_t)topo.size() * 8, 256));
    int32_t* dstatus =
        reinterpret_cast<int32_t*>(reinterpret_cast<char*>(dwords) + round_up((int64_t)C * 32, 256));
    CUDA_CHECK(cudaMemcpyAsync(dtopo, topo.data(), topo.size() * 8, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(dwords, rng_words_host, (size_t)C * 32, cudaMemcpyHostToDevice, st));
    auto kern = d <= 4 ? anneal_kernel<4> : d <= 8 ? anneal_kernel<8> : anneal_kernel<DES_MAXD>;
    kern<<<C, 32, 0, st>>>(v, C, dwords, cur, best, d, dtopo, dtopo + d, dtopo + 2 * d,
                           dtopo + 3 * d, policy, iterations, moves, t_init, cooling, ntasks,
                           slots[0], ntasks > 1 ? slots[1] : 0, sizes[0],
                           ntasks > 1 ? sizes[1] : 1, caps, ws + head, stride, best_time, dstatus);
    LAUNCH_CHECK();
    std::vector<int32_t> hs(C);
    CUDA_CHECK(cudaMemcpyAsync(hs.data(), dstatus, (size_t)C * 4, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    return hs;
  };
  // small queues first; a chain whose heap / link FIFO overflowed makes the whole launch
  // re-run from the saved initial state with capacities that cannot overflow
  const size_t state_bytes = (size_t)C * 2 * v.n * sizeof(int32_t);
  int32_t* saved = nullptr;
  CUDA_CHECK(cudaMallocAsync(&saved, state_bytes, st));
  CUDA_CHECK(cudaMemcpyAsync(saved, cur, state_bytes, cudaMemcpyDeviceToDevice, st));
  std::vector<int32_t> stat = run(DesCaps{64, 64, 64});
  bool redo = false;
  for (int s : stat) {
    if (s == ST_DEADLOCK) GO_THROW(GO_ERR_DEADLOCK, "simulation deadlocked");
    redo |= s != ST_OK;
  }
  if (redo) {
    CUDA_CHECK(cudaMemcpyAsync(cur, saved, state_bytes, cudaMemcpyDeviceToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(best, saved, state_bytes, cudaMemcpyDeviceToDevice, st));
    stat = run(DesCaps{std::max<int64_t>(G, 1), std::max<int64_t>(v.num_edges, 1),
                       std::max<int64_t>(G, 1)});
    for (int s : stat)
      if (s != ST_OK)
        GO_THROW(s == ST_DEADLOCK ? GO_ERR_DEADLOCK : GO_ERR_UNSUPPORTED,
                 "simulation failed (status %d)", s);
  }
  CUDA_CHECK(cudaFreeAsync(saved, st));
  return 0;
}

}  // namespace go

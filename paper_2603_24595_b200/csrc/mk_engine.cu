// mk_engine.cu -- sm_100a checking-stage engine behind include/mk_b200.h.
//
// Replaces, per compiled site problem, the reference's decision
// (solver/builtin.py:705-764 check_assertions) and canonical-witness search
// (engine/report.py:147-203 + solver/interface.py:112-187 bisection) by a
// data-parallel lexicographic branch-and-prune over the problem's box of free
// symbols:
//
//   k_bb      pre-split rounds, one thread per box: incumbent test on the
//             box's best corner, linear bound contraction, interval
//             evaluation of the bytecode, then prune / accept the corner /
//             hand to leaf enumeration / split into K children written in
//             lexicographic order; the host compacts the children
//             (order-preserving scan) until every search unit has a task;
//   k_search  persistent best-first search, one independent unit per WARP:
//             pop the best 32 boxes of the warp's HBM stack (one per lane),
//             process, warp-scan the child counts, write children worst
//             first (best on top), enumerate small boxes warp-wide in
//             lexicographic index order; incumbents are shared through a
//             64-bit atomicMin key plus a per-problem seqlock.  When a
//             quarter of the units idles, busy units dump their stacks and
//             the host relaunches on the dumped boxes (bulk-synchronous
//             redistribution).
//
// Every per-box / per-point routine is instantiated for two value types
// (mk_core.cuh): exact int64 for problems the compiler proved narrow, and
// saturating int128 otherwise; narrow and wide problems run as two
// concurrent persistent grids on two streams.  Small problems (<= 8 free
// symbols, <= 64 registers) use compile-time-sized per-lane arrays.

#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "mk_b200.h"
#include "mk_core.cuh"
#include "mk_jit.cuh"
#include "mk_shreg.cuh"

namespace {

// specialised k_search code paths for small problems (8 symbols: 64-entry
// local register files; 24 registers: the register file in shared memory).
// Off: one generic path per class is faster on every corpus set measured on
// the B200 (config3 40.7 -> 36.2 ms, paged_attention_v2 long 32.2 -> 29.6,
// moe_align 18.4 -> 17.3; profiles/r02_code_paths.jsonl) -- the three inlined
// copies made k_search<int64_t> 46 k SASS instructions, and 40 % of its
// stall samples were instruction fetch (no_inst) -- and a budgeted run
// keeps its budget (the small path overran a 0.5 s budget by 0.49 s)
#ifndef MK_SMALL_PATH
#define MK_SMALL_PATH 0
#endif
#ifndef MK_SHREG_PATH
#define MK_SHREG_PATH 0
#endif

// bound-contraction sweeps per box (each ends early once nothing changes).
// One: a box's children inherit its contracted bounds and are contracted
// again, so further sweeps on the parent mostly repeat work (measured on the
// B200, full sets: config3 15.4 -> 13.2 ms, moe_align 6.4 -> 6.0,
// paged_attention_v2 long 12.6 -> 12.0 at 1 vs 4; profiles/r02_contract_sweeps.jsonl)
#ifndef MK_CONTRACT_SWEEPS
#define MK_CONTRACT_SWEEPS 1
#endif

constexpr unsigned FULL = 0xffffffffu;
constexpr int SMALL_V = 8;    // free symbols of a "small" problem
constexpr int SMALL_R = 64;   // registers of a "small" problem
constexpr int SH_R = 24;      // registers of a narrow problem evaluated from shared memory
// per 128-thread CTA; none without the shared-register path, which leaves
// the whole 256 KB of the SM's L1 / shared storage to the L1 (the generic
// path's register files are local memory)
constexpr int SH_BYTES = MK_SHREG_PATH ? 2 * SH_R * 128 * (int)sizeof(int64_t) : 0;
constexpr int DIVE_CAP = 1024;  // boxes per speculative-dive stack

// dynamic shared memory of k_search<int64_t>: lo / hi interval register files
extern __shared__ int64_t mk_dyn_sh[];

struct Box {
  int32_t prob;
  int32_t pad0;
  int64_t pad1;
  // followed by mk_i128 lo[S], hi[S]
};

struct Incumbent {
  int lock;
  unsigned version;
  int has;
  int err;  // inexact evaluation (saturation) or unsplittable box
  // lexicographic key of the best offered model: each symbol's offset from
  // its best root bound packed into bit fields in witness order (a monotone
  // prefix of the full order when the fields exceed 64 bits)
  unsigned long long key;
};

struct DevSet {
  const mk_problem* probs;
  const mk_insn* insns;
  const mk_i128* consts;
  const int32_t* atom_regs;
  const uint64_t* atom_masks;
  const mk_row* rows;
  const mk_row_term* terms;
  const mk_i128* var_lo;
  const mk_i128* var_hi;
  Incumbent* inc;
  mk_i128* best;  // nvar_total
  int stride;     // S
  size_t box_bytes;
};

struct DevStats {
  unsigned long long boxes, leaves, points, insns_bb, insns_leaf, steps;
  double covered;
};

// per-lane counters, flushed to DevStats once per unit
struct LaneStats {
  unsigned long long boxes, leaves, points, insns_bb, insns_leaf, steps;
  double covered;
  __device__ void zero() {
    boxes = leaves = points = insns_bb = insns_leaf = steps = 0;
    covered = 0.0;
  }
  __device__ void flush(DevStats* st) {
    if (steps) atomicAdd(&st->steps, steps);
    if (boxes) atomicAdd(&st->boxes, boxes);
    if (leaves) atomicAdd(&st->leaves, leaves);
    if (points) atomicAdd(&st->points, points);
    if (insns_bb) atomicAdd(&st->insns_bb, insns_bb);
    if (insns_leaf) atomicAdd(&st->insns_leaf, insns_leaf);
    if (covered != 0.0) atomicAdd(&st->covered, covered);
  }
  __device__ void flush_warp(DevStats* st) {
    for (int o = 16; o > 0; o >>= 1) {
      boxes += __shfl_down_sync(FULL, boxes, o);
      leaves += __shfl_down_sync(FULL, leaves, o);
      points += __shfl_down_sync(FULL, points, o);
      insns_bb += __shfl_down_sync(FULL, insns_bb, o);
      insns_leaf += __shfl_down_sync(FULL, insns_leaf, o);
      steps += __shfl_down_sync(FULL, steps, o);
      covered += __shfl_down_sync(FULL, covered, o);
    }
    if ((threadIdx.x & 31) == 0) flush(st);
  }
};

__device__ __forceinline__ bool is_narrow(const mk_problem& p) {
  return (p.flags & MK_PF_NARROW) != 0;
}
__device__ __forceinline__ bool is_small(const mk_problem& p) {
  return MK_SMALL_PATH && p.nvars <= SMALL_V && p.nregs <= SMALL_R;
}
__device__ __forceinline__ bool is_shreg(const mk_problem& p) {
  return MK_SHREG_PATH && is_narrow(p) && p.nvars <= SMALL_V && p.nregs <= SH_R;
}

__device__ __forceinline__ Box* box_at(void* base, size_t box_bytes, size_t i) {
  return reinterpret_cast<Box*>(reinterpret_cast<char*>(base) + i * box_bytes);
}
__device__ __forceinline__ mk_i128* box_lo(Box* b) { return reinterpret_cast<mk_i128*>(b + 1); }

// box storage: the pre-split stack keeps int128 bounds (mk_i128); the narrow
// search class keeps int64 bounds (half the HBM per box)
template <typename T>
struct Store;
template <>
struct Store<i128> {
  typedef mk_i128 E;
  __device__ static i128 get(const E& e) { return mk_ld(e); }
  __device__ static E put(i128 x) { return mk_st(x); }
};
template <>
struct Store<int64_t> {
  typedef int64_t E;
  __device__ static int64_t get(const E& e) { return e; }
  __device__ static E put(i128 x) { return (int64_t)x; }
};
template <typename T>
__host__ __device__ constexpr size_t box_bytes_of(int S) {
  return sizeof(Box) + 2 * sizeof(typename Store<T>::E) * (size_t)S;
}

template <typename V>
__device__ __forceinline__ V ldv(const mk_i128& v) {
  return MkNum<V>::ld(v);
}
template <typename V>
__device__ __forceinline__ V ldv_volatile(const volatile mk_i128* p) {
  mk_i128 t;
  t.lo = p->lo;
  t.hi = p->hi;
  return MkNum<V>::ld(t);
}

// 64-bit lexicographic key of a point (see Incumbent::key)
// the best corner of a box in witness order, read in place (the corner never
// exists as an array: a materialised copy was one more local-memory array per
// box evaluation)
template <typename V>
struct BoxCorner {
  const V* lo;
  const V* hi;
  uint64_t maxmask;
  __device__ __forceinline__ V operator[](int i) const { return ((maxmask >> i) & 1) ? hi[i] : lo[i]; }
};

template <typename V, typename X>
__device__ unsigned long long lex_key(const DevSet& D, const mk_problem& p, const X& x) {
  typedef typename MkNum<V>::U U;
  unsigned long long key = 0;
  int left = 64;
  for (int i = 0; i < p.nvars && left > 0; ++i) {
    V rlo = ldv<V>(D.var_lo[p.var_off + i]), rhi = ldv<V>(D.var_hi[p.var_off + i]);
    U span = (U)(rhi - rlo);
    int bits = mk_bitlen(span);
    if (bits == 0) continue;
    U d = ((p.maxmask >> i) & 1) ? (U)(rhi - x[i]) : (U)(x[i] - rlo);
    if (bits <= left) {
      key = (bits == 64 ? 0ull : (key << bits)) | (unsigned long long)d;
      left -= bits;
    } else {  // keep the top `left` bits of this field, then stop
      key = (key << left) | (unsigned long long)(d >> (bits - left));
      left = 0;
    }
  }
  if (left > 0 && left < 64) key <<= left;
  return key;
}

// incumbent test: true when the box cannot hold anything better than the
// current incumbent (its best corner is not strictly better)
template <typename V, typename X>
__device__ bool inc_dominates(const DevSet& D, int pid, const mk_problem& p, const X& corner) {
  Incumbent* I = D.inc + pid;
  {
    unsigned long long kmin = *((volatile unsigned long long*)&I->key);
    if (kmin == ~0ull) return false;  // nothing offered yet
    if (p.flags & MK_PF_ANY) return true;  // feasibility only: one model decides
    unsigned long long k = lex_key<V>(D, p, corner);
    if (k > kmin) return true;        // a strictly better model was offered
  }
  unsigned v1 = *((volatile unsigned*)&I->version);
  if (v1 & 1u) return false;
  __threadfence();
  int has = *((volatile int*)&I->has);
  if (!has) return false;
  const volatile mk_i128* B = D.best + p.var_off;
  bool dominated = true;
  for (int i = 0; i < p.nvars; ++i) {
    V b = ldv_volatile<V>(B + i);
    if (corner[i] == b) continue;
    bool mx = (p.maxmask >> i) & 1;
    dominated = !(mx ? corner[i] > b : corner[i] < b);
    break;
  }
  __threadfence();
  unsigned v2 = *((volatile unsigned*)&I->version);
  if (v1 != v2) return false;
  return dominated;
}

template <typename V, typename X>
__device__ void inc_offer(const DevSet& D, int pid, const mk_problem& p, const X& x) {
  Incumbent* I = D.inc + pid;
  // lock-free filter: a candidate whose key prefix is worse than the best
  // offered key loses without touching the lock
  {
    unsigned long long k = lex_key<V>(D, p, x);
    unsigned long long old = atomicMin(&I->key, k);
    if (k > old) return;
    // feasibility only: the first offer records the model (inc_dominates
    // prunes everything once a key exists)
    if ((p.flags & MK_PF_ANY) && old != ~0ull) return;
  }
  if (!(p.flags & MK_PF_ANY) && inc_dominates<V>(D, pid, p, x)) return;
  unsigned ns = 32;
  while (atomicCAS(&I->lock, 0, 1) != 0) {
    __nanosleep(ns);
    if (ns < 2048) ns <<= 1;
  }
  __threadfence();
  bool better = true;
  if (I->has) {  // strictly better in witness order (equal points are not)
    better = false;
    for (int i = 0; i < p.nvars; ++i) {
      V b = ldv<V>(D.best[p.var_off + i]);
      if (x[i] == b) continue;
      bool mx = (p.maxmask >> i) & 1;
      better = mx ? x[i] > b : x[i] < b;
      break;
    }
  }
  if (better) {
    atomicAdd(&I->version, 1u);
    __threadfence();
    for (int i = 0; i < p.nvars; ++i) D.best[p.var_off + i] = mk_st((i128)x[i]);
    I->has = 1;
    __threadfence();
    atomicAdd(&I->version, 1u);
  }
  __threadfence();
  atomicExch(&I->lock, 0);
}

__device__ __forceinline__ MkProb view(const DevSet& D, int pid) {
  return mk_prob_view(D.probs, pid, D.insns, D.consts, D.atom_regs, D.atom_masks, D.rows,
                      D.terms);
}

__global__ void k_roots(DevSet D, int nprob, void* stack, int keep_incumbents) {
  int pid = blockIdx.x * blockDim.x + threadIdx.x;
  if (pid >= nprob) return;
  const mk_problem p = D.probs[pid];
  Box* b = box_at(stack, D.box_bytes, pid);
  b->prob = pid;
  mk_i128* lo = box_lo(b);
  mk_i128* hi = lo + D.stride;
  for (int i = 0; i < p.nvars; ++i) {
    lo[i] = D.var_lo[p.var_off + i];
    hi[i] = D.var_hi[p.var_off + i];
  }
  D.inc[pid].lock = 0;
  D.inc[pid].err = 0;
  if (keep_incumbents) return;  // a model of a previous attempt stays a valid bound
  D.inc[pid].version = 0;
  D.inc[pid].has = 0;
  D.inc[pid].err = 0;
  D.inc[pid].key = ~0ull;
}

// Root bound propagation, one thread per problem, before any search: the
// linear rows (and row groups) contract the root box in the stack to their
// fixpoint (up to `sweeps` FBBT sweeps, exact int128); a root with no model
// is marked empty (lo > hi in its first symbol) and every consumer drops
// it.  This is the device half of the presolve's bound propagation (the host
// half can be switched off: compiler.HOST_FBBT).
__global__ void k_root_contract(DevSet D, int nprob, void* stack, int sweeps) {
  const int pid = blockIdx.x * blockDim.x + threadIdx.x;
  if (pid >= nprob) return;
  const mk_problem p = D.probs[pid];
  if (p.nrows == 0 || p.nvars == 0) return;
  Box* b = box_at(stack, D.box_bytes, pid);
  mk_i128* blo = box_lo(b);
  mk_i128* bhi = blo + D.stride;
  i128 lo[MK_MAXV], hi[MK_MAXV];
  for (int i = 0; i < p.nvars; ++i) {
    lo[i] = ldv<i128>(blo[i]);
    hi[i] = ldv<i128>(bhi[i]);
  }
  const MkProb P = mk_prob_view(D.probs, pid, D.insns, D.consts, D.atom_regs, D.atom_masks,
                                D.rows, D.terms);
  if (!mk_contract<i128>(P, lo, hi, sweeps)) lo[0] = hi[0] + 1;
  for (int i = 0; i < p.nvars; ++i) {
    blo[i] = Store<i128>::put(lo[i]);
    bhi[i] = Store<i128>::put(hi[i]);
  }
}

// ---------------------------------------------------------------------------
// per-box step

enum { ACT_DONE = 0, ACT_LEAF = 1, ACT_SPLIT = 2 };

struct Act {
  int kind;
  int sv;   // split symbol
  int m;    // pieces of sv
  int sv2;  // second split symbol of a product split, -1 for none
  int m2;   // pieces of sv2 (children: m * m2)
};

constexpr int MAX_CHILDREN = 32;  // product splits: at most one child per lane

// lo/hi: the box (contracted in place).  Prunes, accepts the best corner of an
// all-true box, hands small boxes to enumeration, or chooses a split.
// `wide`: the unit's stack is too shallow to keep every lane busy: a split
// whose symbol has fewer than K values also splits a second undecided symbol
// (a product split of up to MAX_CHILDREN children), trading a little pruning
// granularity for lanes that would otherwise idle
template <typename V, int CAPV, int CAPR, int SH = 0>
__device__ Act process_box(const DevSet& D, int pid, const mk_problem& p, V* lo, V* hi, int K,
                           long long leaf_volume, LaneStats& st, bool wide = false) {
  const int nv = p.nvars;
  const MkProb P = view(D, pid);
  Act a;
  a.kind = ACT_DONE;
  a.sv = -1;
  a.m = 0;
  a.sv2 = -1;
  a.m2 = 1;
  const BoxCorner<V> c{lo, hi, p.maxmask};
  st.boxes++;
  for (int v = 0; v < nv; ++v)
    if (lo[v] > hi[v]) return a;  // an empty root (k_root_contract)
  const double vol0 = mk_volume_f(lo, hi, nv);
  if (inc_dominates<V>(D, pid, p, c)) {
    st.covered += vol0;
    return a;
  }
  if (!mk_contract(P, lo, hi, MK_CONTRACT_SWEEPS)) {
    st.covered += vol0;
    return a;
  }
  int64_t cnt = 0;
  MkBoxVerdict v;
  if constexpr (SH != 0) {
    v = sh_eval_box(P, lo, hi, mk_dyn_sh, mk_dyn_sh + SH_R * blockDim.x, &cnt);
  } else {
    MkPair<V> R[CAPR < MK_MAXT ? CAPR : MK_MAXT];   // temporaries only (flags in registers)
    v = mk_eval_box_t(P, lo, hi, R, &cnt);
  }
  st.insns_bb += (unsigned long long)cnt;
  if (v.any_false) {
    st.covered += vol0;
    return a;
  }
  if (v.all_true) {
    inc_offer<V>(D, pid, p, c);   // the contracted box's best corner
    st.covered += vol0;
    return a;
  }
  if (mk_volume(lo, hi, nv) <= leaf_volume) {
    a.kind = ACT_LEAF;
    return a;
  }
  int sv = mk_pick_split(lo, hi, nv, v.und_mask, *((volatile int*)&D.inc[pid].has) != 0);
  if (sv < 0) {  // every symbol of an undecided atom is fixed: saturated arithmetic
    atomicExch(&D.inc[pid].err, 1);
    return a;
  }
  typedef typename MkNum<V>::U U;
  U size = (U)(hi[sv] - lo[sv]) + 1;
  a.kind = ACT_SPLIT;
  a.sv = sv;
  a.m = size < (U)K ? (int)size : K;
  if (wide && a.m < K) {
    const int sv2 = mk_pick_split(lo, hi, nv, v.und_mask & ~(1ull << sv),
                                  *((volatile int*)&D.inc[pid].has) != 0);
    if (sv2 >= 0) {
      const int cap = MAX_CHILDREN / a.m;
      U size2 = (U)(hi[sv2] - lo[sv2]) + 1;
      const int m2 = size2 < (U)cap ? (int)size2 : cap;
      if (m2 >= 2) {
        a.sv2 = sv2;
        a.m2 = m2;
      }
    }
  }
  return a;
}

template <typename T, typename V>
__device__ __forceinline__ void write_box(Box* out, int pid, const V* lo, const V* hi, int nv,
                                          int stride, int sv, V plo, V phi) {
  typedef Store<T> St;
  out->prob = pid;
  typename St::E* olo = reinterpret_cast<typename St::E*>(out + 1);
  for (int k = 0; k < nv; ++k) {
    olo[k] = St::put((i128)(k == sv ? plo : lo[k]));
    olo[stride + k] = St::put((i128)(k == sv ? phi : hi[k]));
  }
}

template <typename T, typename V>
__device__ __forceinline__ void load_box(const Box* in, int nv, int stride, V* lo, V* hi) {
  typedef Store<T> St;
  const typename St::E* blo = reinterpret_cast<const typename St::E*>(in + 1);
  for (int v = 0; v < nv; ++v) {
    lo[v] = (V)St::get(blo[v]);
    hi[v] = (V)St::get(blo[stride + v]);
  }
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// pre-split round kernel: one thread per box

template <typename V, int CAPV, int CAPR>
__device__ void bb_one(const DevSet& D, const Box* in, int pid, const mk_problem& p, int i, int K,
                       long long leaf_volume, void* child_out, int* child_flag, void* leaf_out,
                       int* leaf_flag, LaneStats& st) {
  const int nv = p.nvars;
  V lo[CAPV], hi[CAPV];
  load_box<i128, V>(in, nv, D.stride, lo, hi);
  Act a = process_box<V, CAPV, CAPR>(D, pid, p, lo, hi, K, leaf_volume, st);
  if (a.kind == ACT_LEAF) {
    write_box<i128, V>(box_at(leaf_out, D.box_bytes, i), pid, lo, hi, nv, D.stride, -1, 0, 0);
    leaf_flag[i] = 1;
  } else if (a.kind == ACT_SPLIT) {
    bool mx = (p.maxmask >> a.sv) & 1;
    for (int t = 0; t < a.m; ++t) {
      V plo, phi;
      mk_piece(lo[a.sv], hi[a.sv], a.m, t, mx, &plo, &phi);
      size_t slot = (size_t)i * K + (K - 1 - t);  // best piece in the highest slot
      write_box<i128, V>(box_at(child_out, D.box_bytes, slot), pid, lo, hi, nv, D.stride, a.sv,
                         plo, phi);
      child_flag[slot] = 1;
    }
  }
}

__global__ void __launch_bounds__(128) k_bb(DevSet D, const void* chunk, int n, int K,
                                            long long leaf_volume, void* child_out,
                                            int* child_flag, void* leaf_out, int* leaf_flag,
                                            DevStats* dst) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  LaneStats st;
  st.zero();
  if (i < n) {
    for (int j = 0; j < K; ++j) child_flag[(size_t)i * K + j] = 0;
    leaf_flag[i] = 0;
    const Box* in = box_at(const_cast<void*>(chunk), D.box_bytes, i);
    const int pid = in->prob;
    const mk_problem p = D.probs[pid];
    if (is_narrow(p)) {
      if (is_small(p))
        bb_one<int64_t, SMALL_V, SMALL_R>(D, in, pid, p, i, K, leaf_volume, child_out, child_flag,
                                          leaf_out, leaf_flag, st);
      else
        bb_one<int64_t, MK_MAXV, MK_MAXR>(D, in, pid, p, i, K, leaf_volume, child_out, child_flag,
                                          leaf_out, leaf_flag, st);
    } else {
      bb_one<i128, MK_MAXV, MK_MAXR>(D, in, pid, p, i, K, leaf_volume, child_out, child_flag,
                                     leaf_out, leaf_flag, st);
    }
  }
  st.flush_warp(dst);
}

// ---------------------------------------------------------------------------
// warp-wide exhaustive enumeration of one small box: lane l evaluates index
// 32*r + l of round r (index order == witness order); the first round with a
// model gives the lexicographic optimum of the box (lowest such lane).

template <typename T, typename V, int CAPV, int CAPR, int SH = 0>
__device__ void warp_enumerate(const DevSet& D, int pid, const mk_problem& p, const Box* box,
                               LaneStats& st) {
  const int lane = threadIdx.x & 31;
  const int nv = p.nvars;
  V lo[CAPV], hi[CAPV], x[CAPV];
  load_box<T, V>(box, nv, D.stride, lo, hi);
  int skip = 0;
  if (lane == 0) {
    mk_corner(lo, hi, nv, p.maxmask, x);
    skip = inc_dominates<V>(D, pid, p, x) ? 1 : 0;
  }
  skip = __shfl_sync(FULL, skip, 0);
  const unsigned long long vol = (unsigned long long)mk_volume(lo, hi, nv);
  if (lane == 0) {
    st.leaves++;
    st.covered += (double)vol;
  }
  if (skip) return;
  const MkProb P = view(D, pid);
  V R[SH ? 1 : (CAPR < MK_MAXT ? CAPR : MK_MAXT)];   // temporaries only (flags in a register)
  int64_t cnt = 0;
  bool ovf = false;
  unsigned long long found = ~0ull;
  for (unsigned long long base = 0; base < vol; base += 32) {
    const unsigned long long idx = base + lane;
    bool model = false;
    if (idx < vol) {
      mk_decode(lo, hi, nv, p.maxmask, idx, x);
      st.points++;
      if constexpr (SH != 0) {
        model = sh_eval_point(P, x, mk_dyn_sh);
        cnt += p.ninsn;
      } else {
        model = mk_eval_point_t(P, x, R, &ovf, &cnt);
      }
    }
    unsigned m = __ballot_sync(FULL, model);
    if (m) {
      found = base + (unsigned long long)(__ffs(m) - 1);
      break;
    }
  }
  st.insns_leaf += (unsigned long long)cnt;
  if (__any_sync(FULL, ovf) && lane == 0) atomicExch(&D.inc[pid].err, 1);
  if (lane == 0 && found != ~0ull) {
    mk_decode(lo, hi, nv, p.maxmask, found, x);
    inc_offer<V>(D, pid, p, x);
  }
}

template <typename V, int CAPV, int CAPR>
__device__ void leaf_block(const DevSet& D, const Box* in, LaneStats& st) {
  const int pid = in->prob;
  const mk_problem p = D.probs[pid];
  warp_enumerate<i128, V, CAPV, CAPR>(D, pid, p, in, st);
}

// pre-split leaves: one warp per leaf box
// a leaf is enumerated only inside the run's wall budget (device stamp +
// budget); one left over marks its problem undecided
__global__ void __launch_bounds__(128) k_leaf(DevSet D, const void* leaves, int nleaf,
                                              DevStats* dst, const unsigned long long* stamp,
                                              unsigned long long budget_ns, int* pending) {
  const int w = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  LaneStats st;
  st.zero();
  bool late = false;
  if (w < nleaf && (threadIdx.x & 31) == 0) late = globaltimer_ns() > *stamp + budget_ns;
  late = __shfl_sync(FULL, late, 0);
  if (w < nleaf && late) {
    if ((threadIdx.x & 31) == 0)
      pending[box_at(const_cast<void*>(leaves), D.box_bytes, w)->prob] = 1;
  } else if (w < nleaf) {
    const Box* in = box_at(const_cast<void*>(leaves), D.box_bytes, w);
    const mk_problem p = D.probs[in->prob];
    if (is_narrow(p)) {
      if (is_small(p)) leaf_block<int64_t, SMALL_V, SMALL_R>(D, in, st);
      else leaf_block<int64_t, MK_MAXV, MK_MAXR>(D, in, st);
    } else {
      leaf_block<i128, MK_MAXV, MK_MAXR>(D, in, st);
    }
  }
  st.flush_warp(dst);
}


__global__ void k_stamp(unsigned long long* out) { *out = globaltimer_ns(); }

// ---------------------------------------------------------------------------
// persistent warp-granular search

#define SEARCH_THREADS 128
#define WARPS_PER_CTA (SEARCH_THREADS / 32)

struct SearchArgs {
  const void* tasks;
  int ntasks;
  int* ctl;  // [0] task counter, [1] idle units, [2..3] dumped boxes (u64), [4..5] start stamp
  void* stacks;
  long long cap;  // boxes per unit stack
  void* leafbuf;  // 32 boxes per unit
  int K;
  long long leaf_volume;
  unsigned long long budget_ns, slice_ns;
  void* dump;
  long long dump_cap;
  int* pending;
  DevStats* st;
  int units;
  size_t box_bytes;  // class storage (Store<V>)
  int width;         // boxes popped per step (32; 1 in a dive)
  int max_steps;     // steps per task (0: unbounded)
  int dive;          // incumbent dive: no spills, dumps or pending marks
  const int* stop;   // dive: the main search has finished (polled per step)
  int adapt_k;       // widen the splits of a shallow stack (MK_ADAPT_K)
  int group;         // tasks taken per grab; a run of one problem's tasks shares a stack
};

// TASK_DUMPED: redistribution (every task has been handed out), the unit
// ends this launch
enum { TASK_DONE = 0, TASK_ABORT = 1, TASK_DUMPED = 2 };

// copy the unit's stack [0, top) to the global dump buffer; returns false
// when the dump buffer cannot take it.  The reservation is one atomicAdd (no
// CAS retry storm when every unit dumps at once); a reservation that runs past
// the buffer end marks its in-range slots empty (prob = -1) so the next
// launch skips them, and the host clamps the count to the capacity.
// warp-wide copy of n int4 words with 4 loads in flight per lane (stack
// spills and dumps move megabytes; one dependent load per iteration made a
// spill a multi-millisecond step)
__device__ __forceinline__ void warp_copy16(int4* __restrict__ dst, const int4* __restrict__ src,
                                            size_t n) {
  const int lane = threadIdx.x & 31;
  size_t w = lane;
  for (; w + 96 < n; w += 128) {
    const int4 a = src[w], b = src[w + 32], c = src[w + 64], d = src[w + 96];
    dst[w] = a;
    dst[w + 32] = b;
    dst[w + 64] = c;
    dst[w + 96] = d;
  }
  for (; w < n; w += 32) dst[w] = src[w];
}

__device__ bool dump_stack(const SearchArgs& A, const DevSet& D, char* stack, long long top) {
  const int lane = threadIdx.x & 31;
  unsigned long long off = 0;
  if (lane == 0)
    off = atomicAdd(reinterpret_cast<unsigned long long*>(A.ctl + 2), (unsigned long long)top);
  off = __shfl_sync(FULL, off, 0);
  const unsigned long long cap = (unsigned long long)A.dump_cap;
  if (off + (unsigned long long)top > cap) {
    for (unsigned long long i = off + lane; i < cap; i += 32)
      box_at(A.dump, A.box_bytes, (size_t)i)->prob = -1;
    return false;
  }
  const size_t words = A.box_bytes / sizeof(int4);
  const int4* src = reinterpret_cast<const int4*>(stack);
  int4* dst = reinterpret_cast<int4*>(static_cast<char*>(A.dump) + (size_t)off * A.box_bytes);
  warp_copy16(dst, src, (size_t)top * words);
  return true;
}

template <typename V, int CAPV, int CAPR, int SH = 0>
__device__ int search_task(const SearchArgs& A, const DevSet& D, int pid, const mk_problem& p,
                           char* stack, char* leaves, unsigned long long t_start,
                           LaneStats& st, long long top0 = 1) {
  const int lane = threadIdx.x & 31;
  const int nv = p.nvars;
  const int K = A.K;
  const unsigned long long deadline_ns = t_start + A.budget_ns;
  long long top = top0;
  int steps = 0;
  while (top > 0) {
    long long room = A.cap - top;
    long long n = top < A.width ? top : A.width;
    const bool wide = A.width > 1 && top < 2 * A.width;
    long long fit = room / ((wide ? MAX_CHILDREN : K) - 1);
    if (fit < n) n = fit;
    if (n < 1 && A.dive) return TASK_DONE;
    if (n < 1) {
      // past the deadline a full stack is not spilled: the task is undecided
      {
        int lt = 0;
        if (lane == 0) lt = globaltimer_ns() > deadline_ns;
        if (__shfl_sync(FULL, lt, 0)) return TASK_ABORT;
      }
      // stack full: the bottom (worst) half goes to the next launch's task
      // list, the unit keeps searching its best half
      const long long spill = top - top / 2;
      if (!dump_stack(A, D, stack, spill)) {
        if (lane == 0) atomicExch(&D.inc[pid].err, 1);
        return TASK_DONE;
      }
      const size_t words = A.box_bytes / sizeof(int4);
      const int4* src = reinterpret_cast<const int4*>(stack + (size_t)spill * A.box_bytes);
      int4* dst = reinterpret_cast<int4*>(stack);
      // (top - spill) <= spill boxes: source and destination do not overlap
      warp_copy16(dst, src, (size_t)(top - spill) * words);
      __syncwarp();
      top -= spill;
      continue;
    }
    const long long base = top - n;
    if (lane == 0) st.steps++;
    V lo[CAPV], hi[CAPV];
    Act a;
    a.kind = ACT_DONE;
    a.m = 0;
    a.sv = -1;
    if (lane < n) {
      load_box<V, V>(box_at(stack, A.box_bytes, (size_t)(base + lane)), nv, D.stride, lo, hi);
      // a shallow stack splits wider so the next step fills the warp:
      // n boxes popped -> up to 32 / n pieces each (A.adapt_k)
      int Ke = K;
      if (A.adapt_k && wide && n * K < 32) Ke = (int)(32 / n) < MAX_CHILDREN ? (int)(32 / n) : MAX_CHILDREN;
      a = process_box<V, CAPV, CAPR, SH>(D, pid, p, lo, hi, Ke, A.leaf_volume, st, wide);
    }
    const int nch = a.kind == ACT_SPLIT ? a.m * a.m2 : 0;
    int incl = nch;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int ctot = __shfl_sync(FULL, incl, 31);
    const int coff = incl - nch;
    const unsigned leafmask = __ballot_sync(FULL, a.kind == ACT_LEAF);
    __syncwarp();  // every popped box has been read: its slot may be reused
    if (nch && a.sv2 < 0) {
      bool mx = (p.maxmask >> a.sv) & 1;
      for (int j = 0; j < a.m; ++j) {
        V plo, phi;
        mk_piece(lo[a.sv], hi[a.sv], a.m, a.m - 1 - j, mx, &plo, &phi);  // worst first
        write_box<V, V>(box_at(stack, A.box_bytes, (size_t)(base + coff + j)), pid, lo, hi, nv,
                        D.stride, a.sv, plo, phi);
      }
    } else if (nch) {
      // product split: children in lexicographic order of (earlier symbol's
      // piece, later symbol's piece), best on top of the stack
      const int s1 = a.sv < a.sv2 ? a.sv : a.sv2, s2 = a.sv < a.sv2 ? a.sv2 : a.sv;
      const int m1 = s1 == a.sv ? a.m : a.m2, m2 = s1 == a.sv ? a.m2 : a.m;
      const bool mx1 = (p.maxmask >> s1) & 1, mx2 = (p.maxmask >> s2) & 1;
      const V lo1 = lo[s1], hi1 = hi[s1], lo2 = lo[s2], hi2 = hi[s2];
      for (int j = 0; j < nch; ++j) {
        const int t = nch - 1 - j;  // worst first
        V plo, phi;
        mk_piece(lo1, hi1, m1, t / m2, mx1, &plo, &phi);
        lo[s1] = plo;
        hi[s1] = phi;
        mk_piece(lo2, hi2, m2, t % m2, mx2, &plo, &phi);
        write_box<V, V>(box_at(stack, A.box_bytes, (size_t)(base + coff + j)), pid, lo, hi, nv,
                        D.stride, s2, plo, phi);
      }
      lo[s1] = lo1;
      hi[s1] = hi1;
    }
    if (a.kind == ACT_LEAF) {
      const int loff = __popc(leafmask & ((1u << lane) - 1u));
      write_box<V, V>(box_at(leaves, A.box_bytes, loff), pid, lo, hi, nv, D.stride, -1, 0, 0);
    }
    __syncwarp();
    top = base + ctot;
    const int nleaf = __popc(leafmask);
    bool late = false;
    for (int l = 0; l < nleaf; ++l) {
      // past the deadline the remaining leaves are not enumerated (the
      // problem is undecided): one step never runs long over the budget
      int lt = 0;
      if (lane == 0 && l > 0) lt = globaltimer_ns() > deadline_ns;
      if (__shfl_sync(FULL, lt, 0)) {
        late = true;
        break;
      }
      warp_enumerate<V, V, CAPV, CAPR, SH>(D, pid, p, box_at(leaves, A.box_bytes, l), st);
    }
    if (late) return TASK_ABORT;
    int ctlw = 0;
    if (lane == 0) {
      unsigned long long now = globaltimer_ns();
      if (now > deadline_ns) ctlw = 1;
      // hand the remaining subtrees back when a quarter of the units idles
      int idle = *((volatile int*)(A.ctl + 1));
      if (!ctlw && !A.dive && top > 0 && idle * 4 >= A.units && now - t_start > A.slice_ns)
        ctlw = 2;
    }
    if (A.dive && lane == 0 && *((volatile const int*)A.stop)) ctlw = 3;
    ctlw = __shfl_sync(FULL, ctlw, 0);
    if (ctlw == 3) return TASK_DONE;
    if (A.max_steps && ++steps >= A.max_steps) return TASK_DONE;
    if (ctlw == 1) return top > 0 ? TASK_ABORT : TASK_DONE;
    // a redistribution dump that does not fit simply keeps searching
    if (ctlw == 2 && dump_stack(A, D, stack, top)) return TASK_DUMPED;
  }
  return TASK_DONE;
}

// resident CTAs per SM the register allocation is bounded for (occupancy
// vs. spills; measured)
#ifndef MK_MINB_NARROW
#define MK_MINB_NARROW 4
#endif
#ifndef MK_MINB_WIDE
#define MK_MINB_WIDE 2
#endif
template <typename V>
struct MinBlocks {
  static constexpr int value = MkNum<V>::kWide ? MK_MINB_WIDE : MK_MINB_NARROW;
};

template <typename V>
__global__ void __launch_bounds__(SEARCH_THREADS, MinBlocks<V>::value)
    k_search(DevSet D, SearchArgs A) {
  const int lane = threadIdx.x & 31;
  const int unit = blockIdx.x * WARPS_PER_CTA + threadIdx.x / 32;
  const unsigned long long t_start = *reinterpret_cast<const unsigned long long*>(A.ctl + 4);
  char* stack = static_cast<char*>(A.stacks) + (size_t)unit * (size_t)A.cap * A.box_bytes;
  char* leaves = static_cast<char*>(A.leafbuf) + (size_t)unit * 32 * A.box_bytes;
  const size_t words = A.box_bytes / sizeof(int4);
  LaneStats st;
  st.zero();
  const int G = A.group > 1 ? A.group : 1;
  for (;;) {
    int task = 0;
    if (lane == 0) task = atomicAdd(A.ctl, G);
    task = __shfl_sync(FULL, task, 0);
    if (task >= A.ntasks) {
      if (lane == 0) atomicAdd(A.ctl + 1, 1);  // idle from now on
      break;
    }
    const int tend = task + G < A.ntasks ? task + G : A.ntasks;
    bool dumped = false;
    // tasks are taken best-first (the top of the task stack); a run of
    // consecutive tasks of one problem is searched as one stack -- task box
    // ntasks-1-t for task t, so the run's boxes are contiguous, worst first,
    // exactly the stack order -- which fills the warp's lanes from the
    // first step instead of one root box per unit
    // the grab's problem ids, one per lane, read in parallel (G <= 32)
    const int cnt = tend - task;
    int my_pid = -2;
    if (lane < cnt)
      my_pid = box_at(const_cast<void*>(A.tasks), A.box_bytes, (size_t)(A.ntasks - 1 - task - lane))->prob;
    for (int t = task; t < tend;) {
      const int off = t - task;
      const int pid = __shfl_sync(FULL, my_pid, off);
      // the run: consecutive lanes from `off` holding the same problem
      const unsigned same = __ballot_sync(FULL, lane >= off && lane < cnt && my_pid == pid);
      const unsigned rest = ~(same >> off);
      const int len = rest ? __ffs(rest) - 1 : 32 - off;
      if (dumped) {
        // this unit's launch ended: the rest of its grab goes to the dump
        if (pid >= 0) {
          const int4* src = reinterpret_cast<const int4*>(
              box_at(const_cast<void*>(A.tasks), A.box_bytes, (size_t)(A.ntasks - t - len)));
          warp_copy16(reinterpret_cast<int4*>(stack), src, words * (size_t)len);
          __syncwarp();
          if (!dump_stack(A, D, stack, len) && lane == 0) atomicExch(&D.inc[pid].err, 1);
          __syncwarp();
        }
        t += len;
        continue;
      }
      const size_t first = (size_t)(A.ntasks - t - len);
      t += len;
      if (pid < 0) continue;  // holes left by a dump that did not fit
      if (globaltimer_ns() > t_start + A.budget_ns) {
        if (lane == 0 && !A.dive) A.pending[pid] = 1;
        continue;
      }
      warp_copy16(reinterpret_cast<int4*>(stack),
                  reinterpret_cast<const int4*>(box_at(const_cast<void*>(A.tasks), A.box_bytes, first)),
                  words * (size_t)len);
      __syncwarp();
      const mk_problem p = D.probs[pid];
      int r;
      if constexpr (!MkNum<V>::kWide) {
        if (is_shreg(p)) r = search_task<V, SMALL_V, SH_R, 1>(A, D, pid, p, stack, leaves, t_start, st, len);
        else if (is_small(p)) r = search_task<V, SMALL_V, SMALL_R>(A, D, pid, p, stack, leaves, t_start, st, len);
        else r = search_task<V, MK_MAXV, MK_MAXR>(A, D, pid, p, stack, leaves, t_start, st, len);
      } else {
        if (is_small(p)) r = search_task<V, SMALL_V, SMALL_R>(A, D, pid, p, stack, leaves, t_start, st, len);
        else r = search_task<V, MK_MAXV, MK_MAXR>(A, D, pid, p, stack, leaves, t_start, st, len);
      }
      if (r == TASK_ABORT && lane == 0 && !A.dive) A.pending[pid] = 1;
      if (r == TASK_DUMPED) dumped = true;  // the launch ends for the unit; the host redistributes
    }
    if (dumped) break;
  }
  st.flush_warp(A.st);
}

// problems that still own boxes when the budget runs out are undecided
__global__ void k_mark_pending(const void* stack, size_t box_bytes, long long top, int* pending) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= top) return;
  const Box* b = box_at(const_cast<void*>(stack), box_bytes, (size_t)i);
  if (b->prob >= 0) pending[b->prob] = 1;
}

// flag[i] = box i belongs to a problem of class `narrow` (1) / wide (0)
__global__ void k_class_flags(DevSet D, const void* boxes, long long n, int narrow, int* flag) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Box* b = box_at(const_cast<void*>(boxes), D.box_bytes, (size_t)i);
  flag[i] = (((D.probs[b->prob].flags & MK_PF_NARROW) != 0) == (narrow != 0)) ? 1 : 0;
}

// move flagged fixed-size box records to their scanned positions; the last
// thread also publishes the selected count
__global__ void k_scatter(const char* src, const int* flag, const int* pos, long long n, char* dst,
                          size_t box_bytes, int* count) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == n - 1) *count = pos[i] + flag[i];
  if (!flag[i]) return;
  const int4* s = reinterpret_cast<const int4*>(src + (size_t)i * box_bytes);
  int4* d = reinterpret_cast<int4*>(dst + (size_t)pos[i] * box_bytes);
  for (size_t w = 0; w < box_bytes / sizeof(int4); ++w) d[w] = s[w];
}

// partition: box i of the int128 pre-split stack goes, converted to the
// class storage T, to slot pos[i] when flagged; the last thread publishes
// the selected count
template <typename T>
__global__ void k_to_class(DevSet D, const char* src, const int* flag, const int* pos,
                           long long n, char* dst, int* count) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == n - 1) *count = pos[i] + flag[i];
  if (!flag[i]) return;
  const Box* in = reinterpret_cast<const Box*>(src + (size_t)i * D.box_bytes);
  Box* out = reinterpret_cast<Box*>(dst + (size_t)pos[i] * box_bytes_of<T>(D.stride));
  const int nv = D.probs[in->prob].nvars;
  T lo[MK_MAXV], hi[MK_MAXV];
  load_box<i128, T>(in, nv, D.stride, lo, hi);
  write_box<T, T>(out, in->prob, lo, hi, nv, D.stride, -1, 0, 0);
}

}  // namespace

struct mk_dset {
  void* d = nullptr;
  size_t cap = 0;
  int nprob = 0, S = 1, nvar_total = 0;
  size_t o_probs, o_insn, o_const, o_ar, o_am, o_rows, o_terms, o_vlo, o_vhi, o_best, o_inc,
      o_pend, o_stats, o_counts;
};

struct mk_ctx {
  int device = 0;
  int sms = 148;
  int units[2] = {592, 592};  // search units (warps) of the wide [0] / narrow [1] grid
  int ctas[2] = {148, 148};
  std::string err;
  cudaStream_t stream = nullptr;
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaStream_t dive[2] = {nullptr, nullptr};  // speculative incumbent dives
  cudaEvent_t ev[12] = {};
  // growable device buffers
  mk_dset scratch;
  void* d_work = nullptr;
  size_t d_work_bytes = 0;
  void* h_pinned = nullptr;
  void* h_race = nullptr;  // device side buffer of the race sweep
  mkjit::Cache jit;        // specialised race generators, by source
};

static int fail(mk_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

#define CK(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return fail(ctx, MK_ECUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

extern "C" int mk_abi_version(void) { return MK_ABI_VERSION; }

extern "C" int mk_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) n = 0;
  if (out) *out = n;
  return n > 0 ? MK_OK : MK_ENODEV;
}

extern "C" int mk_ctx_create(int device, mk_ctx** out) {
  if (!out) return MK_EINVAL;
  *out = nullptr;
  mk_ctx* ctx = new mk_ctx();
  ctx->device = device;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device) {
    delete ctx;
    return MK_ENODEV;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    return MK_ECUDA;
  }
  // the wide evaluators keep their register files in local memory
  cudaDeviceSetLimit(cudaLimitStackSize, 32 * 1024);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return MK_ECUDA;
  }
  for (int c = 0; c < 2; ++c) cudaStreamCreateWithFlags(&ctx->side[c], cudaStreamNonBlocking);
  for (int c = 0; c < 2; ++c) cudaStreamCreateWithFlags(&ctx->dive[c], cudaStreamNonBlocking);
  for (int i = 0; i < 12; ++i) cudaEventCreate(&ctx->ev[i]);
  cudaMallocHost(&ctx->h_pinned, 4096);
  {
    int sms = 0, per_wide = 0, per_narrow = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    // the search kernels keep their register files in local memory: all of
    // the SM's unified L1 / shared storage as L1
    cudaFuncSetAttribute(k_search<i128>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         SH_BYTES ? -1 : 0);
    cudaFuncSetAttribute(k_search<int64_t>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         SH_BYTES ? -1 : 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_wide, k_search<i128>, SEARCH_THREADS, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_narrow, k_search<int64_t>, SEARCH_THREADS,
                                                  SH_BYTES);
    if (per_wide < 1) per_wide = 1;
    if (per_narrow < 1) per_narrow = 1;
    ctx->sms = sms;
    ctx->ctas[0] = sms * per_wide;
    ctx->ctas[1] = sms * per_narrow;
    ctx->units[0] = ctx->ctas[0] * WARPS_PER_CTA;
    ctx->units[1] = ctx->ctas[1] * WARPS_PER_CTA;
  }
  *out = ctx;
  return MK_OK;
}

extern "C" int mk_ctx_destroy(mk_ctx* ctx) {
  if (!ctx) return MK_OK;
  cudaSetDevice(ctx->device);
  if (ctx->d_work) cudaFree(ctx->d_work);
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  if (ctx->h_race) cudaFree(ctx->h_race);
  for (int i = 0; i < 12; ++i)
    if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
  if (ctx->scratch.d) cudaFree(ctx->scratch.d);
  for (int c = 0; c < 2; ++c)
    if (ctx->side[c]) cudaStreamDestroy(ctx->side[c]);
  for (int c = 0; c < 2; ++c)
    if (ctx->dive[c]) cudaStreamDestroy(ctx->dive[c]);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return MK_OK;
}

extern "C" const char* mk_last_error(const mk_ctx* ctx) {
  return ctx ? ctx->err.c_str() : "null context";
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static int ensure(mk_ctx* ctx, void** buf, size_t* cap, size_t need) {
  if (*cap >= need) return MK_OK;
  if (*buf) cudaFree(*buf);
  *buf = nullptr;
  size_t want = need + need / 4;
  cudaError_t e = cudaMalloc(buf, want);
  if (e != cudaSuccess) {
    *cap = 0;
    return fail(ctx, MK_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  *cap = want;
  return MK_OK;
}

// search = false: a race / access program (its evaluators keep the whole
// register file, no temporaries limit)
static int upload_set(mk_ctx* ctx, const mk_problem_set* set, mk_dset* ds, bool search = true) {
  const int nprob = set->nprob;
  int S = 1;
  for (int i = 0; i < nprob; ++i) {
    const mk_problem& p = set->probs[i];
    if (p.nvars > MK_MAXV || p.nregs > MK_MAXR ||
        (search && p.nregs - p.nvars - p.nconst > MK_MAXT))
      return fail(ctx, MK_EINVAL,
                  "problem exceeds MK_MAXV symbols, MK_MAXR registers or MK_MAXT temporaries");
    if (p.nvars > S) S = p.nvars;
  }
  size_t off = 0;
  auto place = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  ds->o_probs = place(sizeof(mk_problem) * (nprob + 1));
  ds->o_insn = place(sizeof(mk_insn) * (size_t)set->ninsn_total + 16);
  ds->o_const = place(sizeof(mk_i128) * (size_t)set->nconst_total + 16);
  ds->o_ar = place(sizeof(int32_t) * (size_t)set->natom_total + 16);
  ds->o_am = place(sizeof(uint64_t) * (size_t)set->natom_total + 16);
  ds->o_rows = place(sizeof(mk_row) * (size_t)set->nrow_total + 16);
  ds->o_terms = place(sizeof(mk_row_term) * (size_t)set->nterm_total + 16);
  ds->o_vlo = place(sizeof(mk_i128) * (size_t)set->nvar_total + 16);
  ds->o_vhi = place(sizeof(mk_i128) * (size_t)set->nvar_total + 16);
  ds->o_best = place(sizeof(mk_i128) * (size_t)set->nvar_total + 16);
  ds->o_inc = place(sizeof(Incumbent) * (nprob + 1));
  ds->o_pend = place(sizeof(int) * (nprob + 1));
  ds->o_stats = place(sizeof(DevStats));
  ds->o_counts = place(sizeof(int) * 8);
  int rc = ensure(ctx, &ds->d, &ds->cap, off);
  if (rc) return rc;
  ds->nprob = nprob;
  ds->S = S;
  ds->nvar_total = set->nvar_total;
  char* base = static_cast<char*>(ds->d);
  cudaStream_t s = ctx->stream;
  auto h2d = [&](size_t o, const void* src, size_t bytes) -> cudaError_t {
    if (!bytes || !src) return cudaSuccess;
    return cudaMemcpyAsync(base + o, src, bytes, cudaMemcpyHostToDevice, s);
  };
  CK(h2d(ds->o_probs, set->probs, sizeof(mk_problem) * nprob));
  CK(h2d(ds->o_insn, set->insns, sizeof(mk_insn) * (size_t)set->ninsn_total));
  CK(h2d(ds->o_const, set->consts, sizeof(mk_i128) * (size_t)set->nconst_total));
  CK(h2d(ds->o_ar, set->atom_regs, sizeof(int32_t) * (size_t)set->natom_total));
  CK(h2d(ds->o_am, set->atom_masks, sizeof(uint64_t) * (size_t)set->natom_total));
  CK(h2d(ds->o_rows, set->rows, sizeof(mk_row) * (size_t)set->nrow_total));
  CK(h2d(ds->o_terms, set->row_terms, sizeof(mk_row_term) * (size_t)set->nterm_total));
  CK(h2d(ds->o_vlo, set->var_lo, sizeof(mk_i128) * (size_t)set->nvar_total));
  CK(h2d(ds->o_vhi, set->var_hi, sizeof(mk_i128) * (size_t)set->nvar_total));
  return MK_OK;
}

// one persistent search class (0 = wide / int128, 1 = narrow / int64)
struct ClassRun {
  void* tasks;
  void* dump;
  long long ntasks;
  int* ctl;
  void* stacks;
  void* leafbuf;
  long long cap;
  int launches;
  double ms;
};

static int run_set(mk_ctx* ctx, mk_dset* ds, const mk_limits* lim, int32_t* status,
                   mk_i128* point, mk_stats* stats, std::chrono::steady_clock::time_point t0,
                   bool keep_incumbents = false, bool* budget_out = nullptr) {
  mk_stats local_stats;
  std::memset(&local_stats, 0, sizeof(local_stats));
  const int nprob = ds->nprob;
  const int S = ds->S;
  int64_t max_rounds = lim && lim->max_rounds > 0 ? lim->max_rounds : 200000;
  int64_t max_boxes = lim && lim->max_boxes > 0 ? lim->max_boxes : (int64_t)4e9;
  double max_seconds = lim && lim->max_seconds > 0 ? lim->max_seconds : 30.0;
  // split arity, measured on the B200 (profiles/r02_split_knobs_after_kernel_work.jsonl,
  // r02_split_k_final.jsonl): 8 was best with four contraction sweeps per
  // box; with one sweep, 12 (full sets: config3 13.6 -> 9.1 ms, paged
  // attention v2 long 12.0 -> 10.4, moe_align equal)
  int K = 12;
  if (const char* e = getenv("MK_SPLIT_K")) K = atoi(e) > 1 ? atoi(e) : K;
  // widen the splits of shallow stacks (measured: config3 40 -> 32 ms,
  // racy 8.7 -> 4.6 ms, the rest within noise; profiles/r02_adapt_k.jsonl)
  int adapt_k = 1;
  if (const char* e = getenv("MK_ADAPT_K")) adapt_k = atoi(e);
  // most tasks a unit grabs at once (k_search; 1 = one root per grab)
  long long group_cap = 16;   // measured: profiles/r02_task_group.jsonl
  if (const char* e = getenv("MK_TASK_GROUP")) group_cap = atoi(e) > 0 ? atoi(e) : 1;
  if (group_cap > 32) group_cap = 32;   // one task per lane when a grab is scanned
  if (lim && lim->split_k > 1) K = lim->split_k;
  int chunk = lim && lim->chunk > 0 ? lim->chunk : 65536;
  long long leaf_volume = lim && lim->leaf_volume > 0 ? lim->leaf_volume : 4096;
  // incumbent dive: steps of width 1 from every root before the search
  // (mk_limits.chunk < -1 disables it; a model found early prunes the
  // parallel search, whose units would otherwise explore worse subtrees)
  const int dive_steps = lim && lim->chunk < -1 ? 0 : 4096;
  const size_t box_bytes = sizeof(Box) + 2 * sizeof(mk_i128) * (size_t)S;
  char* base = static_cast<char*>(ds->d);
  cudaStream_t s = ctx->stream;
  int64_t launches = 0;
  CK(cudaEventRecord(ctx->ev[4], s));
  CK(cudaMemsetAsync(base + ds->o_pend, 0, sizeof(int) * nprob, s));
  CK(cudaMemsetAsync(base + ds->o_stats, 0, sizeof(DevStats), s));

  DevSet D;
  D.probs = reinterpret_cast<const mk_problem*>(base + ds->o_probs);
  D.insns = reinterpret_cast<const mk_insn*>(base + ds->o_insn);
  D.consts = reinterpret_cast<const mk_i128*>(base + ds->o_const);
  D.atom_regs = reinterpret_cast<const int32_t*>(base + ds->o_ar);
  D.atom_masks = reinterpret_cast<const uint64_t*>(base + ds->o_am);
  D.rows = reinterpret_cast<const mk_row*>(base + ds->o_rows);
  D.terms = reinterpret_cast<const mk_row_term*>(base + ds->o_terms);
  D.var_lo = reinterpret_cast<const mk_i128*>(base + ds->o_vlo);
  D.var_hi = reinterpret_cast<const mk_i128*>(base + ds->o_vhi);
  D.inc = reinterpret_cast<Incumbent*>(base + ds->o_inc);
  D.best = reinterpret_cast<mk_i128*>(base + ds->o_best);
  D.stride = S;
  D.box_bytes = box_bytes;
  DevStats* d_st = reinterpret_cast<DevStats*>(base + ds->o_stats);
  int* d_counts = reinterpret_cast<int*>(base + ds->o_counts);
  int* d_pend = reinterpret_cast<int*>(base + ds->o_pend);
  int rc = MK_OK;

  // ---- work buffers: pre-split stack, child/leaf staging, flags, cub
  // scratch, and per class: task/dump buffers, unit stacks, leaf lists
  size_t cap_boxes = ((size_t)2 << 30) / box_bytes;  // 2 GiB of pre-split stack in HBM
  if (cap_boxes < (size_t)nprob + (size_t)chunk * K) cap_boxes = (size_t)nprob + (size_t)chunk * K;
  // per class c (0 = wide / int128 storage, 1 = narrow / int64 storage)
  const size_t cbytes[2] = {box_bytes_of<i128>(S), box_bytes_of<int64_t>(S)};
  size_t cls_cap[2];
  for (int c = 0; c < 2; ++c) cls_cap[c] = ((size_t)1 << 30) / cbytes[c];  // 1 GiB per task / dump buffer
  size_t scan_n = (size_t)chunk * K;
  if (scan_n < cap_boxes) scan_n = cap_boxes;
  size_t cub_bytes = 0;
  {
    size_t t1 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t1, (const int*)nullptr, (int*)nullptr, (int)scan_n, s);
    cub_bytes = t1;
  }
  size_t w = 0;
  auto wplace = [&](size_t bytes) {
    size_t o = w;
    w = align_up(w + bytes, 256);
    return o;
  };
  size_t w_stack = wplace(box_bytes * cap_boxes);
  size_t w_child = wplace(box_bytes * (size_t)chunk * K);
  size_t w_cflag = wplace(sizeof(int) * scan_n);
  size_t w_cpos = wplace(sizeof(int) * scan_n);
  size_t w_leaf = wplace(box_bytes * (size_t)chunk);
  size_t w_lflag = wplace(sizeof(int) * (size_t)chunk);
  size_t w_lpos = wplace(sizeof(int) * (size_t)chunk);
  size_t w_leaves = wplace(box_bytes * (size_t)chunk);
  size_t w_cub = wplace(cub_bytes + 256);
  size_t w_cls[2][6];
  size_t w_dive[2][4];
  long long unit_cap[2];
  for (int c = 0; c < 2; ++c) {
    const int units = ctx->units[c];
    long long cap = (long long)(((size_t)3 << 30) / ((size_t)units * cbytes[c]));
    if (cap > 16384) cap = 16384;
    if (cap < 8 * 32) cap = 8 * 32;
    if (lim && lim->unit_stack > 0) cap = lim->unit_stack < 32 ? 32 : lim->unit_stack;
    unit_cap[c] = cap;
    w_cls[c][0] = wplace(cbytes[c] * cls_cap[c]);                    // tasks
    w_cls[c][1] = wplace(cbytes[c] * cls_cap[c]);                    // dump
    w_cls[c][2] = wplace(cbytes[c] * (size_t)cap * units);           // unit stacks
    w_cls[c][3] = wplace(cbytes[c] * (size_t)32 * units);            // unit leaf lists
    w_cls[c][4] = wplace(sizeof(int) * 8);                           // control block
    w_dive[c][0] = wplace(cbytes[c] * (size_t)(nprob + 1));          // dive tasks (roots)
    w_dive[c][1] = wplace(cbytes[c] * (size_t)DIVE_CAP * (nprob + 4)); // dive stacks
    w_dive[c][2] = wplace(cbytes[c] * (size_t)32 * (nprob + 4));     // dive leaf lists
    w_dive[c][3] = wplace(sizeof(int) * 8);                          // dive control block
  }
  const size_t w_stop = wplace(sizeof(int) * 8);
  rc = ensure(ctx, &ctx->d_work, &ctx->d_work_bytes, w);
  if (rc) return rc;
  char* wb = static_cast<char*>(ctx->d_work);
  void* stack = wb + w_stack;
  char* child = wb + w_child;
  int* cflag = reinterpret_cast<int*>(wb + w_cflag);
  int* cpos = reinterpret_cast<int*>(wb + w_cpos);
  char* leafst = wb + w_leaf;
  int* lflag = reinterpret_cast<int*>(wb + w_lflag);
  int* lpos = reinterpret_cast<int*>(wb + w_lpos);
  char* leaves = wb + w_leaves;
  void* cub_tmp = wb + w_cub;
  int* d_stop = reinterpret_cast<int*>(wb + w_stop);
  // device stamp of the run's start (the pre-split leaves' wall budget)
  unsigned long long* run_stamp = reinterpret_cast<unsigned long long*>(d_stop + 2);
  k_stamp<<<1, 1, 0, s>>>(run_stamp);
  ++launches;
  ClassRun cls[2];
  for (int c = 0; c < 2; ++c) {
    cls[c].tasks = wb + w_cls[c][0];
    cls[c].dump = wb + w_cls[c][1];
    cls[c].stacks = wb + w_cls[c][2];
    cls[c].leafbuf = wb + w_cls[c][3];
    cls[c].ctl = reinterpret_cast<int*>(wb + w_cls[c][4]);
    cls[c].cap = unit_cap[c];
    cls[c].ntasks = 0;
    cls[c].launches = 0;
    cls[c].ms = 0.0;
  }
  // pre-split until every unit of the larger persistent grid has a task
  long long presplit_target =
      lim && lim->chunk < 0 ? 0
                            : (long long)(ctx->units[1] > ctx->units[0] ? ctx->units[1] : ctx->units[0]);
  if (const char* e = getenv("MK_PRESPLIT_TARGET")) presplit_target = atoll(e);

  k_roots<<<(nprob + 127) / 128, 128, 0, s>>>(D, nprob, stack, keep_incumbents ? 1 : 0);
  ++launches;
  CK(cudaGetLastError());
  {
    // off by default: measured on the B200 with the host presolve's bound
    // tightening on, a contracted root changes the split order and slows some
    // searches (fused_add_rms_norm 0.8 -> 4.2 ms); with the host tightening
    // off it does not recover the host-presolved speed
    int sweeps = 0;
    if (const char* e = getenv("MK_ROOT_SWEEPS")) sweeps = atoi(e);
    if (sweeps > 0) {
      k_root_contract<<<(nprob + 63) / 64, 64, 0, s>>>(D, nprob, stack, sweeps);
      ++launches;
      CK(cudaGetLastError());
    }
  }
  long long top = nprob;
  int* h_counts = static_cast<int*>(ctx->h_pinned);
  double dive_ms = 0.0;
  bool diving = false;
  int dive_ctas[2] = {0, 0};
  const unsigned long long dive_budget_ns = 3000000ull;

  // split boxes [0, n) of the int128 stack into the two classes' task lists
  // (class storage); ntasks = -1 when they do not fit
  auto partition_to = [&](long long n, void* const dst[2], long long out[2]) -> int {
    if ((size_t)n > cls_cap[0] || (size_t)n > cls_cap[1]) {
      out[0] = out[1] = -1;
      return MK_OK;
    }
    for (int c = 0; c < 2; ++c) {
      k_class_flags<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(D, stack, n, c, cflag);
      ++launches;
      CK(cudaGetLastError());
      size_t tb = cub_bytes;
      CK(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, cflag, cpos, (int)n, s));
      ++launches;
      if (c == 0)
        k_to_class<i128><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(
            D, static_cast<const char*>(stack), cflag, cpos, n, static_cast<char*>(dst[c]),
            d_counts + 2 + c);
      else
        k_to_class<int64_t><<<(unsigned)((n + 127) / 128), 128, 0, s>>>(
            D, static_cast<const char*>(stack), cflag, cpos, n, static_cast<char*>(dst[c]),
            d_counts + 2 + c);
      ++launches;
      CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(h_counts, d_counts + 2, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    out[0] = h_counts[0];
    out[1] = h_counts[1];
    return MK_OK;
  };
  auto partition = [&](long long n) -> int {
    void* const dst[2] = {cls[0].tasks, cls[1].tasks};
    long long out[2];
    int r = partition_to(n, dst, out);
    cls[0].ntasks = out[0];
    cls[1].ntasks = out[1];
    return r;
  };
  // one launch of both classes' persistent grids on their streams; a dive
  // follows only the best box of each root for a few steps (width 1, no
  // spills or dumps) to seed the incumbents
  auto search_round = [&](double left, bool dive, float* out_ms) -> int {
    CK(cudaEventRecord(ctx->ev[0], s));
    for (int c = 0; c < 2; ++c) {
      if (cls[c].ntasks <= 0) continue;
      cudaStream_t cs = ctx->side[c];
      CK(cudaStreamWaitEvent(cs, ctx->ev[0], 0));
      CK(cudaMemsetAsync(cls[c].ctl, 0, sizeof(int) * 8, cs));
      // the wall budget is checked on the device against %globaltimer,
      // stamped stream-ordered just before the launch
      k_stamp<<<1, 1, 0, cs>>>(reinterpret_cast<unsigned long long*>(cls[c].ctl + 4));
      ++launches;
      SearchArgs A;
      A.adapt_k = adapt_k;
      A.tasks = cls[c].tasks;
      A.ntasks = (int)cls[c].ntasks;
      A.ctl = cls[c].ctl;
      A.stacks = cls[c].stacks;
      A.cap = cls[c].cap;
      A.leafbuf = cls[c].leafbuf;
      A.K = K;
      // a dive enumerates only boxes of at most one warp round of points:
      // larger ones are split further (one box per step is cheap), so a
      // dive never stalls a warp on a long unsat enumeration
      A.leaf_volume = dive ? 32 : leaf_volume;
      A.budget_ns = (unsigned long long)(left * 1e9);
      A.slice_ns = 200000ull;
      A.dump = cls[c].dump;
      A.dump_cap = (long long)cls_cap[c];
      A.box_bytes = cbytes[c];
      A.pending = d_pend;
      A.st = d_st;
      A.units = ctx->units[c];
      A.width = dive ? 1 : 32;
      A.max_steps = dive ? dive_steps : 0;
      A.dive = dive ? 1 : 0;
      A.stop = d_stop;
      // always the full persistent grid: units without a task idle at once,
      // which is what triggers redistribution of a lone deep subtree
      // the persistent grid leaves the slots of a running dive free, so
      // every CTA of it is resident at once
      if (dive_ctas[c] && cudaEventQuery(ctx->ev[8 + c]) == cudaSuccess) dive_ctas[c] = 0;
      int grid = ctx->ctas[c] - dive_ctas[c];
      if (grid < ctx->sms) grid = ctx->sms;
      A.units = grid * WARPS_PER_CTA;
      // tasks per grab: with many more tasks than units, a unit takes a few
      // at once (runs of one problem share its stack); never in a dive
      {
        long long g = dive ? 1 : A.ntasks / (2LL * A.units);
        if (g > group_cap) g = group_cap;
        A.group = g < 1 ? 1 : (int)g;
      }
      if (c == 0) k_search<i128><<<grid, SEARCH_THREADS, 0, cs>>>(D, A);
      else k_search<int64_t><<<grid, SEARCH_THREADS, SH_BYTES, cs>>>(D, A);
      ++launches;
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(h_counts + 4 + 2 * c, cls[c].ctl + 2, sizeof(long long),
                         cudaMemcpyDeviceToHost, cs));
      CK(cudaEventRecord(ctx->ev[6 + c], cs));
      cls[c].launches++;
    }
    for (int c = 0; c < 2; ++c) {
      if (cls[c].ntasks <= 0) continue;
      CK(cudaEventSynchronize(ctx->ev[6 + c]));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[6 + c]);
      cls[c].ms += ms;
      long long dumped = dive ? 0 : *reinterpret_cast<long long*>(h_counts + 4 + 2 * c);
      if (dumped > (long long)cls_cap[c]) dumped = (long long)cls_cap[c];
      cls[c].ntasks = dumped;
      void* tmp = cls[c].tasks;
      cls[c].tasks = cls[c].dump;
      cls[c].dump = tmp;
      CK(cudaStreamWaitEvent(s, ctx->ev[6 + c], 0));
    }
    CK(cudaEventRecord(ctx->ev[1], s));
    CK(cudaEventSynchronize(ctx->ev[1]));
    cudaEventElapsedTime(out_ms, ctx->ev[0], ctx->ev[1]);
    return MK_OK;
  };

  // ---- speculative incumbent dives, one warp per root, concurrent with the
  // pre-split and the parallel search: width-1 best-first DFS (the serial
  // search order) that offers models as soon as it meets them, so the wide
  // search prunes by them; stopped through d_stop when the search is done

  CK(cudaMemsetAsync(d_stop, 0, sizeof(int), s));
  // the roots' class partition made for the dive; the search copies it
  // (device to device) instead of partitioning again when no pre-split
  // round runs in between
  long long dive_nt[2] = {-1, -1};
  if (dive_steps > 0) {
    void* const dst[2] = {wb + w_dive[0][0], wb + w_dive[1][0]};
    long long nt[2];
    rc = partition_to(top, dst, nt);
    if (rc) return rc;
    dive_nt[0] = nt[0];
    dive_nt[1] = nt[1];
    if (nt[0] >= 0) {
      CK(cudaEventRecord(ctx->ev[5], s));
      for (int c = 0; c < 2; ++c) {
        if (nt[c] <= 0) continue;
        cudaStream_t ds = ctx->dive[c];
        CK(cudaStreamWaitEvent(ds, ctx->ev[5], 0));
        int* dctl = reinterpret_cast<int*>(wb + w_dive[c][3]);
        CK(cudaMemsetAsync(dctl, 0, sizeof(int) * 8, ds));
        k_stamp<<<1, 1, 0, ds>>>(reinterpret_cast<unsigned long long*>(dctl + 4));
        ++launches;
        SearchArgs A;
        A.adapt_k = 0;   // a dive pops one box per step by design
        A.group = 1;
        A.tasks = dst[c];
        A.ntasks = (int)nt[c];
        A.ctl = dctl;
        A.stacks = wb + w_dive[c][1];
        A.cap = DIVE_CAP;
        A.leafbuf = wb + w_dive[c][2];
        A.K = K;
        A.leaf_volume = 32;
        // a dive is a heuristic: a fixed time budget bounds what it can
        // cost the step (it exits earlier when its tree is exhausted)
        A.budget_ns = dive_budget_ns;
        A.slice_ns = 200000ull;
        A.dump = nullptr;
        A.dump_cap = 0;
        A.box_bytes = cbytes[c];
        A.pending = d_pend;
        A.st = d_st;
        const int grid = (int)((nt[c] + WARPS_PER_CTA - 1) / WARPS_PER_CTA);
        A.units = grid * WARPS_PER_CTA;
        A.width = 1;
        A.max_steps = dive_steps;
        A.dive = 1;
        A.stop = d_stop;
        if (c == 0) k_search<i128><<<grid, SEARCH_THREADS, 0, ds>>>(D, A);
        else k_search<int64_t><<<grid, SEARCH_THREADS, SH_BYTES, ds>>>(D, A);
        ++launches;
        CK(cudaGetLastError());
        CK(cudaEventRecord(ctx->ev[8 + c], ds));
      }
      diving = true;
      for (int c = 0; c < 2; ++c)
        dive_ctas[c] = nt[c] > 0 ? (int)((nt[c] + WARPS_PER_CTA - 1) / WARPS_PER_CTA) : 0;
    }
  }

  int64_t rounds = 0;
  double bb_ms = 0.0, leaf_ms = 0.0;
  bool budget_hit = false;
  while (top > 0) {
    double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (rounds >= max_rounds || el > max_seconds) {
      budget_hit = true;
      break;
    }
    if (top >= presplit_target) break;  // hand over to the persistent search
    long long room = (long long)cap_boxes - top;
    long long n = top < chunk ? top : chunk;
    // popping n boxes frees n slots and their children need up to n*K:
    // n*(K-1) <= room.  A nearly full stack therefore processes fewer, deeper
    // boxes (LIFO top), which drains it.
    long long fit = room / (K - 1);
    if (fit < n) n = fit;
    if (n < 1) {
      budget_hit = true;
      break;
    }
    long long basei = top - n;
    const void* chunk_ptr = static_cast<char*>(stack) + (size_t)basei * box_bytes;
    CK(cudaEventRecord(ctx->ev[0], s));
    int threads = 128;
    k_bb<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(
        D, chunk_ptr, (int)n, K, leaf_volume, child, cflag, leafst, lflag, d_st);
    ++launches;
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev[1], s));
    top = basei;
    // compact children (order preserving) straight onto the stack top and
    // leaves into the leaf list: exclusive scan of the flags, then scatter
    {
      size_t tb = cub_bytes;
      CK(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, cflag, cpos, (int)(n * K), s));
      ++launches;
      long long nc = n * K;
      k_scatter<<<(unsigned)((nc + 127) / 128), 128, 0, s>>>(
          child, cflag, cpos, nc, static_cast<char*>(stack) + (size_t)top * box_bytes, box_bytes,
          d_counts);
      ++launches;
      CK(cudaGetLastError());
      tb = cub_bytes;
      CK(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, lflag, lpos, (int)n, s));
      ++launches;
      k_scatter<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(leafst, lflag, lpos, n, leaves,
                                                             box_bytes, d_counts + 1);
      ++launches;
      CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(h_counts, d_counts, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    long long nchild = h_counts[0];
    long long nleaf = h_counts[1];
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
    bb_ms += ms;
    if (nleaf > 0) {
      CK(cudaEventRecord(ctx->ev[2], s));
      k_leaf<<<(unsigned)((nleaf + 3) / 4), 128, 0, s>>>(
          D, leaves, (int)nleaf, d_st, run_stamp, (unsigned long long)(max_seconds * 1e9), d_pend);
      ++launches;
      CK(cudaGetLastError());
      CK(cudaEventRecord(ctx->ev[3], s));
      CK(cudaEventSynchronize(ctx->ev[3]));
      cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
      leaf_ms += ms;
    }
    top += nchild;
    ++rounds;
    if (rounds % 64 == 0) {
      unsigned long long nb = 0;
      CK(cudaMemcpy(&nb, &d_st->boxes, sizeof(nb), cudaMemcpyDeviceToHost));
      if ((int64_t)nb > max_boxes) {
        budget_hit = true;
        break;
      }
    }
  }
  // ---- persistent search: both classes concurrently, bulk-synchronous
  // redistribution of dumped subtrees between launches
  double search_ms = 0.0;
  int search_launches = 0;
  if (!budget_hit && top > 0) {
    if (rounds == 0 && dive_nt[0] >= 0) {
      for (int c = 0; c < 2; ++c) {
        cls[c].ntasks = dive_nt[c];
        if (dive_nt[c] > 0)
          CK(cudaMemcpyAsync(cls[c].tasks, wb + w_dive[c][0], cbytes[c] * (size_t)dive_nt[c],
                             cudaMemcpyDeviceToDevice, s));
      }
    } else {
      rc = partition(top);
      if (rc) return rc;
    }
    if (cls[0].ntasks < 0) budget_hit = true;
    else top = 0;
  }
  const char* trace_env = getenv("MK_TRACE_RUN");
  const bool trace = trace_env && *trace_env && *trace_env != '0';
  auto tr_el = [&]() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e3;
  };
  if (trace)
    fprintf(stderr, "[mk] presplit done %.2f ms rounds %lld tasks %lld/%lld\n", tr_el(),
            (long long)rounds, cls[0].ntasks, cls[1].ntasks);
  CK(cudaEventRecord(ctx->ev[5], s));
  for (int c = 0; c < 2; ++c) CK(cudaStreamWaitEvent(ctx->side[c], ctx->ev[5], 0));
  while (!budget_hit && (cls[0].ntasks > 0 || cls[1].ntasks > 0)) {
    double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    double left = max_seconds - el;
    if (left <= 0) {
      budget_hit = true;
      break;
    }
    float ms = 0.f;
    rc = search_round(left, false, &ms);
    if (rc) return rc;
    search_ms += ms;
    ++search_launches;
    if (trace)
      fprintf(stderr, "[mk] search launch %d: %.2f ms (left %.2f ms) -> %.2f ms, next tasks %lld/%lld\n",
              search_launches, ms, left * 1e3, tr_el(), cls[0].ntasks, cls[1].ntasks);
  }
  if (diving) {
    CK(cudaMemsetAsync(d_stop, 1, sizeof(int), s));
    for (int c = 0; c < 2; ++c) CK(cudaStreamWaitEvent(s, ctx->ev[8 + c], 0));
    if (trace) {
      CK(cudaStreamSynchronize(s));
      fprintf(stderr, "[mk] dives joined %.2f ms\n", tr_el());
    }
  }
  for (int c = 0; c < 2; ++c) {
    if (budget_hit && cls[c].ntasks > 0) {
      k_mark_pending<<<(unsigned)((cls[c].ntasks + 255) / 256), 256, 0, s>>>(
          cls[c].tasks, cbytes[c], cls[c].ntasks, d_pend);
      ++launches;
      CK(cudaGetLastError());
    }
  }
  if (budget_hit && top > 0) {
    k_mark_pending<<<(unsigned)((top + 255) / 256), 256, 0, s>>>(stack, box_bytes, top, d_pend);
    ++launches;
    CK(cudaGetLastError());
  }
  // ---- results
  std::vector<Incumbent> inc(nprob);
  std::vector<int> pend(nprob);
  DevStats dst;
  CK(cudaMemcpyAsync(inc.data(), D.inc, sizeof(Incumbent) * nprob, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(pend.data(), d_pend, sizeof(int) * nprob, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(point, D.best, sizeof(mk_i128) * (size_t)ds->nvar_total,
                     cudaMemcpyDeviceToHost, s));
  CK(cudaEventRecord(ctx->ev[5], s));
  CK(cudaMemcpyAsync(&dst, d_st, sizeof(DevStats), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int i = 0; i < nprob; ++i) {
    if (inc[i].err || pend[i]) status[i] = MK_UNKNOWN;
    else status[i] = inc[i].has ? MK_SAT : MK_UNSAT;
  }
  if (budget_out) *budget_out = budget_hit;
  local_stats.rounds = rounds + search_launches;
  local_stats.boxes = (int64_t)dst.boxes;
  local_stats.leaves = (int64_t)dst.leaves;
  local_stats.points = (int64_t)dst.points;
  local_stats.covered = dst.covered;
  local_stats.insns_bb = (int64_t)dst.insns_bb;
  local_stats.insns_leaf = (int64_t)dst.insns_leaf;
  local_stats.bb_ms = bb_ms + search_ms + dive_ms;
  local_stats.leaf_ms = leaf_ms;
  local_stats.seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  {
    float dms = 0.f;
    cudaEventElapsedTime(&dms, ctx->ev[4], ctx->ev[5]);
    local_stats.device_ms = dms;
  }
  local_stats.launches = launches;
  local_stats.steps = (int64_t)dst.steps;
  if (stats) *stats = local_stats;
  return MK_OK;
}

// Search strategy: the pre-split (breadth rounds until every persistent unit
// has a task) pays off on long searches -- one deep unsat core spread over
// the whole grid -- but costs host round trips and explores subtrees an
// early model would prune on short ones.  Unless the caller chose (chunk !=
// 0), a short probe runs first with the roots handed straight to the
// persistent search; if it decides every problem inside its budget that is
// the answer (exact either way: the strategy changes the order, not the
// optimum), otherwise the full strategy runs from scratch.
static int run_adaptive(mk_ctx* ctx, mk_dset* ds, const mk_limits* lim, int32_t* status,
                        mk_i128* point, mk_stats* stats, std::chrono::steady_clock::time_point t0) {
  // a large set (hundreds of sites, e.g. the Fig. 7 port's 862) keeps the
  // units busy from the roots on: the probe would only add its budget
  int probe_max = 256;
  if (const char* e = getenv("MK_PROBE_MAX_PROBLEMS")) probe_max = atoi(e);
  if ((lim && lim->chunk != 0) || getenv("MK_NO_PROBE") || ds->nprob > probe_max)
    return run_set(ctx, ds, lim, status, point, stats, t0);
  // a probe step must check its deadline often: small leaves (a warp
  // enumerates at most 32 leaves per step)
  double probe_s = 0.001;
  if (const char* e = getenv("MK_PROBE_MS")) probe_s = atof(e) / 1e3;
  long long probe_leaf = 512;
  if (const char* e = getenv("MK_PROBE_LEAF")) probe_leaf = atoll(e);
  mk_limits probe;
  std::memset(&probe, 0, sizeof(probe));
  if (lim) probe = *lim;
  const double max_s = lim && lim->max_seconds > 0 ? lim->max_seconds : 30.0;
  probe.chunk = -1;
  probe.max_seconds = probe_s < max_s ? probe_s : max_s;
  if (!(lim && lim->leaf_volume > 0)) probe.leaf_volume = probe_leaf;
  mk_stats s1, s2;
  bool hit = false;
  int rc = run_set(ctx, ds, &probe, status, point, &s1, t0, false, &hit);
  bool undecided = false;
  for (int i = 0; i < ds->nprob; ++i) undecided |= status[i] == MK_UNKNOWN;
  if (rc || (!hit && !undecided) || probe.max_seconds >= max_s) {
    s1.strategy = 1;
    if (stats) *stats = s1;
    return rc;
  }
  // a fresh full run: its search order (first-fail splits before any model)
  // is the one the long searches are tuned for
  rc = run_set(ctx, ds, lim, status, point, &s2, t0, false, nullptr);
  if (rc) return rc;
  if (stats) {
    s2.rounds += s1.rounds;
    s2.boxes += s1.boxes;
    s2.leaves += s1.leaves;
    s2.points += s1.points;
    s2.covered += s1.covered;
    s2.bb_ms += s1.bb_ms;
    s2.leaf_ms += s1.leaf_ms;
    s2.insns_bb += s1.insns_bb;
    s2.insns_leaf += s1.insns_leaf;
    s2.device_ms += s1.device_ms;
    s2.launches += s1.launches;
    s2.steps += s1.steps;
    s2.strategy = 2;
    *stats = s2;
  }
  return MK_OK;
}

extern "C" int mk_set_upload(mk_ctx* ctx, const mk_problem_set* set, mk_dset** out) {
  if (!ctx || !set || !out) return fail(ctx, MK_EINVAL, "null argument");
  CK(cudaSetDevice(ctx->device));
  mk_dset* ds = new mk_dset();
  int rc = upload_set(ctx, set, ds);
  if (rc) {
    if (ds->d) cudaFree(ds->d);
    delete ds;
    return rc;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  *out = ds;
  return MK_OK;
}

extern "C" int mk_set_free(mk_ctx* ctx, mk_dset* ds) {
  if (!ds) return MK_OK;
  if (ctx) cudaSetDevice(ctx->device);
  if (ds->d) cudaFree(ds->d);
  delete ds;
  return MK_OK;
}

extern "C" int mk_set_eval(mk_ctx* ctx, mk_dset* ds, const mk_limits* lim, int32_t* status,
                           mk_i128* point, mk_stats* stats) {
  if (!ctx || !ds || !status || !point) return fail(ctx, MK_EINVAL, "null argument");
  auto t0 = std::chrono::steady_clock::now();
  CK(cudaSetDevice(ctx->device));
  if (ds->nprob <= 0) {
    if (stats) std::memset(stats, 0, sizeof(*stats));
    return MK_OK;
  }
  return run_adaptive(ctx, ds, lim, status, point, stats, t0);
}

extern "C" int mk_site_eval(mk_ctx* ctx, const mk_problem_set* set, const mk_limits* lim,
                            int32_t* status, mk_i128* point, mk_stats* stats) {
  if (!ctx || !set || !status || !point) return fail(ctx, MK_EINVAL, "null argument");
  auto t0 = std::chrono::steady_clock::now();
  CK(cudaSetDevice(ctx->device));
  if (set->nprob <= 0) {
    if (stats) std::memset(stats, 0, sizeof(*stats));
    return MK_OK;
  }
  // one-shot: the context's scratch set is reused across calls
  int rc = upload_set(ctx, set, &ctx->scratch);
  if (rc) return rc;
  return run_adaptive(ctx, &ctx->scratch, lim, status, point, stats, t0);
}

// -- INT32 issue microbenchmark (roofline denominator) --------------------------------
// 8 independent chains per thread; each step of a chain is four PTX integer
// instructions kept verbatim by asm volatile -- add (IADD3), lop3 (LOP3),
// min (VIMNMX) and mad.lo (IMAD) -- so one step retires exactly 4 integer
// thread-instructions (the SASS count is in profiles/int_peak_r02.json).
// Seeds come from the launch arguments and the result is stored under a
// condition that never holds at run time, so nothing is folded away.
namespace {
constexpr int kPeakChains = 8;
constexpr int kPeakOpsPerStep = 4;
__global__ void __launch_bounds__(256) k_int_peak(uint32_t seed, int iters, uint32_t* sink) {
  uint32_t a[kPeakChains], b[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) {
    a[c] = seed ^ (threadIdx.x * 0x9e3779b9u + c);
    b[c] = seed + blockIdx.x * 7u + c;
  }
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) {
      uint32_t x, y, z;
      asm volatile("add.u32 %0, %1, %2;" : "=r"(x) : "r"(a[c]), "r"(b[c]));
      asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(y) : "r"(x), "r"(b[c]), "r"(a[c]));
      asm volatile("min.u32 %0, %1, %2;" : "=r"(z) : "r"(y), "r"(x));
      asm volatile("mad.lo.u32 %0, %1, 16777619, %2;" : "=r"(a[c]) : "r"(z), "r"(y));
      b[c] = x;
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) acc ^= a[c] ^ b[c];
  if (acc == 0x7fffffffu && seed == 0x12345u) sink[0] = acc;
}
}  // namespace

extern "C" int mk_int_peak(mk_ctx* ctx, double* ops_per_s, double* ms) {
  if (!ctx || !ops_per_s) return fail(ctx, MK_EINVAL, "null argument");
  CK(cudaSetDevice(ctx->device));
  uint32_t* sink = nullptr;
  CK(cudaMalloc(&sink, 64));
  const int threads = 256, ctas = ctx->sms * 4, iters = 1 << 14;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  k_int_peak<<<ctas, threads, 0, ctx->stream>>>(0x9u, 256, sink);  // warm-up
  CK(cudaEventRecord(e0, ctx->stream));
  k_int_peak<<<ctas, threads, 0, ctx->stream>>>(0x9u, iters, sink);
  CK(cudaEventRecord(e1, ctx->stream));
  CK(cudaEventSynchronize(e1));
  float t = 0.f;
  CK(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  double ops = (double)ctas * threads * iters * kPeakChains * kPeakOpsPerStep;
  *ops_per_s = ops / (t * 1e-3);
  if (ms) *ms = t;
  return MK_OK;
}

#include "mk_race.cuh"
#include "mk_access.cuh"

extern "C" int mk_sort_pairs_u64(mk_ctx* ctx, uint64_t* keys, uint64_t* vals, uint64_t n,
                                 int32_t bits, int32_t force, double* ms, int32_t* passes) {
  if (!ctx || (n && (!keys || !vals))) return fail(ctx, MK_EINVAL, "null argument");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const size_t tb = 8ull * (n + 1);
  size_t off = 0;
  auto place = [&](size_t bytes) {
    size_t o = off;
    off = (off + bytes + 255) / 256 * 256;
    return o;
  };
  const size_t o_k0 = place(tb), o_k1 = place(tb), o_v0 = place(tb), o_v1 = place(tb);
  const size_t o_ws = place(mksort::workspace_bytes(n));
  int rc = ensure(ctx, &ctx->d_work, &ctx->d_work_bytes, off);
  if (rc) return rc;
  char* wb = static_cast<char*>(ctx->d_work);
  typedef unsigned long long u64;
  u64* k0 = reinterpret_cast<u64*>(wb + o_k0);
  u64* k1 = reinterpret_cast<u64*>(wb + o_k1);
  u64* v0 = reinterpret_cast<u64*>(wb + o_v0);
  u64* v1 = reinterpret_cast<u64*>(wb + o_v1);
  CK(cudaMemcpyAsync(k0, keys, 8 * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(v0, vals, 8 * n, cudaMemcpyHostToDevice, s));
  u64* ks = k0;
  u64* vs = v0;
  mksort::SortInfo si{};
  CK(cudaEventRecord(ctx->ev[0], s));
  CK((mksort::sort_pairs<u64, u64>(k0, v0, k1, v1, n, bits, wb + o_ws, ctx->sms, s, &ks, &vs, &si,
                                  force != 0)));
  CK(cudaEventRecord(ctx->ev[1], s));
  CK(cudaMemcpyAsync(keys, ks, 8 * n, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(vals, vs, 8 * n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  float t = 0.f;
  cudaEventElapsedTime(&t, ctx->ev[0], ctx->ev[1]);
  if (ms) *ms = t;
  if (passes) *passes = si.passes_run;
  return MK_OK;
}

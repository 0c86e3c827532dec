// mk_engine.cu -- sm_100a checking-stage engine behind include/mk_b200.h.
//
// Replaces, per compiled site problem, the reference's decision
// (solver/builtin.py:705-764 check_assertions) and canonical-witness search
// (engine/report.py:147-203 + solver/interface.py:112-187 bisection) by a
// data-parallel lexicographic branch-and-prune over the problem's box of free
// symbols:
//
//   k_bb    one thread per box: incumbent test on the box's best corner, linear
//           bound contraction, interval evaluation of the bytecode, then
//           prune / accept the corner / hand to leaf enumeration / split the
//           first undecided symbol (witness order) into K children written in
//           lexicographic order;
//   k_leaf  one CTA per small box: exhaustive concrete evaluation of every
//           instance in lexicographic order, first model per thread, CTA min
//           reduction of the instance index (index order == witness order),
//           incumbent update under a per-problem seqlock;
//   stack   LIFO of boxes in HBM; children are compacted with
//           cub::DeviceSelect::Flagged (order preserving) so the best child
//           of the best box is always on top (depth-first in witness order,
//           which finds the incumbent early and prunes the rest).
//
// The host loop (mk_site_eval) runs rounds until the stack is empty.

#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "mk_b200.h"
#include "mk_core.cuh"

namespace {

struct Box {
  int32_t prob;
  int32_t pad0;
  int64_t pad1;
  // followed by i128 lo[S], hi[S]
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
  unsigned long long boxes, leaves, points, insns_bb, insns_leaf;
  double covered;
};

__device__ __forceinline__ Box* box_at(void* base, size_t box_bytes, size_t i) {
  return reinterpret_cast<Box*>(reinterpret_cast<char*>(base) + i * box_bytes);
}
__device__ __forceinline__ mk_i128* box_lo(Box* b) { return reinterpret_cast<mk_i128*>(b + 1); }

// 64-bit lexicographic key of a point (see Incumbent::key)
__device__ unsigned long long lex_key(const DevSet& D, const mk_problem& p, const i128* x) {
  unsigned long long key = 0;
  int left = 64;
  for (int i = 0; i < p.nvars && left > 0; ++i) {
    i128 rlo = mk_ld(D.var_lo[p.var_off + i]), rhi = mk_ld(D.var_hi[p.var_off + i]);
    u128 span = (u128)(rhi - rlo);
    int bits = mk_bitlen(span);
    if (bits == 0) continue;
    u128 d = ((p.maxmask >> i) & 1) ? (u128)(rhi - x[i]) : (u128)(x[i] - rlo);
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
__device__ bool inc_dominates(const DevSet& D, int pid, const mk_problem& p, const i128* corner) {
  Incumbent* I = D.inc + pid;
  {
    unsigned long long kmin = *((volatile unsigned long long*)&I->key);
    if (kmin != ~0ull) {
      unsigned long long k = lex_key(D, p, corner);
      if (k > kmin) return true;   // a strictly better model was offered
    }
  }
  unsigned v1 = *((volatile unsigned*)&I->version);
  if (v1 & 1u) return false;
  __threadfence();
  int has = *((volatile int*)&I->has);
  if (!has) return false;
  const volatile mk_i128* B = D.best + p.var_off;
  bool dominated = true;
  for (int i = 0; i < p.nvars; ++i) {
    mk_i128 t;
    t.lo = B[i].lo;
    t.hi = B[i].hi;
    i128 b = mk_ld(t);
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

__device__ void inc_offer(const DevSet& D, int pid, const mk_problem& p, const i128* x) {
  Incumbent* I = D.inc + pid;
  // lock-free filter: a candidate whose key prefix is worse than the best
  // offered key loses without touching the lock
  {
    unsigned long long k = lex_key(D, p, x);
    unsigned long long old = atomicMin(&I->key, k);
    if (k > old) return;
  }
  if (inc_dominates(D, pid, p, x)) return;
  unsigned ns = 32;
  while (atomicCAS(&I->lock, 0, 1) != 0) {
    __nanosleep(ns);
    if (ns < 2048) ns <<= 1;
  }
  __threadfence();
  bool better = true;
  if (I->has) {
    i128 cur[MK_MAXV];
    for (int i = 0; i < p.nvars; ++i) cur[i] = mk_ld(D.best[p.var_off + i]);
    better = mk_lex_better(x, cur, p.nvars, p.maxmask);
  }
  if (better) {
    atomicAdd(&I->version, 1u);
    __threadfence();
    for (int i = 0; i < p.nvars; ++i) D.best[p.var_off + i] = mk_st(x[i]);
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

__global__ void k_roots(DevSet D, int nprob, void* stack) {
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
  D.inc[pid].version = 0;
  D.inc[pid].has = 0;
  D.inc[pid].err = 0;
  D.inc[pid].key = ~0ull;
}

// ---------------------------------------------------------------------------
// per-box step shared by the round kernel (k_bb) and the persistent search
// kernel (k_search)

enum { ACT_DONE = 0, ACT_LEAF = 1, ACT_SPLIT = 2 };

struct Act {
  int kind;
  int sv;  // split symbol
  int m;   // number of children
};

// lo/hi: the box (contracted in place).  Prunes, accepts the best corner of an
// all-true box, hands small boxes to enumeration, or chooses a split.
__device__ Act process_box(const DevSet& D, int pid, const mk_problem& p, i128* lo, i128* hi,
                           int K, long long leaf_volume, DevStats* st) {
  const int nv = p.nvars;
  const MkProb P = view(D, pid);
  Act a;
  a.kind = ACT_DONE;
  a.sv = -1;
  a.m = 0;
  i128 c[MK_MAXV];
  atomicAdd(&st->boxes, 1ull);
  mk_corner(lo, hi, nv, p.maxmask, c);
  double vol0 = mk_volume_f(lo, hi, nv);
  if (inc_dominates(D, pid, p, c)) {
    atomicAdd(&st->covered, vol0);
    return a;
  }
  if (!mk_contract(P, lo, hi, 4)) {
    atomicAdd(&st->covered, vol0);
    return a;
  }
  MkIv R[MK_MAXR];
  int64_t cnt = 0;
  MkBoxVerdict v = mk_eval_box(P, lo, hi, R, &cnt);
  atomicAdd(&st->insns_bb, (unsigned long long)cnt);
  if (v.any_false) {
    atomicAdd(&st->covered, vol0);
    return a;
  }
  if (v.all_true) {
    mk_corner(lo, hi, nv, p.maxmask, c);
    inc_offer(D, pid, p, c);
    atomicAdd(&st->covered, vol0);
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
  i128 size = hi[sv] - lo[sv] + 1;
  a.kind = ACT_SPLIT;
  a.sv = sv;
  a.m = size < (i128)K ? (int)size : K;
  return a;
}

__device__ __forceinline__ void write_box(Box* out, int pid, const i128* lo, const i128* hi,
                                          int nv, int stride, int sv, i128 plo, i128 phi) {
  out->prob = pid;
  mk_i128* olo = box_lo(out);
  for (int k = 0; k < nv; ++k) {
    olo[k] = mk_st(k == sv ? plo : lo[k]);
    olo[stride + k] = mk_st(k == sv ? phi : hi[k]);
  }
}

__device__ __forceinline__ void load_box(const Box* in, int nv, int stride, i128* lo, i128* hi) {
  const mk_i128* blo = box_lo(const_cast<Box*>(in));
  for (int v = 0; v < nv; ++v) {
    lo[v] = mk_ld(blo[v]);
    hi[v] = mk_ld(blo[stride + v]);
  }
}

// Exhaustive enumeration of one small box by the whole CTA: every instance in
// lexicographic index order (== witness order), each thread stops at its
// first model, CTA min of the index, incumbent update.  s_lo/s_hi in shared.
__device__ void cta_enumerate(const DevSet& D, int pid, const mk_problem& p, const i128* s_lo,
                              const i128* s_hi, unsigned long long* s_best, int* s_skip,
                              DevStats* st) {
  const int nv = p.nvars;
  if (threadIdx.x == 0) {
    *s_best = ~0ull;
    i128 c[MK_MAXV];
    mk_corner(s_lo, s_hi, nv, p.maxmask, c);
    *s_skip = inc_dominates(D, pid, p, c) ? 1 : 0;
  }
  __syncthreads();
  const unsigned long long vol = (unsigned long long)mk_volume(s_lo, s_hi, nv);
  if (*s_skip) {
    if (threadIdx.x == 0) {
      atomicAdd(&st->covered, (double)vol);
      atomicAdd(&st->leaves, 1ull);
    }
    __syncthreads();
    return;
  }
  const MkProb P = view(D, pid);
  MkCv R[MK_MAXR];
  i128 x[MK_MAXV];
  int64_t cnt = 0;
  unsigned long long evaluated = 0;
  bool ovf = false;
  for (unsigned long long idx = threadIdx.x; idx < vol; idx += blockDim.x) {
    if (idx > *((volatile unsigned long long*)s_best)) break;
    mk_decode(s_lo, s_hi, nv, p.maxmask, idx, x);
    ++evaluated;
    if (mk_eval_point(P, x, R, &ovf, &cnt)) {
      atomicMin(s_best, idx);
      break;
    }
  }
  if (ovf) atomicExch(&D.inc[pid].err, 1);
  atomicAdd(&st->points, evaluated);
  atomicAdd(&st->insns_leaf, (unsigned long long)cnt);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&st->leaves, 1ull);
    atomicAdd(&st->covered, (double)vol);
    if (*s_best != ~0ull) {
      mk_decode(s_lo, s_hi, nv, p.maxmask, *s_best, x);
      inc_offer(D, pid, p, x);
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(128) k_bb(DevSet D, const void* chunk, int n, int K,
                                            long long leaf_volume, void* child_out,
                                            int* child_flag, void* leaf_out, int* leaf_flag,
                                            DevStats* st) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int j = 0; j < K; ++j) child_flag[(size_t)i * K + j] = 0;
  leaf_flag[i] = 0;
  const Box* in = box_at(const_cast<void*>(chunk), D.box_bytes, i);
  const int pid = in->prob;
  const mk_problem p = D.probs[pid];
  const int nv = p.nvars;
  i128 lo[MK_MAXV], hi[MK_MAXV];
  load_box(in, nv, D.stride, lo, hi);
  Act a = process_box(D, pid, p, lo, hi, K, leaf_volume, st);
  if (a.kind == ACT_LEAF) {
    write_box(box_at(leaf_out, D.box_bytes, i), pid, lo, hi, nv, D.stride, -1, 0, 0);
    leaf_flag[i] = 1;
  } else if (a.kind == ACT_SPLIT) {
    bool mx = (p.maxmask >> a.sv) & 1;
    for (int t = 0; t < a.m; ++t) {
      i128 plo, phi;
      mk_piece(lo[a.sv], hi[a.sv], a.m, t, mx, &plo, &phi);
      size_t slot = (size_t)i * K + (K - 1 - t);  // best piece in the highest slot
      write_box(box_at(child_out, D.box_bytes, slot), pid, lo, hi, nv, D.stride, a.sv, plo, phi);
      child_flag[slot] = 1;
    }
  }
}

__global__ void __launch_bounds__(256) k_leaf(DevSet D, const void* leaves, int nleaf,
                                              DevStats* st) {
  const Box* in = box_at(const_cast<void*>(leaves), D.box_bytes, blockIdx.x);
  const int pid = in->prob;
  const mk_problem p = D.probs[pid];
  const int nv = p.nvars;
  __shared__ i128 s_lo[MK_MAXV], s_hi[MK_MAXV];
  __shared__ unsigned long long s_best;
  __shared__ int s_skip;
  const mk_i128* blo = box_lo(const_cast<Box*>(in));
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    s_lo[v] = mk_ld(blo[v]);
    s_hi[v] = mk_ld(blo[D.stride + v]);
  }
  __syncthreads();
  cta_enumerate(D, pid, p, s_lo, s_hi, &s_best, &s_skip, st);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_stamp(unsigned long long* out) { *out = globaltimer_ns(); }

// Persistent search: each CTA takes tasks (pre-split boxes, best first) and
// runs a 128-wide best-first DFS from its own HBM stack: pop the top n boxes,
// one per thread, process, block-scan the children counts, write children in
// lexicographic order (best on top), enumerate leaves CTA-wide; repeat until
// the stack is empty.  Incumbents are shared across CTAs through the seqlock.
#define SEARCH_THREADS 128
// control block: [0] task counter, [1] idle CTAs, [2] dumped boxes,
//                [4..5] start stamp (u64)
__global__ void __launch_bounds__(SEARCH_THREADS) k_search(
    DevSet D, const void* tasks, int ntasks, int* ctl, void* stacks, long long cap,
    void* leafbuf, int K, long long leaf_volume, unsigned long long budget_ns,
    unsigned long long slice_ns, void* dump, long long dump_cap, int* pending, DevStats* st) {
  typedef cub::BlockScan<int, SEARCH_THREADS> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int s_task, s_abort, s_dump;
  __shared__ long long s_top, s_dump_off;
  __shared__ int s_nleaf;
  __shared__ i128 s_lo[MK_MAXV], s_hi[MK_MAXV];
  __shared__ unsigned long long s_best;
  __shared__ int s_skip;
  const unsigned long long t_start = *reinterpret_cast<const unsigned long long*>(ctl + 4);
  const unsigned long long deadline_ns = t_start + budget_ns;
  const int grid = gridDim.x;
  char* my_stack = static_cast<char*>(stacks) + (size_t)blockIdx.x * (size_t)cap * D.box_bytes;
  char* my_leaves = static_cast<char*>(leafbuf) + (size_t)blockIdx.x * SEARCH_THREADS * D.box_bytes;
  const int t = threadIdx.x;
  const size_t words = D.box_bytes / sizeof(int4);
  for (;;) {
    if (t == 0) s_task = atomicAdd(ctl, 1);
    __syncthreads();
    const int task = s_task;
    if (task >= ntasks) {
      if (t == 0) atomicAdd(ctl + 1, 1);  // idle from now on
      return;
    }
    // tasks are taken best-first: the top of the task stack
    const Box* tb = box_at(const_cast<void*>(tasks), D.box_bytes, (size_t)(ntasks - 1 - task));
    const int pid = tb->prob;
    const mk_problem p = D.probs[pid];
    const int nv = p.nvars;
    {
      const int4* src = reinterpret_cast<const int4*>(tb);
      int4* dst = reinterpret_cast<int4*>(my_stack);
      for (size_t w = t; w < words; w += SEARCH_THREADS) dst[w] = src[w];
    }
    if (t == 0) {
      s_top = 1;
      s_abort = globaltimer_ns() > deadline_ns ? 1 : 0;
      s_dump = 0;
    }
    __syncthreads();
    if (s_abort) {
      if (t == 0) pending[pid] = 1;
      __syncthreads();
      continue;
    }
    while (s_top > 0) {
      long long top = s_top;
      long long room = cap - top;
      long long n = top < SEARCH_THREADS ? top : SEARCH_THREADS;
      long long fit = room / (K - 1);
      if (fit < n) n = fit;
      if (n < 1) {  // stack full: give up on this task honestly
        if (t == 0) atomicExch(&D.inc[pid].err, 1);
        break;
      }
      const long long base = top - n;
      i128 lo[MK_MAXV], hi[MK_MAXV];
      Act a;
      a.kind = ACT_DONE;
      a.m = 0;
      a.sv = -1;
      if (t < n) {
        load_box(box_at(my_stack, D.box_bytes, (size_t)(base + t)), nv, D.stride, lo, hi);
        a = process_box(D, pid, p, lo, hi, K, leaf_volume, st);
      }
      int nch = a.kind == ACT_SPLIT ? a.m : 0;
      int isleaf = a.kind == ACT_LEAF ? 1 : 0;
      int coff, ctot, loff, ltot;
      Scan(scan_tmp).ExclusiveSum(nch, coff, ctot);
      __syncthreads();
      Scan(scan_tmp).ExclusiveSum(isleaf, loff, ltot);
      __syncthreads();  // every popped box has been read: its slot may be reused
      if (nch) {
        bool mx = (p.maxmask >> a.sv) & 1;
        for (int j = 0; j < a.m; ++j) {
          i128 plo, phi;
          mk_piece(lo[a.sv], hi[a.sv], a.m, a.m - 1 - j, mx, &plo, &phi);  // worst first
          write_box(box_at(my_stack, D.box_bytes, (size_t)(base + coff + j)), pid, lo, hi, nv,
                    D.stride, a.sv, plo, phi);
        }
      }
      if (isleaf) write_box(box_at(my_leaves, D.box_bytes, loff), pid, lo, hi, nv, D.stride, -1, 0, 0);
      if (t == 0) {
        s_top = base + ctot;
        s_nleaf = ltot;
        unsigned long long now = globaltimer_ns();
        if (now > deadline_ns) s_abort = 1;
        // hand the remaining subtrees back when a quarter of the grid idles
        int idle = *((volatile int*)(ctl + 1));
        if (s_top > 0 && idle * 4 >= grid && now > t_start + slice_ns) s_dump = 1;
      }
      __syncthreads();
      for (int l = 0; l < s_nleaf; ++l) {
        const Box* lb = box_at(my_leaves, D.box_bytes, l);
        for (int v = t; v < nv; v += SEARCH_THREADS) {
          s_lo[v] = mk_ld(box_lo(const_cast<Box*>(lb))[v]);
          s_hi[v] = mk_ld(box_lo(const_cast<Box*>(lb))[D.stride + v]);
        }
        __syncthreads();
        cta_enumerate(D, pid, p, s_lo, s_hi, &s_best, &s_skip, st);
      }
      if (s_abort) {
        if (t == 0 && s_top > 0) pending[pid] = 1;
        break;
      }
      if (s_dump) {
        if (t == 0) {
          long long off = atomicAdd(reinterpret_cast<unsigned long long*>(ctl + 2),
                                    (unsigned long long)s_top);
          s_dump_off = off;
          if (off + s_top > dump_cap) {
            atomicExch(&D.inc[pid].err, 1);
            s_dump_off = -1;
          }
        }
        __syncthreads();
        if (s_dump_off >= 0) {
          const int4* src = reinterpret_cast<const int4*>(my_stack);
          int4* dst = reinterpret_cast<int4*>(static_cast<char*>(dump) +
                                              (size_t)s_dump_off * D.box_bytes);
          size_t total = (size_t)s_top * words;
          for (size_t w = t; w < total; w += SEARCH_THREADS) dst[w] = src[w];
        }
        __syncthreads();
        break;
      }
    }
    __syncthreads();
    if (s_dump) return;  // this launch ends; the host redistributes the dump
  }
}

// problems that still own boxes when the budget runs out are undecided
__global__ void k_mark_pending(DevSet D, const void* stack, long long top, int* pending) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= top) return;
  const Box* b = box_at(const_cast<void*>(stack), D.box_bytes, (size_t)i);
  pending[b->prob] = 1;
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
  int search_ctas = 148;
  std::string err;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  // growable device buffers
  mk_dset scratch;
  void* d_work = nullptr;
  size_t d_work_bytes = 0;
  void* h_pinned = nullptr;
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
  // the evaluators keep their register files in local memory
  cudaDeviceSetLimit(cudaLimitStackSize, 32 * 1024);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return MK_ECUDA;
  }
  for (int i = 0; i < 6; ++i) cudaEventCreate(&ctx->ev[i]);
  cudaMallocHost(&ctx->h_pinned, 4096);
  {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search, SEARCH_THREADS, 0);
    if (per_sm < 1) per_sm = 1;
    ctx->search_ctas = sms * per_sm;
  }
  *out = ctx;
  return MK_OK;
}

extern "C" int mk_ctx_destroy(mk_ctx* ctx) {
  if (!ctx) return MK_OK;
  cudaSetDevice(ctx->device);
  if (ctx->d_work) cudaFree(ctx->d_work);
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  for (int i = 0; i < 6; ++i)
    if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
  if (ctx->scratch.d) cudaFree(ctx->scratch.d);
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


static int upload_set(mk_ctx* ctx, const mk_problem_set* set, mk_dset* ds) {
  const int nprob = set->nprob;
  int S = 1;
  for (int i = 0; i < nprob; ++i) {
    const mk_problem& p = set->probs[i];
    if (p.nvars > MK_MAXV || p.nregs > MK_MAXR)
      return fail(ctx, MK_EINVAL, "problem exceeds MK_MAXV symbols or MK_MAXR registers");
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
  ds->o_counts = place(sizeof(int) * 4);
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

static int run_set(mk_ctx* ctx, mk_dset* ds, const mk_limits* lim, int32_t* status,
                   mk_i128* point, mk_stats* stats, std::chrono::steady_clock::time_point t0) {
  mk_stats local_stats;
  std::memset(&local_stats, 0, sizeof(local_stats));
  const int nprob = ds->nprob;
  const int S = ds->S;
  int64_t max_rounds = lim && lim->max_rounds > 0 ? lim->max_rounds : 200000;
  int64_t max_boxes = lim && lim->max_boxes > 0 ? lim->max_boxes : (int64_t)4e9;
  double max_seconds = lim && lim->max_seconds > 0 ? lim->max_seconds : 30.0;
  int K = lim && lim->split_k > 1 ? lim->split_k : 16;
  int chunk = lim && lim->chunk > 0 ? lim->chunk : 65536;
  long long leaf_volume = lim && lim->leaf_volume > 0 ? lim->leaf_volume : 4096;
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

  // ---- work buffers: stack, child/leaf staging, flags, cub scratch
  size_t cap_boxes = ((size_t)3 << 30) / box_bytes;  // 3 GiB of box stack in HBM
  if (cap_boxes < (size_t)nprob + (size_t)chunk * K) cap_boxes = (size_t)nprob + (size_t)chunk * K;
  size_t cub_bytes = 0;
  {
    size_t t1 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, t1, (const int*)nullptr, (int*)nullptr,
                                  (int)((size_t)chunk * K), s);
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
  size_t w_cflag = wplace(sizeof(int) * (size_t)chunk * K);
  size_t w_cpos = wplace(sizeof(int) * (size_t)chunk * K);
  size_t w_leaf = wplace(box_bytes * (size_t)chunk);
  size_t w_lflag = wplace(sizeof(int) * (size_t)chunk);
  size_t w_lpos = wplace(sizeof(int) * (size_t)chunk);
  size_t w_leaves = wplace(box_bytes * (size_t)chunk);
  size_t w_cub = wplace(cub_bytes + 256);
  // persistent search: per-CTA stacks and leaf lists
  const int grid_max = ctx->search_ctas;
  long long cta_cap = (long long)(((size_t)6 << 30) / ((size_t)grid_max * box_bytes));
  if (cta_cap > 65536) cta_cap = 65536;
  if (cta_cap < 4 * SEARCH_THREADS) cta_cap = 4 * SEARCH_THREADS;
  size_t w_cstack = wplace(box_bytes * (size_t)cta_cap * grid_max);
  size_t w_cleaf = wplace(box_bytes * (size_t)SEARCH_THREADS * grid_max);
  size_t w_tctr = wplace(sizeof(int) * 8);
  // redistribution buffer: the dump of one launch is the task list of the
  // next; it alternates with the pre-split stack (both cap_boxes)
  size_t w_dump = wplace(box_bytes * cap_boxes);
  const long long dump_cap = (long long)cap_boxes;
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
  void* cta_stacks = wb + w_cstack;
  void* cta_leaves = wb + w_cleaf;
  int* ctl = reinterpret_cast<int*>(wb + w_tctr);
  void* cta_dump = wb + w_dump;
  // pre-split until every CTA of the persistent search has a task
  const long long presplit_target = lim && lim->chunk < 0 ? 0 : (long long)grid_max;

  k_roots<<<(nprob + 127) / 128, 128, 0, s>>>(D, nprob, stack);
    ++launches;
  CK(cudaGetLastError());
  long long top = nprob;
  int64_t rounds = 0;
  double bb_ms = 0.0, leaf_ms = 0.0;
  int* h_counts = static_cast<int*>(ctx->h_pinned);
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
      k_leaf<<<(unsigned)nleaf, 256, 0, s>>>(D, leaves, (int)nleaf, d_st);
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
  double search_ms = 0.0;
  int search_launches = 0;
  void* tasks_buf = stack;
  void* dump_buf = cta_dump;
  while (!budget_hit && top > 0) {
    double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    double left = max_seconds - el;
    if (left <= 0) {
      budget_hit = true;
      break;
    }
    // the wall budget is checked on the device against %globaltimer, stamped
    // stream-ordered just before the launch
    CK(cudaMemsetAsync(ctl, 0, sizeof(int) * 8, s));
    k_stamp<<<1, 1, 0, s>>>(reinterpret_cast<unsigned long long*>(ctl + 4));
    ++launches;
    // always the full persistent grid: CTAs without a task idle at once,
    // which is what triggers redistribution of a lone deep subtree
    int grid = grid_max;
    CK(cudaEventRecord(ctx->ev[0], s));
    k_search<<<grid, SEARCH_THREADS, 0, s>>>(
        D, tasks_buf, (int)top, ctl, cta_stacks, cta_cap, cta_leaves, K, leaf_volume,
        (unsigned long long)(left * 1e9), (unsigned long long)200000, dump_buf, dump_cap,
        d_pend, d_st);
    ++launches;
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev[1], s));
    long long dumped = 0;
    CK(cudaMemcpyAsync(&dumped, ctl + 2, sizeof(long long), cudaMemcpyDeviceToHost, s));
    CK(cudaEventSynchronize(ctx->ev[1]));
    CK(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
    search_ms += ms;
    ++search_launches;
    top = dumped;
    void* tmp = tasks_buf;
    tasks_buf = dump_buf;
    dump_buf = tmp;
  }
  if (budget_hit && top > 0 && tasks_buf != stack) {
    k_mark_pending<<<(unsigned)((top + 255) / 256), 256, 0, s>>>(D, tasks_buf, top, d_pend);
    ++launches;
    CK(cudaGetLastError());
    top = 0;
  }
  if (budget_hit && top > 0) {
    k_mark_pending<<<(unsigned)((top + 255) / 256), 256, 0, s>>>(D, stack, top, d_pend);
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
  local_stats.rounds = rounds + search_launches;
  local_stats.boxes = (int64_t)dst.boxes;
  local_stats.leaves = (int64_t)dst.leaves;
  local_stats.points = (int64_t)dst.points;
  local_stats.covered = dst.covered;
  local_stats.insns_bb = (int64_t)dst.insns_bb;
  local_stats.insns_leaf = (int64_t)dst.insns_leaf;
  local_stats.bb_ms = bb_ms + search_ms;
  local_stats.leaf_ms = leaf_ms;
  local_stats.seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  {
    float dms = 0.f;
    cudaEventElapsedTime(&dms, ctx->ev[4], ctx->ev[5]);
    local_stats.device_ms = dms;
  }
  local_stats.launches = launches;
  if (stats) *stats = local_stats;
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
  return run_set(ctx, ds, lim, status, point, stats, t0);
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
  return run_set(ctx, &ctx->scratch, lim, status, point, stats, t0);
}

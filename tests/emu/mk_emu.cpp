// mk_emu.cpp -- TEST-ONLY serial host emulation of libmk_b200.so.
//
// Compiles the same evaluation core (paper_2603_24595_b200/csrc/mk_core.cuh)
// for the host and drives it with a serial depth-first loop that mirrors the
// device rounds (LIFO stack, K-ary splits in witness order, exhaustive leaf
// enumeration in lexicographic index order).  It lets the CPU test suite
// check the compiler + search logic against the reference goldens without a
// GPU.  It is never loaded by the package: paper_2603_24595_b200/native.py
// only loads libmk_b200.so and fails loudly without it.
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "mk_b200.h"
#include "mk_core.cuh"

struct mk_ctx {
  std::string err;
};

extern "C" int mk_abi_version(void) { return MK_ABI_VERSION; }
extern "C" int mk_device_count(int* out) {
  if (out) *out = 1;
  return MK_OK;
}
extern "C" int mk_ctx_create(int device, mk_ctx** out) {
  (void)device;
  *out = new mk_ctx();
  return MK_OK;
}
extern "C" int mk_ctx_destroy(mk_ctx* ctx) {
  delete ctx;
  return MK_OK;
}
extern "C" const char* mk_last_error(const mk_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

namespace {
template <typename V>
struct EBox {
  int prob;
  std::vector<V> lo, hi;
};

// one problem, serial depth-first in the device's order; V = int64_t for
// problems flagged MK_PF_NARROW, i128 otherwise (the device's dispatch)
template <typename V>
void solve_problem(const mk_problem_set* set, int pid, int K, long long leaf_volume,
                   double max_seconds, int64_t max_boxes,
                   std::chrono::steady_clock::time_point t0, mk_stats& st, int& has, int& err,
                   int& pend, std::vector<V>& best) {
  typedef typename MkNum<V>::U U;
  const mk_problem& p = set->probs[pid];
  MkProb P = mk_prob_view(set->probs, pid, set->insns, set->consts, set->atom_regs,
                          set->atom_masks, set->rows, set->row_terms);
  std::vector<MkPair<V>> R(MK_MAXT);
  std::vector<V> C(MK_MAXT);
  const int nv = p.nvars;
  std::vector<EBox<V>> stack;
  EBox<V> root;
  root.prob = pid;
  for (int i = 0; i < nv; ++i) {
    root.lo.push_back(MkNum<V>::ld(set->var_lo[p.var_off + i]));
    root.hi.push_back(MkNum<V>::ld(set->var_hi[p.var_off + i]));
  }
  stack.push_back(root);
  while (!stack.empty()) {
    double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > max_seconds || st.boxes > max_boxes) {
      pend = 1;
      break;
    }
    if (has && (p.flags & MK_PF_ANY)) break;  // feasibility only: one model decides
    EBox<V> b = stack.back();
    stack.pop_back();
    st.boxes++;
    V c[MK_MAXV];
    mk_corner(b.lo.data(), b.hi.data(), nv, p.maxmask, c);
    if (has && !mk_lex_better(c, best.data(), nv, p.maxmask)) {
      st.covered += mk_volume_f(b.lo.data(), b.hi.data(), nv);
      continue;
    }
    double vol0 = mk_volume_f(b.lo.data(), b.hi.data(), nv);
    if (!mk_contract(P, b.lo.data(), b.hi.data(), 4)) {
      st.covered += vol0;
      continue;
    }
    int64_t cnt = 0;
    MkBoxVerdict v = mk_eval_box_t(P, b.lo.data(), b.hi.data(), R.data(), &cnt);
    st.insns_bb += cnt;
    if (v.any_false) {
      st.covered += vol0;
      continue;
    }
    if (v.all_true) {
      mk_corner(b.lo.data(), b.hi.data(), nv, p.maxmask, c);
      if (!has || mk_lex_better(c, best.data(), nv, p.maxmask)) {
        best.assign(c, c + nv);
        has = 1;
      }
      st.covered += vol0;
      continue;
    }
    long long vol = mk_volume(b.lo.data(), b.hi.data(), nv);
    if (vol <= leaf_volume) {
      st.leaves++;
      st.covered += (double)vol;
      if (has) {
        mk_corner(b.lo.data(), b.hi.data(), nv, p.maxmask, c);
        if (!mk_lex_better(c, best.data(), nv, p.maxmask)) continue;
      }
      V x[MK_MAXV];
      bool ovf = false;
      int64_t c2 = 0;
      for (long long idx = 0; idx < vol; ++idx) {
        mk_decode(b.lo.data(), b.hi.data(), nv, p.maxmask, (uint64_t)idx, x);
        st.points++;
        if (mk_eval_point_t(P, x, C.data(), &ovf, &c2)) {
          if (!has || mk_lex_better(x, best.data(), nv, p.maxmask)) {
            best.assign(x, x + nv);
            has = 1;
          }
          break;
        }
      }
      st.insns_leaf += c2;
      if (ovf) err = 1;
      continue;
    }
    int sv = mk_pick_split(b.lo.data(), b.hi.data(), nv, v.und_mask, has != 0);
    if (sv < 0) {
      err = 1;
      continue;
    }
    U size = (U)(b.hi[sv] - b.lo[sv]) + 1;
    int m = size < (U)K ? (int)size : K;
    bool mx = (p.maxmask >> sv) & 1;
    // push worst first so the best piece is popped next
    for (int t = m - 1; t >= 0; --t) {
      EBox<V> ch = b;
      mk_piece(b.lo[sv], b.hi[sv], m, t, mx, &ch.lo[sv], &ch.hi[sv]);
      stack.push_back(ch);
    }
    st.rounds++;
  }
}
}  // namespace

extern "C" int mk_site_eval(mk_ctx* ctx, const mk_problem_set* set, const mk_limits* lim,
                            int32_t* status, mk_i128* point, mk_stats* stats) {
  auto t0 = std::chrono::steady_clock::now();
  mk_stats st;
  std::memset(&st, 0, sizeof(st));
  const int nprob = set->nprob;
  int K = lim && lim->split_k > 1 ? lim->split_k : 16;
  long long leaf_volume = lim && lim->leaf_volume > 0 ? lim->leaf_volume : 4096;
  double max_seconds = lim && lim->max_seconds > 0 ? lim->max_seconds : 30.0;
  int64_t max_boxes = lim && lim->max_boxes > 0 ? lim->max_boxes : (int64_t)50000000;
  for (int pid = 0; pid < nprob; ++pid) {
    const mk_problem& p = set->probs[pid];
    if (p.nvars > MK_MAXV || p.nregs > MK_MAXR) {
      ctx->err = "problem exceeds MK_MAXV symbols or MK_MAXR registers";
      return MK_EINVAL;
    }
  }
  for (int pid = 0; pid < nprob; ++pid) {
    const mk_problem& p = set->probs[pid];
    const int nv = p.nvars;
    int has = 0, err = 0, pend = 0;
    std::vector<i128> best(nv, 0);
    if (p.flags & MK_PF_NARROW) {
      std::vector<int64_t> b64;
      solve_problem<int64_t>(set, pid, K, leaf_volume, max_seconds, max_boxes, t0, st, has, err,
                             pend, b64);
      for (int i = 0; i < (int)b64.size(); ++i) best[i] = b64[i];
    } else {
      solve_problem<i128>(set, pid, K, leaf_volume, max_seconds, max_boxes, t0, st, has, err,
                          pend, best);
    }
    if (err || pend) status[pid] = MK_UNKNOWN;
    else status[pid] = has ? MK_SAT : MK_UNSAT;
    for (int i = 0; i < nv; ++i) point[p.var_off + i] = mk_st(has ? best[i] : (i128)0);
  }
  st.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (stats) *stats = st;
  return MK_OK;
}

struct mk_dset {
  const mk_problem_set* set;
};
extern "C" int mk_set_upload(mk_ctx* ctx, const mk_problem_set* set, mk_dset** out) {
  (void)ctx;
  *out = new mk_dset{set};
  return MK_OK;
}
extern "C" int mk_set_eval(mk_ctx* ctx, mk_dset* d, const mk_limits* lim, int32_t* status,
                           mk_i128* point, mk_stats* stats) {
  return mk_site_eval(ctx, d->set, lim, status, point, stats);
}
extern "C" int mk_set_free(mk_ctx* ctx, mk_dset* d) {
  (void)ctx;
  delete d;
  return MK_OK;
}

// -- race sweep (K2), serial host restatement of csrc/mk_race.cuh ----------------
#include <algorithm>
#include <utility>

// ranged call (a shard of the launch): the fused ordered pass's semantics --
// accesses in instance order, keys must be non-decreasing, adjacent equal keys
// with distinct identities conflict; first / last access reported for the
// combination of shards.  Keys and identities as the device computes them.
static int race_range(mk_ctx* ctx, const mk_race_prog* prog, mk_race_result* out) {
  const mk_problem_set& set = prog->set;
  const mk_problem& p = set.probs[0];
  MkProb P = mk_prob_view(set.probs, 0, set.insns, set.consts, set.atom_regs, set.atom_masks,
                          set.rows, set.row_terms);
  const int nv = p.nvars, n_outer = nv - prog->n_exist;
  std::vector<int64_t> lo(nv), hi(nv);
  unsigned long long inner = 1;
  for (int i = 0; i < nv; ++i) {
    lo[i] = (int64_t)set.var_lo[p.var_off + i].lo;
    hi[i] = (int64_t)set.var_hi[p.var_off + i].lo;
    if (i >= n_outer) inner *= (unsigned long long)(hi[i] - lo[i] + 1);
  }
  // key origin: the root box's offset interval (mk_race_sweep's k_race_root)
  std::vector<MkIvT<int64_t>> Rg(MK_MAXR);
  int64_t cnt0 = 0;
  mk_eval_box<int64_t>(P, lo.data(), hi.data(), Rg.data(), &cnt0);
  const int64_t off_lo = Rg[prog->off_reg].lo;
  unsigned long long nblocks = 1;
  for (int a = 0; a < 3; ++a)
    if (prog->shared && prog->id_var[a] >= 0)
      nblocks *= (unsigned long long)(hi[prog->id_var[a]] - lo[prog->id_var[a]] + 1);
  out->off_lo = off_lo;
  out->nblocks = nblocks;
  out->sorted = 1;
  out->fused = 1;
  std::vector<MkCvT<int64_t>> R(MK_MAXR);
  int64_t x[MK_MAXV];
  bool have = false;
  unsigned long long pk = 0, pid = 0, pidx = 0, best = ~0ull, bkey = 0;
  for (unsigned long long idx = prog->begin; idx < prog->end; ++idx) {
    bool hit = false;
    for (unsigned long long j = 0; j < inner && !hit; ++j) {
      mk_decode(lo.data(), hi.data(), nv, 0ull, idx * inner + j, x);
      bool ovf = false;
      int64_t cnt = 0;
      out->instances++;
      hit = mk_eval_point(P, x, R.data(), &ovf, &cnt);
    }
    if (!hit) continue;
    unsigned long long bk = 0;
    if (prog->shared)
      for (int a = 2; a >= 0; --a) {
        const int v = prog->id_var[a];
        if (v < 0) continue;
        bk = bk * (unsigned long long)(hi[v] - lo[v] + 1) + (unsigned long long)(x[v] - lo[v]);
      }
    const unsigned long long key = (unsigned long long)(R[prog->off_reg].v - off_lo) * nblocks + bk;
    unsigned long long idk = 0;
    for (int a = prog->shared ? 3 : 0; a < 6; ++a) {
      const int v = prog->id_var[a];
      if (v < 0) continue;
      idk = idk * (unsigned long long)(hi[v] - lo[v] + 1) + (unsigned long long)(x[v] - lo[v]);
    }
    out->tuples++;
    if (have) {
      if (key < pk) {
        out->sorted = 0;
        return MK_OK;
      }
      if (key == pk && idk != pid) {
        out->conflicts++;
        const unsigned long long c = (idx << 32) | pidx;
        if (c < best) {
          best = c;
          bkey = key;
        }
      }
    } else {
      out->first_key = key;
      out->first_id = idk;
      out->first_idx = idx;
    }
    have = true;
    pk = key;
    pid = idk;
    pidx = idx;
  }
  out->have = have ? 1 : 0;
  out->last_key = pk;
  out->last_id = pid;
  out->last_idx = pidx;
  out->has_race = out->conflicts > 0;
  if (out->has_race) {
    out->idx_b = best >> 32;
    out->idx_a = best & 0xffffffffull;
    out->offset = (int64_t)(bkey / nblocks) + off_lo;
  }
  (void)ctx;
  return MK_OK;
}

extern "C" int mk_race_sweep(mk_ctx* ctx, const mk_race_prog* prog, mk_race_result* out) {
  std::memset(out, 0, sizeof(*out));
  if (prog->end > 0) return race_range(ctx, prog, out);
  const mk_problem_set& set = prog->set;
  if (set.nprob != 1) {
    ctx->err = "race sweep takes exactly one problem";
    return MK_EINVAL;
  }
  const mk_problem& p = set.probs[0];
  if (!(p.flags & MK_PF_NARROW)) {
    ctx->err = "race sweep needs a narrow problem";
    return MK_EINVAL;
  }
  MkProb P = mk_prob_view(set.probs, 0, set.insns, set.consts, set.atom_regs, set.atom_masks,
                          set.rows, set.row_terms);
  const int nv = p.nvars, n_outer = nv - prog->n_exist;
  std::vector<int64_t> lo(nv), hi(nv);
  unsigned long long vol = 1, inner = 1;
  for (int i = 0; i < nv; ++i) {
    lo[i] = (int64_t)set.var_lo[p.var_off + i].lo;
    hi[i] = (int64_t)set.var_hi[p.var_off + i].lo;
    (i < n_outer ? vol : inner) *= (unsigned long long)(hi[i] - lo[i] + 1);
  }
  std::vector<MkCvT<int64_t>> R(MK_MAXR);
  std::vector<std::pair<std::pair<int64_t, unsigned long long>, unsigned long long>> tuples;
  int64_t x[MK_MAXV], y[MK_MAXV];
  for (unsigned long long idx = 0; idx < vol; ++idx) {
    for (unsigned long long j = 0; j < inner; ++j) {
      mk_decode(lo.data(), hi.data(), nv, p.maxmask, idx * inner + j, x);
      bool ovf = false;
      int64_t cnt = 0;
      out->instances++;
      if (mk_eval_point(P, x, R.data(), &ovf, &cnt)) {
        unsigned long long blk = 0;
        if (prog->shared) {
          for (int a = 2; a >= 0; --a) {
            const int v = prog->id_var[a];
            if (v < 0) continue;
            blk = blk * (unsigned long long)(hi[v] - lo[v] + 1) + (unsigned long long)(x[v] - lo[v]);
          }
        }
        tuples.push_back({{R[prog->off_reg].v, blk}, idx});
        break;
      }
    }
  }
  std::sort(tuples.begin(), tuples.end());
  out->tuples = tuples.size();
  for (size_t i = 1; i < tuples.size(); ++i) {
    if (tuples[i].first != tuples[i - 1].first) continue;
    mk_decode(lo.data(), hi.data(), n_outer, p.maxmask, tuples[i - 1].second, x);
    mk_decode(lo.data(), hi.data(), n_outer, p.maxmask, tuples[i].second, y);
    bool same = true;
    for (int a = prog->shared ? 3 : 0; a < 6; ++a) {
      const int v = prog->id_var[a];
      if (v >= 0 && x[v] != y[v]) same = false;
    }
    if (!same) {
      if (!out->has_race) {
        out->idx_a = tuples[i - 1].second;
        out->idx_b = tuples[i].second;
        out->offset = tuples[i].first.first;
      }
      out->has_race = 1;
      out->conflicts++;
    }
  }
  out->hbm_bytes = 4ull * 12ull * out->tuples;
  return MK_OK;
}

// -- access sweep (K2, oracle semantics), serial restatement of csrc/mk_access.cuh --

extern "C" int mk_access_sweep(mk_ctx* ctx, const mk_access_input* in, mk_access_result* out) {
  std::memset(out, 0, sizeof(*out));
  const mk_problem_set& set = in->set;
  long long grid[3], block[3];
  for (int k = 0; k < 3; ++k) {
    grid[k] = in->grid[k] > 0 ? in->grid[k] : 1;
    block[k] = in->block[k] > 0 ? in->block[k] : 1;
  }
  std::vector<std::pair<unsigned long long, unsigned long long>> tuples;  // (key, val), dense order
  unsigned long long slot = 0;
  std::vector<MkCvT<int64_t>> R(MK_MAXR);
  for (int pi = 0; pi < set.nprob; ++pi) {
    const mk_problem& p = set.probs[pi];
    const mk_access_prog& A = in->progs[pi];
    if (!(p.flags & MK_PF_NARROW)) {
      ctx->err = "access sweep needs narrow problems";
      return MK_EINVAL;
    }
    MkProb P = mk_prob_view(set.probs, pi, set.insns, set.consts, set.atom_regs, set.atom_masks,
                            set.rows, set.row_terms);
    const int nv = p.nvars, n_outer = nv - A.n_exist;
    std::vector<int64_t> lo(nv), hi(nv);
    unsigned long long vol = 1, inner = 1;
    for (int i = 0; i < nv; ++i) {
      lo[i] = (int64_t)set.var_lo[p.var_off + i].lo;
      hi[i] = (int64_t)set.var_hi[p.var_off + i].lo;
      (i < n_outer ? vol : inner) *= (unsigned long long)(hi[i] - lo[i] + 1);
    }
    int64_t x[MK_MAXV];
    for (unsigned long long idx = 0; idx < vol; ++idx, slot += (unsigned long long)A.tuples) {
      bool hit = false;
      int64_t off = 0;
      for (unsigned long long j = 0; j < inner && !hit; ++j) {
        mk_decode(lo.data(), hi.data(), nv, 0ull, idx * inner + j, x);
        bool ovf = false;
        int64_t cnt = 0;
        out->instances++;
        if (mk_eval_point(P, x, R.data(), &ovf, &cnt)) {
          hit = true;
          off = R[A.off_reg].v;
        }
      }
      if (!hit) continue;
      long long id[6];
      for (int k = 0; k < 6; ++k) id[k] = A.id_var[k] >= 0 ? (long long)x[A.id_var[k]] : A.id_fixed[k];
      const unsigned long long blk = ((unsigned long long)id[2] * grid[1] + id[1]) * grid[0] + id[0];
      const unsigned long long thr = ((unsigned long long)id[5] * block[1] + id[4]) * block[0] + id[3];
      const unsigned long long nthr = (unsigned long long)(block[0] * block[1] * block[2]);
      const unsigned long long idk = A.shared ? thr : blk * nthr + thr;
      const long long rel = (long long)off - A.off_lo;
      if (rel < 0 || rel % A.granule) out->misaligned = 1;
      const unsigned long long k0 =
          A.kbase + (A.shared ? blk * A.span : 0ull) + (unsigned long long)(rel / A.granule);
      for (int j = 0; j < A.tuples; ++j)
        tuples.push_back({((k0 + j) << 1) | (A.write ? 0ull : 1ull), (idk << 32) | (slot + j)});
    }
  }
  out->tuples = tuples.size();
  if (out->misaligned) return MK_OK;
  std::stable_sort(tuples.begin(), tuples.end(),
                   [](const std::pair<unsigned long long, unsigned long long>& a,
                      const std::pair<unsigned long long, unsigned long long>& b) {
                     return a.first < b.first;
                   });
  const size_t n = tuples.size();
  for (size_t i = 0; i < n; ++i) {
    const unsigned long long k = tuples[i].first;
    if (i > 0 && (tuples[i - 1].first >> 1) == (k >> 1)) continue;
    if (k & 1ull) continue;
    for (size_t j = i + 1; j < n && (tuples[j].first >> 1) == (k >> 1); ++j) {
      if ((tuples[j].second >> 32) != (tuples[i].second >> 32)) {
        if (!out->has_race) {
          out->slot_a = tuples[i].second & 0xffffffffull;
          out->slot_b = tuples[j].second & 0xffffffffull;
        }
        out->has_race = 1;
        out->racy++;
        break;
      }
    }
  }
  return MK_OK;
}

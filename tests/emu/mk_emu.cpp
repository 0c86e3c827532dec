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
struct EBox {
  int prob;
  std::vector<i128> lo, hi;
};
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
  std::vector<int> has(nprob, 0), err(nprob, 0), pend(nprob, 0);
  std::vector<std::vector<i128>> best(nprob);
  std::vector<MkIv> R(MK_MAXR);
  std::vector<MkCv> C(MK_MAXR);
  for (int pid = 0; pid < nprob; ++pid) {
    const mk_problem& p = set->probs[pid];
    if (p.nvars > MK_MAXV || p.nregs > MK_MAXR) {
      ctx->err = "problem exceeds MK_MAXV symbols or MK_MAXR registers";
      return MK_EINVAL;
    }
    MkProb P = mk_prob_view(set->probs, pid, set->insns, set->consts, set->atom_regs,
                            set->atom_masks, set->rows, set->row_terms);
    const int nv = p.nvars;
    std::vector<EBox> stack;
    EBox root;
    root.prob = pid;
    for (int i = 0; i < nv; ++i) {
      root.lo.push_back(mk_ld(set->var_lo[p.var_off + i]));
      root.hi.push_back(mk_ld(set->var_hi[p.var_off + i]));
    }
    stack.push_back(root);
    while (!stack.empty()) {
      double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > max_seconds || st.boxes > max_boxes) {
        pend[pid] = 1;
        break;
      }
      EBox b = stack.back();
      stack.pop_back();
      st.boxes++;
      i128 c[MK_MAXV];
      mk_corner(b.lo.data(), b.hi.data(), nv, p.maxmask, c);
      if (has[pid] && !mk_lex_better(c, best[pid].data(), nv, p.maxmask)) {
        st.covered += mk_volume_f(b.lo.data(), b.hi.data(), nv);
        continue;
      }
      double vol0 = mk_volume_f(b.lo.data(), b.hi.data(), nv);
      if (!mk_contract(P, b.lo.data(), b.hi.data(), 4)) {
        st.covered += vol0;
        continue;
      }
      int64_t cnt = 0;
      MkBoxVerdict v = mk_eval_box(P, b.lo.data(), b.hi.data(), R.data(), &cnt);
      st.insns_bb += cnt;
      if (v.any_false) {
        st.covered += vol0;
        continue;
      }
      if (v.all_true) {
        mk_corner(b.lo.data(), b.hi.data(), nv, p.maxmask, c);
        if (!has[pid] || mk_lex_better(c, best[pid].data(), nv, p.maxmask)) {
          best[pid].assign(c, c + nv);
          has[pid] = 1;
        }
        st.covered += vol0;
        continue;
      }
      long long vol = mk_volume(b.lo.data(), b.hi.data(), nv);
      if (vol <= leaf_volume) {
        st.leaves++;
        st.covered += (double)vol;
        if (has[pid]) {
          mk_corner(b.lo.data(), b.hi.data(), nv, p.maxmask, c);
          if (!mk_lex_better(c, best[pid].data(), nv, p.maxmask)) continue;
        }
        i128 x[MK_MAXV];
        bool ovf = false;
        int64_t c2 = 0;
        for (long long idx = 0; idx < vol; ++idx) {
          mk_decode(b.lo.data(), b.hi.data(), nv, p.maxmask, (uint64_t)idx, x);
          st.points++;
          if (mk_eval_point(P, x, C.data(), &ovf, &c2)) {
            if (!has[pid] || mk_lex_better(x, best[pid].data(), nv, p.maxmask)) {
              best[pid].assign(x, x + nv);
              has[pid] = 1;
            }
            break;
          }
        }
        st.insns_leaf += c2;
        if (ovf) err[pid] = 1;
        continue;
      }
      int sv = mk_pick_split(b.lo.data(), b.hi.data(), nv, v.und_mask, has[pid] != 0);
      if (sv < 0) {
        err[pid] = 1;
        continue;
      }
      i128 size = b.hi[sv] - b.lo[sv] + 1;
      int m = size < (i128)K ? (int)size : K;
      bool mx = (p.maxmask >> sv) & 1;
      // push worst first so the best piece is popped next
      for (int t = m - 1; t >= 0; --t) {
        EBox ch = b;
        mk_piece(b.lo[sv], b.hi[sv], m, t, mx, &ch.lo[sv], &ch.hi[sv]);
        stack.push_back(ch);
      }
      st.rounds++;
    }
    if (err[pid] || pend[pid]) status[pid] = MK_UNKNOWN;
    else status[pid] = has[pid] ? MK_SAT : MK_UNSAT;
    for (int i = 0; i < nv; ++i)
      point[p.var_off + i] = mk_st(has[pid] ? best[pid][i] : (i128)0);
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

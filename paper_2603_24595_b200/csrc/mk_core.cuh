// mk_core.cuh -- evaluation core of the checking stage, shared by the
// sm_100a kernels (mk_engine.cu) and the test-only host emulator
// (tests/emu/mk_emu.cpp).
//
// Semantics restated from the reference (mathematical mode, sym/expr.py):
//   add/sub/mul exact; div truncates toward zero (:273-279); mod = a - trunc(a/b)*b
//   (:282-285); emod = a mod |b| in [0,|b|) (:288-291); shl = a*2^k, shr = floor
//   shift (:315-318); casts are the identity (:356-364); Cmp -> 0/1; and/or
//   short-circuit (:367-378); division/remainder by zero raises EvalError and the
//   point is not a model (solver/query.py:59-62).
// Values are 128-bit two's complement.  |v| >= MK_INF means "beyond the exact
// range": interval endpoints saturate outward (sound), a concrete value that
// saturates marks the problem inexact (reported unknown, never guessed).
#pragma once
#include <stdint.h>
#include "mk_b200.h"

#if defined(__CUDACC__)
#define MK_HD __host__ __device__ __forceinline__
#else
#define MK_HD static inline
#endif

typedef __int128 i128;
typedef unsigned __int128 u128;

#define MK_INF (((i128)1) << 125)
#define MK_FL_OK 1
#define MK_FL_ERR 2

#ifndef MK_MAXR
#define MK_MAXR 256   /* registers per problem evaluated by the kernels */
#endif
#define MK_MAXV 64    /* free symbols per problem */

MK_HD i128 mk_ld(const mk_i128& v) {
  return (i128)(((u128)(uint64_t)v.hi << 64) | (u128)v.lo);
}
MK_HD mk_i128 mk_st(i128 x) {
  mk_i128 r;
  r.lo = (uint64_t)(u128)x;
  r.hi = (int64_t)(uint64_t)((u128)x >> 64);
  return r;
}
MK_HD i128 mk_clamp(i128 x) {
  if (x >= MK_INF) return MK_INF;
  if (x <= -MK_INF) return -MK_INF;
  return x;
}
MK_HD bool mk_isinf(i128 x) { return x >= MK_INF || x <= -MK_INF; }

MK_HD int mk_clz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
  return __clzll((long long)x);
#else
  return x ? __builtin_clzll(x) : 64;
#endif
}
MK_HD int mk_bitlen(u128 x) {
  uint64_t h = (uint64_t)(x >> 64);
  if (h) return 128 - mk_clz64(h);
  uint64_t l = (uint64_t)x;
  return l ? 64 - mk_clz64(l) : 0;
}
MK_HD u128 mk_abs(i128 x) { return x < 0 ? (u128)(-x) : (u128)x; }

// saturating arithmetic on clamped operands (|a|,|b| <= MK_INF)
MK_HD i128 mk_add(i128 a, i128 b) { return mk_clamp(a + b); }
MK_HD i128 mk_sub(i128 a, i128 b) { return mk_clamp(a - b); }
MK_HD i128 mk_mul(i128 a, i128 b) {
  if (a == 0 || b == 0) return 0;
  bool neg = (a < 0) != (b < 0);
  if (mk_bitlen(mk_abs(a)) + mk_bitlen(mk_abs(b)) > 125) return neg ? -MK_INF : MK_INF;
  return mk_clamp(a * b);
}
// truncating division; b != 0.  infinite numerator stays infinite, an infinite
// divisor drives a finite numerator to 0 (the limit; sound at interval corners)
MK_HD i128 mk_tdiv(i128 a, i128 b) {
  if (mk_isinf(a)) return ((a < 0) != (b < 0)) ? -MK_INF : MK_INF;
  if (mk_isinf(b)) return 0;
  return a / b;
}
MK_HD i128 mk_floordiv(i128 a, i128 b) {
  i128 q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
  return q;
}
MK_HD i128 mk_ceildiv(i128 a, i128 b) {
  i128 q = a / b;
  if ((a % b != 0) && ((a < 0) == (b < 0))) q += 1;
  return q;
}
MK_HD i128 mk_emod_c(i128 a, i128 b) {  // exact, b != 0, finite
  i128 m = b < 0 ? -b : b;
  i128 r = a % m;
  if (r < 0) r += m;
  return r;
}
MK_HD i128 mk_min(i128 a, i128 b) { return a < b ? a : b; }
MK_HD i128 mk_max(i128 a, i128 b) { return a > b ? a : b; }

struct MkProb {
  const mk_problem* p;
  const mk_insn* insns;
  const mk_i128* consts;
  const int32_t* atom_regs;
  const uint64_t* atom_masks;
  const mk_row* rows;
  const mk_row_term* terms;
};

MK_HD MkProb mk_prob_view(const mk_problem* probs, int pid, const mk_insn* insns,
                          const mk_i128* consts, const int32_t* atom_regs,
                          const uint64_t* atom_masks, const mk_row* rows,
                          const mk_row_term* terms) {
  MkProb v;
  v.p = probs + pid;
  v.insns = insns + v.p->insn_off;
  v.consts = consts + v.p->const_off;
  v.atom_regs = atom_regs + v.p->atom_off;
  v.atom_masks = atom_masks + v.p->atom_off;
  v.rows = rows + v.p->row_off;
  v.terms = terms;
  return v;
}

// ---------------------------------------------------------------------------
// interval (box) evaluation
//
// Every register carries [lo,hi] over the points of the box where it
// evaluates without error, plus flags: OK = some point evaluates, ERR = some
// point raises.  Booleans use [0,1].

struct MkIv {
  i128 lo, hi;
  uint8_t fl;
};

MK_HD bool mk_sure_lt(const MkIv& a, const MkIv& b) {
  return a.hi != MK_INF && b.lo != -MK_INF && a.hi < b.lo;
}
MK_HD bool mk_sure_le(const MkIv& a, const MkIv& b) {
  return a.hi != MK_INF && b.lo != -MK_INF && a.hi <= b.lo;
}
MK_HD bool mk_exact1(const MkIv& a) { return a.lo == a.hi && !mk_isinf(a.lo); }

MK_HD void mk_corners(i128 c0, i128 c1, i128 c2, i128 c3, i128* lo, i128* hi) {
  *lo = mk_min(mk_min(c0, c1), mk_min(c2, c3));
  *hi = mk_max(mk_max(c0, c1), mk_max(c2, c3));
}

MK_HD void mk_iv_div_part(i128 xlo, i128 xhi, i128 d1, i128 d2, i128* lo, i128* hi) {
  mk_corners(mk_tdiv(xlo, d1), mk_tdiv(xlo, d2), mk_tdiv(xhi, d1), mk_tdiv(xhi, d2), lo, hi);
}

MK_HD MkIv mk_iv_binop(int op, const MkIv& a, const MkIv& b) {
  MkIv r;
  r.fl = 0;
  bool ok = (a.fl & MK_FL_OK) && (b.fl & MK_FL_OK);
  bool err = (a.fl & MK_FL_ERR) || (b.fl & MK_FL_ERR);
  r.lo = 0;
  r.hi = 0;
  if (!ok) {
    r.fl = err ? MK_FL_ERR : 0;
    return r;
  }
  switch (op) {
    case MK_OP_ADD:
      r.lo = mk_add(a.lo, b.lo);
      r.hi = mk_add(a.hi, b.hi);
      if (a.lo == -MK_INF || b.lo == -MK_INF) r.lo = -MK_INF;
      if (a.hi == MK_INF || b.hi == MK_INF) r.hi = MK_INF;
      break;
    case MK_OP_SUB:
      r.lo = mk_sub(a.lo, b.hi);
      r.hi = mk_sub(a.hi, b.lo);
      if (a.lo == -MK_INF || b.hi == MK_INF) r.lo = -MK_INF;
      if (a.hi == MK_INF || b.lo == -MK_INF) r.hi = MK_INF;
      break;
    case MK_OP_MUL:
      mk_corners(mk_mul(a.lo, b.lo), mk_mul(a.lo, b.hi), mk_mul(a.hi, b.lo), mk_mul(a.hi, b.hi),
                 &r.lo, &r.hi);
      break;
    case MK_OP_SHL: {
      int k = (int)b.lo;  // compiler guarantees a constant in [0,256]
      i128 f = k >= 125 ? MK_INF : ((i128)1 << k);
      mk_corners(mk_mul(a.lo, f), mk_mul(a.hi, f), mk_mul(a.lo, f), mk_mul(a.hi, f), &r.lo, &r.hi);
      break;
    }
    case MK_OP_SHR: {
      int k = (int)b.lo;
      if (k > 126) k = 126;
      r.lo = mk_isinf(a.lo) ? a.lo : (a.lo >> k);
      r.hi = mk_isinf(a.hi) ? a.hi : (a.hi >> k);
      break;
    }
    case MK_OP_DIV:
    case MK_OP_MOD:
    case MK_OP_EMOD: {
      bool has0 = b.lo <= 0 && b.hi >= 0;
      if (has0) err = true;
      if (b.lo == 0 && b.hi == 0) {  // every point divides by zero
        r.fl = MK_FL_ERR;
        return r;
      }
      if (op == MK_OP_DIV) {
        bool first = true;
        if (b.hi >= 1) {  // positive divisor part
          i128 l, h;
          mk_iv_div_part(a.lo, a.hi, mk_max(b.lo, 1), b.hi, &l, &h);
          r.lo = l; r.hi = h; first = false;
        }
        if (b.lo <= -1) {
          i128 l, h;
          mk_iv_div_part(a.lo, a.hi, b.lo, mk_min(b.hi, -1), &l, &h);
          if (first) { r.lo = l; r.hi = h; }
          else { r.lo = mk_min(r.lo, l); r.hi = mk_max(r.hi, h); }
        }
        if (a.lo == -MK_INF || a.hi == MK_INF) {
          // unbounded numerator: be explicit about the sign reach
          if (a.lo == -MK_INF) { if (b.hi >= 1) r.lo = -MK_INF; if (b.lo <= -1) r.hi = MK_INF; }
          if (a.hi == MK_INF) { if (b.hi >= 1) r.hi = MK_INF; if (b.lo <= -1) r.lo = -MK_INF; }
        }
      } else {
        i128 m;  // max |divisor| - 1
        if (mk_isinf(b.lo) || mk_isinf(b.hi)) m = MK_INF;
        else m = mk_max(b.lo < 0 ? -b.lo : b.lo, b.hi < 0 ? -b.hi : b.hi) - 1;
        bool xfin = !mk_isinf(a.lo) && !mk_isinf(a.hi);
        bool dsing = mk_exact1(b);
        if (op == MK_OP_MOD) {
          if (xfin && dsing && a.lo == a.hi) {
            r.lo = r.hi = a.lo % b.lo;
          } else if (xfin && dsing && ((a.lo >= 0 && a.lo / b.lo == a.hi / b.lo) ||
                                       (a.hi <= 0 && a.lo / b.lo == a.hi / b.lo))) {
            r.lo = a.lo % b.lo;
            r.hi = a.hi % b.lo;
            if (r.lo > r.hi) { i128 t = r.lo; r.lo = r.hi; r.hi = t; }
          } else {
            r.lo = (a.lo >= 0) ? 0 : ((a.lo == -MK_INF) ? -m : mk_max(a.lo, -m));
            r.hi = (a.hi <= 0) ? 0 : ((a.hi == MK_INF) ? m : mk_min(a.hi, m));
          }
        } else {
          if (xfin && dsing) {
            i128 M = b.lo < 0 ? -b.lo : b.lo;
            if (mk_floordiv(a.lo, M) == mk_floordiv(a.hi, M)) {
              r.lo = mk_emod_c(a.lo, M);
              r.hi = mk_emod_c(a.hi, M);
            } else {
              r.lo = 0; r.hi = m;
            }
          } else {
            r.lo = 0; r.hi = m;
          }
        }
      }
      break;
    }
    case MK_OP_EQ:
    case MK_OP_NE: {
      bool t = !(mk_sure_lt(a, b) || mk_sure_lt(b, a));
      bool f = !(mk_exact1(a) && mk_exact1(b) && a.lo == b.lo);
      if (op == MK_OP_NE) { bool s = t; t = f; f = s; }
      r.lo = f ? 0 : 1;
      r.hi = t ? 1 : 0;
      break;
    }
    case MK_OP_LT:
    case MK_OP_GE: {
      bool t = !mk_sure_le(b, a);   // a < b possible unless surely b <= a
      bool f = !mk_sure_lt(a, b);
      if (op == MK_OP_GE) { bool s = t; t = f; f = s; }
      r.lo = f ? 0 : 1;
      r.hi = t ? 1 : 0;
      break;
    }
    case MK_OP_LE:
    case MK_OP_GT: {
      bool t = !mk_sure_lt(b, a);   // a <= b possible unless surely b < a
      bool f = !mk_sure_le(a, b);
      if (op == MK_OP_GT) { bool s = t; t = f; f = s; }
      r.lo = f ? 0 : 1;
      r.hi = t ? 1 : 0;
      break;
    }
    default:
      break;
  }
  r.fl = MK_FL_OK | (err ? MK_FL_ERR : 0);
  return r;
}

// short-circuit booleans: a is evaluated first
MK_HD MkIv mk_iv_and(const MkIv& a, const MkIv& b) {
  bool aok = a.fl & MK_FL_OK, bok = b.fl & MK_FL_OK;
  bool a_t = aok && a.hi == 1, a_f = aok && a.lo == 0;
  bool b_t = bok && b.hi == 1, b_f = bok && b.lo == 0;
  bool t = a_t && b_t;
  bool f = a_f || (a_t && b_f);
  bool e = (a.fl & MK_FL_ERR) || (a_t && (b.fl & MK_FL_ERR));
  MkIv r;
  r.lo = f ? 0 : 1;
  r.hi = t ? 1 : 0;
  r.fl = ((t || f) ? MK_FL_OK : 0) | (e ? MK_FL_ERR : 0);
  return r;
}
MK_HD MkIv mk_iv_or(const MkIv& a, const MkIv& b) {
  bool aok = a.fl & MK_FL_OK, bok = b.fl & MK_FL_OK;
  bool a_t = aok && a.hi == 1, a_f = aok && a.lo == 0;
  bool b_t = bok && b.hi == 1, b_f = bok && b.lo == 0;
  bool t = a_t || (a_f && b_t);
  bool f = a_f && b_f;
  bool e = (a.fl & MK_FL_ERR) || (a_f && (b.fl & MK_FL_ERR));
  MkIv r;
  r.lo = f ? 0 : 1;
  r.hi = t ? 1 : 0;
  r.fl = ((t || f) ? MK_FL_OK : 0) | (e ? MK_FL_ERR : 0);
  return r;
}
MK_HD MkIv mk_iv_ite(const MkIv& c, const MkIv& x, const MkIv& y) {
  bool cok = c.fl & MK_FL_OK;
  bool c_t = cok && c.hi == 1, c_f = cok && c.lo == 0;
  MkIv r;
  bool any = false;
  r.lo = 0; r.hi = 0;
  uint8_t e = (c.fl & MK_FL_ERR) ? MK_FL_ERR : 0;
  if (c_t) {
    if (x.fl & MK_FL_OK) { r.lo = x.lo; r.hi = x.hi; any = true; }
    e |= (x.fl & MK_FL_ERR);
  }
  if (c_f) {
    if (y.fl & MK_FL_OK) {
      if (any) { r.lo = mk_min(r.lo, y.lo); r.hi = mk_max(r.hi, y.hi); }
      else { r.lo = y.lo; r.hi = y.hi; any = true; }
    }
    e |= (y.fl & MK_FL_ERR);
  }
  r.fl = (any ? MK_FL_OK : 0) | e;
  return r;
}

// evaluate the program over a box; returns per-atom status in *und_mask
// (undecided atoms' symbol masks OR-ed), *any_false, *all_true.
struct MkBoxVerdict {
  bool any_false;
  bool all_true;
  bool overflow;      // some value saturated although every symbol is fixed
  uint64_t und_mask;  // symbols of undecided atoms
};

MK_HD MkBoxVerdict mk_eval_box(const MkProb& P, const i128* vlo, const i128* vhi, MkIv* R,
                               int64_t* insn_count) {
  const int nv = P.p->nvars;
  const int nc = P.p->nconst;
  for (int i = 0; i < nv; ++i) {
    R[i].lo = vlo[i];
    R[i].hi = vhi[i];
    R[i].fl = MK_FL_OK;
  }
  for (int i = 0; i < nc; ++i) {
    i128 c = mk_ld(P.consts[i]);
    R[nv + i].lo = c;
    R[nv + i].hi = c;
    R[nv + i].fl = MK_FL_OK;
  }
  const int n = P.p->ninsn;
  MkBoxVerdict v;
  v.any_false = false;
  v.all_true = true;
  v.overflow = false;
  v.und_mask = 0;
  for (int k = 0; k < n; ++k) {
    const mk_insn in = P.insns[k];
    switch (in.op) {
      case MK_OP_ATOM: {
        const MkIv r = R[in.a];
        bool ok = r.fl & MK_FL_OK;
        bool may_true = ok && r.hi == 1;
        bool sure_true = ok && r.lo == 1 && !(r.fl & MK_FL_ERR);
        if (!may_true) {
          *insn_count += k + 1;
          v.any_false = true;
          v.all_true = false;
          return v;
        }
        if (!sure_true) {
          v.all_true = false;
          v.und_mask |= P.atom_masks[in.b];
        }
        break;
      }
      case MK_OP_AND: R[in.dst] = mk_iv_and(R[in.a], R[in.b]); break;
      case MK_OP_OR: R[in.dst] = mk_iv_or(R[in.a], R[in.b]); break;
      case MK_OP_NOT: {
        MkIv a = R[in.a], r;
        r.lo = 1 - a.hi;
        r.hi = 1 - a.lo;
        r.fl = a.fl;
        R[in.dst] = r;
        break;
      }
      case MK_OP_ITE: R[in.dst] = mk_iv_ite(R[in.a], R[in.b], R[in.c]); break;
      default: R[in.dst] = mk_iv_binop(in.op, R[in.a], R[in.b]); break;
    }
  }
  *insn_count += n;
  return v;
}

// ---------------------------------------------------------------------------
// bound contraction over the linear rows (one FBBT sweep per call);
// returns false when the box is empty.

MK_HD bool mk_contract(const MkProb& P, i128* lo, i128* hi, int sweeps) {
  const int nr = P.p->nrows;
  for (int s = 0; s < sweeps; ++s) {
    bool changed = false;
    for (int r = 0; r < nr; ++r) {
      const mk_row row = P.rows[r];
      const mk_row_term* T = P.terms + row.term_off;
      i128 fmin = mk_ld(row.c0), fmax = fmin;
      int nmin_inf = 0, nmax_inf = 0;
      for (int k = 0; k < row.nterms; ++k) {
        i128 c = mk_ld(T[k].coef);
        int v = T[k].var;
        i128 a = mk_mul(c, lo[v]), b = mk_mul(c, hi[v]);
        i128 mn = mk_min(a, b), mx = mk_max(a, b);
        if (mn == -MK_INF) nmin_inf++; else fmin = mk_add(fmin, mn);
        if (mx == MK_INF) nmax_inf++; else fmax = mk_add(fmax, mx);
      }
      if (nmin_inf == 0 && fmin > 0 && fmin != MK_INF) return false;  // sum >= fmin > 0
      if (nmin_inf == 0 && fmin == MK_INF) return false;
      if (row.rel == 1 && nmax_inf == 0 && fmax < 0 && fmax != -MK_INF) return false;
      if (row.rel == 1 && nmax_inf == 0 && fmax == -MK_INF) return false;
      for (int k = 0; k < row.nterms; ++k) {
        i128 c = mk_ld(T[k].coef);
        int v = T[k].var;
        i128 a = mk_mul(c, lo[v]), b = mk_mul(c, hi[v]);
        i128 mn = mk_min(a, b), mx = mk_max(a, b);
        // others_min = fmin - mn (when finite)
        int oinf = nmin_inf - (mn == -MK_INF ? 1 : 0);
        if (oinf == 0) {
          i128 omin = (mn == -MK_INF) ? fmin : mk_sub(fmin, mn);
          if (!mk_isinf(omin)) {
            // c*x <= -omin
            if (c > 0) {
              i128 nb = mk_floordiv(-omin, c);
              if (nb < hi[v]) { hi[v] = nb; changed = true; }
            } else {
              i128 nb = mk_ceildiv(-omin, c);
              if (nb > lo[v]) { lo[v] = nb; changed = true; }
            }
          }
        }
        if (row.rel == 1) {
          int oinf2 = nmax_inf - (mx == MK_INF ? 1 : 0);
          if (oinf2 == 0) {
            i128 omax = (mx == MK_INF) ? fmax : mk_sub(fmax, mx);
            if (!mk_isinf(omax)) {
              // c*x >= -omax
              if (c > 0) {
                i128 nb = mk_ceildiv(-omax, c);
                if (nb > lo[v]) { lo[v] = nb; changed = true; }
              } else {
                i128 nb = mk_floordiv(-omax, c);
                if (nb < hi[v]) { hi[v] = nb; changed = true; }
              }
            }
          }
        }
        if (lo[v] > hi[v]) return false;
      }
    }
    if (!changed) break;
  }
  return true;
}

// ---------------------------------------------------------------------------
// concrete (point) evaluation.  Registers hold exact values; an error bit per
// register tracks EvalError with the reference's short-circuit rules.

struct MkCv {
  i128 v;
  uint8_t err;
};

MK_HD bool mk_eval_point(const MkProb& P, const i128* x, MkCv* R, bool* overflow,
                         int64_t* insn_count) {
  const int nv = P.p->nvars;
  const int nc = P.p->nconst;
  for (int i = 0; i < nv; ++i) { R[i].v = x[i]; R[i].err = 0; }
  for (int i = 0; i < nc; ++i) { R[nv + i].v = mk_ld(P.consts[i]); R[nv + i].err = 0; }
  const int n = P.p->ninsn;
  bool ovf = false;
  for (int k = 0; k < n; ++k) {
    const mk_insn in = P.insns[k];
    const MkCv a = R[in.a], b = R[in.b];
    if (in.op == MK_OP_ATOM) {
      if (a.err || !a.v) {
        *insn_count += k + 1;
        if (ovf) *overflow = true;
        return false;
      }
      continue;
    }
    MkCv r;
    r.err = 0;
    r.v = 0;
    switch (in.op) {
      case MK_OP_AND:
        if (a.err) r.err = 1; else if (!a.v) r.v = 0; else { r.v = b.v ? 1 : 0; r.err = b.err; }
        break;
      case MK_OP_OR:
        if (a.err) r.err = 1; else if (a.v) r.v = 1; else { r.v = b.v ? 1 : 0; r.err = b.err; }
        break;
      case MK_OP_NOT:
        r.err = a.err; r.v = a.v ? 0 : 1;
        break;
      case MK_OP_ITE: {
        const MkCv c = R[in.c];
        if (a.err) r.err = 1; else r = a.v ? b : c;
        break;
      }
      default: {
        r.err = a.err | b.err;
        if (!r.err) {
          switch (in.op) {
            case MK_OP_ADD: r.v = mk_add(a.v, b.v); break;
            case MK_OP_SUB: r.v = mk_sub(a.v, b.v); break;
            case MK_OP_MUL: r.v = mk_mul(a.v, b.v); break;
            case MK_OP_SHL: {
              int k2 = (int)b.v;
              r.v = (k2 >= 125) ? (a.v == 0 ? 0 : (a.v < 0 ? -MK_INF : MK_INF))
                                : mk_mul(a.v, (i128)1 << k2);
              break;
            }
            case MK_OP_SHR: {
              int k2 = (int)b.v;
              if (k2 > 126) k2 = 126;
              r.v = a.v >> k2;
              break;
            }
            case MK_OP_DIV:
              if (b.v == 0) r.err = 1; else r.v = a.v / b.v;
              break;
            case MK_OP_MOD:
              if (b.v == 0) r.err = 1; else r.v = a.v % b.v;
              break;
            case MK_OP_EMOD:
              if (b.v == 0) r.err = 1; else r.v = mk_emod_c(a.v, b.v);
              break;
            case MK_OP_EQ: r.v = a.v == b.v; break;
            case MK_OP_NE: r.v = a.v != b.v; break;
            case MK_OP_LT: r.v = a.v < b.v; break;
            case MK_OP_LE: r.v = a.v <= b.v; break;
            case MK_OP_GT: r.v = a.v > b.v; break;
            case MK_OP_GE: r.v = a.v >= b.v; break;
            default: break;
          }
          if (mk_isinf(r.v)) ovf = true;
        }
      }
    }
    R[in.dst] = r;
  }
  *insn_count += n;
  if (ovf) *overflow = true;
  return true;
}

// lexicographic comparison in witness order: true when x is strictly better
MK_HD bool mk_lex_better(const i128* x, const i128* y, int nv, uint64_t maxmask) {
  for (int i = 0; i < nv; ++i) {
    if (x[i] == y[i]) continue;
    bool mx = (maxmask >> i) & 1;
    return mx ? (x[i] > y[i]) : (x[i] < y[i]);
  }
  return false;
}

// the best corner of a box (its lexicographic lower bound)
MK_HD void mk_corner(const i128* lo, const i128* hi, int nv, uint64_t maxmask, i128* out) {
  for (int i = 0; i < nv; ++i) out[i] = ((maxmask >> i) & 1) ? hi[i] : lo[i];
}

// box volume, saturating at 2^62
MK_HD int64_t mk_volume(const i128* lo, const i128* hi, int nv) {
  const i128 cap = ((i128)1) << 62;
  i128 v = 1;
  for (int i = 0; i < nv; ++i) {
    i128 s = hi[i] - lo[i] + 1;
    if (s >= cap) return (int64_t)cap;
    v = v * s;
    if (v >= cap) return (int64_t)cap;
  }
  return (int64_t)v;
}
MK_HD double mk_volume_f(const i128* lo, const i128* hi, int nv) {
  double v = 1.0;
  for (int i = 0; i < nv; ++i) v *= (double)(hi[i] - lo[i] + 1);
  return v;
}

// decode point #idx of a box in lexicographic order (index order == witness order)
MK_HD void mk_decode(const i128* lo, const i128* hi, int nv, uint64_t maxmask, uint64_t idx,
                     i128* x) {
  for (int i = nv - 1; i >= 0; --i) {
    uint64_t s = (uint64_t)(hi[i] - lo[i] + 1);
    uint64_t d = idx % s;
    idx /= s;
    x[i] = ((maxmask >> i) & 1) ? hi[i] - (i128)d : lo[i] + (i128)d;
  }
}

// choose the split symbol among the non-singleton symbols of undecided atoms:
// before any model is known, the smallest domain first (first-fail: refutes
// the narrow core of a query without touching wide launch dimensions); once
// an incumbent exists, the first symbol in witness order (children are then
// lexicographically ordered and the incumbent prunes whole subtrees).
// Returns -1 when every such symbol is fixed.
MK_HD int mk_pick_split(const i128* lo, const i128* hi, int nv, uint64_t und_mask,
                        bool have_incumbent) {
  int best = -1;
  i128 bw = 0;
  for (int i = 0; i < nv; ++i) {
    if (!((und_mask >> i) & 1) || lo[i] >= hi[i]) continue;
    if (have_incumbent) return i;
    i128 w = hi[i] - lo[i];
    if (best < 0 || w < bw) {
      best = i;
      bw = w;
    }
  }
  return best;
}

// piece t (0 = best in the symbol's direction) of m near-equal pieces of [lo,hi]
MK_HD void mk_piece(i128 lo, i128 hi, int m, int t, bool maximize, i128* plo, i128* phi) {
  u128 size = (u128)(hi - lo) + 1;
  u128 q = size / (u128)m, rem = size % (u128)m;
  // ascending piece j covers [lo + j*q + min(j,rem), ...]
  int j = maximize ? (m - 1 - t) : t;
  u128 start = (u128)j * q + (u128)((u128)j < rem ? (u128)j : rem);
  u128 len = q + ((u128)j < rem ? 1 : 0);
  *plo = lo + (i128)start;
  *phi = *plo + (i128)len - 1;
}

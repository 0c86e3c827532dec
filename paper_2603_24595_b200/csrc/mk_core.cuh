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
//
// Every routine is a template over the value type V:
//   V = i128 ("wide"): 128-bit two's complement.  |v| >= MK_INF means "beyond
//     the exact range": interval endpoints saturate outward (sound), a concrete
//     value that saturates marks the problem inexact (reported unknown, never
//     guessed).
//   V = int64_t ("narrow"): used only for problems the site compiler proved
//     narrow (mk_problem.flags & MK_PF_NARROW): every symbol bound, every
//     arithmetic operand and result interval over the root box and every
//     contraction-row sum lies in (-2^61, 2^61), and every register (e.g. a
//     constant that is only compared) fits in int64.  Interval arithmetic is
//     inclusion-isotonic, so every value computed on any sub-box or point
//     stays in those ranges: plain 64-bit arithmetic is exact and no
//     saturation logic is needed.
#pragma once
#include <stdint.h>
#include "mk_b200.h"

#if defined(__CUDACC__)
#define MK_HD __host__ __device__ __forceinline__
#define MK_HDM __host__ __device__ __forceinline__ static
#define MK_HDF __host__ __device__ __forceinline__   /* non-static member functions */
#define MK_HDN __host__ __device__ __noinline__      /* rare, large: one copy, called */
/* runtime-bounded loops stay rolled: unrolled copies of the 64-bit
   division / multiply sequences made the search kernel's code exceed the
   instruction caches (ncu: no_inst the top stall) */
#define MK_NOUNROLL _Pragma("unroll 1")
#else
#define MK_NOUNROLL
#define MK_HD static inline
#define MK_HDM static inline
#define MK_HDF inline
#define MK_HDN static __attribute__((noinline))
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
#define MK_MAXT 64    /* temporaries per problem in the search kernels (flag bit masks) */

MK_HD i128 mk_ld(const mk_i128& v) {
  return (i128)(((u128)(uint64_t)v.hi << 64) | (u128)v.lo);
}
MK_HD mk_i128 mk_st(i128 x) {
  mk_i128 r;
  r.lo = (uint64_t)(u128)x;
  r.hi = (int64_t)(uint64_t)((u128)x >> 64);
  return r;
}

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
MK_HD int mk_bitlen(uint64_t x) { return x ? 64 - mk_clz64(x) : 0; }
MK_HD u128 mk_abs(i128 x) { return x < 0 ? (u128)(-x) : (u128)x; }

// ---------------------------------------------------------------------------
// number traits

template <typename V>
struct MkNum;

template <>
struct MkNum<i128> {
  typedef u128 U;
  static constexpr bool kWide = true;
  MK_HDM i128 inf() { return MK_INF; }
  MK_HDM i128 clamp(i128 x) {
    if (x >= MK_INF) return MK_INF;
    if (x <= -MK_INF) return -MK_INF;
    return x;
  }
  MK_HDM bool isinf(i128 x) { return x >= MK_INF || x <= -MK_INF; }
  // saturating arithmetic on clamped operands (|a|,|b| <= MK_INF)
  MK_HDM i128 add(i128 a, i128 b) { return clamp(a + b); }
  MK_HDM i128 sub(i128 a, i128 b) { return clamp(a - b); }
  MK_HDM i128 mul(i128 a, i128 b) {
    if (a == 0 || b == 0) return 0;
    bool neg = (a < 0) != (b < 0);
    if (mk_bitlen(mk_abs(a)) + mk_bitlen(mk_abs(b)) > 125) return neg ? -MK_INF : MK_INF;
    return clamp(a * b);
  }
  // a * 2^k, k >= 0
  MK_HDM i128 shl(i128 a, int k) {
    if (k >= 125) return a == 0 ? 0 : (a < 0 ? -MK_INF : MK_INF);
    return mul(a, (i128)1 << k);
  }
  MK_HDM i128 shr(i128 a, int k) {
    if (k > 126) k = 126;
    return isinf(a) ? a : (a >> k);
  }
  MK_HDM i128 ld(const mk_i128& v) { return mk_ld(v); }
};

template <>
struct MkNum<int64_t> {
  typedef uint64_t U;
  static constexpr bool kWide = false;
  // never reached: narrow problems stay inside (-2^61, 2^61)
  MK_HDM int64_t inf() { return INT64_MAX; }
  MK_HDM int64_t clamp(int64_t x) { return x; }
  MK_HDM bool isinf(int64_t) { return false; }
  MK_HDM int64_t add(int64_t a, int64_t b) { return a + b; }
  MK_HDM int64_t sub(int64_t a, int64_t b) { return a - b; }
  MK_HDM int64_t mul(int64_t a, int64_t b) { return a * b; }
  MK_HDM int64_t shl(int64_t a, int k) {
    // the narrow proof bounds |a * 2^k| < 2^61, so k < 61 unless a == 0
    return k >= 62 ? 0 : (int64_t)((uint64_t)a << k);
  }
  MK_HDM int64_t shr(int64_t a, int k) { return a >> (k > 63 ? 63 : k); }
  MK_HDM int64_t ld(const mk_i128& v) { return (int64_t)v.lo; }
};

template <typename V>
MK_HD V mk_min(V a, V b) { return a < b ? a : b; }
template <typename V>
MK_HD V mk_max(V a, V b) { return a > b ? a : b; }

// truncating quotient, one division: a 32-bit division when both operands
// fit (the common case for the contraction rows' bounds and coefficients;
// a 64-bit division is a ~70-instruction sequence on the GPU)
// (unit divisors -- most contraction-row coefficients -- need no division)
MK_HD i128 mk_tquot(i128 a, i128 b) {
  if (b == 1) return a;
  if (b == -1) return -a;
  return a / b;
}
MK_HD int64_t mk_tquot(int64_t a, int64_t b) {
  if (b == 1) return a;
  if (b == -1) return -a;
  if (a == (int64_t)(int32_t)a && b == (int64_t)(int32_t)b && !(a == INT32_MIN && b == -1))
    return (int64_t)((int32_t)a / (int32_t)b);
  return a / b;
}

// truncating division; b != 0.  infinite numerator stays infinite, an infinite
// divisor drives a finite numerator to 0 (the limit; sound at interval corners)
template <typename V>
MK_HD V mk_tdiv(V a, V b) {
  typedef MkNum<V> N;
  if (N::isinf(a)) return ((a < 0) != (b < 0)) ? -N::inf() : N::inf();
  if (N::isinf(b)) return 0;
  return mk_tquot(a, b);
}
template <typename V>
MK_HD V mk_floordiv(V a, V b) {
  V q = mk_tquot(a, b);
  if ((a - q * b != 0) && ((a < 0) != (b < 0))) q -= 1;
  return q;
}
template <typename V>
MK_HD V mk_ceildiv(V a, V b) {
  V q = mk_tquot(a, b);
  if ((a - q * b != 0) && ((a < 0) == (b < 0))) q += 1;
  return q;
}
template <typename V>
MK_HD V mk_emod_c(V a, V b) {  // exact, b != 0, finite
  V m = b < 0 ? -b : b;
  V r = a - mk_tquot(a, m) * m;
  if (r < 0) r += m;
  return r;
}

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

template <typename V>
struct MkIvT {
  V lo, hi;
  uint8_t fl;
};
typedef MkIvT<i128> MkIv;

template <typename V>
MK_HD bool mk_sure_lt(const MkIvT<V>& a, const MkIvT<V>& b) {
  typedef MkNum<V> N;
  if (!N::kWide) return a.hi < b.lo;  // narrow: every endpoint is exact
  return a.hi != N::inf() && b.lo != -N::inf() && a.hi < b.lo;
}
template <typename V>
MK_HD bool mk_sure_le(const MkIvT<V>& a, const MkIvT<V>& b) {
  typedef MkNum<V> N;
  if (!N::kWide) return a.hi <= b.lo;
  return a.hi != N::inf() && b.lo != -N::inf() && a.hi <= b.lo;
}
template <typename V>
MK_HD bool mk_exact1(const MkIvT<V>& a) { return a.lo == a.hi && !MkNum<V>::isinf(a.lo); }

template <typename V>
MK_HD void mk_corners(V c0, V c1, V c2, V c3, V* lo, V* hi) {
  *lo = mk_min(mk_min(c0, c1), mk_min(c2, c3));
  *hi = mk_max(mk_max(c0, c1), mk_max(c2, c3));
}

template <typename V>
MK_HD void mk_iv_div_part(V xlo, V xhi, V d1, V d2, V* lo, V* hi) {
  mk_corners(mk_tdiv(xlo, d1), mk_tdiv(xlo, d2), mk_tdiv(xhi, d1), mk_tdiv(xhi, d2), lo, hi);
}

// interval division / remainder (both operands OK): not inlined -- each
// corner is a 64- or 128-bit division sequence, and inlining it into every
// evaluator copy made the search kernel's code too large for the instruction
// caches
template <typename V>
MK_HDN MkIvT<V> mk_iv_divmod(int op, MkIvT<V> a, MkIvT<V> b, bool err) {
  typedef MkNum<V> N;
  const V INF = N::inf();
  MkIvT<V> r;
  r.lo = 0;
  r.hi = 0;
  r.fl = 0;
  {
    bool has0 = b.lo <= 0 && b.hi >= 0;
    if (has0) err = true;
    if (b.lo == 0 && b.hi == 0) {  // every point divides by zero
      r.fl = MK_FL_ERR;
      return r;
    }
    if (op == MK_OP_DIV) {
      bool first = true;
      if (b.hi >= 1) {  // positive divisor part
        V l, h;
        mk_iv_div_part<V>(a.lo, a.hi, mk_max<V>(b.lo, 1), b.hi, &l, &h);
        r.lo = l; r.hi = h; first = false;
      }
      if (b.lo <= -1) {
        V l, h;
        mk_iv_div_part<V>(a.lo, a.hi, b.lo, mk_min<V>(b.hi, -1), &l, &h);
        if (first) { r.lo = l; r.hi = h; }
        else { r.lo = mk_min(r.lo, l); r.hi = mk_max(r.hi, h); }
      }
      if (N::kWide && (a.lo == -INF || a.hi == INF)) {
        // unbounded numerator: be explicit about the sign reach
        if (a.lo == -INF) { if (b.hi >= 1) r.lo = -INF; if (b.lo <= -1) r.hi = INF; }
        if (a.hi == INF) { if (b.hi >= 1) r.hi = INF; if (b.lo <= -1) r.lo = -INF; }
      }
    } else {
      V m;  // max |divisor| - 1
      if (N::isinf(b.lo) || N::isinf(b.hi)) m = INF;
      else m = mk_max<V>(b.lo < 0 ? -b.lo : b.lo, b.hi < 0 ? -b.hi : b.hi) - 1;
      bool xfin = !N::isinf(a.lo) && !N::isinf(a.hi);
      bool dsing = mk_exact1(b);
      if (op == MK_OP_MOD) {
        if (xfin && dsing && a.lo == a.hi) {
          r.lo = r.hi = a.lo % b.lo;
        } else if (xfin && dsing && ((a.lo >= 0 && a.lo / b.lo == a.hi / b.lo) ||
                                     (a.hi <= 0 && a.lo / b.lo == a.hi / b.lo))) {
          r.lo = a.lo % b.lo;
          r.hi = a.hi % b.lo;
          if (r.lo > r.hi) { V t = r.lo; r.lo = r.hi; r.hi = t; }
        } else {
          r.lo = (a.lo >= 0) ? 0 : ((a.lo == -INF) ? -m : mk_max<V>(a.lo, -m));
          r.hi = (a.hi <= 0) ? 0 : ((a.hi == INF) ? m : mk_min<V>(a.hi, m));
        }
      } else {
        if (xfin && dsing) {
          V M = b.lo < 0 ? -b.lo : b.lo;
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
  }
  r.fl = MK_FL_OK | (err ? MK_FL_ERR : 0);
  return r;
}

template <typename V>
MK_HD MkIvT<V> mk_iv_binop(int op, const MkIvT<V>& a, const MkIvT<V>& b) {
  typedef MkNum<V> N;
  const V INF = N::inf();
  MkIvT<V> r;
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
      r.lo = N::add(a.lo, b.lo);
      r.hi = N::add(a.hi, b.hi);
      if (N::kWide) {
        if (a.lo == -INF || b.lo == -INF) r.lo = -INF;
        if (a.hi == INF || b.hi == INF) r.hi = INF;
      }
      break;
    case MK_OP_SUB:
      r.lo = N::sub(a.lo, b.hi);
      r.hi = N::sub(a.hi, b.lo);
      if (N::kWide) {
        if (a.lo == -INF || b.hi == INF) r.lo = -INF;
        if (a.hi == INF || b.lo == -INF) r.hi = INF;
      }
      break;
    case MK_OP_MUL:
      mk_corners(N::mul(a.lo, b.lo), N::mul(a.lo, b.hi), N::mul(a.hi, b.lo), N::mul(a.hi, b.hi),
                 &r.lo, &r.hi);
      break;
    case MK_OP_SHL: {
      int k = (int)b.lo;  // compiler guarantees a constant in [0,256]
      V x = N::shl(a.lo, k), y = N::shl(a.hi, k);
      r.lo = mk_min(x, y);
      r.hi = mk_max(x, y);
      break;
    }
    case MK_OP_SHR: {
      int k = (int)b.lo;
      r.lo = N::shr(a.lo, k);
      r.hi = N::shr(a.hi, k);
      break;
    }
    case MK_OP_DIV:
    case MK_OP_MOD:
    case MK_OP_EMOD:
      return mk_iv_divmod<V>(op, a, b, err);
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
template <typename V>
MK_HD MkIvT<V> mk_iv_and(const MkIvT<V>& a, const MkIvT<V>& b) {
  bool aok = a.fl & MK_FL_OK, bok = b.fl & MK_FL_OK;
  bool a_t = aok && a.hi == 1, a_f = aok && a.lo == 0;
  bool b_t = bok && b.hi == 1, b_f = bok && b.lo == 0;
  bool t = a_t && b_t;
  bool f = a_f || (a_t && b_f);
  bool e = (a.fl & MK_FL_ERR) || (a_t && (b.fl & MK_FL_ERR));
  MkIvT<V> r;
  r.lo = f ? 0 : 1;
  r.hi = t ? 1 : 0;
  r.fl = ((t || f) ? MK_FL_OK : 0) | (e ? MK_FL_ERR : 0);
  return r;
}
template <typename V>
MK_HD MkIvT<V> mk_iv_or(const MkIvT<V>& a, const MkIvT<V>& b) {
  bool aok = a.fl & MK_FL_OK, bok = b.fl & MK_FL_OK;
  bool a_t = aok && a.hi == 1, a_f = aok && a.lo == 0;
  bool b_t = bok && b.hi == 1, b_f = bok && b.lo == 0;
  bool t = a_t || (a_f && b_t);
  bool f = a_f && b_f;
  bool e = (a.fl & MK_FL_ERR) || (a_f && (b.fl & MK_FL_ERR));
  MkIvT<V> r;
  r.lo = f ? 0 : 1;
  r.hi = t ? 1 : 0;
  r.fl = ((t || f) ? MK_FL_OK : 0) | (e ? MK_FL_ERR : 0);
  return r;
}
template <typename V>
MK_HD MkIvT<V> mk_iv_ite(const MkIvT<V>& c, const MkIvT<V>& x, const MkIvT<V>& y) {
  bool cok = c.fl & MK_FL_OK;
  bool c_t = cok && c.hi == 1, c_f = cok && c.lo == 0;
  MkIvT<V> r;
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

// register access policies of the evaluators.  MkIvFile: one file holding
// every register (variables and constants copied in first).  MkIvTemps: the
// file holds only the temporaries (registers >= nvars + nconst); variables
// are read from the box and constants from the problem's constant table, so
// a box evaluation neither copies them nor keeps them in per-thread (local)
// memory -- the k_search hot path.
template <typename V>
struct MkIvFile {
  MkIvT<V>* R;
  MK_HDF MkIvT<V> get(int r) const { return R[r]; }
  MK_HDF void set(int r, const MkIvT<V>& x) { R[r] = x; }
};

// an interval temporary without its flags: one 16-byte (int64) load / store
template <typename V>
struct alignas(16) MkPair {
  V lo, hi;
};

// temporaries only (registers nvars + nconst ...): variables are read from
// the box, constants from the table; the temporaries' OK / ERR flags are bit
// masks held in registers (at most MK_MAXT temporaries), so the register
// file in local memory is {lo, hi} pairs only
template <typename V>
struct MkIvTemps {
  const MkProb* P;
  const V* lo;
  const V* hi;
  MkPair<V>* T;
  int nv, base;
  uint64_t ok = 0, er = 0;
  MK_HDF MkIvT<V> get(int r) const {
    MkIvT<V> o;
    if (r >= base) {
      const int k = r - base;
      const MkPair<V> t = T[k];
      o.lo = t.lo;
      o.hi = t.hi;
      o.fl = (uint8_t)((((ok >> k) & 1) ? MK_FL_OK : 0) | (((er >> k) & 1) ? MK_FL_ERR : 0));
      return o;
    }
    o.fl = MK_FL_OK;
    if (r < nv) {
      o.lo = lo[r];
      o.hi = hi[r];
    } else {
      const V c = MkNum<V>::ld(P->consts[r - nv]);
      o.lo = c;
      o.hi = c;
    }
    return o;
  }
  MK_HDF void set(int r, const MkIvT<V>& x) {
    const int k = r - base;
    MkPair<V> t;
    t.lo = x.lo;
    t.hi = x.hi;
    T[k] = t;
    const uint64_t bit = 1ull << k;
    ok = (x.fl & MK_FL_OK) ? (ok | bit) : (ok & ~bit);
    er = (x.fl & MK_FL_ERR) ? (er | bit) : (er & ~bit);
  }
};

template <typename V, typename Regs>
MK_HD MkBoxVerdict mk_eval_box_impl(const MkProb& P, Regs R, int64_t* insn_count) {
  const int n = P.p->ninsn;
  MkBoxVerdict v;
  v.any_false = false;
  v.all_true = true;
  v.overflow = false;
  v.und_mask = 0;
  MK_NOUNROLL
  for (int k = 0; k < n; ++k) {
    const mk_insn in = P.insns[k];
    switch (in.op) {
      case MK_OP_ATOM: {
        const MkIvT<V> r = R.get(in.a);
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
      case MK_OP_AND: R.set(in.dst, mk_iv_and(R.get(in.a), R.get(in.b))); break;
      case MK_OP_OR: R.set(in.dst, mk_iv_or(R.get(in.a), R.get(in.b))); break;
      case MK_OP_NOT: {
        MkIvT<V> a = R.get(in.a), r;
        r.lo = 1 - a.hi;
        r.hi = 1 - a.lo;
        r.fl = a.fl;
        R.set(in.dst, r);
        break;
      }
      case MK_OP_ITE: R.set(in.dst, mk_iv_ite(R.get(in.a), R.get(in.b), R.get(in.c))); break;
      default: R.set(in.dst, mk_iv_binop<V>(in.op, R.get(in.a), R.get(in.b))); break;
    }
  }
  *insn_count += n;
  return v;
}

// every register in R (variables and constants copied in): the race / access
// generators read arbitrary registers (the offset) after the evaluation
template <typename V>
MK_HD MkBoxVerdict mk_eval_box(const MkProb& P, const V* vlo, const V* vhi, MkIvT<V>* R,
                               int64_t* insn_count) {
  typedef MkNum<V> N;
  const int nv = P.p->nvars;
  const int nc = P.p->nconst;
  MK_NOUNROLL
  for (int i = 0; i < nv; ++i) {
    R[i].lo = vlo[i];
    R[i].hi = vhi[i];
    R[i].fl = MK_FL_OK;
  }
  MK_NOUNROLL
  for (int i = 0; i < nc; ++i) {
    V c = N::ld(P.consts[i]);
    R[nv + i].lo = c;
    R[nv + i].hi = c;
    R[nv + i].fl = MK_FL_OK;
  }
  return mk_eval_box_impl<V>(P, MkIvFile<V>{R}, insn_count);
}

// temporaries only in T (registers nvars + nconst ... nregs - 1)
template <typename V>
MK_HD MkBoxVerdict mk_eval_box_t(const MkProb& P, const V* vlo, const V* vhi, MkPair<V>* T,
                                 int64_t* insn_count) {
  const int nv = P.p->nvars;
  return mk_eval_box_impl<V>(P, MkIvTemps<V>{&P, vlo, vhi, T, nv, nv + P.p->nconst},
                             insn_count);
}

// ---------------------------------------------------------------------------
// bound contraction over the linear rows (one FBBT sweep per call);
// returns false when the box is empty.  Rows of a disjunctive group (group >
// 0, contiguous) contract only when every other row of the group is
// infeasible on the box; a group whose rows are all infeasible empties it.

// activity range of one row over the box: fmin / fmax with the number of
// infinite contributions (wide class only)
template <typename V>
MK_HD void mk_row_range(const mk_row& row, const mk_row_term* T, const V* lo, const V* hi,
                        V& fmin, V& fmax, int& nmin_inf, int& nmax_inf) {
  typedef MkNum<V> N;
  const V INF = N::inf();
  fmin = N::ld(row.c0);
  fmax = fmin;
  nmin_inf = nmax_inf = 0;
  MK_NOUNROLL
  for (int k = 0; k < row.nterms; ++k) {
    V c = N::ld(T[k].coef);
    int v = T[k].var;
    V a = N::mul(c, lo[v]), b = N::mul(c, hi[v]);
    V mn = mk_min(a, b), mx = mk_max(a, b);
    if (N::kWide && mn == -INF) nmin_inf++; else fmin = N::add(fmin, mn);
    if (N::kWide && mx == INF) nmax_inf++; else fmax = N::add(fmax, mx);
  }
}

// the row cannot hold anywhere on the box
template <typename V>
MK_HD bool mk_row_dead(const mk_row& row, V fmin, V fmax, int nmin_inf, int nmax_inf) {
  typedef MkNum<V> N;
  const V INF = N::inf();
  if (nmin_inf == 0 && fmin > 0 && fmin != INF) return true;  // sum >= fmin > 0
  if (N::kWide && nmin_inf == 0 && fmin == INF) return true;
  if (row.rel == 1 && nmax_inf == 0 && fmax < 0 && fmax != -INF) return true;
  if (N::kWide && row.rel == 1 && nmax_inf == 0 && fmax == -INF) return true;
  return false;
}

// tighten every variable of one row; false when a bound crosses
template <typename V>
MK_HD bool mk_row_tighten(const mk_row& row, const mk_row_term* T, V* lo, V* hi, V fmin,
                          V fmax, int nmin_inf, int nmax_inf, bool& changed) {
  typedef MkNum<V> N;
  const V INF = N::inf();
  MK_NOUNROLL
  for (int k = 0; k < row.nterms; ++k) {
    V c = N::ld(T[k].coef);
    int v = T[k].var;
    V a = N::mul(c, lo[v]), b = N::mul(c, hi[v]);
    V mn = mk_min(a, b), mx = mk_max(a, b);
    // others_min = fmin - mn (when finite)
    int oinf = nmin_inf - ((N::kWide && mn == -INF) ? 1 : 0);
    if (oinf == 0) {
      V omin = (N::kWide && mn == -INF) ? fmin : N::sub(fmin, mn);
      if (!N::isinf(omin)) {
        // c*x <= -omin
        if (c > 0) {
          V nb = mk_floordiv<V>(-omin, c);
          if (nb < hi[v]) { hi[v] = nb; changed = true; }
        } else {
          V nb = mk_ceildiv<V>(-omin, c);
          if (nb > lo[v]) { lo[v] = nb; changed = true; }
        }
      }
    }
    if (row.rel == 1) {
      int oinf2 = nmax_inf - ((N::kWide && mx == INF) ? 1 : 0);
      if (oinf2 == 0) {
        V omax = (N::kWide && mx == INF) ? fmax : N::sub(fmax, mx);
        if (!N::isinf(omax)) {
          // c*x >= -omax
          if (c > 0) {
            V nb = mk_ceildiv<V>(-omax, c);
            if (nb > lo[v]) { lo[v] = nb; changed = true; }
          } else {
            V nb = mk_floordiv<V>(-omax, c);
            if (nb < hi[v]) { hi[v] = nb; changed = true; }
          }
        }
      }
    }
    if (lo[v] > hi[v]) return false;
  }
  return true;
}

template <typename V>
MK_HD bool mk_contract(const MkProb& P, V* lo, V* hi, int sweeps) {
  const int nr = P.p->nrows;
  MK_NOUNROLL
  for (int s = 0; s < sweeps; ++s) {
    bool changed = false;
    MK_NOUNROLL
    for (int r = 0; r < nr;) {
      const mk_row row = P.rows[r];
      V fmin, fmax;
      int nmin_inf, nmax_inf;
      if (row.group == 0) {
        const mk_row_term* T = P.terms + row.term_off;
        mk_row_range<V>(row, T, lo, hi, fmin, fmax, nmin_inf, nmax_inf);
        if (mk_row_dead<V>(row, fmin, fmax, nmin_inf, nmax_inf)) return false;
        if (!mk_row_tighten<V>(row, T, lo, hi, fmin, fmax, nmin_inf, nmax_inf, changed))
          return false;
        ++r;
        continue;
      }
      // disjunctive group [r, e): find its live rows
      int e = r + 1;
      while (e < nr && P.rows[e].group == row.group) ++e;
      int live = -1, nlive = 0;
      MK_NOUNROLL
      for (int q = r; q < e && nlive < 2; ++q) {
        const mk_row rq = P.rows[q];
        mk_row_range<V>(rq, P.terms + rq.term_off, lo, hi, fmin, fmax, nmin_inf, nmax_inf);
        if (!mk_row_dead<V>(rq, fmin, fmax, nmin_inf, nmax_inf)) {
          live = q;
          ++nlive;
        }
      }
      if (nlive == 0) return false;
      if (nlive == 1) {
        const mk_row rl = P.rows[live];
        const mk_row_term* T = P.terms + rl.term_off;
        mk_row_range<V>(rl, T, lo, hi, fmin, fmax, nmin_inf, nmax_inf);
        if (!mk_row_tighten<V>(rl, T, lo, hi, fmin, fmax, nmin_inf, nmax_inf, changed))
          return false;
      }
      r = e;
    }
    if (!changed) break;
  }
  return true;
}

// ---------------------------------------------------------------------------
// concrete (point) evaluation.  Registers hold exact values; an error bit per
// register tracks EvalError with the reference's short-circuit rules.

template <typename V>
struct MkCvT {
  V v;
  uint8_t err;
};
typedef MkCvT<i128> MkCv;

template <typename V>
struct MkCvFile {
  MkCvT<V>* R;
  MK_HDF MkCvT<V> get(int r) const { return R[r]; }
  MK_HDF void set(int r, const MkCvT<V>& x) { R[r] = x; }
};

// temporaries only, values in T and the error flags as a bit mask in a
// register (at most MK_MAXT temporaries)
template <typename V>
struct MkCvTemps {
  const MkProb* P;
  const V* x;
  V* T;
  int nv, base;
  uint64_t er = 0;
  MK_HDF MkCvT<V> get(int r) const {
    MkCvT<V> o;
    if (r >= base) {
      const int k = r - base;
      o.v = T[k];
      o.err = (uint8_t)((er >> k) & 1);
      return o;
    }
    o.err = 0;
    o.v = r < nv ? x[r] : MkNum<V>::ld(P->consts[r - nv]);
    return o;
  }
  MK_HDF void set(int r, const MkCvT<V>& v) {
    const int k = r - base;
    T[k] = v.v;
    const uint64_t bit = 1ull << k;
    er = v.err ? (er | bit) : (er & ~bit);
  }
};

template <typename V, typename Regs>
MK_HD bool mk_eval_point_impl(const MkProb& P, Regs R, bool* overflow, int64_t* insn_count) {
  typedef MkNum<V> N;
  const int n = P.p->ninsn;
  bool ovf = false;
  MK_NOUNROLL
  for (int k = 0; k < n; ++k) {
    const mk_insn in = P.insns[k];
    const MkCvT<V> a = R.get(in.a), b = R.get(in.b);
    if (in.op == MK_OP_ATOM) {
      if (a.err || !a.v) {
        *insn_count += k + 1;
        if (ovf) *overflow = true;
        return false;
      }
      continue;
    }
    MkCvT<V> r;
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
        const MkCvT<V> c = R.get(in.c);
        if (a.err) r.err = 1; else r = a.v ? b : c;
        break;
      }
      default: {
        r.err = a.err | b.err;
        if (!r.err) {
          switch (in.op) {
            case MK_OP_ADD: r.v = N::add(a.v, b.v); break;
            case MK_OP_SUB: r.v = N::sub(a.v, b.v); break;
            case MK_OP_MUL: r.v = N::mul(a.v, b.v); break;
            case MK_OP_SHL: r.v = N::shl(a.v, (int)b.v); break;
            case MK_OP_SHR: r.v = N::shr(a.v, (int)b.v); break;
            case MK_OP_DIV:
              if (b.v == 0) r.err = 1; else r.v = mk_tquot(a.v, b.v);
              break;
            case MK_OP_MOD:
              if (b.v == 0) r.err = 1; else r.v = a.v - mk_tquot(a.v, b.v) * b.v;
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
          if (N::isinf(r.v)) ovf = true;
        }
      }
    }
    R.set(in.dst, r);
  }
  *insn_count += n;
  if (ovf) *overflow = true;
  return true;
}

template <typename V>
MK_HD bool mk_eval_point(const MkProb& P, const V* x, MkCvT<V>* R, bool* overflow,
                         int64_t* insn_count) {
  typedef MkNum<V> N;
  const int nv = P.p->nvars;
  const int nc = P.p->nconst;
  MK_NOUNROLL
  for (int i = 0; i < nv; ++i) { R[i].v = x[i]; R[i].err = 0; }
  MK_NOUNROLL
  for (int i = 0; i < nc; ++i) { R[nv + i].v = N::ld(P.consts[i]); R[nv + i].err = 0; }
  return mk_eval_point_impl<V>(P, MkCvFile<V>{R}, overflow, insn_count);
}

// temporaries only in T (the k_search leaf enumeration)
template <typename V>
MK_HD bool mk_eval_point_t(const MkProb& P, const V* x, V* T, bool* overflow,
                           int64_t* insn_count) {
  const int nv = P.p->nvars;
  return mk_eval_point_impl<V>(P, MkCvTemps<V>{&P, x, T, nv, nv + P.p->nconst}, overflow,
                               insn_count);
}

// lexicographic comparison in witness order: true when x is strictly better
template <typename V>
MK_HD bool mk_lex_better(const V* x, const V* y, int nv, uint64_t maxmask) {
  MK_NOUNROLL
  for (int i = 0; i < nv; ++i) {
    if (x[i] == y[i]) continue;
    bool mx = (maxmask >> i) & 1;
    return mx ? (x[i] > y[i]) : (x[i] < y[i]);
  }
  return false;
}

// the best corner of a box (its lexicographic lower bound)
template <typename V>
MK_HD void mk_corner(const V* lo, const V* hi, int nv, uint64_t maxmask, V* out) {
  MK_NOUNROLL
  for (int i = 0; i < nv; ++i) out[i] = ((maxmask >> i) & 1) ? hi[i] : lo[i];
}

// box volume, saturating at 2^62
template <typename V>
MK_HD int64_t mk_volume(const V* lo, const V* hi, int nv) {
  const u128 cap = ((u128)1) << 62;
  u128 v = 1;
  MK_NOUNROLL
  for (int i = 0; i < nv; ++i) {
    u128 s = (u128)(hi[i] - lo[i]) + 1;
    if (s >= cap) return (int64_t)cap;
    v = v * s;
    if (v >= cap) return (int64_t)cap;
  }
  return (int64_t)v;
}
template <typename V>
MK_HD double mk_volume_f(const V* lo, const V* hi, int nv) {
  double v = 1.0;
  MK_NOUNROLL
  for (int i = 0; i < nv; ++i) v *= (double)(hi[i] - lo[i] + 1);
  return v;
}

// decode point #idx of a box in lexicographic order (index order == witness order)
template <typename V>
MK_HD void mk_decode(const V* lo, const V* hi, int nv, uint64_t maxmask, uint64_t idx, V* x) {
  MK_NOUNROLL
  for (int i = nv - 1; i >= 0; --i) {
    uint64_t s = (uint64_t)(hi[i] - lo[i] + 1);
    uint64_t d = idx % s;
    idx /= s;
    x[i] = ((maxmask >> i) & 1) ? hi[i] - (V)d : lo[i] + (V)d;
  }
}

// choose the split symbol among the non-singleton symbols of undecided atoms:
// before any model is known, the smallest domain first (first-fail: refutes
// the narrow core of a query without touching wide launch dimensions); once
// an incumbent exists, the first symbol in witness order (children are then
// lexicographically ordered and the incumbent prunes whole subtrees).
// Returns -1 when every such symbol is fixed.
template <typename V>
MK_HD int mk_pick_split(const V* lo, const V* hi, int nv, uint64_t und_mask,
                        bool have_incumbent) {
  int best = -1;
  V bw = 0;
  MK_NOUNROLL
  for (int i = 0; i < nv; ++i) {
    if (!((und_mask >> i) & 1) || lo[i] >= hi[i]) continue;
    if (have_incumbent) return i;
    V w = hi[i] - lo[i];
    if (best < 0 || w < bw) {
      best = i;
      bw = w;
    }
  }
  return best;
}

// piece t (0 = best in the symbol's direction) of m near-equal pieces of [lo,hi]
template <typename V>
MK_HD void mk_piece(V lo, V hi, int m, int t, bool maximize, V* plo, V* phi) {
  typedef typename MkNum<V>::U U;
  U size = (U)(hi - lo) + 1;
  U q = size / (U)m, rem = size % (U)m;
  // ascending piece j covers [lo + j*q + min(j,rem), ...]
  int j = maximize ? (m - 1 - t) : t;
  U start = (U)j * q + ((U)j < rem ? (U)j : rem);
  U len = q + ((U)j < rem ? 1 : 0);
  *plo = lo + (V)start;
  *phi = *plo + (V)len - 1;
}

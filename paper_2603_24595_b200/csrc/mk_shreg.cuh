// mk_shreg.cuh -- narrow (int64) evaluators with the register file in shared
// memory, for the hot kernels (k_search's small narrow problems, the K2 race
// generator).  Register r of thread t lives at sh[r * blockDim.x + t]
// (consecutive lanes hit consecutive banks); flags are bit masks over the
// registers (these problems have <= 64 registers).  Semantics are exactly
// mk_core.cuh's mk_eval_point<int64_t> / mk_eval_box<int64_t>: the interval
// step calls the same mk_iv_binop / mk_iv_and / mk_iv_or / mk_iv_ite.  The
// local-memory register files of the generic evaluators spill to L2 at
// full occupancy (ncu: long-scoreboard stalls on the register loads).
#pragma once
#include "mk_core.cuh"

// Point evaluation of a narrow problem with the register file in shared
// memory (register r of thread t at sh[r * blockDim.x + t]: consecutive lanes
// hit consecutive banks) and the EvalError flags as a bit mask (small
// problems have <= 64 registers).  Same semantics as mk_core.cuh
// mk_eval_point<int64_t>; the local-memory register file of the generic
// evaluator spills to L2 at full occupancy.
__device__ __forceinline__ bool sh_eval_point(const MkProb& P, const int64_t* x, int64_t* sh) {
  const int nv = P.p->nvars;
  const int nc = P.p->nconst;
  const int bd = blockDim.x, t = threadIdx.x;
  uint64_t err = 0;
  for (int i = 0; i < nv; ++i) sh[i * bd + t] = x[i];
  for (int i = 0; i < nc; ++i) sh[(nv + i) * bd + t] = (int64_t)P.consts[i].lo;
  const int n = P.p->ninsn;
  for (int k = 0; k < n; ++k) {
    const mk_insn in = P.insns[k];
    const int64_t a = sh[in.a * bd + t];
    const bool ea = (err >> in.a) & 1;
    if (in.op == MK_OP_ATOM) {
      if (ea || !a) return false;
      continue;
    }
    const int64_t b = sh[in.b * bd + t];
    const bool eb = (err >> in.b) & 1;
    int64_t r = 0;
    bool e = false;
    switch (in.op) {
      case MK_OP_AND: if (ea) e = true; else if (!a) r = 0; else { r = b ? 1 : 0; e = eb; } break;
      case MK_OP_OR: if (ea) e = true; else if (a) r = 1; else { r = b ? 1 : 0; e = eb; } break;
      case MK_OP_NOT: e = ea; r = a ? 0 : 1; break;
      case MK_OP_ITE: {
        const int64_t c = sh[in.c * bd + t];
        const bool ec = (err >> in.c) & 1;
        if (ea) e = true; else if (a) { r = b; e = eb; } else { r = c; e = ec; }
        break;
      }
      default:
        e = ea || eb;
        if (!e) {
          switch (in.op) {
            case MK_OP_ADD: r = a + b; break;
            case MK_OP_SUB: r = a - b; break;
            case MK_OP_MUL: r = a * b; break;
            case MK_OP_SHL: r = MkNum<int64_t>::shl(a, (int)b); break;
            case MK_OP_SHR: r = MkNum<int64_t>::shr(a, (int)b); break;
            case MK_OP_DIV: if (b == 0) e = true; else r = a / b; break;
            case MK_OP_MOD: if (b == 0) e = true; else r = a % b; break;
            case MK_OP_EMOD: if (b == 0) e = true; else r = mk_emod_c<int64_t>(a, b); break;
            case MK_OP_EQ: r = a == b; break;
            case MK_OP_NE: r = a != b; break;
            case MK_OP_LT: r = a < b; break;
            case MK_OP_LE: r = a <= b; break;
            case MK_OP_GT: r = a > b; break;
            case MK_OP_GE: r = a >= b; break;
            default: break;
          }
        }
    }
    sh[in.dst * bd + t] = r;
    err = e ? (err | (1ull << in.dst)) : (err & ~(1ull << in.dst));
  }
  return true;
}


// interval evaluation of a box; lo/hi register files in shared memory,
// OK / ERR flags as masks
__device__ __forceinline__ MkBoxVerdict sh_eval_box(const MkProb& P, const int64_t* vlo,
                                                    const int64_t* vhi, int64_t* shlo,
                                                    int64_t* shhi, int64_t* insn_count) {
  const int nv = P.p->nvars;
  const int nc = P.p->nconst;
  const int bd = blockDim.x, t = threadIdx.x;
  uint64_t okm = 0, erm = 0;
  for (int i = 0; i < nv; ++i) {
    shlo[i * bd + t] = vlo[i];
    shhi[i * bd + t] = vhi[i];
    okm |= 1ull << i;
  }
  for (int i = 0; i < nc; ++i) {
    const int64_t c = (int64_t)P.consts[i].lo;
    shlo[(nv + i) * bd + t] = c;
    shhi[(nv + i) * bd + t] = c;
    okm |= 1ull << (nv + i);
  }
  auto load = [&](int r) {
    MkIvT<int64_t> v;
    v.lo = shlo[r * bd + t];
    v.hi = shhi[r * bd + t];
    v.fl = (uint8_t)((((okm >> r) & 1) ? MK_FL_OK : 0) | (((erm >> r) & 1) ? MK_FL_ERR : 0));
    return v;
  };
  const int n = P.p->ninsn;
  MkBoxVerdict v;
  v.any_false = false;
  v.all_true = true;
  v.overflow = false;
  v.und_mask = 0;
  for (int k = 0; k < n; ++k) {
    const mk_insn in = P.insns[k];
    if (in.op == MK_OP_ATOM) {
      const MkIvT<int64_t> r = load(in.a);
      const bool ok = r.fl & MK_FL_OK;
      const bool may_true = ok && r.hi == 1;
      const bool sure_true = ok && r.lo == 1 && !(r.fl & MK_FL_ERR);
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
      continue;
    }
    MkIvT<int64_t> r;
    switch (in.op) {
      case MK_OP_AND: r = mk_iv_and(load(in.a), load(in.b)); break;
      case MK_OP_OR: r = mk_iv_or(load(in.a), load(in.b)); break;
      case MK_OP_NOT: {
        const MkIvT<int64_t> a = load(in.a);
        r.lo = 1 - a.hi;
        r.hi = 1 - a.lo;
        r.fl = a.fl;
        break;
      }
      case MK_OP_ITE: r = mk_iv_ite(load(in.a), load(in.b), load(in.c)); break;
      default: r = mk_iv_binop<int64_t>(in.op, load(in.a), load(in.b)); break;
    }
    shlo[in.dst * bd + t] = r.lo;
    shhi[in.dst * bd + t] = r.hi;
    const uint64_t bit = 1ull << in.dst;
    okm = (r.fl & MK_FL_OK) ? (okm | bit) : (okm & ~bit);
    erm = (r.fl & MK_FL_ERR) ? (erm | bit) : (erm & ~bit);
  }
  *insn_count += n;
  return v;
}

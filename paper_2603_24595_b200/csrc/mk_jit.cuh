// mk_jit.cuh -- specialised evaluator for the K2 race generator: the path
// bytecode of one store is compiled at run time (NVRTC, sm_100a cubin) into a
// straight-line CUDA kernel whose registers are scalar locals.  Included by
// mk_engine.cu after mk_race.cuh's device code.
//
// The generated statements restate sh_eval_point (mk_shreg.cuh), i.e. the
// reference's mathematical-mode semantics (sym/expr.py:273-383): exact int64
// arithmetic on a narrow problem, truncating div / mod, Euclidean emod,
// shl = *2^k, shr = floor shift, an error flag per register with the
// short-circuit rules of and / or / ite, division by zero is an error, an
// atom that is false or in error ends the instance (solver/query.py:45-62).
// NVRTC is loaded with dlopen on first use: a host without it (or a compile
// failure) keeps the interpreted generator, which computes the same tuples.
#pragma once
#include <dlfcn.h>
#include <nvrtc.h>

#include <functional>
#include <map>
#include <vector>
#include <sstream>
#include <string>

namespace mkjit {

struct Nvrtc {
  bool tried = false, ok = false;
  void* h = nullptr;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*,
                        const char* const*) = nullptr;
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*cubin)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*log_size)(nvrtcProgram, size_t*) = nullptr;
  nvrtcResult (*log)(nvrtcProgram, char*) = nullptr;
  nvrtcResult (*destroy)(nvrtcProgram*) = nullptr;

  bool load() {
    if (tried) return ok;
    tried = true;
    const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) return false;
    create = (decltype(create))dlsym(h, "nvrtcCreateProgram");
    compile = (decltype(compile))dlsym(h, "nvrtcCompileProgram");
    cubin_size = (decltype(cubin_size))dlsym(h, "nvrtcGetCUBINSize");
    cubin = (decltype(cubin))dlsym(h, "nvrtcGetCUBIN");
    log_size = (decltype(log_size))dlsym(h, "nvrtcGetProgramLogSize");
    log = (decltype(log))dlsym(h, "nvrtcGetProgramLog");
    destroy = (decltype(destroy))dlsym(h, "nvrtcDestroyProgram");
    ok = create && compile && cubin_size && cubin && log_size && log && destroy;
    return ok;
  }
};

inline Nvrtc& nvrtc() {
  static Nvrtc n;
  return n;
}

inline std::string lit(int64_t v) {
  if (v == INT64_MIN) return "(-9223372036854775807LL - 1)";
  std::ostringstream o;
  o << v << "LL";
  return o.str();
}

// Straight-line evaluation of one path program's bytecode (registers as
// locals v<r> with error flags e<r>; an atom that is false or in error
// breaks out of the enclosing do { } while (0)).  Vars are x<i>.
inline void emit_path(std::ostringstream& s, const mk_problem& p, const mk_insn* insns,
                      const mk_i128* consts, const int* rbits) {
  const int nv = p.nvars, nc = p.nconst, nr = p.nregs;
  auto b32 = [&](int r) { return rbits && rbits[r] == 32; };
  auto ty = [&](int r) { return b32(r) ? "int" : "i64"; };
  for (int r = nv + nc; r < nr; ++r) s << "      " << ty(r) << " v" << r << " = 0; bool e" << r << " = false;\n";
  for (int i = 0; i < nv; ++i) s << "      const " << ty(i) << " v" << i << " = x" << i << "; const bool e" << i << " = false;\n";
  for (int i = 0; i < nc; ++i)
    s << "      const " << ty(nv + i) << " v" << (nv + i) << " = " << lit((int64_t)consts[i].lo)
      << "; const bool e" << (nv + i) << " = false;\n";
  for (int k = 0; k < p.ninsn; ++k) {
    const mk_insn in = insns[k];
    const int a = in.a, b = in.b, c = in.c, d = in.dst;
    if (in.op == MK_OP_ATOM) {
      s << "      if (e" << a << " || !v" << a << ") break;\n";
      continue;
    }
    // 32-bit arithmetic only when operands and result are all int32-bounded
    // (then the mathematical result is the int32 result); shifts stay int64
    const bool arith32 = b32(a) && b32(b) && b32(d) && in.op != MK_OP_SHL && in.op != MK_OP_SHR;
    const char* OT = arith32 ? "int" : "i64";
    s << "      { const " << OT << " A = (" << OT << ")v" << a << ", B = (" << OT << ")v" << b
      << "; const bool EA = e" << a << ", EB = e" << b << "; " << OT
      << " R = 0; bool E = false; (void)A; (void)B; (void)EA; (void)EB;\n        ";
    switch (in.op) {
      case MK_OP_AND: s << "if (EA) E = true; else if (!A) R = 0; else { R = B ? 1 : 0; E = EB; }"; break;
      case MK_OP_OR: s << "if (EA) E = true; else if (A) R = 1; else { R = B ? 1 : 0; E = EB; }"; break;
      case MK_OP_NOT: s << "E = EA; R = A ? 0 : 1;"; break;
      case MK_OP_ITE:
        s << "const " << OT << " C = (" << OT << ")v" << c << "; const bool EC = e" << c
          << "; if (EA) E = true; else if (A) { R = B; E = EB; } else { R = C; E = EC; }";
        break;
      default: {
        s << "E = EA || EB; if (!E) { ";
        switch (in.op) {
          case MK_OP_ADD: s << "R = A + B;"; break;
          case MK_OP_SUB: s << "R = A - B;"; break;
          case MK_OP_MUL: s << "R = A * B;"; break;
          case MK_OP_SHL: s << "R = mk_shl(A, B);"; break;
          case MK_OP_SHR: s << "R = mk_shr(A, B);"; break;
          case MK_OP_DIV: s << "if (B == 0) E = true; else R = A / B;"; break;
          case MK_OP_MOD: s << "if (B == 0) E = true; else R = A % B;"; break;
          case MK_OP_EMOD:
            s << "if (B == 0) E = true; else R = " << (arith32 ? "mk_emod32" : "mk_emod") << "(A, B);";
            break;
          case MK_OP_EQ: s << "R = A == B;"; break;
          case MK_OP_NE: s << "R = A != B;"; break;
          case MK_OP_LT: s << "R = A < B;"; break;
          case MK_OP_LE: s << "R = A <= B;"; break;
          case MK_OP_GT: s << "R = A > B;"; break;
          case MK_OP_GE: s << "R = A >= B;"; break;
          default: s << "E = true;"; break;
        }
        s << " }";
      }
    }
    s << "\n        v" << d << " = (" << ty(d) << ")R; e" << d << " = E; }\n";
  }
}

// CUDA source of the race generators for one program (host copy of the
// problem).  Key type, sentinel, offset origin and block radix are baked in.
// Two kernels share one generated access function:
//   mk_race_gen_jit    dense (key, index) tuples for the sort path;
//   mk_race_fused_jit  the ordered fast path: every warp walks a contiguous
//                      instance range (lane l takes base + l + 32 j), compares
//                      each access with the previous one in instance order in
//                      registers (ballot + shuffles), and leaves only a
//                      per-warp summary (first / last access) for the chunk
//                      boundary pass.  Nothing per instance touches HBM.
// rbits[r] (optional) is 32 when register r provably stays inside int32 on
// the whole instance box (interval evaluation of the root box, inclusion
// isotonic): such registers are 32-bit locals and an operation whose
// operands and result are all 32-bit runs on the 32-bit pipe; everything
// else is exact int64 (the narrow class).
// instances per thread of the compacting generator's tile (256 threads)
inline int gc_items() {
  static const int v = [] {
    const char* e = getenv("MK_GC_ITEMS");
    const int x = e ? atoi(e) : 32;
    return x >= 4 && x <= 64 && x % 4 == 0 ? x : 32;   // a multiple of 4 (the count scan)
  }();
  return v;
}

// ", N": the compacting generator asks for N resident 256-thread CTAs per SM
// (a register cap).  Default 5, measured on the B200 (config 1's forced sort
// path: uncapped 115 registers, 2 CTAs per SM, generation 3.38 ms; 5 CTAs
// 2.47 ms; 4: 2.67; 6: 2.59; 8: 3.19; profiles/r02_k2_genc_minb.jsonl).
// MK_GC_MINB=0 leaves the registers uncapped.
inline std::string gc_minb() {
  const char* e = getenv("MK_GC_MINB");
  const int x = e ? atoi(e) : 5;
  return x > 0 && x <= 8 ? ", " + std::to_string(x) : std::string();
}

inline std::string race_gen_source(const mk_problem& p, const mk_insn* insns,
                                   const mk_i128* consts, int n_outer, int off_reg, int shared,
                                   const int id_var[6], const int64_t* lo, const int64_t* hi,
                                   bool key64, const int* rbits = nullptr, int64_t off_lo = 0,
                                   unsigned long long nblocks = 1) {
  const int nv = p.nvars, nc = p.nconst, nr = p.nregs;
  std::ostringstream s;
  const char* KT = key64 ? "unsigned long long" : "unsigned int";
  auto b32 = [&](int r) { return rbits && rbits[r] == 32; };
  auto ty = [&](int r) { return b32(r) ? "int" : "i64"; };
  s << "typedef long long i64;\ntypedef unsigned long long u64;\n"
       "__device__ __forceinline__ i64 mk_emod(i64 a, i64 b) { i64 m = b < 0 ? -b : b; i64 r = a % m;"
       " return r < 0 ? r + m : r; }\n"
       "__device__ __forceinline__ int mk_emod32(int a, int b) { int m = b < 0 ? -b : b; int r = a % m;"
       " return r < 0 ? r + m : r; }\n"
       "__device__ __forceinline__ i64 mk_shl(i64 a, i64 k) { return k >= 62 ? 0 :"
       " (i64)((unsigned long long)a << k); }\n"
       "__device__ __forceinline__ i64 mk_shr(i64 a, i64 k) { return a >> (k > 63 ? 63 : k); }\n";
  for (int i = 0; i < nv; ++i) {
    s << "#define lo" << i << " " << lit(lo[i]) << "\n#define sp" << i << " " << lit(hi[i] - lo[i] + 1)
      << "\n";
  }
  // the access function: leading values in, (hit, key) out
  s << "__device__ __forceinline__ bool mk_acc(";
  for (int i = 0; i < n_outer; ++i) s << (i ? ", " : "") << "const " << ty(i) << " x" << i;
  s << (n_outer ? ", " : "") << "u64& done, " << KT << "& key) {\n";
  unsigned long long inner = 1;
  for (int i = n_outer; i < nv; ++i) inner *= (unsigned long long)(hi[i] - lo[i] + 1);
  // with no existential vars every instance is one evaluation: the callers
  // count them per warp instead of per instance
  const bool count_inner = inner > 1;
  s << "  for (unsigned long long j = 0; j < " << inner << "ULL; ++j) {\n";
  if (nv > n_outer) {
    s << "    unsigned long long jj = j;\n";
    for (int i = nv - 1; i >= n_outer; --i)
      s << "    const " << ty(i) << " x" << i << " = (" << ty(i) << ")(lo" << i
        << " + (i64)(jj % (unsigned long long)sp" << i << ")); jj /= (unsigned long long)sp" << i << ";\n";
  }
  s << (count_inner ? "    ++done;\n" : "") << "    bool hit = false;\n    i64 off = 0;\n    do {\n";
  emit_path(s, p, insns, consts, rbits);
  s << "      hit = true; off = (i64)v" << off_reg << ";\n    } while (0);\n";
  s << "    if (hit) {\n      u64 bk = 0;\n";
  if (shared) {
    for (int ax = 2; ax >= 0; --ax) {
      const int v = id_var[ax];
      if (v < 0) continue;
      s << "      bk = bk * (u64)sp" << v << " + (u64)((i64)x" << v << " - lo" << v << ");\n";
    }
  }
  s << "      key = (" << KT << ")((u64)(off - (" << lit(off_lo) << ")) * " << nblocks
    << "ull + bk);\n      (void)done;\n      return true;\n    }\n"
       "  }\n  (void)done;\n  return false;\n}\n";
  // the identity of an instance as one integer (< 2^31: mixed radix of its
  // thread-identity digits; shared memory: thread ids only, the key holds the
  // block)
  s << "__device__ __forceinline__ unsigned mk_idk(";
  for (int i = 0; i < n_outer; ++i) s << (i ? ", " : "") << "const int d" << i;
  s << ") {\n  unsigned k = 0;\n";
  for (int ax = shared ? 3 : 0; ax < 6; ++ax) {
    const int v = id_var[ax];
    if (v < 0) continue;
    s << "  k = k * (unsigned)sp" << v << " + (unsigned)d" << v << ";\n";
  }
  s << "  return k;\n}\n";
  s << "__device__ __noinline__ unsigned mk_idk_of(unsigned long long a) {\n";
  for (int i = n_outer - 1; i >= 0; --i)
    s << "  const int d" << i << " = (int)(a % (unsigned long long)sp" << i << "); a /= (unsigned long long)sp" << i
      << ";\n";
  s << "  return mk_idk(";
  for (int i = 0; i < n_outer; ++i) s << (i ? ", " : "") << "d" << i;
  s << ");\n}\n";
  // leading digits are int32 (the instance box holds < 2^31 instances)
  auto call_args = [&]() {
    std::ostringstream a;
    for (int i = 0; i < n_outer; ++i) a << "(" << ty(i) << ")(lo" << i << " + d" << i << "), ";
    return a.str();
  };
  auto id_args = [&]() {
    std::ostringstream a;
    for (int i = 0; i < n_outer; ++i) a << (i ? ", " : "") << "d" << i;
    return a.str();
  };
  // mixed-radix odometer over the leading digits; the step's digits are
  // literals (32 for the fused pass), or computed from the grid stride
  auto odometer_init = [&](const char* start, const char* step, unsigned long long cstep) {
    std::ostringstream o;
    for (int i = 0; i < n_outer; ++i) o << "  int d" << i << ", t" << i << ";\n";
    o << "  { unsigned long long a = " << start << ", b = " << step << "; (void)b;\n";
    unsigned long long c = cstep;
    for (int i = n_outer - 1; i >= 0; --i) {
      const unsigned long long sp = (unsigned long long)(hi[i] - lo[i] + 1);
      o << "    d" << i << " = (int)(a % (unsigned long long)sp" << i << "); a /= (unsigned long long)sp" << i << "; ";
      if (cstep) {
        o << "t" << i << " = " << (c % sp) << ";\n";
        c /= sp;
      } else {
        o << "t" << i << " = (int)(b % (unsigned long long)sp" << i << "); b /= (unsigned long long)sp" << i << ";\n";
      }
    }
    o << "  }\n";
    return o.str();
  };
  auto odometer_step = [&]() {
    std::ostringstream o;
    o << "    { int c = 0;\n";
    for (int i = n_outer - 1; i >= 0; --i) {
      o << "      d" << i << " += t" << i << " + c; c = d" << i << " >= (int)sp" << i << "; if (c) d" << i
        << " -= (int)sp" << i << ";\n";
    }
    o << "      (void)c;\n    }\n";
    return o.str();
  };
  // dense generator (sort path)
  s << "extern \"C\" __global__ void __launch_bounds__(256) mk_race_gen_jit(unsigned long long vol, "
    << KT << " sentinel, " << KT
    << "* keys, unsigned int* vals, unsigned long long* count, unsigned long long* evaluated,"
       " i64 off_lo, unsigned long long nblocks) {\n"
       "  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;\n"
       "  unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;\n"
    << odometer_init("idx", "stride", 0)
    << "  unsigned long long done = 0, models = 0;\n"
       "  for (; idx < vol; idx += stride) {\n"
       "    " << KT << " key = sentinel;\n"
       << (count_inner ? "" : "    ++done;\n") <<
       "    if (mk_acc(" << call_args() << "done, key)) ++models; else key = sentinel;\n"
       "    keys[idx] = key;\n    vals[idx] = (unsigned int)idx;\n"
    << odometer_step()
    << "  }\n"
       "  for (int o = 16; o > 0; o >>= 1) { done += __shfl_down_sync(0xffffffffu, done, o);"
       " models += __shfl_down_sync(0xffffffffu, models, o); }\n"
       "  if ((threadIdx.x & 31) == 0) { if (done) atomicAdd(evaluated, done);"
       " if (models) atomicAdd(count, models); }\n}\n";
  // compacting generator (sort path): each CTA takes the next tile of
  // 256 x 8 instances in order (tile counter), evaluates them (item j of
  // thread t is instance base + 256 j + t), counts the accesses per (item,
  // warp), gets the tile's output offset by a decoupled look-back over the
  // tiles before it and writes only the accesses, in instance order -- the
  // separate compaction's full read and write of every tuple never happens
  s << "__device__ __forceinline__ u64 gc_ld(const u64* p) { u64 v; asm volatile(\"ld.volatile.global.u64 %0, [%1];\""
       " : \"=l\"(v) : \"l\"(p)); return v; }\n"
       "__device__ __forceinline__ void gc_st(u64* p, u64 v) { asm volatile(\"st.volatile.global.u64 [%0], %1;\""
       " :: \"l\"(p), \"l\"(v)); }\n"
       "#define GC_ITEMS " << gc_items() << "\n"
       "#define GC_AGG (1ull << 32)\n#define GC_INCL (2ull << 32)\n"
       "extern \"C\" __global__ void __launch_bounds__(256" << gc_minb() << ") mk_race_genc_jit(unsigned long long vol, "
    << KT << "* keys, unsigned int* vals, unsigned long long* count, unsigned long long* evaluated,"
       " u64* lookback, unsigned int* tile_ctr, unsigned long long epoch) {\n"
       "  __shared__ unsigned tile_s;\n  __shared__ unsigned cnt[GC_ITEMS * 8];\n"
       "  __shared__ u64 prefix_s;\n"
       "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n"
       "  if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1u);\n  __syncthreads();\n"
       "  const unsigned tile = tile_s;\n"
       "  const unsigned long long base = (unsigned long long)tile * (256ull * GC_ITEMS);\n"
       "  unsigned long long idx = base + threadIdx.x;\n"
    << odometer_init("idx", "256ull", 256)
    << "  unsigned long long done = 0, models = 0;\n"
       "  " << KT << " key[GC_ITEMS];\n  unsigned keep[GC_ITEMS];\n"
       "#pragma unroll\n"
       "  for (int j = 0; j < GC_ITEMS; ++j) {\n"
       "    " << KT << " k = 0;\n    bool hit = false;\n"
       "    if (idx < vol) {\n"
       << (count_inner ? "" : "      ++done;\n") <<
       "      hit = mk_acc(" << call_args() << "done, k);\n"
       "    }\n"
       "    if (hit) ++models;\n"
       "    key[j] = k;\n"
       "    keep[j] = __ballot_sync(0xffffffffu, hit);\n"
       "    if (lane == 0) cnt[j * 8 + warp] = __popc(keep[j]);\n"
       "    idx += 256;\n"
    << odometer_step()
    << "  }\n  __syncthreads();\n"
       "  if (warp == 0) {\n"
       "    constexpr int E = GC_ITEMS / 4;   // (item, warp) counts per lane, in order\n"
       "    unsigned loc[E], sum = 0;\n"
       "#pragma unroll\n"
       "    for (int e = 0; e < E; ++e) { loc[e] = cnt[lane * E + e]; sum += loc[e]; }\n"
       "    unsigned incl = sum;\n"
       "    for (int o = 1; o < 32; o <<= 1) { const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);"
       " if (lane >= o) incl += y; }\n"
       "    unsigned run = incl - sum;\n"
       "#pragma unroll\n"
       "    for (int e = 0; e < E; ++e) { cnt[lane * E + e] = run; run += loc[e]; }\n"
       "    const unsigned total = __shfl_sync(0xffffffffu, incl, 31);\n"
       "    const u64 tag = epoch << 34;\n"
       "    u64 prefix = 0;\n"
       "    if (tile == 0) {\n      if (lane == 0) gc_st(lookback, tag | GC_INCL | total);\n"
       "    } else {\n"
       "      if (lane == 0) gc_st(lookback + tile, tag | GC_AGG | total);\n"
       "      long long p = (long long)tile - 1;\n"
       "      while (p >= 0) {\n"
       "        const long long q = p - (long long)lane;\n"
       "        u64 e = q >= 0 ? gc_ld(lookback + q) : (tag | GC_INCL);\n"
       "        while ((e >> 34) != epoch || (e & (3ull << 32)) == 0) e = gc_ld(lookback + q);\n"
       "        const unsigned inc = __ballot_sync(0xffffffffu, (e & GC_INCL) != 0);\n"
       "        const unsigned upto = inc ? (unsigned)(__ffs(inc) - 1) : 31u;\n"
       "        u64 c = ((unsigned)lane <= upto && q >= 0) ? (e & 0xffffffffull) : 0ull;\n"
       "        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);\n"
       "        prefix += c;\n"
       "        if (inc) break;\n"
       "        p -= 32;\n"
       "      }\n"
       "      if (lane == 0) gc_st(lookback + tile, tag | GC_INCL | (prefix + total));\n"
       "    }\n"
       "    if (lane == 0) prefix_s = prefix;\n"
       "  }\n  __syncthreads();\n"
       "  const u64 pre = prefix_s;\n"
       "  const unsigned lt = (1u << lane) - 1u;\n"
       "  idx = base + threadIdx.x;\n"
       "#pragma unroll\n"
       "  for (int j = 0; j < GC_ITEMS; ++j) {\n"
       "    if ((keep[j] >> lane) & 1u) {\n"
       "      const u64 o = pre + cnt[j * 8 + warp] + __popc(keep[j] & lt);\n"
       "      keys[o] = key[j];\n      vals[o] = (unsigned int)idx;\n"
       "    }\n"
       "    idx += 256;\n"
       "  }\n"
       "  for (int o = 16; o > 0; o >>= 1) { done += __shfl_down_sync(0xffffffffu, done, o);"
       " models += __shfl_down_sync(0xffffffffu, models, o); }\n"
       "  if (lane == 0) { if (done) atomicAdd(evaluated, done); if (models) atomicAdd(count, models); }\n}\n";
  // one warp step of the fused pass over instances b0 .. b0 + 31 (lane l
  // holds b0 + l); `guarded`: the tail step, lanes past the range idle
  auto step = [&](bool guarded) {
    std::ostringstream o;
    o << "    const unsigned idx = b0 + lane;\n"
         "    " << KT << " key = 0;\n"
         "    bool valid = false;\n";
    if (guarded) o << "    if (idx < uend) valid = mk_acc(" << call_args() << "done, key);\n";
    else o << "    valid = mk_acc(" << call_args() << "done, key);\n";
    o << "    const unsigned mask = __ballot_sync(0xffffffffu, valid);\n"
         "    if (mask) {\n"
         "      const unsigned lower = mask & lt;\n"
         "      const int src = lower ? 31 - __clz(lower) : 0;\n"
         "      " << KT << " pk = __shfl_sync(0xffffffffu, key, src);\n"
         "      if (!lower) pk = ck;\n"
         "      const bool ph = lower ? true : have;\n"
         "      models += valid ? 1u : 0u;\n"
         "      if (valid && ph && key < pk) down = true;\n"
         "      const bool eq = valid && ph && key == pk;\n"
         "      if (__any_sync(0xffffffffu, eq)) {\n"
         "        const unsigned idk = valid ? mk_idk(" << id_args() << ") : 0u;\n"
         "        unsigned pi = __shfl_sync(0xffffffffu, idk, src);\n"
         "        const unsigned px = lower ? b0 + (unsigned)src : cx;\n"
         "        if (eq && !lower) pi = mk_idk_of(cx);\n"
         "        if (eq && idk != pi) { ++conf; const u64 c = ((u64)idx << 32) | px;"
         " if (c < best) { best = c; bkey = (u64)key; } }\n"
         "      }\n"
         "      if (!have) { const int fl = __ffs(mask) - 1; fk = __shfl_sync(0xffffffffu, key, fl);"
         " fx = b0 + (unsigned)fl; }\n"
         "      const int hl = 31 - __clz(mask);\n"
         "      ck = __shfl_sync(0xffffffffu, key, hl); cx = b0 + (unsigned)hl;\n"
         "      have = true;\n"
         "    }\n";
    return o.str();
  };
  // fused ordered scan (fast path).  rec: MK_RACE_REC u64 per warp = have,
  // first key, first identity, first index, last key, last identity, last
  // index, best conflict (idx_b << 32 | idx_a), its key, pad.
  // ctr: [0] accesses [1] conflicts [2] min (idx_b << 32 | idx_a) [3]
  // evaluations [4] out-of-order flag.  Lane l holds instance b0 + l, so
  // instance indices need no shuffle; the hot loop moves only keys (ballot +
  // two shuffles), identities are computed only on the rare equal-key steps.
  s << "extern \"C\" __global__ void __launch_bounds__(256) mk_race_fused_jit(unsigned long long vol, "
       "unsigned long long chunk, unsigned long long start, unsigned long long nblocks_unused, u64* rec,"
       " u64* ctr) {\n"
       "  const unsigned lane = threadIdx.x & 31;\n"
       "  const unsigned long long warp = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;\n"
       "  const unsigned long long base = start + warp * chunk;\n"
       "  unsigned long long end = base + chunk; if (end > start + vol) end = start + vol;\n"
       "  const unsigned uend = (unsigned)(end < base ? base : end);\n"
       "  const unsigned lt = (1u << lane) - 1u;\n"
    << odometer_init("(base + lane)", "32ull", 32)
    << "  u64 done = 0, conf = 0, best = ~0ull, bkey = 0;\n"
       "  unsigned models = 0;\n"
       "  bool have = false, down = false;\n"
       "  " << KT << " ck = 0, fk = 0;\n"
       "  unsigned cx = 0, fx = 0;\n"
       "  unsigned b0 = (unsigned)base;\n"
       "  // full steps (every lane in range), then at most one guarded tail step\n"
       "  for (; b0 + 32u <= uend; b0 += 32) {\n"
    << step(false) << odometer_step()
    << "  }\n"
       "  if (b0 < uend) {\n"
    << step(true)
    << "  }\n"
    << (count_inner ? "" : "  done = (lane == 0 && uend > (unsigned)base) ? (u64)(uend - (unsigned)base) : 0ull;\n")
    << "  u64 m64 = models;\n"
       "  for (int o = 16; o > 0; o >>= 1) {\n"
       "    done += __shfl_down_sync(0xffffffffu, done, o);\n"
       "    m64 += __shfl_down_sync(0xffffffffu, m64, o);\n"
       "    conf += __shfl_down_sync(0xffffffffu, conf, o);\n"
       "    const u64 b2 = __shfl_down_sync(0xffffffffu, best, o), k2 = __shfl_down_sync(0xffffffffu, bkey, o);\n"
       "    if (b2 < best) { best = b2; bkey = k2; }\n"
       "  }\n"
       "  const bool anydown = __any_sync(0xffffffffu, down);\n"
       "  if (lane == 0) {\n"
       "    u64* r = rec + warp * 10;\n"
       "    r[0] = have ? 1ull : 0ull; r[1] = (u64)fk; r[2] = have ? mk_idk_of(fx) : 0u; r[3] = fx;\n"
       "    r[4] = (u64)ck; r[5] = have ? mk_idk_of(cx) : 0u; r[6] = cx;\n"
       "    r[7] = best; r[8] = bkey;\n"
       "    if (m64) atomicAdd(ctr + 0, m64);\n"
       "    if (conf) atomicAdd(ctr + 1, conf);\n"
       "    if (best != ~0ull) atomicMin(ctr + 2, best);\n"
       "    if (done) atomicAdd(ctr + 3, done);\n"
       "    if (anydown) atomicOr(ctr + 4, 1ull);\n"
       "  }\n}\n";
  return s.str();
}

// CUDA source of the multi-access generator (mk_access.cuh): one straight-
// line access function per access program and one kernel that dispatches a
// global instance index to its program with a balanced if-tree over the
// literal instance starts.  mode 0: dense (key, val) tuples; 1 / 2: the
// owner-table write / read passes (semantics of k_acc_gen).
struct AccGenInfo {
  int n_outer = 0;
  unsigned long long start = 0, slot = 0, vol = 0;
  std::vector<int64_t> lo, hi;
  std::vector<int> rbits;
};

inline std::string access_gen_source(const mk_problem_set& set, const mk_access_prog* progs,
                                     const std::vector<AccGenInfo>& info, const long long grid[3],
                                     const long long block[3], unsigned long long total) {
  const int np = set.nprob;
  std::ostringstream s;
  s << "typedef long long i64;\ntypedef unsigned long long u64;\n"
       "__device__ __forceinline__ i64 mk_emod(i64 a, i64 b) { i64 m = b < 0 ? -b : b; i64 r = a % m;"
       " return r < 0 ? r + m : r; }\n"
       "__device__ __forceinline__ int mk_emod32(int a, int b) { int m = b < 0 ? -b : b; int r = a % m;"
       " return r < 0 ? r + m : r; }\n"
       "__device__ __forceinline__ i64 mk_shl(i64 a, i64 k) { return k >= 62 ? 0 :"
       " (i64)((unsigned long long)a << k); }\n"
       "__device__ __forceinline__ i64 mk_shr(i64 a, i64 k) { return a >> (k > 63 ? 63 : k); }\n";
  const unsigned long long nthr = (unsigned long long)(block[0] * block[1] * block[2]);
  for (int pi = 0; pi < np; ++pi) {
    const mk_problem& p = set.probs[pi];
    const mk_access_prog& A = progs[pi];
    const AccGenInfo& I = info[pi];
    const int nv = p.nvars, n_outer = I.n_outer;
    const int* rb = I.rbits.empty() ? nullptr : I.rbits.data();
    auto ty = [&](int r) { return rb && rb[r] == 32 ? "int" : "i64"; };
    s << "__device__ __forceinline__ bool acc_" << pi
      << "(unsigned local, u64& k0, unsigned& idk, bool& mis, u64& done) {\n"
         "  unsigned r = local; (void)r;\n";
    for (int i = n_outer - 1; i >= 0; --i) {
      const unsigned long long sp = (unsigned long long)(I.hi[i] - I.lo[i] + 1);
      s << "  const " << ty(i) << " x" << i << " = (" << ty(i) << ")(" << lit(I.lo[i]) << " + (i64)(r % "
        << sp << "u)); r /= " << sp << "u;\n";
    }
    unsigned long long inner = 1;
    for (int i = n_outer; i < nv; ++i) inner *= (unsigned long long)(I.hi[i] - I.lo[i] + 1);
    s << "  for (unsigned long long j = 0; j < " << inner << "ULL; ++j) {\n";
    if (nv > n_outer) {
      s << "    unsigned long long jj = j;\n";
      for (int i = nv - 1; i >= n_outer; --i) {
        const unsigned long long sp = (unsigned long long)(I.hi[i] - I.lo[i] + 1);
        s << "    const " << ty(i) << " x" << i << " = (" << ty(i) << ")(" << lit(I.lo[i])
          << " + (i64)(jj % " << sp << "ull)); jj /= " << sp << "ull;\n";
      }
    }
    s << "    ++done;\n    bool hit = false;\n    i64 off = 0;\n    do {\n";
    emit_path(s, p, set.insns + p.insn_off, set.consts + p.const_off, rb);
    s << "      hit = true; off = (i64)v" << A.off_reg << ";\n    } while (0);\n";
    s << "    if (hit) {\n";
    for (int k = 0; k < 6; ++k) {
      s << "      const u64 id" << k << " = (u64)";
      if (A.id_var[k] >= 0) s << "(i64)x" << A.id_var[k];
      else s << lit(A.id_fixed[k]);
      s << ";\n";
    }
    s << "      const u64 blk = (id2 * " << grid[1] << "ull + id1) * " << grid[0] << "ull + id0;\n"
      << "      const u64 thr = (id5 * " << block[1] << "ull + id4) * " << block[0] << "ull + id3;\n"
      << "      idk = (unsigned)(" << (A.shared ? "thr" : "blk * " + std::to_string(nthr) + "ull + thr") << ");\n"
      << "      const i64 rel = off - (" << lit(A.off_lo) << ");\n"
      << "      if (rel < 0 || rel % " << A.granule << " != 0) mis = true;\n"
      << "      k0 = " << A.kbase << "ull + " << (A.shared ? "blk * " + std::to_string(A.span) + "ull" : "0ull")
      << " + (u64)(rel / " << A.granule << ");\n"
      << "      (void)blk; (void)thr;\n      return true;\n    }\n  }\n  return false;\n}\n";
  }
  // dispatch tree
  std::function<void(int, int, int)> tree = [&](int a, int b, int ind) {
    const std::string pad(ind, ' ');
    if (a == b) {
      const mk_access_prog& A = progs[a];
      const AccGenInfo& I = info[a];
      s << pad << "if ((mode == 1 && !" << A.write << ") || (mode == 2 && " << A.write << ")) continue;\n"
        << pad << "{ const unsigned l = (unsigned)(g - " << I.start << "ull);\n"
        << pad << "  hit = acc_" << a << "(l, k0, idk, mis, done); T = " << A.tuples << "; W = "
        << A.write << "; slot0 = " << I.slot << "ull + (u64)l * " << A.tuples << "ull; }\n";
      return;
    }
    const int m = (a + b) / 2;
    s << pad << "if (g < " << info[m + 1].start << "ull) {\n";
    tree(a, m, ind + 2);
    s << pad << "} else {\n";
    tree(m + 1, b, ind + 2);
    s << pad << "}\n";
  };
  s << "extern \"C\" __global__ void __launch_bounds__(256) mk_access_jit(int mode, u64* keys, u64* vals,"
       " unsigned* owner, u64* ctr) {\n"
       "  u64 done = 0, emitted = 0;\n  bool mis = false, race = false;\n"
       "  const u64 stride = (u64)gridDim.x * blockDim.x;\n"
       "  for (u64 g = (u64)blockIdx.x * blockDim.x + threadIdx.x; g < " << total << "ull; g += stride) {\n"
       "    u64 k0 = 0, slot0 = 0; unsigned idk = 0; bool hit = false; int T = 1, W = 0;\n";
  tree(0, np - 1, 4);
  s << "    if (!hit) {\n"
       "      if (mode == 0) for (int j = 0; j < T; ++j) { keys[slot0 + j] = ~0ull; vals[slot0 + j] = 0ull; }\n"
       "      continue;\n    }\n"
       "    if (mode == 0) {\n"
       "      for (int j = 0; j < T; ++j) { keys[slot0 + j] = ((k0 + (u64)j) << 1) | (W ? 0ull : 1ull);"
       " vals[slot0 + j] = ((u64)idk << 32) | (slot0 + (u64)j); }\n"
       "    } else if (!mis) {\n"
       "      for (int j = 0; j < T; ++j) {\n"
       "        unsigned* o = owner + (k0 + (u64)j);\n"
       "        if (mode == 1) { const unsigned old = atomicCAS(o, 0xffffffffu, idk);"
       " if (old != 0xffffffffu && old != idk) race = true; }\n"
       "        else { const unsigned w = *o; if (w != 0xffffffffu && w != idk) race = true; }\n"
       "      }\n    }\n"
       "    emitted += (u64)T;\n  }\n"
       "  for (int o = 16; o > 0; o >>= 1) { done += __shfl_down_sync(0xffffffffu, done, o);"
       " emitted += __shfl_down_sync(0xffffffffu, emitted, o); }\n"
       "  const bool am = __any_sync(0xffffffffu, mis), ar = __any_sync(0xffffffffu, race);\n"
       "  if ((threadIdx.x & 31) == 0) { if (done) atomicAdd(ctr + 0, done);"
       " if (emitted) atomicAdd(ctr + 1, emitted); if (am) atomicOr(ctr + 2, 1ull);"
       " if (ar) atomicOr(ctr + 6, 1ull); }\n}\n";
  return s.str();
}

struct Cache {
  std::map<std::string, cudaKernel_t> kernels;
  std::map<std::string, cudaLibrary_t> libs;
  std::string last_error;
};

// compile (or fetch) the kernel for `src`; nullptr on failure
inline cudaKernel_t get_kernel(Cache& cache, const std::string& src, int device,
                               const char* name = "mk_race_gen_jit") {
  const std::string ckey = std::string(name) + "\n" + src;
  auto it = cache.kernels.find(ckey);
  if (it != cache.kernels.end()) return it->second;
  auto lt = cache.libs.find(src);
  cudaLibrary_t lib = nullptr;
  if (lt != cache.libs.end()) lib = lt->second;
  if (!lib) {
    Nvrtc& N = nvrtc();
    if (!N.load()) {
      cache.last_error = "nvrtc unavailable";
      return nullptr;
    }
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    const std::string arch = "--gpu-architecture=sm_" + std::to_string(major * 10 + minor) +
                             (major >= 9 ? "a" : "");
    nvrtcProgram prog;
    if (N.create(&prog, src.c_str(), "mk_race_gen_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
      cache.last_error = "nvrtcCreateProgram failed";
      return nullptr;
    }
    const char* opts[] = {arch.c_str(), "--std=c++17", "-default-device"};
    nvrtcResult rc = N.compile(prog, 3, opts);
    if (rc != NVRTC_SUCCESS) {
      size_t n = 0;
      N.log_size(prog, &n);
      std::string log(n, '\0');
      if (n) N.log(prog, &log[0]);
      cache.last_error = "nvrtc: " + log;
      N.destroy(&prog);
      return nullptr;
    }
    size_t n = 0;
    N.cubin_size(prog, &n);
    std::string bin(n, '\0');
    N.cubin(prog, &bin[0]);
    N.destroy(&prog);
    if (cudaLibraryLoadData(&lib, bin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) !=
        cudaSuccess) {
      cache.last_error = "cudaLibraryLoadData failed";
      cudaGetLastError();
      return nullptr;
    }
    cache.libs[src] = lib;
  }
  cudaKernel_t k;
  if (cudaLibraryGetKernel(&k, lib, name) != cudaSuccess) {
    cache.last_error = "cudaLibraryGetKernel failed";
    cudaGetLastError();
    return nullptr;
  }
  cache.kernels[ckey] = k;
  return k;
}

}  // namespace mkjit

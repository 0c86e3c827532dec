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

#include <map>
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

// CUDA source of the race generator for one program (host copy of the
// problem).  Key type, sentinel, offset origin and block radix are baked in.
inline std::string race_gen_source(const mk_problem& p, const mk_insn* insns,
                                   const mk_i128* consts, int n_outer, int off_reg, int shared,
                                   const int id_var[6], const int64_t* lo, const int64_t* hi,
                                   bool key64) {
  const int nv = p.nvars, nc = p.nconst, nr = p.nregs;
  std::ostringstream s;
  const char* KT = key64 ? "unsigned long long" : "unsigned int";
  s << "typedef long long i64;\n"
       "__device__ __forceinline__ i64 mk_emod(i64 a, i64 b) { i64 m = b < 0 ? -b : b; i64 r = a % m;"
       " return r < 0 ? r + m : r; }\n"
       "__device__ __forceinline__ i64 mk_shl(i64 a, i64 k) { return k >= 62 ? 0 :"
       " (i64)((unsigned long long)a << k); }\n"
       "__device__ __forceinline__ i64 mk_shr(i64 a, i64 k) { return a >> (k > 63 ? 63 : k); }\n";
  s << "extern \"C\" __global__ void __launch_bounds__(256) mk_race_gen_jit(unsigned long long vol, "
    << KT << " sentinel, " << KT
    << "* keys, unsigned int* vals, unsigned long long* count, unsigned long long* evaluated,"
       " i64 off_lo, unsigned long long nblocks) {\n";
  for (int i = 0; i < nv; ++i) {
    s << "  const i64 lo" << i << " = " << lit(lo[i]) << ", sp" << i << " = " << lit(hi[i] - lo[i] + 1)
      << ";\n";
  }
  s << "  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;\n"
       "  unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;\n";
  // odometer digits of idx and of the stride over the leading vars
  for (int i = 0; i < n_outer; ++i) s << "  i64 d" << i << ", t" << i << ";\n";
  s << "  { unsigned long long a = idx, b = stride;\n";
  for (int i = n_outer - 1; i >= 0; --i) {
    s << "    d" << i << " = (i64)(a % (unsigned long long)sp" << i << "); a /= (unsigned long long)sp" << i
      << "; t" << i << " = (i64)(b % (unsigned long long)sp" << i << "); b /= (unsigned long long)sp"
      << i << ";\n";
  }
  s << "  }\n  unsigned long long done = 0, models = 0;\n"
       "  for (; idx < vol; idx += stride) {\n";
  for (int i = 0; i < n_outer; ++i) s << "    const i64 x" << i << " = lo" << i << " + d" << i << ";\n";
  s << "    " << KT << " key = sentinel;\n";
  // existential (trailing) vars: first model wins
  unsigned long long inner = 1;
  for (int i = n_outer; i < nv; ++i) inner *= (unsigned long long)(hi[i] - lo[i] + 1);
  s << "    for (unsigned long long j = 0; j < " << inner << "ULL; ++j) {\n";
  if (nv > n_outer) {
    s << "      unsigned long long jj = j;\n";
    for (int i = nv - 1; i >= n_outer; --i)
      s << "      const i64 x" << i << " = lo" << i << " + (i64)(jj % (unsigned long long)sp" << i
        << "); jj /= (unsigned long long)sp" << i << ";\n";
  }
  s << "      ++done;\n      bool hit = false;\n      i64 off = 0;\n      do {\n";
  for (int r = 0; r < nr; ++r) s << "        i64 v" << r << " = 0; bool e" << r << " = false;\n";
  for (int i = 0; i < nv; ++i) s << "        v" << i << " = x" << i << ";\n";
  for (int i = 0; i < nc; ++i) s << "        v" << (nv + i) << " = " << lit((int64_t)consts[i].lo) << ";\n";
  for (int k = 0; k < p.ninsn; ++k) {
    const mk_insn in = insns[k];
    const int a = in.a, b = in.b, c = in.c, d = in.dst;
    if (in.op == MK_OP_ATOM) {
      s << "        if (e" << a << " || !v" << a << ") break;\n";
      continue;
    }
    s << "        { const i64 A = v" << a << ", B = v" << b << "; const bool EA = e" << a << ", EB = e"
      << b << "; i64 R = 0; bool E = false; (void)A; (void)B; (void)EA; (void)EB;\n          ";
    switch (in.op) {
      case MK_OP_AND: s << "if (EA) E = true; else if (!A) R = 0; else { R = B ? 1 : 0; E = EB; }"; break;
      case MK_OP_OR: s << "if (EA) E = true; else if (A) R = 1; else { R = B ? 1 : 0; E = EB; }"; break;
      case MK_OP_NOT: s << "E = EA; R = A ? 0 : 1;"; break;
      case MK_OP_ITE:
        s << "const i64 C = v" << c << "; const bool EC = e" << c
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
          case MK_OP_EMOD: s << "if (B == 0) E = true; else R = mk_emod(A, B);"; break;
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
    s << "\n          v" << d << " = R; e" << d << " = E; }\n";
  }
  s << "        hit = true; off = v" << off_reg << ";\n      } while (0);\n";
  s << "      if (hit) {\n        unsigned long long bk = 0;\n";
  if (shared) {
    for (int ax = 2; ax >= 0; --ax) {
      const int v = id_var[ax];
      if (v < 0) continue;
      s << "        bk = bk * (unsigned long long)sp" << v << " + (unsigned long long)(x" << v << " - lo" << v
        << ");\n";
    }
  }
  s << "        key = (" << KT << ")((unsigned long long)(off - off_lo) * nblocks + bk);\n"
       "        ++models;\n        break;\n      }\n    }\n"
       "    keys[idx] = key;\n    vals[idx] = (unsigned int)idx;\n";
  // odometer step
  s << "    { i64 carry = 0, dd;\n";
  for (int i = n_outer - 1; i >= 0; --i) {
    s << "      dd = d" << i << " + t" << i << " + carry; carry = dd >= sp" << i << " ? 1 : 0; d" << i
      << " = dd - (carry ? sp" << i << " : 0);\n";
  }
  s << "    }\n  }\n"
       "  for (int o = 16; o > 0; o >>= 1) { done += __shfl_down_sync(0xffffffffu, done, o);"
       " models += __shfl_down_sync(0xffffffffu, models, o); }\n"
       "  if ((threadIdx.x & 31) == 0) { if (done) atomicAdd(evaluated, done);"
       " if (models) atomicAdd(count, models); }\n}\n";
  return s.str();
}

struct Cache {
  std::map<std::string, cudaKernel_t> kernels;
  std::string last_error;
};

// compile (or fetch) the kernel for `src`; nullptr on failure
inline cudaKernel_t get_kernel(Cache& cache, const std::string& src, int device) {
  auto it = cache.kernels.find(src);
  if (it != cache.kernels.end()) return it->second;
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
  cudaLibrary_t lib;
  if (cudaLibraryLoadData(&lib, bin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) !=
      cudaSuccess) {
    cache.last_error = "cudaLibraryLoadData failed";
    cudaGetLastError();
    return nullptr;
  }
  cudaKernel_t k;
  if (cudaLibraryGetKernel(&k, lib, "mk_race_gen_jit") != cudaSuccess) {
    cache.last_error = "cudaLibraryGetKernel failed";
    cudaGetLastError();
    return nullptr;
  }
  cache.kernels[src] = k;
  return k;
}

}  // namespace mkjit

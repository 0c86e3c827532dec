// mk_access.cuh -- K2, oracle semantics: read-write and write-write races
// across instructions over one concrete launch (include/mk_b200.h
// mk_access_sweep).  Included at the end of mk_engine.cu.
//
// Rule (the reference specification's concrete oracle,
// which the reference does not ship): two accesses race when they touch the
// same region at overlapping bytes, come from different threads, at least
// one is a write, and -- for shared memory -- they share the barrier epoch
// (and the block).  Data-parallel form:
//
//   k_acc_gen   one thread per (access, instance): decode the instance,
//               evaluate the access's path bytecode (exact int64), emit one
//               (key, val) tuple per granule the access covers, or sentinels
//               when the path fails;
//   compact     order-preserving compaction of the executed tuples
//               (mksort::compact, mk_sort.cuh);
//   sort        radix sort of the 64-bit keys (value = identity | slot),
//               mksort::sort_pairs (hand-written onesweep, mk_sort.cuh);
//   k_acc_scan  segments of equal granule: a segment races iff its head is a
//               write (writes sort first) and some element has another
//               identity; the head thread walks its segment and stops at the
//               first such element.  First race = the least key.

namespace {

struct AccDev {
  int prob;
  int n_outer;
  int off_reg;
  int write;
  int shared;
  int granule;
  int tuples;
  int id_var[6];
  long long id_fixed[6];
  unsigned long long inner;
  unsigned long long vol;
  unsigned long long start;   // first global instance
  unsigned long long slot;    // first dense tuple slot
  unsigned long long kbase;
  unsigned long long span;
  long long off_lo;
};

struct AccLaunch {
  long long grid[3];
  long long block[3];
};

constexpr int ACC_THREADS = 256;

// MODE 0: dense (key, val) tuples for the sort path.  MODE 1 / 2: the
// owner-table fast path -- writes claim their granules (atomicCAS of the
// writer's identity; a second writer identity is a race), then reads check
// them (a granule owned by another identity is a race).  No tuple reaches
// HBM; a launch without races is decided exactly, one with races goes to the
// sort path for the canonical first pair and the racy-granule count.
constexpr unsigned ACC_EMPTY = 0xffffffffu;

template <int MODE>
__global__ void __launch_bounds__(ACC_THREADS) k_acc_gen(
    const AccDev* __restrict__ progs, int nprog, unsigned long long total, AccLaunch L,
    const mk_problem* probs, const mk_insn* insns, const mk_i128* consts, const int32_t* ar,
    const uint64_t* am, const mk_row* rows, const mk_row_term* terms, const mk_i128* vlo,
    const mk_i128* vhi, unsigned long long* keys, unsigned long long* vals,
    unsigned* owner, unsigned long long* ctr) {
  extern __shared__ int64_t sh[];
  int64_t lo[SMALL_V], hi[SMALL_V], x[SMALL_V];
  unsigned long long done = 0, emitted = 0;
  bool misaligned = false, race = false;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long g = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += stride) {
    // the access owning global instance g (starts are ascending)
    int a = 0, b = nprog - 1;
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (progs[m].start <= g) a = m; else b = m - 1;
    }
    const AccDev& A = progs[a];
    if (MODE == 1 && !A.write) continue;
    if (MODE == 2 && A.write) continue;
    const unsigned long long local = g - A.start;
    const MkProb P = mk_prob_view(probs, A.prob, insns, consts, ar, am, rows, terms);
    const int nv = P.p->nvars;
    for (int i = 0; i < nv; ++i) {
      lo[i] = (int64_t)vlo[P.p->var_off + i].lo;
      hi[i] = (int64_t)vhi[P.p->var_off + i].lo;
    }
    {
      // instance boxes hold < 2^31 instances: 32-bit mixed-radix decode
      unsigned r = (unsigned)local;
      for (int i = A.n_outer - 1; i >= 0; --i) {
        const unsigned sp = (unsigned)(hi[i] - lo[i] + 1);
        x[i] = lo[i] + (int64_t)(r % sp);
        r /= sp;
      }
    }
    bool hit = false;
    int64_t off = 0;
    for (unsigned long long j = 0; j < A.inner && !hit; ++j) {
      unsigned long long jj = j;
      for (int i = nv - 1; i >= A.n_outer; --i) {
        const unsigned long long s = (unsigned long long)(hi[i] - lo[i] + 1);
        x[i] = lo[i] + (int64_t)(jj % s);
        jj /= s;
      }
      ++done;
      if (sh_eval_point(P, x, sh)) {
        hit = true;
        off = sh[A.off_reg * blockDim.x + threadIdx.x];
      }
    }
    const unsigned long long slot0 = A.slot + local * (unsigned long long)A.tuples;
    if (!hit) {
      if (MODE) continue;
      for (int j = 0; j < A.tuples; ++j) {
        keys[slot0 + j] = ~0ull;
        vals[slot0 + j] = 0ull;
      }
      continue;
    }
    long long id[6];
    for (int k = 0; k < 6; ++k) id[k] = A.id_var[k] >= 0 ? (long long)x[A.id_var[k]] : A.id_fixed[k];
    const unsigned long long blk =
        ((unsigned long long)id[2] * L.grid[1] + id[1]) * L.grid[0] + id[0];
    const unsigned long long thr =
        ((unsigned long long)id[5] * L.block[1] + id[4]) * L.block[0] + id[3];
    const unsigned long long nthr = (unsigned long long)(L.block[0] * L.block[1] * L.block[2]);
    const unsigned long long idk = A.shared ? thr : blk * nthr + thr;
    const long long rel = (long long)off - A.off_lo;
    if (rel < 0 || rel % A.granule) misaligned = true;
    const unsigned long long k0 =
        A.kbase + (A.shared ? blk * A.span : 0ull) + (unsigned long long)(rel / A.granule);
    if (MODE == 0) {
      for (int j = 0; j < A.tuples; ++j) {
        keys[slot0 + j] = ((k0 + (unsigned long long)j) << 1) | (A.write ? 0ull : 1ull);
        vals[slot0 + j] = (idk << 32) | (slot0 + (unsigned long long)j);
      }
    } else if (!misaligned) {
      for (int j = 0; j < A.tuples; ++j) {
        unsigned* o = owner + (k0 + (unsigned long long)j);
        if (MODE == 1) {
          const unsigned old = atomicCAS(o, ACC_EMPTY, (unsigned)idk);
          if (old != ACC_EMPTY && old != (unsigned)idk) race = true;
        } else {
          const unsigned w = *o;
          if (w != ACC_EMPTY && w != (unsigned)idk) race = true;
        }
      }
    }
    emitted += (unsigned long long)A.tuples;
  }
  for (int o = 16; o > 0; o >>= 1) {
    done += __shfl_down_sync(FULL, done, o);
    emitted += __shfl_down_sync(FULL, emitted, o);
  }
  const bool mis = __any_sync(FULL, misaligned);
  const bool rc = __any_sync(FULL, race);
  if ((threadIdx.x & 31) == 0) {
    if (done) atomicAdd(ctr + 0, done);
    if (emitted) atomicAdd(ctr + 1, emitted);
    if (mis) atomicOr(ctr + 2, 1ull);
    if (rc) atomicOr(ctr + 6, 1ull);
  }
}

// segment scan over n sorted tuples (n read on the device).  ctr[3] racy
// granules, ctr[4] min (head position << 32 | partner distance).
__global__ void __launch_bounds__(ACC_THREADS) k_acc_scan(const unsigned long long* keys,
                                                          const unsigned long long* vals,
                                                          const unsigned long long* count,
                                                          unsigned long long* ctr) {
  const unsigned long long n = *count;
  unsigned long long racy = 0, first = ~0ull;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[i];
    if (i > 0 && (keys[i - 1] >> 1) == (k >> 1)) continue;   // not a segment head
    if (k & 1ull) continue;                                   // no write in this granule
    const unsigned long long id = vals[i] >> 32;
    for (unsigned long long j = i + 1; j < n && (keys[j] >> 1) == (k >> 1); ++j) {
      if ((vals[j] >> 32) != id) {
        ++racy;
        const unsigned long long c = (i << 32) | (j - i);
        if (c < first) first = c;
        break;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    racy += __shfl_down_sync(FULL, racy, o);
    const unsigned long long f = __shfl_down_sync(FULL, first, o);
    if (f < first) first = f;
  }
  if ((threadIdx.x & 31) == 0) {
    if (racy) atomicAdd(ctr + 3, racy);
    if (first != ~0ull) atomicMin(ctr + 4, first);
  }
}


}  // namespace

extern "C" int mk_access_sweep(mk_ctx* ctx, const mk_access_input* in, mk_access_result* out) {
  if (!ctx || !in || !out) return fail(ctx, MK_EINVAL, "null argument");
  std::memset(out, 0, sizeof(*out));
  CK(cudaSetDevice(ctx->device));
  const mk_problem_set& set = in->set;
  const int np = set.nprob;
  if (np < 1) return MK_OK;
  if (np > (1 << 20)) return fail(ctx, MK_EINVAL, "too many accesses");
  // per-access device descriptors: instance and slot prefix sums
  std::vector<AccDev> dev(np);
  unsigned long long total = 0, slots = 0;
  int maxr = 1;
  for (int i = 0; i < np; ++i) {
    const mk_problem& p = set.probs[i];
    const mk_access_prog& a = in->progs[i];
    if (!(p.flags & MK_PF_NARROW)) return fail(ctx, MK_EINVAL, "access sweep needs narrow problems");
    if (p.nvars > SMALL_V || p.nregs > SMALL_R)
      return fail(ctx, MK_EINVAL, "access program exceeds the small-problem limits");
    if (a.off_reg < 0 || a.off_reg >= p.nregs) return fail(ctx, MK_EINVAL, "bad off_reg");
    if (a.granule < 1 || a.tuples < 1 || a.tuples > 64) return fail(ctx, MK_EINVAL, "bad granule");
    const int n_outer = p.nvars - a.n_exist;
    if (a.n_exist < 0 || n_outer < 0) return fail(ctx, MK_EINVAL, "bad n_exist");
    AccDev& d = dev[i];
    d.prob = i;
    d.n_outer = n_outer;
    d.off_reg = a.off_reg;
    d.write = a.write ? 1 : 0;
    d.shared = a.shared ? 1 : 0;
    d.granule = a.granule;
    d.tuples = a.tuples;
    for (int k = 0; k < 6; ++k) {
      d.id_var[k] = a.id_var[k];
      d.id_fixed[k] = a.id_fixed[k];
      if (a.id_var[k] >= n_outer) return fail(ctx, MK_EINVAL, "identity var must be a leading var");
    }
    long double vf = 1.0L, inf_ = 1.0L;
    unsigned long long vol = 1, inner = 1;
    for (int v = 0; v < p.nvars; ++v) {
      const int64_t l = (int64_t)set.var_lo[p.var_off + v].lo, h = (int64_t)set.var_hi[p.var_off + v].lo;
      const unsigned long long w = (unsigned long long)(h - l + 1);
      if (v < n_outer) {
        vf *= (long double)w;
        vol *= w;
      } else {
        inf_ *= (long double)w;
        inner *= w;
      }
    }
    if (vf * (long double)a.tuples > 2147483647.0L || inf_ > 65536.0L)
      return fail(ctx, MK_EINVAL, "access instance box too large");
    d.vol = vol;
    d.inner = inner;
    d.start = total;
    d.slot = slots;
    d.kbase = a.kbase;
    d.span = a.span;
    d.off_lo = a.off_lo;
    total += vol;
    slots += vol * (unsigned long long)a.tuples;
    if (p.nregs > maxr) maxr = p.nregs;
  }
  if (slots > 2147483647ull) return fail(ctx, MK_EINVAL, "access sweep exceeds 2^31 tuples");
  int rc = upload_set(ctx, &set, &ctx->scratch, false);
  if (rc) return rc;
  mk_dset* ds = &ctx->scratch;
  char* base = static_cast<char*>(ds->d);
  cudaStream_t s = ctx->stream;
  const int n = (int)slots;
  const size_t sort_ws = mksort::workspace_bytes(slots);
  size_t off = 0;
  auto place = [&](size_t bytes) {
    size_t o = off;
    off = (off + bytes + 255) / 256 * 256;
    return o;
  };
  const size_t o_dev = place(sizeof(AccDev) * np);
  const size_t o_ctr = place(sizeof(unsigned long long) * 8);
  const size_t o_k0 = place(8ull * slots + 8), o_k1 = place(8ull * slots + 8);
  const size_t o_v0 = place(8ull * slots + 8), o_v1 = place(8ull * slots + 8);
  const size_t o_ws = place(sort_ws);
  rc = ensure(ctx, &ctx->d_work, &ctx->d_work_bytes, off);
  if (rc) return rc;
  char* wb = static_cast<char*>(ctx->d_work);
  AccDev* d_dev = reinterpret_cast<AccDev*>(wb + o_dev);
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(wb + o_ctr);
  unsigned long long* k0 = reinterpret_cast<unsigned long long*>(wb + o_k0);
  unsigned long long* k1 = reinterpret_cast<unsigned long long*>(wb + o_k1);
  unsigned long long* v0 = reinterpret_cast<unsigned long long*>(wb + o_v0);
  unsigned long long* v1 = reinterpret_cast<unsigned long long*>(wb + o_v1);
  CK(cudaMemcpyAsync(d_dev, dev.data(), sizeof(AccDev) * np, cudaMemcpyHostToDevice, s));
  // [0] evaluations [1] tuples [2] misaligned [3] racy [4] first [5] count
  unsigned long long init[8] = {0ull, 0ull, 0ull, 0ull, ~0ull, 0ull, 0ull, 0ull};
  CK(cudaMemcpyAsync(ctr, init, sizeof(init), cudaMemcpyHostToDevice, s));
  AccLaunch L;
  for (int k = 0; k < 3; ++k) {
    L.grid[k] = in->grid[k] > 0 ? in->grid[k] : 1;
    L.block[k] = in->block[k] > 0 ? in->block[k] : 1;
  }
  const size_t shm = sizeof(int64_t) * (size_t)maxr * ACC_THREADS;
  if (shm > 48 * 1024) {
    CK(cudaFuncSetAttribute(k_acc_gen<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    CK(cudaFuncSetAttribute(k_acc_gen<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    CK(cudaFuncSetAttribute(k_acc_gen<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
  }
  const int grid = ctx->sms * 8;
  const mk_problem* d_probs = reinterpret_cast<const mk_problem*>(base + ds->o_probs);
  const mk_insn* d_insn = reinterpret_cast<const mk_insn*>(base + ds->o_insn);
  const mk_i128* d_const = reinterpret_cast<const mk_i128*>(base + ds->o_const);
  const int32_t* d_ar = reinterpret_cast<const int32_t*>(base + ds->o_ar);
  const uint64_t* d_am = reinterpret_cast<const uint64_t*>(base + ds->o_am);
  const mk_row* d_rows = reinterpret_cast<const mk_row*>(base + ds->o_rows);
  const mk_row_term* d_terms = reinterpret_cast<const mk_row_term*>(base + ds->o_terms);
  const mk_i128* d_vlo = reinterpret_cast<const mk_i128*>(base + ds->o_vlo);
  const mk_i128* d_vhi = reinterpret_cast<const mk_i128*>(base + ds->o_vhi);
  unsigned long long h[8];
  // specialised generator (NVRTC): straight-line access functions with
  // int32-typed registers; the interpreted k_acc_gen<MODE> otherwise
  cudaKernel_t jk = nullptr;
  if (!getenv("MK_NO_JIT") && total) {
    std::vector<mkjit::AccGenInfo> info(np);
    for (int i = 0; i < np; ++i) {
      const mk_problem& p = set.probs[i];
      mkjit::AccGenInfo& I = info[i];
      I.n_outer = dev[i].n_outer;
      I.start = dev[i].start;
      I.slot = dev[i].slot;
      I.vol = dev[i].vol;
      I.lo.resize(p.nvars);
      I.hi.resize(p.nvars);
      for (int v = 0; v < p.nvars; ++v) {
        I.lo[v] = (int64_t)set.var_lo[p.var_off + v].lo;
        I.hi[v] = (int64_t)set.var_hi[p.var_off + v].lo;
      }
      if (!getenv("MK_JIT_WIDE")) I.rbits = register_bits(set, i, I.lo.data(), I.hi.data());
    }
    const std::string src = mkjit::access_gen_source(set, in->progs, info, L.grid, L.block, total);
    if (const char* dump = getenv("MK_JIT_DUMP_ACCESS")) {
      FILE* f = fopen(dump, "w");
      if (f) {
        fputs(src.c_str(), f);
        fclose(f);
      }
    }
    jk = mkjit::get_kernel(ctx->jit, src, ctx->device, "mk_access_jit");
  }
  out->jit = jk != nullptr;
  auto gen = [&](int mode, unsigned long long* keys, unsigned long long* vals,
                 unsigned* owner) -> cudaError_t {
    if (jk) {
      int a_mode = mode;
      unsigned long long* a_keys = keys;
      unsigned long long* a_vals = vals;
      unsigned* a_owner = owner;
      unsigned long long* a_ctr = ctr;
      void* args[] = {&a_mode, &a_keys, &a_vals, &a_owner, &a_ctr};
      return cudaLaunchKernel((const void*)jk, dim3(grid), dim3(ACC_THREADS), args, 0, s);
    }
    if (mode == 0)
      k_acc_gen<0><<<grid, ACC_THREADS, shm, s>>>(d_dev, np, total, L, d_probs, d_insn, d_const, d_ar,
                                                  d_am, d_rows, d_terms, d_vlo, d_vhi, keys, vals,
                                                  owner, ctr);
    else if (mode == 1)
      k_acc_gen<1><<<grid, ACC_THREADS, shm, s>>>(d_dev, np, total, L, d_probs, d_insn, d_const, d_ar,
                                                  d_am, d_rows, d_terms, d_vlo, d_vhi, keys, vals,
                                                  owner, ctr);
    else
      k_acc_gen<2><<<grid, ACC_THREADS, shm, s>>>(d_dev, np, total, L, d_probs, d_insn, d_const, d_ar,
                                                  d_am, d_rows, d_terms, d_vlo, d_vhi, keys, vals,
                                                  owner, ctr);
    return cudaGetLastError();
  };
  // fast path: the owner table (one u32 per granule key) when it fits
  if (total && in->nkeys > 0 && in->nkeys <= (1ull << 30) && !getenv("MK_ACCESS_NO_FAST")) {
    void* otab = nullptr;
    CK(cudaMallocAsync(&otab, sizeof(unsigned) * in->nkeys, s));
    unsigned* owner = static_cast<unsigned*>(otab);
    CK(cudaMemsetAsync(owner, 0xff, sizeof(unsigned) * in->nkeys, s));
    CK(cudaEventRecord(ctx->ev[0], s));
    CK(gen(1, nullptr, nullptr, owner));
    CK(gen(2, nullptr, nullptr, owner));
    CK(cudaEventRecord(ctx->ev[1], s));
    CK(cudaFreeAsync(otab, s));
    CK(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h[2] || !h[6]) {
      // misaligned (host reruns at granule 1) or race-free: decided
      out->instances = h[0];
      out->tuples = h[1];
      out->misaligned = h[2] ? 1 : 0;
      out->fast = 1;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
      out->gen_ms = ms;
      return MK_OK;
    }
    CK(cudaMemcpyAsync(ctr, init, sizeof(init), cudaMemcpyHostToDevice, s));
  }
  CK(cudaEventRecord(ctx->ev[0], s));
  if (total) CK(gen(0, k0, v0, nullptr));
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev[1], s));
  CK(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  out->instances = h[0];
  out->tuples = h[1];
  out->misaligned = h[2] ? 1 : 0;
  if (out->misaligned || h[1] < 2) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
    out->gen_ms = ms;
    return MK_OK;
  }
  // compaction (executed tuples only, order preserved), sort, segment scan
  unsigned long long* kc = k0;
  unsigned long long* ko = k1;
  unsigned long long* vc = v0;
  unsigned long long* vo = v1;
  if (h[1] != slots) {
    CK((mksort::compact<unsigned long long, unsigned long long>(k0, v0, k1, v1, slots, ~0ull,
                                                               wb + o_ws, ctr + 5, s)));
    kc = k1;
    ko = k0;
    vc = v1;
    vo = v0;
  } else {
    CK(cudaMemcpyAsync(ctr + 5, &slots, sizeof(slots), cudaMemcpyHostToDevice, s));
  }
  // key bits in use (host bound: every key < 2^key_bits)
  int bits = in->key_bits;
  if (bits < 1 || bits > 64) bits = 64;
  const unsigned long long m = h[1];
  unsigned long long* ks = kc;
  unsigned long long* vs = vc;
  {
    mksort::SortInfo si{};
    CK((mksort::sort_pairs<unsigned long long, unsigned long long>(kc, vc, ko, vo, m, bits,
                                                                  wb + o_ws, ctx->sms, s, &ks,
                                                                  &vs, &si)));
    out->sort_passes = si.passes_run;
  }
  CK(cudaEventRecord(ctx->ev[2], s));
  k_acc_scan<<<grid, ACC_THREADS, 0, s>>>(ks, vs, ctr + 5, ctr);
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev[3], s));
  CK(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  out->racy = h[3];
  out->has_race = h[3] > 0;
  if (out->has_race) {
    const unsigned long long i = h[4] >> 32, j = i + (h[4] & 0xffffffffull);
    unsigned long long va = 0, vb2 = 0;
    CK(cudaMemcpy(&va, vs + i, sizeof(va), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&vb2, vs + j, sizeof(vb2), cudaMemcpyDeviceToHost));
    out->slot_a = va & 0xffffffffull;
    out->slot_b = vb2 & 0xffffffffull;
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
  out->gen_ms = ms;
  cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]);
  out->sort_ms = ms;
  cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
  out->scan_ms = ms;
  return MK_OK;
}

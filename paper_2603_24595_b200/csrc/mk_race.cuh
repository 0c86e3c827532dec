// mk_race.cuh -- K2: sort-based race sweep over one concrete launch
// (include/mk_b200.h mk_race_sweep).  Included at the end of mk_engine.cu.
//
// Reference semantics (engine/detectors.py:204-273): a DataRace on a store is
// a pair of instances of the store's path, one per thread, with equal
// mathematical byte offsets and distinct thread identities (global memory),
// or the same block and distinct thread ids (shared memory).  With the
// launch fixed, the sweep is the data-parallel form of that definition:
//
//   k_race_root  interval evaluation of the root box: byte-offset range, so
//                the (offset, block) sort key is packed into as few bits as
//                possible;
//   k_race_gen   every instance index of the thread-private box: decode in
//                lexicographic order, evaluate the path bytecode in exact
//                int64, write (key, instance index) to the instance's slot
//                (a sentinel key when the path fails);
//   mksort::sort_pairs (mk_sort.cuh, hand-written onesweep LSD radix sort)
//                over the key bits in HBM;
//   k_race_scan  adjacent tuples with equal key and distinct identity are a
//                conflict (every race has at least one adjacent witness
//                pair after the sort); warp-aggregated count + atomicMin of
//                the first conflicting position.

#include "mk_sort.cuh"

namespace {

constexpr int RACE_THREADS = 256;

struct RaceDev {
  MkProb P;
  const mk_problem* prob;
  const int64_t* lo;   // root box (int64, narrow)
  const int64_t* hi;
  int off_reg;
  int shared;
  int id_var[6];
  int64_t off_lo;
  unsigned long long nblocks;  // block-key radix (1 for global memory)
  int n_outer;                 // leading vars enumerated as instances
  unsigned long long inner;    // volume of the trailing existential vars
};

__device__ __forceinline__ unsigned long long race_block_key(const RaceDev& R, const int64_t* x) {
  unsigned long long k = 0;
  for (int a = 2; a >= 0; --a) {
    const int v = R.id_var[a];
    if (v < 0) continue;
    const unsigned long long span = (unsigned long long)(R.hi[v] - R.lo[v] + 1);
    k = k * span + (unsigned long long)(x[v] - R.lo[v]);
  }
  return k;
}

__global__ void k_race_root(RaceDev R, int64_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  MkIvT<int64_t> Rg[MK_MAXR];
  int64_t cnt = 0;
  mk_eval_box(R.P, R.lo, R.hi, Rg, &cnt);
  out[0] = Rg[R.off_reg].lo;
  out[1] = Rg[R.off_reg].hi;
}

// dense generation: slot idx holds instance idx's key, or the all-ones
// sentinel (sorted past every real key) when the instance is not an access.
// Positions are the instance order, so the stable radix sort leaves equal
// keys in instance order: conflicts and the first conflicting pair are
// deterministic.  Each thread walks a grid-stride sequence of instances with
// a mixed-radix odometer (one addition per symbol instead of 64-bit
// divisions per decode).
template <typename K>
__global__ void __launch_bounds__(RACE_THREADS) k_race_gen(RaceDev R, unsigned long long vol,
                                                           K sentinel, K* keys, uint32_t* vals,
                                                           unsigned long long* count,
                                                           unsigned long long* evaluated) {
  extern __shared__ int64_t sh[];
  const int nv = R.prob->nvars;
  const int nl = R.n_outer;
  int64_t span[SMALL_V], dig[SMALL_V], sdig[SMALL_V], x[SMALL_V];
  for (int i = 0; i < nv; ++i) span[i] = R.hi[i] - R.lo[i] + 1;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  {
    unsigned long long a = idx, b = stride;
    for (int i = nl - 1; i >= 0; --i) {
      dig[i] = (int64_t)(a % (unsigned long long)span[i]);
      a /= (unsigned long long)span[i];
      sdig[i] = (int64_t)(b % (unsigned long long)span[i]);
      b /= (unsigned long long)span[i];
    }
  }
  unsigned long long done = 0, models = 0;
  for (; idx < vol; idx += stride) {
    for (int i = 0; i < nl; ++i) x[i] = R.lo[i] + dig[i];
    // one access per instance of the leading vars: the first model over the
    // trailing existential vars (inner == 1 when there are none)
    K key = sentinel;
    for (unsigned long long j = 0; j < R.inner; ++j) {
      unsigned long long jj = j;
      for (int i = nv - 1; i >= nl; --i) {
        x[i] = R.lo[i] + (int64_t)(jj % (unsigned long long)span[i]);
        jj /= (unsigned long long)span[i];
      }
      ++done;
      if (sh_eval_point(R.P, x, sh)) {
        const unsigned long long ok =
            (unsigned long long)(sh[R.off_reg * blockDim.x + threadIdx.x] - R.off_lo);
        key = (K)(ok * R.nblocks + (R.shared ? race_block_key(R, x) : 0ull));
        ++models;
        break;
      }
    }
    keys[idx] = key;
    vals[idx] = (uint32_t)idx;
    // odometer: dig += sdig (mixed radix); overflow of the top digit means
    // idx >= vol, which the loop test catches
    int64_t carry = 0;
    for (int i = nl - 1; i >= 0; --i) {
      int64_t d = dig[i] + sdig[i] + carry;
      carry = d >= span[i] ? 1 : 0;
      dig[i] = d - (carry ? span[i] : 0);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    done += __shfl_down_sync(FULL, done, o);
    models += __shfl_down_sync(FULL, models, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (done) atomicAdd(evaluated, done);
    if (models) atomicAdd(count, models);
  }
}

// Adjacent-conflict scan over n tuples (n read on the device).  When
// `unsorted` is given the scan also reports whether the keys are out of order
// (the sweep then sorts and scans again: results of an unsorted pass are
// discarded).
template <typename K>
__global__ void __launch_bounds__(RACE_THREADS) k_race_scan(RaceDev R, const K* keys,
                                                            const uint32_t* vals,
                                                            const unsigned long long* count,
                                                            unsigned long long* conflicts,
                                                            unsigned long long* first,
                                                            unsigned long long* unsorted) {
  const unsigned long long n = *count;
  int64_t xa[SMALL_V], xb[SMALL_V];
  unsigned long long mine = 0, my_first = ~0ull;
  bool down = false;
  // warp-contiguous chunks of 8 x 32 tuples: eight independent key loads in
  // flight per lane; each tuple's predecessor comes by shuffle
  constexpr int J = 8;
  const unsigned lane = threadIdx.x & 31;
  const unsigned long long nchunks = (n + 32 * J - 1) / (32 * J);
  const unsigned long long wstride = (unsigned long long)gridDim.x * (blockDim.x / 32);
  for (unsigned long long c = (unsigned long long)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
       c < nchunks; c += wstride) {
    const unsigned long long base = c * 32 * J;
    K kk[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const unsigned long long i = base + j * 32 + lane;
      kk[j] = i < n ? keys[i] : (K)0;
    }
    K carry = (lane == 0 && base > 0) ? keys[base - 1] : (K)0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const unsigned long long i = base + j * 32 + lane;
      K prev = __shfl_up_sync(FULL, kk[j], 1);
      const K last = __shfl_sync(FULL, kk[j], 31);
      if (lane == 0) prev = carry;
      carry = last;
      if (i == 0 || i >= n) continue;
      const K a = prev, b = kk[j];
      if (b < a) down = true;
      if (a != b) continue;
      // identities are leading vars: decode the instance of the leading box
      mk_decode(R.lo, R.hi, R.n_outer, R.prob->maxmask, (unsigned long long)vals[i - 1], xa);
      mk_decode(R.lo, R.hi, R.n_outer, R.prob->maxmask, (unsigned long long)vals[i], xb);
      bool same = true;
      // shared: the key already holds the block, compare thread ids only
      for (int a = R.shared ? 3 : 0; a < 6; ++a) {
        const int v = R.id_var[a];
        if (v >= 0 && xa[v] != xb[v]) same = false;
      }
      if (!same) {
        ++mine;
        if (i < my_first) my_first = i;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    mine += __shfl_down_sync(FULL, mine, o);
    unsigned long long f = __shfl_down_sync(FULL, my_first, o);
    if (f < my_first) my_first = f;
  }
  if ((threadIdx.x & 31) == 0) {
    if (mine) atomicAdd(conflicts, mine);
    if (my_first != ~0ull) atomicMin(first, my_first);
  }
  if (unsorted && __any_sync(FULL, down) && (threadIdx.x & 31) == 0) atomicOr(unsorted, 1ull);
}

// Chunk boundaries of the fused ordered pass (mk_jit.cuh mk_race_fused_jit):
// every warp left its first and last access in instance order; one CTA
// pairs each non-empty chunk's first access with the previous non-empty
// chunk's last one (exclusive max-scan of "last non-empty chunk"), adds the
// boundary conflicts and out-of-order flag, then resolves the key of the
// globally first conflict.  ctr: [1] conflicts [2] min (idx_b << 32 | idx_a)
// [4] out-of-order flag [5] key of the first conflict.
constexpr int MK_RACE_REC = 10;

// exclusive max-scan over a 1024-thread block (identity -1): warp shuffles,
// then the 32 warp maxima
__device__ __forceinline__ int block_excl_max_1024(int x) {
  __shared__ int wmax[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o && a > incl) incl = a;
  }
  if (lane == 31) wmax[warp] = incl;
  __syncthreads();
  int before = -1;
  for (int w = 0; w < warp; ++w)
    if (wmax[w] > before) before = wmax[w];
  int excl = __shfl_up_sync(0xffffffffu, incl, 1);
  if (lane == 0) excl = -1;
  const int out = excl > before ? excl : before;
  __syncthreads();
  return out;
}

__global__ void __launch_bounds__(1024) k_race_bound(const unsigned long long* rec, int W,
                                                     unsigned long long* ctr) {
  const int per = (W + 1023) / 1024;
  const int b = threadIdx.x * per;
  const int e = min(W, b + per);
  int last = -1;
  for (int w = b; w < e; ++w)
    if (rec[(size_t)w * MK_RACE_REC]) last = w;
  int prev = block_excl_max_1024(last);
  const int prev0 = prev;
  // the range's first and last access (shard combination across GPUs)
  __shared__ int s_first, s_last;
  if (threadIdx.x == 0) {
    s_first = 0x7fffffff;
    s_last = -1;
  }
  __syncthreads();
  if (last >= 0) {
    atomicMax(&s_last, last);
    for (int w = b; w < e; ++w)
      if (rec[(size_t)w * MK_RACE_REC]) {
        atomicMin(&s_first, w);
        break;
      }
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_last >= 0) {
    const unsigned long long* f = rec + (size_t)s_first * MK_RACE_REC;
    const unsigned long long* l = rec + (size_t)s_last * MK_RACE_REC;
    ctr[6] = f[1];
    ctr[7] = f[2];
    ctr[8] = f[3];
    ctr[9] = l[4];
    ctr[10] = l[5];
    ctr[11] = l[6];
    ctr[12] = 1;
  }
  unsigned long long conf = 0, best = ~0ull;
  bool down = false;
  for (int w = b; w < e; ++w) {
    const unsigned long long* r = rec + (size_t)w * MK_RACE_REC;
    if (!r[0]) continue;
    if (prev >= 0) {
      const unsigned long long* q = rec + (size_t)prev * MK_RACE_REC;
      if (r[1] < q[4]) {
        down = true;
      } else if (r[1] == q[4] && r[2] != q[5]) {
        ++conf;
        const unsigned long long c = (r[3] << 32) | q[6];
        if (c < best) best = c;
      }
    }
    prev = w;
  }
  if (conf) atomicAdd(ctr + 1, conf);
  if (best != ~0ull) atomicMin(ctr + 2, best);
  if (down) atomicOr(ctr + 4, 1ull);
  __threadfence();
  __syncthreads();
  const unsigned long long g = *(volatile unsigned long long*)(ctr + 2);
  if (g == ~0ull) return;
  prev = prev0;
  for (int w = b; w < e; ++w) {
    const unsigned long long* r = rec + (size_t)w * MK_RACE_REC;
    if (!r[0]) continue;
    if (r[7] == g) ctr[5] = r[8];
    if (prev >= 0) {
      const unsigned long long* q = rec + (size_t)prev * MK_RACE_REC;
      if (r[1] == q[4] && r[2] != q[5] && ((r[3] << 32) | q[6]) == g) ctr[5] = r[1];
    }
    prev = w;
  }
}

}  // namespace


// Register widths of problem `pid` for the specialised generators: interval
// evaluation of its instance box on the host (the device's own interval
// semantics, mk_core.cuh); a register whose range stays inside int32 is 32.
static std::vector<int> register_bits(const mk_problem_set& set, int pid, const int64_t* lo,
                                      const int64_t* hi) {
  const mk_problem& hp = set.probs[pid];
  std::vector<int> rbits(hp.nregs, 64);
  const MkProb HP = mk_prob_view(set.probs, pid, set.insns, set.consts, set.atom_regs,
                                 set.atom_masks, set.rows, set.row_terms);
  std::vector<MkIvT<i128>> Rg(MK_MAXR);
  for (auto& r : Rg) {
    r.lo = 1;
    r.hi = 0;
    r.fl = 0;
  }
  std::vector<i128> vl(hp.nvars), vh(hp.nvars);
  for (int i = 0; i < hp.nvars; ++i) {
    vl[i] = (i128)lo[i];
    vh[i] = (i128)hi[i];
  }
  int64_t cnt = 0;
  const MkBoxVerdict bv = mk_eval_box<i128>(HP, vl.data(), vh.data(), Rg.data(), &cnt);
  if (!bv.any_false) {
    for (int r = 0; r < hp.nregs; ++r) {
      const MkIvT<i128>& g = Rg[r];
      if ((g.fl & MK_FL_OK) && g.lo <= g.hi && g.lo >= (i128)INT32_MIN && g.hi <= (i128)INT32_MAX)
        rbits[r] = 32;
    }
  }
  return rbits;
}

template <typename K>
static int race_run(mk_ctx* ctx, const RaceDev& R, unsigned long long vol, int bits, int nregs,
                    mk_race_result* out, char* base, unsigned long long* ctr,
                    const mk_race_prog* prog, const int64_t* hlo, const int64_t* hhi) {
  cudaStream_t s = ctx->stream;
  // tuples: keys + values, double buffered for the sort (mk_sort.cuh)
  const size_t sort_ws = mksort::workspace_bytes(vol);
  size_t off = 0;
  auto place = [&](size_t bytes) {
    size_t o = off;
    off = (off + bytes + 255) / 256 * 256;
    return o;
  };
  const size_t o_k0 = place(sizeof(K) * vol), o_k1 = place(sizeof(K) * vol);
  const size_t o_v0 = place(sizeof(uint32_t) * vol), o_v1 = place(sizeof(uint32_t) * vol);
  const size_t o_ws = place(sort_ws);
  int rc = ensure(ctx, &ctx->d_work, &ctx->d_work_bytes, off);
  if (rc) return rc;
  char* wb = static_cast<char*>(ctx->d_work);
  K* k0 = reinterpret_cast<K*>(wb + o_k0);
  K* k1 = reinterpret_cast<K*>(wb + o_k1);
  uint32_t* v0 = reinterpret_cast<uint32_t*>(wb + o_v0);
  uint32_t* v1 = reinterpret_cast<uint32_t*>(wb + o_v1);
  (void)base;
  const int grid = ctx->sms * 8;
  const K sentinel = (K)(bits >= (int)(8 * sizeof(K)) ? ~(K)0 : (((K)1 << bits) - 1));
  // specialised generator (NVRTC) when available, else the interpreter
  cudaKernel_t jk = nullptr, jkc = nullptr;
  std::string src;
  if (!getenv("MK_NO_JIT")) {
    const mk_problem_set& set = prog->set;
    const std::vector<int> rbits = register_bits(set, 0, hlo, hhi);
    src = mkjit::race_gen_source(
        set.probs[0], set.insns + set.probs[0].insn_off, set.consts + set.probs[0].const_off,
        R.n_outer, prog->off_reg, prog->shared, prog->id_var, hlo, hhi, sizeof(K) == 8,
        getenv("MK_JIT_WIDE") ? nullptr : rbits.data(), R.off_lo, R.nblocks);
    if (const char* dump = getenv("MK_JIT_DUMP")) {
      FILE* f = fopen(dump, "w");
      if (f) {
        fputs(src.c_str(), f);
        fclose(f);
      }
    }
    jk = mkjit::get_kernel(ctx->jit, src, ctx->device);
    // the compacting generator of the same source (MK_RACE_SEPARATE_COMPACT:
    // dense generation + k_compact, measurement)
    if (jk && !getenv("MK_RACE_SEPARATE_COMPACT"))
      jkc = mkjit::get_kernel(ctx->jit, src, ctx->device, "mk_race_genc_jit");
  }
  out->jit = jk != nullptr;
  // fast path: the fused ordered pass (no per-instance HBM traffic).  When
  // the accesses arrive in non-decreasing key order in instance order (a
  // coalesced store), the stable sort is the identity and the adjacent-pair
  // scan of the sorted tuples is exactly what the pass computes in registers;
  // otherwise its result is discarded and the sort path below runs.
  const bool ranged = prog->end > 0;
  const unsigned long long r_begin = ranged ? prog->begin : 0ull;
  const unsigned long long r_count = ranged ? (prog->end > prog->begin ? prog->end - prog->begin : 0ull)
                                            : vol;
  out->off_lo = R.off_lo;
  out->nblocks = R.nblocks;
  if (ranged && !jk) {
    // a shard is decided by the fused pass only; without it the caller
    // sweeps the whole launch
    out->sorted = 0;
    return MK_OK;
  }
  if (jk && (ranged || (!getenv("MK_RACE_NO_FAST") && !getenv("MK_RACE_FORCE_SORT")))) {
    cudaKernel_t fk = mkjit::get_kernel(ctx->jit, src, ctx->device, "mk_race_fused_jit");
    if (fk) {
      const int fgrid = ctx->sms * 8;
      const unsigned long long warps = (unsigned long long)fgrid * (RACE_THREADS / 32);
      unsigned long long chunk = (r_count + warps - 1) / warps;
      chunk = (chunk + 31) / 32 * 32;
      if (chunk < 32) chunk = 32;
      const size_t rbytes = sizeof(unsigned long long) * MK_RACE_REC * warps;
      int rc0 = ensure(ctx, &ctx->d_work, &ctx->d_work_bytes, rbytes);
      if (rc0) return rc0;
      unsigned long long* rec = static_cast<unsigned long long*>(ctx->d_work);
      unsigned long long init[13] = {0ull, 0ull, ~0ull, 0ull, 0ull, 0ull, 0ull,
                                     0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
      CK(cudaMemcpyAsync(ctr, init, sizeof(init), cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(ctx->ev[0], s));
      unsigned long long a_vol = r_count, a_chunk = chunk, a_nb = R.nblocks, a_start = r_begin;
      unsigned long long* a_rec = rec;
      unsigned long long* a_ctr = ctr;
      void* fargs[] = {&a_vol, &a_chunk, &a_start, &a_nb, &a_rec, &a_ctr};
      CK(cudaLaunchKernel((const void*)fk, dim3(fgrid), dim3(RACE_THREADS), fargs, 0, s));
      CK(cudaEventRecord(ctx->ev[1], s));
      k_race_bound<<<1, 1024, 0, s>>>(rec, (int)warps, ctr);
      CK(cudaGetLastError());
      CK(cudaEventRecord(ctx->ev[2], s));
      unsigned long long h[13];
      CK(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, s));
      CK(cudaEventRecord(ctx->ev[3], s));
      CK(cudaStreamSynchronize(s));
      out->have = h[12] ? 1 : 0;
      out->first_key = h[6];
      out->first_id = h[7];
      out->first_idx = h[8];
      out->last_key = h[9];
      out->last_id = h[10];
      out->last_idx = h[11];
      if (ranged && h[4]) {
        out->sorted = 0;   // out of order: the caller sweeps the whole launch
        return MK_OK;
      }
      if (!h[4]) {
        out->fused = 1;
        out->sorted = 1;
        out->tuples = h[0];
        out->instances = h[3];
        out->conflicts = h[1];
        out->has_race = h[1] > 0;
        out->sort_bits = bits;
        if (out->has_race) {
          out->idx_b = h[2] >> 32;
          out->idx_a = h[2] & 0xffffffffull;
          out->offset = (int64_t)(h[5] / R.nblocks) + R.off_lo;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
        out->gen_ms = ms;
        cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]);
        out->scan_ms = ms;
        out->sort_ms = 0.0;
        out->hbm_bytes = 2ull * rbytes;   // per-warp records: written once, read once
        return MK_OK;
      }
      // out of order: reset the counters for the sort path
      CK(cudaMemcpyAsync(ctr, init, sizeof(init), cudaMemcpyHostToDevice, s));
    }
  }
  if (ranged) {
    out->sorted = 0;   // no specialised fused pass: the caller sweeps the whole launch
    return MK_OK;
  }
  CK(cudaEventRecord(ctx->ev[0], s));
  bool compacted = false;
  if (jkc) {
    // generation and compaction in one pass: only the accesses are written
    mksort::Workspace gw = mksort::carve(wb + o_ws);
    CK(cudaMemsetAsync(gw.tile_ctr + 14, 0, sizeof(unsigned), s));
    unsigned long long a_vol = vol, a_epoch = mksort::next_epoch();
    K* a_keys = k0;
    uint32_t* a_vals = v0;
    unsigned long long* a_cnt = ctr + 0;
    unsigned long long* a_eval = ctr + 3;
    unsigned long long* a_lb = gw.lookback;
    unsigned* a_tc = gw.tile_ctr + 14;
    void* args[] = {&a_vol, &a_keys, &a_vals, &a_cnt, &a_eval, &a_lb, &a_tc, &a_epoch};
    const unsigned long long per = 256ull * (unsigned long long)mkjit::gc_items();
    const unsigned long long tiles = (vol + per - 1) / per;
    CK(cudaLaunchKernel((const void*)jkc, dim3((unsigned)tiles), dim3(RACE_THREADS), args, 0, s));
    compacted = true;
  } else if (jk) {
    unsigned long long a_vol = vol, a_nb = R.nblocks;
    K a_sent = sentinel;
    K* a_keys = k0;
    uint32_t* a_vals = v0;
    unsigned long long* a_cnt = ctr + 0;
    unsigned long long* a_eval = ctr + 3;
    long long a_off = R.off_lo;
    void* args[] = {&a_vol, &a_sent, &a_keys, &a_vals, &a_cnt, &a_eval, &a_off, &a_nb};
    CK(cudaLaunchKernel((const void*)jk, dim3(grid), dim3(RACE_THREADS), args, 0, s));
  } else {
    const size_t shm = sizeof(int64_t) * (size_t)nregs * RACE_THREADS;
    if (shm > 48 * 1024)
      CK(cudaFuncSetAttribute(k_race_gen<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)shm));
    k_race_gen<K><<<grid, RACE_THREADS, shm, s>>>(R, vol, sentinel, k0, v0, ctr + 0, ctr + 3);
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(ctx->ev[1], s));
  // order-preserving compaction of the accesses (sentinels out; skipped when
  // every instance is an access), then one scan that also detects order:
  // keys that already arrive non-decreasing (a coalesced access pattern:
  // offsets grow with the thread index) need no sort, since equal keys are
  // then already adjacent in instance order, exactly as the stable sort would
  // leave them.  MK_RACE_FORCE_SORT sorts regardless (measurement).
  unsigned long long h[6];
  CK(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  K* kc = k0;
  K* ko = k1;
  uint32_t* vc = v0;
  uint32_t* vo = v1;
  if (compacted || h[0] == vol) {
    CK(cudaMemcpyAsync(ctr + 5, &h[0], sizeof(h[0]), cudaMemcpyHostToDevice, s));
  } else {
    CK((mksort::compact<K, uint32_t>(k0, v0, k1, v1, vol, sentinel, wb + o_ws, ctr + 5, s)));
    kc = k1;
    ko = k0;
    vc = v1;
    vo = v0;
  }
  const bool force = getenv("MK_RACE_FORCE_SORT") != nullptr;
  if (!force) {
    k_race_scan<K><<<grid, RACE_THREADS, 0, s>>>(R, kc, vc, ctr + 5, ctr + 1, ctr + 2, ctr + 4);
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (force) h[4] = 1;
  const unsigned long long n = h[5];
  K* ks = kc;
  uint32_t* vs = vc;
  out->sorted = h[4] == 0;
  CK(cudaEventRecord(ctx->ev[2], s));
  if (h[4]) {
    unsigned long long reset[2] = {0ull, ~0ull};
    CK(cudaMemcpyAsync(ctr + 1, reset, sizeof(reset), cudaMemcpyHostToDevice, s));
    mksort::SortInfo si{};
    // MK_RACE_FORCE_SORT runs the sort path on keys the scan saw in order;
    // the sort's own order check then skips every digit pass unless
    // MK_SORT_ALL_PASSES forces them (measurement of the passes themselves)
    CK((mksort::sort_pairs<K, uint32_t>(kc, vc, ko, vo, n, bits, wb + o_ws, ctx->sms, s, &ks, &vs,
                                       &si, getenv("MK_SORT_ALL_PASSES") != nullptr,
                                       /*known_unsorted=*/!force)));
    out->sort_passes = si.passes_run;
    CK(cudaEventRecord(ctx->ev[2], s));
    k_race_scan<K><<<grid, RACE_THREADS, 0, s>>>(R, ks, vs, ctr + 5, ctr + 1, ctr + 2, nullptr);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, s));
  }
  CK(cudaEventRecord(ctx->ev[3], s));
  CK(cudaStreamSynchronize(s));
  out->tuples = h[0];
  out->instances = h[3];
  out->conflicts = h[1];
  out->has_race = h[1] > 0;
  out->sort_bits = bits;
  if (out->has_race) {
    const unsigned long long i = h[2];
    uint32_t va = 0, vb2 = 0;
    K key = 0;
    CK(cudaMemcpy(&va, vs + i - 1, sizeof(va), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&vb2, vs + i, sizeof(vb2), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&key, ks + i, sizeof(key), cudaMemcpyDeviceToHost));
    out->idx_a = va;
    out->idx_b = vb2;
    out->offset = (int64_t)((unsigned long long)key / R.nblocks) + R.off_lo;
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
  out->gen_ms = ms;
  cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]);
  out->sort_ms = ms;
  cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
  out->scan_ms = ms;
  // one tuple write at generation, one read + one write for a
  // single-pass-equivalent sort, one read in the conflict scan
  out->hbm_bytes = 4ull * (unsigned long long)(sizeof(K) + sizeof(uint32_t)) * h[0];
  return MK_OK;
}

extern "C" int mk_race_sweep(mk_ctx* ctx, const mk_race_prog* prog, mk_race_result* out) {
  if (!ctx || !prog || !out) return fail(ctx, MK_EINVAL, "null argument");
  std::memset(out, 0, sizeof(*out));
  CK(cudaSetDevice(ctx->device));
  const mk_problem_set& set = prog->set;
  if (set.nprob != 1) return fail(ctx, MK_EINVAL, "race sweep takes exactly one problem");
  const mk_problem& hp = set.probs[0];
  if (!(hp.flags & MK_PF_NARROW)) return fail(ctx, MK_EINVAL, "race sweep needs a narrow problem");
  if (hp.nvars > SMALL_V || hp.nregs > SMALL_R)
    return fail(ctx, MK_EINVAL, "race sweep program exceeds the small-problem limits");
  if (prog->off_reg < 0 || prog->off_reg >= hp.nregs) return fail(ctx, MK_EINVAL, "bad off_reg");
  // instance box (int64) and volume
  std::vector<int64_t> lo(hp.nvars), hi(hp.nvars);
  const int n_outer = hp.nvars - prog->n_exist;
  if (prog->n_exist < 0 || n_outer < 0) return fail(ctx, MK_EINVAL, "bad n_exist");
  long double volf = 1.0L, innerf = 1.0L;
  unsigned long long vol = 1, inner = 1;
  for (int i = 0; i < hp.nvars; ++i) {
    lo[i] = (int64_t)set.var_lo[hp.var_off + i].lo;
    hi[i] = (int64_t)set.var_hi[hp.var_off + i].lo;
    const long double w = (long double)(hi[i] - lo[i] + 1);
    if (i < n_outer) {
      volf *= w;
      vol *= (unsigned long long)(hi[i] - lo[i] + 1);
    } else {
      innerf *= w;
      inner *= (unsigned long long)(hi[i] - lo[i] + 1);
    }
  }
  if (volf > 2147483647.0L) return fail(ctx, MK_EINVAL, "race sweep box exceeds 2^31 instances");
  if (volf * innerf > 9.0e18L) return fail(ctx, MK_EINVAL, "race sweep box exceeds 2^63 points");
  int rc = upload_set(ctx, &set, &ctx->scratch, false);
  if (rc) return rc;
  mk_dset* ds = &ctx->scratch;
  char* base = static_cast<char*>(ds->d);
  // small side buffer: box bounds, root offset range, counters
  if (!ctx->h_race) {
    CK(cudaMalloc(&ctx->h_race, 4096));
  }
  char* side = static_cast<char*>(ctx->h_race);
  int64_t* d_lo = reinterpret_cast<int64_t*>(side);
  int64_t* d_hi = d_lo + MK_MAXV;
  int64_t* d_rng = d_hi + MK_MAXV;
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(d_rng + 2);
  cudaStream_t s = ctx->stream;
  CK(cudaMemcpyAsync(d_lo, lo.data(), sizeof(int64_t) * hp.nvars, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_hi, hi.data(), sizeof(int64_t) * hp.nvars, cudaMemcpyHostToDevice, s));
  // [0] accesses, [1] conflicts, [2] first conflict, [3] evaluations,
  // [4] unsorted flag, [5] compacted count
  unsigned long long init[6] = {0ull, 0ull, ~0ull, 0ull, 0ull, 0ull};
  CK(cudaMemcpyAsync(ctr, init, sizeof(init), cudaMemcpyHostToDevice, s));
  RaceDev R;
  const mk_problem* dprobs = reinterpret_cast<const mk_problem*>(base + ds->o_probs);
  // the device view of problem 0, built from the host copy's offsets (the
  // problem record itself lives in HBM)
  R.P.p = dprobs;
  R.P.insns = reinterpret_cast<const mk_insn*>(base + ds->o_insn) + hp.insn_off;
  R.P.consts = reinterpret_cast<const mk_i128*>(base + ds->o_const) + hp.const_off;
  R.P.atom_regs = reinterpret_cast<const int32_t*>(base + ds->o_ar) + hp.atom_off;
  R.P.atom_masks = reinterpret_cast<const uint64_t*>(base + ds->o_am) + hp.atom_off;
  R.P.rows = reinterpret_cast<const mk_row*>(base + ds->o_rows) + hp.row_off;
  R.P.terms = reinterpret_cast<const mk_row_term*>(base + ds->o_terms);
  R.prob = dprobs;
  R.lo = d_lo;
  R.hi = d_hi;
  R.off_reg = prog->off_reg;
  R.shared = prog->shared ? 1 : 0;
  unsigned long long nblocks = 1;
  R.n_outer = n_outer;
  R.inner = inner;
  for (int a = 0; a < 6; ++a) {
    R.id_var[a] = prog->id_var[a];
    if (R.id_var[a] >= n_outer) return fail(ctx, MK_EINVAL, "identity var must be a leading var");
    if (a < 3 && R.id_var[a] >= 0 && R.shared)
      nblocks *= (unsigned long long)(hi[R.id_var[a]] - lo[R.id_var[a]] + 1);
  }
  R.nblocks = nblocks;
  R.off_lo = 0;
  k_race_root<<<1, 32, 0, s>>>(R, d_rng);
  CK(cudaGetLastError());
  int64_t rng[2];
  CK(cudaMemcpyAsync(rng, d_rng, sizeof(rng), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  R.off_lo = rng[0];
  const long double keyspan = ((long double)rng[1] - (long double)rng[0] + 1.0L) * (long double)nblocks;
  if (keyspan > 18446744073709551615.0L)
    return fail(ctx, MK_EINVAL, "race sweep key (offset x block) exceeds 64 bits");
  // real keys are <= kmax; kmax + 1 must fit the key width as the sentinel
  const unsigned long long kmax =
      (unsigned long long)((unsigned long long)(rng[1] - rng[0]) * nblocks + (nblocks - 1));
  if (kmax == ~0ull) return fail(ctx, MK_EINVAL, "race sweep key (offset x block) exceeds 64 bits");
  int bits = mk_bitlen((uint64_t)(kmax + 1));
  if (bits < 1) bits = 1;
  if (bits <= 32)
    return race_run<uint32_t>(ctx, R, vol, bits, hp.nregs, out, base, ctr, prog, lo.data(),
                              hi.data());
  return race_run<unsigned long long>(ctx, R, vol, bits, hp.nregs, out, base, ctr, prog, lo.data(),
                                      hi.data());
}

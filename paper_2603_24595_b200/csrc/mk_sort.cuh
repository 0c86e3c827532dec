// mk_sort.cuh -- the K2 race path's HBM sort, hand-written for sm_100a.
//
// Stable LSD radix sort of (key, value) tuples plus an order-preserving
// compaction, replacing cub::DeviceRadixSort / cub::DeviceSelect on the race
// sweep (mk_race.cuh) and the oracle-rule access replay (mk_access.cuh).
//
//   k_sort_order    one read of the keys: keys that arrive non-decreasing
//                   (a coalesced store's tuples) skip the sort entirely --
//                   the stable sort is then the identity.
//   k_sort_hist     ONE read of the keys: the digit histograms of every pass
//                   at once (shared-memory counters per CTA, 4 x 8-bit digits
//                   for u32 keys, up to 8 for u64; run heads of equal digits
//                   across a warp add their run length).  A pass whose digit
//                   is the same for every key moves nothing and is skipped.
//   k_sort_pass     one onesweep pass per remaining digit (decoupled
//                   look-back): tiles of 4096 tuples claim an in-order tile
//                   id, rank their keys per digit with warp match/ballot
//                   (stable: warp-striped input order), publish per-digit
//                   tile counts, look back for the exclusive prefix, stage
//                   the tile digit-sorted in shared memory and write each
//                   digit run contiguously.  Per pass HBM traffic: one read
//                   and one write of every tuple, plus 8 B per (tile, digit)
//                   of look-back state.
//   k_compact       order-preserving removal of sentinel tuples (guarded
//                   accesses that did not execute), one read + one write:
//                   each 4096-tuple tile arrives in shared memory by TMA bulk
//                   copies (cp.async.bulk + mbarrier), per-item ballots, one
//                   warp-parallel decoupled look-back over tile counts.
//
// Look-back entries carry an epoch tag, so the state array is never cleared:
// entry = epoch << 34 | flag << 32 | count (flag 1: tile aggregate, 2:
// inclusive prefix).  Tiles are claimed with an atomic counter in launch
// order, so every tile a CTA waits for is held by a running or finished CTA.

#pragma once

#include <cstdint>

namespace mksort {

constexpr int kThreads = 256;           // 8 warps
constexpr int kWarps = kThreads / 32;
constexpr int kTileMin = kThreads * 16;  // smallest tile: sizes the look-back state

// tuples per thread: 16 for every pair width (measured on the B200: 8 per
// thread for 16-byte pairs -- half the staged tile, no spills -- sorted 6 %
// slower, the look-back costs more per byte than the smaller tile saves)
template <typename K, typename V>
struct Tiling {
  static constexpr int items = 16;
  static constexpr int tile = kThreads * items;
};
// the compaction's tile (its own: it keeps no per-digit state, so larger
// tiles amortise the look-back and the TMA round trip further)
#ifndef MK_COMPACT_ITEMS
#define MK_COMPACT_ITEMS 24   // measured: profiles/r02_compact_tile.jsonl (16: 6.17 ms, 24: 5.74, 32: 6.09)
#endif
template <typename K, typename V>
struct CompactTiling {
  static constexpr int items = MK_COMPACT_ITEMS;
  static constexpr int tile = kThreads * items;
};
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr unsigned long long kFlagAgg = 1ull << 32;
constexpr unsigned long long kFlagIncl = 2ull << 32;
constexpr unsigned long long kCountMask = 0xffffffffull;

template <typename K>
struct KeyTraits {
  static constexpr int kPasses = (int)(8 * sizeof(K)) / kRadixBits;
};

__device__ __forceinline__ unsigned lane_lt_mask() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void st_volatile(unsigned long long* p, unsigned long long v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v));
}

// -- TMA bulk copies (cp.async.bulk) with an mbarrier ----------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// one bulk copy global -> shared of `bytes` (a multiple of 16, both ends
// 16-byte aligned) completing on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n MK_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MK_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Decoupled look-back by one whole warp (tile counts, one entry per tile):
// the lanes read 32 predecessors at once, wait until all of them are
// published, and stop at the nearest inclusive prefix.  Returns the
// exclusive prefix of `tile` (every lane).
__device__ __forceinline__ unsigned long long warp_lookback(const unsigned long long* lookback,
                                                            unsigned tile,
                                                            unsigned long long epoch) {
  const unsigned lane = threadIdx.x & 31;
  unsigned long long prefix = 0;
  long long p = (long long)tile - 1;
  while (p >= 0) {
    const long long idx = p - (long long)lane;
    unsigned long long e = idx >= 0 ? ld_volatile(lookback + idx) : ((epoch << 34) | kFlagIncl);
    while (((e >> 34) != epoch || (e & (3ull << 32)) == 0)) e = ld_volatile(lookback + idx);
    const unsigned incl = __ballot_sync(0xffffffffu, (e & kFlagIncl) != 0);
    const unsigned upto = incl ? (unsigned)(__ffs(incl) - 1) : 31u;   // nearest inclusive lane
    unsigned long long c = (lane <= upto && idx >= 0) ? (e & kCountMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    prefix += c;
    if (incl) break;
    p -= 32;
  }
  return prefix;
}

// -- pass 0: histograms of every digit pass + order check ---------------------------------

// Per key and pass: the run heads among the warp's lanes (consecutive lanes
// hold consecutive keys) add their run length, so ordered keys cost one
// shared atomic per warp and digit instead of 32 conflicting ones.
template <typename K>
__device__ __forceinline__ void hist_add(unsigned* sh, K k, int p, unsigned active) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned d = (unsigned)((k >> (p * kRadixBits)) & (kRadix - 1));
  const unsigned up = __shfl_up_sync(active, d, 1);
  const bool head = lane == 0 || !((active >> (lane - 1)) & 1u) || up != d;
  const unsigned heads = __ballot_sync(active, head);
  if (head) {
    // run = this head up to the next head (or the last active lane)
    const unsigned after = heads & ~((2u << lane) - 1u);
    const unsigned end = after ? (unsigned)(__ffs(after) - 1) : 32u - __clz(active);
    atomicAdd(&sh[p * kRadix + d], end - lane);
  }
}

template <typename K>
__global__ void __launch_bounds__(kThreads)
    k_sort_hist(const K* __restrict__ keys, unsigned long long n, int passes,
                unsigned long long* __restrict__ hist, unsigned* __restrict__ unsorted) {
  __shared__ unsigned sh[KeyTraits<K>::kPasses * kRadix];
  for (int i = threadIdx.x; i < passes * kRadix; i += kThreads) sh[i] = 0;
  __syncthreads();
  bool down = false;
  const unsigned lane = threadIdx.x & 31;
  // warp-contiguous chunks of 8 x 32 keys, grid-stride over the chunks:
  // eight independent loads in flight per lane
  constexpr int J = 8;
  const unsigned long long chunks = (n + 32 * J - 1) / (32 * J);
  const unsigned long long wstride = (unsigned long long)gridDim.x * kWarps;
  for (unsigned long long c = (unsigned long long)blockIdx.x * kWarps + (threadIdx.x >> 5);
       c < chunks; c += wstride) {
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
      const unsigned long long i0 = base + j * 32;
      const bool ok = i0 + lane < n;
      K prev = __shfl_up_sync(0xffffffffu, kk[j], 1);
      const K last = __shfl_sync(0xffffffffu, kk[j], 31);
      if (lane == 0) prev = carry;
      carry = last;
      if (ok && i0 + lane > 0 && kk[j] < prev) down = true;
      if (i0 >= n) break;
      const unsigned active = __ballot_sync(0xffffffffu, ok);
      if (ok) {
#pragma unroll
        for (int p = 0; p < KeyTraits<K>::kPasses; ++p)
          if (p < passes) hist_add<K>(sh, kk[j], p, active);
      }
    }
  }
  if (down) atomicOr(unsorted, 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += kThreads)
    if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

// non-decreasing order check alone (one read of the keys, eight loads in
// flight per lane): keys that arrive ordered need no histogram and no pass
template <typename K>
__global__ void __launch_bounds__(kThreads)
    k_sort_order(const K* __restrict__ keys, unsigned long long n, unsigned* __restrict__ unsorted) {
  constexpr int J = 8;
  const unsigned lane = threadIdx.x & 31;
  const unsigned long long chunks = (n + 32 * J - 1) / (32 * J);
  const unsigned long long wstride = (unsigned long long)gridDim.x * kWarps;
  bool down = false;
  for (unsigned long long c = (unsigned long long)blockIdx.x * kWarps + (threadIdx.x >> 5);
       c < chunks; c += wstride) {
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
      K prev = __shfl_up_sync(0xffffffffu, kk[j], 1);
      const K last = __shfl_sync(0xffffffffu, kk[j], 31);
      if (lane == 0) prev = carry;
      carry = last;
      if (i < n && i > 0 && kk[j] < prev) down = true;
    }
  }
  if (__any_sync(0xffffffffu, down) && lane == 0) atomicOr(unsorted, 1u);
}

// exclusive prefix of each pass's histogram (in place); skip[p] = 1 when one
// digit holds every key (the pass would be the identity)
__global__ void k_sort_hist_scan(unsigned long long* hist, int passes, unsigned long long n,
                                 int* skip) {
  const int p = blockIdx.x;
  if (p >= passes) return;
  __shared__ unsigned long long v[kRadix];
  __shared__ int full;
  if (threadIdx.x == 0) full = 0;
  __syncthreads();
  const unsigned long long c = hist[p * kRadix + threadIdx.x];
  if (c == n) full = 1;
  v[threadIdx.x] = c;
  __syncthreads();
  // Hillis-Steele inclusive scan over 256 counters
  for (int o = 1; o < kRadix; o <<= 1) {
    unsigned long long a = threadIdx.x >= o ? v[threadIdx.x - o] : 0ull;
    __syncthreads();
    v[threadIdx.x] += a;
    __syncthreads();
  }
  hist[p * kRadix + threadIdx.x] = v[threadIdx.x] - c;
  if (threadIdx.x == 0) skip[p] = full;
}

// -- one onesweep pass --------------------------------------------------------------------

template <typename K, typename V>
struct PassSmem {
  K keys[Tiling<K, V>::tile];
  V vals[Tiling<K, V>::tile];
  unsigned wcnt[kWarps][kRadix];   // per-warp digit counts -> exclusive prefix over warps
  unsigned tstart[kRadix];         // digit start inside the tile (exclusive scan)
  unsigned long long gpos[kRadix]; // global start of the digit run of this tile
  unsigned tile;
};

template <typename K, typename V>
__global__ void __launch_bounds__(kThreads, 3)
    k_sort_pass(const K* __restrict__ kin, const V* __restrict__ vin, K* __restrict__ kout,
                V* __restrict__ vout, unsigned long long n, int shift,
                const unsigned long long* __restrict__ gbase, unsigned long long* lookback,
                unsigned* tile_ctr, unsigned long long epoch) {
  constexpr int kItems = Tiling<K, V>::items;
  constexpr int kTile = Tiling<K, V>::tile;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PassSmem<K, V>& S = *reinterpret_cast<PassSmem<K, V>*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    S.tile = atomicAdd(tile_ctr, 1u);
    mbar_init(&bar, 1);
  }
  for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&S.wcnt[0][0])[i] = 0;
  __syncthreads();
  const unsigned tile = S.tile;
  const unsigned long long base = (unsigned long long)tile * kTile;
  // the tile arrives in the staging buffers by TMA bulk copies (16-byte
  // granules; a ragged tail by plain loads); the buffers are only rewritten
  // after every thread has read its items
  {
    const unsigned valid =
        n - base < (unsigned long long)kTile ? (unsigned)(n - base) : (unsigned)kTile;
    const unsigned nb = valid & ~3u;
    if (threadIdx.x == 0 && nb) {
      mbar_expect_tx(&bar, nb * (unsigned)(sizeof(K) + sizeof(V)));
      bulk_g2s(S.keys, kin + base, nb * (unsigned)sizeof(K), &bar);
      bulk_g2s(S.vals, vin + base, nb * (unsigned)sizeof(V), &bar);
    }
    for (unsigned i = nb + threadIdx.x; i < valid; i += kThreads) {
      S.keys[i] = kin[base + i];
      S.vals[i] = vin[base + i];
    }
    if (nb) mbar_wait(&bar, 0);
    __syncthreads();
  }
  // warp-striped: item j of lane l of warp w is tuple base + w*32*kItems + j*32 + l
  K k[kItems];
  V v[kItems];
  unsigned rank[kItems];
  const unsigned long long wbase = base + (unsigned long long)warp * 32 * kItems;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const unsigned long long i = wbase + j * 32 + lane;
    if (i < n) {
      k[j] = S.keys[i - base];
      v[j] = S.vals[i - base];
    }
  }
  // stable rank inside the warp, items in (j, lane) order
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const unsigned long long i = wbase + j * 32 + lane;
    const bool ok = i < n;
    const unsigned active = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      const unsigned d = (unsigned)((k[j] >> shift) & (kRadix - 1));
      const unsigned peers = __match_any_sync(active, d);
      const unsigned before = __popc(peers & lane_lt_mask());
      rank[j] = S.wcnt[warp][d] + before;
      __syncwarp(active);
      if (before == 0) S.wcnt[warp][d] += __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // per digit (thread t = digit t): tile total, exclusive prefix over warps
  const int t = threadIdx.x;
  unsigned total = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const unsigned c = S.wcnt[w][t];
    S.wcnt[w][t] = total;
    total += c;
  }
  // publish the tile aggregate, then look back for the exclusive prefix
  unsigned long long* mine = lookback + (unsigned long long)tile * kRadix + t;
  const unsigned long long tag = epoch << 34;
  if (tile == 0) {
    st_volatile(mine, tag | kFlagIncl | total);
  } else {
    st_volatile(mine, tag | kFlagAgg | total);
  }
  unsigned long long prefix = 0;
  if (tile > 0) {
    long long p = (long long)tile - 1;
    while (p >= 0) {
      const unsigned long long e = ld_volatile(lookback + (unsigned long long)p * kRadix + t);
      if ((e >> 34) != epoch || (e & (3ull << 32)) == 0) continue;   // not yet published
      prefix += e & kCountMask;
      if (e & kFlagIncl) break;
      --p;
    }
    st_volatile(mine, tag | kFlagIncl | (prefix + total));
  }
  // digit starts inside the tile: exclusive scan of the totals (in tstart)
  S.tstart[t] = total;
  __syncthreads();
  for (int o = 1; o < kRadix; o <<= 1) {
    const unsigned a = t >= o ? S.tstart[t - o] : 0u;
    __syncthreads();
    S.tstart[t] += a;
    __syncthreads();
  }
  const unsigned tstart_excl = S.tstart[t] - total;
  __syncthreads();
  S.tstart[t] = tstart_excl;
  S.gpos[t] = gbase[t] + prefix;
  __syncthreads();
  // stage digit-sorted in shared memory
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const unsigned long long i = wbase + j * 32 + lane;
    if (i < n) {
      const unsigned d = (unsigned)((k[j] >> shift) & (kRadix - 1));
      const unsigned pos = S.tstart[d] + S.wcnt[warp][d] + rank[j];
      S.keys[pos] = k[j];
      S.vals[pos] = v[j];
    }
  }
  __syncthreads();
  // write each digit run contiguously
  const unsigned valid = n - base < (unsigned long long)kTile ? (unsigned)(n - base) : (unsigned)kTile;
  for (unsigned i = threadIdx.x; i < valid; i += kThreads) {
    const K kk = S.keys[i];
    const unsigned d = (unsigned)((kk >> shift) & (kRadix - 1));
    const unsigned long long dst = S.gpos[d] + (i - S.tstart[d]);
    kout[dst] = kk;
    vout[dst] = S.vals[i];
  }
}

// -- order-preserving compaction ----------------------------------------------------------

template <typename K, typename V>
__global__ void __launch_bounds__(kThreads)
    k_compact(const K* __restrict__ kin, const V* __restrict__ vin, K* __restrict__ kout,
              V* __restrict__ vout, unsigned long long n, K sentinel,
              unsigned long long* lookback, unsigned* tile_ctr, unsigned long long epoch,
              unsigned long long* count_out) {
  constexpr int kItems = CompactTiling<K, V>::items;
  constexpr int kTile = CompactTiling<K, V>::tile;
  extern __shared__ __align__(128) unsigned char csm[];   // keys[kTile], vals[kTile]
  K* skeys = reinterpret_cast<K*>(csm);
  V* svals = reinterpret_cast<V*>(csm + sizeof(K) * kTile);
  __shared__ unsigned wsum[kWarps];
  __shared__ unsigned tile_s;
  __shared__ unsigned long long prefix_s;
  __shared__ __align__(8) unsigned long long bar;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    tile_s = atomicAdd(tile_ctr, 1u);
    mbar_init(&bar, 1);
  }
  __syncthreads();
  const unsigned tile = tile_s;
  const unsigned long long base = (unsigned long long)tile * kTile;
  const unsigned valid = n - base < (unsigned long long)kTile ? (unsigned)(n - base) : (unsigned)kTile;
  // the tile's keys and values land in shared memory by two TMA bulk copies
  // (multiples of 4 tuples: 16-byte granules); a ragged tail by plain loads
  const unsigned nb = valid & ~3u;
  if (threadIdx.x == 0 && nb) {
    mbar_expect_tx(&bar, nb * (unsigned)(sizeof(K) + sizeof(V)));
    bulk_g2s(skeys, kin + base, nb * (unsigned)sizeof(K), &bar);
    bulk_g2s(svals, vin + base, nb * (unsigned)sizeof(V), &bar);
  }
  for (unsigned i = nb + threadIdx.x; i < valid; i += kThreads) {
    skeys[i] = kin[base + i];
    svals[i] = vin[base + i];
  }
  if (nb) mbar_wait(&bar, 0);
  __syncthreads();
  // warp-striped: item j of lane l of warp w is tuple w*32*kItems + j*32 + l of the
  // tile, so (j, lane) order is input order and every store is coalesced
  const unsigned wloc = (unsigned)warp * 32 * kItems;
  K k[kItems];
  V v[kItems];
  unsigned keep[kItems];
  unsigned mine = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const unsigned i = wloc + j * 32 + lane;
    bool ok = false;
    if (i < valid) {
      k[j] = skeys[i];
      v[j] = svals[i];
      ok = k[j] != sentinel;
    }
    keep[j] = __ballot_sync(0xffffffffu, ok);
    mine += __popc(keep[j]);
  }
  if (lane == 0) wsum[warp] = mine;
  __syncthreads();
  unsigned wpre = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    if (w < warp) wpre += wsum[w];
    total += wsum[w];
  }
  if (warp == 0) {
    unsigned long long* me = lookback + tile;
    const unsigned long long tag = epoch << 34;
    unsigned long long prefix = 0;
    if (tile == 0) {
      if (lane == 0) st_volatile(me, tag | kFlagIncl | total);
    } else {
      if (lane == 0) st_volatile(me, tag | kFlagAgg | total);
      prefix = warp_lookback(lookback, tile, epoch);
      if (lane == 0) st_volatile(me, tag | kFlagIncl | (prefix + total));
    }
    if (lane == 0) {
      prefix_s = prefix;
      const unsigned long long ntiles = (n + kTile - 1) / kTile;
      if (tile == ntiles - 1) *count_out = prefix + total;
    }
  }
  __syncthreads();
  unsigned long long dst = prefix_s + wpre;
  const unsigned lt = lane_lt_mask();
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    if ((keep[j] >> lane) & 1u) {
      const unsigned long long o = dst + __popc(keep[j] & lt);
      kout[o] = k[j];
      vout[o] = v[j];
    }
    dst += __popc(keep[j]);
  }
}

// -- host side ----------------------------------------------------------------------------

// device workspace: histograms, skip flags, order flag, tile counters,
// look-back state (one entry per tile and digit)
inline size_t workspace_bytes(unsigned long long n) {
  const unsigned long long tiles = (n + kTileMin - 1) / kTileMin + 1;
  return 8 * 8 * kRadix + 64 + 64 + 64 * 4 + tiles * kRadix * 8 + 256;
}

struct Workspace {
  unsigned long long* hist;      // [8][256]
  int* skip;                     // [8]
  unsigned* unsorted;            // [1]
  unsigned* tile_ctr;            // [16] one per launch of a call
  unsigned long long* lookback;  // [tiles * 256]
};

inline Workspace carve(void* ws) {
  char* b = static_cast<char*>(ws);
  Workspace w;
  w.hist = reinterpret_cast<unsigned long long*>(b);
  w.skip = reinterpret_cast<int*>(b + 8 * 8 * kRadix);
  w.unsorted = reinterpret_cast<unsigned*>(b + 8 * 8 * kRadix + 64);
  w.tile_ctr = reinterpret_cast<unsigned*>(b + 8 * 8 * kRadix + 128);
  w.lookback = reinterpret_cast<unsigned long long*>(b + 8 * 8 * kRadix + 128 + 64 * 4);
  return w;
}

inline unsigned long long next_epoch() {
  static unsigned long long e = 0;
  e = (e + 1) & ((1ull << 29) - 1);
  if (e == 0) e = 1;
  return e;
}

template <typename K, typename V>
inline size_t pass_smem() {
  return sizeof(PassSmem<K, V>);
}

struct SortInfo {
  int passes_run;      // onesweep passes executed (0: already ordered or one digit)
  int already_sorted;  // keys were non-decreasing: no pass ran
};

// Stable sort of n (key, value) tuples on the low `bits` key bits.  (k0, v0)
// hold the input; on return *kres / *vres point at whichever buffer holds
// the sorted tuples.  Synchronous (reads back the histogram flags).
template <typename K, typename V>
inline cudaError_t sort_pairs(K* k0, V* v0, K* k1, V* v1, unsigned long long n, int bits,
                              void* ws, int sms, cudaStream_t s, K** kres, V** vres,
                              SortInfo* info, bool force_all = false,
                              bool known_unsorted = false) {
  static_assert(kThreads == kRadix, "one thread per digit in the pass kernel");
  *kres = k0;
  *vres = v0;
  if (info) *info = SortInfo{0, 0};
  if (n < 2) return cudaSuccess;
  const int max_passes = KeyTraits<K>::kPasses;
  int passes = (bits + kRadixBits - 1) / kRadixBits;
  if (passes < 1) passes = 1;
  if (passes > max_passes) passes = max_passes;
  Workspace w = carve(ws);
  cudaError_t e;
  if ((e = cudaMemsetAsync(w.hist, 0, 8 * 8 * kRadix + 64 + 64 + 64 * 4, s))) return e;
  if (!force_all && !known_unsorted) {
    // ordered keys: the stable sort is the identity -- one read, no pass
    unsigned unsorted = 0;
    k_sort_order<K><<<sms * 8, kThreads, 0, s>>>(k0, n, w.unsorted);
    if ((e = cudaMemcpyAsync(&unsorted, w.unsorted, sizeof(unsorted), cudaMemcpyDeviceToHost, s)))
      return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    if (!unsorted) {
      if (info) info->already_sorted = 1;
      return cudaSuccess;
    }
  }
  k_sort_hist<K><<<sms * 8, kThreads, 0, s>>>(k0, n, passes, w.hist, w.unsorted);
  k_sort_hist_scan<<<passes, kRadix, 0, s>>>(w.hist, passes, n, w.skip);
  int skip[8] = {0};
  if ((e = cudaMemcpyAsync(skip, w.skip, sizeof(int) * passes, cudaMemcpyDeviceToHost, s))) return e;
  if ((e = cudaStreamSynchronize(s))) return e;
  const size_t smem = pass_smem<K, V>();
  if ((e = cudaFuncSetAttribute(k_sort_pass<K, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem)))
    return e;
  const unsigned long long tiles = (n + Tiling<K, V>::tile - 1) / Tiling<K, V>::tile;
  K* ki = k0;
  V* vi = v0;
  K* ko = k1;
  V* vo = v1;
  int ran = 0;
  for (int p = 0; p < passes; ++p) {
    if (skip[p] && !force_all) continue;
    k_sort_pass<K, V><<<(unsigned)tiles, kThreads, smem, s>>>(
        ki, vi, ko, vo, n, p * kRadixBits, w.hist + p * kRadix, w.lookback, w.tile_ctr + p,
        next_epoch());
    if ((e = cudaGetLastError())) return e;
    K* tk = ki; ki = ko; ko = tk;
    V* tv = vi; vi = vo; vo = tv;
    ++ran;
  }
  *kres = ki;
  *vres = vi;
  if (info) info->passes_run = ran;
  return cudaSuccess;
}

// Order-preserving compaction of the non-sentinel tuples of (kin, vin) into
// (kout, vout); the surviving count lands in *d_count (device).
template <typename K, typename V>
inline cudaError_t compact(const K* kin, const V* vin, K* kout, V* vout, unsigned long long n,
                           K sentinel, void* ws, unsigned long long* d_count, cudaStream_t s) {
  Workspace w = carve(ws);
  cudaError_t e;
  if ((e = cudaMemsetAsync(w.tile_ctr + 15, 0, sizeof(unsigned), s))) return e;
  if (n == 0) return cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s);
  const unsigned long long tiles = (n + CompactTiling<K, V>::tile - 1) / CompactTiling<K, V>::tile;
  const size_t smem = (sizeof(K) + sizeof(V)) * (size_t)CompactTiling<K, V>::tile;
  if ((e = cudaFuncSetAttribute(k_compact<K, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem)))
    return e;
  k_compact<K, V><<<(unsigned)tiles, kThreads, smem, s>>>(kin, vin, kout, vout, n, sentinel,
                                                       w.lookback, w.tile_ctr + 15, next_epoch(),
                                                       d_count);
  return cudaGetLastError();
}

}  // namespace mksort

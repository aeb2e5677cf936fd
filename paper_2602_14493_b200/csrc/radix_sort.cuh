// radix_sort.cuh — stable LSD radix sort of (key, u32 value) pairs, 8-bit digits.
//
// Used three times on the GMR path: the per-view depth order of splats
// (u32 float bits / u64 double bits), the (view, tile) bucketing of tile
// entries (render.py:227 lexsort by (tile, depth, source)),
// and the face->vertex scatter plan.  The element count may live in device
// memory (`n_dev`), so the pipeline never waits on the host for E: grids are
// sized for the capacity and surplus blocks exit.
//
// One pass = upsweep (per-block digit histogram) + scan (per digit over
// blocks) + downsweep (stable in-block rank with warp match_any, scatter).
// Each block owns 4096 consecutive items; each warp a contiguous 512.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>


namespace gmr {

constexpr int kSortThreads = 256;
#ifndef GMR_SORT_PER
#define GMR_SORT_PER 16
#endif
#ifndef GMR_SORT_MINB
#define GMR_SORT_MINB 3
#endif
constexpr int kSortPerThread = GMR_SORT_PER;
constexpr int kSortTile = kSortThreads * kSortPerThread;  // 4096
constexpr int kSortWarps = kSortThreads / 32;

__device__ __forceinline__ unsigned lanemask_lt_sort() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Lanes holding the same digit d (< 512) by nine ballots: they pipeline,
// where __match_any_sync is one long-latency instruction whose cost grows
// with the number of distinct digits in the warp.  Used by the per-list sort
// (bin_depth_sort) and by the radix downsweep on random digits (depth keys,
// tile keys emitted in depth order: config 4 binning 1.449 -> 1.286 ms);
// coherent digits (tile keys emitted in item order) keep match_any.
__device__ __forceinline__ unsigned digit_peers_ballot(uint32_t d) {
  unsigned m = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < 9; ++b) {
    const bool bit = (d >> b) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, bit);
    m &= bit ? bal : ~bal;
  }
  return m;
}

__device__ __forceinline__ uint32_t sort_count(const uint32_t* n_dev, uint32_t n_host) {
  return n_dev ? *n_dev : n_host;
}

// Key-range reduction (32-bit keys): krange = {min, max} of the keys that
// matter, written on the device before the sort (K1's depth keys of kept
// splats).  Digits are those of key - min, and only the passes that
// max - min needs run: a later pass exits at once.  Keys outside the range
// (culled splats, key ~0) land anywhere; their consumers skip them.
struct KeyRange {
  uint32_t lo;
  int passes;   // 8-bit passes max - lo needs (0: all keys equal or none)
};
__device__ __forceinline__ KeyRange key_range(const uint32_t* krange, int bits) {
  KeyRange r{0u, (bits + 7) / 8};
  if (krange) {
    const uint32_t lo = krange[0], hi = krange[1];
    r.lo = lo;
    r.passes = hi > lo ? (39 - __clz(hi - lo)) / 8 : 0;   // bytes of hi - lo
  }
  return r;
}
template <typename K>
__device__ __forceinline__ uint32_t sort_digit(K key, int shift, uint32_t lo) {
  return (uint32_t)((key - (K)lo) >> shift) & 255u;
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) radix_upsweep(const K* __restrict__ keys,
                                                              const uint32_t* n_dev,
                                                              uint32_t n_host, int shift,
                                                              uint32_t* __restrict__ hist,
                                                              int nblocks, const uint32_t* krange, int bits) {
  pdl_wait();
  const KeyRange kr = key_range(krange, bits);
  if (shift >= 8 * kr.passes) return;
  __shared__ uint32_t h[kSortWarps][256];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t n = sort_count(n_dev, n_host);
  const uint32_t base = blockIdx.x * (uint32_t)kSortTile;
  if (base < n) {
    const uint32_t end = min(n, base + (uint32_t)kSortTile);
    for (uint32_t i = base + tid; i < end; i += kSortThreads) {
      atomicAdd(&h[warp][sort_digit(keys[i], shift, kr.lo)], 1u);
    }
  }
  __syncthreads();
  uint32_t s = 0;
#pragma unroll
  for (int w = 0; w < kSortWarps; ++w) s += h[w][tid];
  hist[(size_t)tid * nblocks + blockIdx.x] = s;
}

// block-wide exclusive scan of one value per thread (256 threads)
__device__ __forceinline__ uint32_t block_exclusive_scan_256(uint32_t v, uint32_t* smem_warp,
                                                             uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < kSortWarps ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < kSortWarps; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kSortWarps) smem_warp[lane] = w;  // inclusive per warp
  }
  __syncthreads();
  uint32_t warp_prefix = warp ? smem_warp[warp - 1] : 0;
  if (total) *total = smem_warp[kSortWarps - 1];
  uint32_t r = warp_prefix + x - v;
  __syncthreads();
  return r;
}

// One block per digit: exclusive scan of hist[d][0..nblocks) in place,
// digit total into totals[d].
__global__ void __launch_bounds__(kSortThreads) radix_scan(uint32_t* __restrict__ hist,
                                                           uint32_t* __restrict__ totals,
                                                           int nblocks, const uint32_t* krange, int bits,
                                                           int shift) {
  pdl_wait();
  if (shift >= 8 * key_range(krange, bits).passes) return;
  __shared__ uint32_t sw[kSortWarps];
  uint32_t* row = hist + (size_t)blockIdx.x * nblocks;
  uint32_t carry = 0;
  for (int base = 0; base < nblocks; base += kSortThreads * 4) {
    uint32_t v[4], s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int i = base + threadIdx.x * 4 + k;
      v[k] = i < nblocks ? row[i] : 0;
      s += v[k];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan_256(s, sw, &tot);
    uint32_t run = carry + ex;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int i = base + threadIdx.x * 4 + k;
      if (i < nblocks) row[i] = run;
      run += v[k];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

template <typename K>
struct DownSmem {
  uint32_t wc[kSortWarps][256];   // per-warp digit counts -> exclusive prefixes
  uint32_t boff[257];             // block-local start of each digit
  uint32_t gbase[256];            // global start of each digit for this block
  uint32_t sw[kSortWarps];
  K keys[kSortTile];              // the block's items in sorted (stable) order
  uint32_t vals[kSortTile];
};

// Stable in-block ranking (warp match_any, warps in order), the block's
// items staged in smem in sorted order, then written out in coalesced runs
// per digit.
template <typename K, bool kBallot>
__global__ void __launch_bounds__(kSortThreads, GMR_SORT_MINB) radix_downsweep(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
    uint32_t* __restrict__ vout, const uint32_t* n_dev, uint32_t n_host, int shift,
    const uint32_t* __restrict__ hist, const uint32_t* __restrict__ totals, int nblocks,
    const uint32_t* krange, int bits) {
  pdl_wait();
  const KeyRange kr = key_range(krange, bits);
  if (shift >= 8 * kr.passes) return;
  extern __shared__ __align__(16) unsigned char dsm_raw[];
  DownSmem<K>& sm = *reinterpret_cast<DownSmem<K>*>(dsm_raw);
  const uint32_t n = sort_count(n_dev, n_host);
  const uint32_t base = blockIdx.x * (uint32_t)kSortTile;
  if (base >= n) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t cnt_blk = min((uint32_t)kSortTile, n - base);
  const uint32_t tot_d = totals[tid];
  const bool trivial = __syncthreads_or(tot_d == n);
  const uint32_t seg = base + (uint32_t)warp * (kSortPerThread * 32);
  // a pass whose digit is the same for every key is the identity permutation
  if (trivial) {
    for (uint32_t i = base + tid; i < base + cnt_blk; i += kSortThreads) {
      kout[i] = kin[i];
      vout[i] = vin[i];
    }
    return;
  }
  K key[kSortPerThread];
#pragma unroll
  for (int r = 0; r < kSortPerThread; ++r) {
    const uint32_t idx = seg + r * 32 + lane;
    key[r] = idx < n ? kin[idx] : K(0);
  }
  for (int i = tid; i < kSortWarps * 256; i += kSortThreads) (&sm.wc[0][0])[i] = 0;
  const uint32_t ex = block_exclusive_scan_256(tot_d, sm.sw, nullptr);
  sm.gbase[tid] = ex + hist[(size_t)tid * nblocks + blockIdx.x];
  __syncthreads();
  uint16_t rank[kSortPerThread];
  const unsigned lt = lanemask_lt_sort();
#pragma unroll
  for (int r = 0; r < kSortPerThread; ++r) {
    const uint32_t idx = seg + r * 32 + lane;
    const bool valid = idx < n;
    const uint32_t d = valid ? sort_digit(key[r], shift, kr.lo) : 256u;
    // depth keys: digits of random floats, where the nine pipelined ballots
    // beat one long-latency match_any; tile keys: coherent digits, match_any
    const unsigned peers = kBallot ? digit_peers_ballot(d) : __match_any_sync(0xffffffffu, d);
    const uint32_t c = valid ? sm.wc[warp][d] : 0u;
    rank[r] = (uint16_t)(c + __popc(peers & lt));
    __syncwarp();
    if (valid && (lt & peers) == 0) sm.wc[warp][d] = c + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    // digit tid: per-warp exclusive prefixes and the block-local digit start
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
      const uint32_t c = sm.wc[w][tid];
      sm.wc[w][tid] = run;
      run += c;
    }
    uint32_t tot;
    const uint32_t off = block_exclusive_scan_256(run, sm.sw, &tot);
    sm.boff[tid] = off;
    if (tid == 0) sm.boff[256] = tot;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSortPerThread; ++r) {
    const uint32_t idx = seg + r * 32 + lane;
    if (idx < n) {
      const uint32_t d = sort_digit(key[r], shift, kr.lo);
      const uint32_t lp = sm.boff[d] + sm.wc[warp][d] + rank[r];
      sm.keys[lp] = key[r];
      sm.vals[lp] = vin[idx];
    }
  }
  __syncthreads();
  // coalesced write-out: local position i -> digit run -> global slot
  for (uint32_t i = tid; i < cnt_blk; i += kSortThreads) {
    const K k = sm.keys[i];
    const uint32_t d = sort_digit(k, shift, kr.lo);
    const uint32_t pos = sm.gbase[d] + (i - sm.boff[d]);
    kout[pos] = k;
    vout[pos] = sm.vals[i];
  }
}

// ---------------------------------------------------------------------------
// Small inputs: the whole sort in one 1024-thread block.  Each thread keeps
// PER (key, value) pairs in registers (warp w owns items w*32*PER + r*32 +
// lane); every digit pass ranks them stably exactly like radix_downsweep
// (match_any, warps in order), scatters through one shared buffer and reads
// back in the same striped order.  One launch instead of 3 per pass: small
// meshes / images are launch-latency bound.  The result is written to the
// buffer the multi-kernel path would use (passes & 1).
// ---------------------------------------------------------------------------

constexpr int kSmallThreads = 1024;
constexpr int kSmallWarps = kSmallThreads / 32;

template <typename K> struct SmallSortLimit { static constexpr uint32_t value = 16384; };
template <> struct SmallSortLimit<unsigned long long> { static constexpr uint32_t value = 12288; };

template <typename K>
inline size_t small_sort_smem(uint32_t n_max) {
  return (size_t)n_max * (sizeof(K) + 4) + (size_t)kSmallWarps * 256 * 4 + 1040 * 4;
}

template <typename K, int PER>
__global__ void __launch_bounds__(kSmallThreads, 1) small_radix_sort(K* __restrict__ k0, uint32_t* __restrict__ v0,
                                                                     K* __restrict__ k1, uint32_t* __restrict__ v1,
                                                                     const uint32_t* n_dev, uint32_t n_host,
                                                                     int bits, uint32_t n_max) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char ss_raw[];
  K* skeys = reinterpret_cast<K*>(ss_raw);
  uint32_t* svals = reinterpret_cast<uint32_t*>(ss_raw + (size_t)n_max * sizeof(K));
  uint32_t(*wc)[256] = reinterpret_cast<uint32_t(*)[256]>(ss_raw + (size_t)n_max * (sizeof(K) + 4));
  uint32_t* tot = reinterpret_cast<uint32_t*>(wc + kSmallWarps);   // [256] digit totals, [256..263] scan, [264] flag
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t n = sort_count(n_dev, n_host);
  const uint32_t seg = (uint32_t)warp * (PER * 32);
  K key[PER];
  uint32_t val[PER];
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const uint32_t idx = seg + r * 32 + lane;
    key[r] = idx < n ? k0[idx] : K(0);
    val[r] = idx < n ? v0[idx] : 0u;
  }
  const unsigned lt = lanemask_lt_sort();
  const int passes = (bits + 7) / 8;
  for (int pass = 0; pass < passes; ++pass) {
    const int shift = 8 * pass;
    for (int i = tid; i < kSmallWarps * 256; i += kSmallThreads) (&wc[0][0])[i] = 0;
    __syncthreads();
    uint16_t rank[PER];
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t idx = seg + r * 32 + lane;
      const bool valid = idx < n;
      const uint32_t d = valid ? ((uint32_t)(key[r] >> shift) & 255u) : 256u;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const uint32_t c = valid ? wc[warp][d] : 0u;
      rank[r] = (uint16_t)(c + __popc(peers & lt));
      __syncwarp();
      if (valid && (lt & peers) == 0) wc[warp][d] = c + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // digit tid: per-warp exclusive prefixes; digit totals; exclusive scan
    if (tid < 256) {
      uint32_t run = 0;
      for (int w = 0; w < kSmallWarps; ++w) {
        const uint32_t c = wc[w][tid];
        wc[w][tid] = run;
        run += c;
      }
      tot[tid] = run;
    }
    __syncthreads();
    if (tid < 32) {   // one warp scans the 256 totals (8 per lane)
      uint32_t v[8], s8 = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) { v[k] = tot[lane * 8 + k]; s8 += v[k]; }
      uint32_t x = s8;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      uint32_t run = x - s8;
      bool triv = false;
#pragma unroll
      for (int k = 0; k < 8; ++k) { triv |= v[k] == n; tot[lane * 8 + k] = run; run += v[k]; }
      const bool any_triv = __any_sync(0xffffffffu, triv);
      if (lane == 0) tot[264] = any_triv ? 1u : 0u;
    }
    __syncthreads();
    if (tot[264]) continue;   // identity permutation: the registers are already in order
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t idx = seg + r * 32 + lane;
      if (idx < n) {
        const uint32_t d = (uint32_t)(key[r] >> shift) & 255u;
        const uint32_t lp = tot[d] + wc[warp][d] + rank[r];
        skeys[lp] = key[r];
        svals[lp] = val[r];
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t idx = seg + r * 32 + lane;
      if (idx < n) {
        key[r] = skeys[idx];
        val[r] = svals[idx];
      }
    }
    __syncthreads();
  }
  K* kout = (passes & 1) ? k1 : k0;
  uint32_t* vout = (passes & 1) ? v1 : v0;
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const uint32_t idx = seg + r * 32 + lane;
    if (idx < n) {
      kout[idx] = key[r];
      vout[idx] = val[r];
    }
  }
}

template <typename K, int PER>
inline void launch_small_sort(K* keys[2], uint32_t* vals[2], const uint32_t* n_dev, uint32_t n_host, int bits,
                              uint32_t n_max, cudaStream_t stream) {
  // thread-safe one-time attribute; a failure surfaces as the launch error
  static const cudaError_t attr_rc = cudaFuncSetAttribute(
      small_radix_sort<K, PER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)small_sort_smem<K>(SmallSortLimit<K>::value));
  (void)attr_rc;
  pdl_launch(small_radix_sort<K, PER>, dim3(1), dim3(kSmallThreads), small_sort_smem<K>(n_max), stream, 
      keys[0], vals[0], keys[1], vals[1], n_dev, n_host, bits, n_max);
}

// Host-side driver: sorts [0, n) of (keys[0], vals[0]) by bits [0, bits).
// Ping-pongs between buffer 0 and 1; returns the index (0/1) holding the
// result.  `capacity` bounds n and sizes the grids; hist needs
// 256 * blocks(capacity) + 256 words.
template <typename K>
inline int radix_sort_pairs(K* keys[2], uint32_t* vals[2], const uint32_t* n_dev,
                            uint32_t n_host, uint32_t capacity, int bits, uint32_t* hist,
                            cudaStream_t stream, bool random_digits = false,
                            const uint32_t* krange = nullptr, bool* reduced = nullptr) {
  // krange (32-bit keys, multi-block path only): see KeyRange.  *reduced
  // tells the caller that the result buffer is then chosen on the device
  // (result_buffer) instead of the returned index.
  if (reduced) *reduced = false;
  const int nblocks = (int)((capacity + kSortTile - 1) / kSortTile);
  if (nblocks == 0 || bits <= 0) return 0;
  if (capacity <= SmallSortLimit<K>::value) {   // one block, one launch
    const uint32_t per = (capacity + kSmallThreads - 1) / kSmallThreads;
    if (per <= 2) launch_small_sort<K, 2>(keys, vals, n_dev, n_host, bits, capacity, stream);
    else if (per <= 4) launch_small_sort<K, 4>(keys, vals, n_dev, n_host, bits, capacity, stream);
    else if (per <= 8) launch_small_sort<K, 8>(keys, vals, n_dev, n_host, bits, capacity, stream);
    else if (per <= 12) launch_small_sort<K, 12>(keys, vals, n_dev, n_host, bits, capacity, stream);
    else launch_small_sort<K, 16>(keys, vals, n_dev, n_host, bits, capacity, stream);
    return ((bits + 7) / 8) & 1;
  }
  uint32_t* totals = hist + (size_t)256 * nblocks;
  // thread-safe one-time attribute per K; a failure surfaces as the launch error
  static const cudaError_t attr_rc = cudaFuncSetAttribute(
      radix_downsweep<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DownSmem<K>));
  static const cudaError_t attr_rb = cudaFuncSetAttribute(
      radix_downsweep<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DownSmem<K>));
  (void)attr_rc;
  (void)attr_rb;
  if (sizeof(K) != 4) krange = nullptr;
  if (reduced) *reduced = krange != nullptr;
  int cur = 0;
  for (int shift = 0; shift < bits; shift += 8) {
    pdl_launch(radix_upsweep<K>, dim3(nblocks), dim3(kSortThreads), 0, stream, keys[cur], n_dev, n_host, shift, hist,
                                                           nblocks, krange, bits);
    pdl_launch(radix_scan, dim3(256), dim3(kSortThreads), 0, stream, hist, totals, nblocks, krange, bits, shift);
    auto down = random_digits ? radix_downsweep<K, true> : radix_downsweep<K, false>;
    pdl_launch(down, dim3(nblocks), dim3(kSortThreads), sizeof(DownSmem<K>), stream, 
        keys[cur], vals[cur], keys[cur ^ 1], vals[cur ^ 1], n_dev, n_host, shift, hist, totals, nblocks,
        krange, bits);
    cur ^= 1;
  }
  return cur;
}

// Buffer holding a range-reduced sort's result: the executed passes flip it.
__device__ __forceinline__ const uint32_t* result_buffer(const uint32_t* v0, const uint32_t* v1,
                                                         const uint32_t* krange, int bits) {
  return (key_range(krange, bits).passes & 1) ? v1 : v0;
}

// kernel launches of one radix_sort_pairs call
template <typename K>
inline int radix_sort_launches(uint32_t capacity, int bits) {
  if (capacity == 0 || bits <= 0) return 0;
  return capacity <= SmallSortLimit<K>::value ? 1 : 3 * ((bits + 7) / 8);
}

inline size_t radix_hist_words(uint32_t capacity) {
  const size_t nblocks = (capacity + kSortTile - 1) / kSortTile;
  return 256 * nblocks + 256;
}

}  // namespace gmr

// Warp-level quantizer and the bit-exact 32-bit arithmetic coder (device side).
//
// Quantizer: restates pkg/src/edpc/coder.py:58-80 (_quantize_kernel).
//   base = floor(p * 65280); freq = base + 1; the deficit 65536 - sum(freq)
//   goes one unit each to the largest remainders, ties to the lower symbol
//   (the reference's stable mergesort over base - scaled).  One warp per row,
//   lane l owns symbols 8l..8l+7.  Instead of sorting, the warp finds the
//   deficit-th largest (remainder, -symbol) key with an MSB-first radix
//   select (one __reduce_add_sync per key bit), so no shared memory is used.
//   Remainders are compared as the IEEE bit patterns of the exact float64
//   remainder, which orders non-negative doubles exactly.
//
// Coder: restates coder.py:126-165 (encode), :177-229 (decode), :290-306
//   (finish): 32-bit low/high, TOTAL = 2^16, pending-bit underflow, MSB-first
//   bit packing, decoder reads zeros past bit_length and fails past +64.
#pragma once

#include <stdint.h>

#include "common.cuh"

namespace edpc {

constexpr uint64_t kHalf = 1ull << 31;
constexpr uint64_t kQuarter = 1ull << 30;
constexpr uint64_t kThreeQ = kHalf + kQuarter;
constexpr uint64_t kMask32 = (1ull << 32) - 1;

// ----------------------------------------------------------------- quantizer

// k-th largest of 256 distinct keys spread 8 per lane (k in [1, 256]).
template <typename K, int kBits>
__device__ __forceinline__ K warp_kth_largest(const K (&key)[8], int k, int top_bit) {
  K thr = 0;
  for (int bit = top_bit; bit >= 0; --bit) {
    K cand = thr | ((K)1 << bit);
    int c = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) c += key[j] >= cand ? 1 : 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if (c >= k) thr = cand;
  }
  return thr;
}

// The same selection for the 49-bit keys of fp32-representable rows, in two
// 32-bit levels: the k-th largest of the high 32 bits (key >> 17) first, then
// -- only if several keys tie at that threshold and not all of them are
// selected -- the remaining low 17 bits among the tied keys.  Returns the
// same key as warp_kth_largest<uint64_t, 49> (keys are distinct) in 32 cheap
// iterations instead of 49 64-bit ones (the quantizer was issue-bound).
__device__ __forceinline__ uint64_t warp_kth_largest_49(const uint64_t (&key)[8], int k) {
  uint32_t hi[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) hi[j] = (uint32_t)(key[j] >> 17);
  uint32_t thr = 0;
  for (int bit = 31; bit >= 0; --bit) {
    const uint32_t cand = thr | (1u << bit);
    int c = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) c += hi[j] >= cand ? 1 : 0;
    if (__reduce_add_sync(0xffffffffu, c) >= k) thr = cand;
  }
  int gt = 0, eq = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    gt += hi[j] > thr ? 1 : 0;
    eq += hi[j] == thr ? 1 : 0;
  }
  gt = __reduce_add_sync(0xffffffffu, gt);
  eq = __reduce_add_sync(0xffffffffu, eq);
  const int k2 = k - gt;  // 1 <= k2 <= eq
  uint32_t lo_thr = 0;
  if (k2 < eq) {
    for (int bit = 16; bit >= 0; --bit) {
      const uint32_t cand = lo_thr | (1u << bit);
      int c = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        c += (hi[j] == thr && (uint32_t)(key[j] & 0x1FFFFu) >= cand) ? 1 : 0;
      if (__reduce_add_sync(0xffffffffu, c) >= k2) lo_thr = cand;
    }
  }
  return ((uint64_t)thr << 17) | lo_thr;
}

// Remainder key.  For fp32-representable probabilities p*65280 has at most
// 32 significant bits, so the float64 remainder's low 21 fraction bits are
// zero: (bits >> 21) keeps the full order in 41 bits and leaves room for the
// tie-break (255 - symbol) in the low 8 bits of a 64-bit key.  float64 inputs
// use a 128-bit key with the full 63-bit pattern.
template <bool kF64>
struct QKey;
template <>
struct QKey<false> {
  using T = uint64_t;
  static constexpr int kBits = 49;
  __device__ static T make(double rem, int sym) {
    return ((uint64_t)(__double_as_longlong(rem)) >> 21) << 8 | (uint64_t)(255 - sym);
  }
};
template <>
struct QKey<true> {
  using T = unsigned __int128;
  static constexpr int kBits = 71;
  __device__ static T make(double rem, int sym) {
    return ((unsigned __int128)(uint64_t)__double_as_longlong(rem)) << 8 |
           (unsigned __int128)(255 - sym);
  }
};

// p[j] is symbol 8*lane+j as an exact double.  Produces freq[8] (>= 1, row
// sum exactly 65536).  If the row sums above 1 by more than 1/65280 (never
// for a softmax row) the surplus is taken from the smallest
// remainders among symbols with freq > 1, so the table stays decodable.
template <bool kF64>
__device__ __forceinline__ void warp_quantize(const double (&p)[8], int (&freq)[8]) {
  using Q = QKey<kF64>;
  using K = typename Q::T;
  const int lane = threadIdx.x & 31;
  const double scale = (double)(kTotal - 256);
  K key[8];
  double rem[8];
  int tot = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double scaled = p[j] * scale;
    double fl = floor(scaled);
    int base = (int)fl;
    rem[j] = scaled - fl;  // exact
    freq[j] = base + 1;
    tot += base + 1;
  }
  tot = __reduce_add_sync(0xffffffffu, tot);
  int deficit = kTotal - tot;
  if (deficit > 0) {
#pragma unroll
    for (int j = 0; j < 8; ++j) key[j] = Q::make(rem[j], lane * 8 + j);
    K thr;
    if constexpr (kF64)
      thr = warp_kth_largest<K, Q::kBits>(key, deficit, Q::kBits - 1);
    else
      thr = warp_kth_largest_49(key, deficit);
#pragma unroll
    for (int j = 0; j < 8; ++j) freq[j] += key[j] >= thr ? 1 : 0;
  } else if (deficit < 0) {
    // smallest remainders first (ties to the higher symbol, mirror image of
    // the surplus rule), only where freq > 1
    // top - key is >= 1 for every real key (remainders are < 1)
    const K top = ((K)1 << Q::kBits) - 1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      K kk = Q::make(rem[j], lane * 8 + j);
      key[j] = freq[j] > 1 ? top - kk : (K)0;
    }
    K thr = warp_kth_largest<K, Q::kBits>(key, -deficit, Q::kBits - 1);
#pragma unroll
    for (int j = 0; j < 8; ++j) freq[j] -= (key[j] >= thr && key[j] != 0) ? 1 : 0;
  }
}

// exclusive prefix over the warp: cum[j] = sum of freq of symbols < 8*lane+j
__device__ __forceinline__ void warp_cdf(const int (&freq)[8], uint32_t (&cum)[8]) {
  const int lane = threadIdx.x & 31;
  int local = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) local += freq[j];
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  uint32_t run = (uint32_t)(incl - local);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    cum[j] = run;
    run += (uint32_t)freq[j];
  }
}

// ------------------------------------------------------------------ bit I/O

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// MSB-first bit writer over 32-bit words stored big-endian (byte 0 = bits 0..7).
// Writes past `cap` words are dropped (never out of bounds); the owner
// sizes buffers for the worst case (18 bits/symbol, coder.py:269-270).
struct BitWriter {
  uint32_t* words;
  uint64_t bitpos;
  uint64_t cap;
  uint32_t acc;  // pending bits of word bitpos>>5, MSB-aligned

  __device__ void open(uint32_t* w, uint64_t bp, uint64_t cap_words) {
    words = w;
    bitpos = bp;
    cap = cap_words;
    acc = ((bp & 31) && (bp >> 5) < cap) ? bswap32(w[bp >> 5]) : 0u;
  }
  __device__ __forceinline__ void store(uint64_t wi, uint32_t v) {
    if (wi < cap) words[wi] = bswap32(v);
  }
  __device__ __forceinline__ void put(uint32_t bit) {
    acc |= bit << (31 - (uint32_t)(bitpos & 31));
    ++bitpos;
    if ((bitpos & 31) == 0) {
      store((bitpos >> 5) - 1, acc);
      acc = 0;
    }
  }
  __device__ __forceinline__ void put_run(uint32_t bit, uint64_t n) {
    while (n) {
      uint32_t used = (uint32_t)(bitpos & 31);
      uint32_t room = 32 - used;
      uint32_t k = n < room ? (uint32_t)n : room;
      if (bit) {
        uint32_t ones = k == 32 ? 0xffffffffu : (((1u << k) - 1u) << (room - k));
        acc |= ones;
      }
      bitpos += k;
      n -= k;
      if ((bitpos & 31) == 0) {
        store((bitpos >> 5) - 1, acc);
        acc = 0;
      }
    }
  }
  __device__ void close() {
    if (bitpos & 31) store(bitpos >> 5, acc);
  }
};

struct EncState {
  uint64_t low, high, pending, bitpos;
};

// coder.py:133-161 for one symbol with interval [c_lo, c_hi) of 2^16
__device__ __forceinline__ void enc_symbol(EncState& st, BitWriter& w, uint32_t c_lo,
                                           uint32_t c_hi) {
  uint64_t low = st.low, high = st.high, pending = st.pending;
  uint64_t span = high - low + 1;
  high = low + ((span * c_hi) >> 16) - 1;
  low = low + ((span * c_lo) >> 16);
  for (;;) {
    uint32_t bit;
    if (high < kHalf) {
      bit = 0;
    } else if (low >= kHalf) {
      bit = 1;
      low -= kHalf;
      high -= kHalf;
    } else if (low >= kQuarter && high < kThreeQ) {
      ++pending;
      low = (low - kQuarter) << 1;
      high = ((high - kQuarter) << 1) | 1;
      continue;
    } else {
      break;
    }
    w.put(bit);
    if (pending) {
      w.put_run(bit ^ 1u, pending);
      pending = 0;
    }
    low <<= 1;
    high = (high << 1) | 1;
  }
  st.low = low;
  st.high = high;
  st.pending = pending;
}

// coder.py:290-306: first = (low >= QUARTER), then pending+1 copies of !first
__device__ __forceinline__ void enc_finish(EncState& st, BitWriter& w) {
  uint32_t first = st.low < kQuarter ? 0u : 1u;
  w.put(first);
  w.put_run(first ^ 1u, st.pending + 1);
  st.pending = 0;
}

struct DecState {
  uint64_t low, high, code;
  int64_t bitpos;
  int64_t cidx = -1;   // payload byte cached in cbyte (one load per 8 bits, not per bit)
  uint32_t cbyte = 0;
};

__device__ __forceinline__ uint32_t read_bit(const uint8_t* data, int64_t bit_length,
                                             int64_t bp) {
  return bp < bit_length ? (uint32_t)((data[bp >> 3] >> (7 - (bp & 7))) & 1) : 0u;
}

// Given the decoded symbol's interval, advance the decoder (coder.py:198-223).
// Returns false on exhaustion (bitpos beyond bit_length + 64).
__device__ __forceinline__ bool dec_advance(DecState& st, const uint8_t* data,
                                            int64_t bit_length, uint64_t span, uint32_t c_lo,
                                            uint32_t c_hi) {
  // low <= code <= high < 2^32 throughout (the coder's 32-bit registers), and
  // every shift below starts from a value < 2^31, so the renormalisation runs
  // in 32-bit registers (half the instructions of the 64-bit form on this
  // serial decode chain); only the interval update needs the 64-bit product
  uint32_t code = (uint32_t)st.code;
  uint32_t high = (uint32_t)(st.low + ((span * c_hi) >> 16) - 1);
  uint32_t low = (uint32_t)(st.low + ((span * c_lo) >> 16));
  constexpr uint32_t kH = (uint32_t)kHalf, kQ = (uint32_t)kQuarter, kTQ = (uint32_t)kThreeQ;
  int64_t bp = st.bitpos;
  const int64_t limit = bit_length + 64;
  for (;;) {
    if (high < kH) {
    } else if (low >= kH) {
      low -= kH;
      high -= kH;
      code -= kH;
    } else if (low >= kQ && high < kTQ) {
      low -= kQ;
      high -= kQ;
      code -= kQ;
    } else {
      break;
    }
    low <<= 1;
    high = (high << 1) | 1u;
    uint32_t bit = 0;
    if (bp < bit_length) {
      const int64_t bi = bp >> 3;
      if (bi != st.cidx) {
        st.cidx = bi;
        st.cbyte = data[bi];
      }
      bit = (st.cbyte >> (7 - (bp & 7))) & 1u;
    } else if (bp > limit) {
      st.bitpos = bp;
      return false;
    }
    ++bp;
    code = (code << 1) | bit;
  }
  st.low = low;
  st.high = high;
  st.code = code;
  st.bitpos = bp;
  return true;
}

// coder.py:186: value = ((code - low + 1) * TOTAL - 1) // span.  num < 2^49
// and span <= 2^32 are exact doubles; the correctly rounded quotient floors
// to the true quotient or one above it (rounding up across an integer), so
// one correction makes it exact -- instead of a 64-bit integer division on
// the decoder's serial critical path.
__device__ __forceinline__ uint64_t dec_value(const DecState& st, uint64_t span) {
  const uint64_t num = ((st.code - st.low + 1) << 16) - 1;
  uint64_t q = (uint64_t)((double)num / (double)span);
  if (q * span > num) --q;
  return q;
}

// Warp-cooperative symbol search: lane l holds cum[8l..8l+7] (cum[0] = 0).
// Returns the symbol s with cum[s] <= value < cum[s+1] and its interval.
__device__ __forceinline__ int warp_find_symbol(const uint32_t (&cum)[8], uint64_t value,
                                                uint32_t& c_lo, uint32_t& c_hi) {
  const int lane = threadIdx.x & 31;
  uint32_t nxt = __shfl_down_sync(0xffffffffu, cum[0], 1);
  if (lane == 31) nxt = (uint32_t)kTotal;
  unsigned ball = __ballot_sync(0xffffffffu, (uint64_t)cum[0] <= value);
  int owner = 31 - __clz(ball);
  int jl = 0;
#pragma unroll
  for (int j = 1; j < 8; ++j) jl += ((uint64_t)cum[j] <= value) ? 1 : 0;
  uint32_t lo = cum[0], hi = cum[1];
#pragma unroll
  for (int j = 1; j < 8; ++j) {
    if (jl == j) {
      lo = cum[j];
      hi = j < 7 ? cum[j + 1] : nxt;
    }
  }
  c_lo = __shfl_sync(0xffffffffu, lo, owner);
  c_hi = __shfl_sync(0xffffffffu, hi, owner);
  return owner * 8 + __shfl_sync(0xffffffffu, jl, owner);
}

}  // namespace edpc

// NumPy's pairwise summation order, restated for device code (bit-exact sums).
#pragma once
#include "ks_common.cuh"

namespace {
// ---------------------------------------------------------------- NumPy pairwise summation
// numpy/_core/src/umath/loops_utils.h.src pairwise_sum: n < 8 sequential from 0; n <= 128
// eight interleaved accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the
// remainder; otherwise split at n2 = n/2 rounded down to a multiple of 8.
constexpr int64_t PW_BLOCK = 128;

template <typename Get>
__device__ double pw_leaf(const Get& get, int64_t s, int64_t len) {
  if (len < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < len; i++) res += get(s + i);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; j++) r[j] = get(s + j);
  int64_t i = 8;
#pragma unroll 4
  for (; i < len - (len % 8); i += 8) {  // unrolled: several blocks' loads in flight
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] += get(s + i + j);
  }
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < len; i++) res += get(s + i);
  return res;
}

__device__ __forceinline__ void pw_split(int64_t len, int64_t* n2) {
  int64_t h = len / 2;
  *n2 = h - (h % 8);
}

// Sequential full recursion (explicit stack; depth <= 64).
template <typename Get>
__device__ double pw_sum_seq(const Get& get, int64_t s, int64_t len) {
  if (len <= PW_BLOCK) return pw_leaf(get, s, len);
  // post-order evaluation with an explicit stack of (start, len, state)
  int64_t st_s[64], st_l[64];
  double st_v[64];
  int st_state[64];
  int sp = 0;
  st_s[0] = s; st_l[0] = len; st_state[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    const int64_t cs = st_s[sp], cl = st_l[sp];
    if (cl <= PW_BLOCK) {
      ret = pw_leaf(get, cs, cl);
      sp--;
      if (sp >= 0) {
        if (st_state[sp] == 1) { st_v[sp] = ret; st_state[sp] = 2; }
        else { ret = st_v[sp] + ret; st_state[sp] = 3; }
      }
      continue;
    }
    int64_t n2;
    pw_split(cl, &n2);
    if (st_state[sp] == 0) {
      st_state[sp] = 1;
      sp++;
      st_s[sp] = cs; st_l[sp] = n2; st_state[sp] = 0;
    } else if (st_state[sp] == 2) {
      sp++;
      st_s[sp] = cs + n2; st_l[sp] = cl - n2; st_state[sp] = 0;
    } else {  // state 3: both children done, `ret` holds the sum
      sp--;
      if (sp >= 0) {
        if (st_state[sp] == 1) { st_v[sp] = ret; st_state[sp] = 2; }
        else { ret = st_v[sp] + ret; st_state[sp] = 3; }
      }
    }
  }
  return ret;
}

}  // namespace

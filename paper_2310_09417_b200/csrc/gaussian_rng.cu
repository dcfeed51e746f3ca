// Device draw of numpy's Generator(Philox(key=[seed, stream])).standard_normal
// -- the sketch embedding Omega of `make_gaussian` (`sketching.py:191-204`)
// without the host RNG (SURVEY.md 8f "next #1").
//
// numpy's ziggurat consumes a variable number of 64-bit words per normal
// (1 on the fast path, 98.5%; 2 per wedge test; 3+ for the tail), so the
// word -> normal mapping is resolved in parallel:
//   A  every word position p is evaluated as if an attempt started there:
//      next[p] (offset of the next attempt), end[p] (does the normal end),
//      val[p] (its value) -- Philox4x64-10 is counter based, so any word is
//      directly computable;
//   B  the stream is cut into segments of SEG positions; one warp per
//      segment stages its next/end bytes in shared memory and, for each of
//      ENTRY possible entry offsets, walks the chain 32 positions at a time
//      (pointer doubling over shuffles gives a window's visited set in five
//      rounds) and records (normals ended, exit offset); chains merge within
//      a few words, so entries > 0 stop where they meet chain 0;
//   C  every segment's actual entry follows from its predecessor's exit (all
//      entries exit alike for almost every segment), then a one-CTA prefix
//      sum gives each segment's first output index;
//   D  each segment's warp walks its real chain once more and writes its
//      normals, a window at a time, divided by `scale` (the reference's
//      `omega /= np.sqrt(ell)`).
// Fast-path values are exact products (rabs * wi[idx]).  The tail uses
// libm_log1p (libm_log1p.cuh), a rounding-exact restatement of the host
// libm's log1p, so tail values are bit-identical too.  The wedge test
// compares against CUDA exp(), which is within 1 ulp of glibc's: a decision
// can only differ when the two sides are within 1 ulp (probability ~1e-16
// per wedge event); tests/test_gpu_rng.py checks bit equality with numpy.
#include "common.cuh"
#include "rskel_internal.h"
#include "ziggurat_tables.h"
#include "libm_log1p.cuh"

namespace rs {

constexpr int SEG = 1024;     // word positions per segment (32 windows of 32)
constexpr int ENTRY = 16;     // supported entry offsets into a segment
constexpr int RNG_T = 256;

struct U128 {
  uint64_t hi, lo;
};

RS_DEV void philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3, uint64_t k0, uint64_t k1,
                          uint64_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
    const uint64_t lo1 = 0xCA5A826395121157ull * c2, hi1 = __umul64hi(0xCA5A826395121157ull, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// Word p of the stream: block p/4 uses counter (p/4 + 1) (numpy pre-increments).
RS_DEV uint64_t philox_word(uint64_t p, uint64_t k0, uint64_t k1) {
  const uint64_t blk = (p >> 2) + 1;
  uint64_t o[4];
  philox4x64_10(blk, 0, 0, 0, k0, k1, o);
  return o[p & 3];
}

RS_DEV double word_double(uint64_t w) { return (double)(w >> 11) * (1.0 / 9007199254740992.0); }

constexpr double ZIG_R = 3.6541528853610088;
constexpr double ZIG_INV_R = 0.27366123732975828;

// Pass A: one attempt starting at every position.
__global__ void rng_attempt_kernel(uint64_t k0, uint64_t k1, long long P, uint8_t* __restrict__ next,
                                   uint8_t* __restrict__ ends, double* __restrict__ val) {
  // ki / wi looked up per word with 32 different indices per warp: from
  // shared memory (constant memory serialises divergent indices)
  __shared__ uint64_t s_ki[256], s_wi[256];
  for (int e = threadIdx.x; e < 256; e += blockDim.x) {
    s_ki[e] = zig_ki[e];
    s_wi[e] = zig_wi_bits[e];
  }
  __syncthreads();
  const long long base = 4LL * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
  if (base >= P) return;
  uint64_t w[4];
  philox4x64_10((uint64_t)(base >> 2) + 1, 0, 0, 0, k0, k1, w);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const long long p = base + q;
    if (p >= P) break;
    uint64_t r = w[q];
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const bool neg = r & 1;
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * __longlong_as_double((long long)s_wi[idx]);
    if (neg) x = -x;
    uint8_t nx = 1, en = 1;
    if (rabs >= s_ki[idx]) {
      if (idx == 0) {  // tail: pairs of doubles until accepted
        long long s = p + 1;
        double xx, yy;
        for (;;) {
          xx = __dmul_rn(-ZIG_INV_R, libm_log1p(-word_double(philox_word((uint64_t)s, k0, k1))));
          yy = -libm_log1p(-word_double(philox_word((uint64_t)s + 1, k0, k1)));
          s += 2;
          if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) break;
        }
        x = ((rabs >> 8) & 1) ? -__dadd_rn(ZIG_R, xx) : __dadd_rn(ZIG_R, xx);
        const long long d = s - p;
        nx = d > 255 ? 255 : (uint8_t)d;
      } else {  // wedge
        const double fi_m = __longlong_as_double((long long)zig_fi_bits[idx - 1]);
        const double fi_i = __longlong_as_double((long long)zig_fi_bits[idx]);
        const double u = word_double(philox_word((uint64_t)p + 1, k0, k1));
        nx = 2;
        // numpy's distributions.c is built without FMA contraction: round each op
        en = (__dadd_rn(__dmul_rn(__dsub_rn(fi_m, fi_i), u), fi_i) < exp(__dmul_rn(__dmul_rn(-0.5, x), x))) ? 1 : 0;
      }
    }
    next[p] = nx;
    ends[p] = en;
    val[p] = x;
  }
}

// Warp-collective walk of one 32-position window of a segment held in shared
// memory: lane i starts an attempt chain at offset i; five pointer-doubling
// rounds give every lane the set of offsets its chain visits in the window
// (R) and the first offset past the window (J >= 32).  The caller reads the
// lane where the real chain enters.
struct WinWalk {
  unsigned vis;  // offsets visited (bit i = offset i)
  int exit;      // first offset >= 32 reached (relative to the window start)
};

RS_DEV WinWalk window_walk(const uint8_t* __restrict__ nxt_s, int win, int s0, int lane) {
  int J = lane + (int)nxt_s[win * 32 + lane];
  unsigned R = 1u << lane;
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const int src = J < 32 ? J : 31;
    const unsigned Rj = __shfl_sync(0xffffffffu, R, src);
    const int Jj = __shfl_sync(0xffffffffu, J, src);
    if (J < 32) {
      R |= Rj;
      J = Jj;
    }
  }
  WinWalk w;
  w.vis = __shfl_sync(0xffffffffu, R, s0);
  w.exit = __shfl_sync(0xffffffffu, J, s0);
  return w;
}

constexpr int SEG_WARPS = 4;

// Stage a segment's next/ends bytes into this warp's shared slice (positions
// past P read as fast-path non-ends: next 1, ends 0).
RS_DEV void stage_segment(long long p0, long long P, const uint8_t* __restrict__ next,
                          const uint8_t* __restrict__ ends, uint8_t* nxt_s, uint8_t* end_s, int lane) {
  if (p0 + SEG <= P) {
    const uint4* n4 = reinterpret_cast<const uint4*>(next + p0);
    const uint4* e4 = reinterpret_cast<const uint4*>(ends + p0);
    uint4* ns4 = reinterpret_cast<uint4*>(nxt_s);
    uint4* es4 = reinterpret_cast<uint4*>(end_s);
#pragma unroll
    for (int i = lane; i < SEG / 16; i += 32) {
      ns4[i] = n4[i];
      es4[i] = e4[i];
    }
  } else {
    for (int i = lane; i < SEG; i += 32) {
      const bool in = p0 + i < P;
      nxt_s[i] = in ? next[p0 + i] : 1;
      end_s[i] = in ? ends[p0 + i] : 0;
    }
  }
  __syncwarp();
}

// Pass B (one warp per segment): for each entry offset e < ENTRY, the number
// of normals the chain entering at e ends inside the segment and its exit
// offset into the next segment.  Chains merge within a few words, so entries
// e > 0 stop at the first offset shared with chain 0 and inherit its tail.
__global__ void __launch_bounds__(32 * SEG_WARPS) rng_segment_kernel(
    long long P, int nseg, const uint8_t* __restrict__ next, const uint8_t* __restrict__ ends,
    int* __restrict__ seg_count, uint8_t* __restrict__ seg_exit, uint8_t* __restrict__ seg_uniform,
    int* __restrict__ overflow) {
  __shared__ __align__(16) uint8_t nxt_sh[SEG_WARPS][SEG];
  __shared__ __align__(16) uint8_t end_sh[SEG_WARPS][SEG];
  __shared__ unsigned vis0_sh[SEG_WARPS][SEG / 32];
  __shared__ int cnt0_sh[SEG_WARPS][SEG / 32];  // chain-0 normals ended before window w
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * SEG_WARPS + wid;
  if (s >= nseg) return;
  const long long p0 = (long long)s * SEG;
  uint8_t* nxt_s = nxt_sh[wid];
  uint8_t* end_s = end_sh[wid];
  stage_segment(p0, P, next, ends, nxt_s, end_s, lane);
  if (lane < SEG / 32) vis0_sh[wid][lane] = 0u;
  __syncwarp();
  // chain 0: full walk, remembering visited masks and running counts
  int pos = 0, cnt0 = 0;
  while (pos < SEG) {
    const int win = pos >> 5;
    const WinWalk w = window_walk(nxt_s, win, pos & 31, lane);
    const unsigned E = __ballot_sync(0xffffffffu, end_s[win * 32 + lane] != 0);
    if (lane == 0) {
      vis0_sh[wid][win] = w.vis;
      cnt0_sh[wid][win] = cnt0;
    }
    cnt0 += __popc(w.vis & E);
    pos = win * 32 + w.exit;
  }
  __syncwarp();
  const int ex0 = pos - SEG;
  bool uniform = true;
  for (int e = 0; e < ENTRY; ++e) {
    int cnt = cnt0, ex = ex0;
    if (e > 0) {
      int p = e, c = 0;
      cnt = -1;
      while (p < SEG) {
        const int win = p >> 5;
        const WinWalk w = window_walk(nxt_s, win, p & 31, lane);
        const unsigned E = __ballot_sync(0xffffffffu, end_s[win * 32 + lane] != 0);
        const unsigned common = w.vis & vis0_sh[wid][win];
        if (common) {  // merged with chain 0 at offset q: inherit its tail
          const int q = __ffs(common) - 1;
          const unsigned below = (1u << q) - 1u;
          c += __popc(w.vis & E & below);
          cnt = c + (cnt0 - cnt0_sh[wid][win] - __popc(vis0_sh[wid][win] & E & below));
          ex = ex0;
          break;
        }
        c += __popc(w.vis & E);
        p = win * 32 + w.exit;
      }
      if (cnt < 0) {  // never merged: own exit
        cnt = c;
        ex = p - SEG;
      }
    }
    if (lane == 0) {
      if (ex >= ENTRY) atomicOr(overflow, 1);
      seg_count[s * ENTRY + e] = cnt;
      seg_exit[s * ENTRY + e] = (uint8_t)(ex < ENTRY ? ex : ENTRY - 1);
    }
    if (ex != ex0) uniform = false;
  }
  if (lane == 0) seg_uniform[s] = uniform ? 1 : 0;
}

// Pass C: entry offset of every segment.  Segment s enters where segment s-1
// exits; if s-1 is uniform that is known directly, otherwise compose forward
// from the last uniform segment (rare, short runs).
__global__ void rng_entry_kernel(int nseg, const int* __restrict__ seg_count, const uint8_t* __restrict__ seg_exit,
                                 const uint8_t* __restrict__ seg_uniform, int* __restrict__ seg_entry,
                                 long long* __restrict__ seg_cnt) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  int e = 0;
  if (s > 0) {
    int t = s - 1;
    while (t > 0 && !seg_uniform[t]) --t;
    if (seg_uniform[t] || t > 0) {
      e = seg_exit[t * ENTRY];  // uniform: any entry gives this exit
    } else {
      e = seg_exit[0 * ENTRY + 0];  // t == 0, entry of segment 0 is 0
    }
    for (int u = t + 1; u < s; ++u) e = seg_exit[u * ENTRY + e];
  }
  seg_entry[s] = e;
  seg_cnt[s] = seg_count[s * ENTRY + e];
}

// Pass D: exclusive prefix sum of seg_cnt in place (one CTA, fixed order).
__global__ void rng_prefix_kernel(int nseg, long long* __restrict__ seg_cnt) {
  __shared__ long long part[RNG_T];
  const int per = (nseg + RNG_T - 1) / RNG_T;
  const int a = threadIdx.x * per, b = min(nseg, a + per);
  long long sum = 0;
  for (int i = a; i < b; ++i) sum += seg_cnt[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = 0;
    for (int i = 0; i < RNG_T; ++i) {
      const long long v = part[i];
      part[i] = run;
      run += v;
    }
  }
  __syncthreads();
  long long run = part[threadIdx.x];
  for (int i = a; i < b; ++i) {
    const long long v = seg_cnt[i];
    seg_cnt[i] = run;
    run += v;
  }
}

// Pass E (one warp per segment): walk the real chain from the segment's entry
// and write its normals; a window's outputs go out in parallel, indexed by a
// popcount of the visited-and-ended mask.
__global__ void __launch_bounds__(32 * SEG_WARPS) rng_emit_kernel(
    long long P, int nseg, long long N, const uint8_t* __restrict__ next, const uint8_t* __restrict__ ends,
    const double* __restrict__ val, const int* __restrict__ seg_entry, const long long* __restrict__ seg_base,
    double scale, double* __restrict__ out) {
  __shared__ __align__(16) uint8_t nxt_sh[SEG_WARPS][SEG];
  __shared__ __align__(16) uint8_t end_sh[SEG_WARPS][SEG];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * SEG_WARPS + wid;
  if (s >= nseg) return;
  const long long p0 = (long long)s * SEG;
  uint8_t* nxt_s = nxt_sh[wid];
  uint8_t* end_s = end_sh[wid];
  stage_segment(p0, P, next, ends, nxt_s, end_s, lane);
  long long o = seg_base[s];
  int pos = seg_entry[s];
  while (pos < SEG && o < N) {
    const int win = pos >> 5;
    const WinWalk w = window_walk(nxt_s, win, pos & 31, lane);
    const unsigned E = __ballot_sync(0xffffffffu, end_s[win * 32 + lane] != 0);
    const unsigned take = w.vis & E;
    if ((take >> lane) & 1u) {
      const long long oi = o + __popc(take & ((1u << lane) - 1u));
      if (oi < N) {
        const double x = val[p0 + win * 32 + lane];
        out[oi] = scale == 1.0 ? x : x / scale;
      }
    }
    o += __popc(take);
    pos = win * 32 + w.exit;
  }
}

static long long rng_positions(long long N) {  // 6.25% slack over the 2.2% average overshoot
  const long long P = N + N / 16 + 4096;
  return (P + SEG - 1) / SEG * SEG;
}

size_t gaussian_workspace_bytes(long long N) {
  const long long P = rng_positions(N);
  const long long nseg = P / SEG;
  return (size_t)P * (8 + 1 + 1) + (size_t)nseg * (ENTRY * 4 + ENTRY + 1 + 4 + 8) + 4096;
}

// Returns RS_OK; *status_dev gets 0, or 1 if a chain crossed a segment
// boundary by >= ENTRY words (never observed; the caller then draws on the host).
int launch_gaussian(uint64_t seed, uint64_t stream, long long N, double scale, double* out, void* ws,
                    size_t ws_bytes, int* status_dev, cudaStream_t st) {
  if (N < 0) return RS_ERR_ARG;
  if (N == 0) return RS_OK;
  const long long P = rng_positions(N);
  const int nseg = (int)(P / SEG);
  if (gaussian_workspace_bytes(N) > ws_bytes) return RS_ERR_CAPACITY;
  // 16-byte aligned: val, next, ends (P is a multiple of SEG), then the
  // per-segment arrays, widest first.
  char* w = static_cast<char*>(ws);
  double* val = reinterpret_cast<double*>(w);
  w += (size_t)P * 8;
  uint8_t* next = reinterpret_cast<uint8_t*>(w);
  w += (size_t)P;
  uint8_t* ends = reinterpret_cast<uint8_t*>(w);
  w += (size_t)P;
  long long* seg_cnt = reinterpret_cast<long long*>(w);
  w += (size_t)nseg * 8;
  int* seg_count = reinterpret_cast<int*>(w);
  w += (size_t)nseg * ENTRY * 4;
  int* seg_entry = reinterpret_cast<int*>(w);
  w += (size_t)nseg * 4;
  uint8_t* seg_exit = reinterpret_cast<uint8_t*>(w);
  w += (size_t)nseg * ENTRY;
  uint8_t* seg_uniform = reinterpret_cast<uint8_t*>(w);
  cudaMemsetAsync(status_dev, 0, sizeof(int), st);
  const long long nthr = (P + 3) / 4;
  rng_attempt_kernel<<<(unsigned)((nthr + RNG_T - 1) / RNG_T), RNG_T, 0, st>>>(seed, stream, P, next, ends, val);
  const unsigned seg_grid = (unsigned)((nseg + SEG_WARPS - 1) / SEG_WARPS);
  rng_segment_kernel<<<seg_grid, 32 * SEG_WARPS, 0, st>>>(P, nseg, next, ends, seg_count, seg_exit, seg_uniform,
                                                          status_dev);
  rng_entry_kernel<<<(nseg + RNG_T - 1) / RNG_T, RNG_T, 0, st>>>(nseg, seg_count, seg_exit, seg_uniform,
                                                                  seg_entry, seg_cnt);
  rng_prefix_kernel<<<1, RNG_T, 0, st>>>(nseg, seg_cnt);
  rng_emit_kernel<<<seg_grid, 32 * SEG_WARPS, 0, st>>>(P, nseg, N, next, ends, val, seg_entry, seg_cnt, scale,
                                                       out);
  count_launch(5);
  return cudaGetLastError() == cudaSuccess ? RS_OK : RS_ERR_CUDA;
}

}  // namespace rs

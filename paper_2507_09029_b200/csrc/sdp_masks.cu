// Block-assignment and mask builder (masking.py:56-359) on the device.
//
//   k_assign       one CTA: SeedSequence -> PCG64 stream generated in parallel
//                  (affine jump-ahead) -> Fisher-Yates as warp-speculative
//                  rejection draws + chain-walk final positions -> cyclic
//                  windows (masking.py:56-117); bit-exact with numpy.
//   k_build_masks  HBM-bound expansion: every element ANDs the owner sets of
//                  the units that govern it (masking.py:131-149, 160-169) and
//                  emits owner mask / [N,d] bool / coverage / divisor /
//                  governors / per-worker counts.
//   k_plan_tiles   warp-per-tile AND/OR shuffle reduction: which tiles have one
//                  owner set (block strategy: nearly all) for the sync kernel.
#include "sdp_common.cuh"

namespace sdp {

// ---------------------------------------------------------------------------
// numpy SeedSequence + PCG64 restated (oracle/oracle.py)
// ---------------------------------------------------------------------------
typedef unsigned __int128 u128;

struct Pcg64 {
  u128 state, inc;
  uint32_t half;
  bool has_half;

  __device__ void step() {
    const u128 mult = (static_cast<u128>(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;
    state = state * mult + inc;
  }
  __device__ uint64_t raw() {
    step();
    uint64_t hi = static_cast<uint64_t>(state >> 64);
    uint64_t lo = static_cast<uint64_t>(state);
    uint32_t rot = static_cast<uint32_t>(hi >> 58);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __device__ uint32_t next32() {
    if (has_half) {
      has_half = false;
      return half;
    }
    uint64_t x = raw();
    half = static_cast<uint32_t>(x >> 32);
    has_half = true;
    return static_cast<uint32_t>(x);
  }
  // numpy random_interval: masked rejection, 32-bit draws when max fits.
  __device__ uint64_t interval(uint64_t mx) {
    if (mx == 0) return 0;
    uint64_t mask = mx;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    if (mx <= 0xFFFFFFFFull) {
      uint32_t m32 = static_cast<uint32_t>(mask), v;
      while ((v = (next32() & m32)) > mx) {}
      return v;
    }
    uint64_t v;
    while ((v = (raw() & mask)) > mx) {}
    return v;
  }
};

__device__ void seed_pcg(Pcg64& g, const uint32_t* ent, int n_ent) {
  const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u;
  const uint32_t INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= MULT_A;
    v *= hc;
    return v ^ (v >> 16);
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int k = 4; k < n_ent; ++k)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[k]));
  uint32_t hb = INIT_B, w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t d = pool[i & 3] ^ hb;
    hb *= MULT_B;
    d *= hb;
    w[i] = d ^ (d >> 16);
  }
  uint64_t v0 = w[0] | (static_cast<uint64_t>(w[1]) << 32);
  uint64_t v1 = w[2] | (static_cast<uint64_t>(w[3]) << 32);
  uint64_t v2 = w[4] | (static_cast<uint64_t>(w[5]) << 32);
  uint64_t v3 = w[6] | (static_cast<uint64_t>(w[7]) << 32);
  u128 initstate = (static_cast<u128>(v0) << 64) | v1;
  u128 initseq = (static_cast<u128>(v2) << 64) | v3;
  g.inc = (initseq << 1) | 1;
  g.state = 0;
  g.step();
  g.state += initstate;
  g.step();
  g.has_half = false;
  g.half = 0;
}

struct SeedWords {
  uint32_t w[8];
  int n;
};

// Workers of slot j: {(j*P + t) mod N : t < P} as a bitmask = the low P bits
// rotated left by (j*P) mod N inside an N-bit ring (masking.py:63-65).
__device__ __forceinline__ uint64_t window_bits(uint64_t slot, int n, int p) {
  const uint64_t full = n == 64 ? ~0ull : ((1ull << n) - 1);
  const uint64_t low = p == 64 ? ~0ull : ((1ull << p) - 1);
  const uint32_t start = (static_cast<uint32_t>(slot % static_cast<uint64_t>(n)) * static_cast<uint32_t>(p)) %
                         static_cast<uint32_t>(n);
  if (start == 0) return low;
  return ((low << start) | (low >> (n - start))) & full;
}

// ---- PCG64 stream generated in parallel ------------------------------------
// The LCG step x -> M x + inc (mod 2^128) is affine, so k steps are the affine
// map (M^k, inc (M^(k-1) + ... + 1)): every thread jumps to its own offset by
// binary exponentiation and then steps through its slice of the stream.
struct Affine128 {
  u128 a, c;  // x -> a x + c
};

__device__ __forceinline__ Affine128 compose(const Affine128& f, const Affine128& g) {  // f after g
  return {f.a * g.a, f.a * g.c + f.c};
}

__device__ __forceinline__ u128 pcg_mult() {
  return (static_cast<u128>(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;
}

__device__ __forceinline__ u128 jump(u128 x, u128 inc, uint64_t k) {
  Affine128 r{1, 0}, b{pcg_mult(), inc};
  while (k) {
    if (k & 1) r = compose(b, r);
    b = compose(b, b);
    k >>= 1;
  }
  return r.a * x + r.c;
}

__device__ __forceinline__ uint64_t pcg_output(u128 state) {  // XSL-RR
  const uint64_t hi = static_cast<uint64_t>(state >> 64), lo = static_cast<uint64_t>(state);
  const uint32_t rot = static_cast<uint32_t>(hi >> 58);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

constexpr int kAssignThreads = 1024;
constexpr int kAssignWords = 8192;               // 32-bit words per refill (4096 raw draws)
constexpr int kRawPerThread = kAssignWords / 2 / kAssignThreads;

// words[2k], words[2k+1] = low, high half of the k-th next 64-bit output after
// *state (numpy's buffered 32-bit draws consume them in exactly this order);
// *state advances by kAssignWords / 2 steps.  Whole CTA.
__device__ void refill_words(uint32_t* words, u128* state, u128 inc) {
  const u128 base = *state;
  u128 x = jump(base, inc, static_cast<uint64_t>(threadIdx.x) * kRawPerThread);
  const u128 m = pcg_mult();
  for (int s = 0; s < kRawPerThread; ++s) {
    x = m * x + inc;
    const uint64_t out = pcg_output(x);
    const int k = threadIdx.x * kRawPerThread + s;
    words[2 * k] = static_cast<uint32_t>(out);
    words[2 * k + 1] = static_cast<uint32_t>(out >> 32);
  }
  __syncthreads();  // everyone has read *state
  if (threadIdx.x == kAssignThreads - 1) *state = x;
  __syncthreads();
}

// Block-wide exclusive scan of cnt[0..n) into start[0..n] (start[n] = total).
__device__ void block_exclusive_scan(const int32_t* cnt, int32_t* start, int n, int32_t* s_warp) {
  const int per = (n + kAssignThreads - 1) / kAssignThreads;
  const int b = threadIdx.x * per, e = min(n, b + per);
  int local = 0;
  for (int k = b; k < e; ++k) local += cnt[k];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kAssignThreads / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kAssignThreads / 32) s_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  int run = (warp > 0 ? s_warp[warp - 1] : 0) + incl - local;
  for (int k = b; k < e; ++k) {
    start[k] = run;
    run += cnt[k];
  }
  if (threadIdx.x == kAssignThreads - 1) start[n] = s_warp[kAssignThreads / 32 - 1];
  __syncthreads();
}

// One CTA.  numpy's Generator.shuffle of arange(n) per group (one generator
// across groups, masking.py:107-116) in two parallel phases:
//  (A) per group, in stream order: the masked rejection draws j_i for
//      i = n-1..1 (numpy random_interval) depend on the 32-bit word stream
//      and i only.  Warp 0 takes 32 words at a time: with a_k accepted draws
//      before lane k (a_k <= k), lane k is surely accepted when v_k <= i - k,
//      surely rejected when v_k > i, and only the first lane in between is
//      resolved exactly (ballot + popc); a batch is cut where the mask (set by
//      i's bit length) would change.  Every step records its target as a
//      global unit position: js[first + i] = first + j_i.
//  (B) once, over all groups: the swaps a[i] <-> a[j_i] are evaluated without
//      running them.  The content of position x right before step i is set
//      by the most recent earlier step (the smallest step index > i) that
//      targeted x, so with the steps bucketed by target (counting sort) each
//      final a[i] is a short chain walk:
//        a[i] = g(nxt(i)) if a step s > i has j_s = j_i (nxt = the smallest),
//               else j_i;   a[0] = g(npos(0)), else 0;
//        g(y) = g(npos(y)) if a step s > y has j_s = y (npos = the smallest),
//               else y.
// The PCG64 stream is generated cooperatively into shared memory (affine
// jump-ahead per thread).  scratch: 8 x n_units int32 (device).
__global__ void __launch_bounds__(kAssignThreads)
k_assign(SeedWords seed, const sdp_group_desc* __restrict__ groups, int n_groups, int n_units,
         int n_workers, int replication, uint64_t* __restrict__ unit_bits, int32_t* __restrict__ scratch) {
  extern __shared__ __align__(16) uint32_t s_dyn[];
  uint32_t* words = s_dyn;
  __shared__ u128 s_state, s_inc;
  __shared__ int s_p, s_i;
  __shared__ int32_t s_warp[kAssignThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nu = n_units;
  int32_t* js = scratch;              // step target (global position); -1 group first, -2 no group
  int32_t* slot_of = scratch + nu;    // window slot of each position
  int32_t* cnt = scratch + 2 * nu;    // bucket sizes, then fill cursors, then results
  int32_t* start = scratch + 3 * nu;  // [nu + 1]
  int32_t* bucket = scratch + 4 * nu + 1;
  int32_t* nxt = scratch + 5 * nu + 1;
  int32_t* npos = scratch + 6 * nu + 1;
  int32_t* res = cnt;
  const uint64_t full = n_workers == 64 ? ~0ull : ((1ull << n_workers) - 1);
  for (int u = threadIdx.x; u < nu; u += blockDim.x) {
    unit_bits[u] = full;
    js[u] = -2;
  }
  if (threadIdx.x == 0) {
    Pcg64 g;
    seed_pcg(g, seed.w, seed.n);
    s_state = g.state;
    s_inc = g.inc;
    s_p = 0;
  }
  __syncthreads();
  const u128 inc = s_inc;
  refill_words(words, &s_state, inc);
  // ---- (A) draws, group by group in stream order ---------------------------
  // the first kGroupStage group descriptors are staged in shared memory with
  // one parallel load (not a dependent global round trip per group)
  constexpr int kGroupStage = 512;
  __shared__ int2 s_groups[kGroupStage];
  for (int g = threadIdx.x; g < min(n_groups, kGroupStage); g += blockDim.x)
    s_groups[g] = make_int2(groups[g].first_unit, groups[g].size);
  __syncthreads();
  int slot = 0;
  for (int gi = 0; gi < n_groups; ++gi) {
    const int2 gd = gi < kGroupStage ? s_groups[gi] : make_int2(groups[gi].first_unit, groups[gi].size);
    const int first = gd.x, n = gd.y;
    for (int k = threadIdx.x; k < n; k += blockDim.x) slot_of[first + k] = slot + k;
    // every thread has read the previous group's s_i (its loop exit test)
    // before thread 0 resets it (compute-sanitizer racecheck / synccheck)
    __syncthreads();
    if (threadIdx.x == 0) {
      js[first] = -1;
      s_i = n - 1;
    }
    slot += n;
    __syncthreads();
    while (true) {
      if (warp == 0) {
        int i = s_i, p = s_p;
        while (i > 0 && p < kAssignWords) {
          const uint32_t m = 0xffffffffu >> __clz(i);
          const int lo = static_cast<int>((m >> 1) + 1);  // smallest i with this mask
          const int B = min(min(32, kAssignWords - p), i - lo + 1);
          uint32_t v = 0;
          int t = -1;
          if (lane < B) {
            v = words[p + lane] & m;
            t = i - static_cast<int>(v);
          }
          // classify every lane against the bounds on a_k (accepted draws
          // before lane k), then resolve the undecided lanes one by one from
          // the lowest, re-classifying the rest with the tightened bounds
          const uint32_t live = B >= 32 ? 0xffffffffu : ((1u << B) - 1u);
          uint32_t acc = __ballot_sync(0xffffffffu, lane < B && t >= lane);       // sure accepts
          uint32_t dec = acc | (__ballot_sync(0xffffffffu, t < 0) & live);      // decided lanes
          int u = -1;  // lanes <= u are resolved exactly
          while (dec != live) {
            const uint32_t und = live & ~dec;
            const int k = __ffs(und) - 1;            // lowest undecided lane: its a_k is exact
            const uint32_t below = (1u << k) - 1u;
            const int tk = __shfl_sync(0xffffffffu, t, k);
            if (__popc(acc & below) <= tk) acc |= 1u << k;
            u = k;
            dec |= (1u << k) | below;
            // lanes above k: a in [A, A + (lane - k - 1)], A = accepted up to k
            const int A = __popc(acc & (below | (1u << k)));
            const bool hi = lane > k && ((und >> lane) & 1u);
            const uint32_t sa = __ballot_sync(0xffffffffu, hi && A + (lane - k - 1) <= t);
            const uint32_t sr = __ballot_sync(0xffffffffu, hi && A > t);
            acc |= sa;
            dec |= sa | sr;
          }
          (void)u;
          int consumed = B;
          if (__popc(acc) >= i) {  // the group's last draw: stop right after it
            uint32_t a2 = acc;
            for (int q = 1; q < i; ++q) a2 &= a2 - 1;  // the i-th accepted lane is now lowest
            const int last = __ffs(a2) - 1;
            acc &= last >= 31 ? 0xffffffffu : ((1u << (last + 1)) - 1u);
            consumed = last + 1;
          }
          if ((acc >> lane) & 1u) js[first + i - __popc(acc & ((1u << lane) - 1u))] = first + static_cast<int32_t>(v);
          i -= __popc(acc);
          p += consumed;
        }
        __syncwarp();  // every lane of warp 0 read s_i / s_p at the top
        if (lane == 0) {
          s_i = i;
          s_p = p;
        }
      }
      __syncthreads();
      if (s_i == 0) break;
      refill_words(words, &s_state, inc);  // the stream ran out mid-group
      if (threadIdx.x == 0) s_p = 0;
      __syncthreads();
    }
  }
  // ---- (B) final positions, all groups at once -----------------------------
  for (int k = threadIdx.x; k < nu; k += blockDim.x) cnt[k] = 0;
  __syncthreads();
  for (int q = threadIdx.x; q < nu; q += blockDim.x)
    if (js[q] >= 0) atomicAdd(&cnt[js[q]], 1);
  __syncthreads();
  block_exclusive_scan(cnt, start, nu, s_warp);
  for (int k = threadIdx.x; k < nu; k += blockDim.x) cnt[k] = 0;
  __syncthreads();
  for (int q = threadIdx.x; q < nu; q += blockDim.x) {
    const int x = js[q];
    if (x >= 0) bucket[start[x] + atomicAdd(&cnt[x], 1)] = q;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nu; k += blockDim.x) {
    // npos(k): smallest step > k targeting k;  nxt(k): smallest step > k targeting j_k
    int bp = 0x7fffffff;
    for (int q = start[k]; q < start[k + 1]; ++q) {
      const int c = bucket[q];
      if (c > k && c < bp) bp = c;
    }
    npos[k] = bp == 0x7fffffff ? -1 : bp;
    int bn = 0x7fffffff;
    const int x = js[k];
    if (x >= 0)
      for (int q = start[x]; q < start[x + 1]; ++q) {
        const int c = bucket[q];
        if (c > k && c < bn) bn = c;
      }
    nxt[k] = bn == 0x7fffffff ? -1 : bn;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nu; k += blockDim.x) {
    const int x = js[k];
    if (x == -2) continue;  // not in any group
    int y = x == -1 ? npos[k] : nxt[k];
    int r;
    if (y < 0) {
      r = x == -1 ? k : x;
    } else {
      while (npos[y] >= 0) y = npos[y];
      r = y;
    }
    res[k] = r;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < nu; k += blockDim.x)
    if (js[k] != -2) unit_bits[res[k]] = window_bits(slot_of[k], n_workers, replication);
}

__global__ void k_permutation(SeedWords seed, const int32_t* skip_sizes_dev, int n_skip, int n,
                              int32_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Pcg64 g;
  seed_pcg(g, seed.w, seed.n);
  for (int s = 0; s < n_skip; ++s)
    for (int i = skip_sizes_dev[s] - 1; i > 0; --i) (void)g.interval(static_cast<uint64_t>(i));
  for (int i = 0; i < n; ++i) out[i] = i;
  for (int i = n - 1; i > 0; --i) {
    int j = static_cast<int>(g.interval(static_cast<uint64_t>(i)));
    int32_t t = out[i];
    out[i] = out[j];
    out[j] = t;
  }
}

// ---------------------------------------------------------------------------
// element expansion
// ---------------------------------------------------------------------------
constexpr int kBuildThreads = 256;
constexpr int kStepElems = 256;  // elements a warp writes per grid-stride step

__device__ __forceinline__ int find_param(const sdp_param_desc* __restrict__ p, int n, int64_t j) {
  int lo = 0, hi = n - 1;  // last param with offset <= j
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (p[mid].offset <= j) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint32_t mul, uint32_t shr) {
  return mul ? (__umulhi(n, mul) >> shr) : n;
}

// The parameter an element falls in, with its owner set precomputed when no
// rule varies along the parameter (block rules, dim == 1: the whole block
// strategy and every ungoverned tensor) -- then an element costs no rule walk.
struct ParamCursor {
  int pi;
  int64_t lo, hi;       // [offset, offset + size)
  int32_t rule_begin, rule_count;
  bool uniform;
  uint64_t bits;

  __device__ void load(const sdp_param_desc* __restrict__ params, const sdp_rule_desc* __restrict__ rules,
                       const uint64_t* __restrict__ unit_bits, uint64_t full, int i) {
    const sdp_param_desc pd = params[i];
    pi = i;
    lo = pd.offset;
    hi = pd.offset + pd.size;
    rule_begin = pd.rule_begin;
    rule_count = pd.rule_count;
    uniform = true;
    bits = full;
    for (int r = 0; r < rule_count; ++r) {
      const sdp_rule_desc rd = rules[rule_begin + r];
      if (rd.dim != 1) {
        uniform = false;
        break;
      }
      bits &= __ldg(unit_bits + rd.unit_base);
    }
  }

  __device__ __forceinline__ uint64_t owners(const sdp_rule_desc* __restrict__ rules,
                                             const uint64_t* __restrict__ unit_bits, uint64_t full,
                                             int64_t j) const {
    if (uniform) return bits;
    const uint32_t le = static_cast<uint32_t>(j - lo);
    uint64_t b = full;
    for (int r = 0; r < rule_count; ++r) {
      const sdp_rule_desc rd = rules[rule_begin + r];
      const uint32_t q = fdiv(le, rd.inner_mul, rd.inner_shr);
      const uint32_t u = q - fdiv(q, rd.dim_mul, rd.dim_shr) * static_cast<uint32_t>(rd.dim);
      b &= __ldg(unit_bits + static_cast<uint32_t>(rd.unit_base) + u);
    }
    return b;
  }

  // owners of j and j + 1, both inside this parameter: one rule walk
  __device__ __forceinline__ void owners2(const sdp_rule_desc* __restrict__ rules,
                                          const uint64_t* __restrict__ unit_bits, uint64_t full,
                                          int64_t j, uint64_t& b0, uint64_t& b1) const {
    if (uniform) {
      b0 = b1 = bits;
      return;
    }
    const uint32_t le = static_cast<uint32_t>(j - lo);
    b0 = b1 = full;
    for (int r = 0; r < rule_count; ++r) {
      const sdp_rule_desc rd = rules[rule_begin + r];
      const uint32_t q0 = fdiv(le, rd.inner_mul, rd.inner_shr);
      const uint32_t q1 = fdiv(le + 1, rd.inner_mul, rd.inner_shr);
      const uint32_t u0 = q0 - fdiv(q0, rd.dim_mul, rd.dim_shr) * static_cast<uint32_t>(rd.dim);
      const uint32_t u1 = q1 - fdiv(q1, rd.dim_mul, rd.dim_shr) * static_cast<uint32_t>(rd.dim);
      const uint64_t* ub = unit_bits + static_cast<uint32_t>(rd.unit_base);
      b0 &= __ldg(ub + u0);
      b1 &= __ldg(ub + u1);
    }
  }
};

// bit q of the low nibble -> 16-bit field q (value 0/1), one carry-free multiply
__device__ __forceinline__ uint64_t spread4(uint64_t b) {
  return ((b & 0xf) * 0x0000200040008001ull) & 0x0001000100010001ull;
}

template <typename M>
__device__ __forceinline__ void st_mask_pair(M* p, uint64_t b0, uint64_t b1) {
  if constexpr (sizeof(M) == 1) {
    *reinterpret_cast<uint16_t*>(p) = static_cast<uint16_t>((b0 & 0xff) | ((b1 & 0xff) << 8));
  } else if constexpr (sizeof(M) == 2) {
    *reinterpret_cast<uint32_t*>(p) = static_cast<uint32_t>((b0 & 0xffff) | ((b1 & 0xffff) << 16));
  } else if constexpr (sizeof(M) == 4) {
    *reinterpret_cast<uint64_t*>(p) = (b0 & 0xffffffffull) | (b1 << 32);
  } else {
    *reinterpret_cast<ulonglong2*>(p) = make_ulonglong2(b0, b1);
  }
}

// Grid-stride over 256-element steps: at step k warp w writes elements
// [(k * n_warps + w) * 256, +256) in four 64-element iterations, lane l the
// pair (2l, 2l + 1) of each, so every store instruction writes 64 consecutive
// elements with 16-B (8-B arrays) or 2..16-B (masks) vectors, and the whole
// GPU's write front is one compact window (~7 MB per 8-B array).  A wider front (e.g. 1024-element warp chunks,
// ~40 MB per array) leaves the L2 evicting dirty lines from all over a 120 MB
// window: measured 2.1 TB/s instead of 3.5+ on the 3.1 GB GPT-2 build.
// Output buffers are 16-B aligned (checked by sdp_build_masks).
template <int MB>
__global__ void __launch_bounds__(kBuildThreads)
k_build_masks(const sdp_param_desc* __restrict__ params, int n_params,
              const sdp_rule_desc* __restrict__ rules, const uint64_t* __restrict__ unit_bits,
              int n_workers, int64_t total, typename MaskT<MB>::T* __restrict__ owner_mask,
              uint8_t* __restrict__ param_masks, int64_t* __restrict__ coverage,
              double* __restrict__ divisor, int64_t* __restrict__ governors,
              unsigned long long* __restrict__ active_counts) {
  using M = typename MaskT<MB>::T;
  const uint64_t full = n_workers == 64 ? ~0ull : ((1ull << n_workers) - 1);
  const int lane = threadIdx.x & 31;
  const int64_t n_steps = (total + kStepElems - 1) / kStepElems;
  const int64_t warp0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  // per-worker held counts of this lane: 16-bit counters, four per register;
  // MB mask bytes bound the workers (8 * MB), so only 2 * MB registers exist
  // (a 16-register loop with runtime predicates cost ~70 issued instructions
  // per element at N = 8)
  constexpr int kGroups = 2 * MB;
  uint64_t packed[kGroups];
#pragma unroll
  for (int g = 0; g < kGroups; ++g) packed[g] = 0;
  ParamCursor cur;
  cur.pi = -1;
  // Which steps a warp takes: a contiguous share when the share is small
  // (<= 16 steps: consecutive steps stay in one parameter, so the cursor --
  // binary search + rule loads -- is reused; ResNet-18 C2 / C3 82-87 ->
  // 70-73 / 69 us), else the interleaved grid stride, which keeps the
  // per-warp cost even where the per-element rule walk is dear in some
  // parameters only (GPT-2 channel units: contiguous shares were 4% slower;
  // profiles/r2_build_steps_ab.jsonl).
  const int64_t per_warp = (n_steps + n_warps - 1) / n_warps;
  const bool contiguous = per_warp <= 16;
  const int64_t k0 = contiguous ? warp0 * per_warp : warp0;
  const int64_t k_step = contiguous ? 1 : n_warps;
  const int64_t k_end = contiguous ? min(n_steps, k0 + per_warp) : n_steps;
  for (int64_t k = k0; k < k_end; k += k_step) {  // warp-uniform trip count
    // Whole step inside one parameter with one owner set (block rules or no
    // rule: the block strategy almost everywhere): constant fills, no
    // per-element work.  The cursor is loaded from the step start, so it is
    // warp-uniform here.
    const int64_t jb = k * kStepElems;
    if (cur.pi < 0 || jb < cur.lo || jb >= cur.hi)
      cur.load(params, rules, unit_bits, full, find_param(params, n_params, jb));
    if (cur.uniform && jb + kStepElems <= cur.hi && jb + kStepElems <= total && !(param_masks && (total & 1))) {
      const uint64_t b = cur.bits;
      const int c = __popcll(b);
      const longlong2 cv = make_longlong2(c, c);
      const double dv = static_cast<double>(c > 0 ? c : 1);
      const double2 dvv = make_double2(dv, dv);
      const longlong2 gv = make_longlong2(cur.rule_count, cur.rule_count);
#pragma unroll
      for (int it = 0; it < kStepElems / 64; ++it) {
        const int64_t j = jb + it * 64 + 2 * lane;
        if (owner_mask) st_mask_pair<M>(owner_mask + j, b, b);
        if (coverage) *reinterpret_cast<longlong2*>(coverage + j) = cv;
        if (divisor) *reinterpret_cast<double2*>(divisor + j) = dvv;
        if (governors) *reinterpret_cast<longlong2*>(governors + j) = gv;
        if (param_masks)
          for (int w = 0; w < n_workers; ++w)
            *reinterpret_cast<uint16_t*>(param_masks + static_cast<int64_t>(w) * total + j) =
                static_cast<uint16_t>(((b >> w) & 1ull) * 0x0101u);
      }
      if (active_counts) {  // 2 * kStepElems / 64 elements of this lane, all with owner set b
#pragma unroll
        for (int g = 0; g < kGroups; ++g)
          if (4 * g < n_workers) packed[g] += spread4(b >> (4 * g)) * (2 * kStepElems / 64);
      }
      continue;
    }
#pragma unroll 1
    for (int it = 0; it < kStepElems / 64; ++it) {
      const int64_t j = k * kStepElems + it * 64 + 2 * lane;
      if (j >= total) break;
      const bool two = j + 1 < total;
      if (cur.pi < 0 || j < cur.lo || j >= cur.hi)
        cur.load(params, rules, unit_bits, full, find_param(params, n_params, j));
      uint64_t b0, b1 = 0;
      int32_t g0 = cur.rule_count, g1 = 0;
      if (two && j + 1 < cur.hi) {
        cur.owners2(rules, unit_bits, full, j, b0, b1);
        g1 = g0;
      } else {
        b0 = cur.owners(rules, unit_bits, full, j);
        if (two) {  // the pair straddles a parameter boundary
          cur.load(params, rules, unit_bits, full, find_param(params, n_params, j + 1));
          b1 = cur.owners(rules, unit_bits, full, j + 1);
          g1 = cur.rule_count;
        }
      }
      const int c0 = __popcll(b0), c1 = __popcll(b1);
      if (two) {
        if (owner_mask) st_mask_pair<M>(owner_mask + j, b0, b1);
        if (coverage) *reinterpret_cast<longlong2*>(coverage + j) = make_longlong2(c0, c1);
        if (divisor) *reinterpret_cast<double2*>(divisor + j) = make_double2(c0 > 0 ? c0 : 1, c1 > 0 ? c1 : 1);
        if (governors) *reinterpret_cast<longlong2*>(governors + j) = make_longlong2(g0, g1);
        if (param_masks)
          for (int w = 0; w < n_workers; ++w) {
            uint8_t* pm = param_masks + static_cast<int64_t>(w) * total + j;
            if (total & 1) {  // odd d: row w starts at an odd byte for odd w
              pm[0] = static_cast<uint8_t>((b0 >> w) & 1ull);
              pm[1] = static_cast<uint8_t>((b1 >> w) & 1ull);
            } else {
              *reinterpret_cast<uint16_t*>(pm) =
                  static_cast<uint16_t>(((b0 >> w) & 1ull) | (((b1 >> w) & 1ull) << 8));
            }
          }
      } else {
        if (owner_mask) owner_mask[j] = static_cast<M>(b0);
        if (coverage) coverage[j] = c0;
        if (divisor) divisor[j] = static_cast<double>(c0 > 0 ? c0 : 1);
        if (governors) governors[j] = g0;
        if (param_masks)
          for (int w = 0; w < n_workers; ++w)
            param_masks[static_cast<int64_t>(w) * total + j] = static_cast<uint8_t>((b0 >> w) & 1ull);
      }
      if (active_counts) {
#pragma unroll
        for (int g = 0; g < kGroups; ++g)
          if (4 * g < n_workers) packed[g] += spread4(b0 >> (4 * g)) + spread4(b1 >> (4 * g));
      }
    }
  }
  if (active_counts) {
    // held-parameter count per worker: warp-shuffle reduce, one atomic per warp
#pragma unroll
    for (int g = 0; g < kGroups; ++g) {
      if (4 * g >= n_workers) break;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int w = 4 * g + q;
        if (w >= n_workers) break;
        const unsigned t = __reduce_add_sync(0xffffffffu, static_cast<unsigned>((packed[g] >> (16 * q)) & 0xffff));
        if (lane == 0 && t) atomicAdd(active_counts + w, static_cast<unsigned long long>(t));
      }
    }
  }
}


template <int MB>
__global__ void k_worker_mask(const typename MaskT<MB>::T* __restrict__ owner_mask, int64_t total,
                              int worker, double* __restrict__ mf, uint8_t* __restrict__ mu) {
  for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < total;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const bool on = (static_cast<uint64_t>(owner_mask[j]) >> worker) & 1ull;
    if (mf) mf[j] = on ? 1.0 : 0.0;
    if (mu) mu[j] = on ? 1 : 0;
  }
}

// One warp per tile: uniform iff AND == OR over the tile's owner sets.
template <int MB>
__global__ void k_plan_tiles(const typename MaskT<MB>::T* __restrict__ owner_mask, int64_t total,
                             int tile, int64_t n_tiles, sdp_tile_desc* __restrict__ tiles,
                             int64_t* __restrict__ owned) {
  using M = typename MaskT<MB>::T;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t t = warp; t < n_tiles; t += nwarps) {
    const int64_t s = t * tile;
    const int len = static_cast<int>(min(static_cast<int64_t>(tile), total - s));
    uint64_t a = ~0ull, o = 0;
    uint32_t cnt = 0;  // sum of |O_j| over the tile (<= 2^20 * 64)
    const M* base = owner_mask + s;
    if (len == tile) {
      constexpr int per = 16 / MB;  // mask elements per 16-B vector
      const uint4* v = reinterpret_cast<const uint4*>(base);
      for (int q = lane; q < tile / per; q += 32) {
        uint4 x = __ldg(v + q);
        const M* m = reinterpret_cast<const M*>(&x);
#pragma unroll
        for (int e = 0; e < per; ++e) {
          a &= static_cast<uint64_t>(m[e]);
          o |= static_cast<uint64_t>(m[e]);
          cnt += __popcll(static_cast<uint64_t>(m[e]));
        }
      }
    } else {
      for (int e = lane; e < len; e += 32) {
        uint64_t m = static_cast<uint64_t>(base[e]);
        a &= m;
        o |= m;
        cnt += __popcll(m);
      }
    }
    if (owned) {
      const uint32_t c = __reduce_add_sync(0xffffffffu, cnt);
      if (lane == 0) owned[t] = c;
    }
    const uint32_t alo = __reduce_and_sync(0xffffffffu, static_cast<uint32_t>(a));
    const uint32_t ahi = __reduce_and_sync(0xffffffffu, static_cast<uint32_t>(a >> 32));
    const uint32_t olo = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(o));
    const uint32_t ohi = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(o >> 32));
    if (lane == 0) {
      const uint64_t A = (static_cast<uint64_t>(ahi) << 32) | alo;
      const uint64_t O = (static_cast<uint64_t>(ohi) << 32) | olo;
      sdp_tile_desc d;
      d.owner_bits = O;
      d.tile_index = static_cast<uint32_t>(t);
      d.len_flags = static_cast<uint32_t>(len) | (A == O ? SDP_TILE_UNIFORM : 0u);
      tiles[t] = d;
    }
  }
}

static int check_mask_bytes(int mb) {
  if (mb == 1 || mb == 2 || mb == 4 || mb == 8) return SDP_OK;
  return set_error(SDP_ERR_CONFIG, "mask_bytes must be 1, 2, 4 or 8 (got %d)", mb);
}

static SeedWords make_seed(const uint32_t* w, int n) {
  SeedWords s{};
  s.n = n;
  for (int i = 0; i < n && i < 8; ++i) s.w[i] = w[i];
  return s;
}

}  // namespace sdp

using namespace sdp;

extern "C" {

int sdp_assign_units(const uint32_t* seed_words, int n_seed_words, const sdp_group_desc* groups,
                     int n_groups, int max_group, int n_units, int n_workers, int replication,
                     uint64_t* unit_bits, int32_t* scratch, void* stream) {
  if (n_workers < 1 || n_workers > SDP_MAX_WORKERS)
    return set_error(SDP_ERR_CONFIG, "n_workers must lie in [1, %d], got %d", SDP_MAX_WORKERS, n_workers);
  if (replication < 1 || replication > n_workers)
    return set_error(SDP_ERR_CONFIG, "replication must satisfy 1 <= P <= N, got P=%d, N=%d",
                     replication, n_workers);
  if (n_groups < 1 || max_group < 1) return set_error(SDP_ERR_CONFIG, "assignment requires non-empty groups");
  if (!seed_words || n_seed_words < 1 || n_seed_words > 8)
    return set_error(SDP_ERR_CONFIG, "seed must be given as 1..8 uint32 words");
  if (!unit_bits || !groups) return set_error(SDP_ERR_USAGE, "null device pointer");
  if (!scratch) return set_error(SDP_ERR_USAGE, "k_assign needs an 8 x n_units int32 scratch buffer");
  const size_t smem = kAssignWords * sizeof(uint32_t);
  k_assign<<<1, kAssignThreads, smem, as_stream(stream)>>>(
      make_seed(seed_words, n_seed_words), groups, n_groups, n_units, n_workers, replication,
      unit_bits, scratch);
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_permutation(const uint32_t* seed_words, int n_seed_words, const int32_t* skip_sizes,
                    int n_skip, int n, int32_t* out, void* stream) {
  if (!seed_words || n_seed_words < 1 || n_seed_words > 8)
    return set_error(SDP_ERR_CONFIG, "seed must be given as 1..8 uint32 words");
  if (n < 0 || n_skip < 0) return set_error(SDP_ERR_USAGE, "negative size");
  k_permutation<<<1, 32, 0, as_stream(stream)>>>(make_seed(seed_words, n_seed_words), skip_sizes,
                                                 n_skip, n, out);
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_build_masks(const sdp_param_desc* params, int n_params, const sdp_rule_desc* rules,
                    int n_rules, const uint64_t* unit_bits, int n_workers, int64_t total,
                    void* owner_mask, int mask_bytes, uint8_t* param_masks, int64_t* coverage,
                    double* divisor, int64_t* governors, int64_t* active_counts, void* stream) {
  (void)n_rules;
  if (n_workers < 1 || n_workers > SDP_MAX_WORKERS)
    return set_error(SDP_ERR_CONFIG, "n_workers must lie in [1, %d], got %d", SDP_MAX_WORKERS, n_workers);
  if (owner_mask && (check_mask_bytes(mask_bytes) || mask_bytes * 8 < n_workers))
    return set_error(SDP_ERR_CONFIG, "mask_bytes=%d cannot hold %d workers", mask_bytes, n_workers);
  if (n_params < 1 || total < 1) return set_error(SDP_ERR_TOPOLOGY, "empty topology");
  for (const void* p : {static_cast<const void*>(owner_mask), static_cast<const void*>(param_masks),
                        static_cast<const void*>(coverage), static_cast<const void*>(divisor),
                        static_cast<const void*>(governors)})
    if (reinterpret_cast<uintptr_t>(p) % 16)
      return set_error(SDP_ERR_USAGE, "sdp_build_masks outputs must be 16-byte aligned");
  const int64_t n_steps = (total + 63) / 64;
  const int64_t want = (n_steps + kBuildThreads / 32 - 1) / (kBuildThreads / 32);
  // one wave of resident CTAs (a partial second wave would idle 40% of the GPU)
  int per_sm = 0;
  SDP_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_build_masks<1>, kBuildThreads, 0));
  const int grid = static_cast<int>(std::min<int64_t>(want, static_cast<int64_t>(sm_count()) * std::max(1, per_sm)));
  auto ac = reinterpret_cast<unsigned long long*>(active_counts);
  cudaStream_t s = as_stream(stream);
  // the template width also bounds the per-worker counters: never below N
  const int mb = owner_mask ? mask_bytes : (n_workers <= 8 ? 1 : n_workers <= 16 ? 2 : n_workers <= 32 ? 4 : 8);
#define SDP_BUILD(MB)                                                                         \
  k_build_masks<MB><<<grid, kBuildThreads, 0, s>>>(params, n_params, rules, unit_bits,        \
                                                   n_workers, total,                          \
                                                   static_cast<MaskT<MB>::T*>(owner_mask),    \
                                                   param_masks, coverage, divisor, governors, ac)
  switch (mb) {
    case 1: SDP_BUILD(1); break;
    case 2: SDP_BUILD(2); break;
    case 4: SDP_BUILD(4); break;
    default: SDP_BUILD(8); break;
  }
#undef SDP_BUILD
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_worker_mask(const void* owner_mask, int mask_bytes, int64_t total, int worker,
                    double* mask_f64, uint8_t* mask_u8, void* stream) {
  if (check_mask_bytes(mask_bytes)) return SDP_ERR_CONFIG;
  if (worker < 0 || worker >= mask_bytes * 8)
    return set_error(SDP_ERR_CONFIG, "worker id %d outside the mask width", worker);
  if (total <= 0) return SDP_OK;
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, sm_count() * 8));
  cudaStream_t s = as_stream(stream);
  switch (mask_bytes) {
    case 1: k_worker_mask<1><<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(owner_mask), total, worker, mask_f64, mask_u8); break;
    case 2: k_worker_mask<2><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(owner_mask), total, worker, mask_f64, mask_u8); break;
    case 4: k_worker_mask<4><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(owner_mask), total, worker, mask_f64, mask_u8); break;
    default: k_worker_mask<8><<<grid, 256, 0, s>>>(static_cast<const uint64_t*>(owner_mask), total, worker, mask_f64, mask_u8); break;
  }
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

int sdp_plan_tiles(const void* owner_mask, int mask_bytes, int64_t total, int tile,
                   sdp_tile_desc* tiles, int64_t* owned, void* stream) {
  if (check_mask_bytes(mask_bytes)) return SDP_ERR_CONFIG;
  if (tile < 1024 || tile > (1 << 20) || tile % 1024)
    return set_error(SDP_ERR_CONFIG, "tile must be a multiple of 1024 in [1024, 2^20], got %d", tile);
  if (total <= 0) return SDP_OK;
  const int64_t n_tiles = (total + tile - 1) / tile;
  if (n_tiles > 0xFFFFFFFFll) return set_error(SDP_ERR_CONFIG, "too many tiles");
  const int64_t warps_per_cta = 8;
  const int grid = static_cast<int>(std::min<int64_t>((n_tiles + warps_per_cta - 1) / warps_per_cta, sm_count() * 8));
  cudaStream_t s = as_stream(stream);
  switch (mask_bytes) {
    case 1: k_plan_tiles<1><<<grid, 256, 0, s>>>(static_cast<const uint8_t*>(owner_mask), total, tile, n_tiles, tiles, owned); break;
    case 2: k_plan_tiles<2><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(owner_mask), total, tile, n_tiles, tiles, owned); break;
    case 4: k_plan_tiles<4><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(owner_mask), total, tile, n_tiles, tiles, owned); break;
    default: k_plan_tiles<8><<<grid, 256, 0, s>>>(static_cast<const uint64_t*>(owner_mask), total, tile, n_tiles, tiles, owned); break;
  }
  SDP_LAUNCH_CHECK();
  return SDP_OK;
}

}  // extern "C"

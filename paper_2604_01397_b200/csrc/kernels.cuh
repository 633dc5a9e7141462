// kernels.cuh — sm_100a kernels of the EXaCTz correction loop.
//
// Every kernel is deterministic regardless of thread order:
//  * detection reads a snapshot of g (Jacobi, amb-15) and only ever stores
//    the byte 1 into mark[] (idempotent; a vertex is edited at most once per
//    round);
//  * counts are integer atomics of warp-reduced partial sums;
//  * label pointer jumping only ever replaces a pointer by one of its
//    ancestors, so its fixpoint (the forest roots) is unique;
//  * the edit is a pure function of (g_i, c_i, f_i).
// IEEE float semantics are kept exact: no fast-math, explicit compare-select
// (never fminf/fmaxf, whose result for -0/+0 is unspecified), __fsub_ru /
// __fadd_rd for the bound (O1), __fsub_rn for the step (O9).
#pragma once
#include <stdint.h>

#include "mesh.cuh"

namespace exz {

__constant__ LinkTables c_link = kLink;

enum Counter {
  C_VT = 0,       // distinct marked vertices
  C_APPLIED = 1,  // edits applied
  C_N1 = 2,       // R1 .. R6 per-rule counts: C_N1 + k
  C_CHANGED = 8,  // pointer jumping: some pointer moved this round
  C_BAD_NF = 9,   // validation: non-finite values
  C_BAD_BOUND = 10,
  C_NSADDLE = 11,
  C_KEYMIN = 12,  // eps_from_relative: ordered-key min / max
  C_KEYMAX = 13,
  C_NCOUNTERS = 16
};

struct GridP {
  int nx, ny, nz, V;
  int delta[kSlots];  // linear offset of each slot
};

// ref word layout (one uint32 per vertex, computed once from f):
//   bits  0-13  f-lower mask (slot s set <=> neighbour s <_f i)
//   bits 14-17  dn_f slot (0..13, 14 = self)
//   bits 18-21  up_f slot
//   bits 22-24  nlc_f,  25-27 nuc_f
//   bit  28     f-saddle, 29 join saddle, 30 split saddle
__host__ __device__ constexpr uint32_t ref_flow(uint32_t r) { return r & 0x3FFFu; }
__host__ __device__ constexpr int ref_dn(uint32_t r) { return (r >> 14) & 15; }
__host__ __device__ constexpr int ref_up(uint32_t r) { return (r >> 18) & 15; }
__host__ __device__ constexpr int ref_nlc(uint32_t r) { return (r >> 22) & 7; }
__host__ __device__ constexpr int ref_nuc(uint32_t r) { return (r >> 25) & 7; }
__host__ __device__ constexpr bool ref_saddle(uint32_t r) { return (r >> 28) & 1; }
__host__ __device__ constexpr bool ref_join(uint32_t r) { return (r >> 29) & 1; }
__host__ __device__ constexpr bool ref_split(uint32_t r) { return (r >> 30) & 1; }

__device__ __forceinline__ uint32_t valid_mask(int x, int y, int z, const GridP &G) {
  uint32_t m = 0x3FFFu;
  if (x == 0) m &= ~(uint32_t)c_link.req[0];
  if (x == G.nx - 1) m &= ~(uint32_t)c_link.req[1];
  if (y == 0) m &= ~(uint32_t)c_link.req[2];
  if (y == G.ny - 1) m &= ~(uint32_t)c_link.req[3];
  if (z == 0) m &= ~(uint32_t)c_link.req[4];
  if (z == G.nz - 1) m &= ~(uint32_t)c_link.req[5];
  return m;
}

// Number of connected components of the link graph induced on `set`
// (bit-parallel flood fill; O4).
__device__ __forceinline__ uint32_t link_expand(uint32_t r) {
  uint32_t n = r;
#pragma unroll
  for (int s = 0; s < kSlots; ++s)
    if (r & (1u << s)) n |= c_link.adj[s];
  return n;
}
__device__ __noinline__ int link_components(uint32_t set) {
  int n = 0;
  while (set) {
    uint32_t r = set & (0u - set);
    for (;;) {
      uint32_t r2 = link_expand(r) & set;
      if (r2 == r) break;
      r = r2;
    }
    set &= ~r;
    ++n;
  }
  return n;
}

struct Star {
  uint32_t lower;  // slot s set <=> neighbour s <_h i (SoS)
  int dn, up;      // SoS argmin / argmax of the closed star (slot, 14 = self)
};

// Closed-star evaluation of vertex i of field h (O4 lower mask, O5 steepest).
__device__ __forceinline__ Star eval_star(const float *__restrict__ h, int i, uint32_t valid,
                                          const GridP &G) {
  const float hc = h[i];
  float v[kSlots];
#pragma unroll
  for (int s = 0; s < kSlots; ++s) v[s] = (valid & (1u << s)) ? h[i + G.delta[s]] : 0.0f;
  Star st;
  st.lower = 0;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    bool lo = (s < 7) ? (v[s] <= hc) : (v[s] < hc);
    if ((valid & (1u << s)) && lo) st.lower |= 1u << s;
  }
  // argmin in ascending index order, strict compare: the first minimum wins
  int dn = -1, up = -1;
  float dv = 0.0f, uv = 0.0f;
#pragma unroll
  for (int s = 0; s < 7; ++s)
    if (valid & (1u << s)) {
      if (dn < 0 || v[s] < dv) { dn = s; dv = v[s]; }
      if (up < 0 || v[s] >= uv) { up = s; uv = v[s]; }
    }
  if (dn < 0 || hc < dv) { dn = kSelf; dv = hc; }
  if (up < 0 || hc >= uv) { up = kSelf; uv = hc; }
#pragma unroll
  for (int s = 7; s < kSlots; ++s)
    if (valid & (1u << s)) {
      if (v[s] < dv) { dn = s; dv = v[s]; }
      if (v[s] >= uv) { up = s; uv = v[s]; }
    }
  st.dn = dn;
  st.up = up;
  return st;
}

__device__ __forceinline__ int slot_target(int i, int slot, const GridP &G) {
  return slot == kSelf ? i : i + G.delta[slot];
}

__device__ __forceinline__ void warp_add(unsigned long long *dst, unsigned v) {
  unsigned s = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(dst, (unsigned long long)s);
}

// ordered 32-bit key of a finite float: key order == IEEE order, -0 == +0
__device__ __forceinline__ uint32_t ordered_key(float v) {
  uint32_t b = __float_as_uint(v);
  if (b == 0x80000000u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// ---------------------------------------------------------------- validate (O1)
__global__ void k_validate(const float *__restrict__ f, const float *__restrict__ g, int64_t V,
                           float xi, unsigned long long *cnt) {
  unsigned nf = 0, nb = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    float a = f[i], b = g[i];
    if (!isfinite(a) || !isfinite(b)) {
      ++nf;
      continue;
    }
    float lo = __fsub_ru(a, xi), hi = __fadd_rd(a, xi);
    if (!(lo <= b && b <= hi)) ++nb;
  }
  warp_add(&cnt[C_BAD_NF], nf);
  warp_add(&cnt[C_BAD_BOUND], nb);
}

// ------------------------------------------------------ reference of f (O7)
// One thread per vertex: classification, steepest slots, ref word, the
// pointer forests of f (into labf_dn / labf_up, resolved later by jumping)
// and the SoS keys of the saddles (sorted later).
__global__ void __launch_bounds__(128) k_reference(const float *__restrict__ f, GridP G,
                                                   uint32_t *__restrict__ ref, int32_t *labf_dn,
                                                   int32_t *labf_up, uint64_t *saddle_keys,
                                                   unsigned long long *cnt) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, z = blockIdx.z;
  if (x >= G.nx) return;
  int i = x + G.nx * (y + G.ny * z);
  uint32_t valid = valid_mask(x, y, z, G);
  Star st = eval_star(f, i, valid, G);
  int nlc = link_components(st.lower);
  int nuc = link_components(valid & ~st.lower);
  bool isext = (nlc == 0) || (nuc == 0);
  bool sad = !isext && (nlc >= 2 || nuc >= 2);
  bool join = sad && nlc >= 2, split = sad && nuc >= 2;
  ref[i] = st.lower | ((uint32_t)st.dn << 14) | ((uint32_t)st.up << 18) | ((uint32_t)nlc << 22) |
           ((uint32_t)nuc << 25) | ((uint32_t)sad << 28) | ((uint32_t)join << 29) |
           ((uint32_t)split << 30);
  labf_dn[i] = slot_target(i, st.dn, G);
  labf_up[i] = slot_target(i, st.up, G);
  if (sad) {
    unsigned long long k = atomicAdd(&cnt[C_NSADDLE], 1ull);
    saddle_keys[k] = ((uint64_t)ordered_key(f[i]) << 32) | (uint32_t)i;
  }
}

__global__ void k_keys_to_ids(const uint64_t *__restrict__ keys, int32_t *ids, int n) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) ids[k] = (int32_t)(keys[k] & 0xffffffffu);
}

struct IsJoin {
  const uint32_t *ref;
  __device__ __forceinline__ bool operator()(const int32_t &s) const { return ref_join(ref[s]); }
};
struct IsSplit {
  const uint32_t *ref;
  __device__ __forceinline__ bool operator()(const int32_t &s) const { return ref_split(ref[s]); }
};

__device__ __forceinline__ bool sos_less_g(const float *h, int u, int v) {
  float a = h[u], b = h[v];
  return a < b || (a == b && u < v);
}

// m1(s): the <_f-largest minimum reached from the f-lower link of a join
// saddle; M1(s): the <_f-smallest maximum reached from the upper link of a
// split saddle.
__global__ void k_event_reference(const float *__restrict__ f, const uint32_t *__restrict__ ref,
                                  const int32_t *__restrict__ lab, const int32_t *__restrict__ sl,
                                  int n, int want_max, int32_t *out, GridP G) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  int s = sl[k];
  int x = s % G.nx, y = (s / G.nx) % G.ny, z = s / (G.nx * G.ny);
  uint32_t valid = valid_mask(x, y, z, G);
  uint32_t flow = ref_flow(ref[s]);
  uint32_t set = want_max ? flow : (valid & ~flow);
  int best = -1;
  for (uint32_t m = set; m; m &= m - 1) {
    int slot = __ffs(m) - 1;
    int e = lab[s + G.delta[slot]];
    if (best < 0 || (want_max ? sos_less_g(f, best, e) : sos_less_g(f, e, best))) best = e;
  }
  out[k] = best;
}

// --------------------------------------------------- pointer jumping (O6)
// lab[] holds, for every vertex, a pointer to an ancestor in its steepest
// forest; one round replaces it by an ancestor up to 2^hops further.  Reads
// may see pointers other threads already advanced (still ancestors), which
// only speeds convergence; the fixpoint (roots) is unique.
__global__ void k_jump(int32_t *lab, int64_t V, int hops, unsigned long long *cnt) {
  unsigned changed = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    int w = lab[i];
    int w2 = lab[w];
    if (w2 == w) continue;
    for (int h = 0; h < hops; ++h) {
      int w3 = lab[w2];
      if (w3 == w2) break;
      w2 = w3;
    }
    lab[i] = w2;
    changed = 1;
  }
  if (__any_sync(0xffffffffu, changed) && (threadIdx.x & 31) == 0) atomicOr(&cnt[C_CHANGED], 1ull);
}

// ------------------------------------------------------- detection (O8)
// R1, R2, R3 at every vertex from its closed star in g and its ref word;
// writes the g pointer forests for the labels when `ptrs` is set.
__global__ void __launch_bounds__(128) k_stencil(const float *__restrict__ g,
                                                 const uint32_t *__restrict__ ref,
                                                 uint8_t *mark, int32_t *pdn, int32_t *pup,
                                                 int ptrs, GridP G, unsigned long long *cnt) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, z = blockIdx.z;
  unsigned n1 = 0, n2 = 0, n3 = 0;
  if (x < G.nx) {
    int i = x + G.nx * (y + G.ny * z);
    uint32_t valid = valid_mask(x, y, z, G);
    Star st = eval_star(g, i, valid, G);
    uint32_t r = ref[i];
    // R1: the g-largest neighbour is an impostor -> decrease it
    if (st.up != ref_up(r)) {
      mark[slot_target(i, st.up, G)] = 1;
      n1 = 1;
    }
    // R2: the g-smallest neighbour changed -> decrease the true N_min
    if (st.dn != ref_dn(r)) {
      mark[slot_target(i, ref_dn(r), G)] = 1;
      n2 = 1;
    }
    // R3 (amb-7, amb-8)
    uint32_t flow = ref_flow(r);
    uint32_t flip = st.lower ^ flow;
    if (flip) {
      bool apply = ref_saddle(r);
      if (!apply) {
        int nl = link_components(st.lower);
        int nu = link_components(valid & ~st.lower);
        apply = (nl != ref_nlc(r)) || (nu != ref_nuc(r));
      }
      if (apply) {
        n3 = __popc(flip);
        for (uint32_t m = flip & flow; m; m &= m - 1) mark[i + G.delta[__ffs(m) - 1]] = 1;
        if (flip & ~flow) mark[i] = 1;
      }
    }
    if (ptrs) {
      pdn[i] = slot_target(i, st.dn, G);
      pup[i] = slot_target(i, st.up, G);
    }
  }
  warp_add(&cnt[C_N1 + 0], n1);
  warp_add(&cnt[C_N1 + 1], n2);
  warp_add(&cnt[C_N1 + 2], n3);
}

// R4 (C2): adjacent saddles a = S[k] <_f b = S[k+1]; if b <_g a,
// decrease a (the f-smaller).
__global__ void k_saddle_order(const float *__restrict__ g, const int32_t *__restrict__ S,
                               int nS, uint8_t *mark, unsigned long long *cnt) {
  unsigned n4 = 0;
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k + 1 < nS) {
    int a = S[k], b = S[k + 1];
    if (sos_less_g(g, b, a)) {
      mark[a] = 1;
      n4 = 1;
    }
  }
  warp_add(&cnt[C_N1 + 3], n4);
}

// R5 / R6 (C3): for a join saddle s, m2 = <_g-largest minimum
// reached from the g-lower link; if m2 != m1(s) decrease m2.  For a split
// saddle, M2 = <_g-smallest maximum from the g-upper link; if M2 != M1(s)
// decrease M1(s) (amb-12).
__global__ void k_events(const float *__restrict__ g, const int32_t *__restrict__ sl, int n,
                         const int32_t *__restrict__ lab, const int32_t *__restrict__ ref_ext,
                         int split, uint8_t *mark, GridP G, unsigned long long *cnt) {
  unsigned hit = 0;
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) {
    int s = sl[k];
    int x = s % G.nx, y = (s / G.nx) % G.ny, z = s / (G.nx * G.ny);
    uint32_t valid = valid_mask(x, y, z, G);
    float gs = g[s];
    int best = -1;
    float bv = 0.0f;
#pragma unroll
    for (int slot = 0; slot < kSlots; ++slot) {
      if (!(valid & (1u << slot))) continue;
      int u = s + G.delta[slot];
      float gu = g[u];
      bool lower = (slot < 7) ? (gu <= gs) : (gu < gs);
      if (lower == (bool)split) continue;
      int e = lab[u];
      float ge = g[e];
      bool take;
      if (best < 0) take = true;
      else if (!split) take = (bv < ge) || (bv == ge && best < e);  // max
      else take = (ge < bv) || (ge == bv && e < best);               // min
      if (take) { best = e; bv = ge; }
    }
    int want = ref_ext[k];
    if (best >= 0 && best != want) {
      mark[split ? want : best] = 1;
      hit = 1;
    }
  }
  warp_add(&cnt[C_N1 + 4 + split], hit);
}

// ---------------------------------------------------- count + edit (O9)
// V_t = #marked; for each marked i not at lo = RU(f_i - xi): a step of
// Delta (clamped at lo) while c_i < N, else the lossless clamp; c_i++.
// Marks are cleared for the next round.
__global__ void k_count_edit(float *g, uint8_t *c, uint8_t *mark, const float *__restrict__ f,
                             int64_t V, float xi, float delta, int N, int do_edit,
                             unsigned long long *cnt) {
  unsigned vt = 0, ap = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!mark[i]) continue;
    ++vt;
    mark[i] = 0;
    if (!do_edit) continue;
    float lo = __fsub_ru(f[i], xi);
    float gi = g[i];
    if (gi == lo) continue;
    int ci = c[i];
    float t;
    if (ci < N) {
      t = __fsub_rn(gi, delta);
      t = (t < lo) ? lo : t;
    } else {
      t = lo;
    }
    g[i] = t;
    c[i] = (uint8_t)(ci + 1);
    ++ap;
  }
  warp_add(&cnt[C_VT], vt);
  warp_add(&cnt[C_APPLIED], ap);
}

// ------------------------------------------------------- min / max of f
__global__ void k_minmax(const float *__restrict__ f, int64_t n, unsigned long long *cnt) {
  uint32_t mn = 0xffffffffu, mx = 0u;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t k = ordered_key(f[i]);
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&cnt[C_KEYMIN], (unsigned long long)mn);
    atomicMax(&cnt[C_KEYMAX], (unsigned long long)mx);
  }
}

}  // namespace exz

// kernels.cuh — sm_100a kernels of the EXaCTz correction loop.
//
// Every kernel is deterministic regardless of thread order:
//  * detection reads a snapshot of g (Jacobi, amb-15) and only ever ORs bits
//    into the mark bitmap (idempotent; a vertex is edited at most once per
//    round);
//  * counts are integer atomics of warp-reduced partial sums;
//  * labels are the unique terminus of a steepest path (walks, or pointer
//    jumping whose fixpoint is unique);
//  * the edit is a pure function of (g_i, c_i, f_i).
// IEEE float semantics are kept exact: no fast-math, explicit compare-select
// (never fminf/fmaxf, whose result for -0/+0 is unspecified), __fsub_ru /
// __fadd_rd for the bound (O1), __fsub_rn for the step (O9).
#pragma once
#include <stdint.h>

#include "mesh.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace exz {

__constant__ LinkTables c_link = kLink;
// Slot s decodes arithmetically (no table lookups with divergent indices):
// b = s - 6 for s >= 7, 7 - s for s < 7; offset = sign * (b&1, (b>>1)&1, b>>2).
__host__ __device__ __forceinline__ constexpr int slot_bits(int s) { return s >= 7 ? s - 6 : 7 - s; }
__host__ __device__ __forceinline__ constexpr int slot_sign(int s) { return s >= 7 ? 1 : -1; }

// Number of connected components of the link graph induced on any subset M of
// the 14 slots (O4), built on the host from the Kuhn tables.  The induced
// subgraph on M does not depend on the other slots, so a clipped (boundary)
// link is handled by the same table: nlc = comp[lower], nuc = comp[valid & ~lower].
__device__ uint8_t d_comp[1 << kSlots];

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
  C_NREMOTE = 14,  // sharded: remote marks appended by k_events
  C_WALK = 15,     // diagnostic: steps taken by the label walks of a pass
  C_NCP = 8,       // reference: critical points (shares the slot of C_CHANGED)
  C_NEG = 16,      // validation: lo = RU(f - xi) < 0 or g = -0.0 (k_stencil_fast needs none)
  C_EVAL = 17,     // diagnostic: vertices evaluated by the list / compacted stencils of a pass
  C_LINKS = 18,    // diagnostic: link vertices the C3 walks started from in a pass
  C_NCOUNTERS = 19
};

// Geometry of the (local) grid a kernel works on.  Single GPU: the whole
// field (zoff = 0, gnz = nz, owned planes [zb, ze) = [0, nz)).  Sharded: one
// z-slab with a ghost plane on each side (local plane 0 is global plane
// zoff), owned planes [1, nz-1).
struct GridP {
  int nx, ny, nz, V;  // local extent (V = nx*ny*nz)
  int W;              // 32-bit words per row of the mark bitmap, ceil(nx/32)
  int delta[kSlots];  // linear offset of each slot
  int zoff, gnz;      // global z of local plane 0, global nz
  int zb, ze;         // owned local planes [zb, ze)
  uint32_t mnx, mny, mW;  // division by nx, ny, W: q = (umulhi(n, m) + n) >> l (n < 2^31)
  int lnx, lny, lW;
  // k_stencil_fast key tags as run-time values: (bits & keymask) | tag[k] is
  // one LOP3 with the tag as a constant-bank operand (with both as
  // immediates ptxas emits two)
  uint32_t keymask;   // ~15u
  uint32_t tag[16];   // tag[k] = k
  // k_stencil_key: key of slot s = bits * 16 + kc[s], kc[s] = s - 16 bits(lo_min)
  uint32_t kc[kSlots];
  uint32_t k16;  // 16, as a run-time value: the key products stay IMADs (stencil_key.cuh)
  uint32_t k2up[10];  // 2^(29 - 3r): row r of a pair layout to the top 3 bits by IMAD
};

// Magic numbers of the unsigned division n / d for n < 2^31, d >= 1
// (Granlund-Montgomery): l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1.
inline void fastdiv_magic(uint32_t d, uint32_t &m, int &l) {
  l = 0;
  while ((1ull << l) < d) ++l;
  m = (uint32_t)((((1ull << l) - d) << 32) / d + 1);
}
inline void grid_fastdiv(GridP &G) {
  G.keymask = ~15u;
  G.k16 = 16u;
  for (int r = 0; r < 10; ++r) G.k2up[r] = 1u << (29 - 3 * r);
  for (int k = 0; k < 16; ++k) G.tag[k] = (uint32_t)k;
  fastdiv_magic((uint32_t)G.nx, G.mnx, G.lnx);
  fastdiv_magic((uint32_t)G.ny, G.mny, G.lny);
  fastdiv_magic((uint32_t)G.W, G.mW, G.lW);
}
__device__ __forceinline__ int div_nx(int n, const GridP &G) {
  return (int)((__umulhi((uint32_t)n, G.mnx) + (uint32_t)n) >> G.lnx);
}
__device__ __forceinline__ int div_ny(int n, const GridP &G) {
  return (int)((__umulhi((uint32_t)n, G.mny) + (uint32_t)n) >> G.lny);
}
__device__ __forceinline__ int div_W(int n, const GridP &G) {  // mark-bitmap row of word n
  return (int)((__umulhi((uint32_t)n, G.mW) + (uint32_t)n) >> G.lW);
}

// Change tracking (single GPU, late rounds).
//  * Vertex activity: a vertex whose closed star saw no value change and that
//    did not fire R1-R3 in the previous pass evaluates exactly as before (no
//    fire, same steepest slots), so only act = St(edited) u fired is re-run,
//    by the sparse stencil.  act_next collects the set for the next pass
//    (bitmaps in the mark layout).
//  * Brick stamps for the C3 cache: bricks of 32 x 8 x 8 vertices carry
//      bval[b]  = pass in which a value change inside b becomes visible
//                 (edits of pass t are stamped t + 1),
//      bslot[b] = pass in which a steepest slot inside b changed;
//    a saddle's cached C3 result is reused while no brick its walks touched
//    changed.
#ifndef EXACTZ_BY
#define EXACTZ_BY 8
#endif
#ifndef EXACTZ_BZ
#define EXACTZ_BZ 8
#endif
#ifndef EXACTZ_SB
#define EXACTZ_SB 4
#endif
constexpr int BX = 32, BY = EXACTZ_BY, BZ = EXACTZ_BZ;  // BX = one warp row of the stencils
constexpr int SB = EXACTZ_SB;  // superbrick = SB^3 bricks (4: 128 x 32 x 32 vertices)
struct Track {
  uint16_t *bval, *bslot;       // brick stamps (nullptr: C3 cache off)
  uint16_t *sbval, *sbslot;     // superbrick stamps (max over its bricks)
  uint32_t *act_next;           // vertex activity for the next pass (nullptr: off)
  uint32_t *edited;             // vertices edited by this pass (written by k_count_edit)
  const int32_t *posS;          // position in S of each f-saddle (single GPU; else nullptr)
  uint32_t *gS;                 // g at S[k] (value bits), written by the stencils for C2
  uint32_t *lmS;                // the saddles' link masks in S order (single GPU; else the
                                // stencils write lm[i]); read through per-list positions
  int nbx, nby, nbz, round;
  int nsx, nsy;                 // superbrick grid (x, y extents)
  int tab_round;                // sharded: last pass in which a boundary-table entry changed
  // exactz_correct_host: vertices edited after the result's D2H copy began
  // (patched on the host afterwards); nullptr: off
  int32_t *patch;
  int *npatch;
  int patch_cap;
  // clean-path test of the C3 walks (FPaths below): tiles holding a vertex
  // whose dn_g != dn_f (dirtD) / up_g != up_f (dirtU) in this pass, set by
  // the list stencil (nullptr: off)
  uint8_t *dirtD, *dirtU;  // one byte per tile (plain stores of 1: no read, no atomic)
  int ntx, nty;
};

// Tiles of the clean-path test: 8 x 4 x 4 vertices.
constexpr int FTX_SH = 3, FTY_SH = 2, FTZ_SH = 2;
__host__ __device__ __forceinline__ int ftile(int x, int y, int z, int ntx, int nty) {
  return (x >> FTX_SH) + ntx * ((y >> FTY_SH) + nty * (z >> FTZ_SH));
}

// Outputs of a stencil at an f-saddle i: its g-lower / g-upper link masks
// (for the C3 walks) and its value at its position in S (for C2).
// g at an f-saddle into its entry k of gS (sharded: the changed owned
// entries are listed afterwards by k_gs_diff)
__device__ __forceinline__ void gs_write(const Track &T, int k, uint32_t vbits) { T.gS[k] = vbits; }

// With T.lmS (single GPU) the masks go to the saddle's position in S, a
// compact array the C3 kernels gather from L2 instead of the V-sized lm.
__device__ __forceinline__ void saddle_out(uint32_t *__restrict__ lm, const Track &T, int i,
                                           uint32_t lower, uint32_t valid, uint32_t vbits) {
  const uint32_t m = lower | ((valid & ~lower) << 16);
  if (T.gS) {
    const int k = __ldg(&T.posS[i]);
    gs_write(T, k, vbits);
    if (T.lmS) T.lmS[k] = m;
    else lm[i] = m;
  } else {
    lm[i] = m;
  }
}
// link masks of saddle k of a list (lpos: positions in S, masks in S order)
__device__ __forceinline__ uint32_t saddle_lm(const uint32_t *__restrict__ lm,
                                              const int32_t *__restrict__ lpos, int k, int s) {
  return lpos ? __ldg(&lm[__ldg(&lpos[k])]) : __ldg(&lm[s]);
}

__device__ __forceinline__ void stamp(uint16_t *b, uint16_t *sb, const Track &T, int bx, int by,
                                      int bz, uint16_t v) {
  b[bx + T.nbx * (by + T.nby * bz)] = v;
  sb[bx / SB + T.nsx * (by / SB + T.nsy * (bz / SB))] = v;
}

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

// slots of vertex (x, y, local z) whose neighbour exists in the global domain
// (split into the x/y and the z conditions for the z-marching kernels)
__device__ __forceinline__ uint32_t valid_xy(int x, int y, const GridP &G) {
  uint32_t m = 0x3FFFu;
  if (x == 0) m &= ~(uint32_t)c_link.req[0];
  if (x == G.nx - 1) m &= ~(uint32_t)c_link.req[1];
  if (y == 0) m &= ~(uint32_t)c_link.req[2];
  if (y == G.ny - 1) m &= ~(uint32_t)c_link.req[3];
  return m;
}
__device__ __forceinline__ uint32_t valid_z(int z, const GridP &G) {
  uint32_t m = 0x3FFFu;
  const int zg = z + G.zoff;
  if (zg == 0) m &= ~(uint32_t)c_link.req[4];
  if (zg == G.gnz - 1) m &= ~(uint32_t)c_link.req[5];
  return m;
}
__device__ __forceinline__ uint32_t valid_mask(int x, int y, int z, const GridP &G) {
  uint32_t m = 0x3FFFu;
  const int zg = z + G.zoff;
  if (x == 0) m &= ~(uint32_t)c_link.req[0];
  if (x == G.nx - 1) m &= ~(uint32_t)c_link.req[1];
  if (y == 0) m &= ~(uint32_t)c_link.req[2];
  if (y == G.ny - 1) m &= ~(uint32_t)c_link.req[3];
  if (zg == 0) m &= ~(uint32_t)c_link.req[4];
  if (zg == G.gnz - 1) m &= ~(uint32_t)c_link.req[5];
  return m;
}

// Number of connected components of the link graph induced on `set`
// (bit-parallel flood fill; O4).  Used on the host to build d_comp.
__host__ __device__ __forceinline__ uint32_t link_expand(uint32_t r, const uint16_t *adj) {
  uint32_t n = r;
#pragma unroll
  for (int s = 0; s < kSlots; ++s)
    if (r & (1u << s)) n |= adj[s];
  return n;
}
__host__ __device__ inline int link_components_t(uint32_t set, const uint16_t *adj) {
  int n = 0;
  while (set) {
    uint32_t r = set & (0u - set);
    for (;;) {
      uint32_t r2 = link_expand(r, adj) & set;
      if (r2 == r) break;
      r = r2;
    }
    set &= ~r;
    ++n;
  }
  return n;
}

// (nlc, nuc) of a vertex with lower mask `lower` and valid mask `valid`.
__device__ __forceinline__ void link_type(uint32_t lower, uint32_t valid, int &nl, int &nu) {
  nl = __ldg(&d_comp[lower]);
  nu = __ldg(&d_comp[valid & ~lower]);
}

struct Star {
  uint32_t lower;  // slot s set <=> neighbour s <_h i (SoS)
  int dn, up;      // SoS argmin / argmax of the closed star (slot, 14 = self)
};

// Closed-star evaluation (O4 lower mask, O5 steepest) from the 14 neighbour
// values v[] (slot order) and the centre hc.  SoS by static slot direction:
// candidates are visited in ascending index order (slots 0..6, the centre,
// slots 7..13) with a strict compare for the argmin (first minimum = smallest
// index wins a tie) and a non-strict one for the argmax (last maximum =
// largest index wins).  Missing neighbours hold NaN, for which every compare
// is false: they are never lower, never the argmin, never the argmax.
__device__ __forceinline__ Star eval_values(const float (&v)[kSlots], float hc) {
  Star st;
  st.lower = 0;
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {
    bool lo = (s < 7) ? (v[s] <= hc) : (v[s] < hc);
    st.lower |= lo ? (1u << s) : 0u;
  }
  int dn = kSelf, up = kSelf;
  float dv = __int_as_float(0x7f800000), uv = -__int_as_float(0x7f800000);  // +inf, -inf
#pragma unroll
  for (int s = 0; s < 7; ++s) {
    if (v[s] < dv) { dn = s; dv = v[s]; }
    if (v[s] >= uv) { up = s; uv = v[s]; }
  }
  if (hc < dv) { dn = kSelf; dv = hc; }
  if (hc >= uv) { up = kSelf; uv = hc; }
#pragma unroll
  for (int s = 7; s < kSlots; ++s) {
    if (v[s] < dv) { dn = s; dv = v[s]; }
    if (v[s] >= uv) { up = s; uv = v[s]; }
  }
  st.dn = dn;
  st.up = up;
  return st;
}

__device__ __forceinline__ Star eval_star(const float *__restrict__ h, int i, uint32_t valid,
                                          const GridP &G) {
  float v[kSlots];
#pragma unroll
  for (int s = 0; s < kSlots; ++s)
    v[s] = (valid & (1u << s)) ? h[i + G.delta[s]] : __int_as_float(0x7fc00000);
  return eval_values(v, h[i]);
}

// linear offset of slot s (0..13) by arithmetic decode (no indexed parameter
// loads for a data-dependent slot)
__device__ __forceinline__ int slot_delta(int s, const GridP &G) {
  const int b = slot_bits(s);
  const int d = (b & 1) + ((b >> 1) & 1) * G.nx + (b >> 2) * (G.nx * G.ny);
  return s >= 7 ? d : -d;
}
__device__ __forceinline__ int slot_target(int i, int slot, const GridP &G) {
  return slot == kSelf ? i : i + slot_delta(slot, G);
}

// Statistics counters (V_t, applied, per-rule counts, validation) are summed
// by one atomic per warp into one of kCntRep replicas of the counter array
// chosen by the block: with a single address every warp's atomic queued at
// one L2 slice (ncu, C3 R4 launch: 700 K same-address atomics, one slice's
// atomic unit 34 % busy vs 2 % on average, 1.1 ms for 22 M saddle pairs).
// k_fold_counters adds the replicas into cnt[0 .. C_NCOUNTERS) (and clears
// them) before the host or a collective reads the counters.
constexpr int kCntRep = 32, kCntStride = 32;  // replica r of counter X: cnt[(1 + r) * stride + X]
constexpr int C_NALLOC = (1 + kCntRep) * kCntStride;

__device__ __forceinline__ void warp_add(unsigned long long *dst, unsigned v) {
  unsigned s = __reduce_add_sync(0xffffffffu, v);
  const unsigned r = (blockIdx.x + 7u * blockIdx.y + 13u * blockIdx.z) & (kCntRep - 1);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(dst + (size_t)(1 + r) * kCntStride, (unsigned long long)s);
}

// values (and edit counts) of the patched vertices, for the host patch
__global__ void k_gather_patch(const int32_t *__restrict__ idx, int n, const float *__restrict__ g,
                               const uint8_t *__restrict__ c, float *vals, uint8_t *cnts) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  vals[k] = g[idx[k]];
  if (c) cnts[k] = c[idx[k]];
}

__global__ void k_fold_counters(unsigned long long *cnt, unsigned long long *mirror = nullptr) {
  const int X = threadIdx.x;
  if (X >= C_NCOUNTERS) return;
  unsigned long long t = 0;
  for (int r = 1; r <= kCntRep; ++r) {
    t += cnt[r * kCntStride + X];
    cnt[r * kCntStride + X] = 0;
  }
  t += cnt[X];
  cnt[X] = t;
  if (mirror) mirror[X] = t;  // mapped host memory (Ctx::read)
}

// ordered 32-bit key of a finite float: key order == IEEE order, -0 == +0
__device__ __forceinline__ uint32_t ordered_key(float v) {
  uint32_t b = __float_as_uint(v);
  if (b == 0x80000000u) b = 0u;
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// mark bitmap: row-padded, bit x of word row*W + x/32 (row = y + ny*z)
// Marks only accumulate until the edit pass clears them, so a bit already
// set (by the stencil, which ran before, or by another rule) needs no atomic:
// an L2 read (the 16 MB bitmap of 512^3 stays resident) replaces most
// read-modify-writes in the dense rounds, where most targets are marked.
__device__ __forceinline__ void mark_vertex(uint32_t *marks, int v, const GridP &G) {
  const int row = div_nx(v, G), x = v - row * G.nx;
  uint32_t *w = &marks[(size_t)row * G.W + (x >> 5)];
  const uint32_t b = 1u << (x & 31);
  if (!(__ldcg(w) & b)) atomicOr(w, b);
}

__device__ __forceinline__ bool sos_less_g(const float *h, int u, int v) {
  float a = h[u], b = h[v];
  return a < b || (a == b && u < v);
}

// ---------------------------------------------------------------- validate (O1)
__global__ void k_validate(const float *__restrict__ f, const float *__restrict__ g, int64_t V,
                           float xi, unsigned long long *cnt) {
  unsigned nf = 0, nb = 0, ng = 0;
  uint32_t nlo = 0, ghi = 0;  // ~bits of the smallest lo, bits of the largest g (lo, g >= 0)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    float a = f[i], b = g[i];
    if (!isfinite(a) || !isfinite(b)) {
      ++nf;
      continue;
    }
    float lo = __fsub_ru(a, xi), hi = __fadd_rd(a, xi);
    if (!(lo <= b && b <= hi)) ++nb;
    if (lo < 0.0f || __float_as_uint(b) == 0x80000000u) ++ng;  // -0.0 in g: general stencil
    nlo = max(nlo, ~__float_as_uint(lo));
    ghi = max(ghi, __float_as_uint(b));
  }
  warp_add(&cnt[C_BAD_NF], nf);
  warp_add(&cnt[C_BAD_BOUND], nb);
  warp_add(&cnt[C_NEG], ng);
  // value range of g over the call (k_stencil_key's applicability); only
  // read when C_NEG == 0, where bit order == value order
  nlo = __reduce_max_sync(0xffffffffu, nlo);
  ghi = __reduce_max_sync(0xffffffffu, ghi);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&cnt[C_KEYMIN], (unsigned long long)nlo);
    atomicMax(&cnt[C_KEYMAX], (unsigned long long)ghi);
  }
}

// ------------------------------------------------------ reference of f (O7)
// Classification, steepest slots and the ref word of vertex (x, y, z) of f;
// SoS keys of the saddles are appended (sorted later).
__device__ __forceinline__ void reference_vertex(const float *__restrict__ f, const GridP &G,
                                                 uint32_t *__restrict__ ref,
                                                 uint64_t *saddle_keys, uint64_t *cp_keys,
                                                 unsigned long long *cnt, int x, int y, int z) {
  const bool in = x < G.nx;  // lanes past the row end take part in the ballots only
  const int i = in ? x + G.nx * (y + G.ny * z) : 0;
  bool isext = false, sad = false;
  uint64_t key = 0;
  if (in) {
    uint32_t valid = valid_mask(x, y, z, G);
    Star st = eval_star(f, i, valid, G);
    int nlc, nuc;
    link_type(st.lower, valid, nlc, nuc);
    isext = (nlc == 0) || (nuc == 0);
    sad = !isext && (nlc >= 2 || nuc >= 2);
    const bool join = sad && nlc >= 2, split = sad && nuc >= 2;
    ref[i] = st.lower | ((uint32_t)st.dn << 14) | ((uint32_t)st.up << 18) |
             ((uint32_t)nlc << 22) | ((uint32_t)nuc << 25) | ((uint32_t)sad << 28) |
             ((uint32_t)join << 29) | ((uint32_t)split << 30);
    const uint32_t ig = (uint32_t)(i + G.zoff * G.nx * G.ny);  // global index (SoS)
    key = ((uint64_t)ordered_key(f[i]) << 32) | ig;
  }
  // warp-aggregated appends (one atomic per warp and list; list order is
  // irrelevant: the keys are sorted afterwards)
  const unsigned ms = __ballot_sync(0xffffffffu, sad);
  const unsigned mc = cp_keys ? __ballot_sync(0xffffffffu, sad || isext) : 0u;
  const int lane = threadIdx.x & 31;
  unsigned long long bs = 0, bc = 0;
  if (lane == 0) {
    if (ms) bs = atomicAdd(&cnt[C_NSADDLE], (unsigned long long)__popc(ms));
    if (mc) bc = atomicAdd(&cnt[C_NCP], (unsigned long long)__popc(mc));
  }
  const unsigned below = (1u << lane) - 1u;
  bs = __shfl_sync(0xffffffffu, bs, 0);
  bc = __shfl_sync(0xffffffffu, bc, 0);
  if (sad) saddle_keys[bs + __popc(ms & below)] = key;
  if (cp_keys && (sad || isext)) cp_keys[bc + __popc(mc & below)] = key;
}

// Persistent 2D grid over rows (y + ny*z) and x.
__global__ void __launch_bounds__(128) k_reference(const float *__restrict__ f, GridP G,
                                                   uint32_t *__restrict__ ref,
                                                   uint64_t *saddle_keys, uint64_t *cp_keys,
                                                   unsigned long long *cnt) {
  // warp-uniform trip counts (the appends use warp ballots); lanes past nx idle
  for (int row = G.zb * G.ny + blockIdx.y; row < G.ze * G.ny; row += gridDim.y)
    for (int xb = blockIdx.x * blockDim.x + (threadIdx.x & ~31); xb < G.nx;
         xb += gridDim.x * blockDim.x)
      reference_vertex(f, G, ref, saddle_keys, cp_keys, cnt, xb + (threadIdx.x & 31), row % G.ny,
                       row / G.ny);
}

// The same reference on the stencil's z-marching shared-memory tile (32 x 8
// columns per CTA, f planes z-1 .. z+1 in a 4-deep ring with halo; NaN for
// missing neighbours): neighbour values come from shared memory instead of 14
// global loads per vertex.
__global__ void __launch_bounds__(256) k_reference_tile(const float *__restrict__ f, GridP G,
                                                        int zc, uint32_t *__restrict__ ref,
                                                        uint64_t *saddle_keys, uint64_t *cp_keys,
                                                        unsigned long long *cnt,
                                                        uint8_t *__restrict__ fslots = nullptr) {
  constexpr int TXr = 32, TYr = 8, SXr = TXr + 2, SPr = SXr * (TYr + 2);
  __shared__ float sg[4][SPr];
  __shared__ unsigned wcnt[2][TYr];             // per-warp key counts of the plane
  __shared__ unsigned long long wbase[2][TYr];  // per-warp output offsets
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, tid = threadIdx.x;
  const int x0 = blockIdx.x * TXr, y0 = blockIdx.y * TYr;
  const int z0 = G.zb + blockIdx.z * zc, z1 = min(z0 + zc, G.ze);
  const int x = x0 + tx, y = y0 + ty;
  const bool inside = x < G.nx && y < G.ny;
  const int c = (ty + 1) * SXr + tx + 1;
  int coff[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int cc = tid + k * 256;
    coff[k] = -1;
    if (cc < SPr) {
      const int ly = cc / SXr, lx = cc - ly * SXr;
      const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
      if (gx >= 0 && gx < G.nx && gy >= 0 && gy < G.ny) coff[k] = gx + G.nx * gy;
    }
  }
  auto load = [&](int p, float (&r)[2]) {
    const bool pin = p >= 0 && p < G.nz;
#pragma unroll
    for (int k = 0; k < 2; ++k)
      r[k] = (pin && coff[k] >= 0) ? f[(size_t)p * G.nx * G.ny + coff[k]] : __int_as_float(0x7fc00000);
  };
  auto store = [&](int p, const float (&r)[2]) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (tid + k * 256 < SPr) sg[p & 3][tid + k * 256] = r[k];
  };
  {
    float r[2];
    for (int p = z0 - 1; p <= z0 + 1; ++p) {
      load(p, r);
      store(p, r);
    }
  }
  __syncthreads();
  for (int z = z0; z < z1; ++z) {
    float pre[2];  // plane z+2 in flight while plane z is classified
    const bool prefetch = z + 2 <= z1;
    if (prefetch) load(z + 2, pre);
    bool isext = false, sad = false;
    uint64_t key = 0;
    if (inside) {
      const float *pm = &sg[(z - 1) & 3][c], *p0 = &sg[z & 3][c], *pp = &sg[(z + 1) & 3][c];
      float v[kSlots];
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        const int b = slot_bits(s), sg1 = slot_sign(s);
        const float *pl = (b >> 2) ? (sg1 > 0 ? pp : pm) : p0;
        v[s] = pl[sg1 * ((b & 1) + ((b >> 1) & 1) * SXr)];
      }
      const Star st = eval_values(v, *p0);
      const uint32_t valid = valid_mask(x, y, z, G);
      int nlc, nuc;
      link_type(st.lower, valid, nlc, nuc);
      isext = (nlc == 0) || (nuc == 0);
      sad = !isext && (nlc >= 2 || nuc >= 2);
      const bool join = sad && nlc >= 2, split = sad && nuc >= 2;
      const int i = x + G.nx * (y + G.ny * z);
      ref[i] = st.lower | ((uint32_t)st.dn << 14) | ((uint32_t)st.up << 18) |
               ((uint32_t)nlc << 22) | ((uint32_t)nuc << 25) | ((uint32_t)sad << 28) |
               ((uint32_t)join << 29) | ((uint32_t)split << 30);
      // f's steepest slots as one byte (the f-walks of k_fpaths read 1 B per
      // step instead of the 4 B ref word)
      if (fslots) fslots[i] = (uint8_t)(st.dn | (st.up << 4));
      const uint32_t ig = (uint32_t)(i + G.zoff * G.nx * G.ny);
      key = ((uint64_t)ordered_key(*p0) << 32) | ig;
    }
    // one global atomic per CTA and plane (was: per warp; every one on the
    // same address, queued at one L2 slice): the warps' counts go through
    // shared memory, warp 0 takes the CTA's range
    const unsigned ms = __ballot_sync(0xffffffffu, sad);
    const unsigned mc = cp_keys ? __ballot_sync(0xffffffffu, sad || isext) : 0u;
    if (tx == 0) {
      wcnt[0][ty] = __popc(ms);
      wcnt[1][ty] = __popc(mc);
    }
    __syncthreads();
    if (ty == 0) {
      const unsigned a = tx < TYr ? wcnt[0][tx] : 0u, b = tx < TYr ? wcnt[1][tx] : 0u;
      unsigned ia = a, ib = b;  // inclusive scans over the 8 warps
#pragma unroll
      for (int o = 1; o < TYr; o <<= 1) {
        const unsigned pa = __shfl_up_sync(0xffffffffu, ia, o), pb = __shfl_up_sync(0xffffffffu, ib, o);
        if (tx >= o) { ia += pa; ib += pb; }
      }
      const unsigned ta = __shfl_sync(0xffffffffu, ia, TYr - 1), tb = __shfl_sync(0xffffffffu, ib, TYr - 1);
      unsigned long long ga = 0, gb = 0;
      if (tx == 0) {
        if (ta) ga = atomicAdd(&cnt[C_NSADDLE], (unsigned long long)ta);
        if (tb) gb = atomicAdd(&cnt[C_NCP], (unsigned long long)tb);
      }
      ga = __shfl_sync(0xffffffffu, ga, 0);
      gb = __shfl_sync(0xffffffffu, gb, 0);
      if (tx < TYr) {
        wbase[0][tx] = ga + ia - a;
        wbase[1][tx] = gb + ib - b;
      }
    }
    __syncthreads();
    const unsigned long long bs = wbase[0][ty], bc = wbase[1][ty];
    const unsigned below = (1u << tx) - 1u;
    if (sad) saddle_keys[bs + __popc(ms & below)] = key;
    if (cp_keys && (sad || isext)) cp_keys[bc + __popc(mc & below)] = key;
    if (prefetch) store(z + 2, pre);  // ring slot of plane z-2, last read at step z-1
    __syncthreads();
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

// ------------------------------------------------------- detection (O8)
// Stencil tile: 32 (x) x 8 (y) columns per CTA (one warp per y row),
// marching along z through a chunk of planes.  g planes z-1 .. z+2 live in a
// 4-deep shared-memory ring with a 1-vertex halo; plane z+2 is prefetched
// into registers while plane z is evaluated.
// Marks: every vertex names its targets as a 15-bit mask over its closed
// star; a warp turns the masks into one ballot per slot and ORs them, shifted
// by the slot's x offset, into 64-bit shared rows (bit lx of row ly of a
// plane buffer, lx = 0..33 covering x0-1 .. x0+32).  A plane is complete one
// step after its last contributor and is flushed into the global bitmap with
// at most 3 atomics per row (left halo bit, the 32 interior bits, right halo
// bit).  One barrier per plane.
constexpr int TX = 32, TY = 8, NT = TX * TY;
constexpr int SX = TX + 2, SY = TY + 2, SP = SX * SY;  // 340 cells per plane

// Per-thread offsets of its (up to 2) halo-tile cells within a plane, -1 when
// outside the domain; computed once per CTA (V < 2^31: 32-bit offsets).
struct PlaneCells {
  int off[2];
};
__device__ __forceinline__ PlaneCells plane_cells(int x0, int y0, const GridP &G) {
  const int tid = threadIdx.y * TX + threadIdx.x;
  PlaneCells pc;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    int c = tid + k * NT;
    pc.off[k] = -1;
    if (c < SP) {
      int ly = c / SX, lx = c - ly * SX;
      int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
      if (gx >= 0 && gx < G.nx && gy >= 0 && gy < G.ny) pc.off[k] = gx + G.nx * gy;
    }
  }
  return pc;
}
// Plane p of the tile with its halo into registers; cells outside the domain
// (or a plane outside [0, nz)) read as NaN.
__device__ __forceinline__ void load_plane_regs(const float *__restrict__ g, int p,
                                                const PlaneCells &pc, const GridP &G,
                                                float (&r)[2]) {
  const bool pin = p >= 0 && p < G.nz;
  const float *gp = g + p * (G.nx * G.ny);
#pragma unroll
  for (int k = 0; k < 2; ++k)
    r[k] = (pin && pc.off[k] >= 0) ? gp[pc.off[k]] : __int_as_float(0x7fc00000);
}
__device__ __forceinline__ void store_plane_regs(float *sg, const float (&r)[2]) {
  const int tid = threadIdx.y * TX + threadIdx.x;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    int c = tid + k * NT;
    if (c < SP) sg[c] = r[k];
  }
}

// R1, R2, R3 at one vertex (x, y, z) from its closed star in the shared ring
// (pm, p0, pp: the vertex's cell in planes z-1, z, z+1) and its ref word r.
// Returns the targets as a 15-bit mask over the closed star (bit 14 = self);
// ns receives the packed steepest slots (dn | up << 4), lower the g-lower
// mask.  At the f-saddles the stencils keep lm = lower | upper << 16 (the
// g-lower and g-upper link slots) for the C3 event kernels.
__device__ __forceinline__ uint32_t stencil_rules(const float *pm, const float *p0,
                                                  const float *pp, uint32_t r, uint32_t valid,
                                                  unsigned &n1,
                                                  unsigned &n2, unsigned &n3, uint8_t &ns,
                                                  uint32_t &lower) {
  float v[kSlots];
#pragma unroll
  for (int s = 0; s < kSlots; ++s) {  // s is a compile-time constant here
    const int b = slot_bits(s), sg1 = slot_sign(s);
    const float *pl = (b >> 2) ? (sg1 > 0 ? pp : pm) : p0;
    v[s] = pl[sg1 * ((b & 1) + ((b >> 1) & 1) * SX)];
  }
  const Star st = eval_values(v, *p0);
  uint32_t tgt = 0;
  // R1: the g-largest neighbour is an impostor -> decrease it
  if (st.up != ref_up(r)) { tgt |= 1u << st.up; n1 += 1; }
  // R2: the g-smallest neighbour changed -> decrease the true N_min
  if (st.dn != ref_dn(r)) { tgt |= 1u << ref_dn(r); n2 += 1; }
  // R3 (amb-7, amb-8): flipped pairs at f-saddles and at
  // vertices whose type (nlc, nuc) changed; target = the f-smaller end
  const uint32_t flow = ref_flow(r);
  const uint32_t flip = st.lower ^ flow;
  if (flip) {
    bool apply = ref_saddle(r);
    if (!apply) {
      int nl, nu;
      link_type(st.lower, valid, nl, nu);
      apply = (nl != ref_nlc(r)) || (nu != ref_nuc(r));
    }
    if (apply) {
      n3 += __popc(flip);
      tgt |= flip & flow;
      if (flip & ~flow) tgt |= 1u << kSelf;
    }
  }
  ns = (uint8_t)(st.dn | (st.up << 4));
  lower = st.lower;
  return tgt;
}

// Row masks of the marks, by writer: step z (mod 4) x warp (y row) x the 7
// (dz, dy) target rows, one u64 each (bit 1 + dx + lane; 8th word padding).
// Lane 0 of every warp stores its 7 words every step (zeros when it marked
// nothing); the flush of plane p ORs the words its writers stored at steps
// p+1, p, p-1.
typedef unsigned long long u64;
constexpr int KR = 7;  // k: (dz,dy) = (-1,-1) (-1,0) (0,-1) (0,0) (0,1) (1,0) (1,1)
__host__ __device__ constexpr int kr_dz(int k) { return k < 2 ? -1 : (k < 5 ? 0 : 1); }
__host__ __device__ constexpr int kr_dy(int k) {
  return (k == 0 || k == 2) ? -1 : ((k == 4 || k == 6) ? 1 : 0);
}

// Flush plane p (rows ly = 0..SY-1 of the tile with its halo) into the global
// bitmap: lane ly ORs the words of its writers and issues at most 3 atomics
// (left halo bit, the 32 interior bits, right halo bit).  Writer steps
// outside [z0, z1) did not run and are skipped.
__device__ __forceinline__ void flush_plane(uint32_t *__restrict__ marks,
                                            const u64 (*wr)[TY][8], int p, int z0, int z1,
                                            int x0, int y0, const GridP &G) {
  const int ly = threadIdx.x;
  if (ly >= SY) return;
  u64 val = 0;
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int w = ly - 1 - kr_dy(k), st = p - kr_dz(k);
    if (w >= 0 && w < TY && st >= z0 && st < z1) val |= wr[st & 3][w][k];
  }
  const int gy = y0 - 1 + ly;
  if (!val || gy < 0 || gy >= G.ny || p < 0 || p >= G.nz) return;
  uint32_t *row = marks + (size_t)(gy + G.ny * p) * G.W;
  const int wx = x0 >> 5;
  const uint32_t w = (uint32_t)(val >> 1);
  if (w) atomicOr(&row[wx], w);
  if ((val & 1ull) && x0 > 0) atomicOr(&row[wx - 1], 0x80000000u);
  if (((val >> 33) & 1ull) && x0 + 32 < G.nx) atomicOr(&row[wx + 1], 1u);
}

// Dense pass: R1, R2, R3 at every vertex; writes the packed steepest slots
// used by the label walks.
template <bool TRACK>
__global__ void __launch_bounds__(NT, 5) k_stencil(const float *__restrict__ g,
                                                   const uint32_t *__restrict__ ref,
                                                   uint32_t *__restrict__ marks,
                                                   uint8_t *__restrict__ slots,
                                                   uint32_t *__restrict__ lm, GridP G, int zc,
                                                   Track T, unsigned long long *cnt) {
  __shared__ float sg[4][SP];
  __shared__ __align__(16) u64 wr[4][TY][8];
  const int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int x0 = bx * TX, y0 = by * TY;
  const int z0 = G.zb + bz * zc, z1 = min(z0 + zc, G.ze);
  const int x = x0 + tx, y = y0 + ty;
  const bool inside = x < G.nx && y < G.ny;
  const int c = (ty + 1) * SX + tx + 1;
  const uint32_t vxy = valid_xy(x, y, G);
  unsigned n1 = 0, n2 = 0, n3 = 0;
  const PlaneCells pc = plane_cells(x0, y0, G);

  {  // prologue: planes z0-1, z0, z0+1 (NaN outside the domain)
    float r[2];
    for (int p = z0 - 1; p <= z0 + 1; ++p) {
      load_plane_regs(g, p, pc, G, r);
      store_plane_regs(sg[p & 3], r);
    }
  }
  __syncthreads();

  for (int z = z0; z < z1; ++z) {
    float pre[2];
    const int pz = z + 2;
    const bool prefetch = pz <= z1;
    if (prefetch) load_plane_regs(g, pz, pc, G, pre);

    uint32_t tgt = 0;
    bool schg = false;
    if (inside) {
      const int i = x + G.nx * (y + G.ny * z);
      const uint32_t r = __ldcs(&ref[i]);
      uint8_t ns;
      uint32_t lower;
      const uint32_t valid = vxy & valid_z(z, G);
      tgt = stencil_rules(&sg[(z - 1) & 3][c], &sg[z & 3][c], &sg[(z + 1) & 3][c], r, valid, n1,
                          n2, n3, ns, lower);
      if (TRACK && T.bval) schg = (slots[i] != ns);
      slots[i] = ns;
      if (ref_saddle(r)) saddle_out(lm, T, i, lower, valid, __float_as_uint(sg[z & 3][c]));
    }
    if (TRACK && T.bval) {  // slot-change stamp of this warp's brick
      const unsigned chg = __ballot_sync(0xffffffffu, schg);
      if (tx == 0 && chg) stamp(T.bslot, T.sbslot, T, bx, y / BY, z / BZ, (uint16_t)T.round);
    }
    if (TRACK && T.act_next) {  // fired vertices stay active next pass
      const unsigned fired = __ballot_sync(0xffffffffu, tgt != 0);
      if (tx == 0 && fired) atomicOr(&T.act_next[(size_t)(y + G.ny * z) * G.W + bx], fired);
    }
    // warp-aggregated marks: the targets re-indexed in ascending linear
    // order (slots 0..6, self, 7..13) put each (dz, dy) row's 2-3 slots on
    // adjacent bits; per row, lane l contributes those bits shifted to
    // 1 + dx + l and one OR-reduction per 32-bit half builds the 34-bit row
    u64 rv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (__any_sync(0xffffffffu, tgt)) {
      const uint32_t t = (tgt & 0x7Fu) | ((tgt & 0x3F80u) << 1) | ((tgt >> kSelf) << 7);
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        constexpr int kStart[KR] = {0, 2, 4, 6, 9, 11, 13};
        const uint32_t c = ((t >> kStart[k]) & (k == 3 ? 7u : 3u)) << (k >= 4 ? 1 : 0);
        const uint32_t lo = __reduce_or_sync(0xffffffffu, c << tx);
        const uint32_t hi = __reduce_or_sync(0xffffffffu, tx >= 30 ? c >> (32 - tx) : 0u);
        rv[k] = (u64)lo | ((u64)hi << 32);
      }
    }
    if (tx == 0) {
      ulonglong2 *d = reinterpret_cast<ulonglong2 *>(&wr[z & 3][ty][0]);
#pragma unroll
      for (int k = 0; k < 4; ++k) d[k] = make_ulonglong2(rv[2 * k], rv[2 * k + 1]);
    }
    // plane z-2 is complete (its writers z-3 .. z-1 are done): one warp
    // flushes it
    const int pf = z - 2;
    if (ty == (z & (TY - 1)) && pf >= z0 - 1 && pf >= 0) flush_plane(marks, wr, pf, z0, z1, x0, y0, G);
    if (prefetch) store_plane_regs(sg[pz & 3], pre);
    __syncthreads();
  }
  // epilogue: planes z1-2 .. z1 not flushed by the loop (one warp each)
  {
    const int pf = z1 - 2 + ty;
    if (ty < 3 && pf >= z0 - 1 && pf >= 0 && pf < G.nz) flush_plane(marks, wr, pf, z0, z1, x0, y0, G);
  }

  warp_add(&cnt[C_N1 + 0], n1);
  warp_add(&cnt[C_N1 + 1], n2);
  warp_add(&cnt[C_N1 + 2], n3);
}

// Compacted dense pass (tracking, moderately many active vertices): the same
// z-march and shared ring, but per plane only the active vertices of the tile
// are evaluated, packed onto the first threads of the CTA.  The list of plane
// z+1 is built during step z from the activity words (consumed words are
// cleared); marks go to per-plane shared row words by shared atomics; the
// fired vertices of plane z are written to act_next at step z+1; a brick's
// slot-change stamp comes from the step's barrier (__syncthreads_or).
__global__ void __launch_bounds__(NT, 5) k_stencil_compact(const float *__restrict__ g,
                                                           const uint32_t *__restrict__ ref,
                                                           uint32_t *__restrict__ marks,
                                                           uint8_t *__restrict__ slots,
                                                           uint32_t *__restrict__ lm,
                                                           uint32_t *__restrict__ act, GridP G,
                                                           int zc, Track T,
                                                           unsigned long long *cnt) {
  __shared__ float sg[4][SP];
  __shared__ uint32_t cmI[4][SY], cmH[4][SY];  // interior bits / halo bits (1: x0-1, 2: x0+32)
  __shared__ uint16_t list[4][NT];
  __shared__ int ln[4];
  __shared__ uint32_t fm[2][TY];
  const int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int x0 = bx * TX, y0 = by * TY;
  const int z0 = G.zb + bz * zc, z1 = min(z0 + zc, G.ze);
  const int yw = y0 + ty;  // this warp's row for the list building
  const uint32_t xin = (G.nx - x0 >= 32) ? 0xffffffffu : ((1u << (G.nx - x0)) - 1u);
  unsigned n1 = 0, n2 = 0, n3 = 0;
  const PlaneCells pc = plane_cells(x0, y0, G);
  unsigned ne = 0;  // vertices evaluated (C_EVAL)

  // active lanes of this warp's row in plane p -> list[p & 3]
  auto build = [&](int p) {
    uint32_t a = 0;
    if (yw < G.ny) {
      uint32_t *aw = &act[(size_t)(yw + G.ny * p) * G.W + bx];
      a = *aw;  // warp-uniform address: one broadcast load
      if (a && tx == 0) *aw = 0u;  // consumed
      a &= xin;
    }
    if (!a) return;
    int base = 0;
    if (tx == 0) base = atomicAdd(&ln[p & 3], __popc(a));
    base = __shfl_sync(0xffffffffu, base, 0);
    if ((a >> tx) & 1u) list[p & 3][base + __popc(a & ((1u << tx) - 1u))] = (uint16_t)tid;
  };

  if (tid < 4) ln[tid] = 0;
  if (tid < 4 * SY) {
    (&cmI[0][0])[tid] = 0u;
    (&cmH[0][0])[tid] = 0u;
  }
  if (tid < 2 * TY) (&fm[0][0])[tid] = 0u;
  {  // prologue: planes z0-1, z0, z0+1 (NaN outside the domain)
    float r[2];
    for (int p = z0 - 1; p <= z0 + 1; ++p) {
      load_plane_regs(g, p, pc, G, r);
      store_plane_regs(sg[p & 3], r);
    }
  }
  __syncthreads();
  build(z0);
  __syncthreads();

  for (int z = z0; z < z1; ++z) {
    float pre[2];
    const int pz = z + 2;
    const bool prefetch = pz <= z1;
    if (prefetch) load_plane_regs(g, pz, pc, G, pre);
    if (z + 1 < z1) build(z + 1);
    if (tid == 0) ln[(z + 2) & 3] = 0;  // plane z-2's count, reused by plane z+2
    if (z > z0 && tx == 0) {  // fired vertices of plane z-1 (complete at the last barrier)
      uint32_t &w = fm[(z - 1) & 1][ty];
      if (w) {
        atomicOr(&T.act_next[(size_t)(yw + G.ny * (z - 1)) * G.W + bx], w);
        w = 0u;
      }
    }

    bool schg = false;
    if (tid < ln[z & 3]) {
      ++ne;
      const int cell = list[z & 3][tid];
      const int lx = cell & 31, ly = cell >> 5;
      const int x = x0 + lx, y = y0 + ly;
      const int i = x + G.nx * (y + G.ny * z);
      const int c = (ly + 1) * SX + lx + 1;
      const uint32_t r = ref[i];
      uint8_t ns;
      uint32_t lower;
      const uint32_t valid = valid_mask(x, y, z, G);
      const uint32_t tgt = stencil_rules(&sg[(z - 1) & 3][c], &sg[z & 3][c],
                                         &sg[(z + 1) & 3][c], r, valid, n1, n2, n3, ns, lower);
      if (T.bval) schg = (slots[i] != ns);
      slots[i] = ns;
      if (ref_saddle(r)) saddle_out(lm, T, i, lower, valid, __float_as_uint(sg[z & 3][c]));
      if (tgt) {
        atomicOr(&fm[z & 1][ly], 1u << lx);
        for (uint32_t m = tgt; m; m &= m - 1) {
          const int s = __ffs(m) - 1;
          int dx = 0, dy = 0, dz = 0;
          if (s != kSelf) {
            const int b = slot_bits(s), sg1 = slot_sign(s);
            dx = sg1 * (b & 1);
            dy = sg1 * ((b >> 1) & 1);
            dz = sg1 * (b >> 2);
          }
          const int tx2 = lx + dx, row = ly + 1 + dy, pl = (z + dz) & 3;
          if (tx2 < 0) atomicOr(&cmH[pl][row], 1u);
          else if (tx2 > 31) atomicOr(&cmH[pl][row], 2u);
          else atomicOr(&cmI[pl][row], 1u << tx2);
        }
      }
    }
    // plane z-2 is complete (its writers z-3 .. z-1 are done): one warp
    // flushes and clears it
    const int pf = z - 2;
    if (ty == (z & (TY - 1)) && pf >= z0 - 1 && pf >= 0 && tx < SY) {
      const int ly = tx, gy = y0 - 1 + ly;
      const uint32_t w = cmI[pf & 3][ly], h = cmH[pf & 3][ly];
      cmI[pf & 3][ly] = 0u;
      cmH[pf & 3][ly] = 0u;
      if ((w | h) && gy >= 0 && gy < G.ny && pf < G.nz) {
        uint32_t *row = marks + (size_t)(gy + G.ny * pf) * G.W;
        const int wx = x0 >> 5;
        if (w) atomicOr(&row[wx], w);
        if ((h & 1u) && x0 > 0) atomicOr(&row[wx - 1], 0x80000000u);
        if ((h & 2u) && x0 + 32 < G.nx) atomicOr(&row[wx + 1], 1u);
      }
    }
    if (prefetch) store_plane_regs(sg[pz & 3], pre);
    if (T.bval) {
      if (__syncthreads_or(schg) && tid == 0)  // every brick the CTA's rows cover
        for (int b = y0 / BY, bl = (min(y0 + TY, G.ny) - 1) / BY; b <= bl; ++b)
          stamp(T.bslot, T.sbslot, T, bx, b, z / BZ, (uint16_t)T.round);
    } else {
      __syncthreads();
    }
  }
  // epilogue: fired words of plane z1-1; planes z1-2 .. z1 not flushed yet
  if (tx == 0 && z1 > z0) {
    const uint32_t w = fm[(z1 - 1) & 1][ty];
    if (w) atomicOr(&T.act_next[(size_t)(yw + G.ny * (z1 - 1)) * G.W + bx], w);
  }
  {
    const int pf = z1 - 2 + ty;
    if (ty < 3 && pf >= z0 - 1 && pf >= 0 && pf < G.nz && tx < SY) {
      const int ly = tx, gy = y0 - 1 + ly;
      const uint32_t w = cmI[pf & 3][ly], h = cmH[pf & 3][ly];
      if ((w | h) && gy >= 0 && gy < G.ny) {
        uint32_t *row = marks + (size_t)(gy + G.ny * pf) * G.W;
        const int wx = x0 >> 5;
        if (w) atomicOr(&row[wx], w);
        if ((h & 1u) && x0 > 0) atomicOr(&row[wx - 1], 0x80000000u);
        if ((h & 2u) && x0 + 32 < G.nx) atomicOr(&row[wx + 1], 1u);
      }
    }
  }

  warp_add(&cnt[C_N1 + 0], n1);
  warp_add(&cnt[C_N1 + 1], n2);
  warp_add(&cnt[C_N1 + 2], n3);
  warp_add(&cnt[C_EVAL], ne);
}

// Sparse pass (tracking): re-evaluate only the active vertices (warp per
// 32-bit word of the activity bitmap, consumed words are cleared).  Same
// rules as k_stencil, neighbour values read from global memory.
__global__ void __launch_bounds__(256) k_stencil_sparse(const float *__restrict__ g,
                                                        const uint32_t *__restrict__ ref,
                                                        uint32_t *__restrict__ marks,
                                                        uint8_t *__restrict__ slots,
                                                        uint32_t *__restrict__ lm,
                                                        uint32_t *__restrict__ act, GridP G,
                                                        Track T, unsigned long long *cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)G.ny * G.zb * G.W, nwords = (int64_t)G.ny * G.ze * G.W;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned n1 = 0, n2 = 0, n3 = 0;
  for (int64_t base = w0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32;
       base < nwords; base += nwarps * 32) {
   // 32 words per warp step, one per lane; only the non-zero ones are visited
   const uint32_t mine = (base + lane < nwords) ? act[base + lane] : 0u;
   if (mine) act[base + lane] = 0u;  // consumed
   for (uint32_t nzw = __ballot_sync(0xffffffffu, mine != 0u); nzw; nzw &= nzw - 1) {
    const int j = __ffs(nzw) - 1;
    const uint32_t word = __shfl_sync(0xffffffffu, mine, j);
    const int64_t w = base + j;
    const int row = div_W((int)w, G), wx = (int)w - row * G.W;
    const int z = div_ny(row, G), y = row - z * G.ny, x = wx * 32 + lane;
    uint32_t tgt = 0;
    bool schg = false;
    if (((word >> lane) & 1u) && x < G.nx) {
      const int i = x + G.nx * row;
      const uint32_t valid = valid_mask(x, y, z, G);
      const Star st = eval_star(g, i, valid, G);
      const uint32_t r = ref[i];
      if (st.up != ref_up(r)) { tgt |= 1u << st.up; n1 += 1; }
      if (st.dn != ref_dn(r)) { tgt |= 1u << ref_dn(r); n2 += 1; }
      const uint32_t flow = ref_flow(r);
      const uint32_t flip = st.lower ^ flow;
      if (flip) {
        bool apply = ref_saddle(r);
        if (!apply) {
          int nl, nu;
          link_type(st.lower, valid, nl, nu);
          apply = (nl != ref_nlc(r)) || (nu != ref_nuc(r));
        }
        if (apply) {
          n3 += __popc(flip);
          tgt |= flip & flow;
          if (flip & ~flow) tgt |= 1u << kSelf;
        }
      }
      for (uint32_t m = tgt; m; m &= m - 1) mark_vertex(marks, slot_target(i, __ffs(m) - 1, G), G);
      const uint8_t ns = (uint8_t)(st.dn | (st.up << 4));
      schg = slots[i] != ns;
      slots[i] = ns;
      if (ref_saddle(r)) saddle_out(lm, T, i, st.lower, valid, __float_as_uint(g[i]));
    }
    if (T.bval) {
      const unsigned chg = __ballot_sync(0xffffffffu, schg);
      if (lane == 0 && chg) stamp(T.bslot, T.sbslot, T, wx, y / BY, z / BZ, (uint16_t)T.round);
    }
    if (T.act_next) {
      const unsigned fired = __ballot_sync(0xffffffffu, tgt != 0);
      if (lane == 0 && fired) atomicOr(&T.act_next[w], fired);
    }
   }
  }
  warp_add(&cnt[C_N1 + 0], n1);
  warp_add(&cnt[C_N1 + 1], n2);
  warp_add(&cnt[C_N1 + 2], n3);
}

// act |= closed stars of the vertices edited by the previous pass: the
// edited bitmap dilated by the Freudenthal star (offsets in rows (dz, dy) of
// the KR list; dx in {-1, 0} for rows 0..3 and {0, +1} for rows 3..6).  One
// thread per word; the star is symmetric, so "some edited vertex lies in my
// star" is this pull.
__device__ __forceinline__ uint32_t dilated_word(const uint32_t *__restrict__ edited, int row,
                                                 int wx, const GridP &G) {
  const int z = div_ny(row, G), y = row - z * G.ny;
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int yy = y + kr_dy(k), zz = z + kr_dz(k);
    if (yy < 0 || yy >= G.ny || zz < 0 || zz >= G.nz) continue;
    const uint32_t *r = edited + (size_t)(yy + G.ny * zz) * G.W;
    const uint32_t e = __ldg(&r[wx]);
    acc |= e;
    if (k <= 3) acc |= (e << 1) | ((wx > 0) ? (__ldg(&r[wx - 1]) >> 31) : 0u);
    if (k >= 3) acc |= (e >> 1) | ((wx + 1 < G.W) ? (__ldg(&r[wx + 1]) << 31) : 0u);
  }
  const int rem = G.nx - wx * 32;
  if (rem < 32) acc &= (1u << rem) - 1u;
  return acc;
}

__global__ void __launch_bounds__(256) k_dilate_or(uint32_t *__restrict__ act,
                                                   const uint32_t *__restrict__ edited, GridP G) {
  const int64_t w0 = (int64_t)G.ny * G.zb * G.W, nwords = (int64_t)G.ny * G.ze * G.W;
  for (int64_t w = w0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int row = div_W((int)w, G), wx = (int)w - row * G.W;
    const uint32_t acc = dilated_word(edited, row, wx, G);
    if (acc) act[w] |= acc;
  }
}

// List-based sparse pass (tracking): k_act_list compacts the activity bitmap
// into a list of vertex indices (words consumed and cleared), then
// k_stencil_list evaluates one listed vertex per thread (full parallelism;
// the neighbours come from global memory, mostly L1/L2 hits).  Same rules and
// outputs as k_stencil_sparse.
__global__ void __launch_bounds__(256) k_act_list(uint32_t *__restrict__ act,
                                                  const uint32_t *__restrict__ edited, GridP G,
                                                  int32_t *__restrict__ list, int *count) {
  __shared__ int wsum[8], bbase;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w0 = (int64_t)G.ny * G.zb * G.W, nwords = (int64_t)G.ny * G.ze * G.W;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // the next step's word is loaded one step ahead (the late passes are a
  // latency-bound scan of mostly zero words)
  uint32_t a_next = (w0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x < nwords)
                        ? act[w0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x]
                        : 0u;
  for (int64_t base = w0 + (int64_t)blockIdx.x * blockDim.x; base < nwords;
       base += stride) {  // block-uniform trip count
    const int64_t w = base + threadIdx.x;
    uint32_t a = a_next;
    a_next = (w + stride < nwords) ? act[w + stride] : 0u;
    int row = 0, x0 = 0;
    if (w < nwords) {
      // this pass's set: fired last pass (act, consumed) | stars of its edits
      row = div_W((int)w, G);
      const int wx = (int)w - row * G.W;
      x0 = wx * 32;
      if (a) act[w] = 0u;
      if (edited) a |= dilated_word(edited, row, wx, G);
      if (G.nx - x0 < 32) a &= (1u << (G.nx - x0)) - 1u;
    }
    if (!__syncthreads_or(a != 0u)) continue;  // nothing active in these 256 words
    const int n = __popc(a);
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {  // one atomic per block and step
      int tot = 0;
      for (int k = 0; k < 8; ++k) {
        const int v = wsum[k];
        wsum[k] = tot;
        tot += v;
      }
      bbase = tot ? atomicAdd(count, tot) : 0;
    }
    __syncthreads();
    // coalesced writes: the warp writes one non-zero word at a time, lane l
    // storing vertex x0 + l if its bit is set
    int k = bbase + wsum[warp] + incl - n;
    const int i0 = row * G.nx + x0;
    const unsigned nzw = __ballot_sync(0xffffffffu, a != 0u);
    if ((int)__reduce_max_sync(0xffffffffu, (unsigned)n) * 2 < __popc(nzw)) {
      for (; a; a &= a - 1) list[k++] = i0 + __ffs(a) - 1;  // few bits per word
      a = 0;
    }
    for (unsigned nz = __ballot_sync(0xffffffffu, a != 0u); nz; nz &= nz - 1) {
      const int j = __ffs(nz) - 1;
      const uint32_t aj = __shfl_sync(0xffffffffu, a, j);
      const int kj = __shfl_sync(0xffffffffu, k, j), ij = __shfl_sync(0xffffffffu, i0, j);
      if ((aj >> lane) & 1u) list[kj + __popc(aj & ((1u << lane) - 1u))] = ij + lane;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void vertex_outputs(int i, int x, int y, int z, int row, uint32_t r,
                                               uint32_t valid, uint32_t tgt, uint32_t lower,
                                               int dn, int up, const float *__restrict__ g,
                                               uint32_t *__restrict__ marks,
                                               uint8_t *__restrict__ slots,
                                               uint32_t *__restrict__ lm, const GridP &G,
                                               const Track &T);

// One vertex's pass with neighbours from global memory (the list-based and
// the direct dense passes): R1-R3, marks by atomics, slots / lm, tracking.
__device__ __forceinline__ void vertex_pass(int i, const float *__restrict__ g,
                                            const uint32_t *__restrict__ ref,
                                            uint32_t *__restrict__ marks,
                                            uint8_t *__restrict__ slots,
                                            uint32_t *__restrict__ lm, const GridP &G,
                                            const Track &T, unsigned &n1, unsigned &n2,
                                            unsigned &n3) {
  const int row = div_nx(i, G), x = i - row * G.nx;
  const int z = div_ny(row, G), y = row - z * G.ny;
  const uint32_t valid = valid_mask(x, y, z, G);
  const Star st = eval_star(g, i, valid, G);
  const uint32_t r = __ldg(&ref[i]);
  uint32_t tgt = 0;
  if (st.up != ref_up(r)) { tgt |= 1u << st.up; n1 += 1; }
  if (st.dn != ref_dn(r)) { tgt |= 1u << ref_dn(r); n2 += 1; }
  const uint32_t flow = ref_flow(r);
  const uint32_t flip = st.lower ^ flow;
  if (flip) {
    bool apply = ref_saddle(r);
    if (!apply) {
      int nl, nu;
      link_type(st.lower, valid, nl, nu);
      apply = (nl != ref_nlc(r)) || (nu != ref_nuc(r));
    }
    if (apply) {
      n3 += __popc(flip);
      tgt |= flip & flow;
      if (flip & ~flow) tgt |= 1u << kSelf;
    }
  }
  vertex_outputs(i, x, y, z, row, r, valid, tgt, st.lower, st.dn, st.up, g, marks, slots, lm, G, T);
}

// The outputs of one vertex's evaluation (both list stencils): marks by
// atomics, dirty tiles, slot byte (and its brick stamp), lm / gS at f-saddles,
// activity for the next pass.
__device__ __forceinline__ void vertex_outputs(int i, int x, int y, int z, int row, uint32_t r,
                                               uint32_t valid, uint32_t tgt, uint32_t lower,
                                               int dn, int up, const float *__restrict__ g,
                                               uint32_t *__restrict__ marks,
                                               uint8_t *__restrict__ slots,
                                               uint32_t *__restrict__ lm, const GridP &G,
                                               const Track &T) {
  struct {
    int dn, up;
  } st{dn, up};
  for (uint32_t m = tgt; m; m &= m - 1) mark_vertex(marks, slot_target(i, __ffs(m) - 1, G), G);
  if (T.dirtD) {  // a steepest pointer of g that is not f's: its tile is dirty (FPaths)
    const bool dd = st.dn != ref_dn(r), du = st.up != ref_up(r);
    if (dd || du) {
      const int t = ftile(x, y, z, T.ntx, T.nty);
      if (dd) T.dirtD[t] = 1;
      if (du) T.dirtU[t] = 1;
    }
  }
  const uint8_t ns = (uint8_t)(st.dn | (st.up << 4));
  if (T.bval && slots[i] != ns)  // benign race: every writer stores the same pass number
    stamp(T.bslot, T.sbslot, T, x / BX, y / BY, z / BZ, (uint16_t)T.round);
  slots[i] = ns;
  if (ref_saddle(r)) saddle_out(lm, T, i, lower, valid, __float_as_uint(g[i]));
  if (T.act_next && tgt) atomicOr(&T.act_next[(size_t)row * G.W + (x >> 5)], 1u << (x & 31));
}

#ifndef EXACTZ_LIST_MINB
#define EXACTZ_LIST_MINB 6  // CTAs per SM of the list stencils (latency-bound gathers; 5 / 6 / 8: round 10 of C2 0.90 / 0.83 / 0.87 ms)
#endif
__global__ void __launch_bounds__(256, EXACTZ_LIST_MINB) k_stencil_list(const float *__restrict__ g,
                                                      const uint32_t *__restrict__ ref,
                                                      uint32_t *__restrict__ marks,
                                                      uint8_t *__restrict__ slots,
                                                      uint32_t *__restrict__ lm,
                                                      const int32_t *__restrict__ list,
                                                      const int *__restrict__ count, GridP G,
                                                      Track T, unsigned long long *cnt) {
  const int n = *count;
  unsigned n1 = 0, n2 = 0, n3 = 0, ne = 0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    vertex_pass(__ldg(&list[k]), g, ref, marks, slots, lm, G, T, n1, n2, n3);
    ++ne;
  }
  warp_add(&cnt[C_EVAL], ne);
  warp_add(&cnt[C_N1 + 0], n1);
  warp_add(&cnt[C_N1 + 1], n2);
  warp_add(&cnt[C_N1 + 2], n3);
}

// R4 (C2): adjacent saddles a = S[k] <_f b = S[k+1]; if b <_g a,
// decrease a (the f-smaller).
// (also R7 of the reformulation over the list of all critical points, counted
// in counter `ci`)
__global__ void k_saddle_order(const float *__restrict__ g, const int32_t *__restrict__ S,
                               int nS, uint32_t *marks, GridP G, unsigned long long *cnt,
                               int ci = C_N1 + 3) {
  unsigned n4 = 0;
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k + 1 < nS) {
    int a = S[k], b = S[k + 1];
    if (sos_less_g(g, b, a)) {
      mark_vertex(marks, a, G);
      n4 = 1;
    }
  }
  warp_add(&cnt[ci], n4);
}

// R4 from the saddle values the stencils wrote in S order (gS, value bits):
// pair (S[k], S[k+1]) violates iff S[k+1] <_g S[k]; the f-smaller S[k] is
// marked.  Sequential reads instead of two gathers of g.
__global__ void k_saddle_order_vals(const uint32_t *__restrict__ gS,
                                    const int32_t *__restrict__ S, int nS, uint32_t *marks,
                                    GridP G, unsigned long long *cnt) {
  unsigned n4 = 0;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k + 1 < nS) {
    const float va = __uint_as_float(gS[k]), vb = __uint_as_float(gS[k + 1]);
    const int a = S[k], b = S[k + 1];
    if (vb < va || (vb == va && b < a)) {
      mark_vertex(marks, a, G);
      n4 = 1;
    }
  }
  warp_add(&cnt[C_N1 + 3], n4);
}

__global__ void k_gather_pos(const int32_t *__restrict__ L, int n, const int32_t *__restrict__ pos,
                             int32_t *out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) out[k] = pos[L[k]];
}

__global__ void k_scatter_pos(const int32_t *__restrict__ S, int n, int32_t *pos) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) pos[S[k]] = k;
}

// Terminus of the steepest path from u (O6): follow 4-bit slot pointers.
// FROM_REF: pointers of f (ref word bits 14-17 / 18-21); else of g (slot
// bytes written by the stencil, low / high nibble).  Returns the local root,
// or -(w + 1) for the first vertex w of the path outside the owned planes
// (sharded slabs only; on a single GPU every path stays inside).  A slab's
// ghost-plane slot bytes hold kSelf in both nibbles (set at setup, never
// written), so a g walk stops there by itself and is tested once at its end
// instead of at every step; the ref words of f have no such planes.
template <bool UP, bool FROM_REF, bool SLAB>
__device__ __forceinline__ int walk(int u, const uint8_t *__restrict__ slots,
                                    const uint32_t *__restrict__ ref, const GridP &G) {
  const int A = G.nx * G.ny, lo = G.zb * A, hi = G.ze * A;
  int w = u;
  for (;;) {
    if (SLAB && FROM_REF && (w < lo || w >= hi)) return -(w + 1);
    int s;
    if (FROM_REF) s = (__ldg(&ref[w]) >> (UP ? 18 : 14)) & 15;
    else s = (__ldg(&slots[w]) >> (UP ? 4 : 0)) & 15;
    if (s == kSelf) return (SLAB && !FROM_REF && (w < lo || w >= hi)) ? -(w + 1) : w;
    const int b = slot_bits(s);
    const int d = (b & 1) + ((b >> 1) & 1) * G.nx + (b >> 2) * A;
    w += slot_sign(s) * d;
  }
}

// Boundary tables of a sharded run (z-slabs): for every vertex of the first
// and last owned plane of every rank, the terminus of its steepest path in
// the rank's slab: {label, value bits} (a root) or {-(x+1), 0} (the path
// leaves the slab at global vertex x, which lies in a neighbour's boundary
// plane).  Gathered on every rank; a lookup follows exit -> entry links to
// the root (table_lookup): paths strictly descend (ascend) in SoS order, so
// the chains are acyclic (they visit distinct entries; a path may cross a
// slab border several times, in both z directions).  (r02: resolving the
// whole gathered table on every rank each pass,
// by a cooperative pointer-jumping kernel, was 27 % of the per-rank time of
// an 8-slab C2 run; only the few walks that leave a slab need a chain.)
struct Slabs {
  const int *start;  // start[r] = global first plane of rank r, start[p] = gnz
  int p;
  const int2 *table;  // 2 * p * A entries, or nullptr (single GPU)
  unsigned long long *err;  // set when a chain is longer than the table (never: acyclic)
  int base = 0, extra = 0;  // the split: nz / p planes, the first nz % p ranks one more
};

__device__ __forceinline__ int2 table_entry(const Slabs &S, int xg, int A) {
  const int z = xg / A;
  // the rank owning plane z, from the split rule (exactz_slab_range) instead
  // of a search through start[] (a chain of dependent loads per lookup)
  const int big = S.extra * (S.base + 1);
  const int r = z < big ? z / (S.base + 1) : S.extra + (z - big) / S.base;
  const int zs = r * S.base + min(r, S.extra);
  const int side = (z == zs) ? 0 : 1;
  return S.table[(size_t)(2 * r + side) * A + (xg - z * A)];
}
__device__ __forceinline__ int2 table_lookup(const Slabs &S, int xg, int A) {
  int2 t = table_entry(S, xg, A);
  const int hmax = 2 * S.p * A;  // the table's entries: an acyclic chain visits each once
  for (int h = 0; t.x < 0 && h < hmax; ++h) t = table_entry(S, -t.x - 1, A);
  if (t.x < 0 && S.err) atomicOr(S.err, 1ull);
  return t;
}

template <bool UP, bool FROM_REF>
__global__ void k_boundary_walks(const float *__restrict__ h, const uint8_t *__restrict__ slots,
                                 const uint32_t *__restrict__ ref, GridP G, int2 *out) {
  const int A = G.nx * G.ny;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * A) return;
  const int side = i / A, xy = i - side * A;
  const int v = (side ? G.ze - 1 : G.zb) * A + xy;
  const int e = walk<UP, FROM_REF, true>(v, slots, ref, G);
  const int off = G.zoff * A;
  out[i] = e >= 0 ? make_int2(e + off, __float_as_int(h[e])) : make_int2(-(-e - 1 + off) - 1, 0);
}

// Per-saddle cache of the C3 result (tracking mode).  rnd = round it was
// computed in (0: none), mask = the bricks (relative to the saddle's brick,
// bit (dz+1)*9 + (dy+1)*3 + (dx+1)) holding the saddle's star, every walked
// vertex and the reached extrema; bit 31 = some vertex outside that 3x3x3
// neighbourhood (never reused); tgt = the marked target or -1.
struct EvCache {
  uint16_t *rnd;
  unsigned long long *mask;
  int32_t *tgt;
  const int32_t *lpos;  // positions in S of the list's saddles (masks in S order), or nullptr
};
// mask bits 0..26: bricks (dz+1)*9 + (dy+1)*3 + (dx+1) around the saddle's
// brick; bits 32..58: superbricks likewise for vertices farther away; bit 63:
// a vertex outside both neighbourhoods (never reused).
constexpr unsigned long long kFar = 1ull << 63;
// sharded: some walk left the slab and was completed from the boundary
// tables; the result stays valid while no table entry changed (Track.tab_round)
constexpr unsigned long long kExit = 1ull << 62;
constexpr uint32_t kSuperBits = 0x07FFFFFFu;  // mask bits 32..58

__device__ __forceinline__ void brick_bit(int x, int y, int z, int bsx, int bsy, int bsz,
                                          unsigned long long &mask) {
  // every caller passes in-domain coordinates (>= 0): unsigned shifts
  const unsigned bx = (unsigned)x / BX, by = (unsigned)y / BY, bz = (unsigned)z / BZ;
  const unsigned dx = bx - bsx + 1u, dy = by - bsy + 1u, dz = bz - bsz + 1u;  // 0..2: near
  if (dx <= 2u && dy <= 2u && dz <= 2u) {
    mask |= 1ull << (dz * 9u + dy * 3u + dx);
    return;
  }
  const unsigned ex = bx / SB - (unsigned)bsx / SB + 1u, ey = by / SB - (unsigned)bsy / SB + 1u,
                 ez = bz / SB - (unsigned)bsz / SB + 1u;
  if (ex <= 2u && ey <= 2u && ez <= 2u)
    mask |= 1ull << (32u + ez * 9u + ey * 3u + ex);
  else
    mask |= kFar;
}

// walk() that also records the bricks it visits (g slots).  SLAB: a path
// that leaves the owned planes returns -(w + 1) as walk(); the result then
// depends on the boundary tables (kExit)
template <bool UP, bool SLAB = false>
__device__ __forceinline__ int walk_track(int u, int x, int y, int z,
                                          const uint8_t *__restrict__ slots, const GridP &G,
                                          int bsx, int bsy, int bsz, unsigned long long &mask) {
  const int A = G.nx * G.ny;
  int w = u;
  for (;;) {
    brick_bit(x, y, z, bsx, bsy, bsz, mask);
    const int s = (__ldg(&slots[w]) >> (UP ? 4 : 0)) & 15;
    if (s == kSelf) {  // a root, or (slab) a ghost vertex: see walk()
      if (SLAB && (w < G.zb * A || w >= G.ze * A)) {
        mask |= kExit;
        return -(w + 1);
      }
      return w;
    }
    const int b = slot_bits(s), sg1 = slot_sign(s);
    x += sg1 * (b & 1);
    y += sg1 * ((b >> 1) & 1);
    z += sg1 * (b >> 2);
    w += sg1 * ((b & 1) + ((b >> 1) & 1) * G.nx + (b >> 2) * A);
  }
}

// R5 / R6 (C3): for a join saddle s, m2 = <_h-largest minimum
// reached from the h-lower link; for a split saddle, M2 = <_h-smallest
// maximum from the h-upper link.  16 lanes per saddle, one per slot, each
// walking its own integral path; a 16-lane shuffle reduction picks the
// extremum.  FROM_REF: h = f, the result is m1 / M1 (reference).
// Else h = g: if the pick differs from m1 (M1), mark m2 (join) or
// M1 (split, amb-12).  Saddle lists, m1/M1 and labels are global ids; paths
// leaving a slab are completed from the resolved boundary table; targets
// outside the slab go to `remote` (sharded only).  CACHE: the result, with
// the bricks the saddle depends on, is stored for k_events_check.
template <bool SPLIT, bool FROM_REF, bool CACHE, bool SLAB>
__device__ __forceinline__ unsigned events_group(
    int k, bool active, const float *__restrict__ h, const int32_t *__restrict__ sl,
    const uint8_t *__restrict__ slots, const uint32_t *__restrict__ lm,
    const uint32_t *__restrict__ ref, int32_t *ref_ext, uint32_t *marks, const GridP &G,
    const Slabs &S, int32_t *remote, const EvCache &EC, const Track &T,
    unsigned long long *cnt) {
  const int l16 = threadIdx.x & 15;
  const unsigned gmask = 0xffffu << (threadIdx.x & 16);  // this 16-lane group
  const int A = G.nx * G.ny, off = G.zoff * A;
  int s = 0, sx = 0, sy = 0, sz = 0;
  if (active) {
    s = __ldg(&sl[k]) - off;  // local
    const int yz = div_nx(s, G);
    sx = s - yz * G.nx;
    sz = div_ny(yz, G);
    sy = yz - sz * G.ny;
  }
  const int bsx = sx / BX, bsy = sy / BY, bsz = sz / BZ;
  int best = -1;
  float bv = 0.0f;
  unsigned long long mask = 0;
  if (active && l16 < kSlots) {
    const uint32_t valid = valid_mask(sx, sy, sz, G);
    if (CACHE) brick_bit(sx, sy, sz, bsx, bsy, bsz, mask);
    if (valid & (1u << l16)) {
      const int u = s + slot_delta(l16, G);
      bool lower;
      if (FROM_REF) {
        const float hs = h[s], hu = h[u];
        lower = (l16 < 7) ? (hu <= hs) : (hu < hs);
      } else {
        lower = (saddle_lm(lm, EC.lpos, k, s) >> l16) & 1u;  // the stencil's g-lower mask of s
      }
      const int bb = slot_bits(l16), sg1 = slot_sign(l16);
      const int ux = sx + sg1 * (bb & 1), uy = sy + sg1 * ((bb >> 1) & 1),
                uz = sz + sg1 * (bb >> 2);
      if (CACHE) brick_bit(ux, uy, uz, bsx, bsy, bsz, mask);
      if (lower != SPLIT) {
        if (!FROM_REF) atomicAdd(&cnt[(size_t)(1 + (blockIdx.x & (kCntRep - 1))) * kCntStride + C_LINKS], 1ull);
        int e;
        if constexpr (CACHE) e = walk_track<SPLIT, SLAB>(u, ux, uy, uz, slots, G, bsx, bsy, bsz, mask);
        else e = walk<SPLIT, FROM_REF, SLAB>(u, slots, ref, G);
        if (!SLAB || e >= 0) {
          best = e + off;
          bv = h[e];
        } else {
          const int2 t = table_lookup(S, -e - 1 + off, A);
          best = t.x;
          bv = __int_as_float(t.y);
        }
      }
    }
  }
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) {
    int ob = __shfl_xor_sync(gmask, best, o);
    float ov = __shfl_xor_sync(gmask, bv, o);
    bool take;
    if (ob < 0) take = false;
    else if (best < 0) take = true;
    else if (!SPLIT) take = (bv < ov) || (bv == ov && best < ob);  // SoS max
    else take = (ov < bv) || (ov == bv && ob < best);               // SoS min
    if (take) { best = ob; bv = ov; }
    if (CACHE) mask |= __shfl_xor_sync(gmask, mask, o);
  }
  unsigned hit = 0;
  if (active && l16 == 0) {
    if (FROM_REF) {
      ref_ext[k] = best;
    } else {
      int target = -1;
      const int want = ref_ext[k];
      if (best >= 0 && best != want) target = SPLIT ? want : best;
      if (CACHE) {
        EC.rnd[k] = (uint16_t)T.round;
        EC.mask[k] = mask;
        EC.tgt[k] = target;
      }
      if (target >= 0) {
        const int t = target - off;
        if (!SLAB || (t >= G.zb * A && t < G.ze * A)) mark_vertex(marks, t, G);
        else remote[atomicAdd(&cnt[C_NREMOTE], 1ull)] = target;
        hit = 1;
      }
    }
  }
  return hit;
}

// Same rules, one lane per saddle (the walks are short: a few steps on
// average, so per-lane serial walks keep the issue cost per saddle low).  The
// walk set comes from the stencil's link masks at s (g) or from the f values
// (reference); EXACTZ_EV_KW walks are in flight per lane (independent loads), each
// taking the next slot of the set when it finishes.  Pointer steps decode a
// nibble through a 16-entry shared table of linear offsets (kSelf -> 0).
#ifndef EXACTZ_EV_KW
#define EXACTZ_EV_KW 4  // walks in flight per thread (k_events)
#endif

template <bool UP, bool FROM_REF>
__device__ __forceinline__ int next_slot(int w, const uint8_t *__restrict__ slots,
                                         const uint32_t *__restrict__ ref) {
  if (FROM_REF) return (__ldg(&ref[w]) >> (UP ? 18 : 14)) & 15;
  return (__ldg(&slots[w]) >> (UP ? 4 : 0)) & 15;
}

template <bool SPLIT, bool FROM_REF, bool SLAB>
__global__ void __launch_bounds__(256) k_events(const float *__restrict__ h,
                                                const int32_t *__restrict__ sl, int n,
                                                const uint8_t *__restrict__ slots,
                                                const uint32_t *__restrict__ lm,
                                                const uint32_t *__restrict__ ref,
                                                int32_t *ref_ext, uint32_t *marks, GridP G,
                                                Slabs S, int32_t *remote,
                                                unsigned long long *cnt,
                                                const int *__restrict__ idx = nullptr,
                                                const int *__restrict__ nidx = nullptr,
                                                const int32_t *__restrict__ lpos = nullptr) {
  __shared__ int soff[16];
  if (threadIdx.x < 16) soff[threadIdx.x] = threadIdx.x < kSlots ? slot_delta(threadIdx.x, G) : 0;
  __syncthreads();
  // idx: the saddles to evaluate are idx[0 .. *nidx) (those the clean-path
  // test left, k_fclean), grid-stride over a small grid; else one per thread
  int nact = idx ? *nidx : n;
  if (nact < 0) {  // the clean-path test was skipped (k_fclean's gate): every saddle
    nact = n;
    idx = nullptr;
  }
  const int A = G.nx * G.ny, off = G.zoff * A, lo = G.zb * A, hi = G.ze * A;
  unsigned hit = 0, links = 0;
#ifdef EXACTZ_WALKSTATS
  unsigned nsteps = 0;
#endif
  for (int kk = blockIdx.x * blockDim.x + threadIdx.x; kk < nact;
       kk += gridDim.x * blockDim.x) {
    const int k = idx ? __ldg(&idx[kk]) : kk;
    const int s = __ldg(&sl[k]) - off;  // local
    uint32_t todo;                       // link slots to walk from
    if (FROM_REF) {
      const int yz = div_nx(s, G), sz = div_ny(yz, G);
      const uint32_t valid = valid_mask(s - yz * G.nx, yz - sz * G.ny, sz, G);
      const float hs = h[s];
      uint32_t lower = 0;
#pragma unroll
      for (int q = 0; q < kSlots; ++q)
        if (valid & (1u << q)) {
          const float hu = h[s + soff[q]];
          if ((q < 7) ? (hu <= hs) : (hu < hs)) lower |= 1u << q;
        }
      todo = SPLIT ? (valid & ~lower) : lower;
    } else {
      const uint32_t m = saddle_lm(lm, lpos, k, s);
      todo = SPLIT ? (m >> 16) : (m & 0xFFFFu);
      links += __popc(todo);
    }
    int best = -1;
    float bv = 0.0f;
    // KW walks in flight per thread (independent loads).  The walks are bound
    // by the instructions issued per step, so a step is kept to: the slot
    // load, its nibble, the offset lookup (soff[kSelf] = 0: a root stays put)
    // and the root test; refills run only when a walk has ended.
    constexpr int KW = EXACTZ_EV_KW;
    constexpr unsigned kAll = (1u << KW) - 1u;
    int w[KW];
    unsigned runm = 0;  // bit j: walk j in flight
#pragma unroll
    for (int j = 0; j < KW; ++j) w[j] = 0;
    for (;;) {
      if (runm != kAll && todo) {
#pragma unroll
        for (int j = 0; j < KW; ++j)
          if (!((runm >> j) & 1u) && todo) {
            w[j] = s + soff[__ffs(todo) - 1];
            todo &= todo - 1;
            runm |= 1u << j;
          }
      }
      if (!runm) break;
#ifdef EXACTZ_WALKSTATS
      nsteps += __popc(runm);
#endif
      int sv[KW];
#pragma unroll
      for (int j = 0; j < KW; ++j) {
        sv[j] = kSelf;
        if ((runm >> j) & 1u) {
          // (slab, f walks: the exit into a neighbour's slab is tested per
          // step; g walks stop at the ghost planes' kSelf slots, see walk())
          if (!(SLAB && FROM_REF) || (w[j] >= lo && w[j] < hi))
            sv[j] = next_slot<SPLIT, FROM_REF>(w[j], slots, ref);
          else sv[j] = -1;
        }
      }
#pragma unroll
      for (int j = 0; j < KW; ++j) {
        if (sv[j] >= 0 && sv[j] != kSelf) {
          w[j] += soff[sv[j]];
          continue;
        }
        if (!((runm >> j) & 1u)) continue;
        // a root (or, sharded, the exit into a neighbour's slab)
        runm &= ~(1u << j);
        int lab;
        float val;
        const bool exited = SLAB && (FROM_REF ? sv[j] < 0 : (w[j] < lo || w[j] >= hi));
        if (!exited) {
          lab = w[j] + off;
          val = h[w[j]];
        } else {
          const int2 t = table_lookup(S, w[j] + off, A);
          lab = t.x;
          val = __int_as_float(t.y);
        }
        bool take;
        if (best < 0) take = true;
        else if (!SPLIT) take = (bv < val) || (bv == val && best < lab);  // SoS max
        else take = (val < bv) || (val == bv && lab < best);               // SoS min
        if (take) { best = lab; bv = val; }
      }
    }
    if (FROM_REF) {
      ref_ext[k] = best;
    } else {
      const int want = ref_ext[k];
      if (best >= 0 && best != want) {
        const int target = SPLIT ? want : best;
        const int t = target - off;
        if (!SLAB || (t >= lo && t < hi)) mark_vertex(marks, t, G);
        else remote[atomicAdd(&cnt[C_NREMOTE], 1ull)] = target;
        ++hit;  // (grid-stride over an idx list: several saddles per thread)
      }
    }
  }
  if (!FROM_REF) {
    warp_add(&cnt[C_N1 + 4 + (SPLIT ? 1 : 0)], hit);
    warp_add(&cnt[C_LINKS], links);
#ifdef EXACTZ_WALKSTATS
    warp_add(&cnt[C_WALK], nsteps);
#endif
  }
}

// The rules of k_events (g paths), 16 lanes per saddle, one walk per lane (a
// lane per link slot): the kernel lasts about as long as the longest single
// path instead of a thread's ~7 paths in sequence.  For launches with too few
// saddles to hide the walks' dependent loads (a z-slab holds 1/p of them).
// Same bits as k_events: the same walks, the same SoS pick, the same target.
template <bool SPLIT, bool SLAB>
__global__ void __launch_bounds__(256) k_events16(const float *__restrict__ h,
                                                  const int32_t *__restrict__ sl, int n,
                                                  const uint8_t *__restrict__ slots,
                                                  const uint32_t *__restrict__ lm,
                                                  const int32_t *__restrict__ ref_ext,
                                                  uint32_t *marks, GridP G, Slabs S,
                                                  int32_t *remote, unsigned long long *cnt,
                                                  const int32_t *__restrict__ lpos = nullptr,
                                                  const int *__restrict__ idx = nullptr,
                                                  const int *__restrict__ nidx = nullptr) {
  // idx: the saddles idx[0 .. *nidx) (k_fclean's list; *nidx < 0: the test
  // was skipped, every saddle); else all n
  int nact = idx ? *nidx : n;
  if (nact < 0) {
    nact = n;
    idx = nullptr;
  }
  const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  const int l16 = threadIdx.x & 15;
  const unsigned gmask = 0xffffu << (threadIdx.x & 16);  // this 16-lane group
  const bool active = g < nact;
  const int k = active && idx ? __ldg(&idx[g]) : g;
  const int A = G.nx * G.ny, off = G.zoff * A, lo = G.zb * A, hi = G.ze * A;
  int s = 0;
  uint32_t todo = 0;
  if (active) {
    s = __ldg(&sl[k]) - off;  // local
    const uint32_t m = saddle_lm(lm, lpos, k, s);
    todo = SPLIT ? (m >> 16) : (m & 0xFFFFu);
  }
  int best = -1;
  float bv = 0.0f;
  const bool mine = l16 < kSlots && ((todo >> l16) & 1u);
  if (mine) {
    const int e = walk<SPLIT, false, SLAB>(s + slot_delta(l16, G), slots, nullptr, G);
    if (!SLAB || e >= 0) {
      best = e + off;
      bv = h[e];
    } else {
      const int2 t = table_lookup(S, -e - 1 + off, A);
      best = t.x;
      bv = __int_as_float(t.y);
    }
  }
#pragma unroll
  for (int o = 8; o >= 1; o >>= 1) {
    const int ob = __shfl_xor_sync(gmask, best, o);
    const float ov = __shfl_xor_sync(gmask, bv, o);
    bool take;
    if (ob < 0) take = false;
    else if (best < 0) take = true;
    else if (!SPLIT) take = (bv < ov) || (bv == ov && best < ob);  // SoS max
    else take = (ov < bv) || (ov == bv && ob < best);               // SoS min
    if (take) { best = ob; bv = ov; }
  }
  unsigned hit = 0;
  if (active && l16 == 0) {
    const int want = __ldg(&ref_ext[k]);
    if (best >= 0 && best != want) {
      const int target = SPLIT ? want : best;
      const int t = target - off;
      if (!SLAB || (t >= lo && t < hi)) mark_vertex(marks, t, G);
      else remote[atomicAdd(&cnt[C_NREMOTE], 1ull)] = target;
      hit = 1;
    }
  }
  warp_add(&cnt[C_N1 + 4 + (SPLIT ? 1 : 0)], hit);
  warp_add(&cnt[C_LINKS], mine ? 1u : 0u);
}

// Tracking: a saddle whose cached result is still valid (no brick it depends
// on changed since the cached pass) re-emits it; the others are listed for
// k_events_cached.  One thread per saddle.
// SLAB: saddle ids and targets are global (a target in another slab goes to
// `remote`, as k_events)
template <bool SPLIT, bool SLAB = false>
__global__ void __launch_bounds__(256) k_events_check(const int32_t *__restrict__ sl, int n,
                                                      EvCache EC, Track T, uint32_t *marks,
                                                      GridP G, int *todo, int *ntodo,
                                                      unsigned long long *cnt,
                                                      const int *__restrict__ idx = nullptr,
                                                      const int *__restrict__ nidx = nullptr,
                                                      int32_t *remote = nullptr) {
  const int A = G.nx * G.ny, off = SLAB ? G.zoff * A : 0;
  // idx: only the saddles idx[0 .. *nidx) (left by k_fclean); else all n
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  bool act = k < n;
  if (idx) {
    act = k < *nidx;
    if (act) k = __ldg(&idx[k]);
  }
  bool valid = false;
  unsigned hit = 0;
  if (act) {
    const uint16_t rnd = EC.rnd[k];
    const unsigned long long mask = EC.mask[k];  // zeroed when the cache started
    valid = rnd != 0 && !(mask & kFar) && (!(mask & kExit) || rnd >= T.tab_round);
    if (valid) {
      const int s = sl[k] - off;
      const int yz = div_nx(s, G), sz = div_ny(yz, G), sx = s - yz * G.nx, sy = yz - sz * G.ny;
      const int bsx = sx / BX, bsy = sy / BY, bsz = sz / BZ;
      // the stamps of up to 4 bricks in flight per step (independent loads)
      uint32_t m = (uint32_t)mask, ms = (uint32_t)(mask >> 32) & kSuperBits;
      while ((m | ms) && valid) {
        uint16_t st[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          st[2 * q] = st[2 * q + 1] = 0;
          if (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            const int dz = j / 9 - 1, dy = (j / 3) % 3 - 1, dx = j % 3 - 1;
            const int nb = (bsx + dx) + T.nbx * ((bsy + dy) + T.nby * (bsz + dz));
            st[2 * q] = T.bval[nb];
            st[2 * q + 1] = T.bslot[nb];
          } else if (ms) {
            const int j = __ffs(ms) - 1;
            ms &= ms - 1;
            const int dz = j / 9 - 1, dy = (j / 3) % 3 - 1, dx = j % 3 - 1;
            const int nb = (bsx / SB + dx) + T.nsx * ((bsy / SB + dy) + T.nsy * (bsz / SB + dz));
            st[2 * q] = T.sbval[nb];
            st[2 * q + 1] = T.sbslot[nb];
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (st[q] > rnd) valid = false;
      }
    }
    if (valid) {
      const int t = EC.tgt[k];
      if (t >= 0) {
        if (!SLAB || (t - off >= G.zb * A && t - off < G.ze * A)) mark_vertex(marks, t - off, G);
        else remote[atomicAdd(&cnt[C_NREMOTE], 1ull)] = t;
        hit = 1;
      }
    }
  }
  // CTA-aggregated append of the saddles to recompute: one atomic per CTA
  // (per warp, the same-address atomics queued at one L2 slice)
  __shared__ int wcnt[8], wbase[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned need = __ballot_sync(0xffffffffu, act && !valid);
  if (lane == 0) wcnt[wid] = __popc(need);
  __syncthreads();
  if (wid == 0) {
    const int c = lane < 8 ? wcnt[lane] : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const int tot = __shfl_sync(0xffffffffu, inc, 7);
    int base = 0;
    if (lane == 0 && tot) base = atomicAdd(ntodo, tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (lane < 8) wbase[lane] = base + inc - c;
  }
  __syncthreads();
  if ((need >> lane) & 1u) todo[wbase[wid] + __popc(need & ((1u << lane) - 1u))] = k;
  warp_add(&cnt[C_N1 + 4 + (SPLIT ? 1 : 0)], hit);
}

// Recompute (and cache) the listed saddles, one lane per saddle as in
// k_events, recording the bricks the result depends on: the saddle's closed
// star (its link masks come from those values) and every vertex of every walk
// (a slot change anywhere on a path can move its root).
template <bool SPLIT, bool SLAB = false>
__global__ void __launch_bounds__(256) k_events_cached(const float *__restrict__ h,
                                                       const int32_t *__restrict__ sl,
                                                       const int *__restrict__ todo,
                                                       const int *__restrict__ ntodo,
                                                       const uint8_t *__restrict__ slots,
                                                       const uint32_t *__restrict__ lm,
                                                       int32_t *ref_ext, uint32_t *marks,
                                                       GridP G, EvCache EC, Track T,
                                                       unsigned long long *cnt,
                                                       const int *__restrict__ todo2 = nullptr,
                                                       const int *__restrict__ ntodo2 = nullptr,
                                                       Slabs S = Slabs{nullptr, 1, nullptr},
                                                       int32_t *remote = nullptr) {
  __shared__ int soff[16], sdel[16];  // linear offset; packed (dx+1, dy+1, dz+1)
  if (threadIdx.x < 16) {
    const int q = threadIdx.x;
    soff[q] = q < kSlots ? slot_delta(q, G) : 0;
    int p = 1 | (1 << 2) | (1 << 4);
    if (q < kSlots) {
      const int b = slot_bits(q), sg1 = slot_sign(q);
      p = (1 + sg1 * (b & 1)) | ((1 + sg1 * ((b >> 1) & 1)) << 2) | ((1 + sg1 * (b >> 2)) << 4);
    }
    sdel[q] = p;
  }
  __syncthreads();
  int n = *ntodo;
  if (n < 0) {  // the clean-path test was skipped: the stamp check's list
    todo = todo2;
    n = *ntodo2;
  }
  unsigned hit = 0, links = 0;
#ifdef EXACTZ_WALKSTATS
  unsigned nsteps = 0;
#endif
  if (n * 16 <= (int)(gridDim.x * blockDim.x)) {
    // few saddles (late passes: mostly long walks that never stay cached):
    // 16 lanes per saddle, one walk per lane, for the shortest critical path
    const int g = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
    const bool active = g < n;
    hit = events_group<SPLIT, false, true, SLAB>(active ? todo[g] : 0, active, h, sl, slots, lm,
                                                 nullptr, ref_ext, marks, G, S, remote, EC, T,
                                                 cnt);
    warp_add(&cnt[C_N1 + 4 + (SPLIT ? 1 : 0)], hit);
    return;
  }
  const int A = G.nx * G.ny, off = SLAB ? G.zoff * A : 0, lo = G.zb * A, hi = G.ze * A;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < n; g += gridDim.x * blockDim.x) {
    const int k = todo[g];
    const int s = __ldg(&sl[k]) - off;
    const int yz = div_nx(s, G), sz = div_ny(yz, G);
    const int sx = s - yz * G.nx, sy = yz - sz * G.ny;
    const int bsx = sx / BX, bsy = sy / BY, bsz = sz / BZ;
    const uint32_t m = saddle_lm(lm, EC.lpos, k, s);
    unsigned long long mask = 0;
    brick_bit(sx, sy, sz, bsx, bsy, bsz, mask);
    for (uint32_t v = (m | (m >> 16)) & 0x3FFFu; v; v &= v - 1) {  // the star
      const int p = sdel[__ffs(v) - 1];
      brick_bit(sx + (p & 3) - 1, sy + ((p >> 2) & 3) - 1, sz + (p >> 4) - 1, bsx, bsy, bsz, mask);
    }
    uint32_t rest = SPLIT ? (m >> 16) : (m & 0xFFFFu);
    links += __popc(rest);
    int best = -1;
    float bv = 0.0f;
    int w[2] = {0, 0}, x[2] = {0, 0}, y[2] = {0, 0}, z[2] = {0, 0};
    unsigned runm = 0;  // bit j: walk j in flight (refills only after a walk ends, as k_events)
    for (;;) {
      if (runm != 3u && rest) {
#pragma unroll
        for (int j = 0; j < 2; ++j)
          if (!((runm >> j) & 1u) && rest) {
            const int q = __ffs(rest) - 1, p = sdel[q];
            rest &= rest - 1;
            w[j] = s + soff[q];
            x[j] = sx + (p & 3) - 1;
            y[j] = sy + ((p >> 2) & 3) - 1;
            z[j] = sz + (p >> 4) - 1;
            runm |= 1u << j;
          }
      }
      if (!runm) break;
#ifdef EXACTZ_WALKSTATS
      nsteps += __popc(runm);
#endif
      int sv[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        sv[j] = kSelf;
        if ((runm >> j) & 1u) {
          sv[j] = (__ldg(&slots[w[j]]) >> (SPLIT ? 4 : 0)) & 15;  // (ghosts: kSelf, see walk())
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (sv[j] >= 0 && sv[j] != kSelf) {
          const int p = sdel[sv[j]];
          w[j] += soff[sv[j]];
          x[j] += (p & 3) - 1;
          y[j] += ((p >> 2) & 3) - 1;
          z[j] += (p >> 4) - 1;
          brick_bit(x[j], y[j], z[j], bsx, bsy, bsz, mask);
          continue;
        }
        if (!((runm >> j) & 1u)) continue;
        runm &= ~(1u << j);
        int lab;
        float val;
        if (!SLAB || (w[j] >= lo && w[j] < hi)) {
          lab = w[j] + off;
          val = h[w[j]];
        } else {  // completed from the boundary tables
          const int2 t = table_lookup(S, w[j] + off, A);
          lab = t.x;
          val = __int_as_float(t.y);
          mask |= kExit;
        }
        bool take;
        if (best < 0) take = true;
        else if (!SPLIT) take = (bv < val) || (bv == val && best < lab);  // SoS max
        else take = (val < bv) || (val == bv && lab < best);               // SoS min
        if (take) { best = lab; bv = val; }
      }
    }
    int target = -1;
    const int want = ref_ext[k];
    if (best >= 0 && best != want) target = SPLIT ? want : best;
    EC.rnd[k] = (uint16_t)T.round;
    EC.mask[k] = mask;
    EC.tgt[k] = target;
    if (target >= 0) {
      if (!SLAB || (target - off >= lo && target - off < hi)) mark_vertex(marks, target - off, G);
      else remote[atomicAdd(&cnt[C_NREMOTE], 1ull)] = target;
      ++hit;  // a lane may recompute several saddles (grid-stride)
    }
  }
  warp_add(&cnt[C_N1 + 4 + (SPLIT ? 1 : 0)], hit);
  warp_add(&cnt[C_LINKS], links);
#ifdef EXACTZ_WALKSTATS
  warp_add(&cnt[C_WALK], nsteps);
#endif
}

// ------------------------------------------- clean-path test (NEXT-2)
// Incremental labels (P:309 and P:581 name path tracing
// as the cost).  If no vertex on the f-walks from the f-lower link of a join
// saddle s has dn_g != dn_f, and L_g(s) = L_f(s), then every g-walk of R5 is
// the f-walk from the same vertex, so X = {lab_dn_g(u) : u in L_g(s)} is the
// set X_f of the f-labels, computed once here, and m2 = max_<g X_f needs the
// g-values of its few elements only (no walk).  Split saddles likewise with
// up pointers and U.  "Dirty" is tested per 8x4x4 tile: the list stencil
// flags the tiles of the vertices whose g-pointer differs from f's (a vertex
// not evaluated in a list pass did not fire in its last evaluation, so its
// pointers are f's).  The tiles each saddle's f-walks visit are listed once.
constexpr int kFLab = 8;  // distinct f-labels kept per saddle (more: always walked)
struct FPaths {
  const int64_t *off;    // [n] first tile entry of each saddle (a warp's 32 lists are contiguous)
  const uint16_t *len;   // [n] its number of tile entries
  const int32_t *tiles;  // tiles visited by the f-walks (consecutive repeats dropped)
  const int32_t *lab;    // [n * kFLab] the distinct f-termini X_f
  const uint8_t *nlab;   // [n] |X_f|, 255 when more than kFLab
  const unsigned long long *bmask;  // [n] bricks of the star and the f-walks (EvCache format)
  const uint16_t *flow;  // [n] the saddle's f-lower mask (its link partition in f)
  const int32_t *lpos;   // positions in S (link masks in S order), or nullptr
  const uint8_t *dirt;   // [ntiles] this pass's dirty tiles (dirtD / dirtU)
  int nt;                // ntiles
  unsigned long long cap;  // capacity of tiles (setup)
  const unsigned long long *ndirt;  // dirty tiles of `dirt` this pass (device)
  unsigned long long max_dirt;      // k_fclean's gate: skip above this many
};

// Setup: the f-walks of every saddle of the list, from its f-lower (join) /
// f-upper (split) link along f's steepest slots (ref word), one thread per
// saddle: m1 / M1 (ext; the reference of P:298-299, in place of k_events'
// FROM_REF walks), the tiles visited (buffered per thread, at most kFTileCap; longer
// lists, or a full tile array, make the saddle "always walked"), X_f, and the
// bricks of its star and walks for the brick-stamp cache.  A warp reserves
// one contiguous run for its 32 lists (k_fclean scans it coalesced).
constexpr int kFTileCap = 512;
static_assert(kFTileCap <= 65535, "FPaths::len is 16-bit");
// SLAB (a z-slab of the sharded call): ids local to the slab (lab[] holds
// local vertex ids; k_fclean adds the offset), a walk that leaves the owned
// planes makes its saddle "always walked" (its tiles beyond are another
// rank's), and ext (m1 / M1, from the boundary tables) is not written.
template <bool SPLIT, bool SLAB = false>
__global__ void __launch_bounds__(256) k_fpaths(const int32_t *__restrict__ sl, int n,
                                                const uint32_t *__restrict__ ref, GridP G,
                                                int ntx, int nty, unsigned long long *bump,
                                                unsigned long long cap, int64_t *off,
                                                uint16_t *len, int32_t *tiles, int32_t *lab,
                                                uint8_t *nlab, unsigned long long *bmask,
                                                unsigned long long *diag,
                                                const float *__restrict__ f, int32_t *ext,
                                                uint16_t *fflow,
                                                const uint8_t *__restrict__ fslots) {
  __shared__ int soff[16], sdel[16];  // linear offset; packed (dx+1, dy+1, dz+1)
  if (threadIdx.x < 16) {
    const int q = threadIdx.x;
    soff[q] = q < kSlots ? slot_delta(q, G) : 0;
    int p = 1 | (1 << 2) | (1 << 4);
    if (q < kSlots) {
      const int b = slot_bits(q), sg1 = slot_sign(q);
      p = (1 + sg1 * (b & 1)) | ((1 + sg1 * ((b >> 1) & 1)) << 2) | ((1 + sg1 * (b >> 2)) << 4);
    }
    sdel[q] = p;
  }
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const bool act = k < n;
  int32_t buf[kFTileCap];
  int e = 0, nl = 0;
  int best = -1;  // m1 (join) / M1 (split): the SoS-extreme terminus
  float bv = 0.0f;
  int lb[kFLab];
#pragma unroll
  for (int j = 0; j < kFLab; ++j) lb[j] = -1;
  unsigned long long mask = 0;
  bool exited = false;
  if (act) {
    const int A = G.nx * G.ny, lo = G.zb * A, hi = G.ze * A;
    const int s = __ldg(&sl[k]) - (SLAB ? G.zoff * A : 0);
    const int yz = div_nx(s, G), sz = div_ny(yz, G);
    const int sx = s - yz * G.nx, sy = yz - sz * G.ny;
    const uint32_t valid = valid_mask(sx, sy, sz, G), flow = ref_flow(__ldg(&ref[s]));
    fflow[k] = (uint16_t)flow;
    // bricks a cached result of s depends on while its walks are f's (as
    // k_events_cached records them): the closed star and every walked vertex
    // (tiles nest in bricks: one brick bit per new tile)
    const int bsx = sx / BX, bsy = sy / BY, bsz = sz / BZ;
    brick_bit(sx, sy, sz, bsx, bsy, bsz, mask);
    for (uint32_t v = valid; v; v &= v - 1) {
      const int p = sdel[__ffs(v) - 1];
      brick_bit(sx + (p & 3) - 1, sy + ((p >> 2) & 3) - 1, sz + (p >> 4) - 1, bsx, bsy, bsz, mask);
    }
    int last = -1, last2 = -1;  // the last two tiles listed (walks of one saddle overlap)
    // one walk at a time (two in flight measured slower: C2 0.38 -> 0.51 ms,
    // C3 8.7 -> 10.4 ms for the join list)
    for (uint32_t todo = SPLIT ? (valid & ~flow) : flow; todo; todo &= todo - 1) {
      const int q = __ffs(todo) - 1;
      int p = sdel[q], w = s + soff[q];
      int x = sx + (p & 3) - 1, y = sy + ((p >> 2) & 3) - 1, z = sz + (p >> 4) - 1;
      for (;;) {
        if (SLAB && (w < lo || w >= hi)) {
          exited = true;
          break;
        }
        const int t = ftile(x, y, z, ntx, nty);
        if (t != last && t != last2) {
          if (e < kFTileCap) buf[e] = t;
          ++e;
          last2 = last;
          last = t;
          brick_bit(x, y, z, bsx, bsy, bsz, mask);
        }
        const int sv = fslots ? (__ldg(&fslots[w]) >> (SPLIT ? 4 : 0)) & 15
                              : (__ldg(&ref[w]) >> (SPLIT ? 18 : 14)) & 15;
        if (sv == kSelf) break;
        p = sdel[sv];
        w += soff[sv];
        x += (p & 3) - 1;
        y += ((p >> 2) & 3) - 1;
        z += (p >> 4) - 1;
      }
      if (SLAB && exited) break;
      {  // a terminus: m1 / M1 and X_f
        const float val = SLAB ? 0.0f : f[w];
        bool take;
        if (best < 0) take = true;
        else if (!SPLIT) take = (bv < val) || (bv == val && best < w);  // SoS max
        else take = (val < bv) || (val == bv && w < best);               // SoS min
        if (take) { best = w; bv = val; }
      }
      bool seen = false;
#pragma unroll
      for (int j = 0; j < kFLab; ++j) seen |= lb[j] == w;
      if (!seen) {
#pragma unroll
        for (int j = 0; j < kFLab; ++j)
          if (j == nl) lb[j] = w;
        ++nl;
      }
    }
  }
  // one reservation per warp, lists in lane order
  const int lane = threadIdx.x & 31;
  // (a reserved run holds no holes: k_fclean scans the warp's run whole)
  const bool want = act && e <= kFTileCap && nl <= kFLab && !exited;
  const int c = want ? e : 0;
  int inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  const int tot = __shfl_sync(0xffffffffu, inc, 31);
  unsigned long long base = 0;
  if (lane == 0 && tot) base = atomicAdd(bump, (unsigned long long)tot);
  base = __shfl_sync(0xffffffffu, base, 0);
  const bool fits = base + (unsigned long long)tot <= cap;
  if (!act) return;
  const bool ok = fits && want;
  if (diag) {  // saddles left to the walks: list too long, too many labels, array full; entries
    if (e > kFTileCap) atomicAdd(&diag[0], 1ull);
    if (nl > kFLab) atomicAdd(&diag[1], 1ull);
    if (want && !fits) atomicAdd(&diag[2], 1ull);
    if (ok) atomicAdd(&diag[3], (unsigned long long)e);
  }
  const unsigned long long o0 = base + (unsigned long long)(inc - c);
  if (ok)
    for (int j = 0; j < e; ++j) tiles[o0 + j] = buf[j];
  off[k] = (int64_t)o0;
  len[k] = (uint16_t)(ok ? e : 0);
  bmask[k] = mask;
  nlab[k] = (uint8_t)(ok ? nl : 255);  // 255: always walked
#pragma unroll
  for (int j = 0; j < kFLab; ++j) lab[(size_t)k * kFLab + j] = lb[j];
  if (!SLAB) ext[k] = best;
}

// CTA-aggregated append of k to todo for the threads with `need` (one atomic
// per CTA; any block size <= 1024).  Every thread of the block must call it.
__device__ __forceinline__ void cta_append(bool need, int k, int *todo, int *ntodo) {
  __shared__ int wcnt[32], wbase[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, need);
  if (lane == 0) wcnt[wid] = __popc(m);
  __syncthreads();
  if (wid == 0) {
    const int c = lane < nw ? wcnt[lane] : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const int tot = __shfl_sync(0xffffffffu, inc, 31);
    int base = 0;
    if (lane == 0 && tot) base = atomicAdd(ntodo, tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (lane < nw) wbase[lane] = base + inc - c;
  }
  __syncthreads();
  if ((m >> lane) & 1u) todo[wbase[wid] + __popc(m & ((1u << lane) - 1u))] = k;
  __syncthreads();  // wcnt / wbase are reused by the next call
}

// CTA-aggregated append to a list counted by *n (64-bit): returns this
// thread's position if `need`, else -1; one atomic per CTA.  Every thread of
// the block calls it (it synchronises the block).
__device__ __forceinline__ long long cta_slot(bool need, unsigned long long *n) {
  __shared__ int wcnt[32];
  __shared__ unsigned long long wbase[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  const unsigned m = __ballot_sync(0xffffffffu, need);
  if (lane == 0) wcnt[wid] = __popc(m);
  __syncthreads();
  if (wid == 0) {
    const int c = lane < nw ? wcnt[lane] : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const int tot = __shfl_sync(0xffffffffu, inc, 31);
    unsigned long long base = 0;
    if (lane == 0 && tot) base = atomicAdd(n, (unsigned long long)tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (lane < nw) wbase[lane] = base + (unsigned long long)(inc - c);
  }
  __syncthreads();
  const long long r = need ? (long long)(wbase[wid] + __popc(m & ((1u << lane) - 1u))) : -1;
  __syncthreads();  // wcnt / wbase are reused by the next call
  return r;
}

// Per pass: a saddle whose link partition is f's and whose f-walk tiles are
// all clean takes X = X_f (R5 / R6 without walks); the others are listed in
// todo for the walk kernels.  idx: only the saddles idx[0 .. *nidx) (those
// the brick-stamp cache left, k_events_check); EC.rnd: a clean saddle's
// result is cached with the bricks of its star and f-walks (its g-walks), so
// later passes re-emit it while those bricks are unchanged.  Grid-stride
// (block-uniform trip count): a launch over a short idx list stays small.
// SLAB: saddle ids global, F.lab local (see k_fpaths), a target in another
// slab goes to `remote`
template <bool SPLIT, bool SLAB = false>
__global__ void __launch_bounds__(256) k_fclean(const float *__restrict__ g,
                                                const int32_t *__restrict__ sl, int n,
                                                const uint32_t *__restrict__ lm,
                                                const uint32_t *__restrict__ ref, FPaths F,
                                                const int32_t *__restrict__ ref_ext,
                                                uint32_t *marks, GridP G, int *todo, int *ntodo,
                                                unsigned long long *cnt,
                                                const int *__restrict__ idx,
                                                const int *__restrict__ nidx, EvCache EC,
                                                int round, const unsigned long long *ndirt,
                                                unsigned long long max_dirt,
                                                int32_t *remote = nullptr) {
  const int A = G.nx * G.ny, off = SLAB ? G.zoff * A : 0;
  // gate: with more than max_dirt dirty tiles few saddles are clean; the
  // test is skipped and the walk kernels take every saddle (*ntodo = -1)
  if (*ndirt > max_dirt) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *ntodo = -1;
    return;
  }
  auto dirty = [&](int t) -> uint32_t { return __ldg(&F.dirt[t]); };
  const int lane = threadIdx.x & 31;
  const int nact = idx ? *nidx : n;
  unsigned hit = 0;
  // block-uniform trip count (cta_append synchronises the block)
  for (int base = blockIdx.x * blockDim.x; base < nact; base += gridDim.x * blockDim.x) {
    const int kk = base + threadIdx.x;
    const bool act = kk < nact;
    const int k = act ? (idx ? __ldg(&idx[kk]) : kk) : 0;
    bool need = false;
    int s = 0, nl = 0;
    if (act) {
      s = __ldg(&sl[k]) - off;
      nl = F.nlab[k];
      need = nl > kFLab || ((saddle_lm(lm, F.lpos, k, s) ^ F.flow[k]) & 0x3FFFu) != 0;
    }
    if (!idx) {
      // the warp's 32 saddles own one contiguous run of tile entries: scan it
      // 32 entries at a time (coalesced), each lane testing the dirty entries
      // of the window against its own range
      const int64_t o0 = act ? F.off[k] : 0, o1 = act ? o0 + F.len[k] : 0;
      const int64_t E0 = __shfl_sync(0xffffffffu, o0, 0);
      const int64_t E1 =
          (int64_t)__reduce_max_sync(0xffffffffu, act ? (unsigned)(o1 - E0) : 0u) + E0;
      for (int64_t eb = E0; eb < E1; eb += 32) {
        if (__all_sync(0xffffffffu, need || !act)) break;
        const int64_t e = eb + lane;
        const bool d = e < E1 && dirty(__ldg(&F.tiles[e]));
        const unsigned D = __ballot_sync(0xffffffffu, d);
        if (D && act && !need) {
          const int64_t lo = o0 > eb ? o0 : eb, hi = o1 < eb + 32 ? o1 : eb + 32;
          if (lo < hi) {
            const int a = (int)(lo - eb), b = (int)(hi - eb);
            const unsigned rm = (b >= 32 ? 0xffffffffu : ((1u << b) - 1u)) & ~((1u << a) - 1u);
            need = (D & rm) != 0;
          }
        }
      }
    } else if (act && !need) {
      const int64_t e0 = F.off[k], e1 = e0 + F.len[k];
      for (int64_t e = e0; e < e1 && !need; e += 4) {  // four tiles in flight
        uint32_t d = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (e + j < e1) d |= dirty(__ldg(&F.tiles[e + j]));
        need = d != 0;
      }
    }
    if (act && !need) {
      int best = -1;
      float bv = 0.0f;
      for (int j = 0; j < nl; ++j) {
        const int lab = __ldg(&F.lab[(size_t)k * kFLab + j]);
        const float val = g[lab];
        bool take;
        if (best < 0) take = true;
        else if (!SPLIT) take = (bv < val) || (bv == val && best < lab);  // SoS max
        else take = (val < bv) || (val == bv && lab < best);               // SoS min
        if (take) { best = lab; bv = val; }
      }
      const int want = __ldg(&ref_ext[k]);
      int target = -1;
      if (best >= 0 && best + off != want) {
        target = SPLIT ? want : best + off;  // global
        const int t = target - off;
        if (!SLAB || (t >= G.zb * A && t < G.ze * A)) mark_vertex(marks, t, G);
        else remote[atomicAdd(&cnt[C_NREMOTE], 1ull)] = target;
        ++hit;
      }
      if (EC.rnd) {
        EC.rnd[k] = (uint16_t)round;
        EC.mask[k] = F.bmask[k];
        EC.tgt[k] = target;
      }
    }
    cta_append(act && need, k, todo, ntodo);
  }
  warp_add(&cnt[C_N1 + 4 + (SPLIT ? 1 : 0)], hit);
}

// ------------------------------------------------ sharded helpers (z-slabs)
// The g boundary tables of a pass after the first, both directions in one
// launch (4A entries: dir, side, xy): each entry of this rank is recomputed,
// and one that differs from the replicated table's is written there and
// listed {position in the table pair [dn | up], label, value bits} for the
// other ranks (sparse all-gather); the tables stay equal on every rank.
// CACHE (the C3 cache is on): an entry whose walk visited no brick stamped
// since it was walked (value or slot change, kernels.cuh Track) is unchanged
// and not walked again; the exit into a neighbour's slab is a position, not
// data, so every entry is cacheable (unless its path left the superbrick
// neighbourhood: kFar).  brnd / bmask: the round and bricks of each entry.
template <bool CACHE>
__global__ void k_boundary_delta(const float *__restrict__ h, const uint8_t *__restrict__ slots,
                                 GridP G, int rank, int p, int2 *tab, int4 *upd,
                                 unsigned long long *nupd, Track T = Track{},
                                 uint16_t *brnd = nullptr, unsigned long long *bmask = nullptr) {
  const int A = G.nx * G.ny;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool chg = false;
  int pos = 0;
  int2 val = make_int2(0, 0);
  if (i < 4 * A) {
    const int dir = i >= 2 * A, j = i - dir * 2 * A, side = j >= A, xy = j - side * A;
    const int lo = G.zb * A, hi = G.ze * A, sh = dir ? 4 : 0;
    int y = xy / G.nx, x = xy - y * G.nx, z = side ? G.ze - 1 : G.zb;
    const int bsx = x / BX, bsy = y / BY, bsz = z / BZ;
    bool walk = true;
    if (CACHE) {
      const uint16_t r0 = brnd[i];
      const unsigned long long m0 = bmask[i];
      if (r0 != 0 && !(m0 & kFar)) {
        walk = false;
        uint32_t m = (uint32_t)m0, ms = (uint32_t)(m0 >> 32);
        while ((m | ms) && !walk) {
          uint16_t a, b;
          if (m) {
            const int q = __ffs(m) - 1;
            m &= m - 1;
            const int nb = (bsx + q % 3 - 1) + T.nbx * ((bsy + (q / 3) % 3 - 1) + T.nby * (bsz + q / 9 - 1));
            a = T.bval[nb];
            b = T.bslot[nb];
          } else {
            const int q = __ffs(ms) - 1;
            ms &= ms - 1;
            const int nb = (bsx / SB + q % 3 - 1) +
                           T.nsx * ((bsy / SB + (q / 3) % 3 - 1) + T.nsy * (bsz / SB + q / 9 - 1));
            a = T.sbval[nb];
            b = T.sbslot[nb];
          }
          if (a > r0 || b > r0) walk = true;
        }
      }
    }
    if (walk) {
      unsigned long long mask = 0;
      int w = (side ? G.ze - 1 : G.zb) * A + xy, e;
      for (;;) {  // walk(): the steepest path of g inside the slab (ghosts: kSelf)
        if (CACHE) brick_bit(x, y, z, bsx, bsy, bsz, mask);
        const int sl = (__ldg(&slots[w]) >> sh) & 15;
        if (sl == kSelf) {
          e = (w < lo || w >= hi) ? -(w + 1) : w;
          break;
        }
        const int b = slot_bits(sl), sg1 = slot_sign(sl);
        x += sg1 * (b & 1);
        y += sg1 * ((b >> 1) & 1);
        z += sg1 * (b >> 2);
        w += sg1 * ((b & 1) + ((b >> 1) & 1) * G.nx + (b >> 2) * A);
      }
      if (CACHE) {
        brnd[i] = (uint16_t)T.round;
        bmask[i] = mask;
      }
      const int off = G.zoff * A;
      val = e >= 0 ? make_int2(e + off, __float_as_int(h[e])) : make_int2(-(-e - 1 + off) - 1, 0);
      pos = dir * 2 * p * A + (2 * rank + side) * A + xy;
      const int2 old = tab[pos];
      chg = old.x != val.x || old.y != val.y;
      if (chg) tab[pos] = val;
    }
  }
  // warp-aggregated append
  const long long q = cta_slot(chg, nupd);  // (a dense pass changes most entries)
  if (q >= 0) upd[q] = make_int4(pos, val.x, val.y, 0);
}
// Labels of a slab's owned vertices (the optional label outputs of the
// sharded call): the steepest pointers of the final field inside the slab
// (a pointer into a ghost plane becomes the exit -(global id + 1)), local
// pointer jumping, then exits completed from the boundary tables.
__global__ void k_slab_ptrs(const uint8_t *__restrict__ slots, int32_t *p, GridP G, int up) {
  const int A = G.nx * G.ny, lo = G.zb * A, hi = G.ze * A;
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hi) return;
  const int t = slot_target(i, (slots[i] >> (up ? 4 : 0)) & 15, G);
  p[i] = (t >= lo && t < hi) ? t : -(t + G.zoff * A) - 1;
}
__global__ void k_jump_slab(int32_t *lab, GridP G, unsigned long long *changed) {
  const int A = G.nx * G.ny, lo = G.zb * A, hi = G.ze * A;
  unsigned c = 0;
  for (int i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += gridDim.x * blockDim.x) {
    const int w = lab[i];
    if (w < 0) continue;  // an exit: resolved by the tables
    const int w2 = lab[w];
    if (w2 != w) {
      lab[i] = w2;
      c = 1;
    }
  }
  if (__any_sync(0xffffffffu, c) && (threadIdx.x & 31) == 0) atomicOr(changed, 1ull);
}
__global__ void k_slab_resolve(const int32_t *__restrict__ lab, GridP G, Slabs S, int32_t *out) {
  const int A = G.nx * G.ny, lo = G.zb * A, hi = G.ze * A;
  const int i = lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hi) return;
  const int w = lab[i];
  out[i - lo] = w >= 0 ? w + G.zoff * A : table_lookup(S, -w - 1, A).x;
}

// A slab's ghost planes after the halo refresh: a vertex whose value changed
// (the neighbour's edit of its boundary plane) stamps its brick as an edit of
// this pass does (round + 1), so the C3 cache sees a saddle star or a walk
// that reads it change; prev keeps the planes' last values.
__global__ void k_ghost_stamp(const float *__restrict__ g, float *prev, GridP G, Track T) {
  const int A = G.nx * G.ny;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 2 * A) return;
  const int side = i >= A, xy = i - side * A, z = side ? G.nz - 1 : 0;
  const float v = g[(size_t)z * A + xy];
  if (__float_as_uint(v) == __float_as_uint(prev[i])) return;
  prev[i] = v;
  const int y = xy / G.nx, x = xy - y * G.nx;
  stamp(T.bval, T.sbval, T, x / BX, y / BY, z / BZ, (uint16_t)(T.round + 1));
}

// gathered table updates (position < 0: padding)
__global__ void k_apply_tab(const int4 *__restrict__ upd, int n, int2 *tab) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int4 u = upd[k];
  if (u.x >= 0) tab[u.x] = make_int2(u.y, u.z);
}


// R4 with the replicated saddle values gS (uint32 bit patterns, S order):
// the owner of S[k] checks the pair (S[k], S[k+1]).
// own: only the positions k of the pairs whose S[k] the slab owns (nown of them)
__global__ void k_saddle_order_slab(const uint32_t *__restrict__ gS,
                                    const int32_t *__restrict__ S, int nS, uint32_t *marks,
                                    GridP G, unsigned long long *cnt, int ci = C_N1 + 3,
                                    const int32_t *__restrict__ own = nullptr, int nown = 0) {
  unsigned n4 = 0;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = own ? (j < nown ? __ldg(&own[j]) : nS) : j;
  const int A = G.nx * G.ny, off = G.zoff * A;
  if (k + 1 < nS) {
    const int a = S[k] - off;
    if (a >= G.zb * A && a < G.ze * A) {
      const float va = __int_as_float(gS[k]), vb = __int_as_float(gS[k + 1]);
      if (vb < va || (vb == va && S[k + 1] < S[k])) {
        mark_vertex(marks, a, G);
        n4 = 1;
      }
    }
  }
  warp_add(&cnt[ci], n4);
}

// S[k] lies in the owned planes [lo, hi) (global ids): R4's pairs of a slab
struct OwnedInS {
  const int32_t *S;
  int lo, hi;
  __device__ __forceinline__ bool operator()(int k) const {
    const int a = S[k];
    return a >= lo && a < hi;
  }
};

// gS[k] = bits of g at S[k] for owned saddles, 0 elsewhere (max-all-reduced)
__global__ void k_fill_gS(const float *__restrict__ g, const int32_t *__restrict__ S, int nS,
                          uint32_t *gS, GridP G) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nS) return;
  const int A = G.nx * G.ny, a = S[k] - G.zoff * A;
  gS[k] = (a >= G.zb * A && a < G.ze * A) ? __float_as_uint(g[a]) : 0u;
}

// dirty tiles of this pass in one list's byte array (k_fclean's gate): 16
// bytes per load (the array is padded to a multiple of 16 and zeroed)
__global__ void k_count_dirt(const uint8_t *__restrict__ d, int nt, unsigned long long *n) {
  const uint4 *d4 = reinterpret_cast<const uint4 *>(d);
  const int n4 = (nt + 15) / 16;
  unsigned a = 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n4; t += gridDim.x * blockDim.x) {
    const uint4 v = __ldg(&d4[t]);  // bytes are 0 / 1: the sum of the 16 bytes
    a += __dp4a(v.x, 0x01010101u, 0u) + __dp4a(v.y, 0x01010101u, 0u) +
         __dp4a(v.z, 0x01010101u, 0u) + __dp4a(v.w, 0x01010101u, 0u);
  }
  a = __reduce_add_sync(0xffffffffu, a);
  if ((threadIdx.x & 31) == 0 && a) atomicAdd(n, (unsigned long long)a);
}

// positions in S of the saddles a slab owns (local index -> k; -1 elsewhere)
__global__ void k_local_pos(const int32_t *__restrict__ S, int nS, int32_t *pos, GridP G) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nS) return;
  const int A = G.nx * G.ny, a = S[k] - G.zoff * A;
  if (a >= G.zb * A && a < G.ze * A) pos[a] = k;
}
// The owned entries of the replicated gS (positions own[0 .. n)) that the
// stencil changed this pass, listed (position, value bits) for the sparse
// all-gather; prev keeps the last listed values.  A separate pass over the
// slab's ~nS / p entries: appending from inside the dense stencil made it
// spill (ptxas: 500 bytes of spill stores) and run 1.6x longer.
__global__ void k_gs_diff(const int32_t *__restrict__ own, int n, const uint32_t *__restrict__ gS,
                          uint32_t *prev, int2 *upd, unsigned long long *nupd) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  int k = 0;
  uint32_t v = 0;
  bool chg = false;
  if (j < n) {
    k = __ldg(&own[j]);
    v = gS[k];
    chg = prev[k] != v;
    if (chg) prev[k] = v;
  }
  const long long q = cta_slot(chg, nupd);
  if (q >= 0) upd[q] = make_int2(k, (int)v);
}

// The same over the vertices a list pass evaluated (list[0 .. *nlist), local
// ids): the f-saddles among them are the only owned entries that can change
__global__ void k_gs_diff_list(const int32_t *__restrict__ list, const int *__restrict__ nlist,
                               const uint32_t *__restrict__ ref, const int32_t *__restrict__ posS,
                               const uint32_t *__restrict__ gS, uint32_t *prev, int2 *upd,
                               unsigned long long *nupd) {
  const int n = *nlist;
  // block-uniform trip count (cta_slot synchronises the block)
  for (int b = blockIdx.x * blockDim.x; b < n; b += gridDim.x * blockDim.x) {
    const int j = b + threadIdx.x;
    int k = 0;
    uint32_t v = 0;
    bool chg = false;
    if (j < n) {
      const int i = __ldg(&list[j]);
      if (ref_saddle(__ldg(&ref[i]))) {
        k = __ldg(&posS[i]);
        v = gS[k];
        chg = prev[k] != v;
        if (chg) prev[k] = v;
      }
    }
    const long long q = cta_slot(chg, nupd);
    if (q >= 0) upd[q] = make_int2(k, (int)v);
  }
}

// R4 partner values (static routing): the pair (S[k], S[k+1]) is checked by
// the owner of S[k], which needs g at S[k+1].  Every rank computes, from the
// replicated S, the positions it sends (its own j whose predecessor S[j-1] is
// another rank's: key = that rank) and receives (S[k+1] of its own k owned by
// another rank: key = that rank); sorted by key, both sides list a pair's
// positions in ascending order, so the values need no positions on the wire.
__device__ __forceinline__ int owner_rank(int v, int A, int base, int extra) {
  const int z = v / A, big = extra * (base + 1);
  return z < big ? z / (base + 1) : extra + (z - big) / base;
}
__global__ void k_r4_route(const int32_t *__restrict__ own, int nown,
                           const int32_t *__restrict__ S, int nS, int A, int base, int extra,
                           int me, int p, int32_t *skey, int32_t *spos, int32_t *rkey,
                           int32_t *rpos) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nown) return;
  const int k = __ldg(&own[i]);
  int d = p, r = p;  // p: nothing to send / receive (sorted last)
  if (k >= 1) {
    const int o = owner_rank(__ldg(&S[k - 1]), A, base, extra);
    if (o != me) d = o;
  }
  if (k + 1 < nS) {
    const int o = owner_rank(__ldg(&S[k + 1]), A, base, extra);
    if (o != me) r = o;
  }
  skey[i] = d;
  spos[i] = k;
  rkey[i] = r;
  rpos[i] = k + 1;
}
// first index of each key in a sorted key array (start[0 .. p], start[p] = n
// of the keys < p); start[] preset to n by the caller
__global__ void k_key_starts(const int32_t *__restrict__ key, int n, int p, int *start) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int k = key[i];
  if (i == 0 || key[i - 1] != k)
    for (int q = i == 0 ? 0 : key[i - 1] + 1; q <= k && q <= p; ++q) start[q] = i;
}
__global__ void k_pack_u32(const int32_t *__restrict__ pos, int n, const uint32_t *__restrict__ v,
                           uint32_t *out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = v[pos[i]];
}
__global__ void k_unpack_u32(const int32_t *__restrict__ pos, int n, const uint32_t *__restrict__ in,
                             uint32_t *v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[pos[i]] = in[i];
}

// gathered (position, value bits) updates into the replicated gS (pos < 0: padding)
__global__ void k_apply_gs(const int2 *__restrict__ upd, int n, uint32_t *gS) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int2 u = upd[k];
  if (u.x >= 0) gS[u.x] = (uint32_t)u.y;
}

// apply gathered remote marks (global ids) that this slab owns
__global__ void k_apply_remote(const int32_t *__restrict__ ids, int n, uint32_t *marks, GridP G) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int A = G.nx * G.ny, t = ids[k] - G.zoff * A;
  if (t >= G.zb * A && t < G.ze * A) mark_vertex(marks, t, G);
}

__global__ void k_or_words(uint32_t *__restrict__ dst, const uint32_t *__restrict__ src, int n) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n && src[k]) atomicOr(&dst[k], src[k]);
}

// local ids -> global ids
__global__ void k_add_offset(int32_t *ids, int n, int off) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) ids[k] += off;
}

// ---------------------------------------------------- count + edit (O9)
// Eight threads per mark word (one row segment of 32 vertices), four vertices
// each: a streaming pass over the bitmap in which every marked vertex's f, g,
// c are loaded independently (coalesced across the warp, no serial chain).
// V_t = popcount of the words; for each marked i not at lo = RU(f_i - xi): a
// step of Delta (clamped at lo) while c_i < N, else the lossless clamp;
// c_i++.  Words are cleared for the next round.
__device__ __forceinline__ bool edit_vertex(float *__restrict__ g, uint8_t *__restrict__ c,
                                            const float *__restrict__ f, size_t i, float xi,
                                            float delta, int N) {
  const float lo = __fsub_ru(f[i], xi);
  const float gi = g[i];
  const int ci = c[i];
  if (gi == lo) return false;
  float t;
  if (ci < N) {
    t = __fsub_rn(gi, delta);
    t = (t < lo) ? lo : t;
  } else {
    t = lo;
  }
  g[i] = t;
  c[i] = (uint8_t)(ci + 1);
  return true;
}

template <bool TRACK>
__global__ void __launch_bounds__(256, 8) k_count_edit(float *__restrict__ g,
                                                    uint8_t *__restrict__ c,
                                                    uint32_t *__restrict__ marks,
                                                    const float *__restrict__ f, GridP G,
                                                    float xi, float delta, int N, int do_edit,
                                                    Track T, unsigned long long *cnt) {
  const int lane = threadIdx.x & 31, sub = lane & 7, grp = lane >> 3;
  const unsigned gmask = 0xffu << (lane & 24);  // the 8 lanes of a word
  const int64_t nwords = (int64_t)G.ny * G.ze * G.W;  // owned rows: [zb*ny, ze*ny)
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool vec4 = (G.nx & 3) == 0 && ((reinterpret_cast<uintptr_t>(f) |
                                          reinterpret_cast<uintptr_t>(g)) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(c) & 3) == 0;
  unsigned vt = 0, ap = 0;
  for (int64_t wb = (int64_t)G.ny * G.zb * G.W +
                    (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 128;
       wb < nwords; wb += nwarps * 128) {
   // 4 x 32 words per warp step, loaded together (independent loads: the
   // sparse late passes are a scan of mostly zero words, latency-bound)
   uint32_t mine4[4];
#pragma unroll
   for (int q = 0; q < 4; ++q) mine4[q] = (wb + 32 * q + lane < nwords) ? marks[wb + 32 * q + lane] : 0u;
#pragma unroll 1
   for (int q = 0; q < 4; ++q) {
    const int64_t w0 = wb + 32 * q;
    if (w0 >= nwords) break;  // warp-uniform
    // 32 words per warp step (one per lane, coalesced, cleared); the non-zero
    // ones are edited four at a time, 8 lanes x 4 vertices per word
    const uint32_t mine = mine4[q];
    if (mine) {
      vt += __popc(mine);
      marks[w0 + lane] = 0u;
    }
    uint32_t nzw = __ballot_sync(0xffffffffu, mine != 0u);
    while (nzw) {
      // the grp-th remaining non-zero word (if any) goes to lanes 8 grp .. 8 grp + 7
      uint32_t m = nzw;
      for (int k = 0; k < grp && m; ++k) m &= m - 1;
      const int j = m ? __ffs(m) - 1 : 0;
      const uint32_t word = __shfl_sync(0xffffffffu, mine, j);
      for (int k = 0; k < 4 && nzw; ++k) nzw &= nzw - 1;
      if (!m) continue;  // uniform over the 8 lanes of the group
      const int64_t w = w0 + j;
      const int64_t row = div_W((int)w, G);
      const int wx = (int)(w - row * G.W);
      const uint32_t bits = (word >> (4 * sub)) & 15u;
      const size_t base = (size_t)G.nx * row + (size_t)wx * 32 + 4 * sub;
      uint32_t e = 0;  // edited vertices of this word (bit = x - 32 wx)
      if (do_edit && bits && vec4) {
        // rows of a multiple of 4: the lane's 4 vertices as one 16-byte f and
        // g load and one 4-byte c load (independent, in flight together);
        // written back whole (the unmarked ones unchanged)
        const float4 fv = *reinterpret_cast<const float4 *>(f + base);
        float4 gv = *reinterpret_cast<const float4 *>(g + base);
        uint32_t cv = *reinterpret_cast<const uint32_t *>(c + base);
        float *ga = reinterpret_cast<float *>(&gv);
        const float fa[4] = {fv.x, fv.y, fv.z, fv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (!((bits >> q) & 1u)) continue;
          const float lo = __fsub_ru(fa[q], xi);
          if (ga[q] == lo) continue;
          const int ci = (cv >> (8 * q)) & 0xFFu;
          float t;
          if (ci < N) {
            t = __fsub_rn(ga[q], delta);
            t = (t < lo) ? lo : t;
          } else {
            t = lo;
          }
          ga[q] = t;
          cv = (cv & ~(0xFFu << (8 * q))) | ((uint32_t)((ci + 1) & 0xFF) << (8 * q));
          e |= 1u << (4 * sub + q);
        }
        if (e) {
          *reinterpret_cast<float4 *>(g + base) = gv;
          *reinterpret_cast<uint32_t *>(c + base) = cv;
        }
      } else if (do_edit) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if ((bits >> q) & 1u)
            if (edit_vertex(g, c, f, base + q, xi, delta, N)) e |= 1u << (4 * sub + q);
      }
      ap += __popc(e);
      if (TRACK && T.patch && e) {
        const int n = __popc(e);
        const int k0 = atomicAdd(T.npatch, n);
        uint32_t m = e;
        for (int j = 0; j < n; ++j, m &= m - 1)
          if (k0 + j < T.patch_cap)
            T.patch[k0 + j] = (int32_t)((size_t)G.nx * row + (size_t)wx * 32 + (__ffs(m) - 1));
      }
      if (TRACK && (T.bval || T.act_next)) {
        uint32_t E = e;  // OR over the 8 lanes of the word
        E |= __shfl_xor_sync(gmask, E, 1);
        E |= __shfl_xor_sync(gmask, E, 2);
        E |= __shfl_xor_sync(gmask, E, 4);
        if (E) {
          const int z = div_ny((int)row, G), y = (int)row - z * G.ny;
          if (T.bval && sub == 0)
            stamp(T.bval, T.sbval, T, wx, y / BY, z / BZ, (uint16_t)(T.round + 1));
          if (T.edited && sub == 0) T.edited[w] = E;  // one writer per word (pulled later)
          if (!T.edited && T.act_next && sub < 7) {
            // few edits: push the closed stars of the edited vertices into
            // act_next directly (7 (dz, dy) rows, x-1 / x+1 spill into the
            // neighbouring words)
            const int z = div_ny((int)row, G), y = (int)row - z * G.ny;
            const int dz = kr_dz(sub), dy = kr_dy(sub);
            const bool neg = sub <= 3, pos = sub >= 3;  // x-1 for rows 0..3, x+1 for 3..6
            const int yy = y + dy, zz = z + dz;
            if (yy >= 0 && yy < G.ny && zz >= 0 && zz < G.nz) {
              uint32_t *r = T.act_next + (size_t)(yy + G.ny * zz) * G.W;
              const int rem = G.nx - wx * 32;  // vertices of this row in the word
              const uint32_t valid = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
              const uint32_t mm = (E | (neg ? (E >> 1) : 0u) | (pos ? (E << 1) : 0u)) & valid;
              atomicOr(&r[wx], mm);
              if (neg && (E & 1u) && wx > 0) atomicOr(&r[wx - 1], 0x80000000u);
              if (pos && (E >> 31) && wx + 1 < G.W) atomicOr(&r[wx + 1], 1u);
            }
          }
        }
      }
    }
   }
  }
  warp_add(&cnt[C_VT], vt);
  warp_add(&cnt[C_APPLIED], ap);
}

// ------------------------------------------ full labels (outputs only, O6)
__global__ void k_slots_to_ptrs(const uint8_t *__restrict__ slots, int32_t *pdn, int32_t *pup,
                                GridP G) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= G.V) return;
  uint8_t s = slots[i];
  pdn[i] = slot_target((int)i, s & 15, G);
  pup[i] = slot_target((int)i, s >> 4, G);
}

// lab[] holds, for every vertex, a pointer to an ancestor in its steepest
// forest; a round replaces it by its pointer's pointer.  Reads may see
// pointers other threads already advanced (still ancestors), which only
// speeds convergence; the fixpoint (roots) is unique.
__global__ void k_jump(int32_t *lab, int64_t V, unsigned long long *cnt) {
  unsigned changed = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    int w = lab[i];
    int w2 = lab[w];
    if (w2 != w) {
      lab[i] = w2;
      changed = 1;
    }
  }
  if (__any_sync(0xffffffffu, changed) && (threadIdx.x & 31) == 0) atomicOr(&cnt[C_CHANGED], 1ull);
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

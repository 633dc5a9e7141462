// stencil_key.cuh — the dense CheckConstraints stencil (R1, R2, R3 and the
// steepest slots of g) on exact SoS keys.
//
// Applies when every value g can take during the call lies in
// [lo_min, ghat_max] with lo_min >= 2^-41, ghat_max < 2^63 and
// bits(ghat_max) - bits(lo_min) < 2^28 (validation measures both ends; every
// BASELINE config qualifies).  Then:
//
//  * SoS keys (P:178 footnote: value first, the larger index wins a tie):
//    key_s = (bits(v_s) - bits(lo_min)) * 16 + s for neighbour slot s.  For
//    non-negative floats the bit pattern orders like the value, the range
//    bound keeps the product below 2^32, and the slot order IS the index
//    order (mesh.cuh), so unsigned key order == SoS order, exactly.  argmax /
//    argmin over the 14 neighbours are 3-input integer max / min trees
//    (VIMNMX3) whose winner's low 4 bits are its slot: no verification.
//  * The centre is not in the trees: it is the SoS max iff its upper link is
//    empty, the min iff its lower link is empty (O5 over the closed star);
//    otherwise the star's extremum is a neighbour, the tree's winner.
//  * The g-lower mask on the FMA pipe: [v_s > v_c] = sat(fma(v_s, 2^64,
//    -v_c 2^64)) is exact (the rounded difference of two distinct values is
//    >= 2^64 ulp(2^-41) = 1 in magnitude and never overflows below 2^63), and
//    the 14 bits are summed into a float mantissa by FFMA (immediate forms).
//  * Missing neighbours (domain faces): the keys of a warp that holds one are
//    masked to 0 for the max and to ~0 for the min (a real winner always
//    beats them when the link side is non-empty); the lower mask is ANDed
//    with the valid mask.
//  * Marks: the 15-bit target mask (slots, self) is re-indexed in ascending
//    linear order, each (dz, dy) row's 2-3 bits are placed at lane + dx + 1
//    and OR-reduced (REDUX) into a 32-bit word covering x0-1 .. x0+30; the
//    two bits a row can carry past x0+30 come from lanes 30 and 31 only,
//    whose re-indexed masks are fetched with two shuffles and expanded by the
//    plane flush.
#pragma once

namespace exz {

constexpr uint32_t kKeyLoMinBits = 0x2B000000u;  // 2^-41
constexpr uint32_t kKeyHiMaxBits = 0x5F000000u;  // 2^63 (exclusive)
constexpr uint32_t kKeySpan = 1u << 28;

// d_comp2[m] = nlc | nuc << 3 of an interior vertex (all 14 slots present)
// with lower mask m: one lookup instead of two
__device__ uint8_t d_comp2[1 << kSlots];

__device__ __forceinline__ float fma_sat(float a, float b, float c) {
  float d;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 14-input unsigned max / min trees (7 VIMNMX each)
__device__ __forceinline__ uint32_t umax14(const uint32_t (&k)[kSlots]) {
  const uint32_t a = __vimax3_u32(k[0], k[1], k[2]), b = __vimax3_u32(k[3], k[4], k[5]);
  const uint32_t c = __vimax3_u32(k[6], k[7], k[8]), d = __vimax3_u32(k[9], k[10], k[11]);
  const uint32_t e = __vimax3_u32(a, b, c);
  return __vimax3_u32(e, d, max(k[12], k[13]));
}
__device__ __forceinline__ uint32_t umin14(const uint32_t (&k)[kSlots]) {
  const uint32_t a = __vimin3_u32(k[0], k[1], k[2]), b = __vimin3_u32(k[3], k[4], k[5]);
  const uint32_t c = __vimin3_u32(k[6], k[7], k[8]), d = __vimin3_u32(k[9], k[10], k[11]);
  const uint32_t e = __vimin3_u32(a, b, c);
  return __vimin3_u32(e, d, min(k[12], k[13]));
}

// Flush plane p of the key stencil's mark ring into the global bitmap.  An
// entry holds the 7 row words (bit j <-> x0 - 1 + j) and, in word 7, the
// re-indexed target masks of lanes 30 (low half) and 31 (high half), from
// which the bits at x0 + 31 and x0 + 32 are rebuilt.
__device__ __forceinline__ void flush_plane_key(uint32_t *__restrict__ marks,
                                                const uint32_t (*wr)[TY][8], int p, int z0,
                                                int z1, int x0, int y0, const GridP &G) {
  const int ly = threadIdx.x;
  if (ly >= SY) return;
  u64 val = 0;
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int w = ly - 1 - kr_dy(k), st = p - kr_dz(k);
    if (w >= 0 && w < TY && st >= z0 && st < z1) {
      constexpr int kStart[KR] = {0, 2, 4, 6, 9, 11, 13};
      constexpr uint32_t kMask[KR] = {3u, 3u, 3u, 7u, 6u, 6u, 6u};  // in frame: dx + 1
      const uint32_t e = wr[st & 3][w][7];
      const uint32_t t30 = e & 0xFFFFu, t31 = e >> 16;
      // row bits of lane l sit at l + (dx + 1); bits >= 32 of lanes 30, 31
      const u64 c30 = (u64)(((t30 >> kStart[k]) << (k >= 4 ? 1 : 0)) & kMask[k]) << 30;
      const u64 c31 = (u64)(((t31 >> kStart[k]) << (k >= 4 ? 1 : 0)) & kMask[k]) << 31;
      val |= (u64)wr[st & 3][w][k] | ((c30 | c31) & ~0xFFFFFFFFull);
    }
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

template <bool TRACK>
__global__ void __launch_bounds__(NT, 4) k_stencil_key(const float *__restrict__ g,
                                                       const uint32_t *__restrict__ ref,
                                                       uint32_t *__restrict__ marks,
                                                       uint8_t *__restrict__ slots,
                                                       uint32_t *__restrict__ lm, GridP G,
                                                       int zc, Track T,
                                                       unsigned long long *cnt) {
  __shared__ uint32_t sb[4][SP];                   // staged value bits, 4-plane ring
  __shared__ __align__(16) uint32_t wr[4][TY][8];  // mark rows by writer (see flush_plane_key)
  const int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int x0 = bx * TX, y0 = by * TY;
  const int z0 = G.zb + bz * zc, z1 = min(z0 + zc, G.ze);
  const int x = x0 + tx, y = y0 + ty;
  const bool inside = x < G.nx && y < G.ny;
  const int c = (ty + 1) * SX + tx + 1;
  const uint32_t vxy = valid_xy(x, y, G);
  const uint32_t ptx = 1u << tx;
  unsigned n1 = 0, n2 = 0, n3 = 0;
  const int A = G.nx * G.ny;

  int coff[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int cc = tid + k * NT;
    coff[k] = -1;
    if (cc < SP) {
      const int ly = cc / SX, lx = cc - ly * SX;
      const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
      if (gx >= 0 && gx < G.nx && gy >= 0 && gy < G.ny) coff[k] = gx + G.nx * gy;
    }
  }
  auto load = [&](int p, uint32_t (&r)[2]) {
    const bool pin = p >= 0 && p < G.nz;
    const uint32_t *gp = reinterpret_cast<const uint32_t *>(g) + (size_t)p * A;
#pragma unroll
    for (int k = 0; k < 2; ++k) r[k] = (pin && coff[k] >= 0) ? __ldg(gp + coff[k]) : 0xFFFFFFFFu;
  };
  auto store = [&](int p, const uint32_t (&r)[2]) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (tid + k * NT < SP) sb[p & 3][tid + k * NT] = r[k];
  };
  {
    uint32_t r[2];
    for (int p = z0 - 1; p <= z0 + 1; ++p) {
      load(p, r);
      store(p, r);
    }
  }
  __syncthreads();

  const int i00 = x + G.nx * (y + G.ny * z0);
  uint32_t rc = 0, rn = 0;
  int pc = 0;
  if (inside) {
    rc = __ldcs(&ref[i00]);
    if (T.gS && ref_saddle(rc)) pc = __ldg(&T.posS[i00]);
    if (z0 + 1 < z1) rn = __ldcs(&ref[i00 + A]);
  }
  for (int z = z0; z < z1; ++z) {
    uint32_t pre[2];
    const int pz = z + 2;
    const bool prefetch = pz <= z1;
    if (prefetch) load(pz, pre);
    int pn = 0;
    uint32_t rnn = 0;
    if (inside) {
      const int in1 = x + G.nx * (y + G.ny * (z + 1));
      if (T.gS && z + 1 < z1 && ref_saddle(rn)) pn = __ldg(&T.posS[in1]);
      if (z + 2 < z1) rnn = __ldcs(&ref[in1 + A]);
    }

    uint32_t tgt = 0;
    bool schg = false;
    const uint32_t valid = vxy & valid_z(z, G);
    uint32_t bv[kSlots], hb = 0;
#pragma unroll
    for (int s = 0; s < kSlots; ++s) bv[s] = 0u;
    if (inside) {
      const uint32_t *P0 = &sb[z & 3][c];
      const uint32_t *Pm = &sb[(z - 1) & 3][c];
      const uint32_t *Pp = &sb[(z + 1) & 3][c];
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        const int b = slot_bits(s), sg1 = slot_sign(s);
        const uint32_t *pl = (b >> 2) ? (sg1 > 0 ? Pp : Pm) : P0;
        bv[s] = pl[sg1 * ((b & 1) + ((b >> 1) & 1) * SX)];
      }
      hb = *P0;
    }
    // exact SoS keys; a warp holding a missing neighbour masks them
    uint32_t kmax = 0, kmin = 0;
    {
      uint32_t k[kSlots];
#pragma unroll
      for (int s = 0; s < kSlots; ++s) k[s] = bv[s] * 16u + G.kc[s];
      if (__any_sync(0xffffffffu, valid != 0x3FFFu)) {
        uint32_t km[kSlots];
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
          const bool v = (valid >> s) & 1u;
          km[s] = v ? k[s] : 0u;
          k[s] = v ? k[s] : ~0u;
        }
        kmax = umax14(km);
        kmin = umin14(k);
      } else {
        kmax = umax14(k);
        kmin = umin14(k);
      }
    }
    if (inside) {
      const int i = x + G.nx * (y + G.ny * z);
      const uint32_t r = rc;
      // g-lower mask: slot s < 7 is lower iff v_s <= v_c, s >= 7 iff v_s < v_c
      const float hc = __uint_as_float(hb);
      const float sc = __fmul_rn(hc, 0x1p64f);
      float acc = 8388735.0f;  // 2^23 + 127 (bits 0..6 preset)
#pragma unroll
      for (int s = 0; s < 7; ++s)
        acc = __fmaf_rn(fma_sat(__uint_as_float(bv[s]), 0x1p64f, -sc), -(float)(1 << s), acc);
#pragma unroll
      for (int s = 7; s < kSlots; ++s)
        acc = __fmaf_rn(fma_sat(__uint_as_float(bv[s]), -0x1p64f, sc), (float)(1 << s), acc);
      const uint32_t lower = (__float_as_uint(acc) - 0x4B000000u) & valid;
      const uint32_t upper = valid & ~lower;
      const int up = upper ? (int)(kmax & 15u) : kSelf;
      const int dn = lower ? (int)(kmin & 15u) : kSelf;
      // R1, R2
      if (up != ref_up(r)) { tgt |= 1u << up; n1 += 1; }
      if (dn != ref_dn(r)) { tgt |= 1u << ref_dn(r); n2 += 1; }
      // R3 (amb-7, amb-8)
      const uint32_t flow = ref_flow(r);
      const uint32_t flip = lower ^ flow;
      if (flip) {
        bool apply = ref_saddle(r);
        if (!apply) {
          uint32_t t;
          if (valid == 0x3FFFu) {
            t = __ldg(&d_comp2[lower]);
          } else {
            t = (uint32_t)__ldg(&d_comp[lower]) | ((uint32_t)__ldg(&d_comp[upper]) << 3);
          }
          apply = t != ((r >> 22) & 63u);
        }
        if (apply) {
          n3 += __popc(flip);
          tgt |= flip & flow;
          if (flip & ~flow) tgt |= 1u << kSelf;
        }
      }
      const uint8_t ns = (uint8_t)(dn | (up << 4));
      if (TRACK && T.bval) schg = (slots[i] != ns);
      slots[i] = ns;
      if (ref_saddle(r)) {
        if (T.lmS) T.lmS[pc] = lower | (upper << 16);
        else lm[i] = lower | (upper << 16);
        if (T.gS) T.gS[pc] = hb;
      }
    }
    if (TRACK && T.bval) {
      const unsigned chg = __ballot_sync(0xffffffffu, schg);
      if (tx == 0 && chg) stamp(T.bslot, T.sbslot, T, bx, y / BY, z / BZ, (uint16_t)T.round);
    }
    if (TRACK && T.act_next) {
      const unsigned fired = __ballot_sync(0xffffffffu, tgt != 0);
      if (tx == 0 && fired) atomicOr(&T.act_next[(size_t)(y + G.ny * z) * G.W + bx], fired);
    }
    // mark rows: targets re-indexed in ascending linear order (slots 0..6,
    // self, 7..13); row k's bits placed at lane + dx + 1 (low 32 bits); the
    // bits past bit 31 are rebuilt at the flush from lanes 30 and 31
    uint32_t rv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (__any_sync(0xffffffffu, tgt)) {
      const uint32_t t = (tgt & 0x7Fu) | ((tgt & 0x3F80u) << 1) | ((tgt >> kSelf) << 7);
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        constexpr int kStart[KR] = {0, 2, 4, 6, 9, 11, 13};
        const uint32_t cb = ((t >> kStart[k]) & (k == 3 ? 7u : 3u)) << (k >= 4 ? 1 : 0);
        rv[k] = __reduce_or_sync(0xffffffffu, cb * ptx);
      }
      const uint32_t t30 = __shfl_sync(0xffffffffu, t, 30), t31 = __shfl_sync(0xffffffffu, t, 31);
      rv[7] = t30 | (t31 << 16);
    }
    if (tx == 0) {
      uint4 *d = reinterpret_cast<uint4 *>(&wr[z & 3][ty][0]);
      d[0] = make_uint4(rv[0], rv[1], rv[2], rv[3]);
      d[1] = make_uint4(rv[4], rv[5], rv[6], rv[7]);
    }
    const int pf = z - 2;
    if (ty == (z & (TY - 1)) && pf >= z0 - 1 && pf >= 0)
      flush_plane_key(marks, wr, pf, z0, z1, x0, y0, G);
    if (prefetch) store(pz, pre);
    rc = rn;
    pc = pn;
    rn = rnn;
    __syncthreads();
  }
  {
    const int pf = z1 - 2 + ty;
    if (ty < 3 && pf >= z0 - 1 && pf >= 0 && pf < G.nz)
      flush_plane_key(marks, wr, pf, z0, z1, x0, y0, G);
  }
  warp_add(&cnt[C_N1 + 0], n1);
  warp_add(&cnt[C_N1 + 1], n2);
  warp_add(&cnt[C_N1 + 2], n3);
}


// ---------------------------------------------------------------------------
// k_stencil_key2: the same rules, two rows per thread.  The per-step cost of
// k_stencil_key was mostly overhead around the ~130 instructions of rules
// (ncu, round 1 of C2: 375 warp-instructions per 32 vertices: plane and ref
// prefetch addressing, ring addressing, convergence barriers, the REDUX
// results moved out of uniform registers); a thread evaluating the vertices
// (x, ya, z) and (x, ya + 1, z) pays it once for both, shares 8 of the 15
// staged values, and the two vertices' mark rows that land on the same
// global row are ORed before the reduction (10 REDUX per pair, not 14).
// Tile: 32 x 16 columns (8 warps x 2 rows), halo 34 x 18.
constexpr int K2W = 8, K2TY = 2 * K2W, K2SX = TX + 2, K2SY = K2TY + 2, K2SP = K2SX * K2SY;
constexpr int K2ROWS = 10;  // combined (dz, dy') target rows of a row pair, dy' = -1 .. 2
// combined row r: (dz, dy') and the rows of vertex a (ka) / b (kb) it merges
// (row indices of kr_dz / kr_dy above; -1: none)
__host__ __device__ constexpr int k2_dz(int r) { return r < 3 ? -1 : (r < 7 ? 0 : 1); }
__host__ __device__ constexpr int k2_dy(int r) {
  return r < 3 ? r - 1 : (r < 7 ? r - 4 : r - 7);
}
__host__ __device__ constexpr int k2_ka(int r) {
  return r == 0 ? 0 : r == 1 ? 1 : r == 3 ? 2 : r == 4 ? 3 : r == 5 ? 4 : r == 7 ? 5 : r == 8 ? 6 : -1;
}
__host__ __device__ constexpr int k2_kb(int r) {
  return r == 1 ? 0 : r == 2 ? 1 : r == 4 ? 2 : r == 5 ? 3 : r == 6 ? 4 : r == 8 ? 5 : r == 9 ? 6 : -1;
}
// frame field of row k of a position-ordered target mask: bit j <-> dx = j - 1
__host__ __device__ constexpr uint32_t k2_field(uint32_t t, int k) {
  constexpr int kStart[KR] = {0, 2, 4, 6, 9, 11, 13};
  constexpr uint32_t kMask[KR] = {3u, 3u, 3u, 7u, 6u, 6u, 6u};
  return ((t >> kStart[k]) << (k >= 4 ? 1 : 0)) & kMask[k];
}
__host__ __device__ constexpr uint32_t k2_row(uint32_t ta, uint32_t tb, int r) {
  return (k2_ka(r) >= 0 ? k2_field(ta, k2_ka(r)) : 0u) | (k2_kb(r) >= 0 ? k2_field(tb, k2_kb(r)) : 0u);
}

struct KeyOut {
  uint32_t tgt;  // targets, slot order, bit 14 = self
  uint32_t lower, upper;
  uint8_t ns;    // dn | up << 4
  uint32_t d;    // ns ^ (dn_f | up_f << 4): non-zero nibbles = pointers that are not f's
};

// R1-R3 of one vertex from its 14 neighbour value bits (slot order) and
// centre bits hb (see the header of this file)
// k16: 16 as a kernel-parameter value the compiler cannot fold (callers),
// so the 14 key products stay IMADs (FMA pipe) instead of LEAs on the ALU
// pipe that bounds the kernel
__device__ __forceinline__ KeyOut key_rules(const uint32_t (&bv)[kSlots], uint32_t hb,
                                            uint32_t valid, bool edge_warp, uint32_t r,
                                            const GridP &G, unsigned &n1, unsigned &n2,
                                            unsigned &n3, uint32_t k16 = 16u) {
  uint32_t kmax, kmin;
  {
    uint32_t k[kSlots];
#pragma unroll
    for (int s = 0; s < kSlots; ++s) k[s] = bv[s] * k16 + G.kc[s];
    if (edge_warp) {
      uint32_t km[kSlots];
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        const bool v = (valid >> s) & 1u;
        km[s] = v ? k[s] : 0u;
        k[s] = v ? k[s] : ~0u;
      }
      kmax = umax14(km);
      kmin = umin14(k);
    } else {
      kmax = umax14(k);
      kmin = umin14(k);
    }
  }
  const float hc = __uint_as_float(hb);
  const float sc = __fmul_rn(hc, 0x1p64f);
  float acc = 8388735.0f;
#pragma unroll
  for (int s = 0; s < 7; ++s)
    acc = __fmaf_rn(fma_sat(__uint_as_float(bv[s]), 0x1p64f, -sc), -(float)(1 << s), acc);
#pragma unroll
  for (int s = 7; s < kSlots; ++s)
    acc = __fmaf_rn(fma_sat(__uint_as_float(bv[s]), -0x1p64f, sc), (float)(1 << s), acc);
  KeyOut o;
  o.lower = (__float_as_uint(acc) - 0x4B000000u) & valid;
  o.upper = valid & ~o.lower;
  const uint32_t up = o.upper ? (kmax & 15u) : (uint32_t)kSelf;
  const uint32_t dn = o.lower ? (kmin & 15u) : (uint32_t)kSelf;
  // R1 / R2: the packed slot byte against f's (ref bits 14..21 = dn_f | up_f << 4)
  const uint32_t ns = dn | (up << 4), rf = (r >> 14) & 0xFFu, d = ns ^ rf;
  uint32_t tgt = 0;
  if (d & 0xF0u) { tgt |= 1u << up; n1 += 1; }
  if (d & 0x0Fu) { tgt |= 1u << (rf & 15u); n2 += 1; }
  // R3, branch-free (in the dense passes nearly every vertex has a flipped
  // pair): the type from the interior LUT, re-read for the rare face vertex
  const uint32_t flow = ref_flow(r);
  const uint32_t flip = o.lower ^ flow;
  uint32_t t = __ldg(&d_comp2[o.lower]);
  if (valid != 0x3FFFu)
    t = (uint32_t)__ldg(&d_comp[o.lower]) | ((uint32_t)__ldg(&d_comp[o.upper]) << 3);
  const bool apply = ref_saddle(r) || t != ((r >> 22) & 63u);
  const uint32_t fl = apply ? flip : 0u;
  n3 += __popc(fl);
  tgt |= (fl & flow) | ((fl & ~flow) ? (1u << kSelf) : 0u);
  o.tgt = tgt;
  o.ns = (uint8_t)ns;
  o.d = d;
  return o;
}

// Pair layout of the targets: a 3-bit field per combined row r (bit dx + 1),
// vertex a's (dz, dy) rows at r = 0,1 | 3,4,5 | 7,8 and vertex b's the same
// one row (3 bits) up, so the pair's 10 rows are C = A_a | A_b << 3.
// k2_lay(s): the bit of slot s (14: self) in A.
__host__ __device__ constexpr int k2_lay(int s) {
  // slot s = sign * (b & 1, (b >> 1) & 1, b >> 2) (slot_bits / slot_sign)
  return s == kSelf ? 13
                    : 3 * (slot_sign(s) * (slot_bits(s) >> 2) + 1 == 0
                               ? slot_sign(s) * ((slot_bits(s) >> 1) & 1) + 1
                               : (slot_sign(s) * (slot_bits(s) >> 2) == 0
                                      ? slot_sign(s) * ((slot_bits(s) >> 1) & 1) + 4
                                      : slot_sign(s) * ((slot_bits(s) >> 1) & 1) + 7)) +
                          slot_sign(s) * (slot_bits(s) & 1) + 1;
}
static_assert(k2_lay(0) == 0 && k2_lay(3) == 4 && k2_lay(4) == 9 && k2_lay(6) == 12 &&
                  k2_lay(7) == 14 && k2_lay(9) == 17 && k2_lay(10) == 22 && k2_lay(13) == 26 &&
                  k2_lay(kSelf) == 13,
              "pair layout of the mark rows");

// List pass on exact SoS keys (C.keyed): one listed vertex per thread, its
// 15 values from global memory (mostly L1/L2: the list is in index order),
// the rules of key_rules, the outputs of vertex_outputs.  Same bits as
// k_stencil_list (the keys order like SoS, see the top of this file).
__global__ void __launch_bounds__(256, EXACTZ_LIST_MINB) k_stencil_list_key(const float *__restrict__ g,
                                                          const uint32_t *__restrict__ ref,
                                                          uint32_t *__restrict__ marks,
                                                          uint8_t *__restrict__ slots,
                                                          uint32_t *__restrict__ lm,
                                                          const int32_t *__restrict__ list,
                                                          const int *__restrict__ count, GridP G,
                                                          Track T, unsigned long long *cnt) {
  const int n = *count;
  const uint32_t *gb = reinterpret_cast<const uint32_t *>(g);
  unsigned n1 = 0, n2 = 0, n3 = 0, ne = 0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int i = __ldg(&list[k]);
    const int row = div_nx(i, G), x = i - row * G.nx;
    const int z = div_ny(row, G), y = row - z * G.ny;
    const uint32_t valid = valid_mask(x, y, z, G);
    uint32_t bv[kSlots];
#pragma unroll
    for (int s = 0; s < kSlots; ++s) bv[s] = ((valid >> s) & 1u) ? __ldg(&gb[i + G.delta[s]]) : 0u;
    const uint32_t r = __ldg(&ref[i]);
    const KeyOut o = key_rules(bv, __ldg(&gb[i]), valid, valid != 0x3FFFu, r, G, n1, n2, n3,
                               G.k16);
    vertex_outputs(i, x, y, z, row, r, valid, o.tgt, o.lower, o.ns & 15, o.ns >> 4, g, marks,
                   slots, lm, G, T);
    ++ne;
  }
  warp_add(&cnt[C_EVAL], ne);
  warp_add(&cnt[C_N1 + 0], n1);
  warp_add(&cnt[C_N1 + 1], n2);
  warp_add(&cnt[C_N1 + 2], n3);
}

// Flush plane p of k_stencil_key2's ring: lane ly = target row y0 - 1 + ly.
// Entry words 0..9: combined rows (bit j <-> x0 - 1 + j); words 10 / 11: the
// pair layouts C of lanes 30 / 31 (their bits past x0 + 30).
constexpr int K2WR = 16;  // mark-ring entries (steps): a flush every 8 steps reads 10
__device__ __forceinline__ void flush_plane_key2(uint32_t *__restrict__ marks,
                                                 const uint32_t (*wr)[K2W][12], int p, int z0,
                                                 int z1, int x0, int y0, const GridP &G) {
  const int ly = threadIdx.x & 31;
  if (ly >= K2SY) return;
  u64 val = 0;
#pragma unroll
  for (int r = 0; r < K2ROWS; ++r) {
    // writer warp w covers rows 1 + 2w, 2 + 2w of the halo tile; its row r
    // lands on halo row 1 + 2w + dy'
    const int d = ly - 1 - k2_dy(r);
    const int w = d >> 1, st = p - k2_dz(r);
    if (d >= 0 && !(d & 1) && w < K2W && st >= z0 && st < z1) {
      const uint32_t *e = wr[st & (K2WR - 1)][w];
      const u64 c = ((u64)((e[10] >> (3 * r)) & 7u) << 30) | ((u64)((e[11] >> (3 * r)) & 7u) << 31);
      val |= (u64)e[r] | (c & ~0xFFFFFFFFull);
    }
  }
  const int gy = y0 - 1 + ly;
  if (!val || gy < 0 || gy >= G.ny || p < 0 || p >= G.nz) return;
  uint32_t *row = marks + (size_t)(gy + G.ny * p) * G.W;
  const int wx = x0 >> 5;
  const uint32_t wv = (uint32_t)(val >> 1);
  if (wv) atomicOr(&row[wx], wv);
  if ((val & 1ull) && x0 > 0) atomicOr(&row[wx - 1], 0x80000000u);
  if (((val >> 33) & 1ull) && x0 + 32 < G.nx) atomicOr(&row[wx + 1], 1u);
}

// --- TMA / mbarrier helpers (plane staging of k_stencil_key2<*, true>)
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_plane(void *dst, const CUtensorMap *map, uint64_t *bar, int x,
                                          int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// TMA: the halo tile of a plane lands in a ring slot by one bulk-tensor copy
// per plane, issued by one thread three planes ahead, with an mbarrier per
// slot; no per-thread loads, stores or address arithmetic.  The box starts at
// x0 - 4 (the innermost start coordinate must be 16-byte aligned: x0 - 1 is
// an illegal instruction, measured) and is 40 x 18 floats; out-of-domain
// cells are zero-filled and masked by the valid masks.  Needs nx % 4 == 0
// (16-byte row stride); else the threads stage the 34 x 18 cells.
template <bool TMA>
struct K2Stage {
  static constexpr int SXS = TMA ? 40 : K2SX;    // smem row stride (TMA box width)
  static constexpr int X0 = TMA ? 4 : 1;         // tile column of x0
  static constexpr int SLOT = TMA ? 736 : K2SP;  // words per ring slot (TMA: 128-B multiple)
};

#ifndef EXACTZ_K2_MINB
#define EXACTZ_K2_MINB 3  // CTAs per SM (80 registers)
#endif
template <bool TRACK, bool TMA>
__global__ void __launch_bounds__(TX * K2W, EXACTZ_K2_MINB) k_stencil_key2(const float *__restrict__ g,
                                                              const uint32_t *__restrict__ ref,
                                                              uint32_t *__restrict__ marks,
                                                              uint8_t *__restrict__ slots,
                                                              uint32_t *__restrict__ lm, GridP G,
                                                              int zc, Track T,
                                                              unsigned long long *cnt,
                                                              const __grid_constant__ CUtensorMap tmap) {
  constexpr int NT2 = TX * K2W;
  constexpr int SXS = K2Stage<TMA>::SXS, SLOT = K2Stage<TMA>::SLOT;
  __shared__ __align__(128) uint32_t sb[4][SLOT];
  __shared__ __align__(16) uint32_t wr[K2WR][K2W][12];
  __shared__ __align__(8) uint64_t bar[4];
  // slot-order targets -> pair layout (k2_lay): bits 0..7 and 8..14 by table
  __shared__ uint32_t lay0[256], lay1[128];
  const int tid = threadIdx.x, tx = tid & 31, w = tid >> 5;
  for (int m = tid; m < 256 + 128; m += TX * K2W) {
    const int base = m < 256 ? 0 : 8, bits = m < 256 ? m : m - 256;
    uint32_t a = 0;
    for (int j = 0; j < 8; ++j)
      if ((bits >> j) & 1) a |= 1u << k2_lay(base + j);
    if (m < 256) lay0[m] = a;
    else lay1[m - 256] = a;
  }
  const int bx = blockIdx.x;
  const int x0 = bx * TX, y0 = blockIdx.y * K2TY;
  const int z0 = G.zb + blockIdx.z * zc, z1 = min(z0 + zc, G.ze);
  const int x = x0 + tx, ya = y0 + 2 * w, yb = ya + 1;
  const bool ina = x < G.nx && ya < G.ny, inb = x < G.nx && yb < G.ny;
  const int ca = (2 * w + 1) * SXS + tx + K2Stage<TMA>::X0;  // row a's cell; row b's: + SXS
  const uint32_t vxya = valid_xy(x, ya, G), vxyb = valid_xy(x, yb, G);
  // 2^tx, opaque to the compiler: the row placement cb * 2^tx stays an IMAD
  // (FMA pipe) instead of becoming a shift on the busier ALU pipe
  uint32_t ptx = 1u << tx;
  asm volatile("mov.b32 %0, %0;" : "+r"(ptx));
  const uint32_t k16 = G.k16;  // likewise for the key products (key_rules)
  unsigned n1 = 0, n2 = 0, n3 = 0;
  const int A = G.nx * G.ny;
  auto slot_of = [&](int p) { return (p - z0 + 1) & 3; };  // ring slot of plane p

  // staged cells of this thread (3 of the 34 x 18 halo tile; non-TMA only):
  // 32-bit offsets from a plane pointer advanced by one plane per step
  int coff[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int cc = tid + k * NT2;
    coff[k] = -1;
    if (!TMA && cc < K2SP) {
      const int ly = cc / K2SX, lx = cc - ly * K2SX;
      const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
      if (gx >= 0 && gx < G.nx && gy >= 0 && gy < G.ny) coff[k] = gx + G.nx * gy;
    }
  }
  auto load = [&](const uint32_t *gp, bool pin, uint32_t (&rr)[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k) rr[k] = (pin && coff[k] >= 0) ? __ldg(gp + coff[k]) : 0xFFFFFFFFu;
  };
  auto store = [&](int p, const uint32_t (&rr)[3]) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (tid + k * NT2 < K2SP) sb[slot_of(p)][tid + k * NT2] = rr[k];
  };
  auto issue = [&](int p) {  // TMA: one thread, plane p into its slot
    const int sl = slot_of(p);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bar[sl], (uint32_t)(SXS * K2SY * 4));
    tma_plane(&sb[sl][0], &tmap, &bar[sl], x0 - 4, y0 - 1, p);
  };
  auto wait_plane = [&](int p) { mbar_wait(&bar[slot_of(p)], (uint32_t)(((p - z0 + 1) >> 2) & 1)); };
  const uint32_t *gpl = reinterpret_cast<const uint32_t *>(g) + (size_t)(z0 - 1) * A;
  if (TMA) {
    if (tid == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) mbar_init(&bar[k], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0)
      for (int p = z0 - 1; p <= min(z0 + 2, z1); ++p) issue(p);
    wait_plane(z0 - 1);
    wait_plane(z0);
  } else {
    uint32_t rr[3];
    for (int p = z0 - 1; p <= z0 + 1; ++p, gpl += A) {
      load(gpl, p >= 0 && p < G.nz, rr);
      store(p, rr);
    }
    // gpl -> plane z0 + 2
    __syncthreads();
  }

  // ref words (and, at f-saddles, the position in S) planes ahead in
  // register sets of a loop unrolled by three: no moves, so a load's latency
  // is covered by whole steps
  const int ia0 = x + G.nx * (ya + G.ny * z0);
  const uint32_t *rp = ref + ia0;  // row a of plane z; row b is rp[G.nx]
  const uint32_t *pp = T.gS ? reinterpret_cast<const uint32_t *>(T.posS) + ia0 : nullptr;
  struct Pre {
    uint32_t ra, rb;
    uint32_t pa, pb;  // unsigned: no sign extension issued behind the load
  };
  auto fetch = [&](int dz, Pre &q) {  // plane z0 + dz, relative to rp / pp of plane z0
    q.ra = q.rb = 0u;
    q.pa = q.pb = 0u;
    if (dz >= zc || z0 + dz >= z1) return;
    const size_t o = (size_t)dz * A;
    if (ina) q.ra = __ldcs(rp + o);
    if (inb) q.rb = __ldcs(rp + o + G.nx);
  };
  auto fetch_pos = [&](int dz, Pre &q) {  // needs q.ra / q.rb loaded
    if (!pp) return;
    const size_t o = (size_t)dz * A;
    if (ina && ref_saddle(q.ra)) q.pa = __ldg(pp + o);
    if (inb && ref_saddle(q.rb)) q.pb = __ldg(pp + o + G.nx);
  };
  // three register sets: set d % 3 holds plane z0 + d; a step refills its
  // set with the ref words of plane + 3, and issues the posS loads of plane
  // + 2 (whose ref words arrived during the previous step)
  Pre q0, q1, q2;
  fetch(0, q0);
  fetch(1, q1);
  fetch(2, q2);
  fetch_pos(0, q0);
  fetch_pos(1, q1);
  int flushed = z0 - 2;  // planes <= flushed are in the global bitmap
  // output pointers of row a in plane z (row b: + nx), advanced per step
  uint8_t *slp = slots + ia0;
  uint32_t *lmp = lm + ia0;

  auto step = [&](int z, Pre &cur) {
    const int dz = z - z0;
    uint32_t pre[3];
    const bool prefetch = !TMA && z + 2 <= z1;
    if (prefetch) load(gpl, z + 2 < G.nz, pre);
    gpl += A;
    if (TMA) wait_plane(z + 1);
    const uint32_t vz = valid_z(z, G);
    const uint32_t va = vxya & vz, vb = vxyb & vz;
    const bool edge = __any_sync(0xffffffffu, (va & vb) != 0x3FFFu);
    const uint32_t *P0 = &sb[slot_of(z)][ca];
    const uint32_t *Pm = &sb[slot_of(z - 1)][ca];
    const uint32_t *Pp = &sb[slot_of(z + 1)][ca];
    // the 22 staged values of the pair (offsets (dx, dy) from row a's cell)
    // plane z-1: (0,-1) (-1,-1) (-1,0) (0,0) (-1,1) (0,1)
    const uint32_t m0m = Pm[-SXS], mmm = Pm[-SXS - 1], mm0 = Pm[-1], m00 = Pm[0],
                   mm1 = Pm[SXS - 1], m01 = Pm[SXS];
    // plane z: (0,-1) (-1,-1) (-1,0) (0,0) (1,0) (-1,1) (0,1) (1,1) (0,2) (1,2)
    const uint32_t c0m = P0[-SXS], cmm = P0[-SXS - 1], cm0 = P0[-1], c00 = P0[0], c10 = P0[1],
                   cm1 = P0[SXS - 1], c01 = P0[SXS], c11 = P0[SXS + 1],
                   c02 = P0[2 * SXS], c12 = P0[2 * SXS + 1];
    // plane z+1: (0,0) (1,0) (0,1) (1,1) (0,2) (1,2)
    const uint32_t p00 = Pp[0], p10 = Pp[1], p01 = Pp[SXS], p11 = Pp[SXS + 1],
                   p02 = Pp[2 * SXS], p12 = Pp[2 * SXS + 1];
    // slot order (mesh.cuh kOff): (-1,-1,-1) (0,-1,-1) (-1,0,-1) (0,0,-1)
    // (-1,-1,0) (0,-1,0) (-1,0,0) | (1,0,0) (0,1,0) (1,1,0) (0,0,1) (1,0,1)
    // (0,1,1) (1,1,1).  Lanes outside the domain evaluate staged values too
    // (never stored, never counted: no divergent branch around the rules).
    unsigned m1 = 0, m2 = 0, m3 = 0;
    KeyOut oa, ob;
    {
      const uint32_t bv[kSlots] = {mmm, m0m, mm0, m00, cmm, c0m, cm0, c10, c01, c11, p00, p10, p01, p11};
      oa = key_rules(bv, c00, va, edge, cur.ra, G, m1, m2, m3, k16);
    }
    if (!ina) { oa.tgt = 0; m1 = m2 = m3 = 0; }
    n1 += m1; n2 += m2; n3 += m3;
    m1 = m2 = m3 = 0;
    {
      const uint32_t bv[kSlots] = {mm0, m00, mm1, m01, cm0, c00, cm1, c11, c02, c12, p01, p11, p02, p12};
      ob = key_rules(bv, c01, vb, edge, cur.rb, G, m1, m2, m3, k16);
    }
    if (!inb) { ob.tgt = 0; m1 = m2 = m3 = 0; }
    n1 += m1; n2 += m2; n3 += m3;
    bool schg = false;
    if (ina) {
      if (TRACK && T.bval) schg = *slp != oa.ns;
      *slp = oa.ns;
      if (ref_saddle(cur.ra)) {
        if (T.lmS) T.lmS[cur.pa] = oa.lower | (oa.upper << 16);
        else *lmp = oa.lower | (oa.upper << 16);
        if (T.gS) T.gS[cur.pa] = c00;
      }
    }
    if (inb) {
      if (TRACK && T.bval) schg |= slp[G.nx] != ob.ns;
      slp[G.nx] = ob.ns;
      if (ref_saddle(cur.rb)) {
        if (T.lmS) T.lmS[cur.pb] = ob.lower | (ob.upper << 16);
        else lmp[G.nx] = ob.lower | (ob.upper << 16);
        if (T.gS) T.gS[cur.pb] = c01;
      }
    }
    slp += A;
    lmp += A;
    fetch(dz + 3, cur);
    if (TRACK && T.bval) {
      const unsigned chg = __ballot_sync(0xffffffffu, schg);
      if (tx == 0 && chg) stamp(T.bslot, T.sbslot, T, bx, ya / BY, z / BZ, (uint16_t)T.round);
    }
    if (TRACK && T.act_next) {
      const unsigned fa = __ballot_sync(0xffffffffu, oa.tgt != 0);
      const unsigned fb = __ballot_sync(0xffffffffu, ob.tgt != 0);
      if (tx == 0 && fa) atomicOr(&T.act_next[(size_t)(ya + G.ny * z) * G.W + bx], fa);
      if (tx == 0 && fb) atomicOr(&T.act_next[(size_t)(yb + G.ny * z) * G.W + bx], fb);
    }
    // combined mark rows of the pair: the layouts by table (k2_lay), row r
    // = bits 3r .. 3r+2 of C, placed at lane + dx + 1 by the multiply
    {
      const uint32_t Ca = lay0[oa.tgt & 0xFFu] | lay1[oa.tgt >> 8];
      const uint32_t Cb = lay0[ob.tgt & 0xFFu] | lay1[ob.tgt >> 8];
      const uint32_t Cc = Ca | (Cb << 3);
      uint32_t rv[12];
#pragma unroll
      for (int r = 0; r < K2ROWS; ++r)
        rv[r] = __reduce_or_sync(0xffffffffu, ((Cc * G.k2up[r]) >> 29) * ptx);
      rv[10] = __shfl_sync(0xffffffffu, Cc, 30);
      rv[11] = __shfl_sync(0xffffffffu, Cc, 31);
      if (tx == 0) {
        uint4 *d = reinterpret_cast<uint4 *>(&wr[z & (K2WR - 1)][w][0]);
        d[0] = make_uint4(rv[0], rv[1], rv[2], rv[3]);
        d[1] = make_uint4(rv[4], rv[5], rv[6], rv[7]);
        d[2] = make_uint4(rv[8], rv[9], rv[10], rv[11]);
      }
    }
    if (prefetch) store(z + 2, pre);
    __syncthreads();
    // plane z + 3 into the slot plane z - 1 just left
    if (TMA && tid == 0 && z + 3 <= z1) issue(z + 3);
    // every 8 steps the 8 warps flush the 8 complete planes, one each
    if (((dz + 1) & (K2W - 1)) == 0) {
      flush_plane_key2(marks, wr, flushed + 1 + w, z0, z1, x0, y0, G);
      flushed += K2W;
    }
  };
  for (int z = z0; z < z1; z += 3) {
    step(z, q0);
    fetch_pos(z - z0 + 2, q2);
    if (z + 1 >= z1) break;
    step(z + 1, q1);
    fetch_pos(z - z0 + 3, q0);
    if (z + 2 >= z1) break;
    step(z + 2, q2);
    fetch_pos(z - z0 + 4, q1);
  }
  // the remaining planes (writers up to step z1 - 1 are complete)
  for (int p = flushed + 1 + w; p <= z1; p += K2W)
    if (p >= 0 && p < G.nz) flush_plane_key2(marks, wr, p, z0, z1, x0, y0, G);
  warp_add(&cnt[C_N1 + 0], n1);
  warp_add(&cnt[C_N1 + 1], n2);
  warp_add(&cnt[C_N1 + 2], n3);
}

}  // namespace exz

// stencil_fast.cuh — the dense CheckConstraints stencil (R1, R2, R3 and the
// steepest slots of g) for fields whose values
// are all >= 0, balanced between the ALU and FMA pipes.
//
// The first dense stencil (kernels.cuh k_stencil) was bound by the ALU pipe
// (ncu: sm__inst_executed_pipe_alu 87 % of peak, FMA pipe 10 %, ~250 of ~400
// warp instructions per 32 vertices on the ALU pipe, which issues at half
// rate).  This kernel computes the same bits with fewer ALU instructions:
//
//  * argmin / argmax of the closed star by 3-input integer min/max trees
//    (VIMNMX3).  For non-negative floats the IEEE bit pattern read as an
//    integer is order-preserving, so a candidate's key is its value bits with
//    the low 4 bits replaced by its position in index order (slots 0..6, the
//    centre, slots 7..13 -> 0..14).  Within a bucket of equal upper 28 bits
//    the position decides, which is the SoS tie break (largest index wins the
//    argmax, smallest the argmin; P:178 footnote).  A winner is exact iff its
//    full value equals the exact extremum (a second tree over the full bits);
//    otherwise (two different values in the top bucket, rare) the lane falls
//    back to the sequential SoS scan (eval_values).
//  * the g-lower mask from the FMA pipe: sign of the rounded difference
//    (exact: no underflow to zero with gradual underflow), amplified by
//    2^252 and saturated to 0/1, then packed by FFMA into a float whose
//    mantissa is the mask.
//  * marks by PULL: each vertex stores its 15-bit target mask in a shared
//    ring; two planes later a vertex ORs the bits of its 14 neighbours that
//    point back at it (slot 13 - s) plus its own self bit and the warp writes
//    one mark word (one atomicOr).  Targets outside the CTA's tile (rows
//    y0-1 / y0+8, planes z0-1 / z1, columns x0-1 / x0+32) are pushed with
//    global atomics: a warp ballot per slot for whole rows, single bits for
//    the two edge lanes.
//
// Missing neighbours (outside the domain) are staged as 0xFFFFFFFF, the bit
// pattern of the NaN that fills the ghost planes of a slab: negative as a
// signed key (never the max), the largest unsigned key (never the min), NaN
// as a float (never lower; masked by the valid mask anyway).  Used only when
// every lo_i = RU(f_i - xi) is >= 0 and no input value is -0.0 (validation
// counts both): then every value of g is a non-negative float other than -0
// for the whole call (edits produce max(RN(g - Delta), lo) >= +0), so the bit
// patterns are the keys as loaded.  Otherwise k_stencil runs.
#pragma once

namespace exz {

constexpr uint32_t kMissing = 0xFFFFFFFFu;

// star position (index order) of slot s; the centre is 7
__host__ __device__ constexpr int slot_pos(int s) { return s < 7 ? s : s + 1; }

// 3-input integer max / min (VIMNMX3 on sm_100a)
__device__ __forceinline__ int imax3(int a, int b, int c) { return __vimax3_s32(a, b, c); }
__device__ __forceinline__ uint32_t umin3(uint32_t a, uint32_t b, uint32_t c) {
  return __vimin3_u32(a, b, c);
}

// 1.0 if d > 0, else 0.0 (NaN -> 0)
__device__ __forceinline__ float pos01(float d) {
  return __saturatef(__fmul_rn(__fmul_rn(d, 0x1p126f), 0x1p126f));
}

// flush_plane (kernels.cuh) for the packed ring of k_stencil_fast: row k of
// a writer = low word k | carry nibble k of word 7 above bit 32
__device__ __forceinline__ void flush_plane_packed(uint32_t *__restrict__ marks,
                                                   const uint32_t (*wr)[TY][8], int p, int z0,
                                                   int z1, int x0, int y0, const GridP &G) {
  const int ly = threadIdx.x;
  if (ly >= SY) return;
  u64 val = 0;
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int w = ly - 1 - kr_dy(k), st = p - kr_dz(k);
    if (w >= 0 && w < TY && st >= z0 && st < z1)
      val |= (u64)wr[st & 3][w][k] | ((u64)((wr[st & 3][w][7] >> (4 * k)) & 15u) << 32);
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

template <bool TRACK, bool LALU = false>
__global__ void __launch_bounds__(NT, 4) k_stencil_fast(const float *__restrict__ g,
                                                        const uint32_t *__restrict__ ref,
                                                        uint32_t *__restrict__ marks,
                                                        uint8_t *__restrict__ slots,
                                                        uint32_t *__restrict__ lm, GridP G,
                                                        int zc, Track T,
                                                        unsigned long long *cnt) {
  __shared__ uint32_t sb[4][SP];  // staged value bits, 4-plane ring
  __shared__ __align__(16) uint32_t wr[4][TY][8];  // mark rows by writer: 7 low words + packed carries
  __shared__ int stab[4][16];     // per z mod 4: star position -> word offset from the centre cell
  __shared__ uint8_t sslot[16];   // star position -> slot code
  const int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int x0 = bx * TX, y0 = by * TY;
  const int z0 = G.zb + bz * zc, z1 = min(z0 + zc, G.ze);
  const int x = x0 + tx, y = y0 + ty;
  const bool inside = x < G.nx && y < G.ny;
  const int c = (ty + 1) * SX + tx + 1;
  const uint32_t vxy = valid_xy(x, y, G);
  const uint32_t ptx = 1u << tx;  // mark-row placement multiplier (see the row masks)
  unsigned n1 = 0, n2 = 0, n3 = 0;
  const int A = G.nx * G.ny;

  // the (up to 2) halo-tile cells this thread stages: plane offsets, or -1
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
    for (int k = 0; k < 2; ++k) r[k] = (pin && coff[k] >= 0) ? __ldg(gp + coff[k]) : kMissing;
  };
  auto store = [&](int p, const uint32_t (&r)[2]) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (tid + k * NT < SP) sb[p & 3][tid + k * NT] = r[k];
  };
  auto table = [&](int z, int q, int *dst) {  // entry of star position q for steps = z mod 4
    int dx = 0, dy = 0, dz = 0;
    if (q != 7) {
      const int s = q < 7 ? q : q - 1;
      const int b = slot_bits(s), sg1 = slot_sign(s);
      dx = sg1 * (b & 1);
      dy = sg1 * ((b >> 1) & 1);
      dz = sg1 * (b >> 2);
    }
    dst[q] = (((z + dz) & 3) - (z & 3)) * SP + dy * SX + dx;
  };
  if (tid < 15) sslot[tid] = (uint8_t)(tid < 7 ? tid : (tid == 7 ? kSelf : tid - 1));
  if (tid < 60) table(tid / 15, tid % 15, stab[tid / 15]);
  {  // prologue: planes z0-1, z0, z0+1
    uint32_t r[2];
    for (int p = z0 - 1; p <= z0 + 1; ++p) {
      load(p, r);
      store(p, r);
    }
  }
  __syncthreads();

  // ref words one plane ahead and, at f-saddles, the position in S (for the
  // gS write) one plane ahead of its use: no dependent load inside a step
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
    if (inside) {
      const int i = x + G.nx * (y + G.ny * z);
      const uint32_t r = rc;
      const uint32_t valid = vxy & valid_z(z, G);
      const uint32_t *P0 = &sb[z & 3][c];
      const uint32_t *Pm = &sb[(z - 1) & 3][c];
      const uint32_t *Pp = &sb[(z + 1) & 3][c];
      uint32_t bv[15];
#pragma unroll
      for (int s = 0; s < kSlots; ++s) {
        const int b = slot_bits(s), sg1 = slot_sign(s);
        const uint32_t *pl = (b >> 2) ? (sg1 > 0 ? Pp : Pm) : P0;
        bv[slot_pos(s)] = pl[sg1 * ((b & 1) + ((b >> 1) & 1) * SX)];
      }
      bv[7] = *P0;
      // g-lower mask: slot s < 7 is lower iff v_s <= h, s >= 7 iff v_s < h
      const float hc = __uint_as_float(bv[7]);
      uint32_t lower = 0;
      if (LALU) {  // compare-select on the ALU pipe (missing = NaN: never lower)
#pragma unroll
        for (int s = 0; s < kSlots; ++s) {
          const float vs = __uint_as_float(bv[slot_pos(s)]);
          lower |= ((s < 7) ? (vs <= hc) : (vs < hc)) ? (1u << s) : 0u;
        }
      } else {  // FMA pipe: saturated, amplified signs packed into a float mantissa
        float acc = 8388735.0f;  // 2^23 + 127 (bits 0..6 preset)
#pragma unroll
        for (int s = 0; s < 7; ++s)
          acc = __fmaf_rn(pos01(__fsub_rn(__uint_as_float(bv[s]), hc)), -(float)(1 << s), acc);
#pragma unroll
        for (int s = 7; s < kSlots; ++s)
          acc = __fmaf_rn(pos01(__fsub_rn(hc, __uint_as_float(bv[s + 1]))), (float)(1 << s), acc);
        lower = (__float_as_uint(acc) - 0x4B000000u) & valid;
      }
      // argmax / argmin by position-tagged keys, verified against the exact trees
      int q[15];
#pragma unroll
      for (int k = 0; k < 15; ++k) q[k] = (int)((bv[k] & G.keymask) | G.tag[k]);
      const int qmax = imax3(imax3(imax3(q[0], q[1], q[2]), imax3(q[3], q[4], q[5]),
                                   imax3(q[6], q[7], q[8])),
                             imax3(q[9], q[10], q[11]), imax3(q[12], q[13], q[14]));
      const uint32_t qmin = umin3(umin3(umin3(q[0], q[1], q[2]), umin3(q[3], q[4], q[5]),
                                        umin3(q[6], q[7], q[8])),
                                  umin3(q[9], q[10], q[11]), umin3(q[12], q[13], q[14]));
      auto I = [&](int k) { return (int)bv[k]; };
      const int emax = imax3(imax3(imax3(I(0), I(1), I(2)), imax3(I(3), I(4), I(5)),
                                   imax3(I(6), I(7), I(8))),
                             imax3(I(9), I(10), I(11)), imax3(I(12), I(13), I(14)));
      const uint32_t emin =
          umin3(umin3(umin3(bv[0], bv[1], bv[2]), umin3(bv[3], bv[4], bv[5]),
                      umin3(bv[6], bv[7], bv[8])),
                umin3(bv[9], bv[10], bv[11]), umin3(bv[12], bv[13], bv[14]));
      const int wu = qmax & 15, wd = (int)(qmin & 15u);
      const int *tb = stab[z & 3];
      int up = sslot[wu], dn = sslot[wd];
      if ((int)P0[tb[wu]] != emax || P0[tb[wd]] != emin) {
        // a bucket held two different values: the exact sequential scan
        float v[kSlots];
#pragma unroll
        for (int s = 0; s < kSlots; ++s)
          v[s] = ((valid >> s) & 1u) ? __uint_as_float(bv[slot_pos(s)]) : __int_as_float(0x7fc00000);
        const Star sx = eval_values(v, hc);
        up = sx.up;
        dn = sx.dn;
      }
      // R1, R2
      if (up != ref_up(r)) { tgt |= 1u << up; n1 += 1; }
      if (dn != ref_dn(r)) { tgt |= 1u << ref_dn(r); n2 += 1; }
      // R3 (amb-7, amb-8)
      const uint32_t flow = ref_flow(r);
      const uint32_t flip = lower ^ flow;
      if (flip) {
        bool apply = ref_saddle(r);
        if (!apply) {
          int nl, nu;
          link_type(lower, valid, nl, nu);
          apply = (nl != ref_nlc(r)) || (nu != ref_nuc(r));
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
        const uint32_t m = lower | ((valid & ~lower) << 16);
        if (T.lmS) T.lmS[pc] = m;
        else lm[i] = m;
        if (T.gS) gs_write(T, pc, bv[7]);
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
    // warp-aggregated mark rows (as k_stencil): the targets re-indexed in
    // ascending linear order put each (dz, dy) row's 2-3 slots on adjacent
    // bits; one OR-reduction per 32-bit half builds the 34-bit row
    uint32_t rv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (__any_sync(0xffffffffu, tgt)) {
      const uint32_t t = (tgt & 0x7Fu) | ((tgt & 0x3F80u) << 1) | ((tgt >> kSelf) << 7);
      uint32_t hp = 0;  // the rows' carry-outs, 4 bits per row
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        constexpr int kStart[KR] = {0, 2, 4, 6, 9, 11, 13};
        const uint32_t cb = ((t >> kStart[k]) & (k == 3 ? 7u : 3u)) << (k >= 4 ? 1 : 0);
        // cb << tx and the bits it shifts out (cb <= 7: only lanes 30, 31
        // carry, <= 3 bits) as the low and high words of cb * 2^tx, on the
        // FMA pipe (IMAD / IMAD.HI); the carries of the 7 rows share one
        // OR-reduction (packed by IMAD: disjoint nibbles)
        rv[k] = __reduce_or_sync(0xffffffffu, cb * ptx);
        hp = __umulhi(cb, ptx) * (1u << (4 * k)) + hp;
      }
      rv[7] = __reduce_or_sync(0xffffffffu, hp);
    }
    if (tx == 0) {
      uint4 *d = reinterpret_cast<uint4 *>(&wr[z & 3][ty][0]);
      d[0] = make_uint4(rv[0], rv[1], rv[2], rv[3]);
      d[1] = make_uint4(rv[4], rv[5], rv[6], rv[7]);
    }
    const int pf = z - 2;
    if (ty == (z & (TY - 1)) && pf >= z0 - 1 && pf >= 0) flush_plane_packed(marks, wr, pf, z0, z1, x0, y0, G);
    if (prefetch) store(pz, pre);
    rc = rn;
    pc = pn;
    rn = rnn;
    __syncthreads();
  }
  {
    const int pf = z1 - 2 + ty;
    if (ty < 3 && pf >= z0 - 1 && pf >= 0 && pf < G.nz) flush_plane_packed(marks, wr, pf, z0, z1, x0, y0, G);
  }

  warp_add(&cnt[C_N1 + 0], n1);
  warp_add(&cnt[C_N1 + 1], n2);
  warp_add(&cnt[C_N1 + 2], n3);
}

}  // namespace exz

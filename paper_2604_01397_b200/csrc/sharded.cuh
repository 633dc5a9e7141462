// sharded.cuh — z-slab decomposition of the correction loop.
//
// Each rank owns the planes [z0, z0 + nzl) of the field and keeps one ghost
// plane on each side (local planes 0 and nzl + 1; NaN at the global faces).
// Per round (Alg. 1), bit-exact with the single-GPU call:
//   1. stencil R1-R3 on the owned planes (needs the ghost g planes): the key
//      stencils of exactz_correct (TMA-staged dense pass, list passes once
//      the marks are sparse), which also keep the owned entries of the
//      replicated saddle values gS and list the changed ones;
//   2. the g boundary tables (every vertex of the first / last owned plane:
//      the terminus of its steepest path inside the slab) recomputed, the
//      changed entries listed;
//   3. exchange A: one count all-reduce sizes two sparse all-gathers, the
//      changed gS entries and the changed table entries (the whole tables in
//      the first pass, or when more than half of a rank's entries changed);
//   4. C2 (R4) on the pairs whose lower saddle the rank owns;
//   5. C3 (R5/R6): label walks inside the slab; a path that leaves the slab
//      is completed from the gathered tables (table_lookup); once the marks
//      are sparse at brick scale, the brick-stamp cache of exactz_correct
//      re-emits the results whose walks stayed inside the slab;
//   6. exchange B: targets owned by another rank (sparse all-gather);
//   7. marks that fall in a ghost plane go back to the owning neighbour;
//   8. the owners count and edit; the round counters are all-reduced;
//   9. the new g boundary planes refresh the neighbours' ghost planes.
// The paper's distributed protocol exchanges ghost layers and
// uses "a consistent rule ... prioritizing smaller scalar modifications";
// here owners compute every edit and marks are ORed, so no tie rule is
// needed (amb-23) and the result equals the single-GPU result bit for bit.
//
// Transport: NCCL (one rank per process/GPU, exactz_correct_sharded) or a
// loopback that runs every rank of the decomposition in one process on one
// GPU (exactz_correct_slabs), used to test the decomposition on one device;
// its collectives are single kernels over the ranks' buffers.
#pragma once
#include <nccl.h>

#include <algorithm>
#include <memory>

namespace exz {

#define NK(call)                                                     \
  do {                                                               \
    ncclResult_t r_ = (call);                                        \
    if (r_ != ncclSuccess) {                                         \
      set_err(#call, ncclGetErrorString(r_));                        \
      throw Error{EXACTZ_ENCCL};                                     \
    }                                                                \
  } while (0)

// Collectives over the ranks of the decomposition.  Every call lists one
// buffer per LOCAL rank (1 with NCCL, all of them with the loopback).
struct Transport {
  virtual ~Transport() {}
  virtual int nranks() const = 0;
  virtual int nlocal() const = 0;
  virtual int rank_of(int l) const = 0;
  // lo_send of rank r -> hi_recv of rank r-1; hi_send of r -> lo_recv of r+1
  virtual void halo(const std::vector<const void *> &lo_send,
                    const std::vector<const void *> &hi_send, const std::vector<void *> &lo_recv,
                    const std::vector<void *> &hi_recv, size_t bytes) = 0;
  virtual void allgather(const std::vector<const void *> &send, const std::vector<void *> &recv,
                         size_t bytes) = 0;
  virtual void allreduce_sum_u64(const std::vector<unsigned long long *> &buf, size_t n) = 0;
  virtual void allreduce_max_u32(const std::vector<uint32_t *> &buf, size_t n) = 0;
  // All-to-all of 4-byte words with per-peer counts and offsets (words),
  // one entry per local rank: send[soff[q] ..+ scnt[q]) -> peer q's recv at
  // its roff[me].  The plans are static for a run (the loopback caches them).
  struct Ata {
    const uint32_t *send = nullptr;
    uint32_t *recv = nullptr;
    std::vector<size_t> soff, scnt, roff, rcnt;
  };
  virtual void alltoallv_u32(const std::vector<Ata> &a) = 0;
};

__global__ void k_sum_u64(unsigned long long *acc, const unsigned long long *src, int n) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) acc[k] += src[k];
}
__global__ void k_max_u32(uint32_t *acc, const uint32_t *src, size_t n) {
  size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (k < n) acc[k] = src[k] > acc[k] ? src[k] : acc[k];
}

// Loopback collectives as single launches (up to kLoopMax ranks): the
// ranks' buffers are all on this GPU, so a collective is one kernel over its
// segments instead of p or p^2 stream-ordered copies, whose launch costs
// would otherwise dominate the loopback's per-pass time (an artifact: with
// NCCL each rank issues one collective).
constexpr int kLoopMax = 16;
struct LoopPtrs {
  const char *a[kLoopMax];
};
struct LoopMPtrs {
  char *a[kLoopMax];
};
// block-strided copy of one segment (16-byte vectors when everything is aligned)
__device__ __forceinline__ void seg_copy(char *dst, const char *src, size_t bytes) {
  if (dst == src) return;
  const size_t t0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  if ((((uintptr_t)dst | (uintptr_t)src | bytes) & 15) == 0) {
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    for (size_t k = t0; k < bytes / 16; k += st) d4[k] = s4[k];
  } else {
    for (size_t k = t0; k < bytes; k += st) dst[k] = src[k];
  }
}
// segment y = l * p + r: recv[l] + r * bytes <- send[r]
__global__ void k_loop_allgather(LoopPtrs send, LoopMPtrs recv, int p, size_t bytes) {
  const int l = blockIdx.y / p, r = blockIdx.y - l * p;
  seg_copy(recv.a[l] + r * bytes, send.a[r], bytes);
}
// segment y = 2 r + d: d = 0: hi_recv[r - 1] <- lo_send[r]; d = 1: lo_recv[r + 1] <- hi_send[r]
__global__ void k_loop_halo(LoopPtrs lo_send, LoopPtrs hi_send, LoopMPtrs lo_recv,
                            LoopMPtrs hi_recv, int p, size_t bytes) {
  const int r = blockIdx.y >> 1, d = blockIdx.y & 1;
  if (d == 0 && r > 0) seg_copy(hi_recv.a[r - 1], lo_send.a[r], bytes);
  if (d == 1 && r + 1 < p) seg_copy(lo_recv.a[r + 1], hi_send.a[r], bytes);
}
template <class T, bool MAX>
__global__ void k_loop_reduce(LoopMPtrs buf, int p, size_t n) {
  const size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  T v = reinterpret_cast<T *>(buf.a[0])[k];
  for (int l = 1; l < p; ++l) {
    const T x = reinterpret_cast<T *>(buf.a[l])[k];
    v = MAX ? (x > v ? x : v) : v + x;
  }
  for (int l = 0; l < p; ++l) reinterpret_cast<T *>(buf.a[l])[k] = v;
}

struct CopySeg {
  const char *src;
  char *dst;
  size_t bytes;
};
// segment blockIdx.y of a descriptor list
__global__ void k_loop_segs(const CopySeg *__restrict__ seg) {
  const CopySeg g = seg[blockIdx.y];
  seg_copy(g.dst, g.src, g.bytes);
}

struct LoopTransport : Transport {
  int p;
  cudaStream_t s;
  Arena &arena;
  CopySeg *ata_seg = nullptr;  // the cached all-to-all plan (device), its key
  const void *ata_key = nullptr;
  int ata_n = 0;
  size_t ata_max = 0;
  LoopTransport(int p_, cudaStream_t s_, Arena &a) : p(p_), s(s_), arena(a) {}
  int nranks() const override { return p; }
  int nlocal() const override { return p; }
  int rank_of(int l) const override { return l; }
  template <class V>
  static LoopPtrs cptrs(const V &v) {
    LoopPtrs q{};
    for (size_t k = 0; k < v.size(); ++k) q.a[k] = (const char *)v[k];
    return q;
  }
  template <class V>
  static LoopMPtrs mptrs(const V &v) {
    LoopMPtrs q{};
    for (size_t k = 0; k < v.size(); ++k) q.a[k] = (char *)v[k];
    return q;
  }
  static unsigned seg_blocks(size_t bytes) {
    return (unsigned)std::min<size_t>(std::max<size_t>((bytes / 16 + 255) / 256, 1), 256);
  }
  void halo(const std::vector<const void *> &lo_send, const std::vector<const void *> &hi_send,
            const std::vector<void *> &lo_recv, const std::vector<void *> &hi_recv,
            size_t bytes) override {
    if (p < 2 || !bytes) return;
    if (p <= kLoopMax) {
      k_loop_halo<<<dim3(seg_blocks(bytes), 2 * p), 256, 0, s>>>(
          cptrs(lo_send), cptrs(hi_send), mptrs(lo_recv), mptrs(hi_recv), p, bytes);
      CK(cudaGetLastError());
      return;
    }
    for (int r = 0; r < p; ++r) {
      if (r > 0) CK(cudaMemcpyAsync(hi_recv[r - 1], lo_send[r], bytes, cudaMemcpyDefault, s));
      if (r + 1 < p) CK(cudaMemcpyAsync(lo_recv[r + 1], hi_send[r], bytes, cudaMemcpyDefault, s));
    }
  }
  void allgather(const std::vector<const void *> &send, const std::vector<void *> &recv,
                 size_t bytes) override {
    if (!bytes) return;
    if (p <= kLoopMax) {
      k_loop_allgather<<<dim3(seg_blocks(bytes), p * p), 256, 0, s>>>(cptrs(send), mptrs(recv), p,
                                                                      bytes);
      CK(cudaGetLastError());
      return;
    }
    for (int l = 0; l < p; ++l)
      for (int r = 0; r < p; ++r)
        if ((const char *)recv[l] + r * bytes != send[r])  // (in place: nothing to copy)
          CK(cudaMemcpyAsync((char *)recv[l] + r * bytes, send[r], bytes, cudaMemcpyDefault, s));
  }
  void allreduce_sum_u64(const std::vector<unsigned long long *> &buf, size_t n) override {
    if (p < 2 || !n) return;
    if (p <= kLoopMax) {
      k_loop_reduce<unsigned long long, false><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
          mptrs(buf), p, n);
      CK(cudaGetLastError());
      return;
    }
    for (int l = 1; l < p; ++l)
      k_sum_u64<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(buf[0], buf[l], (int)n);
    CK(cudaGetLastError());
    for (int l = 1; l < p; ++l) CK(cudaMemcpyAsync(buf[l], buf[0], n * 8, cudaMemcpyDefault, s));
  }
  void alltoallv_u32(const std::vector<Ata> &a) override {
    if (ata_key != (const void *)a[0].send) {  // build the segment list once per plan
      std::vector<CopySeg> segs;
      size_t mx = 0;
      for (int r = 0; r < p; ++r)
        for (int q = 0; q < p; ++q)
          if (q != r && a[r].scnt[q]) {
            segs.push_back(CopySeg{(const char *)(a[r].send + a[r].soff[q]),
                                   (char *)(a[q].recv + a[q].roff[r]), a[r].scnt[q] * 4});
            mx = std::max(mx, a[r].scnt[q] * 4);
          }
      ata_n = (int)segs.size();
      ata_max = mx;
      if (ata_n) {
        ata_seg = arena.get<CopySeg>(segs.size());
        CK(cudaMemcpyAsync(ata_seg, segs.data(), segs.size() * sizeof(CopySeg),
                           cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));  // (segs is a host temporary)
      }
      ata_key = a[0].send;
    }
    if (!ata_n) return;
    k_loop_segs<<<dim3(seg_blocks(ata_max), ata_n), 256, 0, s>>>(ata_seg);
    CK(cudaGetLastError());
  }
  void allreduce_max_u32(const std::vector<uint32_t *> &buf, size_t n) override {
    if (p < 2 || !n) return;
    if (p <= kLoopMax) {
      k_loop_reduce<uint32_t, true><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(mptrs(buf), p, n);
      CK(cudaGetLastError());
      return;
    }
    for (int l = 1; l < p; ++l)
      k_max_u32<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(buf[0], buf[l], n);
    CK(cudaGetLastError());
    for (int l = 1; l < p; ++l) CK(cudaMemcpyAsync(buf[l], buf[0], n * 4, cudaMemcpyDefault, s));
  }
};

}  // namespace exz

struct exactz_comm {
  ncclComm_t nccl;
  int nranks, rank, device;
};

namespace exz {

struct NcclTransport : Transport {
  exactz_comm *c;
  cudaStream_t s;
  NcclTransport(exactz_comm *c_, cudaStream_t s_) : c(c_), s(s_) {}
  int nranks() const override { return c->nranks; }
  int nlocal() const override { return 1; }
  int rank_of(int) const override { return c->rank; }
  void halo(const std::vector<const void *> &lo_send, const std::vector<const void *> &hi_send,
            const std::vector<void *> &lo_recv, const std::vector<void *> &hi_recv,
            size_t bytes) override {
    const int r = c->rank, p = c->nranks;
    NK(ncclGroupStart());
    if (r > 0) {
      NK(ncclSend(lo_send[0], bytes, ncclUint8, r - 1, c->nccl, s));
      NK(ncclRecv(lo_recv[0], bytes, ncclUint8, r - 1, c->nccl, s));
    }
    if (r + 1 < p) {
      NK(ncclSend(hi_send[0], bytes, ncclUint8, r + 1, c->nccl, s));
      NK(ncclRecv(hi_recv[0], bytes, ncclUint8, r + 1, c->nccl, s));
    }
    NK(ncclGroupEnd());
  }
  void allgather(const std::vector<const void *> &send, const std::vector<void *> &recv,
                 size_t bytes) override {
    NK(ncclAllGather(send[0], recv[0], bytes, ncclUint8, c->nccl, s));
  }
  void allreduce_sum_u64(const std::vector<unsigned long long *> &buf, size_t n) override {
    NK(ncclAllReduce(buf[0], buf[0], n, ncclUint64, ncclSum, c->nccl, s));
  }
  void allreduce_max_u32(const std::vector<uint32_t *> &buf, size_t n) override {
    if (n) NK(ncclAllReduce(buf[0], buf[0], n, ncclUint32, ncclMax, c->nccl, s));
  }
  void alltoallv_u32(const std::vector<Ata> &a) override {
    const int me = c->rank, p = c->nranks;
    NK(ncclGroupStart());
    for (int q = 0; q < p; ++q) {
      if (q == me) continue;
      if (a[0].scnt[q]) NK(ncclSend(a[0].send + a[0].soff[q], a[0].scnt[q], ncclUint32, q, c->nccl, s));
      if (a[0].rcnt[q]) NK(ncclRecv(a[0].recv + a[0].roff[q], a[0].rcnt[q], ncclUint32, q, c->nccl, s));
    }
    NK(ncclGroupEnd());
  }
};

// Planes of rank r in an nz-plane field split over p ranks: the first nz % p
// ranks get one extra plane.
static void slab_range(int64_t nz, int p, int r, int64_t *z0, int64_t *cnt) {
  int64_t base = nz / p, extra = nz % p;
  *cnt = base + (r < extra ? 1 : 0);
  *z0 = r * base + (r < extra ? r : extra);
}

// One rank's state (device buffers in the local slab layout).
struct Slab {
  int rank = 0, z0 = 0, nzl = 0;
  GridP G{};
  dim3 sgrid;
  int zc = 1;
  bool fast = false;  // every lo >= 0 (all ranks): k_stencil_fast
  bool keyed = false; // the call's value range fits exact SoS keys: the key stencils
  bool tma = false;   // k_stencil_key2 stages planes by TMA (tmap over this slab's g)
  CUtensorMap tmap{};
  uint32_t *kmm = nullptr;  // ~bits(lo_min), bits(g_max) of this rank, max-reduced
  int32_t *own = nullptr;   // positions k in S whose S[k] this slab owns (R4 pairs)
  int nown = 0;
  float *f = nullptr, *g = nullptr;
  uint32_t *ref = nullptr, *marks = nullptr, *ghost_lo = nullptr, *ghost_hi = nullptr;
  uint8_t *slots = nullptr, *c = nullptr;
  uint32_t *lm = nullptr;  // g-lower | g-upper << 16 link masks at the f-saddles (stencil -> C3 events)
  uint64_t *keys = nullptr, *allkeys = nullptr, *sorted = nullptr;
  int32_t *S = nullptr, *J = nullptr, *P = nullptr, *m1 = nullptr, *M1 = nullptr;
  int nJ = 0, nP = 0;
  int2 *tdn = nullptr, *tup = nullptr;  // gathered boundary tables (2 p A each, contiguous)
  int4 *tupd = nullptr, *alltupd = nullptr;  // changed table entries: this rank's / gathered
  size_t alltupd_cap = 0;
  uint32_t *gS = nullptr;
  uint64_t *cpkeys = nullptr;
  int32_t *CP = nullptr;  // reformulation: all critical points, replicated
  uint32_t *gC = nullptr;
  int32_t *remote = nullptr, *allremote = nullptr;
  size_t allremote_cap = 0;  // grown on demand (geometric)
  // sparse exchange of the replicated gS: positions in S of the owned
  // saddles (local index), this round's changed entries, all ranks' lists
  int32_t *posS = nullptr;
  uint32_t *gSprev = nullptr;  // the owned entries as last listed (k_gs_diff)
  // R4 partner values by static routing (k_r4_route): positions sent /
  // received (grouped by peer), their buffers, the per-peer plan
  int32_t *r4s = nullptr, *r4r = nullptr;
  uint32_t *r4sbuf = nullptr, *r4rbuf = nullptr;
  int r4ns = 0, r4nr = 0;
  std::vector<size_t> r4soff, r4scnt, r4roff, r4rcnt;
  int2 *upd = nullptr, *allupd = nullptr;
  unsigned long long *cnt = nullptr, *hcnt = nullptr;  // device counters / host mirror
  unsigned long long *nrem = nullptr;                    // per-rank remote counts (p)
  // vertex activity (list-based passes, as exactz_correct): act[cur] = this
  // pass's set (owned planes), edited = the last pass's edits with the
  // neighbours' boundary planes in the ghost planes
  uint32_t *act[2] = {nullptr, nullptr}, *edited = nullptr;
  int32_t *list = nullptr;
  int *nlist = nullptr;
  // the C3 cache (brick stamps, as exactz_correct's Tracking) over the local
  // buffer; results whose walks leave the slab are never reused (kFar)
  int nbx = 0, nby = 0, nbz = 0, nsx = 0, nsy = 0, nsz = 0;
  uint16_t *bval = nullptr, *bslot = nullptr, *sbval = nullptr, *sbslot = nullptr;
  EvCache ecJ{}, ecP{};
  int *todo = nullptr, *todoP = nullptr, *ntodo = nullptr;
  // the clean-path test of the C3 walks (exactz_correct's FPaths, slab-local)
  FPaths fpJ{}, fpP{};
  uint8_t *dirtD = nullptr, *dirtU = nullptr;
  unsigned long long *ndirt = nullptr;
  int ntx = 0, nty = 0, nt = 0;
  int *ftodo = nullptr, *ftodoP = nullptr, *nftodo = nullptr;
  float *ghost_prev = nullptr;         // the ghost planes' values as last stamped
  uint16_t *brnd = nullptr;            // boundary-table entries: round and bricks of the
  unsigned long long *bmask = nullptr; // last walk (k_boundary_delta<true>)
  size_t plane() const { return (size_t)G.nx * G.ny; }
  size_t words_per_plane() const { return (size_t)G.ny * G.W; }
};

struct ShardedRun {
  Transport &T;
  cudaStream_t s;
  Arena &A;
  std::vector<Slab> &sl;
  int p, nx, ny, nz, nS = 0, nC = 0;
  bool reform = false;
  int *d_start = nullptr;  // slab starts (device), p + 1 entries
  int N;
  float xi, delta;
  uint32_t flags;
  bool act_on = false, ready = false;  // vertex activity started / act[cur] valid
  bool cache_on = false;               // the C3 cache started
  // stars of this pass's edits: pulled next pass (edited bitmap, dilated by
  // k_act_list) when many, pushed into act_next by the edit when few, as
  // exactz_correct decides (set by the caller from the global V_t)
  bool pull = true, edited_valid = false;
  bool fp_on = false;                  // the clean-path test is set up (list passes use it)
  int rnd = 0;                         // pass number (16-bit stamps of the cache)
  int tab_round = 0;                   // last pass in which a g boundary-table entry changed
  bool tables_ready = false;           // the g boundary tables hold a previous pass's
  int cur = 0;

  ShardedRun(Transport &t, cudaStream_t st, Arena &a, std::vector<Slab> &slabs, int nx_, int ny_,
             int nz_, float xi_, int N_, uint32_t flags_)
      : T(t), s(st), A(a), sl(slabs), p(t.nranks()), nx(nx_), ny(ny_), nz(nz_), N(N_), xi(xi_),
        flags(flags_) {
    delta = xi / (float)N;
    reform = (flags & EXACTZ_REFORMULATED) != 0;
  }

  template <class F>
  void each(F fn) {
    for (auto &x : sl) fn(x);
  }
  void sync() { CK(cudaStreamSynchronize(s)); }
  void read_counters() {
    each([&](Slab &x) {
      k_fold_counters<<<1, 32, 0, s>>>(x.cnt);  // warp_add replicas (kernels.cuh)
      g_launches++;
      CK(cudaMemcpyAsync(x.hcnt, x.cnt, C_NCOUNTERS * 8, cudaMemcpyDeviceToHost, s));
    });
    sync();
  }
  void zero_counters() {
    each([&](Slab &x) { CK(cudaMemsetAsync(x.cnt, 0, C_NALLOC * 8, s)); });
  }

  void start_act() {
    each([&](Slab &x) {
      const size_t n = (size_t)x.G.nz * x.words_per_plane();
      for (int k = 0; k < 2; ++k) {
        x.act[k] = A.get<uint32_t>(n);
        CK(cudaMemsetAsync(x.act[k], 0, n * 4, s));
      }
      x.edited = A.get<uint32_t>(n);
      CK(cudaMemsetAsync(x.edited, 0, n * 4, s));
      x.list = A.get<int32_t>((size_t)x.G.V);
      x.nlist = A.get<int>(1);
    });
    act_on = true;
  }
  // The clean-path test (exactz_correct's Tracking::start_fpaths): the f-walks
  // of every saddle inside its slab, their tiles and f-labels; a saddle whose
  // f-walks leave the slab is always walked.  gate: see exactz_correct.
  void start_fpaths(double gate) {
    each([&](Slab &x) {
      x.ntx = (nx + (1 << FTX_SH) - 1) >> FTX_SH;
      x.nty = (ny + (1 << FTY_SH) - 1) >> FTY_SH;
      const int ntz = (x.G.nz + (1 << FTZ_SH) - 1) >> FTZ_SH;
      x.nt = x.ntx * x.nty * ntz;
      const size_t nt16 = ((size_t)x.nt + 15) / 16 * 16;
      x.dirtD = A.get<uint8_t>(2 * nt16 + 16);
      x.dirtU = x.dirtD + nt16;
      x.ndirt = reinterpret_cast<unsigned long long *>(x.dirtD + 2 * nt16);
      unsigned long long *bump = A.get<unsigned long long>(2);
      CK(cudaMemsetAsync(bump, 0, 16, s));
      auto alloc = [&](int n) {
        FPaths F{};
        const size_t m = n ? (size_t)n : 1;
        F.off = A.get<int64_t>(m);
        F.len = A.get<uint16_t>(m);
        F.lab = A.get<int32_t>(m * kFLab);
        F.nlab = A.get<uint8_t>(m);
        F.bmask = A.get<unsigned long long>(m);
        F.flow = A.get<uint16_t>(m);
        F.cap = 24ull * m + 4096;
        F.tiles = A.get<int32_t>(F.cap);
        return F;
      };
      x.fpJ = alloc(x.nJ);
      x.fpP = alloc(x.nP);
      for (int sp = 0; sp < 2; ++sp) {
        const FPaths &F = sp ? x.fpP : x.fpJ;
        const int n = sp ? x.nP : x.nJ;
        if (n <= 0) continue;
        auto go = [&](auto kern) {
          kern<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
              sp ? x.P : x.J, n, x.ref, x.G, x.ntx, x.nty, bump + sp, F.cap,
              const_cast<int64_t *>(F.off), const_cast<uint16_t *>(F.len),
              const_cast<int32_t *>(F.tiles), const_cast<int32_t *>(F.lab),
              const_cast<uint8_t *>(F.nlab), const_cast<unsigned long long *>(F.bmask), nullptr,
              x.f, nullptr, const_cast<uint16_t *>(F.flow), nullptr);
        };
        if (sp) go(k_fpaths<true, true>);
        else go(k_fpaths<false, true>);
      }
      CK(cudaGetLastError());
      unsigned long long h[2] = {0, 0};
      CK(cudaMemcpyAsync(h, bump, sizeof(h), cudaMemcpyDeviceToHost, s));
      sync();
      for (int sp = 0; sp < 2; ++sp) {
        FPaths &F = sp ? x.fpP : x.fpJ;
        const int n = sp ? x.nP : x.nJ;
        const double L = n ? (double)h[sp] / n : 0.0;
        const double fr = gate > 0.0 && L > 0.0 ? 1.0 - std::pow(gate, 1.0 / L) : 1.0;
        F.max_dirt = gate > 0.0 ? (unsigned long long)(fr * x.nt) : ~0ull;
        F.dirt = sp ? x.dirtU : x.dirtD;
        F.nt = x.nt;
        F.ndirt = x.ndirt + sp;
      }
      x.ftodo = A.get<int>(std::max(x.nJ, 1));
      x.ftodoP = A.get<int>(std::max(x.nP, 1));
      x.nftodo = A.get<int>(2);
    });
    fp_on = true;
  }

  void start_cache() {
    each([&](Slab &x) {
      x.nbx = (x.G.nx + BX - 1) / BX;
      x.nby = (x.G.ny + BY - 1) / BY;
      x.nbz = (x.G.nz + BZ - 1) / BZ;
      x.nsx = (x.nbx + SB - 1) / SB;
      x.nsy = (x.nby + SB - 1) / SB;
      x.nsz = (x.nbz + SB - 1) / SB;
      const size_t nb = (size_t)x.nbx * x.nby * x.nbz, nsb = (size_t)x.nsx * x.nsy * x.nsz;
      uint16_t *st = A.get<uint16_t>(2 * (nb + nsb));
      CK(cudaMemsetAsync(st, 0, 2 * (nb + nsb) * 2, s));
      x.bval = st;
      x.bslot = st + nb;
      x.sbval = st + 2 * nb;
      x.sbslot = x.sbval + nsb;
      auto cache = [&](int n) {
        EvCache e{};
        const size_t m = n > 0 ? (size_t)n : 1;
        e.rnd = A.get<uint16_t>(m);
        e.mask = A.get<unsigned long long>(m);
        e.tgt = A.get<int32_t>(m);
        CK(cudaMemsetAsync(e.rnd, 0, m * 2, s));
        CK(cudaMemsetAsync(e.mask, 0, m * 8, s));
        return e;
      };
      x.ecJ = cache(x.nJ);
      x.ecP = cache(x.nP);
      const size_t A4 = 4 * x.plane();
      x.ghost_prev = A.get<float>(2 * x.plane());
      CK(cudaMemcpyAsync(x.ghost_prev, x.g, x.plane() * 4, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(x.ghost_prev + x.plane(), x.g + (size_t)(x.G.nz - 1) * x.plane(),
                         x.plane() * 4, cudaMemcpyDeviceToDevice, s));
      x.brnd = A.get<uint16_t>(A4);
      x.bmask = A.get<unsigned long long>(A4);
      CK(cudaMemsetAsync(x.brnd, 0, A4 * 2, s));
      x.todo = A.get<int>(std::max(x.nJ, 1));
      x.todoP = A.get<int>(std::max(x.nP, 1));
      x.ntodo = A.get<int>(2);
    });
    cache_on = true;
  }

  // the neighbours' edits of their boundary planes into the ghost planes of
  // `edited` (stars that cross the slab border)
  void halo_edited() {
    std::vector<const void *> lo, hi;
    std::vector<void *> rlo, rhi;
    each([&](Slab &x) {
      const size_t W = x.words_per_plane();
      lo.push_back(x.edited + W * 1);
      hi.push_back(x.edited + W * x.nzl);
      rlo.push_back(x.edited);
      rhi.push_back(x.edited + W * (x.nzl + 1));
    });
    T.halo(lo, hi, rlo, rhi, sl[0].words_per_plane() * 4);
  }

  void halo_planes(bool of_f) {
    std::vector<const void *> lo, hi;
    std::vector<void *> rlo, rhi;
    each([&](Slab &x) {
      float *b = of_f ? x.f : x.g;
      const size_t P = x.plane();
      lo.push_back(b + P * 1);
      hi.push_back(b + P * x.nzl);
      rlo.push_back(b);
      rhi.push_back(b + P * (x.nzl + 1));
    });
    T.halo(lo, hi, rlo, rhi, (size_t)nx * ny * sizeof(float));
  }

  void setup(const std::vector<const float *> &f_in, const std::vector<const float *> &g_in) {
    int64_t gz0 = 0, gc = 0;
    std::vector<int> starts(p + 1);
    for (int r = 0; r < p; ++r) {
      slab_range(nz, p, r, &gz0, &gc);
      starts[r] = (int)gz0;
    }
    starts[p] = nz;
    d_start = A.get<int>(p + 1);
    CK(cudaMemcpyAsync(d_start, starts.data(), (p + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
    for (size_t l = 0; l < sl.size(); ++l) {
      Slab &x = sl[l];
      x.rank = T.rank_of((int)l);
      slab_range(nz, p, x.rank, &gz0, &gc);
      x.z0 = (int)gz0;
      x.nzl = (int)gc;
      GridP &G = x.G;
      G.nx = nx;
      G.ny = ny;
      G.nz = x.nzl + 2;
      G.V = nx * ny * G.nz;
      G.W = (nx + 31) / 32;
      grid_fastdiv(G);
      for (int k = 0; k < kSlots; ++k)
        G.delta[k] = kOff[k][0] + nx * (kOff[k][1] + ny * kOff[k][2]);
      G.zoff = x.z0 - 1;
      G.gnz = nz;
      G.zb = 1;
      G.ze = x.nzl + 1;
      {  // z chunk per stencil CTA, as exactz_correct: enough CTAs for several
         // waves on 148 SMs (a slab of 64 planes in chunks of 32 left the key
         // stencil 2.3 waves, 30 % lost to the tail), >= 8 planes per chunk
        const int64_t cols = (int64_t)((nx + TX - 1) / TX) * ((ny + TY - 1) / TY), want = 148 * 24;
        const int64_t z = cols >= want ? x.nzl : (x.nzl * cols + want - 1) / want;
        x.zc = (int)std::min<int64_t>(std::max<int64_t>(z, 8), 64);
        x.zc = std::max(1, std::min(x.zc, x.nzl));
      }
      x.sgrid = dim3((unsigned)((nx + TX - 1) / TX), (unsigned)((ny + TY - 1) / TY),
                     (unsigned)((x.nzl + x.zc - 1) / x.zc));
      const size_t P = x.plane(), Vl = (size_t)G.V;
      x.f = A.get<float>(Vl);
      x.g = A.get<float>(Vl);
      x.ref = A.get<uint32_t>(Vl);
      x.slots = A.get<uint8_t>(Vl);
      x.lm = A.get<uint32_t>(Vl);
      x.c = A.get<uint8_t>(Vl);
      x.marks = A.get<uint32_t>((size_t)G.nz * x.words_per_plane());
      x.ghost_lo = A.get<uint32_t>(x.words_per_plane());
      x.ghost_hi = A.get<uint32_t>(x.words_per_plane());
      x.cnt = A.get<unsigned long long>(C_NALLOC);
      CK(cudaMallocHost(&x.hcnt, C_NCOUNTERS * 8));
      x.nrem = A.get<unsigned long long>(3 * p);
      x.keys = A.get<uint64_t>(x.nzl * P);
      if (reform) x.cpkeys = A.get<uint64_t>(x.nzl * P);
      // the table pair [dn | up] (k_boundary_delta's positions), this rank's
      // changed entries, and the gathered changes (at most A / 2 per rank:
      // beyond that the whole chunks travel)
      x.tdn = A.get<int2>(4 * p * P);
      x.tup = x.tdn + 2 * p * P;
      x.tupd = A.get<int4>(4 * P);
      x.alltupd = A.get<int4>(p * (P / 2 + 1));
      x.alltupd_cap = p * (P / 2 + 1);
      // owned planes from the caller; ghost planes NaN until the halo exchange
      CK(cudaMemsetAsync(x.f, 0xff, Vl * 4, s));
      CK(cudaMemsetAsync(x.g, 0xff, Vl * 4, s));
      CK(cudaMemcpyAsync(x.f + P, f_in[l], (size_t)x.nzl * P * 4, cudaMemcpyDefault, s));
      CK(cudaMemcpyAsync(x.g + P, g_in[l], (size_t)x.nzl * P * 4, cudaMemcpyDefault, s));
      CK(cudaMemsetAsync(x.c, 0, Vl, s));
      // ghost-plane slots: kSelf in both nibbles, never written (a g walk
      // stops at a ghost vertex by itself; walk())
      CK(cudaMemsetAsync(x.slots, 0xEE, P, s));
      CK(cudaMemsetAsync(x.slots + (size_t)(x.nzl + 1) * P, 0xEE, P, s));
      CK(cudaMemsetAsync(x.marks, 0, (size_t)G.nz * x.words_per_plane() * 4, s));
    }
    halo_planes(true);
    halo_planes(false);
    // O1 validation on the owned planes, agreed by all ranks
    zero_counters();
    each([&](Slab &x) {
      const size_t P = x.plane();
      k_validate<<<blocks_for(x.nzl * P, 256), 256, 0, s>>>(x.f + P, x.g + P, x.nzl * P, xi, x.cnt);
    });
    CK(cudaGetLastError());
    // the value range of the call (the key stencils' applicability, as
    // exactz_correct decides it from the whole field): max over the ranks
    {
      std::vector<uint32_t *> km;
      each([&](Slab &x) {
        x.kmm = A.get<uint32_t>(2);
        CK(cudaMemcpyAsync(x.kmm, reinterpret_cast<const uint32_t *>(x.cnt + C_KEYMIN), 4,
                           cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(x.kmm + 1, reinterpret_cast<const uint32_t *>(x.cnt + C_KEYMAX), 4,
                           cudaMemcpyDeviceToDevice, s));
        km.push_back(x.kmm);
      });
      T.allreduce_max_u32(km, 2);
    }
    uint32_t hk[2] = {0, 0};
    CK(cudaMemcpyAsync(hk, sl[0].kmm, sizeof(hk), cudaMemcpyDeviceToHost, s));
    // C_NEG too: every slab must make the single-GPU call's fast/general
    // stencil choice, which depends on the whole field (the halo planes of a
    // slab hold a neighbour's values).  The other counters are zero here.
    allreduce_counters(C_NEG + 1);
    read_counters();
    if (sl[0].hcnt[C_BAD_NF]) {
      set_err("validate", "non-finite value in f or g");
      throw Error{EXACTZ_EINVAL};
    }
    if (sl[0].hcnt[C_BAD_BOUND]) {
      set_err("validate", "|f - g| > eps for some vertex");
      throw Error{EXACTZ_EBOUND};
    }
    each([&](Slab &x) {
      x.fast = x.hcnt[C_NEG] == 0 && !(flags & 0x800u);
      // exact SoS keys (stencil_key.cuh), as exactz_correct (debug 0x2000: off)
      const uint32_t lo_min = ~hk[0], g_max = hk[1];
      x.keyed = x.fast && !(flags & 0x2000u) && lo_min >= kKeyLoMinBits &&
                g_max < kKeyHiMaxBits && g_max >= lo_min && g_max - lo_min < kKeySpan;
      for (int q = 0; q < kSlots; ++q) x.G.kc[q] = (uint32_t)q - 16u * lo_min;
      // (debug 0x8000: thread-staged planes)
      x.tma = x.keyed && !(flags & 0x8000u) && encode_plane_map(&x.tmap, x.g, nx, ny, x.G.nz);
    });
    // O7 reference of f on the owned planes
    zero_counters();
    each([&](Slab &x) {
      // the z-marching tile kernel of exactz_correct over the owned planes
      k_reference_tile<<<x.sgrid, 256, 0, s>>>(x.f, x.G, x.zc, x.ref, x.keys, x.cpkeys, x.cnt);
    });
    CK(cudaGetLastError());
    read_counters();
    // S: the saddle keys of every rank, gathered and sorted identically
    std::vector<unsigned long long *> nb;
    unsigned long long maxk = 0;
    each([&](Slab &x) {
      CK(cudaMemsetAsync(x.nrem, 0, 2 * p * 8, s));
      CK(cudaMemcpyAsync(x.nrem + x.rank, x.cnt + C_NSADDLE, 8, cudaMemcpyDeviceToDevice, s));
      nb.push_back(x.nrem);
    });
    T.allreduce_sum_u64(nb, p);
    std::vector<unsigned long long> counts(p);
    CK(cudaMemcpyAsync(counts.data(), sl[0].nrem, p * 8, cudaMemcpyDeviceToHost, s));
    sync();
    nS = 0;
    for (int r = 0; r < p; ++r) {
      nS += (int)counts[r];
      maxk = std::max(maxk, counts[r]);
    }
    const size_t slot = std::max<size_t>(maxk, 1);
    std::vector<const void *> ks;
    std::vector<void *> ka;
    each([&](Slab &x) {
      uint64_t *pad = A.get<uint64_t>(slot);
      CK(cudaMemsetAsync(pad, 0xff, slot * 8, s));  // UINT64_MAX sorts last
      // each rank sorts its own keys; the gathered sorted runs are merged
      // below (a replicated radix sort of all nS keys cost every rank ~2 ms
      // at C5 / 8)
      const int nk = (int)counts[x.rank];
      if (nk) {
        size_t tb0 = 0;
        CK(cub::DeviceRadixSort::SortKeys(nullptr, tb0, x.keys, pad, nk, 0, 64, s));
        void *tmp0 = A.get<uint8_t>(tb0);
        CK(cub::DeviceRadixSort::SortKeys(tmp0, tb0, x.keys, pad, nk, 0, 64, s));
      }
      x.allkeys = A.get<uint64_t>(slot * p);
      x.sorted = A.get<uint64_t>(slot * p);
      ks.push_back(pad);
      ka.push_back(x.allkeys);
    });
    T.allgather(ks, ka, slot * 8);
    each([&](Slab &x) {
      x.S = A.get<int32_t>(std::max(nS, 1));
      // pairwise merges of the p sorted runs (padding sorts last in each run
      // and stays after the nS keys)
      uint64_t *a = x.allkeys, *b = x.sorted;
      const size_t total = slot * p;
      size_t tbm = 0;
      if (p > 1) {
        const int h = (int)std::min<size_t>(total / 2, (size_t)INT32_MAX);
        CK(cub::DeviceMerge::MergeKeys(nullptr, tbm, a, h, a + h, h, b, ::cuda::std::less<>{}, s));
      }
      void *tmpm = tbm ? A.get<uint8_t>(tbm) : nullptr;
      for (size_t L = slot; L < total; L *= 2) {
        for (size_t st = 0; st < total; st += 2 * L) {
          const size_t n1 = std::min(L, total - st), n2 = st + L < total ? std::min(L, total - st - L) : 0;
          if (n2) {
            size_t need = 0;
            CK(cub::DeviceMerge::MergeKeys(nullptr, need, a + st, (int)n1, a + st + L, (int)n2, b + st,
                                           ::cuda::std::less<>{}, s));
            if (need > tbm) {
              tbm = need;
              tmpm = A.get<uint8_t>(tbm);
            }
            CK(cub::DeviceMerge::MergeKeys(tmpm, need, a + st, (int)n1, a + st + L, (int)n2, b + st,
                                           ::cuda::std::less<>{}, s));
          } else {
            CK(cudaMemcpyAsync(b + st, a + st, n1 * 8, cudaMemcpyDeviceToDevice, s));
          }
        }
        std::swap(a, b);
      }
      x.sorted = a;  // (the merged keys)
      if (nS) k_keys_to_ids<<<(nS + 255) / 256, 256, 0, s>>>(a, x.S, nS);
      x.gS = A.get<uint32_t>(std::max(nS, 1));
      // (a walk target per join and per split saddle the slab owns)
      x.remote = A.get<int32_t>(2 * (size_t)std::max(nS, 1));
      x.posS = A.get<int32_t>(x.G.V);
      CK(cudaMemsetAsync(x.posS, 0xff, (size_t)x.G.V * 4, s));
      if (nS) k_local_pos<<<(nS + 255) / 256, 256, 0, s>>>(x.S, nS, x.posS, x.G);
      x.upd = A.get<int2>(slot);          // at most the owned saddles
      x.allupd = A.get<int2>(slot * p);
      // J, P: owned saddles in index order (global ids)
      const int lo = x.G.zb * (int)x.plane(), n = x.nzl * (int)x.plane();
      x.J = A.get<int32_t>(std::max<int64_t>(counts[x.rank], 1));
      x.P = A.get<int32_t>(std::max<int64_t>(counts[x.rank], 1));
      int *nsel = A.get<int>(3);
      cub::CountingInputIterator<int32_t> ids(lo);
      // R4 pairs (S[k], S[k+1]) whose S[k] this slab owns: their positions k
      x.own = A.get<int32_t>(std::max(nS, 1));
      cub::CountingInputIterator<int32_t> ks(0);
      const OwnedInS ow{x.S, x.z0 * (int)x.plane(), (x.z0 + x.nzl) * (int)x.plane()};
      size_t t2 = 0, t3 = 0, t4 = 0;
      CK(cub::DeviceSelect::If(nullptr, t2, ids, x.J, nsel, n, IsJoin{x.ref}, s));
      CK(cub::DeviceSelect::If(nullptr, t3, ids, x.P, nsel + 1, n, IsSplit{x.ref}, s));
      CK(cub::DeviceSelect::If(nullptr, t4, ks, x.own, nsel + 2, std::max(nS, 1), ow, s));
      void *tmp2 = A.get<uint8_t>(std::max(std::max(t2, t3), t4));
      CK(cub::DeviceSelect::If(tmp2, t2, ids, x.J, nsel, n, IsJoin{x.ref}, s));
      CK(cub::DeviceSelect::If(tmp2, t3, ids, x.P, nsel + 1, n, IsSplit{x.ref}, s));
      if (nS) CK(cub::DeviceSelect::If(tmp2, t4, ks, x.own, nsel + 2, nS, ow, s));
      else CK(cudaMemsetAsync(nsel + 2, 0, sizeof(int), s));
      int h[3];
      CK(cudaMemcpyAsync(h, nsel, sizeof(h), cudaMemcpyDeviceToHost, s));
      sync();
      x.nJ = h[0];
      x.nP = h[1];
      x.nown = h[2];
      const int off = x.G.zoff * (int)x.plane();
      if (x.nJ) k_add_offset<<<(x.nJ + 255) / 256, 256, 0, s>>>(x.J, x.nJ, off);
      if (x.nP) k_add_offset<<<(x.nP + 255) / 256, 256, 0, s>>>(x.P, x.nP, off);
      x.m1 = A.get<int32_t>(std::max(x.nJ, 1));
      x.M1 = A.get<int32_t>(std::max(x.nP, 1));
    });
    CK(cudaGetLastError());
    // the replicated saddle values of the input: one full exchange (owners
    // fill, max-all-reduce); afterwards only the entries that change travel
    if (nS > 1) {
      std::vector<uint32_t *> b;
      each([&](Slab &x) {
        k_fill_gS<<<(nS + 255) / 256, 256, 0, s>>>(x.g, x.S, nS, x.gS, x.G);
        b.push_back(x.gS);
      });
      T.allreduce_max_u32(b, nS);
      each([&](Slab &x) {
        x.gSprev = A.get<uint32_t>(nS);
        CK(cudaMemcpyAsync(x.gSprev, x.gS, (size_t)nS * 4, cudaMemcpyDeviceToDevice, s));
      });
      if (p > 1) r4_routes();
    }
    if (reform) {
      gather_sorted(C_NCP, [](Slab &x) { return x.cpkeys; },
                    [](Slab &x, int32_t *ids) { x.CP = ids; }, nC);
      each([&](Slab &x) { x.gC = A.get<uint32_t>(std::max(nC, 1)); });
      return;
    }
    // m1 / M1 from f's paths, completed across slabs
    zero_counters();
    boundary_tables(true);
    each([&](Slab &x) {
      events<false, true>(x, x.f, x.J, x.nJ, x.m1);
      events<true, true>(x, x.f, x.P, x.nP, x.M1);
    });
    read_counters();
    each([&](Slab &x) {
      if (x.hcnt[C_CHANGED]) {
        set_err("boundary_tables", "an exit chain is longer than the table (a cycle)");
        throw Error{EXACTZ_ECUDA};
      }
    });
    // the clean-path test for the list passes, as exactz_correct decides it
    // (debug 0x80000: off; 0x200000: run whatever the dirty-tile count)
    if (!(flags & (EXACTZ_NO_TRACK | EXACTZ_NO_C3 | 0x80000u | 0x100u | 0x400u))) {
      static const double gate = [] {
        const char *e = std::getenv("EXACTZ_FP_GATE");
        return e ? std::atof(e) : 0.1;
      }();
      start_fpaths((flags & 0x200000u) ? 0.0 : gate);
    }
  }

  // The static R4 routing (see k_r4_route): per slab the positions it sends
  // and receives, grouped by peer, in ascending order within a peer.
  void r4_routes() {
    const int A2 = nx * ny, base = nz / p, extra = nz % p;
    int bits = 1;
    while ((1 << bits) <= p) ++bits;
    each([&](Slab &x) {
      x.r4soff.assign(p, 0);
      x.r4scnt.assign(p, 0);
      x.r4roff.assign(p, 0);
      x.r4rcnt.assign(p, 0);
      const int n = x.nown;
      x.r4sbuf = A.get<uint32_t>(std::max(n, 1));
      x.r4rbuf = A.get<uint32_t>(std::max(n, 1));
      if (!n) return;
      int32_t *k0 = A.get<int32_t>(n), *p0 = A.get<int32_t>(n), *k1 = A.get<int32_t>(n),
              *p1 = A.get<int32_t>(n);
      int32_t *sk = A.get<int32_t>(n), *rk = A.get<int32_t>(n);
      x.r4s = A.get<int32_t>(n);
      x.r4r = A.get<int32_t>(n);
      k_r4_route<<<(n + 255) / 256, 256, 0, s>>>(x.own, n, x.S, nS, A2, base, extra, x.rank, p, k0,
                                                 p0, k1, p1);
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, sk, p0, x.r4s, n, 0, bits, s));
      void *tmp = A.get<uint8_t>(tb);
      CK(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, sk, p0, x.r4s, n, 0, bits, s));
      CK(cub::DeviceRadixSort::SortPairs(tmp, tb, k1, rk, p1, x.r4r, n, 0, bits, s));
      int *st = A.get<int>(2 * (p + 1));
      std::vector<int> init(2 * (p + 1), n);
      CK(cudaMemcpyAsync(st, init.data(), init.size() * sizeof(int), cudaMemcpyHostToDevice, s));
      k_key_starts<<<(n + 255) / 256, 256, 0, s>>>(sk, n, p, st);
      k_key_starts<<<(n + 255) / 256, 256, 0, s>>>(rk, n, p, st + p + 1);
      CK(cudaGetLastError());
      std::vector<int> h(2 * (p + 1));
      CK(cudaMemcpyAsync(h.data(), st, h.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
      sync();
      for (int q = 0; q < p; ++q) {
        x.r4soff[q] = (size_t)h[q];
        x.r4scnt[q] = (size_t)(h[q + 1] - h[q]);
        x.r4roff[q] = (size_t)h[p + 1 + q];
        x.r4rcnt[q] = (size_t)(h[p + 2 + q] - h[p + 1 + q]);
      }
      x.r4ns = h[p];
      x.r4nr = h[2 * p + 1];
    });
  }
  // The partner values of this pass's R4 pairs, by the static routing
  void r4_exchange() {
    std::vector<Transport::Ata> plan;
    each([&](Slab &x) {
      if (x.r4ns) k_pack_u32<<<(x.r4ns + 255) / 256, 256, 0, s>>>(x.r4s, x.r4ns, x.gS, x.r4sbuf);
      Transport::Ata a;
      a.send = x.r4sbuf;
      a.recv = x.r4rbuf;
      a.soff = x.r4soff;
      a.scnt = x.r4scnt;
      a.roff = x.r4roff;
      a.rcnt = x.r4rcnt;
      plan.push_back(a);
    });
    CK(cudaGetLastError());
    T.alltoallv_u32(plan);
    each([&](Slab &x) {
      if (x.r4nr) k_unpack_u32<<<(x.r4nr + 255) / 256, 256, 0, s>>>(x.r4r, x.r4nr, x.r4rbuf, x.gS);
    });
    CK(cudaGetLastError());
  }

  // Gather every rank's keys (count in counter ci), sort identically on every
  // rank, keep the global ids (the same list everywhere).
  template <class GetKeys, class SetIds>
  void gather_sorted(int ci, GetKeys keys_of, SetIds set_ids, int &total) {
    std::vector<unsigned long long *> nb;
    each([&](Slab &x) {
      CK(cudaMemsetAsync(x.nrem, 0, 2 * p * 8, s));
      CK(cudaMemcpyAsync(x.nrem + x.rank, x.cnt + ci, 8, cudaMemcpyDeviceToDevice, s));
      nb.push_back(x.nrem);
    });
    T.allreduce_sum_u64(nb, p);
    std::vector<unsigned long long> counts(p);
    CK(cudaMemcpyAsync(counts.data(), sl[0].nrem, p * 8, cudaMemcpyDeviceToHost, s));
    sync();
    unsigned long long mx = 1;
    total = 0;
    for (int r = 0; r < p; ++r) {
      total += (int)counts[r];
      mx = std::max(mx, counts[r]);
    }
    std::vector<const void *> ks;
    std::vector<void *> ka;
    std::vector<uint64_t *> all;
    each([&](Slab &x) {
      uint64_t *pad = A.get<uint64_t>(mx);
      CK(cudaMemsetAsync(pad, 0xff, mx * 8, s));
      CK(cudaMemcpyAsync(pad, keys_of(x), counts[x.rank] * 8, cudaMemcpyDeviceToDevice, s));
      uint64_t *a = A.get<uint64_t>(mx * p);
      ks.push_back(pad);
      ka.push_back(a);
      all.push_back(a);
    });
    T.allgather(ks, ka, mx * 8);
    int l = 0;
    each([&](Slab &x) {
      uint64_t *sorted = A.get<uint64_t>(mx * p);
      int32_t *ids = A.get<int32_t>(std::max(total, 1));
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, all[l], sorted, (int)(mx * p), 0, 64, s));
      void *tmp = A.get<uint8_t>(tb);
      CK(cub::DeviceRadixSort::SortKeys(tmp, tb, all[l], sorted, (int)(mx * p), 0, 64, s));
      if (total) k_keys_to_ids<<<(total + 255) / 256, 256, 0, s>>>(sorted, ids, total);
      set_ids(x, ids);
      ++l;
    });
    CK(cudaGetLastError());
  }

  // (the gathered table changes exceed A / 2 per rank only under debug 0x800000)
  size_t x_alltupd_cap() const { return sl[0].alltupd_cap; }
  void grow_alltupd(size_t n) {
    each([&](Slab &x) {
      x.alltupd = A.get<int4>(n);
      x.alltupd_cap = n;
    });
  }

  Slabs slabs_of(const int2 *table, unsigned long long *err = nullptr) const {
    return Slabs{d_start, p, table, err, nz / p, nz % p};
  }

  // gather the boundary walk termini of every rank and resolve them
  void boundary_tables(bool from_ref) {
    for (int up = 0; up < 2; ++up) {
      std::vector<const void *> snd;
      std::vector<void *> rcv;
      const size_t P = (size_t)nx * ny;
      each([&](Slab &x) {
        int2 *mine = A.get<int2>(2 * P);
        const unsigned b = (unsigned)((2 * P + 255) / 256);
        const float *h = from_ref ? x.f : x.g;
        if (from_ref && up) k_boundary_walks<true, true><<<b, 256, 0, s>>>(h, x.slots, x.ref, x.G, mine);
        if (from_ref && !up) k_boundary_walks<false, true><<<b, 256, 0, s>>>(h, x.slots, x.ref, x.G, mine);
        if (!from_ref && up) k_boundary_walks<true, false><<<b, 256, 0, s>>>(h, x.slots, x.ref, x.G, mine);
        if (!from_ref && !up) k_boundary_walks<false, false><<<b, 256, 0, s>>>(h, x.slots, x.ref, x.G, mine);
        snd.push_back(mine);
        rcv.push_back(up ? x.tup : x.tdn);
      });
      CK(cudaGetLastError());
      T.allgather(snd, rcv, 2 * P * sizeof(int2));
      // no resolve pass: lookups follow the exit chains (table_lookup)
    }
  }

  template <bool SPLIT, bool FROM_REF>
  void events(Slab &x, const float *h, const int32_t *list, int n, int32_t *ext,
              const Track *tr = nullptr, bool fpass = false) {
    if (n <= 0) return;
    if (!FROM_REF && fpass && tr) {
      // a list pass with the clean-path test (exactz_correct's launch_events):
      // the saddles whose f-walk tiles are all clean take X_f; the rest (or
      // what the stamp check left, with the cache on) are walked
      const FPaths fp = SPLIT ? x.fpP : x.fpJ;
      int *ftodo = SPLIT ? x.ftodoP : x.ftodo, *nft = x.nftodo + (SPLIT ? 1 : 0);
      k_count_dirt<<<148, 256, 0, s>>>(fp.dirt, fp.nt, const_cast<unsigned long long *>(fp.ndirt));
      CK(cudaMemsetAsync(nft, 0, sizeof(int), s));
      const Slabs sb = slabs_of(SPLIT ? x.tup : x.tdn, x.cnt + C_CHANGED);
      if (cache_on) {
        const EvCache ec = SPLIT ? x.ecP : x.ecJ;
        int *todo = SPLIT ? x.todoP : x.todo, *ntodo = x.ntodo + (SPLIT ? 1 : 0);
        CK(cudaMemsetAsync(ntodo, 0, sizeof(int), s));
        k_events_check<SPLIT, true><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
            list, n, ec, *tr, x.marks, x.G, todo, ntodo, x.cnt, nullptr, nullptr, x.remote);
        k_fclean<SPLIT, true><<<148 * 4, 256, 0, s>>>(h, list, n, x.lm, x.ref, fp, ext, x.marks,
                                                      x.G, ftodo, nft, x.cnt, todo, ntodo, ec,
                                                      tr->round, fp.ndirt, fp.max_dirt, x.remote);
        k_events_cached<SPLIT, true><<<148 * 16, 256, 0, s>>>(
            h, list, ftodo, nft, x.slots, x.lm, ext, x.marks, x.G, ec, *tr, x.cnt, todo, ntodo, sb,
            x.remote);
        g_launches += 4;
      } else {
        k_fclean<SPLIT, true><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
            h, list, n, x.lm, x.ref, fp, ext, x.marks, x.G, ftodo, nft, x.cnt, nullptr, nullptr,
            EvCache{}, 0, fp.ndirt, fp.max_dirt, x.remote);
        // grids sized for every saddle (the list's length is on the device;
        // a grid-stride grid made the walks slower)
        if (n <= (1 << 19))
          k_events16<SPLIT, true><<<(unsigned)((16 * (int64_t)n + 255) / 256), 256, 0, s>>>(
              h, list, n, x.slots, x.lm, ext, x.marks, x.G, sb, x.remote, x.cnt, nullptr, ftodo,
              nft);
        else
          k_events<SPLIT, false, true><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
              h, list, n, x.slots, x.lm, x.ref, ext, x.marks, x.G, sb, x.remote, x.cnt, ftodo, nft);
        g_launches += 3;
      }
      CK(cudaGetLastError());
      return;
    }
    if (!FROM_REF && cache_on && tr) {
      // the stamp check re-emits the still valid results, the rest is walked
      // (k_events_cached, which caches what stays inside the slab)
      const EvCache ec = SPLIT ? x.ecP : x.ecJ;
      int *todo = SPLIT ? x.todoP : x.todo, *ntodo = x.ntodo + (SPLIT ? 1 : 0);
      CK(cudaMemsetAsync(ntodo, 0, sizeof(int), s));
      k_events_check<SPLIT, true><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
          list, n, ec, *tr, x.marks, x.G, todo, ntodo, x.cnt, nullptr, nullptr, x.remote);
      k_events_cached<SPLIT, true><<<148 * 16, 256, 0, s>>>(
          h, list, todo, ntodo, x.slots, x.lm, ext, x.marks, x.G, ec, *tr, x.cnt, nullptr,
          nullptr, slabs_of(SPLIT ? x.tup : x.tdn, x.cnt + C_CHANGED), x.remote);
      CK(cudaGetLastError());
      g_launches += 2;
      return;
    }
    // g walks: 16 lanes per saddle (k_events16; a slab holds 1/p of the
    // saddles, too few to hide a thread's walks in sequence)
    // (a slab with many saddles keeps k_events: its waves hide the walks and
    // 16 lanes per saddle issue more; A/B knob EXACTZ_SLAB_EV1: always k_events)
    // (debug 0x2000000: k_events)
    static const bool ev1 = std::getenv("EXACTZ_SLAB_EV1") != nullptr;
    if (!FROM_REF && !ev1 && !(flags & 0x2000000u) && n <= (1 << 19)) {
      k_events16<SPLIT, true><<<(unsigned)((16 * (int64_t)n + 255) / 256), 256, 0, s>>>(
          h, list, n, x.slots, x.lm, ext, x.marks, x.G,
          slabs_of(SPLIT ? x.tup : x.tdn, x.cnt + C_CHANGED), x.remote, x.cnt);
      CK(cudaGetLastError());
      g_launches++;
      return;
    }
    const int64_t threads = n;  // one lane per saddle
    k_events<SPLIT, FROM_REF, true><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
        h, list, n, x.slots, FROM_REF ? nullptr : x.lm, x.ref, ext, x.marks, x.G,
        slabs_of(SPLIT ? x.tup : x.tdn, x.cnt + C_CHANGED), x.remote,
        x.cnt);
    CK(cudaGetLastError());
  }

  // Labels of the final field (optional outputs): the boundary tables of its
  // slots (recomputed whole, whatever the passes kept), then per slab local
  // pointer jumping and the exits through the tables.  lo_out / hi_out: the
  // owned planes of label_min / label_max per local rank (nullptr: not wanted)
  void labels(const std::vector<int32_t *> &dn_out, const std::vector<int32_t *> &up_out) {
    boundary_tables(false);
    for (int up = 0; up < 2; ++up) {
      int l = 0;
      each([&](Slab &x) {
        int32_t *dst = (up ? up_out : dn_out)[l++];
        if (!dst) return;
        const int n = x.nzl * (int)x.plane();
        int32_t *lab = A.get<int32_t>((size_t)x.G.V);
        k_slab_ptrs<<<(n + 255) / 256, 256, 0, s>>>(x.slots, lab, x.G, up);
        for (int round = 0;; ++round) {
          if (round > 64) {
            set_err("labels", "pointer jumping did not converge");
            throw Error{EXACTZ_ECUDA};
          }
          CK(cudaMemsetAsync(x.cnt + C_CHANGED, 0, 8, s));
          k_jump_slab<<<blocks_for(n, 256), 256, 0, s>>>(lab, x.G, x.cnt + C_CHANGED);
          unsigned long long ch = 0;
          CK(cudaMemcpyAsync(&ch, x.cnt + C_CHANGED, 8, cudaMemcpyDeviceToHost, s));
          sync();
          if (!ch) break;
        }
        CK(cudaMemsetAsync(x.cnt + C_CHANGED, 0, 8, s));
        k_slab_resolve<<<(n + 255) / 256, 256, 0, s>>>(lab, x.G, slabs_of(up ? x.tup : x.tdn,
                                                                          x.cnt + C_CHANGED), dst);
        unsigned long long bad = 0;
        CK(cudaMemcpyAsync(&bad, x.cnt + C_CHANGED, 8, cudaMemcpyDeviceToHost, s));
        sync();
        if (bad) {
          set_err("labels", "an exit chain is longer than the table (a cycle)");
          throw Error{EXACTZ_ECUDA};
        }
      });
    }
    CK(cudaGetLastError());
  }

  // Sums counters [0, n) over the ranks.  Per pass only C_VT .. C_BAD_BOUND
  // are global; C_NREMOTE / C_WALK stay per rank.
  void allreduce_counters(int n = C_BAD_BOUND + 1) {
    std::vector<unsigned long long *> b;
    each([&](Slab &x) {
      k_fold_counters<<<1, 32, 0, s>>>(x.cnt);  // warp_add replicas first
      g_launches++;
      b.push_back(x.cnt);
    });
    T.allreduce_sum_u64(b, n);
  }

  // One CheckConstraints pass (+ edits): returns {V_t, applied, n1..n6}
  void round(bool do_edit, unsigned long long out[8]) {
    const bool c3 = !(flags & EXACTZ_NO_C3);
    zero_counters();
    const bool c2 = !(flags & EXACTZ_NO_C2) && nS > 1;
    ++rnd;
    if (cache_on && rnd >= 65000) cache_on = false;  // 16-bit stamps (as exactz_correct)
    const bool tracked = act_on || cache_on;  // the stencils / edit keep tracking state
    // the clean-path test in list passes (the list stencil flags the tiles
    // holding a pointer that is not f's; an unlisted vertex has f's pointers)
    const bool fpass = fp_on && act_on && ready && c3 && !reform;
    if (fpass)
      each([&](Slab &x) {
        CK(cudaMemsetAsync(x.dirtD, 0, 2 * (((size_t)x.nt + 15) / 16 * 16) + 16, s));
      });
    auto track = [&](Slab &x) {
      Track t{};
      t.round = rnd;
      t.tab_round = tab_round;
      if (fpass) {
        t.dirtD = x.dirtD;
        t.dirtU = x.dirtU;
        t.ntx = x.ntx;
        t.nty = x.nty;
      }
      if (act_on) {
        t.act_next = x.act[cur ^ 1];
        t.edited = pull ? x.edited : nullptr;
      }
      if (cache_on) {
        t.bval = x.bval;
        t.bslot = x.bslot;
        t.sbval = x.sbval;
        t.sbslot = x.sbslot;
        t.nbx = x.nbx;
        t.nby = x.nby;
        t.nbz = x.nbz;
        t.nsx = x.nsx;
        t.nsy = x.nsy;
      }
      if (c2) {  // the stencils keep the owned entries of gS (k_gs_diff lists the changes)
        t.posS = x.posS;
        t.gS = x.gS;
      }
      return t;
    };
    if (c2) each([&](Slab &x) { CK(cudaMemsetAsync(x.nrem + p, 0, p * 8, s)); });
    if (c3 && !reform) each([&](Slab &x) { CK(cudaMemsetAsync(x.nrem + 2 * p, 0, p * 8, s)); });
    if (act_on && ready) {  // list-based pass: fired | stars of the last pass's edits
      if (edited_valid) halo_edited();
      each([&](Slab &x) {
        CK(cudaMemsetAsync(x.nlist, 0, sizeof(int), s));
        k_act_list<<<148 * 16, 256, 0, s>>>(x.act[cur], edited_valid ? x.edited : nullptr, x.G,
                                            x.list, x.nlist);
        if (x.keyed)
          k_stencil_list_key<<<148 * 16, 256, 0, s>>>(x.g, x.ref, x.marks, x.slots, x.lm, x.list,
                                                       x.nlist, x.G, track(x), x.cnt);
        else
          k_stencil_list<<<148 * 16, 256, 0, s>>>(x.g, x.ref, x.marks, x.slots, x.lm, x.list,
                                                   x.nlist, x.G, track(x), x.cnt);
      });
    } else {
      each([&](Slab &x) {
        const Track t = track(x);
        const dim3 g2(x.sgrid.x, (unsigned)((ny + K2TY - 1) / K2TY), x.sgrid.z);
        if (x.keyed && tracked && x.tma)
          k_stencil_key2<true, true><<<g2, TX * K2W, 0, s>>>(x.g, x.ref, x.marks, x.slots, x.lm,
                                                             x.G, x.zc, t, x.cnt, x.tmap);
        else if (x.keyed && x.tma)
          k_stencil_key2<false, true><<<g2, TX * K2W, 0, s>>>(x.g, x.ref, x.marks, x.slots, x.lm,
                                                              x.G, x.zc, t, x.cnt, x.tmap);
        else if (x.keyed && tracked)
          k_stencil_key2<true, false><<<g2, TX * K2W, 0, s>>>(x.g, x.ref, x.marks, x.slots, x.lm,
                                                              x.G, x.zc, t, x.cnt, x.tmap);
        else if (x.keyed)
          k_stencil_key2<false, false><<<g2, TX * K2W, 0, s>>>(x.g, x.ref, x.marks, x.slots,
                                                               x.lm, x.G, x.zc, t, x.cnt, x.tmap);
        else if (x.fast && tracked)
          k_stencil_fast<true><<<x.sgrid, dim3(TX, TY), 0, s>>>(x.g, x.ref, x.marks, x.slots, x.lm,
                                                                 x.G, x.zc, t, x.cnt);
        else if (x.fast)
          k_stencil_fast<false><<<x.sgrid, dim3(TX, TY), 0, s>>>(x.g, x.ref, x.marks, x.slots,
                                                                 x.lm, x.G, x.zc, t, x.cnt);
        else if (tracked)
          k_stencil<true><<<x.sgrid, dim3(TX, TY), 0, s>>>(x.g, x.ref, x.marks, x.slots, x.lm,
                                                           x.G, x.zc, t, x.cnt);
        else
          k_stencil<false><<<x.sgrid, dim3(TX, TY), 0, s>>>(x.g, x.ref, x.marks, x.slots, x.lm,
                                                            x.G, x.zc, t, x.cnt);
      });
    }
    CK(cudaGetLastError());
    if (c3 && reform && nC > 1) {  // R7 on replicated critical-point values
      std::vector<uint32_t *> b;
      each([&](Slab &x) {
        k_fill_gS<<<(nC + 255) / 256, 256, 0, s>>>(x.g, x.CP, nC, x.gC, x.G);
        b.push_back(x.gC);
      });
      T.allreduce_max_u32(b, nC);
      each([&](Slab &x) {
        k_saddle_order_slab<<<(nC + 255) / 256, 256, 0, s>>>(x.gC, x.CP, nC, x.marks, x.G, x.cnt,
                                                            C_N1 + 4);
      });
      CK(cudaGetLastError());
    }
    const bool c3w = c3 && !reform;
    // the boundary tables serve walks that leave a slab, the exchanges other
    // replicas and other owners: none of them with one rank
    const bool tabs = c3w && p > 1;
    if (c2 && p > 1)
      each([&](Slab &x) {
        // a late list pass (the cache on: the lists are short) re-evaluated
        // only the listed vertices: only their saddles can have changed (an
        // early list holds up to a quarter of the slab, more than its saddles)
        if (act_on && ready && cache_on)
          k_gs_diff_list<<<148 * 8, 256, 0, s>>>(x.list, x.nlist, x.ref, x.posS, x.gS, x.gSprev,
                                                 x.upd, x.nrem + p + x.rank);
        else if (x.nown)
          k_gs_diff<<<(x.nown + 255) / 256, 256, 0, s>>>(x.own, x.nown, x.gS, x.gSprev, x.upd,
                                                         x.nrem + p + x.rank);
      });
    // the g boundary tables (C3 walks that leave a slab): this rank's entries
    // recomputed; after the first pass only the changed ones travel
    const size_t A2 = (size_t)nx * ny;
    if (tabs)
      each([&](Slab &x) {
        CK(cudaMemsetAsync(x.nrem + 2 * p + x.rank, 0, 8, s));
        const unsigned nb = (unsigned)((4 * A2 + 255) / 256);
        if (cache_on)
          k_boundary_delta<true><<<nb, 256, 0, s>>>(x.g, x.slots, x.G, x.rank, p, x.tdn, x.tupd,
                                                    x.nrem + 2 * p + x.rank, track(x), x.brnd,
                                                    x.bmask);
        else
          k_boundary_delta<false><<<nb, 256, 0, s>>>(x.g, x.slots, x.G, x.rank, p, x.tdn, x.tupd,
                                                     x.nrem + 2 * p + x.rank);
      });
    CK(cudaGetLastError());
    // exchange A (before C2 and the walks): nrem[p, 2p) = each rank's changed
    // gS entries (counted by the stencils), nrem[2p, 3p) = its changed table
    // entries; one count exchange sizes both sparse all-gathers
    if ((c2 || tabs) && p > 1) {
      std::vector<unsigned long long *> nb;
      each([&](Slab &x) { nb.push_back(x.nrem); });
      T.allreduce_sum_u64(nb, 3 * p);
      std::vector<unsigned long long> counts(3 * p);
      CK(cudaMemcpyAsync(counts.data(), sl[0].nrem, 3 * p * 8, cudaMemcpyDeviceToHost, s));
      sync();
      unsigned long long mu = 0, mt = 0;
      for (int r = 0; r < p; ++r) {
        mu = std::max(mu, counts[p + r]);
        mt = std::max(mt, counts[2 * p + r]);
      }
      // R4 needs only the partners' values: when the changes are many (the
      // dense passes), the static routing moves ~nS / p words per rank
      // instead of p x mu (position, value) pairs (the same decision on every
      // rank; debug 0x10000000: never, 0x20000000: always)
      const bool r4static = c2 && !(flags & 0x10000000u) &&
                            ((flags & 0x20000000u) ||
                             (unsigned long long)mu * p * p > (unsigned long long)nS);
      if (r4static) {
        r4_exchange();
      } else if (c2 && mu) {
        std::vector<const void *> snd;
        std::vector<void *> rcv;
        each([&](Slab &x) {  // pad to mu with position -1
          if (mu > counts[p + x.rank])
            CK(cudaMemsetAsync(x.upd + counts[p + x.rank], 0xff, (mu - counts[p + x.rank]) * 8, s));
          snd.push_back(x.upd);
          rcv.push_back(x.allupd);
        });
        T.allgather(snd, rcv, mu * 8);
        each([&](Slab &x) {
          const int n = (int)(mu * p);
          k_apply_gs<<<(n + 255) / 256, 256, 0, s>>>(x.allupd, n, x.gS);
        });
      }
      // (debug 0x800000: sparse after the first pass, whatever the count;
      // 0x1000000: whole chunks every pass)
      const bool full = !tables_ready || (flags & 0x1000000u) ||
                        (2 * mt > A2 && !(flags & 0x800000u));
      if (tabs && full) {
        // the first pass (or many changes): every rank's whole chunk, in place
        for (int up = 0; up < 2; ++up) {
          std::vector<const void *> snd;
          std::vector<void *> rcv;
          each([&](Slab &x) {
            int2 *t = up ? x.tup : x.tdn;
            snd.push_back(t + 2 * A2 * x.rank);
            rcv.push_back(t);
          });
          T.allgather(snd, rcv, 2 * A2 * sizeof(int2));
        }
        tables_ready = true;
        tab_round = rnd;
      } else if (tabs && mt) {
        tab_round = rnd;  // (cached walks that used the tables are stale)
        if (mt * p > x_alltupd_cap()) grow_alltupd(mt * p);
        std::vector<const void *> snd;
        std::vector<void *> rcv;
        each([&](Slab &x) {  // pad to mt with position -1
          const unsigned long long c = counts[2 * p + x.rank];
          if (mt > c) CK(cudaMemsetAsync(x.tupd + c, 0xff, (mt - c) * 16, s));
          snd.push_back(x.tupd);
          rcv.push_back(x.alltupd);
        });
        T.allgather(snd, rcv, mt * 16);
        each([&](Slab &x) {
          const int n = (int)(mt * p);
          k_apply_tab<<<(n + 255) / 256, 256, 0, s>>>(x.alltupd, n, x.tdn);
        });
      }
      CK(cudaGetLastError());
    }
    // C2 (R4) on the updated replicas, the owned pairs only
    if (c2)
      each([&](Slab &x) {
        if (x.nown)
          k_saddle_order_slab<<<(x.nown + 255) / 256, 256, 0, s>>>(x.gS, x.S, nS, x.marks, x.G,
                                                                   x.cnt, C_N1 + 3, x.own, x.nown);
      });
    if (c3w)
      each([&](Slab &x) {
        const Track t = track(x);
        events<false, false>(x, x.g, x.J, x.nJ, x.m1, &t, fpass);
        events<true, false>(x, x.g, x.P, x.nP, x.M1, &t, fpass);
      });
    CK(cudaGetLastError());
    // exchange B: the walks' targets owned by another rank (all-gathered)
    if (c3w && p > 1) {
      std::vector<unsigned long long *> nb;
      each([&](Slab &x) {
        CK(cudaMemsetAsync(x.nrem, 0, p * 8, s));
        CK(cudaMemcpyAsync(x.nrem + x.rank, x.cnt + C_NREMOTE, 8, cudaMemcpyDeviceToDevice, s));
        nb.push_back(x.nrem);
      });
      T.allreduce_sum_u64(nb, p);
      std::vector<unsigned long long> counts(p);
      CK(cudaMemcpyAsync(counts.data(), sl[0].nrem, p * 8, cudaMemcpyDeviceToHost, s));
      sync();
      unsigned long long mr = 0;
      for (int r = 0; r < p; ++r) mr = std::max(mr, counts[r]);
      if (mr) {
        std::vector<const void *> snd;
        std::vector<void *> rcv;
        each([&](Slab &x) {
          if (mr * p > x.allremote_cap) {
            x.allremote_cap = 2 * mr * p;
            x.allremote = A.get<int32_t>(x.allremote_cap);
          }
          if (mr > counts[x.rank])
            CK(cudaMemsetAsync(x.remote + counts[x.rank], 0xff, (mr - counts[x.rank]) * 4, s));
          snd.push_back(x.remote);
          rcv.push_back(x.allremote);
        });
        T.allgather(snd, rcv, mr * 4);
        each([&](Slab &x) {
          const int n = (int)(mr * p);
          k_apply_remote<<<(n + 255) / 256, 256, 0, s>>>(x.allremote, n, x.marks, x.G);
        });
      }
      CK(cudaGetLastError());
    }
    // marks in the ghost planes belong to the neighbours
    {
      std::vector<const void *> lo, hi;
      std::vector<void *> rlo, rhi;
      each([&](Slab &x) {
        const size_t W = x.words_per_plane();
        CK(cudaMemsetAsync(x.ghost_lo, 0, W * 4, s));
        CK(cudaMemsetAsync(x.ghost_hi, 0, W * 4, s));
        lo.push_back(x.marks);                          // local plane 0 -> rank-1
        hi.push_back(x.marks + (x.nzl + 1) * W);        // local plane nzl+1 -> rank+1
        rlo.push_back(x.ghost_lo);                      // from rank-1 (its top ghost)
        rhi.push_back(x.ghost_hi);                      // from rank+1 (its bottom ghost)
      });
      T.halo(lo, hi, rlo, rhi, sl[0].words_per_plane() * 4);
      each([&](Slab &x) {
        const int W = (int)x.words_per_plane();
        k_or_words<<<(W + 255) / 256, 256, 0, s>>>(x.marks + 1 * W, x.ghost_lo, W);
        k_or_words<<<(W + 255) / 256, 256, 0, s>>>(x.marks + x.nzl * W, x.ghost_hi, W);
        CK(cudaMemsetAsync(x.marks, 0, W * 4, s));
        CK(cudaMemsetAsync(x.marks + (x.nzl + 1) * W, 0, W * 4, s));
      });
      CK(cudaGetLastError());
    }
    each([&](Slab &x) {
      if (tracked) {
        if (act_on && pull)
          CK(cudaMemsetAsync(x.edited, 0, (size_t)x.G.nz * x.words_per_plane() * 4, s));
        k_count_edit<true><<<148 * 8, 256, 0, s>>>(x.g, x.c, x.marks, x.f, x.G, xi, delta, N,
                                                    do_edit ? 1 : 0, track(x), x.cnt);
      } else {
        k_count_edit<false><<<148 * 8, 256, 0, s>>>(x.g, x.c, x.marks, x.f, x.G, xi, delta, N,
                                                     do_edit ? 1 : 0, Track{}, x.cnt);
      }
    });
    CK(cudaGetLastError());
    if (act_on && !pull && p > 1) {
      // pushed stars that fall in a ghost plane belong to the neighbour's
      // boundary plane (as the marks above)
      std::vector<const void *> lo, hi;
      std::vector<void *> rlo, rhi;
      each([&](Slab &x) {
        const size_t W = x.words_per_plane();
        uint32_t *an = x.act[cur ^ 1];
        CK(cudaMemsetAsync(x.ghost_lo, 0, W * 4, s));
        CK(cudaMemsetAsync(x.ghost_hi, 0, W * 4, s));
        lo.push_back(an);
        hi.push_back(an + (x.nzl + 1) * W);
        rlo.push_back(x.ghost_lo);
        rhi.push_back(x.ghost_hi);
      });
      T.halo(lo, hi, rlo, rhi, sl[0].words_per_plane() * 4);
      each([&](Slab &x) {
        const int W = (int)x.words_per_plane();
        uint32_t *an = x.act[cur ^ 1];
        k_or_words<<<(W + 255) / 256, 256, 0, s>>>(an + 1 * W, x.ghost_lo, W);
        k_or_words<<<(W + 255) / 256, 256, 0, s>>>(an + x.nzl * W, x.ghost_hi, W);
        CK(cudaMemsetAsync(an, 0, W * 4, s));
        CK(cudaMemsetAsync(an + (x.nzl + 1) * W, 0, W * 4, s));
      });
      CK(cudaGetLastError());
    }
    if (act_on) {  // act_next (| stars of `edited`) is the next pass's set
      cur ^= 1;
      ready = true;
    }
    edited_valid = act_on && pull;
    allreduce_counters();
    read_counters();
    if (c3 && !reform && sl[0].hcnt[C_CHANGED]) {  // the boundary tables' verification round
      set_err("boundary_tables", "an exit chain is longer than the table (a cycle)");
      throw Error{EXACTZ_ECUDA};
    }
    for (int k = 0; k < 8; ++k) out[k] = sl[0].hcnt[k];
    halo_planes(false);  // the edited boundary planes refresh the neighbours' ghosts
    if (cache_on)        // ... and their changes stamp the ghost bricks (C3 cache)
      each([&](Slab &x) {
        k_ghost_stamp<<<(unsigned)((2 * x.plane() + 255) / 256), 256, 0, s>>>(x.g, x.ghost_prev,
                                                                              x.G, track(x));
      });
  }
};

static exactz_status sharded_impl(Transport &T, std::vector<const float *> f_in,
                                  std::vector<const float *> g_in, std::vector<float *> out,
                                  std::vector<uint8_t *> counts_out,
                                  std::vector<int32_t *> lmin_out, std::vector<int32_t *> lmax_out,
                                  const int64_t dims[3],
                                  float eps, uint32_t *iters, const exactz_opts *opts,
                                  cudaStream_t s) {
  int64_t V = 0;
  if (check_dims(dims, &V) != EXACTZ_OK || !iters) return EXACTZ_EINVAL;
  if (!std::isfinite(eps) || !(eps >= 0.0f)) return EXACTZ_EINVAL;
  int N = (opts && opts->N) ? (int)opts->N : 5;
  if (N < 1 || N > 254) return EXACTZ_EINVAL;
  if (dims[2] < T.nranks()) return EXACTZ_EINVAL;  // every rank owns >= 1 plane
  uint32_t flags = opts ? opts->flags : 0u;
  uint32_t max_iters = opts ? opts->max_iters : 0u;
  exactz_stats *stats = opts ? opts->stats : nullptr;
  Ctx::keep_pool();
  upload_luts(s);
  Arena A(s);
  std::vector<Slab> slabs(T.nlocal());
  struct HostFree {
    std::vector<Slab> &v;
    ~HostFree() {
      for (auto &x : v)
        if (x.hcnt) cudaFreeHost(x.hcnt);
    }
  } hf{slabs};
  ShardedRun R(T, s, A, slabs, (int)dims[0], (int)dims[1], (int)dims[2], eps, N, flags);
  R.setup(f_in, g_in);
  uint32_t it = 0, rows = 0;
  exactz_status st = EXACTZ_OK;
  unsigned long long prev_vt = (unsigned long long)V;
  for (;;) {
    const bool may_edit = !(max_iters && it >= max_iters);
    // vertex activity (list-based passes) once <= V/8 vertices are marked,
    // from the globally reduced V_t (the same decision on every rank)
    if (!(flags & EXACTZ_NO_TRACK) && !R.act_on && rows >= 1 && prev_vt * 8 <= (unsigned long long)V)
      R.start_act();
    // the C3 cache once the marks are sparse at brick scale (exactz_correct's
    // rule over the global brick grid; debug 0x200: off)
    {
      static const unsigned long long cache_div = [] {
        const char *e = std::getenv("EXACTZ_SLAB_CACHE_DIV");  // A/B knob (dev)
        if (!e) e = std::getenv("EXACTZ_CACHE_DIV");
        return e ? std::strtoull(e, nullptr, 10) : 4ull;
      }();
      const unsigned long long nbg = (unsigned long long)((dims[0] + BX - 1) / BX) *
                                     ((dims[1] + BY - 1) / BY) * ((dims[2] + BZ - 1) / BZ);
      if (!(flags & (EXACTZ_NO_TRACK | EXACTZ_REFORMULATED | 0x200u)) && !R.cache_on && rows >= 1 &&
          rows < 65000 && prev_vt * cache_div <= nbg)
        R.start_cache();
    }
    // (debug 0x40000000: always pull, the r02 behaviour before)
    R.pull = (flags & 0x40000000u) || prev_vt * 256 > (unsigned long long)V;
    unsigned long long o[8];
    R.round(may_edit, o);
    prev_vt = o[C_VT];
    if (stats && stats->rows && rows < stats->cap) {
      exactz_iter_stats &r = stats->rows[rows];
      r.violations = o[C_VT];
      r.applied = o[C_APPLIED];
      for (int k = 0; k < 6; ++k) r.n[k] = o[C_N1 + k];
      r.walk_steps = 0;
      r.evaluated = 0;
      r.links = 0;
      r.ms = 0.0;  // per-pass spans: single-GPU call only
    }
    ++rows;
    if (o[C_VT] == 0) break;
    if (!may_edit || o[C_APPLIED] == 0) {
      st = EXACTZ_ESTUCK;
      break;
    }
    ++it;
  }
  // labels of the final field: its slots are the last pass's (no edit followed)
  if (opts && (opts->label_min || opts->label_max)) R.labels(lmin_out, lmax_out);
  for (size_t l = 0; l < slabs.size(); ++l) {
    Slab &x = slabs[l];
    const size_t P = x.plane();
    CK(cudaMemcpyAsync(out[l], x.g + P, x.nzl * P * 4, cudaMemcpyDefault, s));
    if (counts_out.size() > l && counts_out[l])
      CK(cudaMemcpyAsync(counts_out[l], x.c + P, x.nzl * P, cudaMemcpyDefault, s));
  }
  CK(cudaStreamSynchronize(s));
  if (stats) stats->nrows = rows;
  *iters = it;
  return st;
}

}  // namespace exz

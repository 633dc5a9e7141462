// sharded.cuh — z-slab decomposition of the correction loop.
//
// Each rank owns the planes [z0, z0 + nzl) of the field and keeps one ghost
// plane on each side (local planes 0 and nzl + 1; NaN at the global faces).
// Per round (Alg. 1), bit-exact with the single-GPU call:
//   1. stencil R1-R3 on the owned planes (needs the ghost g planes);
//   2. C2 (R4) on the replicated saddle values gS: every rank fills the
//      entries it owns, a max-all-reduce over the uint32 bit patterns gives
//      every rank all values (exactly one non-zero contribution per entry);
//   3. C3 (R5/R6): label walks inside the slab; a path that leaves the slab
//      is completed from the gathered boundary table (§ k_boundary_walks);
//      targets owned by another rank travel in an all-gathered list;
//   4. marks that fall in a ghost plane go back to the owning neighbour;
//   5. the owners count and edit; the 8 round counters are all-reduced;
//   6. the new g boundary planes refresh the neighbours' ghost planes.
// The paper's distributed protocol exchanges ghost layers and
// uses "a consistent rule ... prioritizing smaller scalar modifications";
// here owners compute every edit and marks are ORed, so no tie rule is
// needed (amb-23) and the result equals the single-GPU result bit for bit.
//
// Transport: NCCL (one rank per process/GPU, exactz_correct_sharded) or a
// loopback that runs every rank of the decomposition in one process on one
// GPU (exactz_correct_slabs), used to test the decomposition on one device.
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
};

__global__ void k_sum_u64(unsigned long long *acc, const unsigned long long *src, int n) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) acc[k] += src[k];
}
__global__ void k_max_u32(uint32_t *acc, const uint32_t *src, size_t n) {
  size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (k < n) acc[k] = src[k] > acc[k] ? src[k] : acc[k];
}

struct LoopTransport : Transport {
  int p;
  cudaStream_t s;
  Arena &arena;
  LoopTransport(int p_, cudaStream_t s_, Arena &a) : p(p_), s(s_), arena(a) {}
  int nranks() const override { return p; }
  int nlocal() const override { return p; }
  int rank_of(int l) const override { return l; }
  void halo(const std::vector<const void *> &lo_send, const std::vector<const void *> &hi_send,
            const std::vector<void *> &lo_recv, const std::vector<void *> &hi_recv,
            size_t bytes) override {
    for (int r = 0; r < p; ++r) {
      if (r > 0) CK(cudaMemcpyAsync(hi_recv[r - 1], lo_send[r], bytes, cudaMemcpyDefault, s));
      if (r + 1 < p) CK(cudaMemcpyAsync(lo_recv[r + 1], hi_send[r], bytes, cudaMemcpyDefault, s));
    }
  }
  void allgather(const std::vector<const void *> &send, const std::vector<void *> &recv,
                 size_t bytes) override {
    for (int l = 0; l < p; ++l)
      for (int r = 0; r < p; ++r)
        CK(cudaMemcpyAsync((char *)recv[l] + r * bytes, send[r], bytes, cudaMemcpyDefault, s));
  }
  void allreduce_sum_u64(const std::vector<unsigned long long *> &buf, size_t n) override {
    for (int l = 1; l < p; ++l)
      k_sum_u64<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(buf[0], buf[l], (int)n);
    CK(cudaGetLastError());
    for (int l = 1; l < p; ++l) CK(cudaMemcpyAsync(buf[l], buf[0], n * 8, cudaMemcpyDefault, s));
  }
  void allreduce_max_u32(const std::vector<uint32_t *> &buf, size_t n) override {
    if (!n) return;
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
  bool fast = false;  // every owned lo >= 0: k_stencil_fast
  float *f = nullptr, *g = nullptr;
  uint32_t *ref = nullptr, *marks = nullptr, *ghost_lo = nullptr, *ghost_hi = nullptr;
  uint8_t *slots = nullptr, *c = nullptr;
  uint32_t *lm = nullptr;  // g-lower | g-upper << 16 link masks at the f-saddles (stencil -> C3 events)
  uint64_t *keys = nullptr, *allkeys = nullptr, *sorted = nullptr;
  int32_t *S = nullptr, *J = nullptr, *P = nullptr, *m1 = nullptr, *M1 = nullptr;
  int nJ = 0, nP = 0;
  int2 *tdn = nullptr, *tup = nullptr;  // gathered boundary tables (2 p A)
  uint32_t *gS = nullptr;
  uint64_t *cpkeys = nullptr;
  int32_t *CP = nullptr;  // reformulation: all critical points, replicated
  uint32_t *gC = nullptr;
  int32_t *remote = nullptr, *allremote = nullptr;
  // sparse exchange of the replicated gS: positions in S of the owned
  // saddles (local index), this round's changed entries, all ranks' lists
  int32_t *posS = nullptr;
  int2 *upd = nullptr, *allupd = nullptr;
  unsigned long long *cnt = nullptr, *hcnt = nullptr;  // device counters / host mirror
  unsigned long long *nrem = nullptr;                    // per-rank remote counts (p)
  // vertex activity (list-based passes, as exactz_correct): act[cur] = this
  // pass's set (owned planes), edited = the last pass's edits with the
  // neighbours' boundary planes in the ghost planes
  uint32_t *act[2] = {nullptr, nullptr}, *edited = nullptr;
  int32_t *list = nullptr;
  int *nlist = nullptr;
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
      x.zc = std::min(32, std::max(1, x.nzl));
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
      x.nrem = A.get<unsigned long long>(2 * p);
      x.keys = A.get<uint64_t>(x.nzl * P);
      if (reform) x.cpkeys = A.get<uint64_t>(x.nzl * P);
      x.tdn = A.get<int2>(2 * p * P);
      x.tup = A.get<int2>(2 * p * P);
      // owned planes from the caller; ghost planes NaN until the halo exchange
      CK(cudaMemsetAsync(x.f, 0xff, Vl * 4, s));
      CK(cudaMemsetAsync(x.g, 0xff, Vl * 4, s));
      CK(cudaMemcpyAsync(x.f + P, f_in[l], (size_t)x.nzl * P * 4, cudaMemcpyDefault, s));
      CK(cudaMemcpyAsync(x.g + P, g_in[l], (size_t)x.nzl * P * 4, cudaMemcpyDefault, s));
      CK(cudaMemsetAsync(x.c, 0, Vl, s));
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
    each([&](Slab &x) { x.fast = x.hcnt[C_NEG] == 0 && !(flags & 0x800u); });
    // O7 reference of f on the owned planes
    zero_counters();
    each([&](Slab &x) {
      unsigned bx = std::min(8u, (unsigned)((nx + 127) / 128));
      unsigned by = (unsigned)std::min<int64_t>((int64_t)x.nzl * ny, 148 * 16 / bx + 1);
      k_reference<<<dim3(bx, by), 128, 0, s>>>(x.f, x.G, x.ref, x.keys, x.cpkeys, x.cnt);
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
      CK(cudaMemcpyAsync(pad, x.keys, counts[x.rank] * 8, cudaMemcpyDeviceToDevice, s));
      x.allkeys = A.get<uint64_t>(slot * p);
      x.sorted = A.get<uint64_t>(slot * p);
      ks.push_back(pad);
      ka.push_back(x.allkeys);
    });
    T.allgather(ks, ka, slot * 8);
    each([&](Slab &x) {
      x.S = A.get<int32_t>(std::max(nS, 1));
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, x.allkeys, x.sorted, (int)(slot * p), 0, 64,
                                        s));
      void *tmp = A.get<uint8_t>(tb);
      CK(cub::DeviceRadixSort::SortKeys(tmp, tb, x.allkeys, x.sorted, (int)(slot * p), 0, 64, s));
      if (nS) k_keys_to_ids<<<(nS + 255) / 256, 256, 0, s>>>(x.sorted, x.S, nS);
      x.gS = A.get<uint32_t>(std::max(nS, 1));
      x.remote = A.get<int32_t>(std::max(nS, 1));
      x.posS = A.get<int32_t>(x.G.V);
      CK(cudaMemsetAsync(x.posS, 0xff, (size_t)x.G.V * 4, s));
      if (nS) k_local_pos<<<(nS + 255) / 256, 256, 0, s>>>(x.S, nS, x.posS, x.G);
      x.upd = A.get<int2>(slot);          // at most the owned saddles
      x.allupd = A.get<int2>(slot * p);
      // J, P: owned saddles in index order (global ids)
      const int lo = x.G.zb * (int)x.plane(), n = x.nzl * (int)x.plane();
      x.J = A.get<int32_t>(std::max<int64_t>(counts[x.rank], 1));
      x.P = A.get<int32_t>(std::max<int64_t>(counts[x.rank], 1));
      int *nsel = A.get<int>(2);
      cub::CountingInputIterator<int32_t> ids(lo);
      size_t t2 = 0, t3 = 0;
      CK(cub::DeviceSelect::If(nullptr, t2, ids, x.J, nsel, n, IsJoin{x.ref}, s));
      CK(cub::DeviceSelect::If(nullptr, t3, ids, x.P, nsel + 1, n, IsSplit{x.ref}, s));
      void *tmp2 = A.get<uint8_t>(std::max(t2, t3));
      CK(cub::DeviceSelect::If(tmp2, t2, ids, x.J, nsel, n, IsJoin{x.ref}, s));
      CK(cub::DeviceSelect::If(tmp2, t3, ids, x.P, nsel + 1, n, IsSplit{x.ref}, s));
      int h[2];
      CK(cudaMemcpyAsync(h, nsel, sizeof(h), cudaMemcpyDeviceToHost, s));
      sync();
      x.nJ = h[0];
      x.nP = h[1];
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

  Slabs slabs_of(const int2 *table, unsigned long long *err = nullptr) const {
    return Slabs{d_start, p, table, err};
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
  void events(Slab &x, const float *h, const int32_t *list, int n, int32_t *ext) {
    if (n <= 0) return;
    const int64_t threads = n;  // one lane per saddle
    k_events<SPLIT, FROM_REF, true><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
        h, list, n, x.slots, FROM_REF ? nullptr : x.lm, x.ref, ext, x.marks, x.G,
        slabs_of(SPLIT ? x.tup : x.tdn, x.cnt + C_CHANGED), x.remote,
        x.cnt);
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
    auto track = [&](Slab &x) {
      Track t{};
      if (act_on) {
        t.act_next = x.act[cur ^ 1];
        t.edited = x.edited;
      }
      if (c2) {  // the stencils keep the owned entries of gS and list the changes
        t.posS = x.posS;
        t.gS = x.gS;
        t.gsupd = x.upd;
        t.ngsupd = x.nrem + p + x.rank;
      }
      return t;
    };
    if (c2) each([&](Slab &x) { CK(cudaMemsetAsync(x.nrem + p, 0, p * 8, s)); });
    if (act_on && ready) {  // list-based pass: fired | stars of the last pass's edits
      halo_edited();
      each([&](Slab &x) {
        CK(cudaMemsetAsync(x.nlist, 0, sizeof(int), s));
        k_act_list<<<148 * 16, 256, 0, s>>>(x.act[cur], x.edited, x.G, x.list, x.nlist);
        k_stencil_list<<<148 * 16, 256, 0, s>>>(x.g, x.ref, x.marks, x.slots, x.lm, x.list,
                                                 x.nlist, x.G, track(x), x.cnt);
      });
    } else {
      each([&](Slab &x) {
        const Track t = track(x);
        if (x.fast && act_on)
          k_stencil_fast<true><<<x.sgrid, dim3(TX, TY), 0, s>>>(x.g, x.ref, x.marks, x.slots, x.lm,
                                                                 x.G, x.zc, t, x.cnt);
        else if (x.fast)
          k_stencil_fast<false><<<x.sgrid, dim3(TX, TY), 0, s>>>(x.g, x.ref, x.marks, x.slots,
                                                                 x.lm, x.G, x.zc, t, x.cnt);
        else if (act_on)
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
    } else if (c3 && !reform) {
      boundary_tables(false);
      each([&](Slab &x) {
        events<false, false>(x, x.g, x.J, x.nJ, x.m1);
        events<true, false>(x, x.g, x.P, x.nP, x.M1);
      });
    }
    // one count exchange for the two sparse all-gathers of the round:
    // nrem[0, p) = each rank's remote C3 targets, nrem[p, 2p) = each rank's
    // changed gS entries (counted by the stencils); then C2 (R4) on the
    // updated replicas and the owners' remote marks
    const bool c3w = c3 && !reform;
    if (c2 || c3w) {
      std::vector<unsigned long long *> nb;
      each([&](Slab &x) {
        CK(cudaMemsetAsync(x.nrem, 0, p * 8, s));
        if (c3w)
          CK(cudaMemcpyAsync(x.nrem + x.rank, x.cnt + C_NREMOTE, 8, cudaMemcpyDeviceToDevice, s));
        nb.push_back(x.nrem);
      });
      T.allreduce_sum_u64(nb, 2 * p);
      std::vector<unsigned long long> counts(2 * p);
      CK(cudaMemcpyAsync(counts.data(), sl[0].nrem, 2 * p * 8, cudaMemcpyDeviceToHost, s));
      sync();
      unsigned long long mr = 0, mu = 0;
      for (int r = 0; r < p; ++r) {
        mr = std::max(mr, counts[r]);
        mu = std::max(mu, counts[p + r]);
      }
      if (c2 && mu) {
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
      if (c2)
        each([&](Slab &x) {
          k_saddle_order_slab<<<(nS + 255) / 256, 256, 0, s>>>(x.gS, x.S, nS, x.marks, x.G, x.cnt);
        });
      if (c3w && mr) {
        std::vector<const void *> snd;
        std::vector<void *> rcv;
        each([&](Slab &x) {
          int32_t *pad = A.get<int32_t>(mr);
          CK(cudaMemsetAsync(pad, 0xff, mr * 4, s));  // -1: no vertex
          CK(cudaMemcpyAsync(pad, x.remote, counts[x.rank] * 4, cudaMemcpyDeviceToDevice, s));
          x.allremote = A.get<int32_t>(mr * p);
          snd.push_back(pad);
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
      if (act_on) {
        CK(cudaMemsetAsync(x.edited, 0, (size_t)x.G.nz * x.words_per_plane() * 4, s));
        k_count_edit<true><<<148 * 8, 256, 0, s>>>(x.g, x.c, x.marks, x.f, x.G, xi, delta, N,
                                                    do_edit ? 1 : 0, track(x), x.cnt);
      } else {
        k_count_edit<false><<<148 * 8, 256, 0, s>>>(x.g, x.c, x.marks, x.f, x.G, xi, delta, N,
                                                     do_edit ? 1 : 0, Track{}, x.cnt);
      }
    });
    CK(cudaGetLastError());
    if (act_on) {  // act_next (| stars of `edited`) is the next pass's set
      cur ^= 1;
      ready = true;
    }
    allreduce_counters();
    read_counters();
    if (c3 && !reform && sl[0].hcnt[C_CHANGED]) {  // the boundary tables' verification round
      set_err("boundary_tables", "an exit chain is longer than the table (a cycle)");
      throw Error{EXACTZ_ECUDA};
    }
    for (int k = 0; k < 8; ++k) out[k] = sl[0].hcnt[k];
    halo_planes(false);  // the edited boundary planes refresh the neighbours' ghosts
  }
};

static exactz_status sharded_impl(Transport &T, std::vector<const float *> f_in,
                                  std::vector<const float *> g_in, std::vector<float *> out,
                                  std::vector<uint8_t *> counts_out, const int64_t dims[3],
                                  float eps, uint32_t *iters, const exactz_opts *opts,
                                  cudaStream_t s) {
  int64_t V = 0;
  if (check_dims(dims, &V) != EXACTZ_OK || !iters) return EXACTZ_EINVAL;
  if (!std::isfinite(eps) || !(eps >= 0.0f)) return EXACTZ_EINVAL;
  int N = (opts && opts->N) ? (int)opts->N : 5;
  if (N < 1 || N > 254) return EXACTZ_EINVAL;
  if (opts && (opts->label_min || opts->label_max)) {
    set_err("exactz_correct_sharded", "label outputs are not supported by the sharded path");
    return EXACTZ_EUNSUPPORTED;
  }
  if (dims[2] < T.nranks()) return EXACTZ_EINVAL;  // every rank owns >= 1 plane
  uint32_t flags = opts ? opts->flags : 0u;
  uint32_t max_iters = opts ? opts->max_iters : 0u;
  exactz_stats *stats = opts ? opts->stats : nullptr;
  Ctx::keep_pool();
  {
    static thread_local uint8_t lut[1 << kSlots];
    static thread_local bool ready = false;
    if (!ready) {
      for (uint32_t m = 0; m < (1u << kSlots); ++m) lut[m] = (uint8_t)link_components_t(m, kLink.adj);
      ready = true;
    }
    CK(cudaMemcpyToSymbolAsync(d_comp, lut, sizeof(lut), 0, cudaMemcpyHostToDevice, s));
  }
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

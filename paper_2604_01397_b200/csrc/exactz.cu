// exactz.cu — C ABI (include/exactz.h) and host orchestration of the B200
// EXaCTz correction loop.  Alg. 1:
//   validate (O1) -> reference of f (O7) -> loop { CheckConstraints (O8);
//   if no violation: stop; ApplyBoundedEdits (O9) }.
// All scratch lives in device memory allocated on the caller's stream; the
// host reads back 16 counters per round (termination, stats).
#include <cuda.h>  // CUtensorMap (TMA descriptors; the driver entry point is fetched at run time)
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cub/device/device_merge.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <algorithm>
#include <dlfcn.h>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/exactz.h"
#include "kernels.cuh"
#include "stencil_fast.cuh"
#include "stencil_key.cuh"
#include "vulnerability.cuh"
#include "editlog.cuh"

#ifndef EXACTZ_GIT
#define EXACTZ_GIT "dev"
#endif

namespace exz {

static thread_local std::string g_last_error;

struct Error {
  exactz_status st;
};

static void set_err(const char *what, const char *detail) {
  g_last_error = std::string(what) + ": " + (detail ? detail : "");
}

#define CK(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      set_err(#call, cudaGetErrorString(e_));                                     \
      throw Error{e_ == cudaErrorMemoryAllocation ? EXACTZ_ENOMEM : EXACTZ_ECUDA}; \
    }                                                                             \
  } while (0)

// Device allocations tied to one call; freed (stream-ordered) on scope exit.
class Arena {
 public:
  explicit Arena(cudaStream_t s) : s_(s) {}
  ~Arena() {
    for (void *p : ptrs_) cudaFreeAsync(p, s_);
  }
  template <class T>
  T *get(size_t n) {
    void *p = nullptr;
    CK(cudaMallocAsync(&p, (n ? n : 1) * sizeof(T), s_));
    ptrs_.push_back(p);
    return static_cast<T *>(p);
  }

 private:
  cudaStream_t s_;
  std::vector<void *> ptrs_;
};

static int blocks_for(int64_t n, int threads, int cap = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

static std::atomic<uint64_t> g_launches{0};

// Per-kernel-class CUDA-event timing (EXACTZ_PROFILE).  Events are recorded
// on the launch stream around each kernel and read at the next host sync.
struct Prof {
  bool on = false;
  struct Rec {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<cudaEvent_t> pool;
  std::vector<Rec> pending;
  double ms[EXACTZ_K_CLASSES] = {};
  uint64_t launches[EXACTZ_K_CLASSES] = {}, bytes[EXACTZ_K_CLASSES] = {};
  ~Prof() {
    for (auto &r : pending) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
  }
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  void drain() {  // call after a stream sync
    for (auto &r : pending) {
      float t = 0;
      CK(cudaEventElapsedTime(&t, r.a, r.b));
      ms[r.cls] += t;
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    pending.clear();
  }
};

// Per-thread, per-device resources a call needs but should not create each
// time (cudaHostAlloc, stream and event creation cost milliseconds per call
// in the timed steps): the mapped counter mirror, the two side streams and
// their fork/join events.  A Ctx borrows the kit when it is free (one call
// at a time per thread) and otherwise makes its own.
struct Kit {
  int dev = -1;
  bool busy = false;
  unsigned long long *hcnt = nullptr;
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaEvent_t fj[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t fev[2] = {nullptr, nullptr};
};
static thread_local Kit g_kit;

// The component LUTs of the stencils (d_comp: components of a link mask;
// d_comp2: nlc | nuc << 3 of an interior vertex), built once per thread.
static void upload_luts(cudaStream_t s) {
  static thread_local uint8_t lut[1 << kSlots];
  static thread_local uint8_t lut2[1 << kSlots];
  static thread_local bool ready = false;
  if (!ready) {
    for (uint32_t m = 0; m < (1u << kSlots); ++m) lut[m] = (uint8_t)link_components_t(m, kLink.adj);
    for (uint32_t m = 0; m < (1u << kSlots); ++m)
      lut2[m] = (uint8_t)(lut[m] | (lut[~m & ((1u << kSlots) - 1)] << 3));
    ready = true;
  }
  CK(cudaMemcpyToSymbolAsync(d_comp, lut, sizeof(lut), 0, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyToSymbolAsync(d_comp2, lut2, sizeof(lut2), 0, cudaMemcpyHostToDevice, s));
}

// TMA descriptor of a float32 field the dense key stencil reads
// (k_stencil_key2): 3D {nx, ny, nz}, box {40, 18, 1} from x0 - 4 (the 34 x 18
// halo tile, 16-byte aligned in x), zero fill outside the domain.  False when
// the field does not qualify (nx % 4, alignment) or the driver call fails.
static bool encode_plane_map(CUtensorMap *m, const void *g, int nx, int ny, int nz) {
  if (nx % 4 != 0 || ((uintptr_t)g & 15)) return false;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }();
  if (!encode) return false;
  const cuuint64_t dim[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
  const cuuint64_t stride[2] = {(cuuint64_t)nx * 4, (cuuint64_t)nx * ny * 4};
  const cuuint32_t box[3] = {(cuuint32_t)K2Stage<true>::SXS, (cuuint32_t)K2SY, 1},
                   estr[3] = {1, 1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void *>(g), dim, stride, box,
                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct Ctx {
  cudaStream_t s;
  bool kit = false;  // borrowing g_kit
  Prof prof;
  // Launch one kernel (or library call) of class `cls`; `ours` counts it as
  // one of this library's kernels.
  template <class Fn>
  void run(int cls, uint64_t bytes, bool ours, Fn fn) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (prof.on) {
      a = prof.get();
      CK(cudaEventRecord(a, s));
    }
    fn();
    CK(cudaGetLastError());
    if (prof.on) {
      b = prof.get();
      CK(cudaEventRecord(b, s));
      prof.pending.push_back({cls, a, b});
    }
    if (ours) {
      prof.launches[cls]++;
      g_launches++;
    }
    prof.bytes[cls] += bytes;
  }
  GridP G{};
  int64_t V = 0;
  dim3 sgrid, sblock;                 // stencil: 32x8 columns, z chunks
  dim3 rgrid, vblock;                 // persistent row-parallel grid, 128 x-threads
  int zc = 1;
  uint32_t dbg = 0;                   // the call's flags (debug variants of kernels)
  bool fast = false;                  // every lo >= 0: k_stencil_fast (set by validation)
  bool keyed = false;                 // value range fits exact SoS keys: k_stencil_key
  // TMA descriptor of the field the dense stencil reads (k_stencil_key2):
  // 3D {nx, ny, nz} float32, box {40, 18, 1} from x0 - 4 (the 34 x 18 halo
  // tile, 16-byte aligned in x), zero fill outside the domain
  CUtensorMap tmap{};
  const void *tmap_ptr = nullptr;
  bool plane_map(const void *g) {
    if (g == tmap_ptr) return true;
    if (G.zoff != 0 || !encode_plane_map(&tmap, g, G.nx, G.ny, G.nz)) return false;
    tmap_ptr = g;
    return true;
  }
  unsigned long long *cnt = nullptr;  // device counters
  unsigned long long *hcnt = nullptr; // pinned, mapped host mirror
  unsigned long long *hcnt_dev = nullptr;  // its device alias
  Arena arena;
  explicit Ctx(cudaStream_t st) : s(st), arena(st) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    if (!g_kit.busy) {
      if (g_kit.dev != dev) g_kit = Kit{};  // another device's handles are left to the driver
      g_kit.dev = dev;
      g_kit.busy = true;
      kit = true;
      hcnt = g_kit.hcnt;
      for (int k = 0; k < 2; ++k) side[k] = g_kit.side[k];
      for (int k = 0; k < 3; ++k) fj[k] = g_kit.fj[k];
      for (int k = 0; k < 2; ++k) fev[k] = g_kit.fev[k];
    }
  }
  ~Ctx() {
    if (kit) {  // hand the (possibly just created) handles back
      g_kit.hcnt = hcnt;
      for (int k = 0; k < 2; ++k) g_kit.side[k] = side[k];
      for (int k = 0; k < 3; ++k) g_kit.fj[k] = fj[k];
      for (int k = 0; k < 2; ++k) g_kit.fev[k] = fev[k];
      g_kit.busy = false;
      return;
    }
    if (hcnt) cudaFreeHost(hcnt);
    for (int k = 0; k < 2; ++k)
      if (side[k]) cudaStreamDestroy(side[k]);
    for (int k = 0; k < 3; ++k)
      if (fj[k]) cudaEventDestroy(fj[k]);
    for (int k = 0; k < 2; ++k)
      if (fev[k]) cudaEventDestroy(fev[k]);
  }
  // fork/join of two side streams (independent kernels of one pass)
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaEvent_t fj[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t fev[2] = {nullptr, nullptr};  // fold of counter buffer 0 / 1 done
  cudaStream_t main_s = nullptr;
  void fork() {
    if (!side[0]) {
      // side streams at the highest priority: their short, latency-bound
      // kernels (C2 during the stencil) get SMs as soon as stencil CTAs retire
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      static const bool noprio = std::getenv("EXACTZ_NO_PRIO") != nullptr;  // diagnostic
      for (int k = 0; k < 2; ++k)
        CK(cudaStreamCreateWithPriority(&side[k], cudaStreamNonBlocking, noprio ? lo : hi));
      for (int k = 0; k < 3; ++k) CK(cudaEventCreateWithFlags(&fj[k], cudaEventDisableTiming));
    }
    main_s = s;
    CK(cudaEventRecord(fj[0], s));
    for (int k = 0; k < 2; ++k) CK(cudaStreamWaitEvent(side[k], fj[0], 0));
  }
  void on_side(int k) {
    static const bool serial = std::getenv("EXACTZ_SERIAL") != nullptr;  // diagnostic
    s = serial ? main_s : side[k];
  }
  void join() {
    for (int k = 0; k < 2; ++k) {
      CK(cudaEventRecord(fj[1 + k], side[k]));
      CK(cudaStreamWaitEvent(main_s, fj[1 + k], 0));
    }
    s = main_s;
  }
  void init(const int64_t dims[3]) {
    keep_pool();
    G.nx = (int)dims[0];
    G.ny = (int)dims[1];
    G.nz = (int)dims[2];
    G.V = (int)V;
    G.W = (G.nx + 31) / 32;
    grid_fastdiv(G);
    for (int s = 0; s < kSlots; ++s)
      G.delta[s] = kOff[s][0] + G.nx * (kOff[s][1] + G.ny * kOff[s][2]);
    G.zoff = 0;
    G.gnz = G.nz;
    G.zb = 0;
    G.ze = G.nz;
    // z chunk per stencil CTA: enough CTAs to fill 148 SMs several times over,
    // few enough halo planes (2 per chunk) to keep re-reads small
    int64_t cols = (int64_t)((G.nx + TX - 1) / TX) * ((G.ny + TY - 1) / TY);
    int64_t want = 148 * 24;
    int64_t z = cols >= want ? G.nz : (G.nz * cols + want - 1) / want;
    zc = (int)(z < 8 ? 8 : (z > 64 ? 64 : z));
    static const int zc_env = [] {  // tuning knob (dev)
      const char *e = std::getenv("EXACTZ_ZC");
      return e ? std::atoi(e) : 0;
    }();
    if (zc_env > 0) zc = zc_env;
    if (zc > G.nz) zc = G.nz;
    sblock = dim3(TX, TY, 1);
    sgrid = dim3((unsigned)((G.nx + TX - 1) / TX), (unsigned)((G.ny + TY - 1) / TY),
                 (unsigned)((G.nz + zc - 1) / zc));
    vblock = dim3(128, 1, 1);
    {
      unsigned bx = (unsigned)((G.nx + 127) / 128);
      if (bx > 8) bx = 8;
      int64_t rows = (int64_t)G.ny * G.nz, by = (148 * 16 + bx - 1) / bx;
      rgrid = dim3(bx, (unsigned)(rows < by ? rows : by), 1);
    }
    cnt = arena.get<unsigned long long>(C_NALLOC);
    // mapped: the fold kernel writes the counters straight into host memory,
    // so a pass's read needs no copy-engine transfer (a bulk D2H of the
    // result on a side stream would otherwise queue every pass behind it)
    // two buffers: a pass's counters are read while the next pass runs
    if (!hcnt)
      CK(cudaHostAlloc((void **)&hcnt, 2 * C_NCOUNTERS * sizeof(unsigned long long),
                       cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer((void **)&hcnt_dev, hcnt, 0));
    upload_lut();
  }
  // Keep freed stream-ordered memory in the device's default pool between
  // calls (the default release threshold 0 returns it to the OS at every
  // sync, making each call re-map its scratch).
  static void keep_pool() {  // also used by the sharded path
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  void upload_lut() { upload_luts(s); }
  size_t mark_words() const { return (size_t)G.ny * G.nz * G.W; }
  void zero() { CK(cudaMemsetAsync(cnt, 0, C_NALLOC * sizeof(unsigned long long), s)); }
  void read() {
    // warp_add replicas -> cnt[0 .. C_NCOUNTERS), mirrored into hcnt
    k_fold_counters<<<1, 32, 0, s>>>(cnt, hcnt_dev);
    g_launches++;
    CK(cudaStreamSynchronize(s));
    if (prof.on) prof.drain();
  }
  // Asynchronous counter read of a pass: fold into mapped buffer `buf` and
  // record its event; counters(buf) waits for that event only, so the host can
  // enqueue the next pass before this one has finished.
  void fold(int buf) {
    if (!fev[buf]) CK(cudaEventCreateWithFlags(&fev[buf], cudaEventDisableTiming));
    k_fold_counters<<<1, 32, 0, s>>>(cnt, hcnt_dev + (size_t)buf * C_NCOUNTERS);
    g_launches++;
    CK(cudaGetLastError());
    CK(cudaEventRecord(fev[buf], s));
  }
  const unsigned long long *counters(int buf) {
    CK(cudaEventSynchronize(fev[buf]));
    return hcnt + (size_t)buf * C_NCOUNTERS;
  }
};

static exactz_status check_dims(const int64_t dims[3], int64_t *V) {
  if (!dims) return EXACTZ_EINVAL;
  for (int k = 0; k < 3; ++k)
    if (dims[k] < 1 || dims[k] > (1 << 30)) return EXACTZ_EINVAL;
  int64_t v = dims[0] * dims[1] * dims[2];
  if (v >= ((int64_t)1 << 31)) return EXACTZ_EINVAL;
  if (dims[1] > 65535 || dims[2] > 65535) return EXACTZ_EINVAL;  // launch grid limits
  *V = v;
  return EXACTZ_OK;
}

// Resolve pointer forests to their roots (O6) by pointer jumping; only for the
// optional full label outputs.
static void full_labels(Ctx &C, const uint8_t *slots, int32_t *lab_dn, int32_t *lab_up) {
  C.run(EXACTZ_K_LABELS, 9 * (uint64_t)C.V, true, [&] {
    k_slots_to_ptrs<<<blocks_for(C.V, 256, 1 << 30), 256, 0, C.s>>>(slots, lab_dn, lab_up, C.G);
  });
  for (int32_t *lab : {lab_dn, lab_up}) {
    if (!lab) continue;
    for (int round = 0;; ++round) {
      if (round > 64) {
        set_err("full_labels", "pointer jumping did not converge");
        throw Error{EXACTZ_ECUDA};
      }
      CK(cudaMemsetAsync(&C.cnt[C_CHANGED], 0, sizeof(unsigned long long), C.s));
      C.run(EXACTZ_K_LABELS, 8 * (uint64_t)C.V, true, [&] {
        k_jump<<<blocks_for(C.V, 256), 256, 0, C.s>>>(lab, C.V, C.cnt);
      });
      unsigned long long ch = 0;
      CK(cudaMemcpyAsync(&ch, &C.cnt[C_CHANGED], sizeof(ch), cudaMemcpyDeviceToHost, C.s));
      CK(cudaStreamSynchronize(C.s));
      if (C.prof.on) C.prof.drain();
      if (!ch) break;
    }
  }
}

struct Reference {
  uint32_t *ref = nullptr;
  int32_t *S = nullptr, *J = nullptr, *P = nullptr, *m1 = nullptr, *M1 = nullptr;
  int nS = 0, nJ = 0, nP = 0;
  int32_t *CP = nullptr;  // reformulation: all critical points sorted by (f, idx)
  int nC = 0;
  int32_t *posS = nullptr;  // [V]: position in S of each f-saddle (other entries unused)
  uint32_t *gS = nullptr;   // [nS]: g at S[k] (value bits), written by the stencils
  uint32_t *lmS = nullptr;  // [nS]: g link masks of S[k], written by the stencils
  uint8_t *fslots = nullptr;  // [V]: dn_f | up_f << 4 (k_fpaths; nullptr: not built)
  int32_t *Jpos = nullptr, *Ppos = nullptr;  // [nJ] / [nP]: positions in S of J[k] / P[k]
};

// Sort 64-bit SoS keys (ordered(f) << 32 | idx) and keep the indices.
static void sort_ids(Ctx &C, uint64_t *keys, int n, int32_t *ids) {
  if (n <= 0) return;
  uint64_t *sorted = C.arena.get<uint64_t>(n);
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, n, 0, 64, C.s));
  void *tmp = C.arena.get<uint8_t>(tb);
  C.run(EXACTZ_K_REFERENCE, 32ull * n, false, [&] {
    CK(cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, n, 0, 64, C.s));
  });
  C.run(EXACTZ_K_REFERENCE, 12ull * n, true, [&] {
    k_keys_to_ids<<<blocks_for(n, 256, 1 << 30), 256, 0, C.s>>>(sorted, ids, n);
  });
}

// k_fclean over all n saddles (one per thread) or over an idx list (a small
// grid-stride grid: the list is short in late passes)
template <bool SPLIT>
static void launch_fclean(Ctx &C, const float *h, const int32_t *sl, int n, const uint32_t *lm,
                          const uint32_t *ref, const FPaths &fp, const int32_t *ext,
                          uint32_t *marks, int *out, int *nout, const int *idx, const int *nidx,
                          EvCache ec, int round) {
  const unsigned grid = idx ? 148u * 4u : (unsigned)((n + 255) / 256);
  k_fclean<SPLIT><<<grid, 256, 0, C.s>>>(h, sl, n, lm, ref, fp, ext, marks, C.G, out, nout,
                                         C.cnt, idx, nidx, ec, round, fp.ndirt, fp.max_dirt);
}

// The C3 walks of one saddle list.  fp.off (tracking, list passes): the
// clean-path test first (k_fclean), only the saddles it leaves (ftodo) go on;
// ec.rnd: the brick-stamp cache (k_events_check), then the walks of what is
// left (k_events_cached); else every saddle is walked (k_events).
template <bool SPLIT, bool FROM_REF>
static void launch_events(Ctx &C, const float *h, const int32_t *sl, int n, const uint8_t *slots,
                          const uint32_t *lm, const uint32_t *ref, int32_t *ext, uint32_t *marks,
                          EvCache ec = EvCache{}, Track tr = Track{}, int *todo = nullptr,
                          int *ntodo = nullptr, FPaths fp = FPaths{}, int *ftodo = nullptr,
                          int *nftodo = nullptr, const int32_t *lpos = nullptr,
                          bool dense = false) {
  ec.lpos = lpos;
  fp.lpos = lpos;
  if (n <= 0) return;
  const int64_t threads = n;  // one lane per saddle
  // algorithmic bytes: 8 per saddle (id, m1 / M1) here, 8 per
  // link vertex walked from (its label and the label's value) added after
  // the pass from the C_LINKS count
  const int cls = FROM_REF ? EXACTZ_K_REFERENCE : EXACTZ_K_EVENTS;
  const int *idx = nullptr, *nidx = nullptr;
  if (!FROM_REF && fp.off)  // this list's dirty tiles (k_fclean's gate), on its stream
    C.run(cls, 0, true, [&] {
      k_count_dirt<<<148, 256, 0, C.s>>>(fp.dirt, fp.nt, const_cast<unsigned long long *>(fp.ndirt));
    });
  if (!FROM_REF && fp.off && !ec.rnd) {
    CK(cudaMemsetAsync(nftodo, 0, sizeof(int), C.s));
    // bytes: id, lm, ref word, offsets (16 B per saddle); the tile entries
    // and their flags are not counted (test overhead)
    C.run(cls, 16ull * n, true, [&] {
      launch_fclean<SPLIT>(C, h, sl, n, lm, ref, fp, ext, marks, ftodo, nftodo, nullptr, nullptr,
                           EvCache{}, 0);
    });
    idx = ftodo;
    nidx = nftodo;
  }
  if (!ec.rnd) {
    // (an idx list: a small grid-stride grid)
    // (an idx list in a list pass: a small grid-stride grid; a dense pass,
    // where the test is usually skipped: one thread per saddle)
    const unsigned grid = idx && !dense ? 148u * 8u : (unsigned)((threads + 255) / 256);
    C.run(cls, 8ull * n, true, [&] {
      k_events<SPLIT, FROM_REF, false><<<grid, 256, 0, C.s>>>(
          h, sl, n, slots, lm, ref, ext, marks, C.G, Slabs{nullptr, 1, nullptr}, nullptr, C.cnt,
          idx, nidx, lpos);
    });
    return;
  }
  CK(cudaMemsetAsync(ntodo, 0, sizeof(int), C.s));
  C.run(cls, 16ull * n, true, [&] {
    k_events_check<SPLIT><<<(unsigned)((n + 255) / 256), 256, 0, C.s>>>(
        sl, n, ec, tr, marks, C.G, todo, ntodo, C.cnt, idx, nidx);
  });
  int *todo2 = nullptr, *ntodo2 = nullptr;  // the stamp check's list if k_fclean skips
  if (fp.off) {  // the clean-path test on what the stamps left (caching the clean ones)
    CK(cudaMemsetAsync(nftodo, 0, sizeof(int), C.s));
    C.run(cls, 0, true, [&] {
      launch_fclean<SPLIT>(C, h, sl, n, lm, ref, fp, ext, marks, ftodo, nftodo, todo, ntodo, ec,
                           tr.round);
    });
    todo2 = todo;
    ntodo2 = ntodo;
    todo = ftodo;
    ntodo = nftodo;
  }
  C.run(cls, 0, true, [&] {
    k_events_cached<SPLIT><<<148 * 16, 256, 0, C.s>>>(h, sl, todo, ntodo, slots, lm, ext, marks,
                                                      C.G, ec, tr, C.cnt, todo2, ntodo2);
  });
}

// O7: reference topology of f, computed once per call.
static void build_reference(Ctx &C, const float *f, Reference &R, bool reform = false,
                            bool ext_by_fpaths = false) {
  int64_t V = C.V;
  R.ref = C.arena.get<uint32_t>(V);
  uint64_t *keys = C.arena.get<uint64_t>(V);
  uint64_t *cpkeys = reform ? C.arena.get<uint64_t>(V) : nullptr;
  C.zero();
  if (ext_by_fpaths) R.fslots = C.arena.get<uint8_t>(V);
  C.run(EXACTZ_K_REFERENCE, 8 * (uint64_t)V, true, [&] {
    k_reference_tile<<<C.sgrid, 256, 0, C.s>>>(f, C.G, C.zc, R.ref, keys, cpkeys, C.cnt,
                                               R.fslots);
  });
  C.read();
  R.nS = (int)C.hcnt[C_NSADDLE];
  if (reform) {  // the sorted sequence of all critical points of f
    R.nC = (int)C.hcnt[C_NCP];
    R.CP = C.arena.get<int32_t>(R.nC);
    sort_ids(C, cpkeys, R.nC, R.CP);
  }
  // S: all saddles sorted by the SoS key of f.  J, P: join / split
  // saddles in index (spatial) order, so that consecutive event checks walk
  // nearby integral paths (L1/L2 reuse); their order is otherwise irrelevant.
  // They are selected from the saddle ids sorted by index (Sx).
  uint64_t *sorted = C.arena.get<uint64_t>(R.nS);
  R.S = C.arena.get<int32_t>(R.nS);
  R.J = C.arena.get<int32_t>(R.nS);
  R.P = C.arena.get<int32_t>(R.nS);
  int32_t *Sx = C.arena.get<int32_t>(R.nS);
  int *nsel = C.arena.get<int>(2);
  if (R.nS > 0) {
    size_t tb = 0, tb1 = 0, tb2 = 0, tb3 = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, R.nS, 0, 64, C.s));
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tb1, R.S, Sx, R.nS, 0, 32, C.s));
    CK(cub::DeviceSelect::If(nullptr, tb2, Sx, R.J, nsel, R.nS, IsJoin{R.ref}, C.s));
    CK(cub::DeviceSelect::If(nullptr, tb3, Sx, R.P, nsel + 1, R.nS, IsSplit{R.ref}, C.s));
    size_t tmax = tb > tb1 ? tb : tb1;
    tmax = tmax > tb2 ? tmax : tb2;
    tmax = tmax > tb3 ? tmax : tb3;
    void *tmp = C.arena.get<uint8_t>(tmax);
    C.run(EXACTZ_K_REFERENCE, 32ull * R.nS, false, [&] {
      CK(cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, R.nS, 0, 64, C.s));
    });
    C.run(EXACTZ_K_REFERENCE, 12ull * R.nS, true, [&] {
      k_keys_to_ids<<<blocks_for(R.nS, 256, 1 << 30), 256, 0, C.s>>>(sorted, R.S, R.nS);
    });
    C.run(EXACTZ_K_REFERENCE, 16ull * R.nS, false, [&] {
      CK(cub::DeviceRadixSort::SortKeys(tmp, tb1, R.S, Sx, R.nS, 0, 32, C.s));
      CK(cub::DeviceSelect::If(tmp, tb2, Sx, R.J, nsel, R.nS, IsJoin{R.ref}, C.s));
      CK(cub::DeviceSelect::If(tmp, tb3, Sx, R.P, nsel + 1, R.nS, IsSplit{R.ref}, C.s));
    });
    // C2 by saddle values in S order: posS for the stencils' writes of gS
    R.posS = C.arena.get<int32_t>((size_t)V);
    R.gS = C.arena.get<uint32_t>(R.nS);
    R.lmS = C.arena.get<uint32_t>(R.nS);
    C.run(EXACTZ_K_REFERENCE, 8ull * R.nS, true, [&] {
      k_scatter_pos<<<blocks_for(R.nS, 256, 1 << 30), 256, 0, C.s>>>(R.S, R.nS, R.posS);
    });
    int h[2];
    CK(cudaMemcpyAsync(h, nsel, sizeof(h), cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
    if (C.prof.on) C.prof.drain();
    R.nJ = h[0];
    R.nP = h[1];
    // the C3 kernels read the link masks in S order through these positions
    R.Jpos = C.arena.get<int32_t>(R.nJ);
    R.Ppos = C.arena.get<int32_t>(R.nP);
    C.run(EXACTZ_K_REFERENCE, 8ull * (R.nJ + R.nP), true, [&] {
      if (R.nJ) k_gather_pos<<<blocks_for(R.nJ, 256, 1 << 30), 256, 0, C.s>>>(R.J, R.nJ, R.posS, R.Jpos);
      if (R.nP) k_gather_pos<<<blocks_for(R.nP, 256, 1 << 30), 256, 0, C.s>>>(R.P, R.nP, R.posS, R.Ppos);
    });
  }
  R.m1 = C.arena.get<int32_t>(R.nJ);
  R.M1 = C.arena.get<int32_t>(R.nP);
  // m1 / M1 by walking f's steepest paths from each saddle's link
  if (!reform && !ext_by_fpaths) {  // the two lists concurrently on the side streams
    C.fork();
    C.on_side(0);
    launch_events<false, true>(C, f, R.J, R.nJ, nullptr, nullptr, R.ref, R.m1, nullptr);
    C.on_side(1);
    launch_events<true, true>(C, f, R.P, R.nP, nullptr, nullptr, R.ref, R.M1, nullptr);
    C.join();
  }
}

struct PassOut {
  unsigned long long vt, applied, n[6], walk, evaluated, links;
};

// One CheckConstraints pass on g (O8) followed by the count and, when
// do_edit, the bounded edits (O9).  slots receives g's steepest slots.
// Change-tracking state of a call (single GPU, late passes; kernels.cuh Track).
struct Tracking {
  // vertex activity: act[cur] = this pass's active set (valid when `ready`)
  bool act_on = false, ready = false;
  bool sparse = false;  // few active vertices: the sparse stencil, else the compacted one
  uint32_t *act[2] = {nullptr, nullptr};
  int cur = 0;
  int32_t *list = nullptr;  // active vertices of a sparse pass (k_act_list)
  int *nlist = nullptr;
  uint32_t *edited = nullptr;  // vertices edited by the last pass (k_count_edit)
  bool pull_stars = true;      // this pass: edited bitmap (pulled next pass) or pushed stars
  bool edited_valid = false;   // `edited` holds the previous pass's edits
  // C3 cache with brick stamps
  bool cache_on = false;
  int nbx = 0, nby = 0, nbz = 0, nb = 0, nsx = 0, nsy = 0, nsz = 0, nsb = 0;
  uint16_t *bval = nullptr, *bslot = nullptr, *sbval = nullptr, *sbslot = nullptr;
  EvCache ecJ{}, ecP{};
  int *todo = nullptr, *ntodo = nullptr, *todoP = nullptr;
  // clean-path test of the C3 walks (kernels.cuh FPaths; list passes only)
  bool fp_on = false;
  // k_fclean's gate, per list (join, split), decided on the device from this
  // pass's dirty-tile count d: the test runs when P(a saddle is clean) ~
  // (1 - d / ntiles)^L >= gate, L the average tile entries per saddle
  double fpL[2] = {0.0, 0.0};
  unsigned long long *ndirt = nullptr;  // [2] dirty tiles this pass (D, U)
  void fp_gate(double gate) {
    for (int k = 0; k < 2; ++k) {
      const double f = gate > 0.0 && fpL[k] > 0.0 ? 1.0 - std::pow(gate, 1.0 / fpL[k]) : 1.0;
      (k ? fpP : fpJ).max_dirt = gate > 0.0 ? (unsigned long long)(f * nt) : ~0ull;
    }
  }
  int ntx = 0, nty = 0, ntz = 0, nt = 0;
  FPaths fpJ{}, fpP{};
  uint8_t *dirtD = nullptr, *dirtU = nullptr;  // one byte per tile
  int *ftodo = nullptr, *ftodoP = nullptr, *nftodo = nullptr;
  // FPaths buffers of a list (allocated on the call's stream, before the fork)
  static FPaths fpaths_alloc(Ctx &C, int n) {
    FPaths F{};
    const size_t m = n ? (size_t)n : 1;
    F.off = C.arena.get<int64_t>(m);
    F.len = C.arena.get<uint16_t>(m);
    F.lab = C.arena.get<int32_t>(m * kFLab);
    F.nlab = C.arena.get<uint8_t>(m);
    F.bmask = C.arena.get<unsigned long long>(m);
    F.flow = C.arena.get<uint16_t>(m);
    // tile entries: 24 per saddle on average (C2 7.2, C3 11.8 join / 5.2
    // split); a warp that does not fit leaves its saddles to the walks
    F.cap = 24ull * m + 4096;
    F.tiles = C.arena.get<int32_t>(F.cap);
    return F;
  }
  template <bool SPLIT>
  void fpaths_launch(Ctx &C, const Reference &R, const int32_t *sl, int n, const FPaths &F,
                     unsigned long long *bump, unsigned long long *diag, const float *f,
                     int32_t *ext) {
    if (n > 0)
      C.run(EXACTZ_K_REFERENCE, 8ull * n, true, [&] {
        k_fpaths<SPLIT><<<(unsigned)((n + 255) / 256), 256, 0, C.s>>>(
            sl, n, R.ref, C.G, ntx, nty, bump, F.cap, const_cast<int64_t *>(F.off),
            const_cast<uint16_t *>(F.len), const_cast<int32_t *>(F.tiles),
            const_cast<int32_t *>(F.lab), const_cast<uint8_t *>(F.nlab),
            const_cast<unsigned long long *>(F.bmask), diag, f, ext,
            const_cast<uint16_t *>(F.flow), R.fslots);
      });
  }
  // at setup, in place of the reference walks of build_reference: also
  // writes R.m1 / R.M1
  void start_fpaths(Ctx &C, const Reference &R, const float *f) {
    ntx = (C.G.nx + (1 << FTX_SH) - 1) >> FTX_SH;
    nty = (C.G.ny + (1 << FTY_SH) - 1) >> FTY_SH;
    ntz = (C.G.nz + (1 << FTZ_SH) - 1) >> FTZ_SH;
    nt = ntx * nty * ntz;
    // the two byte arrays (each padded to 16 bytes), then the two counts
    // (cleared by one memset per pass)
    const size_t nt16 = ((size_t)nt + 15) / 16 * 16;
    dirtD = C.arena.get<uint8_t>(2 * nt16 + 16);
    dirtU = dirtD + nt16;
    ndirt = reinterpret_cast<unsigned long long *>(dirtD + 2 * nt16);
    unsigned long long *bump = C.arena.get<unsigned long long>(2);
    CK(cudaMemsetAsync(bump, 0, 2 * sizeof(unsigned long long), C.s));
    static const bool tl = std::getenv("EXACTZ_TIMELINE") != nullptr;  // diagnostic
    unsigned long long *diag = nullptr;
    if (tl) {
      diag = C.arena.get<unsigned long long>(8);
      CK(cudaMemsetAsync(diag, 0, 8 * sizeof(unsigned long long), C.s));
    }
    fpJ = fpaths_alloc(C, R.nJ);
    fpP = fpaths_alloc(C, R.nP);
    C.fork();  // the two lists concurrently
    C.on_side(0);
    fpaths_launch<false>(C, R, R.J, R.nJ, fpJ, bump, diag, f, R.m1);
    C.on_side(1);
    fpaths_launch<true>(C, R, R.P, R.nP, fpP, bump + 1, diag ? diag + 4 : nullptr, f, R.M1);
    C.join();
    if (tl) {
      unsigned long long h[8];
      CK(cudaMemcpyAsync(h, diag, sizeof(h), cudaMemcpyDeviceToHost, C.s));
      CK(cudaStreamSynchronize(C.s));
      std::fprintf(stderr,
                   "fpaths J %d: long %llu labels %llu full %llu entries %llu | P %d: long %llu "
                   "labels %llu full %llu entries %llu\n",
                   R.nJ, h[0], h[1], h[2], h[3], R.nP, h[4], h[5], h[6], h[7]);
    }
    fpJ.dirt = dirtD;
    fpP.dirt = dirtU;
    fpJ.nt = fpP.nt = nt;
    fpJ.ndirt = ndirt;
    fpP.ndirt = ndirt + 1;
    {  // average tile entries per saddle (the gate below)
      unsigned long long h[2];
      CK(cudaMemcpyAsync(h, bump, sizeof(h), cudaMemcpyDeviceToHost, C.s));
      CK(cudaStreamSynchronize(C.s));
      fpL[0] = R.nJ ? (double)h[0] / R.nJ : 0.0;
      fpL[1] = R.nP ? (double)h[1] / R.nP : 0.0;
    }
    ftodo = C.arena.get<int>(R.nJ > 0 ? R.nJ : 1);
    ftodoP = C.arena.get<int>(R.nP > 0 ? R.nP : 1);
    nftodo = C.arena.get<int>(2);
    fp_on = true;
  }
  void geometry(const Ctx &C) {
    nbx = (C.G.nx + BX - 1) / BX;
    nby = (C.G.ny + BY - 1) / BY;
    nbz = (C.G.nz + BZ - 1) / BZ;
    nb = nbx * nby * nbz;
    nsx = (nbx + SB - 1) / SB;
    nsy = (nby + SB - 1) / SB;
    nsz = (nbz + SB - 1) / SB;
    nsb = nsx * nsy * nsz;
  }
  void start_act(Ctx &C) {
    for (int k = 0; k < 2; ++k) {
      act[k] = C.arena.get<uint32_t>(C.mark_words());
      CK(cudaMemsetAsync(act[k], 0, C.mark_words() * 4, C.s));
    }
    list = C.arena.get<int32_t>((size_t)C.V);
    nlist = C.arena.get<int>(1);
    edited = C.arena.get<uint32_t>(C.mark_words());
    act_on = true;
  }
  void start_cache(Ctx &C, const Reference &R) {
    uint16_t *st = C.arena.get<uint16_t>(2 * (size_t)(nb + nsb));
    CK(cudaMemsetAsync(st, 0, 2 * (size_t)(nb + nsb) * 2, C.s));
    bval = st;
    bslot = st + nb;
    sbval = st + 2 * (size_t)nb;
    sbslot = sbval + nsb;
    auto cache = [&](int n) {
      EvCache e;
      e.rnd = C.arena.get<uint16_t>(n);
      e.mask = C.arena.get<unsigned long long>(n);
      e.tgt = C.arena.get<int32_t>(n);
      CK(cudaMemsetAsync(e.rnd, 0, (size_t)(n ? n : 1) * 2, C.s));
      CK(cudaMemsetAsync(e.mask, 0, (size_t)(n ? n : 1) * 8, C.s));  // read with rnd
      return e;
    };
    ecJ = cache(R.nJ);
    ecP = cache(R.nP);
    todo = C.arena.get<int>(R.nJ > 0 ? R.nJ : 1);
    ntodo = C.arena.get<int>(2);
    todoP = C.arena.get<int>(R.nP > 0 ? R.nP : 1);
    cache_on = true;
  }
  Track track(int round) const {
    Track T{};
    T.nbx = nbx;
    T.nby = nby;
    T.nbz = nbz;
    T.round = round;
    T.nsx = nsx;
    T.nsy = nsy;
    if (cache_on) {
      T.bval = bval;
      T.bslot = bslot;
      T.sbval = sbval;
      T.sbslot = sbslot;
    }
    if (act_on) {
      T.act_next = act[cur ^ 1];
      T.edited = pull_stars ? edited : nullptr;
    }
    T.patch = patch;
    T.npatch = npatch;
    T.patch_cap = patch_cap;
    return T;
  }
  int32_t *patch = nullptr;  // see HostSnap
  int *npatch = nullptr;
  int patch_cap = 0;
};

// exactz_correct_host: once the passes are sparse, the result's D2H copy
// starts on a side stream while the remaining passes run; the vertices they
// edit are listed by k_count_edit and patched into the host copy at the end
// (a vertex not listed was final before the copy began).
struct HostSnap {
  float *out_host = nullptr;
  uint8_t *counts_host = nullptr;  // nullptr: edit counts not requested
  cudaStream_t cs = nullptr;
  bool started = false, overflow = false;
};

// One CheckConstraints pass on g (O8) followed by the count and, when
// do_edit, the bounded edits (O9).  slots receives g's steepest slots.
// With tracking: a sparse pass re-evaluates only the active vertices, and
// cached C3 results are reused while their bricks are unchanged (exact; see
// kernels.cuh Track).
struct PassTicket {
  int buf = 0;            // counter buffer of the pass (Ctx::fold)
  bool listed = false;    // the stencil counted the vertices it evaluated (C_EVAL)
};
static PassTicket enqueue_pass(Ctx &C, const Reference &R, const float *f, float *g, uint8_t *c,
                               uint32_t *marks, uint8_t *slots, uint32_t *lm, float xi,
                               float delta, int N, uint32_t flags, bool do_edit,
                               Tracking *trk = nullptr, int round = 0, int buf = 0,
                               Tracking *fpk = nullptr) {
  bool c3 = !(flags & EXACTZ_NO_C3);
  C.zero();
  Track T = trk ? trk->track(round) : Track{};
  T.posS = R.posS;  // the stencils write g at the saddles into gS (C2 below)
  T.gS = R.gS;
  T.lmS = R.lmS;  // and their link masks, in S order (C3 below)
  const bool sparse = trk && trk->ready && trk->sparse;
  const bool compact = trk && trk->ready && !trk->sparse;
  // the clean-path test needs every vertex with a non-f pointer flagged: the
  // list stencil flags them in list passes (an unlisted vertex has f's
  // pointers).  Dense passes do not run it: flagging from the key stencil
  // cost C3 1.8 -> 2.0 ms per dense pass and in those passes nearly every
  // tile is dirty (the gate skipped the test in all of them)
  const bool fpass = fpk && fpk->fp_on && sparse;
  if (fpass) {  // this pass's dirty tiles and their counts
    CK(cudaMemsetAsync(fpk->dirtD, 0, 2 * (((size_t)fpk->nt + 15) / 16 * 16) + 16, C.s));
    T.dirtD = fpk->dirtD;
    T.dirtU = fpk->dirtU;
    T.ntx = fpk->ntx;
    T.nty = fpk->nty;
  }
  // algorithmic bytes per vertex: g 4 + ref 4 read, slots 1 + mark bits 1/8
  // written; a sparse or compacted pass: the active vertices
  // only (plus the activity bitmap)
  if (compact && trk->edited_valid) {  // this pass's set: fired | stars of last pass's edits
    C.run(EXACTZ_K_SPARSE, (uint64_t)C.V / 4, true, [&] {
      k_dilate_or<<<148 * 16, 256, 0, C.s>>>(trk->act[trk->cur], trk->edited, C.G);
    });
  }
  if (compact) {
    C.run(EXACTZ_K_SPARSE, (uint64_t)C.V / 8, true, [&] {
      k_stencil_compact<<<C.sgrid, C.sblock, 0, C.s>>>(g, R.ref, marks, slots, lm, trk->act[trk->cur],
                                                        C.G, C.zc, T, C.cnt);
    });
  } else if (!sparse) {
    // algorithmic bytes: g 4 + packed ref 4 read, mark bit 1/8
    // written and read: 8.25 B per vertex
    C.run(EXACTZ_K_STENCIL, (uint64_t)C.V * 33 / 4, true, [&] {
      // (debug flag 0x4000: the one-row key stencil)
      const dim3 g2(C.sgrid.x, (unsigned)((C.G.ny + K2TY - 1) / K2TY), C.sgrid.z);
      // (debug flag 0x8000: thread-staged planes instead of TMA)
      const bool tma = !(flags & 0x8000u) && C.plane_map(g);
      if (C.keyed && !(flags & 0x4000u) && trk && tma)
        k_stencil_key2<true, true><<<g2, TX * K2W, 0, C.s>>>(g, R.ref, marks, slots, lm, C.G, C.zc,
                                                             T, C.cnt, C.tmap);
      else if (C.keyed && !(flags & 0x4000u) && tma)
        k_stencil_key2<false, true><<<g2, TX * K2W, 0, C.s>>>(g, R.ref, marks, slots, lm, C.G,
                                                              C.zc, T, C.cnt, C.tmap);
      else if (C.keyed && !(flags & 0x4000u) && trk)
        k_stencil_key2<true, false><<<g2, TX * K2W, 0, C.s>>>(g, R.ref, marks, slots, lm, C.G,
                                                              C.zc, T, C.cnt, C.tmap);
      else if (C.keyed && !(flags & 0x4000u))
        k_stencil_key2<false, false><<<g2, TX * K2W, 0, C.s>>>(g, R.ref, marks, slots, lm, C.G,
                                                               C.zc, T, C.cnt, C.tmap);
      else if (C.keyed && trk)
        k_stencil_key<true><<<C.sgrid, C.sblock, 0, C.s>>>(g, R.ref, marks, slots, lm, C.G, C.zc,
                                                           T, C.cnt);
      else if (C.keyed)
        k_stencil_key<false><<<C.sgrid, C.sblock, 0, C.s>>>(g, R.ref, marks, slots, lm, C.G, C.zc,
                                                            T, C.cnt);
      else if (C.fast && trk)
        k_stencil_fast<true><<<C.sgrid, C.sblock, 0, C.s>>>(g, R.ref, marks, slots, lm, C.G, C.zc,
                                                            T, C.cnt);
      else if (C.fast && (flags & 0x1000u))  // experiment: ALU-pipe lower mask
        k_stencil_fast<false, true><<<C.sgrid, C.sblock, 0, C.s>>>(g, R.ref, marks, slots, lm,
                                                                   C.G, C.zc, T, C.cnt);
      else if (C.fast)
        k_stencil_fast<false><<<C.sgrid, C.sblock, 0, C.s>>>(g, R.ref, marks, slots, lm, C.G,
                                                             C.zc, T, C.cnt);
      else if (trk)
        k_stencil<true><<<C.sgrid, C.sblock, 0, C.s>>>(g, R.ref, marks, slots, lm, C.G, C.zc, T,
                                                       C.cnt);
      else
        k_stencil<false><<<C.sgrid, C.sblock, 0, C.s>>>(g, R.ref, marks, slots, lm, C.G, C.zc, T,
                                                        C.cnt);
    });
  } else {
    CK(cudaMemsetAsync(trk->nlist, 0, sizeof(int), C.s));
    C.run(EXACTZ_K_SPARSE, (uint64_t)C.V / 8, true, [&] {
      k_act_list<<<148 * 16, 256, 0, C.s>>>(trk->act[trk->cur],
                                            trk->edited_valid ? trk->edited : nullptr, C.G,
                                            trk->list, trk->nlist);
    });
    C.run(EXACTZ_K_SPARSE, 0, true, [&] {
      // (debug flag 0x400000: the float-compare list stencil for keyed fields)
      if (C.keyed && !(flags & 0x400000u))
        k_stencil_list_key<<<148 * 16, 256, 0, C.s>>>(g, R.ref, marks, slots, lm, trk->list,
                                                      trk->nlist, C.G, T, C.cnt);
      else
        k_stencil_list<<<148 * 16, 256, 0, C.s>>>(g, R.ref, marks, slots, lm, trk->list,
                                                  trk->nlist, C.G, T, C.cnt);
    });
  }
  // R4 (C2) from the saddle values the stencil wrote in S order (gS), and
  // the two C3 event kernels: independent (all read the snapshot and the
  // stencil's outputs, all only OR marks and add counters); the events run
  // on the two side streams, joined before the count/edit.
  C.fork();
  if (!(flags & EXACTZ_NO_C2) && R.nS > 1) {
    C.run(EXACTZ_K_SADDLE_ORDER, 8ull * R.nS, true, [&] {
      k_saddle_order_vals<<<blocks_for(R.nS, 256, 1 << 30), 256, 0, C.s>>>(R.gS, R.S, R.nS,
                                                                           marks, C.G, C.cnt);
    });
  }
  C.on_side(1);
  if (c3 && (flags & EXACTZ_REFORMULATED) && R.nC > 1) {
    // R7: adjacent critical points in the f order
    C.run(EXACTZ_K_EVENTS, 8ull * R.nC, true, [&] {
      k_saddle_order<<<blocks_for(R.nC, 256, 1 << 30), 256, 0, C.s>>>(g, R.CP, R.nC, marks, C.G,
                                                                      C.cnt, C_N1 + 4);
    });
  } else if (c3 && !(flags & EXACTZ_REFORMULATED)) {
    const bool cache = trk && trk->cache_on;
    launch_events<true, false>(C, g, R.P, R.nP, slots, R.lmS, R.ref, R.M1, marks,
                               cache ? trk->ecP : EvCache{}, T, cache ? trk->todoP : nullptr,
                               cache ? trk->ntodo + 1 : nullptr,
                               fpass ? fpk->fpP : FPaths{},
                               fpass ? fpk->ftodoP : nullptr, fpass ? fpk->nftodo + 1 : nullptr,
                               R.Ppos, !sparse && !compact);
    C.on_side(0);
    launch_events<false, false>(C, g, R.J, R.nJ, slots, R.lmS, R.ref, R.m1, marks,
                                cache ? trk->ecJ : EvCache{}, T, cache ? trk->todo : nullptr,
                                cache ? trk->ntodo : nullptr,
                                fpass ? fpk->fpJ : FPaths{},
                                fpass ? fpk->ftodo : nullptr, fpass ? fpk->nftodo : nullptr,
                                R.Jpos, !sparse && !compact);
  }
  C.join();
  if (trk && trk->act_on && trk->pull_stars)  // read by this pass's stencil, rewritten below
    CK(cudaMemsetAsync(trk->edited, 0, C.mark_words() * 4, C.s));
  // bytes: mark words read (the per-edit 14 B are added once V_t is known)
  C.run(EXACTZ_K_EDIT, (uint64_t)C.V / 8, true, [&] {
    if (trk)
      k_count_edit<true><<<148 * 8, 256, 0, C.s>>>(g, c, marks, f, C.G, xi, delta, N,
                                                   do_edit ? 1 : 0, T, C.cnt);
    else
      k_count_edit<false><<<148 * 8, 256, 0, C.s>>>(g, c, marks, f, C.G, xi, delta, N,
                                                    do_edit ? 1 : 0, T, C.cnt);
  });
  C.fold(buf);
  if (trk && trk->act_on) {  // act_next (| stars of `edited`) is the next pass's set
    trk->cur ^= 1;
    trk->ready = true;
    trk->edited_valid = trk->pull_stars;
  }
  PassTicket t;
  t.buf = buf;
  t.listed = sparse || compact;
  return t;
}

// The counters of an enqueued pass (waits for that pass only).
static PassOut collect_pass(Ctx &C, const PassTicket &t) {
  const unsigned long long *h = C.counters(t.buf);
  if (C.prof.on) {
    CK(cudaStreamSynchronize(C.s));
    C.prof.drain();
  }
  PassOut o;
  o.vt = h[C_VT];
  o.applied = h[C_APPLIED];
  C.prof.bytes[EXACTZ_K_EDIT] += 14ull * o.applied;  // f, g, c read; g, c written
  for (int k = 0; k < 6; ++k) o.n[k] = h[C_N1 + k];
  o.walk = h[C_WALK];
  // vertices the stencil evaluated: all of them in a dense pass, the list
  // otherwise (counted by the list / compacted stencils)
  o.evaluated = t.listed ? h[C_EVAL] : (unsigned long long)C.V;
  o.links = h[C_LINKS];
  C.prof.bytes[EXACTZ_K_EVENTS] += 8ull * o.links;
  return o;
}

static PassOut detect_and_edit(Ctx &C, const Reference &R, const float *f, float *g, uint8_t *c,
                               uint32_t *marks, uint8_t *slots, uint32_t *lm, float xi,
                               float delta, int N, uint32_t flags, bool do_edit,
                               Tracking *trk = nullptr, int round = 0) {
  return collect_pass(C, enqueue_pass(C, R, f, g, c, marks, slots, lm, xi, delta, N, flags,
                                      do_edit, trk, round, 0));
}

static void validate_inputs(Ctx &C, const float *f, const float *g, float xi,
                            uint32_t flags = 0) {
  C.zero();
  C.run(EXACTZ_K_VALIDATE, 8 * (uint64_t)C.V, true,
        [&] { k_validate<<<blocks_for(C.V, 256), 256, 0, C.s>>>(f, g, C.V, xi, C.cnt); });
  C.read();
  // debug flag 0x800: the general stencil even for non-negative fields
  C.fast = C.hcnt[C_NEG] == 0 && !(flags & 0x800u);
  // exact SoS keys (stencil_key.cuh) when every value g takes, [lo_min,
  // ghat_max], is within [2^-41, 2^63) and spans < 2^28 bit patterns
  // (debug flag 0x2000: off)
  {
    const uint32_t lo_min = ~(uint32_t)C.hcnt[C_KEYMIN], g_max = (uint32_t)C.hcnt[C_KEYMAX];
    C.keyed = C.fast && !(flags & 0x2000u) && lo_min >= kKeyLoMinBits && g_max < kKeyHiMaxBits &&
              g_max >= lo_min && g_max - lo_min < kKeySpan;
    for (int s = 0; s < kSlots; ++s) C.G.kc[s] = (uint32_t)s - 16u * lo_min;
  }
  if (C.hcnt[C_BAD_NF]) {
    set_err("validate", "non-finite value in f or g");
    throw Error{EXACTZ_EINVAL};
  }
  if (C.hcnt[C_BAD_BOUND]) {
    set_err("validate", "|f - g| > eps for some vertex");
    throw Error{EXACTZ_EBOUND};
  }
}

// Timing events of the per-pass stats rows, kept across calls (per thread and
// device): creating two events per pass cost the timed bench steps ~4 ms.
struct EventPool {
  int dev = -1;
  std::vector<cudaEvent_t> free;
};
static thread_local EventPool g_evpool;
static cudaEvent_t pass_event() {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev != g_evpool.dev) {
    g_evpool.free.clear();  // events of another device are left to the driver
    g_evpool.dev = dev;
  }
  if (!g_evpool.free.empty()) {
    cudaEvent_t e = g_evpool.free.back();
    g_evpool.free.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}
static void pass_event_put(cudaEvent_t e) { g_evpool.free.push_back(e); }

// g_ready (exactz_correct_host): an event recorded after g_in's host->device
// copy, which may still be running when the call starts; the reference of f
// (after a finiteness check of f alone) then overlaps that copy, and the full
// validation waits for it.
static exactz_status correct_impl(const float *f, const float *g_in, const int64_t dims[3],
                                  float eps, float *out, uint32_t *iters, const exactz_opts *opts,
                                  cudaStream_t s, cudaEvent_t g_ready = nullptr,
                                  HostSnap *hs = nullptr) {
  int64_t V = 0;
  if (!f || !g_in || !out || !iters) return EXACTZ_EINVAL;
  if (check_dims(dims, &V) != EXACTZ_OK) return EXACTZ_EINVAL;
  if (!std::isfinite(eps) || !(eps >= 0.0f)) return EXACTZ_EINVAL;
  int N = (opts && opts->N) ? (int)opts->N : 5;
  if (N < 1 || N > 254) return EXACTZ_EINVAL;
  uint32_t flags = opts ? opts->flags : 0u;
  uint32_t max_iters = opts ? opts->max_iters : 0u;
  exactz_stats *stats = opts ? opts->stats : nullptr;

  Ctx C(s);
  C.V = V;
  C.dbg = flags;
  C.prof.on = (flags & EXACTZ_PROFILE) != 0;
  C.init(dims);
  cudaEvent_t e0, e1, e2;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  CK(cudaEventRecord(e0, s));
  Reference R;
  Tracking trk;
  trk.geometry(C);
  // the clean-path test's f-walks (FPaths) replace the reference walks of
  // m1 / M1 whenever list passes can run (they may use the test)
  const bool fp_setup = !(flags & (EXACTZ_NO_TRACK | EXACTZ_REFORMULATED | EXACTZ_NO_C3 |
                                   0x80000u | 0x100u | 0x400u));
  static const double fp_gate = [] {
    // tuning knob (default 0.1): k_fclean runs when the estimated clean
    // fraction (1 - dirty tiles / tiles)^L reaches it (0: always)
    const char *e = std::getenv("EXACTZ_FP_GATE");
    return e ? std::atof(e) : 0.1;
  }();
  auto reference = [&] {
    build_reference(C, f, R, (flags & EXACTZ_REFORMULATED) != 0, fp_setup);
    if (fp_setup) {
      trk.start_fpaths(C, R, f);
      trk.fp_gate((flags & 0x200000u) ? 0.0 : fp_gate);  // (debug flag 0x200000: always)
    }
  };
  if (g_ready) {
    // f alone first (k_validate of (f, f) flags exactly the non-finite f),
    // its reference while g_in is still in flight, then the full check
    C.zero();
    C.run(EXACTZ_K_VALIDATE, 4 * (uint64_t)C.V, true,
          [&] { k_validate<<<blocks_for(C.V, 256), 256, 0, C.s>>>(f, f, C.V, 0.0f, C.cnt); });
    C.read();
    if (C.hcnt[C_BAD_NF]) {
      set_err("validate", "non-finite value in f or g");
      throw Error{EXACTZ_EINVAL};
    }
    reference();
    CK(cudaStreamWaitEvent(s, g_ready, 0));
    validate_inputs(C, f, g_in, eps, flags);
    if (out != g_in) CK(cudaMemcpyAsync(out, g_in, V * sizeof(float), cudaMemcpyDeviceToDevice, s));
  } else {
    validate_inputs(C, f, g_in, eps, flags);
    if (out != g_in) CK(cudaMemcpyAsync(out, g_in, V * sizeof(float), cudaMemcpyDeviceToDevice, s));
    reference();
  }
  uint8_t *c = (opts && opts->edit_counts) ? opts->edit_counts : C.arena.get<uint8_t>(V);
  uint32_t *marks = C.arena.get<uint32_t>(C.mark_words());
  uint8_t *slots = C.arena.get<uint8_t>(V);
  // (the stencils write the saddles' link masks into R.lmS, S order)
  uint32_t *lm = C.arena.get<uint32_t>(1);
  CK(cudaMemsetAsync(c, 0, V, s));
  CK(cudaMemsetAsync(marks, 0, C.mark_words() * sizeof(uint32_t), s));
  CK(cudaEventRecord(e1, s));

  const float delta = eps / (float)N;  // Delta = RN(xi / N)
  uint32_t it = 0, rows = 0;
  exactz_status st = EXACTZ_OK;
  static const unsigned long long act_div = [] {
    const char *e = std::getenv("EXACTZ_ACT_DIV");  // tuning knob (default 8)
    return e ? std::strtoull(e, nullptr, 10) : 8ull;
  }();
  static const unsigned long long cache_div = [] {
    const char *e = std::getenv("EXACTZ_CACHE_DIV");  // tuning knob (default 4)
    return e ? std::strtoull(e, nullptr, 10) : 4ull;
  }();
  static const unsigned long long compact_div = [] {
    const char *e = std::getenv("EXACTZ_COMPACT_DIV");  // tuning knob (default 0: off)
    return e ? std::strtoull(e, nullptr, 10) : 0ull;
  }();
  unsigned long long prev_vt = (unsigned long long)V;
  const bool allow_track = !(flags & EXACTZ_NO_TRACK);
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pass_ev;
  static const bool tl = std::getenv("EXACTZ_TIMELINE") != nullptr;  // diagnostic
  // Pipelined loop: pass r+1 is enqueued before pass r's counters are read
  // (they arrive through mapped memory, Ctx::fold), so the host's read,
  // decision and launches overlap the GPU's work instead of idling it
  // between passes.  If pass r turns out to be the last (V_t = 0, or no edit
  // applied), pass r+1 evaluated an unchanged g: it marks the same set, edits
  // nothing, and its counters are dropped.  The tracking choices made for
  // pass r+1 (from V_t of pass r-1) change only the speed, never the bits.
  // Not after a pass that may not edit (max_iters: that pass is the last);
  // off when profiling or with the per-pass timeline (debug flag 0x100000).
  const bool pipe = !C.prof.on && !tl && !(flags & 0x100000u);
  struct Enq {
    PassTicket t;
    int round = 0;
    bool may_edit = true;
    cudaEvent_t pa = nullptr, pb = nullptr, ta = nullptr, tb = nullptr;
    std::chrono::steady_clock::time_point h0;
  };
  auto enqueue = [&](int round) {
    Enq e;
    e.round = round;  // stamps are 16-bit pass numbers
    // every pass before this one edited (else the loop has ended)
    e.may_edit = !(max_iters && (uint32_t)(round - 1) >= max_iters);
    if (allow_track && round >= 2 && round < 65000) {
      // vertex activity once <= V/act_div vertices are marked: the pass after
      // uses the list-based sparse stencil; the C3 cache once the marks are
      // sparse at brick scale
      // (debug flag 0x400: compacted passes from the second pass on instead
      // of the list-based ones)
      const bool force_compact = (flags & 0x400u) != 0;
      trk.sparse = !force_compact;
      // stars of this pass's edits: pulled (dilation of an edited bitmap) when
      // many are expected, pushed by the edit kernel when few
      trk.pull_stars = prev_vt * 256 > (unsigned long long)V;
      if (!(flags & 0x100u) && !trk.act_on &&
          (force_compact || prev_vt * act_div <= (unsigned long long)V ||
           (compact_div && prev_vt * compact_div <= (unsigned long long)V)))
        trk.start_act(C);
      if (!(flags & (0x200u | EXACTZ_REFORMULATED)) && !trk.cache_on &&
          prev_vt * cache_div <= (unsigned long long)trk.nb)
        trk.start_cache(C, R);
      // the clean-path test with the list passes (debug flag 0x80000: off)
    }
    // (debug 0x40000: passes after the host copy began run untracked, the
    // path a run beyond round 65000 takes)
    const bool tracked = allow_track && round < 65000 && (trk.act_on || trk.cache_on) &&
                         !((flags & 0x40000u) && hs && hs->started);
    // an untracked pass lists no edits for the host copy's patch: once the
    // copy has begun, the caller must copy the whole result instead
    if (hs && hs->started && !tracked) hs->overflow = true;
    e.h0 = std::chrono::steady_clock::now();
    if (tl) {
      CK(cudaEventCreate(&e.ta));
      CK(cudaEventCreate(&e.tb));
      CK(cudaEventRecord(e.ta, s));
    }
    static const unsigned long long snap_div = [] {
      const char *v = std::getenv("EXACTZ_SNAP_DIV");  // tuning knob (default 1024)
      return v ? std::strtoull(v, nullptr, 10) : 1024ull;
    }();
    // (debug 0x10000: start as soon as vertex activity is on; 0x20000: a
    // one-entry patch list, so any later edit overflows it)
    if (hs && !hs->started && trk.act_on && e.may_edit &&
        ((flags & 0x10000u) || prev_vt * snap_div <= (unsigned long long)V)) {
      trk.patch_cap = (flags & 0x20000u) ? 1 : (int)std::min<int64_t>(V, V / 64 + 4096);
      trk.patch = C.arena.get<int32_t>(trk.patch_cap);
      trk.npatch = C.arena.get<int>(1);
      CK(cudaMemsetAsync(trk.npatch, 0, sizeof(int), s));
      cudaEvent_t ev;
      CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CK(cudaEventRecord(ev, s));
      CK(cudaStreamWaitEvent(hs->cs, ev, 0));
      CK(cudaEventDestroy(ev));
      CK(cudaMemcpyAsync(hs->out_host, out, V * sizeof(float), cudaMemcpyDeviceToHost, hs->cs));
      if (hs->counts_host)
        CK(cudaMemcpyAsync(hs->counts_host, c, V, cudaMemcpyDeviceToHost, hs->cs));
      hs->started = true;
    }
    // per-pass GPU span for the stats rows (events read after the final sync)
    if (stats && stats->rows && (uint32_t)(round - 1) < stats->cap) {
      e.pa = pass_event();
      e.pb = pass_event();
      CK(cudaEventRecord(e.pa, s));
    }
    e.t = enqueue_pass(C, R, f, out, c, marks, slots, lm, eps, delta, N, flags, e.may_edit,
                       tracked ? &trk : nullptr, round, round & 1, &trk);
    if (e.pa) CK(cudaEventRecord(e.pb, s));
    return e;
  };
  Enq cur = enqueue(1);
  for (;;) {
    Enq nxt;
    bool have_next = false;
    if (pipe && cur.may_edit) {  // speculative: cur may turn out to be the last pass
      nxt = enqueue(cur.round + 1);
      have_next = true;
    }
    PassOut o = collect_pass(C, cur.t);
    if (cur.pa) pass_ev.push_back({cur.pa, cur.pb});
    if (tl) {  // GPU span of the pass (main stream) vs host wall-clock span
      CK(cudaEventRecord(cur.tb, s));
      CK(cudaEventSynchronize(cur.tb));
      float gms = 0;
      CK(cudaEventElapsedTime(&gms, cur.ta, cur.tb));
      const double hms = std::chrono::duration<double, std::milli>(
                             std::chrono::steady_clock::now() - cur.h0).count();
      std::fprintf(stderr, "pass %3d vt %12llu gpu %8.3f ms host %8.3f ms\n", cur.round, o.vt,
                   gms, hms);
      cudaEventDestroy(cur.ta);
      cudaEventDestroy(cur.tb);
    }
    prev_vt = o.vt;
    if (stats && stats->rows && rows < stats->cap) {
      exactz_iter_stats &r = stats->rows[rows];
      r.violations = o.vt;
      r.applied = o.applied;
      for (int k = 0; k < 6; ++k) r.n[k] = o.n[k];
      r.walk_steps = o.walk;
      r.evaluated = o.evaluated;
      r.links = o.links;
      r.ms = 0.0;  // set from the pass events after the final sync
    }
    ++rows;
    bool last = false;
    if (o.vt == 0) {
      last = true;
    } else if (!cur.may_edit || o.applied == 0) {
      st = EXACTZ_ESTUCK;
      last = true;
    }
    if (last) {
      if (have_next && nxt.pa) {  // the dropped speculative pass
        pass_event_put(nxt.pa);
        pass_event_put(nxt.pb);
      }
      break;
    }
    ++it;
    cur = have_next ? nxt : enqueue(cur.round + 1);
  }
  CK(cudaEventRecord(e2, s));
  if (hs && hs->started) {  // patch the host copy with the vertices edited since it began
    int np = 0;
    CK(cudaMemcpyAsync(&np, trk.npatch, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hs->overflow || np > trk.patch_cap) {
      hs->overflow = true;  // the caller copies the whole result
    } else if (np == 0) {
      CK(cudaStreamSynchronize(hs->cs));
    } else {
      float *vals = C.arena.get<float>(np);
      uint8_t *cnts = hs->counts_host ? C.arena.get<uint8_t>(np) : nullptr;
      k_gather_patch<<<(np + 255) / 256, 256, 0, s>>>(trk.patch, np, out, hs->counts_host ? c : nullptr,
                                                       vals, cnts);
      g_launches++;
      CK(cudaGetLastError());
      std::vector<int32_t> hi(np);
      std::vector<float> hv(np);
      std::vector<uint8_t> hc(cnts ? np : 0);
      CK(cudaMemcpyAsync(hi.data(), trk.patch, np * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(hv.data(), vals, np * sizeof(float), cudaMemcpyDeviceToHost, s));
      if (cnts) CK(cudaMemcpyAsync(hc.data(), cnts, np, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      CK(cudaStreamSynchronize(hs->cs));
      for (int k = 0; k < np; ++k) {
        hs->out_host[hi[k]] = hv[k];
        if (cnts) hs->counts_host[hi[k]] = hc[k];
      }
    }
  }
  // labels of the final field: the last pass ran on it (no edit followed), so
  // `slots` holds its steepest pointers
  if (opts && (opts->label_min || opts->label_max)) {
    int32_t *ld = opts->label_min ? opts->label_min : C.arena.get<int32_t>(V);
    int32_t *lu = opts->label_max ? opts->label_max : C.arena.get<int32_t>(V);
    full_labels(C, slots, ld, lu);
  }
  CK(cudaStreamSynchronize(s));
  if (stats) {
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, e0, e1);
    cudaEventElapsedTime(&b, e1, e2);
    stats->ms_setup = a;
    stats->ms_loop = b;
    stats->nrows = rows;
    stats->n_saddles = (uint64_t)R.nS;
    stats->n_join = (uint64_t)R.nJ;
    stats->n_split = (uint64_t)R.nP;
    for (size_t k = 0; k < pass_ev.size(); ++k) {
      float ms = 0;
      cudaEventElapsedTime(&ms, pass_ev[k].first, pass_ev[k].second);
      stats->rows[k].ms = ms;
    }
    for (int k = 0; k < EXACTZ_K_CLASSES; ++k) {
      stats->kernel_ms[k] = C.prof.ms[k];
      stats->kernel_launches[k] = C.prof.launches[k];
      stats->kernel_bytes[k] = C.prof.bytes[k];
    }
  }
  for (auto &e : pass_ev) {
    pass_event_put(e.first);
    pass_event_put(e.second);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  *iters = it;
  return st;
}

}  // namespace exz

#include "sharded.cuh"

using namespace exz;

template <class Fn>
static exactz_status guarded(Fn fn) {
  try {
    return fn();
  } catch (const Error &e) {
    return e.st;
  } catch (const std::bad_alloc &) {
    set_err("host", "out of memory");
    return EXACTZ_ENOMEM;
  } catch (...) {
    set_err("host", "unexpected exception");
    return EXACTZ_ECUDA;
  }
}

extern "C" {

exactz_status exactz_correct(const float *f, const float *g_in, const int64_t dims[3],
                             float eps_abs, float *out, uint32_t *iters, const exactz_opts *opts,
                             void *stream) {
  return guarded([&] {
    return correct_impl(f, g_in, dims, eps_abs, out, iters, opts, (cudaStream_t)stream);
  });
}

exactz_status exactz_correct_host(const float *f_host, const float *g_in_host,
                                  const int64_t dims[3], float eps_abs, float *out_host,
                                  uint32_t *iters, const exactz_opts *opts_host, void *stream) {
  return guarded([&]() -> exactz_status {
    int64_t V = 0;
    if (!f_host || !g_in_host || !out_host || !iters) return EXACTZ_EINVAL;
    if (check_dims(dims, &V) != EXACTZ_OK) return EXACTZ_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    Arena A(s);
    float *df = A.get<float>(V), *dg = A.get<float>(V);
    // f on the call's stream, g on a side stream behind it (one copy engine
    // direction: f arrives first); the reference of f overlaps g's copy
    cudaStream_t cs;
    cudaEvent_t fdone, gdone;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&fdone, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&gdone, cudaEventDisableTiming));
    struct Guard {
      cudaStream_t cs;
      cudaEvent_t a, b;
      ~Guard() {
        cudaStreamSynchronize(cs);
        cudaStreamDestroy(cs);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
      }
    } guard{cs, fdone, gdone};
    CK(cudaMemcpyAsync(df, f_host, V * sizeof(float), cudaMemcpyHostToDevice, s));
    // g's copy starts when f's is done (also orders dg's stream-ordered
    // allocation on s before its use on cs)
    CK(cudaEventRecord(fdone, s));
    CK(cudaStreamWaitEvent(cs, fdone, 0));
    CK(cudaMemcpyAsync(dg, g_in_host, V * sizeof(float), cudaMemcpyHostToDevice, cs));
    CK(cudaEventRecord(gdone, cs));
    exactz_opts o{};
    if (opts_host) o = *opts_host;
    if (o.edit_counts) o.edit_counts = A.get<uint8_t>(V);
    if (o.label_min) o.label_min = A.get<int32_t>(V);
    if (o.label_max) o.label_max = A.get<int32_t>(V);
    HostSnap hs;
    hs.out_host = out_host;
    hs.counts_host = (opts_host && opts_host->edit_counts) ? opts_host->edit_counts : nullptr;
    hs.cs = cs;
    exactz_status st = correct_impl(df, dg, dims, eps_abs, dg, iters, &o, s, gdone, &hs);
    if (st != EXACTZ_OK && st != EXACTZ_ESTUCK) return st;
    if (!hs.started || hs.overflow) {
      CK(cudaStreamSynchronize(cs));  // a partial copy must not land after the full one
      CK(cudaMemcpyAsync(out_host, dg, V * sizeof(float), cudaMemcpyDeviceToHost, s));
      if (opts_host && opts_host->edit_counts)
        CK(cudaMemcpyAsync(opts_host->edit_counts, o.edit_counts, V, cudaMemcpyDeviceToHost, s));
    }
    if (opts_host && opts_host->label_min)
      CK(cudaMemcpyAsync(opts_host->label_min, o.label_min, V * 4, cudaMemcpyDeviceToHost, s));
    if (opts_host && opts_host->label_max)
      CK(cudaMemcpyAsync(opts_host->label_max, o.label_max, V * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return st;
  });
}

exactz_status exactz_check(const float *f, const float *g, const int64_t dims[3], float eps_abs,
                           uint64_t *violations, exactz_iter_stats *row, uint32_t flags,
                           void *stream) {
  return guarded([&]() -> exactz_status {
    int64_t V = 0;
    if (!f || !g || !violations) return EXACTZ_EINVAL;
    if (check_dims(dims, &V) != EXACTZ_OK) return EXACTZ_EINVAL;
    if (!std::isfinite(eps_abs) || !(eps_abs >= 0.0f)) return EXACTZ_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    Ctx C(s);
    C.V = V;
    C.init(dims);
    validate_inputs(C, f, g, eps_abs, flags);
    Reference R;
    build_reference(C, f, R, (flags & EXACTZ_REFORMULATED) != 0);
    uint32_t *marks = C.arena.get<uint32_t>(C.mark_words());
    uint8_t *slots = C.arena.get<uint8_t>(V);
  uint32_t *lm = C.arena.get<uint32_t>(1);  // (link masks go to R.lmS)
    CK(cudaMemsetAsync(marks, 0, C.mark_words() * sizeof(uint32_t), s));
    PassOut o = detect_and_edit(C, R, f, const_cast<float *>(g), nullptr, marks, slots, lm, eps_abs,
                                0.0f, 5, flags, false);
    *violations = o.vt;
    if (row) {
      row->violations = o.vt;
      row->applied = 0;
      for (int k = 0; k < 6; ++k) row->n[k] = o.n[k];
      row->walk_steps = o.walk;
      row->evaluated = o.evaluated;
      row->links = o.links;
      row->ms = 0.0;
    }
    CK(cudaStreamSynchronize(s));
    return EXACTZ_OK;
  });
}

exactz_status exactz_eps_from_relative(const float *f, int64_t n, double rel, float *eps_abs,
                                       void *stream) {
  return guarded([&]() -> exactz_status {
    if (!f || n < 1 || !eps_abs || !std::isfinite(rel) || rel < 0) return EXACTZ_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    Arena A(s);
    unsigned long long *cnt = A.get<unsigned long long>(C_NALLOC);
    CK(cudaMemsetAsync(cnt, 0, C_NALLOC * 8, s));
    unsigned long long init[C_NCOUNTERS] = {};
    init[C_KEYMIN] = 0xffffffffull;
    CK(cudaMemcpyAsync(cnt, init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_minmax<<<blocks_for(n, 256), 256, 0, s>>>(f, n, cnt);
    g_launches++;
    CK(cudaGetLastError());
    unsigned long long h[C_NCOUNTERS];
    CK(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    auto unkey = [](uint32_t k) {
      uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
      float v;
      std::memcpy(&v, &b, 4);
      return v;
    };
    double mn = unkey((uint32_t)h[C_KEYMIN]), mx = unkey((uint32_t)h[C_KEYMAX]);
    *eps_abs = (float)(rel * (mx - mn));
    return EXACTZ_OK;
  });
}

exactz_status exactz_vulnerability(const float *f, const float *ghat, const int64_t dims[3],
                                   float eps_abs, int64_t out[5], uint32_t *sweeps,
                                   void *stream) {
  return guarded([&]() -> exactz_status {
    int64_t V = 0;
    if (!f || !ghat || !out) return EXACTZ_EINVAL;
    if (check_dims(dims, &V) != EXACTZ_OK) return EXACTZ_EINVAL;
    if (!std::isfinite(eps_abs) || !(eps_abs >= 0.0f)) return EXACTZ_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    Ctx C(s);
    C.V = V;
    C.init(dims);
    uint8_t *flags = C.arena.get<uint8_t>((size_t)(V + 3) & ~(size_t)3);
    uint16_t *smask = C.arena.get<uint16_t>(V);
    int32_t *dep = C.arena.get<int32_t>(V);
    CK(cudaMemsetAsync(flags, 0, (size_t)(V + 3) & ~(size_t)3, s));
    C.zero();
    const unsigned nb = (unsigned)blocks_for(V, 256);
    k_vuln_classify<<<nb, 256, 0, s>>>(f, ghat, C.G, eps_abs, flags, smask, C.cnt);
    k_vuln_init_dep<<<nb, 256, 0, s>>>(flags, (int)V, dep);
    g_launches += 2;
    CK(cudaGetLastError());
    C.read();
    const unsigned long long nseeds = C.hcnt[C_NSADDLE];
    uint32_t n = 0;
    for (;;) {  // sweeps to the fixpoint, checked every 4
      CK(cudaMemsetAsync(&C.cnt[C_CHANGED], 0, sizeof(unsigned long long), s));
      for (int k = 0; k < 4; ++k, ++n) {
        k_vuln_relax<<<nb, 256, 0, s>>>(smask, C.G, dep, C.cnt);
        g_launches++;
      }
      CK(cudaGetLastError());
      unsigned long long ch = 0;
      CK(cudaMemcpyAsync(&ch, &C.cnt[C_CHANGED], sizeof(ch), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (!ch) break;
      if (n > (uint32_t)V + 8) {
        set_err("exactz_vulnerability", "relaxation did not converge");
        throw Error{EXACTZ_ECUDA};
      }
    }
    C.zero();
    k_vuln_gr<<<nb, 256, 0, s>>>(smask, C.G, dep, flags);
    k_vuln_count<<<nb, 256, 0, s>>>(flags, dep, (int)V, C.cnt);
    g_launches += 2;
    CK(cudaGetLastError());
    C.read();
    out[0] = (int64_t)C.hcnt[C_KEYMAX];
    out[1] = (int64_t)C.hcnt[C_N1 + 0];
    out[2] = (int64_t)C.hcnt[C_N1 + 1];
    out[3] = (int64_t)C.hcnt[C_N1 + 2];
    out[4] = (int64_t)nseeds;
    if (sweeps) *sweeps = n;
    return EXACTZ_OK;
  });
}

// ------------------------------------------------------------ edit log (NEXT-4)
namespace {
// libzstd through dlopen (the image has the runtime library, no headers)
struct Zstd {
  void *h = nullptr;
  size_t (*bound)(size_t) = nullptr;
  size_t (*comp)(void *, size_t, const void *, size_t, int) = nullptr;
  size_t (*decomp)(void *, size_t, const void *, size_t) = nullptr;
  unsigned (*iserr)(size_t) = nullptr;
};
const Zstd *zstd() {
  static Zstd z = [] {
    Zstd t;
    t.h = dlopen("libzstd.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!t.h) return t;
    t.bound = (size_t(*)(size_t))dlsym(t.h, "ZSTD_compressBound");
    t.comp = (size_t(*)(void *, size_t, const void *, size_t, int))dlsym(t.h, "ZSTD_compress");
    t.decomp = (size_t(*)(void *, size_t, const void *, size_t))dlsym(t.h, "ZSTD_decompress");
    t.iserr = (unsigned (*)(size_t))dlsym(t.h, "ZSTD_isError");
    if (!t.bound || !t.comp || !t.decomp || !t.iserr) t.h = nullptr;
    return t;
  }();
  return z.h ? &z : nullptr;
}
struct ExceHeader {
  char magic[4];
  uint8_t version, codec;
  uint16_t reserved;
  float xi;
  uint32_t N;
  int64_t nx, ny, nz;
  uint64_t entries, payload, raw;
};
static_assert(sizeof(ExceHeader) == 64, "EXCE header is 64 bytes");
}  // namespace

exactz_status exactz_edit_log(const float *g_in, const float *out, const uint8_t *edit_counts,
                              const int64_t dims[3], float eps_abs, uint32_t N, int level,
                              uint8_t *buf, uint64_t *bytes, uint64_t *entries, void *stream) {
  return guarded([&]() -> exactz_status {
    int64_t V = 0;
    if (!g_in || !out || !edit_counts || !bytes) return EXACTZ_EINVAL;
    if (check_dims(dims, &V) != EXACTZ_OK) return EXACTZ_EINVAL;
    if (!std::isfinite(eps_abs) || !(eps_abs >= 0.0f)) return EXACTZ_EINVAL;
    if (N == 0) N = 5;
    if (N > 254 || level < 0) return EXACTZ_EINVAL;
    if (level > 0 && !zstd()) {
      set_err("exactz_edit_log", "libzstd.so.1 not available (use level 0)");
      return EXACTZ_EUNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    Arena A(s);
    const float delta = eps_abs / (float)N;
    uint8_t *kind = A.get<uint8_t>(V);
    k_edit_kind<<<blocks_for(V, 256), 256, 0, s>>>(g_in, out, edit_counts, V, delta, (int)N, kind);
    g_launches++;
    CK(cudaGetLastError());
    int64_t *idx = A.get<int64_t>(V), *nsel = A.get<int64_t>(1);
    cub::CountingInputIterator<int64_t> it(0);
    size_t tb = 0;
    CK(cub::DeviceSelect::If(nullptr, tb, it, idx, nsel, V, HasEntry{kind}, s));
    void *tmp = A.get<uint8_t>(tb);
    CK(cub::DeviceSelect::If(tmp, tb, it, idx, nsel, V, HasEntry{kind}, s));
    int64_t n = 0;
    CK(cudaMemcpyAsync(&n, nsel, sizeof(n), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<uint8_t> raw;
    if (n) {  // the raw payload is built on the GPU (lengths, scan, bytes)
      uint8_t *ek = A.get<uint8_t>(n);
      float *ev = A.get<float>(n);
      uint64_t *len = A.get<uint64_t>(n + 1), *pos = A.get<uint64_t>(n + 1);
      k_edit_gather<<<blocks_for(n, 256), 256, 0, s>>>(idx, n, kind, out, ek, ev);
      k_edit_len<<<blocks_for(n, 256), 256, 0, s>>>(idx, ek, n, len);
      g_launches += 2;
      CK(cudaGetLastError());
      CK(cudaMemsetAsync(len + n, 0, sizeof(uint64_t), s));
      size_t ts = 0;
      CK(cub::DeviceScan::ExclusiveSum(nullptr, ts, len, pos, n + 1, s));
      void *tsc = A.get<uint8_t>(ts);
      CK(cub::DeviceScan::ExclusiveSum(tsc, ts, len, pos, n + 1, s));
      uint64_t total_raw = 0;
      CK(cudaMemcpyAsync(&total_raw, pos + n, 8, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      uint8_t *draw = A.get<uint8_t>(total_raw);
      k_edit_write<<<blocks_for(n, 256), 256, 0, s>>>(idx, ek, ev, n, pos, draw);
      g_launches++;
      CK(cudaGetLastError());
      raw.resize(total_raw);
      CK(cudaMemcpyAsync(raw.data(), draw, total_raw, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
    }
    std::vector<uint8_t> pay;
    uint8_t codec = 0;
    if (level > 0 && !raw.empty()) {
      const Zstd *z = zstd();
      pay.resize(z->bound(raw.size()));
      const size_t r = z->comp(pay.data(), pay.size(), raw.data(), raw.size(), level);
      if (z->iserr(r)) {
        set_err("exactz_edit_log", "ZSTD_compress failed");
        return EXACTZ_ECUDA;
      }
      pay.resize(r);
      codec = 1;
    } else {
      pay.swap(raw);
      raw.assign(pay.begin(), pay.end());
    }
    ExceHeader h{};
    std::memcpy(h.magic, "EXCE", 4);
    h.version = 1;
    h.codec = codec;
    h.xi = eps_abs;
    h.N = N;
    h.nx = dims[0];
    h.ny = dims[1];
    h.nz = dims[2];
    h.entries = (uint64_t)n;
    h.payload = pay.size();
    h.raw = raw.size();
    const uint64_t total = sizeof(h) + pay.size();
    if (entries) *entries = (uint64_t)n;
    if (!buf) {
      *bytes = total;
      return EXACTZ_OK;
    }
    if (*bytes < total) {
      *bytes = total;
      set_err("exactz_edit_log", "buffer too small (*bytes = size needed)");
      return EXACTZ_EINVAL;
    }
    std::memcpy(buf, &h, sizeof(h));
    if (!pay.empty()) std::memcpy(buf + sizeof(h), pay.data(), pay.size());
    *bytes = total;
    return EXACTZ_OK;
  });
}

exactz_status exactz_edit_log_apply(const uint8_t *buf, uint64_t bytes, const float *g_in,
                                    float *out, int64_t n_elems, void *stream) {
  return guarded([&]() -> exactz_status {
    if (!buf || !g_in || !out || bytes < sizeof(ExceHeader)) return EXACTZ_EINVAL;
    ExceHeader h;
    std::memcpy(&h, buf, sizeof(h));
    int64_t V = 0;
    const int64_t dims[3] = {h.nx, h.ny, h.nz};
    if (std::memcmp(h.magic, "EXCE", 4) || h.version != 1 || h.codec > 1 || h.N < 1 ||
        h.N > 254 || check_dims(dims, &V) != EXACTZ_OK || h.payload > bytes - sizeof(h) ||
        h.entries > (uint64_t)V || h.raw > (uint64_t)V * 15) {
      set_err("exactz_edit_log_apply", "malformed EXCE stream");
      return EXACTZ_EINVAL;
    }
    if (V != n_elems) {
      set_err("exactz_edit_log_apply", "stream dims do not match the caller's element count");
      return EXACTZ_EINVAL;
    }
    std::vector<uint8_t> raw;
    const uint8_t *pay = buf + sizeof(h);
    if (h.codec == 1) {
      const Zstd *z = zstd();
      if (!z) {
        set_err("exactz_edit_log_apply", "libzstd.so.1 not available");
        return EXACTZ_EUNSUPPORTED;
      }
      raw.resize(h.raw);
      const size_t r = z->decomp(raw.data(), raw.size(), pay, h.payload);
      if (z->iserr(r) || r != h.raw) {
        set_err("exactz_edit_log_apply", "corrupt zstd payload");
        return EXACTZ_EINVAL;
      }
    } else {
      if (h.payload != h.raw) return EXACTZ_EINVAL;
      raw.assign(pay, pay + h.payload);
    }
    std::vector<int64_t> hi;
    std::vector<uint8_t> hk;
    std::vector<float> hv;
    hi.reserve(h.entries);
    size_t p = 0;
    int64_t prev = -1;
    for (uint64_t e = 0; e < h.entries; ++e) {
      uint64_t d = 0;
      int sh = 0;
      for (;;) {
        if (p >= raw.size() || sh > 63) {
          set_err("exactz_edit_log_apply", "truncated EXCE payload");
          return EXACTZ_EINVAL;
        }
        const uint8_t b = raw[p++];
        d |= (uint64_t)(b & 0x7F) << sh;
        sh += 7;
        if (!(b & 0x80)) break;
      }
      // d <= V - 1 - (prev + 1) keeps i in [0, V) without signed overflow
      if (prev + 1 >= V || d > (uint64_t)(V - 1 - (prev + 1)) || p >= raw.size()) {
        set_err("exactz_edit_log_apply", "entry out of range or truncated");
        return EXACTZ_EINVAL;
      }
      const int64_t i = prev + 1 + (int64_t)d;
      if (i >= V) {
        set_err("exactz_edit_log_apply", "entry out of range or truncated");
        return EXACTZ_EINVAL;
      }
      prev = i;
      const uint8_t k = raw[p++];
      float v = 0.0f;
      if (k == 0) {
        if (p + 4 > raw.size()) {
          set_err("exactz_edit_log_apply", "truncated EXCE payload");
          return EXACTZ_EINVAL;
        }
        std::memcpy(&v, &raw[p], 4);
        p += 4;
      } else if (k > h.N) {
        set_err("exactz_edit_log_apply", "stepped count above N");
        return EXACTZ_EINVAL;
      }
      hi.push_back(i);
      hk.push_back(k);
      hv.push_back(v);
    }
    if (p != raw.size()) {
      set_err("exactz_edit_log_apply", "trailing bytes in the EXCE payload");
      return EXACTZ_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    Arena A(s);
    if (out != g_in) CK(cudaMemcpyAsync(out, g_in, V * sizeof(float), cudaMemcpyDeviceToDevice, s));
    const int64_t n = (int64_t)hi.size();
    if (n) {
      int64_t *di = A.get<int64_t>(n);
      uint8_t *dk = A.get<uint8_t>(n);
      float *dv = A.get<float>(n);
      CK(cudaMemcpyAsync(di, hi.data(), n * 8, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(dk, hk.data(), n, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(dv, hv.data(), n * 4, cudaMemcpyHostToDevice, s));
      k_edit_apply<<<blocks_for(n, 256), 256, 0, s>>>(di, dk, dv, n, g_in, out, h.xi / (float)h.N);
      g_launches++;
      CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(s));
    return EXACTZ_OK;
  });
}

exactz_status exactz_slab_range(int64_t nz, int nranks, int rank, int64_t *z_begin,
                                int64_t *z_count) {
  if (nz < 1 || nranks < 1 || rank < 0 || rank >= nranks || !z_begin || !z_count)
    return EXACTZ_EINVAL;
  slab_range(nz, nranks, rank, z_begin, z_count);
  return EXACTZ_OK;
}

exactz_status exactz_nccl_unique_id(uint8_t id[128]) {
  return guarded([&]() -> exactz_status {
    if (!id) return EXACTZ_EINVAL;
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    NK(ncclGetUniqueId(&u));
    std::memcpy(id, &u, 128);
    return EXACTZ_OK;
  });
}

exactz_status exactz_comm_init(const uint8_t id[128], int nranks, int rank, int cuda_device,
                               exactz_comm **out) {
  return guarded([&]() -> exactz_status {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return EXACTZ_EINVAL;
    CK(cudaSetDevice(cuda_device));
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    exactz_comm *c = new exactz_comm{nullptr, nranks, rank, cuda_device};
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
    if (r != ncclSuccess) {
      set_err("ncclCommInitRank", ncclGetErrorString(r));
      delete c;
      return EXACTZ_ENCCL;
    }
    *out = c;
    return EXACTZ_OK;
  });
}

exactz_status exactz_comm_destroy(exactz_comm *comm) {
  return guarded([&]() -> exactz_status {
    if (!comm) return EXACTZ_EINVAL;
    ncclResult_t r = ncclCommDestroy(comm->nccl);
    delete comm;
    if (r != ncclSuccess) {
      set_err("ncclCommDestroy", ncclGetErrorString(r));
      return EXACTZ_ENCCL;
    }
    return EXACTZ_OK;
  });
}

exactz_status exactz_correct_sharded(exactz_comm *comm, const float *f_local, const float *g_local,
                                     const int64_t global_dims[3], int64_t z_begin,
                                     int64_t z_count, float eps_abs, float *out_local,
                                     uint32_t *iters, const exactz_opts *opts, void *stream) {
  return guarded([&]() -> exactz_status {
    if (!comm || !f_local || !g_local || !out_local || !global_dims) return EXACTZ_EINVAL;
    int64_t z0 = 0, cnt = 0;
    slab_range(global_dims[2], comm->nranks, comm->rank, &z0, &cnt);
    if (z_begin != z0 || z_count != cnt) {
      set_err("exactz_correct_sharded", "slab does not match slab_range(nz, nranks, rank)");
      return EXACTZ_EINVAL;
    }
    NcclTransport T(comm, (cudaStream_t)stream);
    return sharded_impl(T, {f_local}, {g_local}, {out_local},
                        {opts ? opts->edit_counts : nullptr}, {opts ? opts->label_min : nullptr},
                        {opts ? opts->label_max : nullptr}, global_dims, eps_abs, iters, opts,
                        (cudaStream_t)stream);
  });
}

exactz_status exactz_correct_slabs(const float *f, const float *g_in, const int64_t dims[3],
                                   float eps_abs, int nslabs, float *out, uint32_t *iters,
                                   const exactz_opts *opts, void *stream) {
  return guarded([&]() -> exactz_status {
    int64_t V = 0;
    if (!f || !g_in || !out || nslabs < 1 || check_dims(dims, &V) != EXACTZ_OK)
      return EXACTZ_EINVAL;
    if (dims[2] < nslabs) return EXACTZ_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    Arena A(s);
    LoopTransport T(nslabs, s, A);
    std::vector<const float *> fi, gi;
    std::vector<float *> o;
    std::vector<uint8_t *> co;
    std::vector<int32_t *> ln, lx;
    const size_t P = (size_t)dims[0] * dims[1];
    for (int r = 0; r < nslabs; ++r) {
      int64_t z0 = 0, cnt = 0;
      slab_range(dims[2], nslabs, r, &z0, &cnt);
      fi.push_back(f + z0 * P);
      gi.push_back(g_in + z0 * P);
      o.push_back(out + z0 * P);
      co.push_back(opts && opts->edit_counts ? opts->edit_counts + z0 * P : nullptr);
      ln.push_back(opts && opts->label_min ? opts->label_min + z0 * P : nullptr);
      lx.push_back(opts && opts->label_max ? opts->label_max + z0 * P : nullptr);
    }
    return sharded_impl(T, fi, gi, o, co, ln, lx, dims, eps_abs, iters, opts, s);
  });
}

const char *exactz_strerror(exactz_status s) {
  switch (s) {
    case EXACTZ_OK: return "ok";
    case EXACTZ_EINVAL: return "invalid argument";
    case EXACTZ_EBOUND: return "input violates the error bound";
    case EXACTZ_ESTUCK: return "violations remain at a fixpoint or at max_iters";
    case EXACTZ_EUNSUPPORTED: return "unsupported";
    case EXACTZ_ECUDA: return "CUDA error";
    case EXACTZ_ENCCL: return "NCCL error";
    case EXACTZ_ENOMEM: return "out of memory";
  }
  return "unknown status";
}

const char *exactz_last_error(void) { return g_last_error.c_str(); }

uint64_t exactz_kernel_launches(void) { return g_launches.load(); }

const char *exactz_version(void) { return "exactz sm_100a " EXACTZ_GIT; }

}  // extern "C"

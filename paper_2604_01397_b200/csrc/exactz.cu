// exactz.cu — C ABI (include/exactz.h) and host orchestration of the B200
// EXaCTz correction loop.  Alg. 1:
//   validate (O1) -> reference of f (O7) -> loop { CheckConstraints (O8);
//   if no violation: stop; ApplyBoundedEdits (O9) }.
// All scratch lives in device memory allocated on the caller's stream; the
// host reads back 16 counters per round (termination, stats).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/exactz.h"
#include "kernels.cuh"

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

struct Ctx {
  cudaStream_t s;
  GridP G{};
  int64_t V = 0;
  dim3 sgrid, sblock;
  unsigned long long *cnt = nullptr;  // device counters
  unsigned long long *hcnt = nullptr; // pinned host mirror
  Arena arena;
  explicit Ctx(cudaStream_t st) : s(st), arena(st) {}
  ~Ctx() {
    if (hcnt) cudaFreeHost(hcnt);
  }
  void init(const int64_t dims[3]) {
    G.nx = (int)dims[0];
    G.ny = (int)dims[1];
    G.nz = (int)dims[2];
    G.V = (int)V;
    for (int s = 0; s < kSlots; ++s)
      G.delta[s] = kOff[s][0] + G.nx * (kOff[s][1] + G.ny * kOff[s][2]);
    sblock = dim3(128, 1, 1);
    sgrid = dim3((unsigned)((G.nx + 127) / 128), (unsigned)G.ny, (unsigned)G.nz);
    cnt = arena.get<unsigned long long>(C_NCOUNTERS);
    CK(cudaMallocHost(&hcnt, C_NCOUNTERS * sizeof(unsigned long long)));
  }
  void zero() { CK(cudaMemsetAsync(cnt, 0, C_NCOUNTERS * sizeof(unsigned long long), s)); }
  void read() {
    CK(cudaMemcpyAsync(hcnt, cnt, C_NCOUNTERS * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
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

// Resolve a pointer forest to its roots (O6).
static void resolve_labels(Ctx &C, int32_t *lab) {
  for (int round = 0; round < 64; ++round) {
    CK(cudaMemsetAsync(&C.cnt[C_CHANGED], 0, sizeof(unsigned long long), C.s));
    k_jump<<<blocks_for(C.V, 256), 256, 0, C.s>>>(lab, C.V, 8, C.cnt);
    CK(cudaGetLastError());
    unsigned long long ch = 0;
    CK(cudaMemcpyAsync(&ch, &C.cnt[C_CHANGED], sizeof(ch), cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
    if (!ch) return;
  }
  set_err("resolve_labels", "pointer jumping did not converge");
  throw Error{EXACTZ_ECUDA};
}

struct Reference {
  uint32_t *ref = nullptr;
  int32_t *labf_dn = nullptr, *labf_up = nullptr;
  int32_t *S = nullptr, *J = nullptr, *P = nullptr, *m1 = nullptr, *M1 = nullptr;
  int nS = 0, nJ = 0, nP = 0;
};

// O7: reference topology of f, computed once per call.
static void build_reference(Ctx &C, const float *f, Reference &R) {
  int64_t V = C.V;
  R.ref = C.arena.get<uint32_t>(V);
  R.labf_dn = C.arena.get<int32_t>(V);
  R.labf_up = C.arena.get<int32_t>(V);
  uint64_t *keys = C.arena.get<uint64_t>(V);
  C.zero();
  k_reference<<<C.sgrid, C.sblock, 0, C.s>>>(f, C.G, R.ref, R.labf_dn, R.labf_up, keys, C.cnt);
  CK(cudaGetLastError());
  C.read();
  R.nS = (int)C.hcnt[C_NSADDLE];
  resolve_labels(C, R.labf_dn);
  resolve_labels(C, R.labf_up);
  // saddles sorted by the SoS key of f
  uint64_t *sorted = C.arena.get<uint64_t>(R.nS);
  R.S = C.arena.get<int32_t>(R.nS);
  R.J = C.arena.get<int32_t>(R.nS);
  R.P = C.arena.get<int32_t>(R.nS);
  int *nsel = C.arena.get<int>(2);
  if (R.nS > 0) {
    size_t tb = 0, tb2 = 0, tb3 = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys, sorted, R.nS, 0, 64, C.s));
    CK(cub::DeviceSelect::If(nullptr, tb2, R.S, R.J, nsel, R.nS, IsJoin{R.ref}, C.s));
    CK(cub::DeviceSelect::If(nullptr, tb3, R.S, R.P, nsel + 1, R.nS, IsSplit{R.ref}, C.s));
    size_t tmax = tb > tb2 ? tb : tb2;
    tmax = tmax > tb3 ? tmax : tb3;
    void *tmp = C.arena.get<uint8_t>(tmax);
    CK(cub::DeviceRadixSort::SortKeys(tmp, tb, keys, sorted, R.nS, 0, 64, C.s));
    k_keys_to_ids<<<blocks_for(R.nS, 256, 1 << 30), 256, 0, C.s>>>(sorted, R.S, R.nS);
    CK(cudaGetLastError());
    CK(cub::DeviceSelect::If(tmp, tb2, R.S, R.J, nsel, R.nS, IsJoin{R.ref}, C.s));
    CK(cub::DeviceSelect::If(tmp, tb3, R.S, R.P, nsel + 1, R.nS, IsSplit{R.ref}, C.s));
    int h[2];
    CK(cudaMemcpyAsync(h, nsel, sizeof(h), cudaMemcpyDeviceToHost, C.s));
    CK(cudaStreamSynchronize(C.s));
    R.nJ = h[0];
    R.nP = h[1];
  }
  R.m1 = C.arena.get<int32_t>(R.nJ);
  R.M1 = C.arena.get<int32_t>(R.nP);
  if (R.nJ)
    k_event_reference<<<blocks_for(R.nJ, 128, 1 << 30), 128, 0, C.s>>>(
        f, R.ref, R.labf_dn, R.J, R.nJ, 1, R.m1, C.G);
  if (R.nP)
    k_event_reference<<<blocks_for(R.nP, 128, 1 << 30), 128, 0, C.s>>>(
        f, R.ref, R.labf_up, R.P, R.nP, 0, R.M1, C.G);
  CK(cudaGetLastError());
}

struct PassOut {
  unsigned long long vt, applied, n[6];
  bool ptr_mismatch;
};

// One CheckConstraints pass on g (O8) followed by the count and, when
// do_edit, the bounded edits (O9).  lab_dn/lab_up receive the g pointer
// forests (resolved when they differ from f's).
static PassOut detect_and_edit(Ctx &C, const Reference &R, const float *f, float *g, uint8_t *c,
                               uint8_t *mark, int32_t *lab_dn, int32_t *lab_up, float xi,
                               float delta, int N, uint32_t flags, bool do_edit,
                               const int32_t **lab_used_dn, const int32_t **lab_used_up) {
  bool c3 = !(flags & EXACTZ_NO_C3);
  C.zero();
  k_stencil<<<C.sgrid, C.sblock, 0, C.s>>>(g, R.ref, mark, lab_dn, lab_up, 1, C.G, C.cnt);
  CK(cudaGetLastError());
  if (!(flags & EXACTZ_NO_C2) && R.nS > 1)
    k_saddle_order<<<blocks_for(R.nS, 256, 1 << 30), 256, 0, C.s>>>(g, R.S, R.nS, mark, C.cnt);
  CK(cudaGetLastError());
  C.read();
  bool mismatch_dn = C.hcnt[C_N1 + 1] != 0, mismatch_up = C.hcnt[C_N1 + 0] != 0;
  // Labels of g equal those of f exactly when no steepest pointer differs.
  const int32_t *ldn = R.labf_dn, *lup = R.labf_up;
  if (mismatch_dn) {
    resolve_labels(C, lab_dn);
    ldn = lab_dn;
  }
  if (mismatch_up) {
    resolve_labels(C, lab_up);
    lup = lab_up;
  }
  if (c3) {
    if (R.nJ)
      k_events<<<blocks_for(R.nJ, 128, 1 << 30), 128, 0, C.s>>>(g, R.J, R.nJ, ldn, R.m1, 0, mark,
                                                                C.G, C.cnt);
    if (R.nP)
      k_events<<<blocks_for(R.nP, 128, 1 << 30), 128, 0, C.s>>>(g, R.P, R.nP, lup, R.M1, 1, mark,
                                                                C.G, C.cnt);
    CK(cudaGetLastError());
  }
  k_count_edit<<<blocks_for(C.V, 256), 256, 0, C.s>>>(g, c, mark, f, C.V, xi, delta, N,
                                                       do_edit ? 1 : 0, C.cnt);
  CK(cudaGetLastError());
  C.read();
  PassOut o;
  o.vt = C.hcnt[C_VT];
  o.applied = C.hcnt[C_APPLIED];
  for (int k = 0; k < 6; ++k) o.n[k] = C.hcnt[C_N1 + k];
  o.ptr_mismatch = mismatch_dn || mismatch_up;
  if (lab_used_dn) *lab_used_dn = ldn;
  if (lab_used_up) *lab_used_up = lup;
  return o;
}

static void validate_inputs(Ctx &C, const float *f, const float *g, float xi) {
  C.zero();
  k_validate<<<blocks_for(C.V, 256), 256, 0, C.s>>>(f, g, C.V, xi, C.cnt);
  CK(cudaGetLastError());
  C.read();
  if (C.hcnt[C_BAD_NF]) {
    set_err("validate", "non-finite value in f or g");
    throw Error{EXACTZ_EINVAL};
  }
  if (C.hcnt[C_BAD_BOUND]) {
    set_err("validate", "|f - g| > eps for some vertex");
    throw Error{EXACTZ_EBOUND};
  }
}

static exactz_status correct_impl(const float *f, const float *g_in, const int64_t dims[3],
                                  float eps, float *out, uint32_t *iters, const exactz_opts *opts,
                                  cudaStream_t s) {
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
  C.init(dims);
  cudaEvent_t e0, e1, e2;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  CK(cudaEventRecord(e0, s));
  validate_inputs(C, f, g_in, eps);
  if (out != g_in) CK(cudaMemcpyAsync(out, g_in, V * sizeof(float), cudaMemcpyDeviceToDevice, s));
  Reference R;
  build_reference(C, f, R);
  uint8_t *c = (opts && opts->edit_counts) ? opts->edit_counts : C.arena.get<uint8_t>(V);
  uint8_t *mark = C.arena.get<uint8_t>(V);
  int32_t *lab_dn = C.arena.get<int32_t>(V), *lab_up = C.arena.get<int32_t>(V);
  CK(cudaMemsetAsync(c, 0, V, s));
  CK(cudaMemsetAsync(mark, 0, V, s));
  CK(cudaEventRecord(e1, s));

  const float delta = eps / (float)N;  // Delta = RN(xi / N)
  uint32_t it = 0, rows = 0;
  exactz_status st = EXACTZ_OK;
  const int32_t *ldn = R.labf_dn, *lup = R.labf_up;
  for (;;) {
    bool may_edit = !(max_iters && it >= max_iters);
    PassOut o = detect_and_edit(C, R, f, out, c, mark, lab_dn, lab_up, eps, delta, N, flags,
                                may_edit, &ldn, &lup);
    if (stats && stats->rows && rows < stats->cap) {
      exactz_iter_stats &r = stats->rows[rows];
      r.violations = o.vt;
      r.applied = o.applied;
      for (int k = 0; k < 6; ++k) r.n[k] = o.n[k];
    }
    ++rows;
    if (o.vt == 0) break;
    if (!may_edit || o.applied == 0) {
      st = EXACTZ_ESTUCK;
      break;
    }
    ++it;
  }
  CK(cudaEventRecord(e2, s));
  // labels of the final field: the last pass ran on it (no edit followed)
  if (opts && opts->label_min)
    CK(cudaMemcpyAsync(opts->label_min, ldn, V * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  if (opts && opts->label_max)
    CK(cudaMemcpyAsync(opts->label_max, lup, V * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  CK(cudaStreamSynchronize(s));
  if (stats) {
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, e0, e1);
    cudaEventElapsedTime(&b, e1, e2);
    stats->ms_setup = a;
    stats->ms_loop = b;
    stats->nrows = rows;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  *iters = it;
  return st;
}

}  // namespace exz

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
    CK(cudaMemcpyAsync(df, f_host, V * sizeof(float), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(dg, g_in_host, V * sizeof(float), cudaMemcpyHostToDevice, s));
    exactz_opts o{};
    if (opts_host) o = *opts_host;
    if (o.edit_counts) o.edit_counts = A.get<uint8_t>(V);
    if (o.label_min) o.label_min = A.get<int32_t>(V);
    if (o.label_max) o.label_max = A.get<int32_t>(V);
    exactz_status st = correct_impl(df, dg, dims, eps_abs, dg, iters, &o, s);
    if (st != EXACTZ_OK && st != EXACTZ_ESTUCK) return st;
    CK(cudaMemcpyAsync(out_host, dg, V * sizeof(float), cudaMemcpyDeviceToHost, s));
    if (opts_host && opts_host->edit_counts)
      CK(cudaMemcpyAsync(opts_host->edit_counts, o.edit_counts, V, cudaMemcpyDeviceToHost, s));
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
    validate_inputs(C, f, g, eps_abs);
    Reference R;
    build_reference(C, f, R);
    uint8_t *mark = C.arena.get<uint8_t>(V);
    int32_t *lab_dn = C.arena.get<int32_t>(V), *lab_up = C.arena.get<int32_t>(V);
    CK(cudaMemsetAsync(mark, 0, V, s));
    PassOut o = detect_and_edit(C, R, f, const_cast<float *>(g), nullptr, mark, lab_dn, lab_up,
                                eps_abs, 0.0f, 5, flags, false, nullptr, nullptr);
    *violations = o.vt;
    if (row) {
      row->violations = o.vt;
      row->applied = 0;
      for (int k = 0; k < 6; ++k) row->n[k] = o.n[k];
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
    unsigned long long *cnt = A.get<unsigned long long>(C_NCOUNTERS);
    unsigned long long init[C_NCOUNTERS] = {};
    init[C_KEYMIN] = 0xffffffffull;
    CK(cudaMemcpyAsync(cnt, init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_minmax<<<blocks_for(n, 256), 256, 0, s>>>(f, n, cnt);
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

exactz_status exactz_nccl_unique_id(uint8_t id[128]) {
  (void)id;
  set_err("exactz_nccl_unique_id", "sharded path not built");
  return EXACTZ_EUNSUPPORTED;
}
exactz_status exactz_comm_init(const uint8_t id[128], int nranks, int rank, int cuda_device,
                               exactz_comm **out) {
  (void)id; (void)nranks; (void)rank; (void)cuda_device; (void)out;
  set_err("exactz_comm_init", "sharded path not built");
  return EXACTZ_EUNSUPPORTED;
}
exactz_status exactz_comm_destroy(exactz_comm *comm) {
  (void)comm;
  return EXACTZ_EUNSUPPORTED;
}
exactz_status exactz_correct_sharded(exactz_comm *comm, const float *f_local, const float *g_local,
                                     const int64_t global_dims[3], int64_t z_begin,
                                     int64_t z_count, float eps_abs, float *out_local,
                                     uint32_t *iters, const exactz_opts *opts, void *stream) {
  (void)comm; (void)f_local; (void)g_local; (void)global_dims; (void)z_begin; (void)z_count;
  (void)eps_abs; (void)out_local; (void)iters; (void)opts; (void)stream;
  set_err("exactz_correct_sharded", "sharded path not built");
  return EXACTZ_EUNSUPPORTED;
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

const char *exactz_version(void) { return "exactz sm_100a " EXACTZ_GIT; }

}  // extern "C"

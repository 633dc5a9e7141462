/*
 * exactz.h — C ABI of the B200 (sm_100a) EXaCTz topology-correction hot path.
 *
 * The operation (PAPER.md, arXiv 2604.01397):
 *   Alg. 1: given the original field f, its decompressed version
 *   f^ with |f_i - f^_i| <= xi and the bound xi, set g <- f^ and repeat
 *     S <- CheckConstraints(g, f)        (C1 P:284-290, C2 P:292-294,
 *                                         C3 P:297-302)
 *     if S is empty: stop
 *     g <- ApplyBoundedEdits(g, S, xi)   (one step Delta = xi/N down,
 *                                         lossless clamp f - xi after N steps)
 *   The returned field g (and the per-vertex edit counts = the edit set E)
 *   preserve the extremum graph and the join/split trees of f.
 *
 * Exact semantics (bit-level) are SURVEY.md §8(c) O0-O10 with the readings
 * listed in DESIGN.md §3; the CPU oracle (oracle/) implements the same
 * definition independently and the test suite checks bit equality.
 *
 * Conventions common to every call
 *  - Grid: dims = {nx, ny, nz}; nz = 1 gives the 2D path, ny = nz = 1 a 1D
 *    path.  Linear index i = x + nx*(y + ny*z) (x fastest); V = nx*ny*nz must
 *    be < 2^31 (labels are int32 global ids).
 *  - Mesh: Freudenthal/Kuhn triangulation (14 neighbours, clipped at faces).
 *  - Order: Simulation of Simplicity (P:178 footnote): u < v iff
 *    h_u < h_v or (h_u == h_v and u < v), IEEE compares (-0 == +0).
 *  - Values: float32; every f and f^ value must be finite.
 *  - Ownership: the caller owns every buffer.  Scratch is allocated with
 *    cudaMallocAsync on `stream` and freed before return.  f and g_in are
 *    never written unless out == g_in (allowed).
 *  - Device pointers: unless a name ends in _host, array arguments are CUDA
 *    device pointers of the current device, 16-byte aligned.  `stream` is a
 *    cudaStream_t (NULL = legacy default stream).
 *  - Blocking: every call returns after the result is known on the host
 *    (*iters etc.); device outputs are complete in stream order.
 *  - Errors: no exception crosses the ABI.  Validation failures (EXACTZ_EINVAL,
 *    EXACTZ_EBOUND) return before anything is written to `out`.  CUDA errors
 *    map to EXACTZ_ECUDA, allocation failures to EXACTZ_ENOMEM; details in
 *    exactz_last_error() (thread-local).
 */
#ifndef EXACTZ_H
#define EXACTZ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  EXACTZ_OK = 0,
  EXACTZ_EINVAL = 2,       /* null pointer, bad dims, non-finite value, N out of range */
  EXACTZ_EBOUND = 3,       /* some f^_i outside [RU(f_i - xi), RD(f_i + xi)] */
  EXACTZ_ESTUCK = 4,       /* violations remain at a fixpoint or at max_iters (amb-17) */
  EXACTZ_EUNSUPPORTED = 5, /* requested mode not built */
  EXACTZ_ECUDA = 6,
  EXACTZ_ENCCL = 7,
  EXACTZ_ENOMEM = 8
} exactz_status;

/* flags */
#define EXACTZ_NO_C2 0x1u   /* debug: skip the saddle-ordering rule (C2, R4) */
#define EXACTZ_NO_C3 0x2u   /* debug: skip the event rules (C3, R5/R6) */
#define EXACTZ_PROFILE 0x4u /* time every kernel class with CUDA events on `stream`
                               (exactz_stats.kernel_ms); results are unchanged */
#define EXACTZ_NO_TRACK 0x8u /* debug: dense passes only (no change tracking; results
                                are identical) */
#define EXACTZ_REFORMULATED 0x10u /* reformulated event constraints: the
                                     f-order of ALL critical points is checked on
                                     adjacent pairs (rule R7, counted in n[4]) instead
                                     of the label-based C3 rules R5/R6 */

/* kernel classes reported by EXACTZ_PROFILE */
enum {
  EXACTZ_K_VALIDATE = 0, /* bound check (O1) */
  EXACTZ_K_REFERENCE,    /* reference of f: classify, sort saddles, m1/M1 (O7) */
  EXACTZ_K_STENCIL,      /* R1-R3 + steepest slots, per round (O8) */
  EXACTZ_K_SADDLE_ORDER, /* R4 (C2) */
  EXACTZ_K_EVENTS,       /* R5/R6 (C3) incl. the label walks (O6) */
  EXACTZ_K_EDIT,         /* count + bounded edits (O9) */
  EXACTZ_K_LABELS,       /* full label outputs (pointer jumping) */
  EXACTZ_K_SPARSE,       /* sparse R1-R3 passes over the active vertices (tracking) */
  EXACTZ_K_CLASSES = 8
};

/* One row per CheckConstraints pass (the last row is the clean pass on OK). */
typedef struct {
  uint64_t violations; /* V_t: distinct vertices marked for an edit */
  uint64_t applied;    /* edits applied this round (marked and not yet at f - xi) */
  uint64_t n[6];       /* per-rule counts: R1 max-neighbour, R2 min-neighbour,
                          R3 flipped (vertex, link-vertex) pairs at saddles / type
                          changes, R4 flipped adjacent saddles, R5 join events
                          (R7 flipped adjacent critical points when REFORMULATED),
                          R6 split events */
  uint64_t walk_steps; /* diagnostics: steps of the C3 label walks (0 when not counted) */
  uint64_t evaluated;  /* vertices the stencil evaluated this pass (V for a dense pass, the
                          active set of a change-tracked one; SURVEY 8(d) per-pass bytes) */
  uint64_t links;      /* link vertices the C3 walks started from this pass (join: |L_g(s)|,
                          split: |U_g(s)|, summed over the saddles walked) */
  double ms;           /* GPU span of the pass on `stream` (CUDA events; exactz_correct
                          only, 0 elsewhere): detection, edits and the counter read */
} exactz_iter_stats;

typedef struct {
  exactz_iter_stats *rows; /* HOST array of `cap` rows, may be NULL */
  uint32_t cap;
  uint32_t nrows;          /* out: number of detection passes (may exceed cap) */
  double ms_setup;         /* out: validate + reference setup (CUDA events) */
  double ms_loop;          /* out: all iterations */
  /* EXACTZ_PROFILE only: per kernel class (EXACTZ_K_*), summed over the call */
  double kernel_ms[EXACTZ_K_CLASSES];       /* CUDA-event time on `stream` */
  uint64_t kernel_launches[EXACTZ_K_CLASSES];
  uint64_t kernel_bytes[EXACTZ_K_CLASSES];  /* algorithmic bytes */
  uint64_t n_saddles;      /* out: |S|, f-saddles (O7; exactz_correct only) */
  uint64_t n_join, n_split; /* out: |J|, |P| */
} exactz_stats;

typedef struct {
  uint32_t N;            /* steps before the lossless clamp; 0 => 5; <= 254 */
  uint32_t max_iters;    /* 0 => none: the loop ends at a fixpoint */
  uint32_t flags;        /* EXACTZ_NO_C2 | EXACTZ_NO_C3 */
  uint8_t *edit_counts;  /* optional out [V]: c_i in 0..N+1, N+1 == stored losslessly */
  int32_t *label_min;    /* optional out [V]: steepest-descent terminus of i in out */
  int32_t *label_max;    /* optional out [V]: steepest-ascent terminus of i in out */
  exactz_stats *stats;   /* optional HOST struct */
} exactz_opts;

/* The iterative correction (Alg. 1).  Returns EXACTZ_OK with zero violations
 * left, or EXACTZ_ESTUCK with out = the last g.  *iters (HOST) = number of
 * edit rounds (0 when f^ is already clean). */
exactz_status exactz_correct(const float *f, const float *g_in, const int64_t dims[3],
                             float eps_abs, float *out, uint32_t *iters,
                             const exactz_opts *opts, void *stream);

/* Same call with HOST buffers (f_host, g_in_host, out_host and the optional
 * opts arrays are host memory; pinned memory is fastest).  The host<->device
 * copies are part of the call. */
exactz_status exactz_correct_host(const float *f_host, const float *g_in_host,
                                  const int64_t dims[3], float eps_abs, float *out_host,
                                  uint32_t *iters, const exactz_opts *opts_host, void *stream);

/* One CheckConstraints(g, f) pass without editing: *violations (HOST)
 * = V_t, per-rule counts into row (HOST, may be NULL).  g must satisfy the
 * bound (else EXACTZ_EBOUND).  Used to verify a corrected field. */
exactz_status exactz_check(const float *f, const float *g, const int64_t dims[3], float eps_abs,
                           uint64_t *violations, exactz_iter_stats *row, uint32_t flags,
                           void *stream);

/* The Theorem 1 bound at full size:
 * the weak / strong / reduced vulnerability graphs of (f, ghat) over mesh
 * edges oriented u -> v when v <_f u (weak: f_u - f_v <= 2 eps; strong: weak
 * and ghat_v >= f_u - eps, both exact in double; seed: strong and u <_ghat v)
 * and D_max, the most vertices on a path of G_R from a seed endpoint, so
 * that iterations <= N * D_max.  f, ghat: device, layout as exactz_correct
 * (not validated against the bound).  out (HOST) = {D_max, |V(G_V)|,
 * |V(G_S)|, |V(G_R)|, #seed edges}; *sweeps (HOST, may be NULL) = relaxation
 * sweeps to the fixpoint.  Scratch ~7 bytes per vertex, freed on return. */
exactz_status exactz_vulnerability(const float *f, const float *ghat, const int64_t dims[3],
                                   float eps_abs, int64_t out[5], uint32_t *sweeps,
                                   void *stream);

/* The edit set E of a correction as a compact log (Alg. 1 "E"; P:178
 * lossless edits; P:433 edits compressed losslessly).
 * g_in, out, edit_counts: DEVICE, as given to / returned by exactz_correct
 * (out = corrected field, edit_counts = opts.edit_counts).  Entries: every
 * vertex with edit_counts > 0, in index order, as Stepped(k) when out equals
 * k sequential steps RN(g - Delta) from g_in (Delta = RN(eps/N)), else
 * Lossless(out value, the clamp RU(f - eps)).  Byte format "EXCE" v1
 * (editlog.cuh): 64-byte header, then varint index gaps, a kind byte and the
 * 4 value bytes of lossless entries; level > 0 compresses that payload with
 * zstd at that level (libzstd.so.1 loaded at run time; EXACTZ_EUNSUPPORTED
 * when absent).  buf (HOST) may be NULL: *bytes (HOST) then receives the
 * size; else *bytes is the capacity on entry (EXACTZ_EINVAL and the size
 * needed when too small) and the size written on return.  *entries (HOST,
 * may be NULL) = number of entries. */
exactz_status exactz_edit_log(const float *g_in, const float *out, const uint8_t *edit_counts,
                              const int64_t dims[3], float eps_abs, uint32_t N, int level,
                              uint8_t *buf, uint64_t *bytes, uint64_t *entries, void *stream);

/* Decode an EXCE stream (buf, bytes: HOST) and apply it to g_in (DEVICE):
 * out (DEVICE, may alias g_in) = g_in with every entry replayed (Stepped) or
 * stored (Lossless).  n_elems = the element count of g_in and out; it must
 * equal nx*ny*nz of the stream's header.  The stream is untrusted input:
 * EXACTZ_EINVAL on a malformed or truncated stream, a header whose sizes do
 * not fit `bytes`, an index gap past the end of the field or a dims mismatch,
 * always before any device write.
 * Format note: the header is this library's own (64 bytes: magic "EXCE",
 * version, codec, xi as float32 — the ABI's eps type —, N, the dims, entry
 * count, payload and raw sizes); SPEC's CPU program writes xi as f64 in a
 * shorter header, so the two streams are not interchangeable byte for byte
 * (NEXT-4). */
exactz_status exactz_edit_log_apply(const uint8_t *buf, uint64_t bytes, const float *g_in,
                                    float *out, int64_t n_elems, void *stream);

/* xi = RN_f32(rel * (max f - min f)) computed in double (amb-19). */
exactz_status exactz_eps_from_relative(const float *f, int64_t n, double rel, float *eps_abs,
                                       void *stream);

/* Sharded variant: z-slabs, one rank per GPU, NCCL over NVLink.  Collective:
 * every rank calls with identical scalars.  `id` is 128 bytes from
 * exactz_nccl_unique_id on rank 0, broadcast by the caller. */
typedef struct exactz_comm exactz_comm;
/* The z-slab of `rank` in an nz-plane field over `nranks` ranks: planes
 * [*z_begin, *z_begin + *z_count); the first nz % nranks ranks get one extra. */
exactz_status exactz_slab_range(int64_t nz, int nranks, int rank, int64_t *z_begin,
                                int64_t *z_count);
exactz_status exactz_nccl_unique_id(uint8_t id[128]);
exactz_status exactz_comm_init(const uint8_t id[128], int nranks, int rank, int cuda_device,
                               exactz_comm **out);
exactz_status exactz_comm_destroy(exactz_comm *comm);
/* f_local / g_local / out_local: the z_count planes [z_begin, z_begin+z_count)
 * of the global field (global_dims = {nx, ny, nz}); rank r must own exactly
 * the planes of the split "the first nz % nranks ranks get one extra plane"
 * (else EXACTZ_EINVAL).  edit_counts, label_min and label_max cover the local
 * planes (labels are global vertex ids, equal to exactz_correct's).  out_local is bit-equal to
 * the same planes of the single-GPU out; *iters identical on every rank. */
exactz_status exactz_correct_sharded(exactz_comm *comm, const float *f_local,
                                     const float *g_local, const int64_t global_dims[3],
                                     int64_t z_begin, int64_t z_count, float eps_abs,
                                     float *out_local, uint32_t *iters, const exactz_opts *opts,
                                     void *stream);

/* Single-process slab decomposition: runs the sharded algorithm with
 * `nslabs` virtual ranks on the current device (loopback transport instead of
 * NCCL); f, g_in, out are whole-field device buffers.  Validates the sharded
 * path on one GPU: out (and edit_counts, label_min, label_max: whole-field
 * buffers) is bit-equal to exactz_correct's. */
exactz_status exactz_correct_slabs(const float *f, const float *g_in, const int64_t dims[3],
                                   float eps_abs, int nslabs, float *out, uint32_t *iters,
                                   const exactz_opts *opts, void *stream);

const char *exactz_strerror(exactz_status s);
const char *exactz_last_error(void);
/* Number of this library's own kernels launched by the calling process so far
 * (diagnostic; library kernels such as CUB's sort are not counted). */
uint64_t exactz_kernel_launches(void);

/* build identification, e.g. "exactz sm_100a <git-describe>" */
const char *exactz_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EXACTZ_H */

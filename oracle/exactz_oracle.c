/*
 * exactz_oracle.c — the CPU ORACLE for the EXaCTz topology-correction loop.
 *
 *   *** TEST INFRASTRUCTURE ONLY. ***
 *   Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 *   --impl reference legs may load this library.  The product path
 *   (paper_2604_01397_b200/) never imports, links or executes it, and this file
 *   shares no code, header, table or constant generator with the CUDA path.
 *
 * Plain, slow, single-threaded C.  Every function follows the paper
 * (/root/reference/PAPER.md, cited as P:<line> §<section>) in its own order and
 * notation, with the readings of SURVEY.md §8(c) (amb-N) where the paper is
 * silent; DESIGN.md §3 lists every reading.  Floating point is IEEE binary32
 * (the configs are float32 fields, BASELINE.json), round-to-nearest-even, except
 * where RU/RD (directed rounding) is written; compiled -O2 -ffp-contract=off,
 * no fast-math.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (see the "Pinned by" line of each); none is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL 2
#define ORC_EBOUND 3
#define ORC_ESTUCK 4
#define ORC_ENOMEM 8

#define ORC_NO_C2 1u    /* debug: skip rule R4 (C2) */
#define ORC_NO_C3 2u    /* debug: skip rules R5/R6 (C3) */
#define ORC_REFORM 16u  /* reformulated event constraints: R7 instead of R5/R6 */

#define CLS_REGULAR 0
#define CLS_MIN 1
#define CLS_MAX 2
#define CLS_SADDLE 3

typedef struct {
  int64_t nx, ny, nz, V;
} Grid;

/* ------------------------------------------------------------------------ */
/* O3. Mesh: Freudenthal / Kuhn triangulation (amb-1).      */
/* Neighbour offsets D = { d, -d : d in {0,1}^3 \ {0} } (14 offsets).         */
/* Pinned by: test_oracle_mesh.py (SPEC S:47-49 examples, symmetry, Euler     */
/* characteristic 14-36+24=2, plane restriction = 6-cycle).                   */
/* ------------------------------------------------------------------------ */
static int OFF[14][3];
static int LINK_ADJ[14][14];
static int mesh_ready = 0;

static int is_nonneg(const int *a) { return a[0] >= 0 && a[1] >= 0 && a[2] >= 0; }

/* Two link vertices a, b of the centre 0 are adjacent iff {0, a, b} is a
 * triangle of the Kuhn subdivision, i.e. {0,a,b} lies on one chain:
 *   same sign     -> a and b are componentwise comparable;
 *   opposite sign -> the positive one and the negation of the negative one
 *                    have disjoint supports. */
static int kuhn_adjacent(const int *a, const int *b) {
  int sa = is_nonneg(a), sb = is_nonneg(b);
  if (sa == sb) {
    int a_le_b = 1, b_le_a = 1;
    for (int c = 0; c < 3; c++) {
      int x = abs(a[c]), y = abs(b[c]);
      if (x > y) a_le_b = 0;
      if (y > x) b_le_a = 0;
    }
    return a_le_b || b_le_a;
  }
  for (int c = 0; c < 3; c++)
    if (a[c] != 0 && b[c] != 0) return 0;
  return 1;
}

static void init_mesh(void) {
  if (mesh_ready) return;
  int k = 0;
  for (int dz = 0; dz <= 1; dz++)
    for (int dy = 0; dy <= 1; dy++)
      for (int dx = 0; dx <= 1; dx++) {
        if (!dx && !dy && !dz) continue;
        OFF[k][0] = dx; OFF[k][1] = dy; OFF[k][2] = dz;
        OFF[k + 7][0] = -dx; OFF[k + 7][1] = -dy; OFF[k + 7][2] = -dz;
        k++;
      }
  for (int a = 0; a < 14; a++)
    for (int b = 0; b < 14; b++) LINK_ADJ[a][b] = (a != b) && kuhn_adjacent(OFF[a], OFF[b]);
  mesh_ready = 1;
}

/* Lk(v): the clipped neighbours of v, in ascending linear index.
 * nb[j] = neighbour id, ko[j] = which of the 14 offsets it is. */
static int neighbors(const Grid *G, int64_t v, int64_t *nb, int *ko) {
  int64_t x = v % G->nx, y = (v / G->nx) % G->ny, z = v / (G->nx * G->ny);
  int n = 0;
  for (int k = 0; k < 14; k++) {
    int64_t a = x + OFF[k][0], b = y + OFF[k][1], c = z + OFF[k][2];
    if (a < 0 || b < 0 || c < 0 || a >= G->nx || b >= G->ny || c >= G->nz) continue;
    nb[n] = a + G->nx * (b + G->ny * c);
    ko[n] = k;
    n++;
  }
  for (int i = 1; i < n; i++) /* insertion sort by id */
    for (int j = i; j > 0 && nb[j - 1] > nb[j]; j--) {
      int64_t t = nb[j]; nb[j] = nb[j - 1]; nb[j - 1] = t;
      int s = ko[j]; ko[j] = ko[j - 1]; ko[j - 1] = s;
    }
  return n;
}

/* ------------------------------------------------------------------------ */
/* O2. Simulation of Simplicity (§3.3 footnote): equal values are       */
/* ordered by global index, the larger index being larger.  IEEE compares.   */
/* Pinned by: test_oracle_mesh.py::test_sos_examples.          */
/* ------------------------------------------------------------------------ */
static int sos_less(const float *h, int64_t u, int64_t v) {
  return h[u] < h[v] || (h[u] == h[v] && u < v);
}

/* ------------------------------------------------------------------------ */
/* O1. Directed rounding without rounding-mode state: TwoSum (exact error of  */
/* a float addition, in RN) then one ulp toward +/-inf when the rounding     */
/* error has the wrong sign.                                                  */
/* Pinned by: test_oracle_edit.py (exact rational comparison in Python).     */
/* ------------------------------------------------------------------------ */
static float two_sum_err(float a, float b, float s) {
  float bb = s - a;
  return (a - (s - bb)) + (b - bb);
}
float oracle_ru_sub(float a, float b) { /* RU(a - b) */
  float nb = -b;
  float s = a + nb;
  if (two_sum_err(a, nb, s) > 0.0f) s = nextafterf(s, INFINITY);
  return s;
}
float oracle_rd_add(float a, float b) { /* RD(a + b) */
  float s = a + b;
  if (two_sum_err(a, b, s) < 0.0f) s = nextafterf(s, -INFINITY);
  return s;
}

/* ------------------------------------------------------------------------ */
/* O4. Classification (§3.2 Step 1; fig:saddle_class P:150):       */
/* L(i) = {u in Lk(i): u < i}, U(i) = Lk(i) \ L(i); nlc, nuc = number of     */
/* connected components of the link graph induced on L and on U.  Extrema    */
/* take precedence (amb-5).                                                   */
/* Pinned by: test_oracle_topology.py (Alexander-duality identity            */
/* nlc - nuc + 1 = chi(L) on all 2^14 interior masks;        */
/* union-find minima count).                                                  */
/* ------------------------------------------------------------------------ */
static int count_components(int n, const int *ko, const int *in_set) {
  int seen[14] = {0}, stack[14], comps = 0;
  for (int s = 0; s < n; s++) {
    if (!in_set[s] || seen[s]) continue;
    comps++;
    int sp = 0;
    seen[s] = 1;
    stack[sp++] = s;
    while (sp) {
      int a = stack[--sp];
      for (int b = 0; b < n; b++)
        if (in_set[b] && !seen[b] && LINK_ADJ[ko[a]][ko[b]]) {
          seen[b] = 1;
          stack[sp++] = b;
        }
    }
  }
  return comps;
}

static void link_components(const Grid *G, const float *h, int64_t i, int *nlc, int *nuc) {
  int64_t nb[14];
  int ko[14], lower[14], upper[14];
  int n = neighbors(G, i, nb, ko);
  for (int j = 0; j < n; j++) {
    lower[j] = sos_less(h, nb[j], i);
    upper[j] = !lower[j];
  }
  *nlc = count_components(n, ko, lower);
  *nuc = count_components(n, ko, upper);
}

static int class_of(int nlc, int nuc) {
  if (nlc == 0) return CLS_MIN;
  if (nuc == 0) return CLS_MAX;
  if (nlc >= 2 || nuc >= 2) return CLS_SADDLE;
  return CLS_REGULAR;
}

/* ------------------------------------------------------------------------ */
/* O5. Steepest neighbours over the closed star St(i) = {i} u Lk(i)           */
/* (§3.1 "highest (or lowest) adjacent neighbor"; P:286 N_max/N_min;   */
/* amb-6: closed star so an extremum points to itself).                       */
/* Pinned by: test_oracle_topology.py (monotone closed forms; brute force).  */
/* ------------------------------------------------------------------------ */
static void steepest(const Grid *G, const float *h, int64_t i, int32_t *up, int32_t *dn) {
  int64_t nb[14];
  int ko[14];
  int n = neighbors(G, i, nb, ko);
  int64_t lo = i, hi = i;
  for (int j = 0; j < n; j++) {
    if (sos_less(h, nb[j], lo)) lo = nb[j];
    if (sos_less(h, hi, nb[j])) hi = nb[j];
  }
  *up = (int32_t)hi;
  *dn = (int32_t)lo;
}

/* ------------------------------------------------------------------------ */
/* O6. Labels: lab(i) = the fixpoint of i -> ptr(i) -> ... (the extremum the  */
/* integral path from i reaches).  Memoised path walks.         */
/* ------------------------------------------------------------------------ */
static void path_labels(int64_t V, const int32_t *ptr, int32_t *lab, int32_t *stack) {
  for (int64_t v = 0; v < V; v++) lab[v] = -1;
  for (int64_t v = 0; v < V; v++) {
    if (lab[v] >= 0) continue;
    int64_t sp = 0, w = v;
    while (lab[w] < 0 && ptr[w] != w) {
      stack[sp++] = (int32_t)w;
      w = ptr[w];
    }
    if (lab[w] < 0) lab[w] = (int32_t)w;
    int32_t root = lab[w];
    while (sp) lab[stack[--sp]] = root;
  }
}

/* ------------------------------------------------------------------------ */
/* O7. Reference topology of f, computed once.      */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint8_t *nlc, *nuc, *cls;
  int32_t *up, *dn, *lab_dn, *lab_up;
  int64_t nS, nJ, nP, nC;
  int32_t *S, *J, *P, *m1, *M1; /* m1 indexed like J, M1 like P */
  int32_t *CP;                  /* all critical points sorted by <_f (reformulation) */
} Ref;

static const float *sort_h; /* single-threaded qsort context */
static int cmp_sos_asc(const void *a, const void *b) {
  int32_t u = *(const int32_t *)a, v = *(const int32_t *)b;
  if (u == v) return 0;
  return sos_less(sort_h, u, v) ? -1 : 1;
}

static void free_ref(Ref *R) {
  free(R->nlc); free(R->nuc); free(R->cls); free(R->up); free(R->dn);
  free(R->lab_dn); free(R->lab_up); free(R->S); free(R->J); free(R->P);
  free(R->m1); free(R->M1); free(R->CP);
  memset(R, 0, sizeof(*R));
}

static int build_ref(const Grid *G, const float *f, Ref *R, int32_t *stack) {
  int64_t V = G->V;
  memset(R, 0, sizeof(*R));
  R->nlc = malloc(V); R->nuc = malloc(V); R->cls = malloc(V);
  R->up = malloc(4 * V); R->dn = malloc(4 * V);
  R->lab_dn = malloc(4 * V); R->lab_up = malloc(4 * V);
  if (!R->nlc || !R->nuc || !R->cls || !R->up || !R->dn || !R->lab_dn || !R->lab_up) {
    free_ref(R);
    return ORC_ENOMEM;
  }
  int64_t nS = 0, nJ = 0, nP = 0;
  for (int64_t i = 0; i < V; i++) {
    int a, b;
    link_components(G, f, i, &a, &b);
    R->nlc[i] = (uint8_t)a;
    R->nuc[i] = (uint8_t)b;
    R->cls[i] = (uint8_t)class_of(a, b);
    steepest(G, f, i, &R->up[i], &R->dn[i]);
    if (R->cls[i] == CLS_SADDLE) {
      nS++;
      if (a >= 2) nJ++; /* join saddle: lower link splits */
      if (b >= 2) nP++; /* split saddle: upper link splits */
    }
  }
  path_labels(V, R->dn, R->lab_dn, stack);
  path_labels(V, R->up, R->lab_up, stack);
  int64_t nC = 0;
  for (int64_t i = 0; i < V; i++) nC += (R->cls[i] != CLS_REGULAR);
  R->S = malloc(4 * (nS + 1)); R->J = malloc(4 * (nJ + 1)); R->P = malloc(4 * (nP + 1));
  R->m1 = malloc(4 * (nJ + 1)); R->M1 = malloc(4 * (nP + 1)); R->CP = malloc(4 * (nC + 1));
  if (!R->S || !R->J || !R->P || !R->m1 || !R->M1 || !R->CP) {
    free_ref(R);
    return ORC_ENOMEM;
  }
  /* Reformulation: "the reformulated event constraints preserve
   * the ordering of all critical points" -- every non-regular vertex of f,
   * sorted by <_f. */
  R->nC = nC;
  {
    int64_t c = 0;
    for (int64_t i = 0; i < V; i++)
      if (R->cls[i] != CLS_REGULAR) R->CP[c++] = (int32_t)i;
    sort_h = f;
    qsort(R->CP, nC, 4, cmp_sos_asc);
  }
  R->nS = nS; R->nJ = nJ; R->nP = nP;
  int64_t s = 0;
  for (int64_t i = 0; i < V; i++)
    if (R->cls[i] == CLS_SADDLE) R->S[s++] = (int32_t)i;
  /* S sorted ascending by the SoS order of f: "We compute saddle ordering in f
   * as the reference ordering".  J and P are taken in the same order. */
  sort_h = f;
  qsort(R->S, nS, 4, cmp_sos_asc);
  int64_t j = 0, p = 0;
  for (int64_t k = 0; k < nS; k++) {
    int32_t v = R->S[k];
    if (R->nlc[v] >= 2) R->J[j++] = v;
    if (R->nuc[v] >= 2) R->P[p++] = v;
  }
  /* m1(s) = the largest (under <_f) minimum reached from the lower link of s:
   * "the pair <i,s> is extracted if i is the largest minimum among all minima
   * connected to s".  M1(s) symmetric for split saddles. */
  int64_t nb[14];
  int ko[14];
  for (int64_t k = 0; k < nJ; k++) {
    int32_t sdl = R->J[k];
    int n = neighbors(G, sdl, nb, ko);
    int64_t best = -1;
    for (int q = 0; q < n; q++) {
      if (!sos_less(f, nb[q], sdl)) continue;
      int64_t m = R->lab_dn[nb[q]];
      if (best < 0 || sos_less(f, best, m)) best = m;
    }
    R->m1[k] = (int32_t)best;
  }
  for (int64_t k = 0; k < nP; k++) {
    int32_t sdl = R->P[k];
    int n = neighbors(G, sdl, nb, ko);
    int64_t best = -1;
    for (int q = 0; q < n; q++) {
      if (sos_less(f, nb[q], sdl)) continue;
      int64_t M = R->lab_up[nb[q]];
      if (best < 0 || sos_less(f, M, best)) best = M;
    }
    R->M1[k] = (int32_t)best;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* O8. CheckConstraints(g, f) (Alg. 1 line "S <- CheckConstraints(g,f)",     */
/* P:251) on a snapshot of g (Jacobi, amb-15).  Writes mark[] (0/1) and the  */
/* per-rule counts cnt[0..6] = {V_t, n1, n2, n3, n4, n5, n6}.                */
/* Work arrays: upg, dng, labdn, labup, stack of V int32 each.               */
/* Pinned by: tests/golden/edit_strategy_1x3.json (fig:edit_strategy),*/
/* SPEC C1/C2/C3 examples, and the post-correction recall tests.     */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t *upg, *dng, *labdn, *labup, *stack;
} Work;

static void detect(const Grid *G, const float *f, const Ref *R, const float *g, uint32_t flags,
                   uint8_t *mark, Work *W, int64_t cnt[7]) {
  int64_t V = G->V;
  for (int k = 0; k < 7; k++) cnt[k] = 0;
  memset(mark, 0, V);
  for (int64_t i = 0; i < V; i++) steepest(G, g, i, &W->upg[i], &W->dng[i]);

  int64_t nb[14];
  int ko[14];
  for (int64_t i = 0; i < V; i++) {
    /* R1: "If N^_max(i) != N_max(i), we decrease the value of N^_max(i)". */
    if (W->upg[i] != R->up[i]) {
      mark[W->upg[i]] = 1;
      cnt[1]++;
    }
    /* R2: "if N^_min(i) != N_min(i), we decrease the value of N_min(i)". */
    if (W->dng[i] != R->dn[i]) {
      mark[R->dn[i]] = 1;
      cnt[2]++;
    }
    /* R3 (P:290 + C1(1) P:220; amb-7, amb-8): at f-saddles, and wherever the
     * type T=(nlc,nuc) differs, every link vertex whose order against i flipped
     * is a violation; the target is the f-smaller endpoint. */
    int n = neighbors(G, i, nb, ko);
    int flipped[14], any = 0;
    for (int q = 0; q < n; q++) {
      flipped[q] = sos_less(g, nb[q], i) != sos_less(f, nb[q], i);
      any |= flipped[q];
    }
    if (!any) continue; /* no flipped pair: R3 has nothing to mark at i */
    int apply = (R->cls[i] == CLS_SADDLE);
    if (!apply) {
      int a, b;
      link_components(G, g, i, &a, &b);
      apply = (a != R->nlc[i]) || (b != R->nuc[i]);
    }
    if (!apply) continue;
    for (int q = 0; q < n; q++) {
      if (!flipped[q]) continue;
      cnt[3]++;
      if (sos_less(f, nb[q], i)) mark[nb[q]] = 1;
      else mark[i] = 1;
    }
  }

  /* R4 (C2; amb-9, amb-10): adjacent saddles a=S[k] <_f b=S[k+1];
   * "if f_i < f_j but g_i > g_j, we decrease g_i". */
  if (!(flags & ORC_NO_C2)) {
    for (int64_t k = 0; k + 1 < R->nS; k++) {
      int32_t a = R->S[k], b = R->S[k + 1];
      if (sos_less(g, b, a)) {
        mark[a] = 1;
        cnt[4]++;
      }
    }
  }

  /* R7 (reformulated C3): "each iteration only requires
   * exchanging the scalar value of each critical point with its immediate
   * predecessor and successor (determined by the sorted sequence in the
   * original data). Violations are detected by comparing the current
   * ordering with the original one ... and corrected by applying edits to
   * restore the correct order": adjacent a = CP[k] <_f b = CP[k+1]; if
   * b <_g a, decrease a (the f-smaller, as for C2).  Counted in cnt[5]. */
  if (!(flags & ORC_NO_C3) && (flags & ORC_REFORM)) {
    for (int64_t k = 0; k + 1 < R->nC; k++) {
      int32_t a = R->CP[k], b = R->CP[k + 1];
      if (sos_less(g, b, a)) {
        mark[a] = 1;
        cnt[5]++;
      }
    }
  }
  /* R5/R6 (C3; amb-11, amb-12): the extremum EGP selects for each
   * saddle, evaluated on the extremum graph of g (labels of g). */
  if (!(flags & ORC_NO_C3) && !(flags & ORC_REFORM)) {
    path_labels(V, W->dng, W->labdn, W->stack);
    path_labels(V, W->upg, W->labup, W->stack);
    for (int64_t k = 0; k < R->nJ; k++) {
      int32_t s = R->J[k];
      int n = neighbors(G, s, nb, ko);
      int64_t m2 = -1;
      for (int q = 0; q < n; q++) {
        if (!sos_less(g, nb[q], s)) continue;
        int64_t m = W->labdn[nb[q]];
        if (m2 < 0 || sos_less(g, m2, m)) m2 = m;
      }
      /* "we decrease g_{m2} to enforce g_{m2} < g_{m1}" */
      if (m2 >= 0 && m2 != R->m1[k]) {
        mark[m2] = 1;
        cnt[5]++;
      }
    }
    for (int64_t k = 0; k < R->nP; k++) {
      int32_t s = R->P[k];
      int n = neighbors(G, s, nb, ko);
      int64_t M2 = -1;
      for (int q = 0; q < n; q++) {
        if (sos_less(g, nb[q], s)) continue;
        int64_t M = W->labup[nb[q]];
        if (M2 < 0 || sos_less(g, M, M2)) M2 = M;
      }
      /* "The same argument applies to split events": under
       * decrease-only edits the fix is lowering the f-selected M1 (amb-12). */
      if (M2 >= 0 && M2 != R->M1[k]) {
        mark[R->M1[k]] = 1;
        cnt[6]++;
      }
    }
  }
  for (int64_t i = 0; i < V; i++) cnt[0] += mark[i];
}

/* ------------------------------------------------------------------------ */
/* O9. ApplyBoundedEdits (§3.3): one step of Delta = xi/N down,  */
/* never below lo = RU(f - xi); the (N+1)-th edit is the lossless clamp to    */
/* f - xi ("If a vertex i requires more than N edits, we store the edit in a */
/* lossless manner as the absolute lower bound").  Returns the number */
/* of applied edits (marked vertices not already at lo).                     */
/* Pinned by: test_oracle_edit.py (P-9).                     */
/* ------------------------------------------------------------------------ */
static int64_t apply_edits(int64_t V, const float *f, float xi, int N, const uint8_t *mark,
                           float *g, uint8_t *c) {
  float delta = xi / (float)N;
  int64_t applied = 0;
  for (int64_t i = 0; i < V; i++) {
    if (!mark[i]) continue;
    float lo = oracle_ru_sub(f[i], xi);
    if (g[i] == lo) continue; /* saturated: nothing left to do */
    if (c[i] < N) {
      float t = g[i] - delta;
      g[i] = (t < lo) ? lo : t;
    } else {
      g[i] = lo;
    }
    c[i]++;
    applied++;
  }
  return applied;
}

/* ------------------------------------------------------------------------ */
/* Public entry points (ctypes, see oracle/oracle.py).                       */
/* ------------------------------------------------------------------------ */
static int make_grid(Grid *G, int64_t nx, int64_t ny, int64_t nz) {
  if (nx < 1 || ny < 1 || nz < 1) return ORC_EINVAL;
  G->nx = nx; G->ny = ny; G->nz = nz; G->V = nx * ny * nz;
  if (G->V >= ((int64_t)1 << 31)) return ORC_EINVAL;
  init_mesh();
  return ORC_OK;
}

int oracle_offsets(int32_t *out /* [14*3] */) {
  init_mesh();
  for (int k = 0; k < 14; k++)
    for (int c = 0; c < 3; c++) out[3 * k + c] = OFF[k][c];
  return 14;
}

int oracle_link_adjacent(int a, int b) {
  init_mesh();
  if (a < 0 || b < 0 || a >= 14 || b >= 14) return -1;
  return LINK_ADJ[a][b];
}

/* components of an interior link subset given as a 14-bit mask over OFF order */
int oracle_mask_components(uint32_t mask) {
  init_mesh();
  int ko[14], in_set[14];
  for (int k = 0; k < 14; k++) {
    ko[k] = k;
    in_set[k] = (mask >> k) & 1u;
  }
  return count_components(14, ko, in_set);
}

int oracle_neighbors(int64_t nx, int64_t ny, int64_t nz, int64_t v, int64_t *out) {
  Grid G;
  if (make_grid(&G, nx, ny, nz) || v < 0 || v >= G.V) return -1;
  int ko[14];
  return neighbors(&G, v, out, ko);
}

int oracle_sos_less(const float *h, int64_t u, int64_t v) { return sos_less(h, u, v); }

int oracle_classify(const float *h, int64_t nx, int64_t ny, int64_t nz, uint8_t *nlc, uint8_t *nuc,
                    uint8_t *cls) {
  Grid G;
  if (make_grid(&G, nx, ny, nz)) return ORC_EINVAL;
  for (int64_t i = 0; i < G.V; i++) {
    int a, b;
    link_components(&G, h, i, &a, &b);
    nlc[i] = (uint8_t)a;
    nuc[i] = (uint8_t)b;
    cls[i] = (uint8_t)class_of(a, b);
  }
  return ORC_OK;
}

int oracle_steepest(const float *h, int64_t nx, int64_t ny, int64_t nz, int32_t *up, int32_t *dn) {
  Grid G;
  if (make_grid(&G, nx, ny, nz)) return ORC_EINVAL;
  for (int64_t i = 0; i < G.V; i++) steepest(&G, h, i, &up[i], &dn[i]);
  return ORC_OK;
}

int oracle_labels(const float *h, int64_t nx, int64_t ny, int64_t nz, int32_t *lab_dn, int32_t *lab_up) {
  Grid G;
  if (make_grid(&G, nx, ny, nz)) return ORC_EINVAL;
  int32_t *up = malloc(4 * G.V), *dn = malloc(4 * G.V), *st = malloc(4 * G.V);
  if (!up || !dn || !st) {
    free(up); free(dn); free(st);
    return ORC_ENOMEM;
  }
  for (int64_t i = 0; i < G.V; i++) steepest(&G, h, i, &up[i], &dn[i]);
  path_labels(G.V, dn, lab_dn, st);
  path_labels(G.V, up, lab_up, st);
  free(up); free(dn); free(st);
  return ORC_OK;
}

/* Reference lists of f: S (sorted saddles), J, P, m1, M1; counts in n[0..2].
 * Buffers must hold V entries each. */
int oracle_reference(const float *f, int64_t nx, int64_t ny, int64_t nz, int32_t *S, int32_t *J,
                     int32_t *P, int32_t *m1, int32_t *M1, int64_t *n) {
  Grid G;
  if (make_grid(&G, nx, ny, nz)) return ORC_EINVAL;
  int32_t *st = malloc(4 * G.V);
  if (!st) return ORC_ENOMEM;
  Ref R;
  int rc = build_ref(&G, f, &R, st);
  free(st);
  if (rc) return rc;
  memcpy(S, R.S, 4 * R.nS); memcpy(J, R.J, 4 * R.nJ); memcpy(P, R.P, 4 * R.nP);
  memcpy(m1, R.m1, 4 * R.nJ); memcpy(M1, R.M1, 4 * R.nP);
  n[0] = R.nS; n[1] = R.nJ; n[2] = R.nP;
  free_ref(&R);
  return ORC_OK;
}

static int alloc_work(int64_t V, Work *W) {
  W->upg = malloc(4 * V); W->dng = malloc(4 * V); W->labdn = malloc(4 * V);
  W->labup = malloc(4 * V); W->stack = malloc(4 * V);
  if (!W->upg || !W->dng || !W->labdn || !W->labup || !W->stack) {
    free(W->upg); free(W->dng); free(W->labdn); free(W->labup); free(W->stack);
    return ORC_ENOMEM;
  }
  return ORC_OK;
}
static void free_work(Work *W) {
  free(W->upg); free(W->dng); free(W->labdn); free(W->labup); free(W->stack);
}

/* One CheckConstraints pass: marks (V bytes) and cnt[7] = {V_t, n1..n6}. */
int oracle_check(const float *f, const float *g, int64_t nx, int64_t ny, int64_t nz, uint32_t flags,
                 uint8_t *mark, int64_t *cnt) {
  Grid G;
  if (make_grid(&G, nx, ny, nz)) return ORC_EINVAL;
  Work W;
  if (alloc_work(G.V, &W)) return ORC_ENOMEM;
  Ref R;
  int rc = build_ref(&G, f, &R, W.stack);
  if (rc) {
    free_work(&W);
    return rc;
  }
  detect(&G, f, &R, g, flags, mark, &W, cnt);
  free_ref(&R);
  free_work(&W);
  return ORC_OK;
}

/* O1 validation: finite inputs, xi finite >= 0, RU(f-xi) <= ghat <= RD(f+xi). */
int oracle_validate(const float *f, const float *ghat, int64_t V, float xi, int N) {
  if (!(xi >= 0.0f) || !isfinite(xi) || N < 1 || N > 254) return ORC_EINVAL;
  for (int64_t i = 0; i < V; i++)
    if (!isfinite(f[i]) || !isfinite(ghat[i])) return ORC_EINVAL;
  for (int64_t i = 0; i < V; i++) {
    float lo = oracle_ru_sub(f[i], xi), hi = oracle_rd_add(f[i], xi);
    if (!(lo <= ghat[i] && ghat[i] <= hi)) return ORC_EBOUND;
  }
  return ORC_OK;
}

/* Alg. 1: g <- f^; loop { S <- CheckConstraints(g,f); if S = {}
 * break; (g, dE) <- ApplyBoundedEdits(g,S,xi) }.
 * iters = number of edit rounds (amb-18).  ESTUCK when a round applies no edit
 * (fixpoint with violations left, amb-17) or when max_iters rounds were done
 * and violations remain.  stats (optional) gets one row of 8 int64 per
 * detection pass: {V_t, applied, n1, n2, n3, n4, n5, n6}. */
int oracle_correct(const float *f, const float *ghat, int64_t nx, int64_t ny, int64_t nz, float xi,
                   int N, uint32_t flags, uint32_t max_iters, float *out, uint8_t *counts,
                   int32_t *lab_min, int32_t *lab_max, uint32_t *iters_out, int64_t *stats,
                   int64_t stats_cap, int64_t *stats_rows) {
  Grid G;
  if (make_grid(&G, nx, ny, nz)) return ORC_EINVAL;
  int rc = oracle_validate(f, ghat, G.V, xi, N);
  if (rc) return rc;
  int64_t V = G.V;
  Work W;
  if (alloc_work(V, &W)) return ORC_ENOMEM;
  uint8_t *mark = malloc(V), *c = counts ? counts : malloc(V);
  Ref R;
  if (!mark || !c || build_ref(&G, f, &R, W.stack)) {
    free(mark);
    if (!counts) free(c);
    free_work(&W);
    return ORC_ENOMEM;
  }
  memmove(out, ghat, 4 * V); /* g <- f^ */
  memset(c, 0, V);
  uint32_t iters = 0;
  int64_t rows = 0;
  int status = ORC_OK;
  for (;;) {
    int64_t cnt[7];
    detect(&G, f, &R, out, flags, mark, &W, cnt);
    int64_t applied = 0;
    int done = (cnt[0] == 0);
    if (!done && max_iters && iters >= max_iters) {
      status = ORC_ESTUCK;
      done = 1;
    }
    if (!done) {
      applied = apply_edits(V, f, xi, N, mark, out, c);
      if (applied == 0) {
        status = ORC_ESTUCK;
        done = 1;
      } else {
        iters++;
      }
    }
    if (stats && rows < stats_cap) {
      int64_t *row = stats + 8 * rows;
      row[0] = cnt[0]; row[1] = applied;
      for (int k = 1; k <= 6; k++) row[1 + k] = cnt[k];
    }
    rows++;
    if (done) break;
  }
  if (lab_min || lab_max) {
    for (int64_t i = 0; i < V; i++) steepest(&G, out, i, &W.upg[i], &W.dng[i]);
    if (lab_min) path_labels(V, W.dng, lab_min, W.stack);
    if (lab_max) path_labels(V, W.upg, lab_max, W.stack);
  }
  if (iters_out) *iters_out = iters;
  if (stats_rows) *stats_rows = rows;
  free_ref(&R);
  free_work(&W);
  free(mark);
  if (!counts) free(c);
  return status;
}

/* ------------------------------------------------------------------------ */
/* O11. Verification-only tools (tests; never on the hot path).              */
/* ------------------------------------------------------------------------ */

/* (a) Extremum graph: {(s, lab_dn(u)) : s join saddle, u in L(s)} for
 * split=0, {(s, lab_up(u)) : s split saddle, u in U(s)} for split=1;
 * deduplicated.  edges: int32 pairs, capacity cap pairs.  Returns #edges. */
int64_t oracle_extremum_graph(const float *h, int64_t nx, int64_t ny, int64_t nz, int split,
                              int32_t *edges, int64_t cap) {
  Grid G;
  if (make_grid(&G, nx, ny, nz)) return -1;
  int64_t V = G.V;
  int32_t *lab_dn = malloc(4 * V), *lab_up = malloc(4 * V);
  if (!lab_dn || !lab_up) {
    free(lab_dn); free(lab_up);
    return -1;
  }
  oracle_labels(h, nx, ny, nz, lab_dn, lab_up);
  int64_t ne = 0, nb[14];
  int ko[14];
  for (int64_t s = 0; s < V; s++) {
    int a, b;
    link_components(&G, h, s, &a, &b);
    if (class_of(a, b) != CLS_SADDLE) continue;
    if (split ? (b < 2) : (a < 2)) continue;
    int n = neighbors(&G, s, nb, ko);
    int32_t seen[14];
    int ns = 0;
    for (int q = 0; q < n; q++) {
      int lower = sos_less(h, nb[q], s);
      if (split ? lower : !lower) continue;
      int32_t e = split ? lab_up[nb[q]] : lab_dn[nb[q]];
      int dup = 0;
      for (int t = 0; t < ns; t++) dup |= (seen[t] == e);
      if (dup) continue;
      seen[ns++] = e;
      if (ne < cap) {
        edges[2 * ne] = (int32_t)s;
        edges[2 * ne + 1] = e;
      }
      ne++;
    }
  }
  free(lab_dn); free(lab_up);
  return ne;
}

/* (b) Merge tree by brute force: a textbook union-find sweep of the sublevel
 * sets L^-(c) over the mesh graph, in ascending SoS order (join
 * tree) or the exactly reversed order (split tree, amb-3).  A vertex touching
 * >= 2 components is a merge node: it emits tree arcs (head(C), v) for every
 * merged C and elder pairs (birth(C), v) for all but the oldest-born C.  At the
 * end: root arc (head, last vertex) and pair (first vertex, last vertex).
 * Returns #arcs in n[0], #pairs in n[1]; arcs/pairs need 2*V int32 each. */
static int64_t uf_find(int64_t *parent, int64_t x) {
  while (parent[x] != x) {
    parent[x] = parent[parent[x]];
    x = parent[x];
  }
  return x;
}

int oracle_merge_tree(const float *h, int64_t nx, int64_t ny, int64_t nz, int split, int32_t *arcs,
                      int32_t *pairs, int64_t *n) {
  Grid G;
  if (make_grid(&G, nx, ny, nz)) return ORC_EINVAL;
  int64_t V = G.V;
  int32_t *order = malloc(4 * V);
  int64_t *parent = malloc(8 * V), *rank = malloc(8 * V);
  int32_t *head = malloc(4 * V), *birth = malloc(4 * V);
  int64_t *pos = malloc(8 * V);
  if (!order || !parent || !head || !birth || !pos || !rank) {
    free(order); free(parent); free(head); free(birth); free(pos); free(rank);
    return ORC_ENOMEM;
  }
  for (int64_t i = 0; i < V; i++) order[i] = (int32_t)i;
  sort_h = h;
  qsort(order, V, 4, cmp_sos_asc);
  if (split) /* exactly reversed total order */
    for (int64_t i = 0; i < V / 2; i++) {
      int32_t t = order[i]; order[i] = order[V - 1 - i]; order[V - 1 - i] = t;
    }
  for (int64_t i = 0; i < V; i++) {
    pos[order[i]] = i; /* processing time */
    parent[i] = -1;
  }
  int64_t na = 0, np = 0, nb[14];
  int ko[14];
  for (int64_t t = 0; t < V; t++) {
    int64_t v = order[t];
    int n = neighbors(&G, v, nb, ko);
    int64_t roots[14];
    int nr = 0;
    for (int q = 0; q < n; q++) {
      if (pos[nb[q]] >= t) continue; /* not yet processed */
      int64_t r = uf_find(parent, nb[q]);
      int dup = 0;
      for (int k = 0; k < nr; k++) dup |= (roots[k] == r);
      if (!dup) roots[nr++] = r;
    }
    parent[v] = v;
    rank[v] = 0;
    if (nr == 0) { /* a new component is born: a minimum of the sweep */
      head[v] = (int32_t)v;
      birth[v] = (int32_t)v;
      continue;
    }
    if (nr == 1) {
      int64_t r = roots[0];
      parent[v] = r;
      continue;
    }
    /* merge node */
    int oldest = 0;
    for (int k = 1; k < nr; k++)
      if (pos[birth[roots[k]]] < pos[birth[roots[oldest]]]) oldest = k;
    for (int k = 0; k < nr; k++) {
      arcs[2 * na] = head[roots[k]];
      arcs[2 * na + 1] = (int32_t)v;
      na++;
      if (k != oldest) {
        pairs[2 * np] = birth[roots[k]];
        pairs[2 * np + 1] = (int32_t)v;
        np++;
      }
    }
    int32_t old_birth = birth[roots[oldest]];
    for (int k = 0; k < nr; k++) parent[roots[k]] = v;
    head[v] = (int32_t)v;
    birth[v] = old_birth;
  }
  int64_t r = uf_find(parent, order[V - 1]);
  arcs[2 * na] = head[r];
  arcs[2 * na + 1] = order[V - 1];
  na++;
  pairs[2 * np] = order[0];
  pairs[2 * np + 1] = order[V - 1];
  np++;
  n[0] = na;
  n[1] = np;
  free(order); free(parent); free(head); free(birth); free(pos); free(rank);
  return ORC_OK;
}

/* (d) Vulnerability graphs and the Theorem 1 bound (amb-21/22).
 * Mesh edges {u,v} oriented u->v when v <_f u.
 *   weak   : f_u - f_v <= 2 xi                    (double)
 *   strong : weak and ghat_v >= f_u - xi          (double)
 *   seed   : strong and u <=_ghat v, read under SoS as u <_ghat v
 * G_R = strong edges whose tail is reachable from a seed endpoint along strong
 * edges; dep(v) = most vertices on a path from a seed endpoint;
 * D_max = max dep (0 without seeds).
 * out[0]=D_max, out[1]=|V(G_V)|, out[2]=|V(G_S)|, out[3]=|V(G_R)|, out[4]=#seeds. */
int oracle_vulnerability(const float *f, const float *ghat, int64_t nx, int64_t ny, int64_t nz,
                         float xi, int64_t *out) {
  Grid G;
  if (make_grid(&G, nx, ny, nz)) return ORC_EINVAL;
  int64_t V = G.V;
  int32_t *order = malloc(4 * V);
  uint8_t *inV = calloc(V, 1), *inS = calloc(V, 1), *inR = calloc(V, 1), *reach = calloc(V, 1);
  int64_t *dep = calloc(V, 8);
  if (!order || !inV || !inS || !inR || !reach || !dep) {
    free(order); free(inV); free(inS); free(inR); free(reach); free(dep);
    return ORC_ENOMEM;
  }
  double x2 = 2.0 * (double)xi, x1 = (double)xi;
  int64_t nb[14], nseeds = 0;
  int ko[14];
  /* edge classification; reach[] seeded with seed endpoints */
  for (int64_t u = 0; u < V; u++) {
    int n = neighbors(&G, u, nb, ko);
    for (int q = 0; q < n; q++) {
      int64_t v = nb[q];
      if (!sos_less(f, v, u)) continue; /* orient u -> v, v <_f u */
      if (!((double)f[u] - (double)f[v] <= x2)) continue;
      inV[u] = inV[v] = 1;
      if (!((double)ghat[v] >= (double)f[u] - x1)) continue;
      inS[u] = inS[v] = 1;
      if (sos_less(ghat, u, v)) {
        reach[u] = reach[v] = 1;
        nseeds++;
      }
    }
  }
  /* descending f order is a topological order of every stage (edges go from
   * f-larger to f-smaller) */
  for (int64_t i = 0; i < V; i++) order[i] = (int32_t)i;
  sort_h = f;
  qsort(order, V, 4, cmp_sos_asc);
  for (int64_t i = 0; i < V; i++) dep[i] = reach[i] ? 1 : 0;
  int64_t dmax = 0;
  for (int64_t t = V - 1; t >= 0; t--) {
    int64_t u = order[t];
    if (!reach[u]) continue;
    if (dep[u] > dmax) dmax = dep[u];
    int n = neighbors(&G, u, nb, ko);
    for (int q = 0; q < n; q++) {
      int64_t v = nb[q];
      if (!sos_less(f, v, u)) continue;
      if (!((double)f[u] - (double)f[v] <= x2)) continue;
      if (!((double)ghat[v] >= (double)f[u] - x1)) continue;
      /* strong edge with reachable tail: in G_R */
      inR[u] = inR[v] = 1;
      reach[v] = 1;
      if (dep[u] + 1 > dep[v]) dep[v] = dep[u] + 1;
    }
  }
  int64_t cV = 0, cS = 0, cR = 0;
  for (int64_t i = 0; i < V; i++) {
    cV += inV[i];
    cS += inS[i];
    cR += inR[i];
  }
  out[0] = dmax; out[1] = cV; out[2] = cS; out[3] = cR; out[4] = nseeds;
  free(order); free(inV); free(inS); free(inR); free(reach); free(dep);
  return ORC_OK;
}

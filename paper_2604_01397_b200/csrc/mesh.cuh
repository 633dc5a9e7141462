// mesh.cuh — Freudenthal neighbourhood of the B200 path (SURVEY §8(c) O3,
// amb-1): 14 neighbour slots and the 36-edge link graph.
//
// Slot order = ascending linear-index offset (x + nx*(y + ny*z)), which is the
// lexicographic (dz, dy, dx) order for every grid whose clipped axes have
// length 1.  With this order the Simulation-of-Simplicity tie break of
// P:178 (footnote: "the vertex with the larger global index [is] larger")
// becomes a STATIC direction per slot:
//   slot s < 7 (neighbour index smaller):  u <_h i  <=>  h_u <= h_i
//   slot s >= 7 (neighbour index larger):  u <_h i  <=>  h_u <  h_i
// and an argmin (argmax) over the closed star taken in slot order with a
// strict (non-strict) compare is the SoS argmin (argmax).
//
// The link adjacency is generated here from the 24 Kuhn tetrahedra around a
// vertex (the 6 permutation chains of each of the 8 incident cubes), NOT from
// the oracle's pairwise chain rule; the two constructions are checked against
// each other only through end-to-end results (tests/test_gpu_*.py).
#pragma once
#include <stdint.h>

namespace exz {

constexpr int kSlots = 14;
constexpr int kSelf = 14;  // "slot" code of the centre vertex

// (dx, dy, dz) of each slot, ascending linear offset.
constexpr int kOff[kSlots][3] = {
    {-1, -1, -1}, {0, -1, -1}, {-1, 0, -1}, {0, 0, -1}, {-1, -1, 0}, {0, -1, 0}, {-1, 0, 0},
    {1, 0, 0},    {0, 1, 0},   {1, 1, 0},   {0, 0, 1},  {1, 0, 1},   {0, 1, 1},  {1, 1, 1}};

struct LinkTables {
  uint16_t adj[kSlots];  // adj[s] = bitmask of slots link-adjacent to s
  uint16_t req[6];       // slots needing x-1, x+1, y-1, y+1, z-1, z+1 to exist
};

constexpr int slot_of(int dx, int dy, int dz) {
  for (int s = 0; s < kSlots; ++s)
    if (kOff[s][0] == dx && kOff[s][1] == dy && kOff[s][2] == dz) return s;
  return -1;
}

constexpr LinkTables make_link_tables() {
  LinkTables t{};
  const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  for (int cz = -1; cz <= 0; ++cz)
    for (int cy = -1; cy <= 0; ++cy)
      for (int cx = -1; cx <= 0; ++cx)
        for (int p = 0; p < 6; ++p) {
          // tetrahedron {c, c+e_a, c+e_a+e_b, c+(1,1,1)} of the Kuhn subdivision
          int pts[4][3] = {{cx, cy, cz}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
          for (int j = 1; j < 4; ++j) {
            for (int c = 0; c < 3; ++c) pts[j][c] = pts[j - 1][c];
            pts[j][perms[p][j - 1]] += 1;
          }
          int centre = -1;
          for (int j = 0; j < 4; ++j)
            if (pts[j][0] == 0 && pts[j][1] == 0 && pts[j][2] == 0) centre = j;
          if (centre < 0) continue;
          // the opposite triangle lies in the link: its 3 edges are link edges
          for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) {
              if (a == centre || b == centre || a == b) continue;
              int sa = slot_of(pts[a][0], pts[a][1], pts[a][2]);
              int sb = slot_of(pts[b][0], pts[b][1], pts[b][2]);
              t.adj[sa] = (uint16_t)(t.adj[sa] | (1u << sb));
            }
        }
  for (int s = 0; s < kSlots; ++s)
    for (int c = 0; c < 3; ++c) {
      if (kOff[s][c] < 0) t.req[2 * c] = (uint16_t)(t.req[2 * c] | (1u << s));
      if (kOff[s][c] > 0) t.req[2 * c + 1] = (uint16_t)(t.req[2 * c + 1] | (1u << s));
    }
  return t;
}

constexpr LinkTables kLink = make_link_tables();

constexpr int popcount16(unsigned v) {
  int n = 0;
  for (; v; v &= v - 1) ++n;
  return n;
}
constexpr int link_edge_count() {
  int n = 0;
  for (int s = 0; s < kSlots; ++s) n += popcount16(kLink.adj[s]);
  return n / 2;
}
static_assert(link_edge_count() == 36, "Freudenthal link must have 36 edges");
static_assert(kLink.adj[0] != 0 && kLink.adj[13] != 0, "link tables");
// symmetric negation: slot s and 13 - s are opposite offsets
static_assert(kOff[3][2] == -kOff[10][2] && kOff[6][0] == -kOff[7][0], "slot order");

}  // namespace exz

// editlog.cuh — the edit set E of a correction as a compact log (SURVEY §8(f)
// NEXT-4; Alg. 1 "Set of applied edits E" P:245, "store the edit in a
// lossless manner as the absolute lower bound", P:433 edits compressed
// losslessly; S:104-138 EditLog / serialize_edit_log).
//
// Entries are the vertices with edit count c_i > 0, in index order:
//   Stepped(k), 1 <= k <= N : out_i = k sequential steps RN(. - Delta) from
//                             g_in_i (no step was clamped), Delta = RN(xi/N);
//   Lossless(v)             : out_i = v (the clamp at lo = RU(f_i - xi), the
//                             only other value a correction produces).
// The decoder needs g_in only (not f): it replays the steps or stores v.
//
// Byte format "EXCE" v1 (little endian):
//   magic 'E','X','C','E', u8 version = 1, u8 codec (0 raw, 1 zstd),
//   u16 reserved, f32 xi, u32 N, i64 nx, ny, nz, u64 entries,
//   u64 payload bytes (after the codec), u64 raw payload bytes, payload.
// Raw payload, per entry: varint(index - previous index - 1) (the first entry:
//   varint(index)), u8 kind (0 = Lossless, k = Stepped(k)), and for Lossless
//   the 4 bytes of v.
#pragma once

namespace exz {

// kind per vertex: 0xFF = no entry, 0 = Lossless, k = Stepped(k)
__global__ void __launch_bounds__(256) k_edit_kind(const float *__restrict__ g_in,
                                                   const float *__restrict__ out,
                                                   const uint8_t *__restrict__ c, int64_t V,
                                                   float delta, int N, uint8_t *kind) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < V;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ci = c[i];
    uint8_t k = 0xFFu;
    if (ci > 0) {
      k = 0;
      if (ci <= N) {
        float t = g_in[i];
        for (int s = 0; s < ci; ++s) t = __fsub_rn(t, delta);
        if (__float_as_uint(t) == __float_as_uint(out[i])) k = (uint8_t)ci;
      }
    }
    kind[i] = k;
  }
}

struct HasEntry {
  const uint8_t *kind;
  __device__ __forceinline__ bool operator()(const int64_t &i) const { return kind[i] != 0xFFu; }
};

__global__ void k_edit_gather(const int64_t *__restrict__ idx, int64_t n,
                              const uint8_t *__restrict__ kind, const float *__restrict__ out,
                              uint8_t *ek, float *ev) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx[e];
    ek[e] = kind[i];
    ev[e] = out[i];
  }
}

// raw payload on the GPU: per entry its byte length (varint of the index gap,
// the kind byte, 4 value bytes for Lossless), an exclusive scan, the bytes
__device__ __forceinline__ int varint_len(uint64_t v) {
  int n = 1;
  while (v >= 0x80) {
    v >>= 7;
    ++n;
  }
  return n;
}
__global__ void k_edit_len(const int64_t *__restrict__ idx, const uint8_t *__restrict__ ek,
                           int64_t n, uint64_t *len) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t gap = (uint64_t)(idx[e] - (e ? idx[e - 1] : -1) - 1);
    len[e] = (uint64_t)(varint_len(gap) + 1 + (ek[e] == 0 ? 4 : 0));
  }
}
__global__ void k_edit_write(const int64_t *__restrict__ idx, const uint8_t *__restrict__ ek,
                             const float *__restrict__ ev, int64_t n,
                             const uint64_t *__restrict__ pos, uint8_t *out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint64_t v = (uint64_t)(idx[e] - (e ? idx[e - 1] : -1) - 1);
    uint8_t *o = out + pos[e];
    while (v >= 0x80) {
      *o++ = (uint8_t)(v | 0x80);
      v >>= 7;
    }
    *o++ = (uint8_t)v;
    *o++ = ek[e];
    if (ek[e] == 0) {
      const uint32_t b = __float_as_uint(ev[e]);
      o[0] = (uint8_t)b;
      o[1] = (uint8_t)(b >> 8);
      o[2] = (uint8_t)(b >> 16);
      o[3] = (uint8_t)(b >> 24);
    }
  }
}

// apply decoded entries: out = g_in except at the entries
__global__ void k_edit_apply(const int64_t *__restrict__ idx, const uint8_t *__restrict__ ek,
                             const float *__restrict__ ev, int64_t n,
                             const float *__restrict__ g_in, float *out, float delta) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx[e];
    const int k = ek[e];
    if (k == 0) {
      out[i] = ev[e];
    } else {
      float t = g_in[i];
      for (int s = 0; s < k; ++s) t = __fsub_rn(t, delta);
      out[i] = t;
    }
  }
}

}  // namespace exz

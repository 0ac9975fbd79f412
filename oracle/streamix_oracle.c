/*
 * streamix_oracle.c — CPU restatement of the reference enqueue path.
 * TEST INFRASTRUCTURE ONLY (see streamix_oracle.h). Each function cites the
 * reference file:line it restates; paths are relative to /root/reference.
 */
#include "streamix_oracle.h"

#include <stdlib.h>
#include <string.h>

static const char *const kErrNames[] = {
    /* proj/src/result.cpp:5-32 */
    "OK", "POOL_EXHAUSTED", "NO_EXPLICIT_POOL", "PENDING_OPS", "IN_USE", "BAD_HINT",
    "INVALID_STREAM", "INVALID_COMM", "INVALID_RANK", "INVALID_COUNT", "INVALID_TAG",
    "INVALID_REQUEST", "INVALID_INDEX", "MULTIPLEX_COMM", "NOT_MULTIPLEX", "WILDCARD_DST",
    "EMPTY_LIST", "NOT_ENQUEUE_COMM", "STREAM_MISMATCH", "QUEUE_BUSY", "CONFIG_INVALID",
    "NOT_FOUND", "BAD_ENCODING"};

const char *orc_err_name(int code) {
  if (code < 0 || code > ORC_BAD_ENCODING) return "UNKNOWN";
  return kErrNames[code];
}

/* proj/src/info.cpp:37-46 */
void orc_hex_encode(const uint8_t *in, size_t len, char *out) {
  static const char d[] = "0123456789abcdef";
  for (size_t i = 0; i < len; ++i) {
    out[2 * i] = d[in[i] >> 4];
    out[2 * i + 1] = d[in[i] & 15];
  }
  out[2 * len] = 0;
}

/* proj/src/info.cpp:10-15 (nibble) and 48-59 (decode) */
static int orc_nibble(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  return -1;
}

int orc_hex_decode(const char *s, size_t slen, uint8_t *out, size_t *outlen) {
  if (slen % 2) return ORC_BAD_ENCODING;
  for (size_t i = 0; i < slen; i += 2) {
    int hi = orc_nibble(s[i]), lo = orc_nibble(s[i + 1]);
    if (hi < 0 || lo < 0) return ORC_BAD_ENCODING;
    out[i / 2] = (uint8_t)((hi << 4) | lo);
  }
  *outlen = slen / 2;
  return ORC_OK;
}

/* proj/src/wire.cpp:9-29 (put/get), 31-51 (encode/decode) */
static void put_le(uint8_t *p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static uint64_t get_le(const uint8_t *p, int n) {
  uint64_t v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

void orc_encode_header(const orc_envelope *e, uint8_t out[36]) {
  put_le(out + 0, e->context_id, 4);
  put_le(out + 4, e->src_rank, 4);
  put_le(out + 8, (uint32_t)e->src_idx, 4);
  put_le(out + 12, (uint32_t)e->dst_idx, 4);
  put_le(out + 16, (uint32_t)e->tag, 4);
  put_le(out + 20, e->seq, 8);
  put_le(out + 28, e->payload_len, 8);
}

void orc_decode_header(const uint8_t in[36], orc_envelope *e) {
  e->context_id = (uint32_t)get_le(in + 0, 4);
  e->src_rank = (uint32_t)get_le(in + 4, 4);
  e->src_idx = (int32_t)(uint32_t)get_le(in + 8, 4);
  e->dst_idx = (int32_t)(uint32_t)get_le(in + 12, 4);
  e->tag = (int32_t)(uint32_t)get_le(in + 16, 4);
  e->seq = get_le(in + 20, 8);
  e->payload_len = get_le(in + 28, 8);
}

/* proj/include/streamix/wire.hpp:38-43 */
uint32_t orc_wire_ctx(uint32_t comm_ctx, int collective) {
  return (comm_ctx << 1) | (collective ? 1u : 0u);
}

/* proj/src/proc_enqueue.cpp:8-20 */
int orc_check_enqueue_args(int n_ranks, int count, int peer, int tag, int recv_side) {
  if (recv_side) {
    if (peer != ORC_ANY && (peer < 0 || peer >= n_ranks)) return ORC_INVALID_RANK;
    if (tag != ORC_ANY && tag < 0) return ORC_INVALID_TAG;
  } else {
    if (peer < 0 || peer >= n_ranks) return ORC_INVALID_RANK;
    if (tag < 0) return ORC_INVALID_TAG;
  }
  if (count < 0) return ORC_INVALID_COUNT;
  return ORC_OK;
}

/* proj/src/proc_p2p.cpp:9-23 */
int orc_check_p2p_args(int n_ranks, int count, int peer, int tag, int recv_side) {
  if (recv_side) {
    if (peer != ORC_ANY && (peer < 0 || peer >= n_ranks)) return ORC_INVALID_RANK;
    if (count < 0) return ORC_INVALID_COUNT;
    if (tag != ORC_ANY && tag < 0) return ORC_INVALID_TAG;
  } else {
    if (peer < 0 || peer >= n_ranks) return ORC_INVALID_RANK;
    if (count < 0) return ORC_INVALID_COUNT;
    if (tag < 0) return ORC_INVALID_TAG;
  }
  return ORC_OK;
}

/* proj/src/endpoint.cpp:17-24 */
void orc_deliver(uint64_t len, uint64_t cap, uint64_t *delivered, int *truncated) {
  *delivered = len < cap ? len : cap;
  *truncated = len > cap;
}

/* ---- matching ------------------------------------------------------------ */
typedef struct {
  int src, tag;
  uint64_t id;
} orc_msg;
typedef struct {
  int source, tag;
  uint64_t id;
} orc_recv;

static int accepts(const orc_recv *r, const orc_msg *m) { /* oracle.cpp:27-30 */
  return (r->source == ORC_ANY || r->source == m->src) && (r->tag == ORC_ANY || r->tag == m->tag);
}

static uint64_t op_id(int rank, int pos) { return ((uint64_t)rank << 16) | (uint64_t)pos; }

/* proj/src/oracle.cpp:33-74: one posted list and one unexpected list per
 * destination; arrival side takes the first accepting posted receive, post
 * side the first accepting unexpected message. */
void orc_match_reference(int n_ranks, const orc_op *const *progs, const int *lens,
                         const int *order, int n_order, uint64_t *pairs_out, int max_pos) {
  int total = 0;
  for (int r = 0; r < n_ranks; ++r) total += lens[r];
  orc_recv **posted = calloc((size_t)n_ranks, sizeof(*posted));
  orc_msg **unexp = calloc((size_t)n_ranks, sizeof(*unexp));
  int *np = calloc((size_t)n_ranks, sizeof(int)), *nu = calloc((size_t)n_ranks, sizeof(int));
  int *pos = calloc((size_t)n_ranks, sizeof(int));
  for (int r = 0; r < n_ranks; ++r) {
    posted[r] = calloc((size_t)total + 1, sizeof(orc_recv));
    unexp[r] = calloc((size_t)total + 1, sizeof(orc_msg));
  }
  for (int i = 0; i < n_ranks * max_pos; ++i) pairs_out[i] = UINT64_MAX;
  for (int k = 0; k < n_order; ++k) {
    int rank = order[k];
    const orc_op *op = &progs[rank][pos[rank]];
    uint64_t id = op_id(rank, pos[rank]);
    int me_pos = pos[rank]++;
    if (op->is_send) {
      orc_msg m = {rank, op->tag, id};
      int d = op->peer, hit = -1;
      for (int j = 0; j < np[d]; ++j)
        if (accepts(&posted[d][j], &m)) { hit = j; break; }
      if (hit >= 0) {
        uint64_t rid = posted[d][hit].id;
        pairs_out[(int)(rid >> 16) * max_pos + (int)(rid & 0xffff)] = m.id;
        memmove(&posted[d][hit], &posted[d][hit + 1], (size_t)(np[d] - hit - 1) * sizeof(orc_recv));
        --np[d];
      } else {
        unexp[d][nu[d]++] = m;
      }
    } else {
      orc_recv rv = {op->peer, op->tag, id};
      int hit = -1;
      for (int j = 0; j < nu[rank]; ++j)
        if (accepts(&rv, &unexp[rank][j])) { hit = j; break; }
      if (hit >= 0) {
        pairs_out[rank * max_pos + me_pos] = unexp[rank][hit].id;
        memmove(&unexp[rank][hit], &unexp[rank][hit + 1],
                (size_t)(nu[rank] - hit - 1) * sizeof(orc_msg));
        --nu[rank];
      } else {
        posted[rank][np[rank]++] = rv;
      }
    }
  }
  for (int r = 0; r < n_ranks; ++r) { free(posted[r]); free(unexp[r]); }
  free(posted); free(unexp); free(np); free(nu); free(pos);
}

void orc_match_static(int n_ranks, const orc_op *const *progs, const int *lens,
                      uint64_t *pairs_out, int max_pos) {
  for (int i = 0; i < n_ranks * max_pos; ++i) pairs_out[i] = UINT64_MAX;
  for (int d = 0; d < n_ranks; ++d) {
    for (int k = 0; k < lens[d]; ++k) {
      const orc_op *rv = &progs[d][k];
      if (rv->is_send) continue;
      int s = rv->peer, t = rv->tag;
      /* m = index of this receive among d's receives for (s, t) */
      int m = 0;
      for (int j = 0; j < k; ++j)
        if (!progs[d][j].is_send && progs[d][j].peer == s && progs[d][j].tag == t) ++m;
      /* the m-th send s->d with tag t */
      int c = 0;
      for (int j = 0; j < lens[s]; ++j) {
        const orc_op *sd = &progs[s][j];
        if (sd->is_send && sd->peer == d && sd->tag == t) {
          if (c == m) { pairs_out[d * max_pos + k] = op_id(s, j); break; }
          ++c;
        }
      }
    }
  }
}

/* ---- allreduce ----------------------------------------------------------- */
#define FOLD(acc, x, op) \
  ((op) == 1 ? (acc) + (x) : (op) == 2 ? ((x) > (acc) ? (x) : (acc)) : ((x) < (acc) ? (x) : (acc)))

void orc_allreduce_f32(const float *const *in, int P, size_t n, int op, float *out) {
  for (size_t i = 0; i < n; ++i) {
    volatile float acc = in[0][i];
    for (int q = 1; q < P; ++q) acc = FOLD(acc, in[q][i], op);
    out[i] = acc;
  }
}

void orc_allreduce_f64(const double *const *in, int P, size_t n, int op, double *out) {
  for (size_t i = 0; i < n; ++i) {
    volatile double acc = in[0][i];
    for (int q = 1; q < P; ++q) acc = FOLD(acc, in[q][i], op);
    out[i] = acc;
  }
}

void orc_allreduce_i32(const int32_t *const *in, int P, size_t n, int op, int32_t *out) {
  for (size_t i = 0; i < n; ++i) {
    uint32_t acc = (uint32_t)in[0][i];
    for (int q = 1; q < P; ++q) {
      int32_t x = in[q][i], a = (int32_t)acc;
      if (op == 1) acc += (uint32_t)x; /* wrapping */
      else acc = (uint32_t)(op == 2 ? (x > a ? x : a) : (x < a ? x : a));
    }
    out[i] = (int32_t)acc;
  }
}

static float bf16_to_f32(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

uint16_t orc_f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40); /* quiet NaN */
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

void orc_allreduce_bf16(const uint16_t *const *in, int P, size_t n, int op, uint16_t *out) {
  for (size_t i = 0; i < n; ++i) {
    volatile float acc = bf16_to_f32(in[0][i]);
    for (int q = 1; q < P; ++q) acc = FOLD(acc, bf16_to_f32(in[q][i]), op);
    out[i] = orc_f32_to_bf16_rne(acc);
  }
}

uint32_t orc_hash32(uint64_t i, uint32_t r) {
  uint64_t z = i * 0x9E3779B97F4A7C15ull + (uint64_t)r * 0xD1B54A32D192ED03ull + 1;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (uint32_t)(z ^ (z >> 31));
}

float orc_exact_f32(uint64_t i, uint32_t r) {
  return (float)((int)(orc_hash32(i, r) % 2048u) - 1024) / 256.0f;
}

uint16_t orc_exact_bf16(uint64_t i, uint32_t r) {
  return orc_f32_to_bf16_rne((float)((int)(orc_hash32(i, r) % 256u) - 128) / 16.0f);
}

/* ---- helper-kernel mirrors (paper_2208_13707_b200/csrc/mpix_testing.cu) --- */
uint32_t orc_pattern_u32(uint32_t seed, uint32_t iter, uint64_t i) {
  uint32_t x = seed ^ (iter * 0x9E3779B9u) ^ (uint32_t)i ^ (uint32_t)(i >> 32) * 0x85EBCA6Bu;
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

void orc_fill_pattern(void *buf, uint64_t nbytes, uint32_t seed, uint32_t iter) {
  uint64_t nw = nbytes / 4;
  uint8_t *b = (uint8_t *)buf;
  for (uint64_t i = 0; i < nw; ++i) {
    uint32_t v = orc_pattern_u32(seed, iter, i);
    memcpy(b + 4 * i, &v, 4);
  }
  uint32_t v = orc_pattern_u32(seed, iter, nw);
  for (uint64_t t = 0; t < nbytes - nw * 4; ++t) b[nw * 4 + t] = (uint8_t)(v >> (8 * t));
}

static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t orc_checksum64(const void *buf, uint64_t nbytes) {
  const uint8_t *b = (const uint8_t *)buf;
  uint64_t nw = nbytes / 8, acc = 0;
  for (uint64_t i = 0; i < nw; ++i) {
    uint64_t v;
    memcpy(&v, b + 8 * i, 8);
    acc += mix64(v ^ (i * 0x9E3779B97F4A7C15ull));
  }
  if (nbytes & 7) {
    uint64_t v = 0;
    for (uint64_t k = nw * 8; k < nbytes; ++k) v |= (uint64_t)b[k] << (8 * (k - nw * 8));
    acc += mix64(v ^ (nw * 0x9E3779B97F4A7C15ull));
  }
  return acc;
}

uint64_t orc_fnv1a64(const void *buf, uint64_t nbytes) {
  const uint8_t *b = (const uint8_t *)buf;
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < nbytes; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* ---- cfg5 stencil ----------------------------------------------------------- */
static uint64_t hidx(int x, int y, int z, int nx, int ny) {
  return ((uint64_t)z * (ny + 2) + y) * (uint64_t)(nx + 2) + x;
}

void orc_stencil7(const float *u, float *out, int nx, int ny, int nz, float w0, float w1) {
  const uint64_t sx = 1, sy = nx + 2, sz = (uint64_t)(nx + 2) * (ny + 2);
  for (int z = 1; z <= nz; ++z)
    for (int y = 1; y <= ny; ++y)
      for (int x = 1; x <= nx; ++x) {
        uint64_t c = hidx(x, y, z, nx, ny);
        volatile float a = u[c - sx] + u[c + sx];
        volatile float b = u[c - sy] + u[c + sy];
        volatile float d = u[c - sz] + u[c + sz];
        volatile float s = a + b;
        s = s + d;
        volatile float p0 = w0 * u[c];
        volatile float p1 = w1 * s;
        out[c] = p0 + p1;
      }
}

static void face_walk(float *u, int nx, int ny, int nz, int face, float *buf, int pack) {
  int axis = face >> 1, hi = face & 1, na, nb;
  if (axis == 0) { na = ny; nb = nz; }
  else if (axis == 1) { na = nx; nb = nz; }
  else { na = nx; nb = ny; }
  int layer = pack ? 1 : 0;
  for (int b = 0; b < nb; ++b)
    for (int a = 0; a < na; ++a) {
      int x, y, z;
      if (axis == 0) { x = hi ? nx + 1 - layer : layer; y = a + 1; z = b + 1; }
      else if (axis == 1) { x = a + 1; y = hi ? ny + 1 - layer : layer; z = b + 1; }
      else { x = a + 1; y = b + 1; z = hi ? nz + 1 - layer : layer; }
      uint64_t c = hidx(x, y, z, nx, ny);
      uint64_t i = (uint64_t)b * na + a;
      if (pack) buf[i] = u[c];
      else u[c] = buf[i];
    }
}

void orc_halo_pack(const float *u, int nx, int ny, int nz, int face, float *buf) {
  face_walk((float *)u, nx, ny, nz, face, buf, 1);
}

void orc_halo_unpack(float *u, int nx, int ny, int nz, int face, const float *buf) {
  face_walk(u, nx, ny, nz, face, (float *)buf, 0);
}

/* proj/src/wire.cpp:53-62 (append_frame) + proj/src/endpoint.cpp:15-27 (deliver) */
uint64_t orc_loopback_message(const void *src, uint64_t len, void *dst, uint64_t cap,
                              void *frame_scratch) {
  uint8_t *f = (uint8_t *)frame_scratch;
  orc_envelope e = {0, 0, -2, -2, 0, 1, len};
  orc_encode_header(&e, f);
  if (len) memcpy(f + 36, src, len);
  uint64_t n;
  int trunc;
  orc_deliver(len, cap, &n, &trunc);
  if (n) memcpy(dst, f + 36, n);
  return n;
}

/* ---- cfg3 at full size ----------------------------
 * Inputs are generated per (element, rank) instead of materialised, so the
 * rank-ordered fold of P x 256 MiB runs in host memory of one chunk.
 *   set 0 "exact":           f32 (h%2048-1024)/256, bf16 (h%256-128)/16
 *   set 1 "order-sensitive": uniform(-1,1) = (h >> 8) * 2^-23 - 1 (exact in
 *                            f32; bf16 = its RNE rounding)
 * The device generator (MPIXT_Fill_values, mpix_testing.cu) computes the
 * same bits. */
float orc_value_f32(uint64_t i, uint32_t r, int set) {
  if (set == 0) return orc_exact_f32(i, r);
  return (float)(orc_hash32(i, r) >> 8) * (1.0f / 8388608.0f) - 1.0f;
}

uint16_t orc_value_bf16(uint64_t i, uint32_t r, int set) {
  if (set == 0) return orc_exact_bf16(i, r);
  return orc_f32_to_bf16_rne(orc_value_f32(i, r, 1));
}

/* checksum64 of bytes [0, nbytes) of a buffer whose 8-byte word 0 is word
 * `w0` of the whole buffer (nbytes a multiple of 8 except at the end). */
static uint64_t checksum_part(const uint8_t *b, uint64_t nbytes, uint64_t w0) {
  uint64_t nw = nbytes / 8, acc = 0;
  for (uint64_t i = 0; i < nw; ++i) {
    uint64_t v;
    memcpy(&v, b + 8 * i, 8);
    acc += mix64(v ^ ((w0 + i) * 0x9E3779B97F4A7C15ull));
  }
  if (nbytes & 7) {
    uint64_t v = 0;
    for (uint64_t k = nw * 8; k < nbytes; ++k) v |= (uint64_t)b[k] << (8 * (k - nw * 8));
    acc += mix64(v ^ ((w0 + nw) * 0x9E3779B97F4A7C15ull));
  }
  return acc;
}

uint64_t orc_gen_checksum(uint32_t r, uint64_t count, int dt, int set) {
  const uint64_t chunk = 1u << 20; /* elements, a multiple of 4 */
  const int es = dt == 1 ? 4 : 2;
  uint8_t *buf = (uint8_t *)malloc(chunk * es);
  uint64_t acc = 0;
  for (uint64_t c0 = 0; c0 < count; c0 += chunk) {
    uint64_t n = count - c0 < chunk ? count - c0 : chunk;
    for (uint64_t k = 0; k < n; ++k) {
      if (dt == 1) { float v = orc_value_f32(c0 + k, r, set); memcpy(buf + 4 * k, &v, 4); }
      else { uint16_t v = orc_value_bf16(c0 + k, r, set); memcpy(buf + 2 * k, &v, 2); }
    }
    acc += checksum_part(buf, n * es, c0 * es / 8);
  }
  free(buf);
  return acc;
}

uint64_t orc_allreduce_gen(int P, uint64_t count, int dt, int set, int op, int ns,
                           const uint64_t *sample_idx, void *sample_out) {
  const uint64_t chunk = 1u << 20;
  const int es = dt == 1 ? 4 : 2;
  uint8_t *buf = (uint8_t *)malloc(chunk * es);
  uint64_t acc = 0;
  for (uint64_t c0 = 0; c0 < count; c0 += chunk) {
    uint64_t n = count - c0 < chunk ? count - c0 : chunk;
    for (uint64_t k = 0; k < n; ++k) {
      const uint64_t i = c0 + k;
      if (dt == 1) { /* same fold as orc_allreduce_f32 */
        volatile float a = orc_value_f32(i, 0, set);
        for (int q = 1; q < P; ++q) a = FOLD(a, orc_value_f32(i, (uint32_t)q, set), op);
        float v = a;
        memcpy(buf + 4 * k, &v, 4);
      } else { /* same fold as orc_allreduce_bf16 */
        volatile float a = bf16_to_f32(orc_value_bf16(i, 0, set));
        for (int q = 1; q < P; ++q) a = FOLD(a, bf16_to_f32(orc_value_bf16(i, (uint32_t)q, set)), op);
        uint16_t v = orc_f32_to_bf16_rne(a);
        memcpy(buf + 2 * k, &v, 2);
      }
    }
    for (int s = 0; s < ns; ++s)
      if (sample_idx[s] >= c0 && sample_idx[s] < c0 + n)
        memcpy((uint8_t *)sample_out + (size_t)s * es, buf + (sample_idx[s] - c0) * es, es);
    acc += checksum_part(buf, n * es, c0 * es / 8);
  }
  free(buf);
  return acc;
}

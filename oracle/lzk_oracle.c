/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see lzk_oracle.h). Plain C11, no CUDA,
 * no product code. Restates the reference algorithms for the snapshot path.
 */
#include "lzk_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---- FNV-1a 64: include/lzckpt/checksum.hpp:12-24 ---------------------- */
uint64_t lzo_fnv1a64(uint64_t h, const uint8_t* p, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
  return h;
}

/* ---- generators ---------------------------------------------------------- */
/* MT19937-64 (Matsumoto & Nishimura), identical to std::mt19937_64(seed). */
#define MT_NN 312
#define MT_MM 156
typedef struct {
  uint64_t mt[MT_NN];
  int mti;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_NN; ++i) s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = MT_NN;
}

static uint64_t mt64_next(mt64* s) {
  static const uint64_t mag[2] = {0ull, 0xB5026F5AA96619E9ull};
  const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
  if (s->mti >= MT_NN) {
    int i;
    uint64_t x;
    for (i = 0; i < MT_NN - MT_MM; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + MT_MM] ^ (x >> 1) ^ mag[x & 1];
    }
    for (; i < MT_NN - 1; ++i) {
      x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
      s->mt[i] = s->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ mag[x & 1];
    }
    x = (s->mt[MT_NN - 1] & UM) | (s->mt[0] & LM);
    s->mt[MT_NN - 1] = s->mt[MT_MM - 1] ^ (x >> 1) ^ mag[x & 1];
    s->mti = 0;
  }
  uint64_t x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= (x >> 43);
  return x;
}

static void put_le(uint8_t* p, uint64_t v, int w) {
  for (int i = 0; i < w; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

/* Words little-endian; a final partial word donates its leading bytes
 * (reference tests/test_support.hpp:20-31 fill). */
void lzo_fill_mt19937_64(uint64_t seed, uint64_t n_leaves, const uint64_t* sizes, uint8_t* const* out) {
  mt64* s = (mt64*)malloc(sizeof(mt64));
  mt64_seed(s, seed);
  for (uint64_t l = 0; l < n_leaves; ++l) {
    uint64_t k = 0;
    for (; k + 8 <= sizes[l]; k += 8) put_le(out[l] + k, mt64_next(s), 8);
    if (k < sizes[l]) {
      uint8_t w[8];
      put_le(w, mt64_next(s), 8);
      memcpy(out[l] + k, w, sizes[l] - k);
    }
  }
  free(s);
}

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void lzo_fill_splitmix(uint64_t seed, uint64_t leaf, uint64_t size, uint8_t* out) {
  const uint64_t base = seed ^ (leaf * 0xD1B54A32D192ED03ull);
  uint64_t k = 0, w = 0;
  for (; k + 8 <= size; k += 8, ++w) put_le(out + k, mix64(base + (w + 1) * 0x9E3779B97F4A7C15ull), 8);
  if (k < size) {
    uint8_t b[8];
    put_le(b, mix64(base + (w + 1) * 0x9E3779B97F4A7C15ull), 8);
    memcpy(out + k, b, size - k);
  }
}

uint64_t lzo_splitmix_fnv(uint64_t seed, uint64_t leaf, uint64_t size) {
  const uint64_t base = seed ^ (leaf * 0xD1B54A32D192ED03ull);
  uint64_t h = 0xcbf29ce484222325ull, k = 0, w = 0;
  for (; k + 8 <= size; k += 8, ++w) {
    const uint64_t v = mix64(base + (w + 1) * 0x9E3779B97F4A7C15ull);
    for (int b = 0; b < 8; ++b) h = (h ^ ((v >> (8 * b)) & 0xff)) * 0x100000001b3ull;
  }
  if (k < size) {
    const uint64_t v = mix64(base + (w + 1) * 0x9E3779B97F4A7C15ull);
    for (uint64_t b = 0; b < size - k; ++b) h = (h ^ ((v >> (8 * b)) & 0xff)) * 0x100000001b3ull;
  }
  return h;
}

/* ---- ring: src/ring_core.cpp:21-139 -------------------------------------- */
typedef struct {
  uint64_t id, off, len;
  int state; /* 0 Reserved 1 Filled 2 Flushing */
  int gap;
} lzo_slot;

struct lzo_ring {
  uint64_t capacity, head, next_id, live;
  lzo_slot* q; /* FIFO in reservation order: q[first .. first+count) */
  size_t first, count, cap;
};

lzo_ring* lzo_ring_new(uint64_t capacity) {
  lzo_ring* r = (lzo_ring*)calloc(1, sizeof(lzo_ring));
  r->capacity = capacity;
  r->next_id = 1;
  r->cap = 64;
  r->q = (lzo_slot*)calloc(r->cap, sizeof(lzo_slot));
  return r;
}

void lzo_ring_free(lzo_ring* r) {
  if (!r) return;
  free(r->q);
  free(r);
}

static void ring_push(lzo_ring* r, lzo_slot s) {
  if (r->first + r->count == r->cap) {
    if (r->first > 0) {
      memmove(r->q, r->q + r->first, r->count * sizeof(lzo_slot));
      r->first = 0;
    } else {
      r->cap *= 2;
      r->q = (lzo_slot*)realloc(r->q, r->cap * sizeof(lzo_slot));
    }
  }
  r->q[r->first + r->count++] = s;
}

int lzo_ring_try_reserve(lzo_ring* r, uint64_t size, uint64_t* id, uint64_t* offset) {
  if (size == 0 || size > r->capacity) return 0;
  uint64_t at = 0;
  int gap = 0;
  if (r->count == 0) {
    r->head = 0;
  } else {
    const uint64_t tail = r->q[r->first].off; /* oldest entry, never a gap */
    if (r->head > tail) {
      if (size <= r->capacity - r->head) {
        at = r->head;
      } else if (size <= tail) {
        gap = r->head < r->capacity;
        at = 0;
      } else {
        return 0;
      }
    } else if (r->head < tail) {
      if (size > tail - r->head) return 0;
      at = r->head;
    } else {
      return 0;
    }
  }
  if (gap) {
    lzo_slot g = {0, r->head, r->capacity - r->head, 0, 1};
    ring_push(r, g);
  }
  lzo_slot s = {r->next_id++, at, size, 0, 0};
  ring_push(r, s);
  r->head = at + size;
  if (r->head == r->capacity) r->head = 0;
  r->live += size;
  *id = s.id;
  *offset = at;
  return 1;
}

static lzo_slot* ring_find(lzo_ring* r, uint64_t id) {
  for (size_t i = 0; i < r->count; ++i) {
    lzo_slot* s = &r->q[r->first + i];
    if (!s->gap && s->id == id) return s;
  }
  return NULL;
}

int lzo_ring_mark_filled(lzo_ring* r, uint64_t id) {
  lzo_slot* s = ring_find(r, id);
  if (!s || s->state != 0) return -1;
  s->state = 1;
  return 0;
}

int lzo_ring_begin_flush(lzo_ring* r, uint64_t id) {
  lzo_slot* s = ring_find(r, id);
  if (!s || s->state != 1) return -1;
  s->state = 2;
  return 0;
}

int lzo_ring_release(lzo_ring* r, uint64_t id) {
  if (r->count == 0) return -1;
  lzo_slot* f = &r->q[r->first];
  if (f->gap || f->id != id || f->state != 2) return -1;
  r->live -= f->len;
  ++r->first;
  --r->count;
  while (r->count && r->q[r->first].gap) {
    ++r->first;
    --r->count;
  }
  if (r->count == 0) {
    r->head = 0;
    r->first = 0;
  }
  return 0;
}

uint64_t lzo_ring_live_bytes(const lzo_ring* r) { return r->live; }

/* ---- header: src/format.cpp:79-115 ---------------------------------------- */
uint64_t lzo_header_size(uint32_t n, const uint32_t* key_lens) {
  uint64_t s = 8 + 4 + 4 + 8;
  for (uint32_t i = 0; i < n; ++i) s += 4 + (uint64_t)key_lens[i] + 24;
  return s;
}

uint64_t lzo_header_serialize(uint32_t n, const char* const* keys, const uint32_t* key_lens,
                              const uint64_t* offsets, const uint64_t* lengths, const uint64_t* checksums,
                              uint8_t* out) {
  uint8_t* p = out;
  memcpy(p, "LZCKPT01", 8);
  p += 8;
  put_le(p, 1, 4);
  p += 4;
  put_le(p, n, 4);
  p += 4;
  for (uint32_t i = 0; i < n; ++i) {
    put_le(p, key_lens[i], 4);
    p += 4;
    memcpy(p, keys[i], key_lens[i]);
    p += key_lens[i];
    put_le(p, offsets[i], 8);
    put_le(p + 8, lengths[i], 8);
    put_le(p + 16, checksums[i], 8);
    p += 24;
  }
  put_le(p, lzo_fnv1a64(0xcbf29ce484222325ull, out, (uint64_t)(p - out)), 8);
  p += 8;
  return (uint64_t)(p - out);
}

/* ---- flatten order: src/state_tree.cpp:103-120 ---------------------------- */
static const char* const* g_paths; /* qsort context (single-threaded test use) */

static int cmp_components(const char* a, const char* b) {
  for (;;) {
    const char* ea = strchr(a, '/');
    const char* eb = strchr(b, '/');
    size_t la = ea ? (size_t)(ea - a) : strlen(a);
    size_t lb = eb ? (size_t)(eb - b) : strlen(b);
    size_t m = la < lb ? la : lb;
    int c = memcmp(a, b, m); /* std::string operator<: unsigned bytewise */
    if (c) return c;
    if (la != lb) return la < lb ? -1 : 1;
    if (!ea || !eb) return (ea ? 1 : 0) - (eb ? 1 : 0);
    a = ea + 1;
    b = eb + 1;
  }
}

static int cmp_idx(const void* x, const void* y) {
  return cmp_components(g_paths[*(const uint32_t*)x], g_paths[*(const uint32_t*)y]);
}

void lzo_flatten_order(uint32_t n, const char* const* paths, uint32_t* order) {
  for (uint32_t i = 0; i < n; ++i) order[i] = i;
  g_paths = paths;
  qsort(order, n, sizeof(uint32_t), cmp_idx);
}

/* ---- one shard file: engine.cpp:96-231, state_tree.cpp:195-210,
 *      flush_pipeline.cpp:194-263 ---------------------------------------------- */
uint64_t lzo_compose_shard(uint32_t n, const char* const* paths, const uint8_t* is_region, const uint64_t* sizes,
                           const uint8_t* const* data, uint64_t threshold, uint8_t* out) {
  /* __meta__ := u32 n, n x { u32 len, path, u8 flags(1 region|2 inlined), u64 size, [bytes] } */
  uint64_t meta = 4;
  uint32_t n_large = 0;
  for (uint32_t i = 0; i < n; ++i) {
    meta += 4 + strlen(paths[i]) + 1 + 8;
    if (sizes[i] < threshold) {
      meta += sizes[i];
    } else {
      ++n_large;
    }
  }
  const uint32_t n_entries = 1 + n_large;
  const char** keys = (const char**)malloc(n_entries * sizeof(char*));
  uint32_t* klen = (uint32_t*)malloc(n_entries * sizeof(uint32_t));
  uint64_t* off = (uint64_t*)malloc(n_entries * sizeof(uint64_t));
  uint64_t* len = (uint64_t*)malloc(n_entries * sizeof(uint64_t));
  uint64_t* sum = (uint64_t*)malloc(n_entries * sizeof(uint64_t));
  const uint8_t** src = (const uint8_t**)malloc(n_entries * sizeof(uint8_t*));
  keys[0] = "__meta__";
  klen[0] = 8;
  len[0] = meta;
  uint32_t e = 1;
  for (uint32_t i = 0; i < n; ++i) {
    if (sizes[i] >= threshold) {
      keys[e] = paths[i];
      klen[e] = (uint32_t)strlen(paths[i]);
      len[e] = sizes[i];
      src[e] = data[i];
      ++e;
    }
  }
  const uint64_t hsize = lzo_header_size(n_entries, klen);
  uint64_t cursor = hsize;
  for (uint32_t k = 0; k < n_entries; ++k) {
    off[k] = cursor;
    cursor += len[k];
  }
  const uint64_t total = cursor;
  if (out) {
    uint8_t* m = out + hsize; /* meta is entry 0, right after the header */
    put_le(m, n, 4);
    m += 4;
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t pl = (uint32_t)strlen(paths[i]);
      const int inl = sizes[i] < threshold;
      put_le(m, pl, 4);
      m += 4;
      memcpy(m, paths[i], pl);
      m += pl;
      *m++ = (uint8_t)((is_region[i] ? 1 : 0) | (inl ? 2 : 0));
      put_le(m, sizes[i], 8);
      m += 8;
      if (inl && sizes[i]) {
        memcpy(m, data[i], sizes[i]);
        m += sizes[i];
      }
    }
    sum[0] = lzo_fnv1a64(0xcbf29ce484222325ull, out + hsize, meta);
    for (uint32_t k = 1; k < n_entries; ++k) {
      if (len[k]) memcpy(out + off[k], src[k], len[k]);
      sum[k] = lzo_fnv1a64(0xcbf29ce484222325ull, out + off[k], len[k]);
    }
    lzo_header_serialize(n_entries, keys, klen, off, len, sum, out); /* header last */
  }
  free(keys);
  free(klen);
  free(off);
  free(len);
  free(sum);
  free(src);
  return total;
}

/* ---- plan: src/topology.cpp:100-185 ------------------------------------------- */
static uint64_t piece(uint64_t total, uint64_t parts, uint64_t i) {
  return total / parts + (i < total % parts ? 1 : 0);
}

int lzo_plan_rank(uint32_t dp, uint32_t pp, uint32_t tp, uint64_t params, uint32_t layers, uint32_t bpp_model,
                  uint32_t bpp_opt, uint32_t flat_rank, uint32_t* kind, uint64_t* size, uint32_t* first_layer,
                  uint32_t* layer_count, uint32_t* partition) {
  const uint32_t ranks = dp * pp * tp;
  const uint32_t rtp = flat_rank % tp, rpp = (flat_rank / tp) % pp, rdp = flat_rank / (tp * pp);
  /* stage rpp: contiguous layers; stage bytes = sum of per-layer param bytes */
  uint32_t first = 0;
  for (uint32_t s = 0; s < rpp; ++s) first += (uint32_t)piece(layers, pp, s);
  const uint32_t count = (uint32_t)piece(layers, pp, rpp);
  uint64_t stage_bytes = 0;
  for (uint32_t l = first; l < first + count; ++l) stage_bytes += piece(params, layers, l) * bpp_model;
  int n = 0;
  const uint32_t slice = rdp * tp + rtp;
  const uint64_t layer_slice = piece(stage_bytes, (uint64_t)tp * dp, slice);
  if (count > 0 && layer_slice > 0) {
    kind[n] = 0;
    size[n] = layer_slice;
    first_layer[n] = first;
    layer_count[n] = count;
    partition[n] = slice;
    ++n;
  }
  const uint64_t opt = piece(params * bpp_opt, ranks, flat_rank);
  if (opt > 0) {
    kind[n] = 1;
    size[n] = opt;
    first_layer[n] = 0;
    layer_count[n] = 0;
    partition[n] = flat_rank;
    ++n;
  }
  return n;
}

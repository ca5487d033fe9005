// K10: text example lines -> canonical hashed features (Fe:175-235, H:28-50),
// the step before the forward / training path.
//
// Line grammar (Fe:3-10): label ws '|' field_name (ws token[':' value])* ...
// The reference parses one line at a time in Python (~340 µs per line);
// here every line is independent:
//   A  fw_parse_lines, thread per line: label (Fe:223-229), '|' blocks,
//      ASCII-whitespace atoms (Fe:190), field-name lookup, values (Python
//      float() grammar: sign, digits with single '_' separators, '.', exponent;
//      non-finite rejected, Fe:201-208), raw '@digits' indices (Fe:209-214),
//      FNV-1a 32 of name 0x1F token masked to hash_bits (H:43-50), log1p for
//      numeric fields (Fe:33-39) -> raw (field, index, value) entries in token
//      order into a per-line scratch window (a token needs >= 2 bytes of line,
//      so len/2 + 1 entries always fit).
//   B  warp per line: bitonic sort of (field, index, token position) keys in
//      shared memory (<= 1024 features per line, else PS_TOO_LONG), duplicates
//      summed in occurrence order in f64 (Fe:219), per-field counts (<= 255);
//   C  exclusive scan of the per-line feature counts -> ex_off;
//   D  fw_parse_emit, warp per line: the canonical entries -> the ragged batch
//      (ex_off, cnt, idx i32, val f32 and optionally val f64) that K9 / K1 take.
// Values: exactly rounded on Clinger's fast path (<= 19 significant digits
// whose mantissa fits 2^53 and |exp10| <= 22 -- every short decimal); else a
// double-double product with 10^e (error ~2^-100 before the final rounding).
// Lines holding a byte sequence that decodes to Unicode (non-ASCII)
// whitespace, or non-ASCII bytes in a value or raw index, are rejected with
// PARSE_UNSUPPORTED instead of being tokenised differently from str.split().
#include <math.h>

#include "common.cuh"
#include "pow10_dd.h"

namespace dffm {

enum ParseStatus {
  PS_OK = 0, PS_LABEL = 1, PS_NO_BLOCKS = 2, PS_EMPTY_BLOCK = 3, PS_UNKNOWN_FIELD = 4,
  PS_BAD_VALUE = 5, PS_NONFINITE = 6, PS_RAW_RANGE = 7, PS_UNSUPPORTED = 8, PS_TOO_LONG = 9,
  PS_FIELD_CAP = 10, PS_BLANK = 11
};

constexpr int PB_WARPS = 2;
constexpr int PB_CAP = 1024;  // raw entries per line the sort stage takes

__device__ __forceinline__ bool is_ws(uint32_t c) {
  return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}

// exact m * 10^e10 for m < 2^53, |e10| <= 22 (Clinger: both operands exact, one
// IEEE rounding); else the double-double product (m_hi + m_lo)(t_hi + t_lo)
// rounded once (relative error ~2^-100 before that rounding).  Results below
// ~1e-290 are scaled through 10^-60 (a second rounding: subnormals may differ
// by one ulp).
__device__ double decimal_to_double(uint64_t m, int e10) {
  if (m == 0) return 0.0;
  if (m < (1ull << 53) && e10 >= -22 && e10 <= 22) {
    const double a = (double)m;
    return e10 >= 0 ? a * c_pow10_dd[e10 - POW10_MIN].x : a / c_pow10_dd[-e10 - POW10_MIN].x;
  }
  if (e10 > POW10_MAX) return INFINITY;
  if (e10 < -290) {
    if (e10 < -400) return 0.0;
    return decimal_to_double(m, e10 + 60) * 1e-60;
  }
  const double mh = (double)m;
  const double ml = (double)(int64_t)(m - (uint64_t)mh);  // exact remainder (|.| < 2^11)
  const double2 t = c_pow10_dd[e10 - POW10_MIN];
  const double ph = mh * t.x;
  const double pl = fma(mh, t.x, -ph) + (mh * t.y + ml * t.x);
  return ph + pl;
}

// Python float() over bytes [b, e) (no surrounding whitespace: atoms are
// whitespace-split).  Returns PS_OK / PS_BAD_VALUE / PS_NONFINITE / PS_UNSUPPORTED.
__device__ int parse_float(const uint8_t* s, int64_t b, int64_t e, double* out) {
  int64_t i = b;
  bool neg = false;
  if (i < e && (s[i] == '+' || s[i] == '-')) { neg = s[i] == '-'; ++i; }
  // inf / infinity / nan (any case): valid float() spellings, non-finite here
  {
    const int64_t L = e - i;
    auto lower = [&](int64_t k) { uint32_t c = s[i + k]; return (c >= 'A' && c <= 'Z') ? c + 32 : c; };
    if (L == 3 && ((lower(0) == 'i' && lower(1) == 'n' && lower(2) == 'f') ||
                   (lower(0) == 'n' && lower(1) == 'a' && lower(2) == 'n')))
      return PS_NONFINITE;
    if (L == 8) {
      const char* w = "infinity";
      bool m = true;
      for (int k = 0; k < 8; ++k) m &= lower(k) == (uint32_t)w[k];
      if (m) return PS_NONFINITE;
    }
  }
  uint64_t m = 0;
  int nd = 0;          // significant digits kept in m (<= 19)
  int drop = 0;        // integer digits dropped past 19 (scale up)
  int frac = 0;        // fraction digits kept (scale down)
  bool any = false, zero_lead = true;
  // integer part: digits with single '_' between digits
  int64_t j = i;
  bool prev_digit = false;
  for (; j < e; ++j) {
    const uint32_t c = s[j];
    if (c >= '0' && c <= '9') {
      any = true;
      prev_digit = true;
      if (zero_lead && c == '0') continue;
      zero_lead = false;
      if (nd < 19) { m = m * 10 + (c - '0'); ++nd; } else { ++drop; }
    } else if (c == '_') {
      if (!prev_digit || j + 1 >= e || s[j + 1] < '0' || s[j + 1] > '9') return PS_BAD_VALUE;
      prev_digit = false;
    } else {
      break;
    }
  }
  bool any_frac = false;
  if (j < e && s[j] == '.') {
    ++j;
    prev_digit = false;
    for (; j < e; ++j) {
      const uint32_t c = s[j];
      if (c >= '0' && c <= '9') {
        any_frac = true;
        prev_digit = true;
        if (zero_lead && c == '0') { ++frac; continue; }
        zero_lead = false;
        if (nd < 19) { m = m * 10 + (c - '0'); ++nd; ++frac; }
      } else if (c == '_') {
        if (!prev_digit || j + 1 >= e || s[j + 1] < '0' || s[j + 1] > '9') return PS_BAD_VALUE;
        prev_digit = false;
      } else {
        break;
      }
    }
  }
  if (!any && !any_frac) {
    for (int64_t k = i; k < e; ++k) if (s[k] >= 0x80) return PS_UNSUPPORTED;
    return PS_BAD_VALUE;
  }
  int64_t ex = 0;
  if (j < e && (s[j] == 'e' || s[j] == 'E')) {
    ++j;
    bool eneg = false;
    if (j < e && (s[j] == '+' || s[j] == '-')) { eneg = s[j] == '-'; ++j; }
    bool ed = false;
    prev_digit = false;
    for (; j < e; ++j) {
      const uint32_t c = s[j];
      if (c >= '0' && c <= '9') {
        ed = true;
        prev_digit = true;
        if (ex < 100000000) ex = ex * 10 + (c - '0');
      } else if (c == '_') {
        if (!prev_digit || j + 1 >= e || s[j + 1] < '0' || s[j + 1] > '9') return PS_BAD_VALUE;
        prev_digit = false;
      } else {
        break;
      }
    }
    if (!ed) return PS_BAD_VALUE;
    if (eneg) ex = -ex;
  }
  if (j != e) {
    for (int64_t k = i; k < e; ++k) if (s[k] >= 0x80) return PS_UNSUPPORTED;
    return PS_BAD_VALUE;
  }
  double v;
  if (m == 0) {
    v = 0.0;
  } else {
    int64_t e10 = ex + drop - frac;
    if (e10 > 400) v = INFINITY;
    else if (e10 < -420) v = 0.0;
    else v = decimal_to_double(m, (int)e10);
  }
  if (!isfinite(v)) return PS_NONFINITE;
  *out = neg ? -v : v;
  return PS_OK;
}

// the Unicode whitespace code points str.split() also splits on, as UTF-8
__device__ __forceinline__ bool unicode_ws_at(const uint8_t* s, int64_t p, int64_t e) {
  const uint32_t c0 = s[p];
  if (c0 == 0xC2 && p + 1 < e) return s[p + 1] == 0x85 || s[p + 1] == 0xA0;
  if (c0 == 0xE1 && p + 2 < e) return s[p + 1] == 0x9A && s[p + 2] == 0x80;
  if (c0 == 0xE2 && p + 2 < e) {
    const uint32_t c1 = s[p + 1], c2 = s[p + 2];
    if (c1 == 0x80) return (c2 >= 0x80 && c2 <= 0x8A) || c2 == 0xA8 || c2 == 0xA9 || c2 == 0xAF;
    if (c1 == 0x81) return c2 == 0x9F;
    return false;
  }
  if (c0 == 0xE3 && p + 2 < e) return s[p + 1] == 0x80 && s[p + 2] == 0x80;
  return false;
}

struct ParseParams {
  const uint8_t* text;
  const int64_t* line_off;
  int64_t n;
  const uint8_t* names;
  const int32_t* name_off;
  const uint8_t* numeric;
  int F;
  int hash_bits;
  uint64_t* ent_key;  // (fid << 40) | (index << 11) | token position   (scratch)
  double* ent_val;    // scratch
  int32_t* ent_n;     // [n] raw entries, then canonical entries per line
  uint8_t* labels;
  int32_t* status;
};

__device__ __forceinline__ int64_t ent_base(const ParseParams& p, int64_t i) {
  return (p.line_off[i] - p.line_off[0]) / 2 + i;
}

// first q in [from, e) with s[q] == c, else e; aligned 8-byte words, bytes only
// in a word that may hold c (the zero-byte test has no false negatives)
__device__ __forceinline__ int64_t find_byte(const uint8_t* s, int64_t from, int64_t e,
                                             uint32_t c) {
  int64_t q = from;
  const int64_t head = (int64_t)((8 - ((uintptr_t)(s + q) & 7)) & 7);
  for (const int64_t qa = q + head < e ? q + head : e; q < qa; ++q)
    if (s[q] == c) return q;
  const uint64_t pat = 0x0101010101010101ull * c;
  for (; q + 8 <= e; q += 8) {
    const uint64_t x = *reinterpret_cast<const uint64_t*>(s + q) ^ pat;
    if ((x - 0x0101010101010101ull) & ~x & 0x8080808080808080ull) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (((x >> (8 * k)) & 0xffu) == 0) return q + k;
    }
  }
  for (; q < e; ++q)
    if (s[q] == c) return q;
  return e;
}

__global__ void __launch_bounds__(128) parse_lines_kernel(ParseParams p) {
  // schema lookup table: (name length << 32) | FNV-1a of the name, per field
  __shared__ uint64_t ftab[256];
  for (int f = threadIdx.x; f < p.F; f += blockDim.x) {
    const int32_t o0 = p.name_off[f], o1 = p.name_off[f + 1];
    uint32_t h = 0x811C9DC5u;
    for (int32_t k = o0; k < o1; ++k) h = (h ^ p.names[k]) * 0x01000193u;
    ftab[f] = ((uint64_t)(uint32_t)(o1 - o0) << 32) | h;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  const uint8_t* s = p.text;
  const int64_t b = p.line_off[i], e = p.line_off[i + 1];
  const int64_t eb = ent_base(p, i);
  int st = PS_OK, ne = 0;
  uint8_t label = 0;
  // unsupported (non-ASCII whitespace) anywhere in the line; whitespace-only
  // lines are "blank" (skipped by the stream loops, T:176)
  // (8-byte words where aligned: an all-ASCII word needs no per-byte reload)
  bool blank = true;
  {
    const int64_t head = (int64_t)((8 - ((uintptr_t)(s + b) & 7)) & 7);
    const int64_t qa = b + head < e ? b + head : e;
    int64_t q = b;
    for (; q < qa && st == PS_OK; ++q) {
      blank &= is_ws(s[q]);
      if (s[q] >= 0xC2 && unicode_ws_at(s, q, e)) st = PS_UNSUPPORTED;
    }
    for (; q + 8 <= e && st == PS_OK; q += 8) {
      const uint64_t w = *reinterpret_cast<const uint64_t*>(s + q);
      if (w & 0x8080808080808080ull) {
        for (int k = 0; k < 8 && st == PS_OK; ++k) {
          blank &= is_ws(s[q + k]);
          if (s[q + k] >= 0xC2 && unicode_ws_at(s, q + k, e)) st = PS_UNSUPPORTED;
        }
      } else if (blank) {
#pragma unroll
        for (int k = 0; k < 8; ++k) blank &= is_ws((uint32_t)(w >> (8 * k)) & 0xffu);
      }
    }
    for (; q < e && st == PS_OK; ++q) {
      blank &= is_ws(s[q]);
      if (s[q] >= 0xC2 && unicode_ws_at(s, q, e)) st = PS_UNSUPPORTED;
    }
  }
  if (st == PS_OK && blank) st = PS_BLANK;
  // label (Fe:223-229)
  const int64_t bar = find_byte(s, b, e, '|');
  if (st == PS_OK) {
    int64_t h0 = b, h1 = bar;
    while (h0 < h1 && is_ws(s[h0])) ++h0;
    while (h1 > h0 && is_ws(s[h1 - 1])) --h1;
    const int64_t L = h1 - h0;
    if (L == 1 && s[h0] == '1') label = 1;
    else if ((L == 1 && s[h0] == '0') || (L == 2 && s[h0] == '-' && s[h0 + 1] == '1')) label = 0;
    else st = PS_LABEL;
    if (st == PS_OK && bar >= e) st = PS_NO_BLOCKS;
  }
  const uint32_t mask = (uint32_t)((1ull << p.hash_bits) - 1);
  const int64_t max_index = 1ll << p.hash_bits;
  int64_t q = bar;
  while (st == PS_OK && q < e) {  // one '|' block per iteration; q at its '|'
    const int64_t se = find_byte(s, q + 1, e, '|');
    int64_t a = q + 1;
    while (a < se && is_ws(s[a])) ++a;
    if (a >= se) { st = PS_EMPTY_BLOCK; break; }
    int64_t ae = a;
    uint32_t hname = 0x811C9DC5u;
    for (; ae < se; ++ae) {
      const uint32_t c = s[ae];
      if (is_ws(c)) break;
      hname = (hname ^ c) * 0x01000193u;
    }
    // field name lookup (InputSchema.field_id): the first field whose name equals
    // the atom; fields whose (length, hash) differ cannot, the rest are compared
    int fid = -1;
    const int64_t nl = ae - a;
    const uint64_t key = nl <= 0xFFFFFFFFll ? ((uint64_t)nl << 32) | hname : ~0ull;
    for (int f = 0; f < p.F && fid < 0; ++f) {
      if (ftab[f] != key) continue;
      const int32_t o0 = p.name_off[f];
      bool eq = true;
      for (int64_t k = 0; k < nl && eq; ++k) eq = p.names[o0 + k] == s[a + k];
      if (eq) fid = f;
    }
    if (fid < 0) { st = PS_UNKNOWN_FIELD; break; }
    hname = (hname ^ 0x1Fu) * 0x01000193u;
    const bool numeric = p.numeric[fid] != 0;
    int64_t t = ae;
    while (st == PS_OK) {  // atoms after the name
      while (t < se && is_ws(s[t])) ++t;
      if (t >= se) break;
      // one pass over the atom: its end, its first ':' and the FNV-1a of the
      // bytes before it (used when the atom is not a raw @index)
      int64_t te = t, colon = -1;
      uint32_t htok = hname;
      for (; te < se; ++te) {
        const uint32_t c = s[te];
        if (is_ws(c)) break;
        if (colon < 0) {
          if (c == ':') colon = te;
          else htok = (htok ^ c) * 0x01000193u;
        }
      }
      if (colon < 0) colon = te;
      double value = 1.0;
      if (colon < te) {
        const int r = parse_float(s, colon + 1, te, &value);
        if (r != PS_OK) { st = r; break; }
      }
      int64_t index;
      bool raw = s[t] == '@' && colon - t >= 2;
      for (int64_t k = t + 1; raw && k < colon; ++k) {
        if (s[k] >= 0x80) { st = PS_UNSUPPORTED; break; }
        raw = s[k] >= '0' && s[k] <= '9';
      }
      if (st != PS_OK) break;
      if (raw) {  // Fe:209-214
        int64_t v = 0;
        bool big = false;
        for (int64_t k = t + 1; k < colon; ++k) {
          v = v * 10 + (s[k] - '0');
          if (v >= max_index) { big = true; break; }
        }
        if (big) { st = PS_RAW_RANGE; break; }
        index = v;
      } else {  // H:43-50 (+ Fe:215-218 numeric transform)
        index = htok & mask;
        if (numeric && value > 0) value = log1p(value);
      }
      p.ent_key[eb + ne] = ((uint64_t)fid << 40) | ((uint64_t)index << 11) | (uint64_t)ne;
      p.ent_val[eb + ne] = value;
      ++ne;
      t = te;
    }
    q = se;
  }
  if (st == PS_OK && ne > PB_CAP) st = PS_TOO_LONG;
  p.labels[i] = label;
  p.status[i] = st;
  p.ent_n[i] = st == PS_OK ? ne : 0;
}

// B: per line, sort the raw entries by (field, index, position), sum
// duplicates in occurrence order, count per field; canonical entries are
// written back to the line's scratch window
// Two tiers: <CAP_S, 8 warps> takes every line with <= CAP_S raw entries (the
// common case, many warps per SM), <PB_CAP, 2 warps> then takes the rest (a
// line is processed by the tier whose range holds its raw count LO < ne <= CAP;
// processed lines hold their canonical count <= their raw count afterwards).
template <int CAP, int WARPS, int LO>
__global__ void __launch_bounds__(WARPS * 32) parse_canon_kernel(ParseParams p, uint8_t* cnt,
                                                                 int32_t* max_cnt) {
  __shared__ uint64_t key[WARPS][CAP];
  __shared__ double sval[WARPS][CAP];
  __shared__ int fcnt[WARPS][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* k = key[warp];
  double* sv = sval[warp];
  int* fc = fcnt[warp];
  auto line = [&](int64_t i, int ne) {
    const int64_t eb = ent_base(p, i);
    for (int f = lane; f < p.F; f += 32) fc[f] = 0;
    int np2 = 1;
    while (np2 < ne) np2 <<= 1;
    if (np2 <= 64) {
      // keys unique (position in the low bits): bitonic sort of 64 in registers,
      // element t = lane + 32 j in slot j, partners by shuffle (stride < 32)
      uint64_t r0 = lane < ne ? p.ent_key[eb + lane] : ~0ull;
      uint64_t r1 = lane + 32 < ne ? p.ent_key[eb + lane + 32] : ~0ull;
      if (lane < ne) sv[lane] = p.ent_val[eb + lane];
      if (lane + 32 < ne) sv[lane + 32] = p.ent_val[eb + lane + 32];
#pragma unroll
      for (int size = 2; size <= 64; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          if (stride == 32) {  // size 64: slot 0 (t < 32) keeps the min
            const uint64_t lo = r0 < r1 ? r0 : r1, hi = r0 < r1 ? r1 : r0;
            r0 = lo, r1 = hi;
          } else {
            const bool lower = (lane & stride) == 0;
            const uint64_t y0 = __shfl_xor_sync(0xffffffffu, r0, stride);
            const uint64_t y1 = __shfl_xor_sync(0xffffffffu, r1, stride);
            const bool up0 = (lane & size) == 0, up1 = ((lane + 32) & size) == 0;
            r0 = (lower == up0) ? (r0 < y0 ? r0 : y0) : (r0 < y0 ? y0 : r0);
            r1 = (lower == up1) ? (r1 < y1 ? r1 : y1) : (r1 < y1 ? y1 : r1);
          }
        }
      }
      k[lane] = r0;
      k[lane + 32] = r1;
      __syncwarp();
      np2 = 0;  // sorted: skip the shared-memory network below
    } else {
      for (int t = lane; t < np2; t += 32) {
        k[t] = t < ne ? p.ent_key[eb + t] : ~0ull;
        if (t < ne) sv[t] = p.ent_val[eb + t];
      }
      __syncwarp();
    }
    for (int size = 2; size <= np2; size <<= 1) {  // bitonic sort, ascending
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = lane; t < np2; t += 32) {
          const int u = t ^ stride;
          if (u > t) {
            const uint64_t x = k[t], y = k[u];
            const bool up = (t & size) == 0;
            if ((x > y) == up) { k[t] = y; k[u] = x; }
          }
        }
        __syncwarp();
      }
    }
    // runs of equal (field, index): the run's first lane sums it in position order
    int nu = 0;
    for (int t0 = 0; t0 < ne; t0 += 32) {
      const int t = t0 + lane;
      bool start = false;
      uint64_t kk = 0;
      if (t < ne) {
        kk = k[t] >> 11;
        start = t == 0 || (k[t - 1] >> 11) != kk;
      }
      const uint32_t bm = __ballot_sync(0xffffffffu, start);
      if (start) {
        double v = 0.0;
        for (int r = t; r < ne && (k[r] >> 11) == kk; ++r) v += sv[k[r] & 2047];  // Fe:219 order
        const int u = nu + __popc(bm & ((1u << lane) - 1u));
        p.ent_val[eb + u] = v;  // raw entries live in shared memory now
        p.ent_key[eb + u] = kk;
        atomicAdd(&fc[(int)(kk >> 29)], 1);
      }
      nu += __popc(bm);
    }
    __syncwarp();
    int big = 0, mx = 0;
    for (int f = lane; f < p.F; f += 32) {
      const int c = fc[f];
      big |= c > 255;
      mx = max(mx, c);
      cnt[i * p.F + f] = (uint8_t)min(c, 255);
    }
    big = __any_sync(0xffffffffu, big);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
      if (big && p.status[i] == PS_OK) p.status[i] = PS_FIELD_CAP;
      p.ent_n[i] = big ? 0 : nu;
      if (!big) atomicMax(max_cnt, mx);
    }
    if (big)
      for (int f = lane; f < p.F; f += 32) cnt[i * p.F + f] = 0;
    __syncwarp();
  };
  const int64_t w0 = (int64_t)blockIdx.x * WARPS + warp, nw = (int64_t)gridDim.x * WARPS;
  if (LO == 0) {
    for (int64_t i = w0; i < p.n; i += nw) {
      const int ne = p.ent_n[i];
      if (ne <= CAP) line(i, ne);  // longer lines: the other tier's
    }
  } else {
    // the long-line tier sees few lines: 32 counts per coalesced load, a ballot
    // picks this tier's lines
    for (int64_t g = w0 * 32; g < p.n; g += nw * 32) {
      const int64_t il = g + lane;
      const int nel = il < p.n ? p.ent_n[il] : 0;
      uint32_t pend = __ballot_sync(0xffffffffu, nel > LO && nel <= CAP);
      while (pend) {
        const int b = __ffs(pend) - 1;
        pend &= pend - 1;
        line(g + b, __shfl_sync(0xffffffffu, nel, b));
      }
    }
  }
}

// C: ex_off = exclusive scan of the canonical counts: per-tile sums, a scan of
// the tile sums in one CTA, then each tile's local scan plus its offset
constexpr int SC_TILE = 4096;
__global__ void __launch_bounds__(256) parse_tile_sum_kernel(const int32_t* ent_n, int64_t n,
                                                             int64_t* tsum) {
  __shared__ int64_t red[8];
  const int64_t b = (int64_t)blockIdx.x * SC_TILE;
  int64_t s = 0;
  for (int64_t i = b + threadIdx.x; i < min(n, b + SC_TILE); i += 256) s += ent_n[i];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < 8; ++w) t += red[w];
    tsum[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) parse_tile_scan_kernel(int64_t* tsum, int64_t ntiles,
                                                               int64_t* total) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t per = (ntiles + 1023) / 1024;
  const int64_t b = t * per, e = min(ntiles, b + per);
  int64_t s = 0;
  for (int64_t i = b; i < e; ++i) s += tsum[i];
  part[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = t ? part[t - 1] : 0;
  for (int64_t i = b; i < e; ++i) { const int64_t v = tsum[i]; tsum[i] = run; run += v; }
  if (t == 1023) *total = part[1023];
}

__global__ void __launch_bounds__(256) parse_tile_apply_kernel(const int32_t* ent_n, int64_t n,
                                                               const int64_t* tsum,
                                                               int64_t* ex_off) {
  __shared__ int64_t wsum[8];
  const int64_t b = (int64_t)blockIdx.x * SC_TILE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t run = tsum[blockIdx.x];
  for (int64_t c0 = b; c0 < min(n, b + SC_TILE); c0 += 256) {
    const int64_t i = c0 + threadIdx.x;
    const int64_t v = i < n ? ent_n[i] : 0;
    int64_t x = v;  // inclusive scan within the warp, then across the 8 warps
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int64_t before = 0, all = 0;
    for (int w = 0; w < 8; ++w) {
      if (w < warp) before += wsum[w];
      all += wsum[w];
    }
    if (i < n) ex_off[i] = run + before + x - v;
    run += all;
    __syncthreads();
  }
}

// D: canonical entries -> ragged batch arrays
__global__ void __launch_bounds__(256) parse_emit_kernel(ParseParams p, const int64_t* ex_off,
                                                         int32_t* idx, float* val, double* val64) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < p.n; i += (int64_t)gridDim.x * 8) {
    const int nu = p.ent_n[i];
    const int64_t eb = ent_base(p, i), o = ex_off[i];
    for (int u = lane; u < nu; u += 32) {
      const uint64_t kk = p.ent_key[eb + u];
      idx[o + u] = (int32_t)(kk & ((1ull << 29) - 1));
      const double v = p.ent_val[eb + u];
      val[o + u] = (float)v;
      if (val64) val64[o + u] = v;
    }
  }
}

}  // namespace dffm

using namespace dffm;

static ParseParams parse_params(const int64_t* line_off, int64_t n, int64_t text_bytes,
                                void* scratch) {
  ParseParams p{};
  p.line_off = line_off;
  p.n = n;
  const int64_t cap = text_bytes / 2 + n + 1;
  p.ent_key = (uint64_t*)scratch;
  p.ent_val = (double*)(p.ent_key + cap);
  p.ent_n = (int32_t*)(p.ent_val + cap);
  return p;
}

extern "C" int64_t fw_parse_scratch_bytes(int64_t n_lines, int64_t text_bytes) {
  const int64_t cap = text_bytes / 2 + n_lines + 1;
  return cap * 16 + n_lines * 4 + 256 + ((n_lines + SC_TILE - 1) / SC_TILE) * 8 + 16;
}

extern "C" int fw_parse_lines(const uint8_t* text, const int64_t* line_off, int64_t n_lines,
                              int64_t text_bytes, const uint8_t* names, const int32_t* name_off,
                              const uint8_t* numeric, int32_t n_fields, int32_t hash_bits,
                              void* scratch, uint8_t* labels, int32_t* line_status, uint8_t* cnt,
                              int64_t* ex_off, int32_t* max_cnt, void* stream) {
  if (n_lines < 0 || n_fields < 1 || n_fields > 255 || hash_bits < 1 || hash_bits > 29) {
    set_error("bad parse args (n=%lld F=%d bits=%d)", (long long)n_lines, n_fields, hash_bits);
    return DFFM_CONTRACT;
  }
  if (!text || !line_off || !names || !name_off || !numeric || !scratch || !labels ||
      !line_status || !cnt || !ex_off || !max_cnt) {
    set_error("null buffer");
    return DFFM_CONTRACT;
  }
  cudaStream_t s = (cudaStream_t)stream;
  DFFM_CUDA_TRY(cudaMemsetAsync(max_cnt, 0, 4, s), "memset(max_cnt)");
  if (!n_lines) {
    DFFM_CUDA_TRY(cudaMemsetAsync(ex_off, 0, 8, s), "memset(ex_off)");
    return DFFM_OK;
  }
  ParseParams p = parse_params(line_off, n_lines, text_bytes, scratch);
  p.text = text;
  p.names = names;
  p.name_off = name_off;
  p.numeric = numeric;
  p.F = n_fields;
  p.hash_bits = hash_bits;
  p.labels = labels;
  p.status = line_status;
  note_launches(1), parse_lines_kernel<<<(unsigned)((n_lines + 127) / 128), 128, 0, s>>>(p);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(parse_lines)");
  const int64_t sms = sm_count_current();
  constexpr int CAP_S = 128;
  const unsigned g1 = (unsigned)std::min<int64_t>((n_lines + 7) / 8, sms * 8);
  note_launches(1), parse_canon_kernel<CAP_S, 8, 0><<<g1, 256, 0, s>>>(p, cnt, max_cnt);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(parse_canon)");
  const unsigned gb = (unsigned)std::min<int64_t>((n_lines + PB_WARPS - 1) / PB_WARPS, sms * 16);
  note_launches(1), parse_canon_kernel<PB_CAP, PB_WARPS, CAP_S><<<gb, PB_WARPS * 32, 0, s>>>(
      p, cnt, max_cnt);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(parse_canon long lines)");
  // ex_off via tile sums: the tile-sum array lives past the ent_n array in scratch
  const int64_t ntiles = (n_lines + SC_TILE - 1) / SC_TILE;
  int64_t* tsum = (int64_t*)(((uintptr_t)(p.ent_n + n_lines) + 15) & ~(uintptr_t)15);
  note_launches(1), parse_tile_sum_kernel<<<(unsigned)ntiles, 256, 0, s>>>(p.ent_n, n_lines, tsum);
  note_launches(1), parse_tile_scan_kernel<<<1, 1024, 0, s>>>(tsum, ntiles, ex_off + n_lines);
  note_launches(1), parse_tile_apply_kernel<<<(unsigned)ntiles, 256, 0, s>>>(p.ent_n, n_lines, tsum,
                                                                          ex_off);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(parse_scan)");
  return DFFM_OK;
}

extern "C" int fw_parse_emit(const int64_t* line_off, int64_t n_lines, int64_t text_bytes,
                             const void* scratch, const int64_t* ex_off, int32_t* idx, float* val,
                             double* val64_opt, void* stream) {
  if (n_lines < 0) { set_error("bad n_lines"); return DFFM_CONTRACT; }
  if (!n_lines) return DFFM_OK;
  if (!line_off || !scratch || !ex_off || !idx || !val) { set_error("null buffer"); return DFFM_CONTRACT; }
  ParseParams p = parse_params(line_off, n_lines, text_bytes, const_cast<void*>(scratch));
  const int64_t sms = sm_count_current();
  const unsigned g = (unsigned)std::min<int64_t>((n_lines + 7) / 8, sms * 16);
  note_launches(1), parse_emit_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(p, ex_off, idx, val,
                                                                         val64_opt);
  DFFM_CUDA_TRY(cudaGetLastError(), "launch(parse_emit)");
  return DFFM_OK;
}

/*
 * oracle/fier_oracle.c -- CPU restatement of the reference's Fier hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library, and only as the
 * checker (or the timed CPU baseline); the product path never calls it.
 *
 * Parity is pinned: tests/test_oracle.py checks every function below against
 * (a) the reference's own known-answer tests restated in tests/golden/kats.json
 * (test_io.cpp:25-98, test_quant1bit.cpp:48-122, test_kvcore.cpp:84-94) and
 * (b) fixtures produced by the reference itself, compiled here from
 * /root/reference/proj/include by oracle/Makefile into oracle/_ref/
 * (tests/golden/make_golden.py).
 *
 * Arithmetic is IEEE fp64 with contraction disabled (-ffp-contract=off), the
 * same evaluation order as the reference, so results are bit-identical to the
 * reference's default (non-FMA x86-64) build.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define FO_OK 0
#define FO_EINVAL 1
#define FO_EDATA 2

/* ---- binary16 (half.hpp) --------------------------------------------------- */

/* half.hpp:13-28: exact widening. */
double fo_half_to_double(uint16_t h) {
    const uint16_t sign = h & 0x8000u;
    const uint16_t ex = (h >> 10) & 0x1Fu;
    const uint16_t frac = h & 0x03FFu;
    double mag;
    if (ex == 0) {
        mag = (double)frac * 0x1.0p-24;
    } else if (ex == 31) {
        mag = frac == 0 ? INFINITY : NAN;
    } else {
        mag = ldexp(1024.0 + frac, (int)ex - 25);
    }
    return sign ? -mag : mag;
}

/* half.hpp:30-61: round to nearest even, >= 65520 -> inf, NaN -> 0x7E00. */
uint16_t fo_double_to_half(double x) {
    uint64_t bits;
    memcpy(&bits, &x, sizeof bits);
    const uint16_t sign = (uint16_t)((bits >> 48) & 0x8000u);
    const uint64_t a = bits & 0x7FFFFFFFFFFFFFFFull;
    if (a > 0x7FF0000000000000ull) return sign | 0x7E00u;
    if (a >= 0x40EFFE0000000000ull) return sign | 0x7C00u;
    const int e = (int)(a >> 52) - 1023;
    if (e < -1022) return sign;
    uint64_t sig = (a & 0xFFFFFFFFFFFFFull) | (1ull << 52);
    int shift = 42;
    if (e < -14) shift += -14 - e;
    if (shift >= 64) return sign;
    uint64_t kept = sig >> shift;
    const uint64_t rem = sig & ((1ull << shift) - 1);
    const uint64_t halfway = 1ull << (shift - 1);
    if (rem > halfway || (rem == halfway && (kept & 1))) ++kept;
    uint16_t out;
    if (e < -14) out = (uint16_t)kept;
    else out = (uint16_t)(((uint64_t)(e + 15) << 10) + (kept - 1024));
    return sign | out;
}

/* ---- 1-bit quantizer (quant1bit.hpp) ----------------------------------------- */

size_t fo_words_per_row(size_t d) { return (d + 63) / 64; }          /* quant1bit.hpp:44 */
size_t fo_groups(size_t l, size_t g) { return (l + g - 1) / g; }     /* quant1bit.hpp:75 */
size_t fo_payload_bytes(size_t l, size_t d, size_t g) {               /* quant1bit.hpp:60-62 */
    return l * ((d + 7) / 8) + d * fo_groups(l, g) * 4;
}

/*
 * quant1bit.hpp:65-103.  K is row-major l x d fp64.  code_words: l * ceil(d/64)
 * u64 (zeroed here), scales/zeros: ceil(l/g) * d fp64 indexed [gi*d + j].
 */
int fo_quantize(const double* K, size_t l, size_t d, size_t g, uint64_t* code_words,
                double* scales, double* zeros) {
    if (g < 1) return FO_EINVAL;                    /* :66 */
    if (l < 1 || d < 1) return FO_EINVAL;           /* :67 */
    for (size_t i = 0; i < l * d; ++i)              /* :68 */
        if (!isfinite(K[i])) return FO_EINVAL;
    const size_t wpr = fo_words_per_row(d), G = fo_groups(l, g);
    memset(code_words, 0, l * wpr * sizeof(uint64_t));
    for (size_t j = 0; j < d; ++j) {
        for (size_t gi = 0; gi < G; ++gi) {
            const size_t t0 = gi * g;
            const size_t t1 = (t0 + g < l) ? t0 + g : l;  /* :84 short final group */
            double mn = K[t0 * d + j], mx = mn;
            for (size_t t = t0 + 1; t < t1; ++t) {
                const double v = K[t * d + j];
                mn = (v < mn) ? v : mn;  /* std::min(mn, v): first seen wins ties */
                mx = (mx < v) ? v : mx;  /* std::max(mx, v) */
            }
            const double z = (mx + mn) / 2.0;
            const double s = (mx - mn) / 2.0;
            scales[gi * d + j] = s;
            zeros[gi * d + j] = z;
            for (size_t t = t0; t < t1; ++t) {
                if (s == 0.0 || K[t * d + j] >= z)  /* :96 */
                    code_words[t * wpr + j / 64] |= (uint64_t)1 << (j % 64);
            }
        }
    }
    return FO_OK;
}

/* io.hpp:197-225: FIER serialization.  out must hold 18 + payload bytes. */
size_t fo_serialize_packed(size_t l, size_t d, size_t g, const uint64_t* code_words,
                           const double* scales, const double* zeros, unsigned char* out) {
    const size_t G = fo_groups(l, g), wpr = fo_words_per_row(d);
    size_t p = 0;
    memcpy(out, "FIER", 4); p = 4;
    out[p++] = 1; out[p++] = 0;  /* version u16 */
    const uint32_t hdr[3] = {(uint32_t)l, (uint32_t)d, (uint32_t)g};
    for (int i = 0; i < 3; ++i)
        for (int b = 0; b < 4; ++b) out[p++] = (unsigned char)((hdr[i] >> (8 * b)) & 0xFF);
    for (size_t j = 0; j < d; ++j) {
        for (size_t gi = 0; gi < G; ++gi) {
            const uint16_t hs = fo_double_to_half(scales[gi * d + j]);
            const uint16_t hz = fo_double_to_half(zeros[gi * d + j]);
            out[p++] = hs & 0xFF; out[p++] = hs >> 8;
            out[p++] = hz & 0xFF; out[p++] = hz >> 8;
        }
    }
    const size_t row_bytes = (d + 7) / 8;
    for (size_t t = 0; t < l; ++t) {
        for (size_t b = 0; b < row_bytes; ++b) {
            unsigned char byte = 0;
            for (size_t bit = 0; bit < 8; ++bit) {
                const size_t j = b * 8 + bit;
                if (j < d && ((code_words[t * wpr + j / 64] >> (j % 64)) & 1u)) byte |= (unsigned char)(1u << bit);
            }
            out[p++] = byte;
        }
    }
    return p;
}

static uint32_t rd_u32(const unsigned char* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

/* io.hpp:227-277: header fields of a FIER buffer (no payload decode). */
int fo_parse_header(const unsigned char* buf, size_t len, size_t* l, size_t* d, size_t* g) {
    if (len < 4 || memcmp(buf, "FIER", 4) != 0) return FO_EDATA;
    if (len < 18) return FO_EDATA;
    if ((buf[4] | (buf[5] << 8)) != 1) return FO_EDATA;
    *l = rd_u32(buf + 6); *d = rd_u32(buf + 10); *g = rd_u32(buf + 14);
    if (*l == 0 || *d == 0 || *g == 0) return FO_EDATA;
    if (len - 18 != fo_payload_bytes(*l, *d, *g)) return FO_EDATA;
    return FO_OK;
}

/* io.hpp:227-277: decode into in-memory form with half-rounded parameters. */
int fo_parse_packed(const unsigned char* buf, size_t len, uint64_t* code_words, double* scales,
                    double* zeros) {
    size_t l, d, g;
    int rc = fo_parse_header(buf, len, &l, &d, &g);
    if (rc) return rc;
    const size_t G = fo_groups(l, g), wpr = fo_words_per_row(d);
    const unsigned char* p = buf + 18;
    for (size_t j = 0; j < d; ++j) {
        for (size_t gi = 0; gi < G; ++gi) {
            scales[gi * d + j] = fo_half_to_double((uint16_t)(p[0] | (p[1] << 8)));
            zeros[gi * d + j] = fo_half_to_double((uint16_t)(p[2] | (p[3] << 8)));
            p += 4;
        }
    }
    memset(code_words, 0, l * wpr * sizeof(uint64_t));
    const size_t row_bytes = (d + 7) / 8;
    for (size_t t = 0; t < l; ++t) {
        for (size_t b = 0; b < row_bytes; ++b) {
            const unsigned char byte = p[b];
            for (size_t bit = 0; bit < 8; ++bit) {
                const size_t j = b * 8 + bit;
                if (j < d && (byte & (1u << bit))) code_words[t * wpr + j / 64] |= (uint64_t)1 << (j % 64);
            }
        }
        p += row_bytes;
    }
    return FO_OK;
}

/* quant1bit.hpp:121-140: estimated logits, channel order, no K~ materialized. */
void fo_approx_scores(const double* q, size_t l, size_t d, size_t g, const uint64_t* code_words,
                      const double* scales, const double* zeros, double* out) {
    const size_t wpr = fo_words_per_row(d);
    for (size_t t = 0; t < l; ++t) {
        const size_t grow = (t / g) * d;
        const uint64_t* w = code_words + t * wpr;
        double acc = 0.0;
        for (size_t j = 0; j < d; ++j) {
            const double s = scales[grow + j], z = zeros[grow + j];
            const int bit = (int)((w[j / 64] >> (j % 64)) & 1u);
            acc += q[j] * ((bit ? s : -s) + z);
        }
        out[t] = acc;
    }
}

/* core.hpp:98-112 */
void fo_exact_scores(const double* q, const double* K, size_t l, size_t d, int scaled, double* out) {
    const double inv = scaled ? 1.0 / sqrt((double)d) : 1.0;
    for (size_t i = 0; i < l; ++i) {
        double acc = 0.0;
        for (size_t j = 0; j < d; ++j) acc += q[j] * K[i * d + j];
        out[i] = acc * inv;
    }
}

/* core.hpp:134-148: k largest; ties -> lower index; output ascending. */
static int cmp_desc(const void* a, const void* b, void* arg) {
    const double* sc = (const double*)arg;
    const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
    const double sa = sc[ia], sb = sc[ib];
    if (sa != sb) return sa > sb ? -1 : 1;
    return ia < ib ? -1 : (ia > ib);
}
static int cmp_asc(const void* a, const void* b) {
    const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
    return ia < ib ? -1 : (ia > ib);
}
int fo_topk(const double* scores, size_t l, size_t k, int64_t* out) {
    if (k < 1 || k > l) return FO_EINVAL;  /* core.hpp:136 */
    int64_t* order = (int64_t*)malloc(l * sizeof(int64_t));
    if (!order) return FO_EINVAL;
    for (size_t i = 0; i < l; ++i) order[i] = (int64_t)i;
    qsort_r(order, l, sizeof(int64_t), cmp_desc, (void*)scores);
    memcpy(out, order, k * sizeof(int64_t));
    qsort(out, k, sizeof(int64_t), cmp_asc);
    free(order);
    return FO_OK;
}

/* core.hpp:152-179 (softmax core.hpp:115-130). */
int fo_gather_attention(const double* q, const double* K, const double* V, size_t l, size_t d,
                        const int64_t* idx, size_t n, int scaled, double* out) {
    if (n == 0) return FO_EINVAL;                                   /* :158 */
    for (size_t s = 0; s < n; ++s) {                                /* :159 valid_against */
        if (idx[s] < 0 || (size_t)idx[s] >= l) return FO_EINVAL;
        if (s > 0 && idx[s] <= idx[s - 1]) return FO_EINVAL;
    }
    double* w = (double*)malloc(n * sizeof(double));
    if (!w) return FO_EINVAL;
    const double inv = scaled ? 1.0 / sqrt((double)d) : 1.0;
    for (size_t s = 0; s < n; ++s) {
        const double* k = K + (size_t)idx[s] * d;
        double acc = 0.0;
        for (size_t j = 0; j < d; ++j) acc += q[j] * k[j];
        w[s] = acc * inv;
    }
    double mx = w[0];
    for (size_t s = 1; s < n; ++s) mx = (mx < w[s]) ? w[s] : mx;  /* std::max_element */
    if (!isfinite(mx)) { free(w); return FO_EINVAL; }                /* :122 */
    double sum = 0.0;
    for (size_t s = 0; s < n; ++s) { w[s] = exp(w[s] - mx); sum += w[s]; }
    for (size_t s = 0; s < n; ++s) w[s] /= sum;
    for (size_t j = 0; j < d; ++j) out[j] = 0.0;
    for (size_t s = 0; s < n; ++s) {
        const double* v = V + (size_t)idx[s] * d;
        for (size_t j = 0; j < d; ++j) out[j] += w[s] * v[j];
    }
    free(w);
    return FO_OK;
}

/* evalharness.hpp:25-34 (recall on sorted selections). */
double fo_recall(const int64_t* got, const int64_t* want, size_t n) {
    size_t hit = 0, a = 0, b = 0;
    while (a < n && b < n) {
        if (got[a] == want[b]) { ++hit; ++a; ++b; }
        else if (got[a] < want[b]) ++a;
        else ++b;
    }
    return (double)hit / (double)n;
}

/* core.hpp:181-190 */
double fo_relative_l2_error(const double* got, const double* want, size_t n) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < n; ++i) {
        num += (got[i] - want[i]) * (got[i] - want[i]);
        den += want[i] * want[i];
    }
    if (den == 0.0) return num == 0.0 ? 0.0 : INFINITY;
    return sqrt(num / den);
}

/*
 * fier_attend minus bookkeeping (retrieval.hpp:136-146) for one q head over a
 * pre-built (hoisted) index with half-rounded parameters: the
 * "port" CPU baseline.  scratch: l doubles + l int64.
 */
int fo_fier_attend(const double* q, const double* K, const double* V, size_t l, size_t d, size_t g,
                   const uint64_t* code_words, const double* scales, const double* zeros, size_t n,
                   int64_t* sel_out, double* out) {
    if (n < 1 || n > l) return FO_EINVAL;
    double* est = (double*)malloc(l * sizeof(double));
    if (!est) return FO_EINVAL;
    fo_approx_scores(q, l, d, g, code_words, scales, zeros, est);
    int rc = fo_topk(est, l, n, sel_out);
    if (!rc) rc = fo_gather_attention(q, K, V, l, d, sel_out, n, 1, out);
    free(est);
    return rc;
}

/* ---- Quest page retrieval (baselines.hpp), SURVEY 8(f) row 2 ------------------- */

/* build_page_summaries (baselines.hpp:34-56): per page, channel-wise min / max of the
 * page's actual members (the last page may be short).  kmax/kmin: [ceil(l/L)][d]. */
int fo_page_summaries(const double* K, size_t l, size_t d, size_t L, double* kmax, double* kmin) {
    if (L < 1) return FO_EINVAL; /* :35 */
    const size_t pages = (l + L - 1) / L;
    for (size_t p = 0; p < pages; ++p) {
        const size_t t0 = p * L, t1 = t0 + L < l ? t0 + L : l;
        for (size_t j = 0; j < d; ++j) {
            double mn = K[t0 * d + j], mx = mn;
            for (size_t t = t0 + 1; t < t1; ++t) {
                const double v = K[t * d + j];
                mn = v < mn ? v : mn; /* std::min / std::max: first-seen on ties */
                mx = mx < v ? v : mx;
            }
            kmax[p * d + j] = mx;
            kmin[p * d + j] = mn;
        }
    }
    return FO_OK;
}

/* quest_page_scores (baselines.hpp:60-79): term_j = max(q_j kmax_j, q_j kmin_j);
 * variant 1 = sum over channels, 0 = max over channels. */
int fo_quest_page_scores(const double* q, const double* kmax, const double* kmin, size_t pages, size_t d,
                         int variant, double* out) {
    for (size_t p = 0; p < pages; ++p) {
        double acc = 0.0, best = -INFINITY;
        for (size_t j = 0; j < d; ++j) {
            const double hi = q[j] * kmax[p * d + j], lo = q[j] * kmin[p * d + j];
            const double term = hi < lo ? lo : hi; /* std::max(hi, lo) */
            acc += term;
            best = best < term ? term : best;
        }
        out[p] = variant == 1 ? acc : best;
    }
    return FO_OK;
}

/* quest_select_quantized page scores (baselines.hpp:131-139): mean of the members'
 * estimated scores, summed in token order. */
int fo_page_mean(const double* est, size_t l, size_t L, double* out) {
    if (L < 1) return FO_EINVAL; /* :122 */
    const size_t pages = (l + L - 1) / L;
    for (size_t p = 0; p < pages; ++p) {
        const size_t t0 = p * L, t1 = t0 + L < l ? t0 + L : l;
        double acc = 0.0;
        for (size_t t = t0; t < t1; ++t) acc += est[t];
        out[p] = acc / (double)(t1 - t0);
    }
    return FO_OK;
}

/* detail::select_by_page_scores (baselines.hpp:85-111): pages ranked by (score desc,
 * index asc); whole pages while they fit, then the next page's lowest indices; the
 * n indices ascending. */
int fo_select_by_page_scores(const double* ps, size_t l, size_t L, size_t n, int64_t* out) {
    if (n < 1 || n > l || L < 1) return FO_EINVAL; /* :87 */
    const size_t pages = (l + L - 1) / L;
    int64_t* order = (int64_t*)malloc(pages * sizeof(int64_t));
    if (!order) return FO_EINVAL;
    for (size_t i = 0; i < pages; ++i) order[i] = (int64_t)i;
    qsort_r(order, pages, sizeof(int64_t), cmp_desc, (void*)ps);
    size_t taken = 0;
    for (size_t r = 0; r < pages && taken < n; ++r) {
        const size_t t0 = (size_t)order[r] * L, t1 = t0 + L < l ? t0 + L : l;
        const size_t take = taken + (t1 - t0) <= n ? t1 - t0 : n - taken;
        for (size_t t = t0; t < t0 + take; ++t) out[taken++] = (int64_t)t;
    }
    qsort(out, n, sizeof(int64_t), cmp_asc);
    free(order);
    return FO_OK;
}

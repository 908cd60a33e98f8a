/*
 * oracle.c: fp64 CPU ORACLE for balanced sparsity (arXiv 1811.00206).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path (paper_1811_00206_b200) never
 * imports, links or executes it, and this file shares no code, header, table or constant generator
 * with the CUDA library. The only thing the two share is the seeded input generator (synth/), which
 * holds none of the method's arithmetic.
 *
 * Everything here is plain, slow and single-threaded. It follows the paper's definitions:
 *   - Balanced Sparsity pattern: "each matrix row is split into multiple equal-sized blocks
 *     and each block has the same number of non-zero weights".
 *   - One pruning step, Alg. 1 inner loop: "sorts the weights in each block by
 *     their absolute magnitude and then zeros out a fraction of weights with smallest absolute
 *     magnitudes". Implemented literally: a stable sort of each block by magnitude, then keep the
 *     first k. This is the count-based reading: ties go to the lower offset, and a
 *     NaN ranks above +Inf with all NaNs equal (A17).
 *   - k = lround((1 - s) * B).
 *   - The FC layer Y = W·X + B with B = 0 (Eq. 1), summed in fp64:
 *     y_r = sum_c W_bs[r][c] * x_c. With its bias (Eq. 1's +B) and an activation for the fused layer
 *     epilogue: y_r = act(sum + b_r), act = ReLU, logistic sigmoid or tanh.
 *   - The SPMV/SPMM/SP24 byte layouts, written from docs/layout.md (not from kernel code).
 *
 * Half-precision decoding is written out from the IEEE 754 binary16 and bfloat16 definitions.
 *
 * Parity pinning: every function here is pinned by tests/test_oracle_pins.py against values the
 * paper prints, SPEC worked examples, closed forms, brute force on tiny inputs,
 * and special cases that reduce to textbook routines. See DESIGN.md §3.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_F32 0
#define ORC_F16 1
#define ORC_BF16 2

#define ORC_SPMV 1
#define ORC_SPMM 2
#define ORC_SP24 3

/* ------------------------------------------------------------------ element decoding */

/* IEEE 754 binary16: 1 sign, 5 exponent (bias 15), 10 fraction bits. */
static double half_to_double(uint16_t h) {
  int sign = (h >> 15) & 1;
  int e = (h >> 10) & 0x1f;
  int f = h & 0x3ff;
  double v;
  if (e == 0)
    v = ldexp((double)f, -24); /* subnormal: f * 2^-14 * 2^-10 */
  else if (e == 31)
    v = f ? NAN : INFINITY;
  else
    v = ldexp((double)(f + 1024), e - 25); /* (1 + f/1024) * 2^(e-15) */
  return sign ? -v : v;
}

/* bfloat16 is the high half of an IEEE 754 binary32. */
static double bf16_to_double(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

static double f32_to_double(const void* p) {
  float f;
  memcpy(&f, p, 4);
  return (double)f;
}

static int dtype_size(int dt) { return dt == ORC_F32 ? 4 : 2; }

/* Element i of an array of dtype dt, converted exactly to double. */
double orc_elem(const void* base, int dt, int64_t i) {
  const unsigned char* p = (const unsigned char*)base + i * dtype_size(dt);
  if (dt == ORC_F32) return f32_to_double(p);
  uint16_t h;
  memcpy(&h, p, 2);
  return dt == ORC_F16 ? half_to_double(h) : bf16_to_double(h);
}

/* ------------------------------------------------------------------ k */

int orc_k_from_sparsity(int B, double s) {
  if (B < 1 || !(s >= 0.0) || !(s < 1.0)) return -1;
  return (int)lround((1.0 - s) * (double)B);
}

/* ------------------------------------------------------------------ pruning (Alg. 1 step) */

/* "a ranks above b" in magnitude: NaN above everything else, all NaNs equal; otherwise |a| > |b|. */
static int mag_above(double a, double b) {
  if (isnan(a)) return !isnan(b);
  if (isnan(b)) return 0;
  return fabs(a) > fabs(b);
}

/* One balance-aware pruning step over W (M×K, leading dim ldw, dtype dt).
 * Output: canonical vals[M][NB][k] (dtype dt, bit copies) and idx[M][NB][k] (ascending offsets).
 * Returns 0, or -1 on a shape or argument error. */
int orc_prune(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int B, int k, void* vals,
              uint16_t* idx) {
  if (M < 1 || K < 1 || B < 1 || K % B != 0 || k < 0 || k > B || ldw < K) return -1;
  int64_t NB = K / B;
  int es = dtype_size(dt);
  int* order = (int*)malloc(sizeof(int) * (size_t)B);
  double* mag = (double*)malloc(sizeof(double) * (size_t)B);
  for (int64_t r = 0; r < M; ++r) {
    for (int64_t b = 0; b < NB; ++b) {
      int64_t c0 = r * ldw + b * B;
      for (int j = 0; j < B; ++j) {
        mag[j] = orc_elem(W, dt, c0 + j);
        order[j] = j;
      }
      /* stable insertion sort of offsets by magnitude, largest first: an element moves before
       * its predecessor only if it ranks strictly above it, so equal keys keep ascending offsets */
      for (int i = 1; i < B; ++i) {
        int cur = order[i];
        int j = i - 1;
        while (j >= 0 && mag_above(mag[cur], mag[order[j]])) {
          order[j + 1] = order[j];
          --j;
        }
        order[j + 1] = cur;
      }
      /* keep the first k; emit them in ascending offset order (insertion sort again) */
      for (int i = 1; i < k; ++i) {
        int cur = order[i];
        int j = i - 1;
        while (j >= 0 && order[j] > cur) {
          order[j + 1] = order[j];
          --j;
        }
        order[j + 1] = cur;
      }
      for (int t = 0; t < k; ++t) {
        int64_t pos = (r * NB + b) * k + t;
        idx[pos] = (uint16_t)order[t];
        memcpy((unsigned char*)vals + pos * es, (const unsigned char*)W + (c0 + order[t]) * es, es);
      }
    }
  }
  free(order);
  free(mag);
  return 0;
}

/* W_bs as a dense fp64 M×K matrix: kept values at (r, b·B + idx), zeros elsewhere. */
int orc_decode(const void* vals, const uint16_t* idx, int dt, int64_t M, int64_t K, int B, int k,
               double* Wd) {
  if (K % B != 0) return -1;
  int64_t NB = K / B;
  memset(Wd, 0, sizeof(double) * (size_t)(M * K));
  for (int64_t r = 0; r < M; ++r)
    for (int64_t b = 0; b < NB; ++b)
      for (int t = 0; t < k; ++t) {
        int64_t pos = (r * NB + b) * k + t;
        Wd[r * K + b * B + idx[pos]] = orc_elem(vals, dt, pos);
      }
  return 0;
}

/* Position of every element in its block's magnitude order (Alg. 1's "sorts the weights in each block
 * by their absolute magnitude"; ties to the lower offset, NaN above Inf, as orc_prune):
 * rank[r*K + c] = position of W[r][c] in the stable descending sort of its block. A pruning step at
 * any k keeps exactly the entries with rank < k, so one rank pass gives the masks of a whole gradual
 * schedule (Alg. 1's outer loop) without retraining. Requires B <= 256 (u8 ranks). */
int orc_block_rank(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int B, uint8_t* rank) {
  if (M < 1 || K < 1 || B < 1 || B > 256 || K % B != 0 || ldw < K) return -1;
  int64_t NB = K / B;
  int* order = (int*)malloc(sizeof(int) * (size_t)B);
  double* mag = (double*)malloc(sizeof(double) * (size_t)B);
  for (int64_t r = 0; r < M; ++r)
    for (int64_t b = 0; b < NB; ++b) {
      int64_t c0 = r * ldw + b * B;
      for (int j = 0; j < B; ++j) {
        mag[j] = orc_elem(W, dt, c0 + j);
        order[j] = j;
      }
      for (int i = 1; i < B; ++i) { /* the same stable insertion sort as orc_prune */
        int cur = order[i];
        int j = i - 1;
        while (j >= 0 && mag_above(mag[cur], mag[order[j]])) {
          order[j + 1] = order[j];
          --j;
        }
        order[j + 1] = cur;
      }
      for (int t = 0; t < B; ++t) rank[r * K + b * B + order[t]] = (uint8_t)t;
    }
  free(order);
  free(mag);
  return 0;
}

/* ------------------------------------------------------------------ Alg. 1's outer loop and the comparison patterns */

/* GraduallyIncrease (Alg. 1 line "tmp_sparsity = GraduallyIncrease(tmp_sparsity)"): "This threshold
 * percentage is gradually increased from 0 to the target sparsity while the increase rate decreases with
 * pruning iteration". The paper gives no formula; SPEC S:205 fixes the cubic trajectory
 * s_i = target * (1 - (1 - i/n)^3), i = 0..n (rate 3·target/n·(1 - i/n)^2, decreasing). Returns -1 on
 * bad arguments (n < 1, i outside [0, n], target outside [0, 1)). */
double orc_schedule(double target, int n, int i) {
  if (n < 1 || i < 0 || i > n || !(target >= 0.0) || !(target < 1.0)) return -1.0;
  double u = 1.0 - (double)i / (double)n;
  return target * (1.0 - u * u * u);
}

/* The pruned matrix M_p of Alg. 1 (its output) in dense form after one pruning step at k kept
 * per block: Wp[r][c] = W[r][c] (bit copy) if (r, c) is kept by orc_prune, else +0 of dtype dt.
 * Wp is M×K with leading dimension K. */
int orc_prune_dense(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int B, int k, void* Wp) {
  if (M < 1 || K < 1 || B < 1 || K % B != 0 || k < 0 || k > B || ldw < K) return -1;
  int64_t NB = K / B;
  int es = dtype_size(dt);
  void* vals = malloc((size_t)(M * NB * (k > 0 ? k : 1)) * (size_t)es);
  uint16_t* idx = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(M * NB * (k > 0 ? k : 1)));
  if (orc_prune(W, dt, M, K, ldw, B, k, vals, idx)) {
    free(vals);
    free(idx);
    return -1;
  }
  memset(Wp, 0, (size_t)(M * K) * (size_t)es);
  for (int64_t r = 0; r < M; ++r)
    for (int64_t b = 0; b < NB; ++b)
      for (int t = 0; t < k; ++t) {
        int64_t pos = (r * NB + b) * k + t;
        memcpy((unsigned char*)Wp + (r * K + b * B + idx[pos]) * es, (const unsigned char*)vals + pos * es, es);
      }
  free(vals);
  free(idx);
  return 0;
}

/* A scored unit (an element or a tile) for the global selections below. */
typedef struct {
  double score;  /* magnitude, or a tile score; NaN = above everything */
  int64_t index; /* row-major position of the element / tile */
} orc_unit;

/* Descending score, NaN first (all NaNs equal), then ascending index: a total order. */
static int unit_cmp(const void* pa, const void* pb) {
  const orc_unit* a = (const orc_unit*)pa;
  const orc_unit* b = (const orc_unit*)pb;
  int an = isnan(a->score), bn = isnan(b->score);
  if (an != bn) return an ? -1 : 1;
  if (!an && a->score != b->score) return a->score > b->score ? -1 : 1;
  return a->index < b->index ? -1 : (a->index > b->index ? 1 : 0);
}

/* keep[u] = 1 for the `keep` first units in unit_cmp order (a library sort as one step). */
static void select_top(orc_unit* units, int64_t n, int64_t keep, uint8_t* keep_flag) {
  qsort(units, (size_t)n, sizeof(orc_unit), unit_cmp);
  memset(keep_flag, 0, (size_t)n);
  for (int64_t i = 0; i < keep && i < n; ++i) keep_flag[units[i].index] = 1;
}

/* Number of units kept at sparsity s: lround((1 - s) * n), the same rounding as k. */
int64_t orc_keep_count(int64_t n, double s) {
  if (n < 0 || !(s >= 0.0) || !(s < 1.0)) return -1;
  return (int64_t)llround((1.0 - s) * (double)n);
}

/* Random sparsity (Han et al.; "performs pruning in each independent weight
 * matrix"): magnitude pruning over the WHOLE matrix. Keeps the keep_count(M·K, s) entries of largest
 * |w| (NaN above Inf; ties to the lower row-major index). mask[r*K + c] = 1 if kept. */
int orc_random_mask(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, double s, uint8_t* mask) {
  if (M < 1 || K < 1 || ldw < K) return -1;
  int64_t n = M * K, keep = orc_keep_count(n, s);
  if (keep < 0) return -1;
  orc_unit* u = (orc_unit*)malloc(sizeof(orc_unit) * (size_t)n);
  for (int64_t r = 0; r < M; ++r)
    for (int64_t c = 0; c < K; ++c) {
      double v = orc_elem(W, dt, r * ldw + c);
      u[r * K + c].score = isnan(v) ? NAN : fabs(v);
      u[r * K + c].index = r * K + c;
    }
  select_top(u, n, keep, mask);
  free(u);
  return 0;
}

/* Block sparsity (Narang et al.): the matrix is tiled into bh×bw tiles (row-major tile
 * order); each tile is scored by "the maximum magnitude or the average magnitude of the weights within
 * one block as a representative": criterion 0 = max |w| (NaN above Inf), criterion 1 =
 * mean |w|, compared as the fp64 sum of |w| in row-major order inside the tile (the mean times the fixed
 * tile size; a NaN sum ranks above everything). The keep_count(#tiles, s) best tiles survive whole
 * (ties to the lower tile index). mask[r*K + c] = 1 if (r, c) lies in a kept tile.
 * Vector sparsity (Mao et al.) is the same rule with whole rows (bh = 1, bw = K) or whole columns
 * (bh = M, bw = 1) as the unit and the mean criterion. */
int orc_block_mask(const void* W, int dt, int64_t M, int64_t K, int64_t ldw, int64_t bh, int64_t bw, double s,
                   int criterion, uint8_t* mask) {
  if (M < 1 || K < 1 || ldw < K || bh < 1 || bw < 1 || M % bh || K % bw || criterion < 0 || criterion > 1)
    return -1;
  int64_t TR = M / bh, TC = K / bw, n = TR * TC, keep = orc_keep_count(n, s);
  if (keep < 0) return -1;
  orc_unit* u = (orc_unit*)malloc(sizeof(orc_unit) * (size_t)n);
  uint8_t* tk = (uint8_t*)malloc((size_t)n);
  for (int64_t tr = 0; tr < TR; ++tr)
    for (int64_t tc = 0; tc < TC; ++tc) {
      double score = criterion == 0 ? -1.0 : 0.0;
      int seen_nan = 0;
      for (int64_t i = 0; i < bh; ++i)
        for (int64_t j = 0; j < bw; ++j) {
          double v = orc_elem(W, dt, (tr * bh + i) * ldw + tc * bw + j);
          if (isnan(v)) {
            seen_nan = 1;
            continue;
          }
          if (criterion == 0) {
            if (fabs(v) > score) score = fabs(v);
          } else {
            score += fabs(v);
          }
        }
      u[tr * TC + tc].score = seen_nan ? NAN : score;
      u[tr * TC + tc].index = tr * TC + tc;
    }
  select_top(u, n, keep, tk);
  for (int64_t r = 0; r < M; ++r)
    for (int64_t c = 0; c < K; ++c) mask[r * K + c] = tk[(r / bh) * TC + c / bw];
  free(u);
  free(tk);
  return 0;
}

/* ------------------------------------------------------------------ layouts (docs/layout.md) */

static int64_t align256(int64_t n) { return (n + 255) / 256 * 256; }

static int64_t pad16(int64_t n) { return (n + 15) / 16 * 16; }

/* bytes of one SPMM blob: mt rows x cb blocks x k entries, values then indices, each 16-padded */
static int64_t blob_bytes(int64_t mt, int64_t cb, int k, int es, int is) {
  return pad16(mt * cb * k * es) + pad16(mt * cb * k * is);
}

typedef struct {
  int64_t V, P, NBf, T;
  int es, is;                 /* value bytes, index bytes */
  int64_t ri;                 /* SPMV: bytes of a step's index run (160: 5-bit runs, 128: 4-bit runs, else P*is) */
  int64_t offA, offB, offC, total;  /* SP24: offA = values, offB = metadata */
} orc_geom;

static int geom(int64_t M, int64_t K, int B, int k, int dt, int layout, orc_geom* g) {
  if (M < 1 || K < 1 || B < 1 || K % B != 0 || k < 0 || k > B) return -1;
  if (dt != ORC_F32 && dt != ORC_F16 && dt != ORC_BF16) return -1;
  int64_t NB = K / B;
  g->es = dtype_size(dt);
  g->is = B <= 256 ? 1 : 2;
  if (layout == ORC_SPMM) {
    /* docs/layout.md SPMM: 128-row tiles x CB-block chunks, one 16-byte-padded blob each */
    g->V = B <= 64 ? (64 + B - 1) / B : 1; /* CB (chunk blocks) kept in V */
    g->P = (M + 127) / 128;                /* MT */
    g->NBf = (NB + g->V - 1) / g->V;       /* NC */
    g->T = 0;
    int64_t mt_last = M - 128 * (g->P - 1), cb_last = NB - g->V * (g->NBf - 1);
    int64_t tb_full = (g->NBf - 1) * blob_bytes(128, g->V, k, g->es, g->is) + blob_bytes(128, cb_last, k, g->es, g->is);
    int64_t tb_last = (g->NBf - 1) * blob_bytes(mt_last, g->V, k, g->es, g->is) + blob_bytes(mt_last, cb_last, k, g->es, g->is);
    g->offA = 0;
    g->offB = tb_full; /* tile stride */
    g->offC = 0;
    g->total = align256((g->P - 1) * tb_full + tb_last);
    return 0;
  }
  if (layout == ORC_SPMV) {
    int64_t vmax = 16 / g->es;
    int64_t V = 1;
    while (V * 2 <= vmax && 32 * V * 2 <= NB) V *= 2;
    g->V = V;
    g->P = 32 * V;
    g->NBf = NB / g->P;
    g->T = NB - g->NBf * g->P;
    /* docs/layout.md: 5-bit index runs when B = 32 and V = 8 (two planes: 32 u32 words + 32 bytes);
     * 4-bit index runs when B <= 16 and V = 8 (32 u32 words) */
    g->ri = (B == 32 && V == 8) ? 160 : (B <= 16 && V == 8) ? 128 : g->P * g->is;
    g->offA = 0;
    g->offB = align256(M * g->NBf * k * (g->P * g->es + g->ri));
    g->offC = g->offB + align256(M * k * g->T * g->es);
    g->total = g->offC + align256(M * k * g->T * g->is);
    return 0;
  }
  if (layout == ORC_SP24) {
    if (B != 4 || k != 2 || K % 8 != 0) return -1;
    g->V = g->P = g->NBf = g->T = 0;
    g->offA = 0;
    g->offB = align256(M * (K / 2) * g->es);
    g->offC = 0;
    g->total = g->offB + align256(M * (NB / 2));
    return 0;
  }
  return -1;
}

size_t orc_packed_bytes(int64_t M, int64_t K, int B, int k, int dt, int layout) {
  orc_geom g;
  if (geom(M, K, B, k, dt, layout, &g)) return 0;
  return (size_t)g.total;
}

static void put_index(unsigned char* dst, int is, uint16_t v) {
  dst[0] = (unsigned char)(v & 0xff);
  if (is == 2) dst[1] = (unsigned char)(v >> 8);
}

/* Reference permutation pi_L(canonical) -> packed bytes (docs/layout.md). Padding bytes are zero. */
int orc_pack(const void* vals, const uint16_t* idx, int64_t M, int64_t K, int B, int k, int dt,
             int layout, void* packed) {
  orc_geom g;
  if (geom(M, K, B, k, dt, layout, &g)) return -1;
  int64_t NB = K / B;
  unsigned char* out = (unsigned char*)packed;
  const unsigned char* in = (const unsigned char*)vals;
  memset(out, 0, (size_t)g.total);
  if (layout == ORC_SP24) {
    for (int64_t r = 0; r < M; ++r)
      for (int64_t b = 0; b < NB; ++b) {
        int64_t pos = (r * NB + b) * 2;
        memcpy(out + g.offA + pos * g.es, in + pos * g.es, 2 * g.es);
        int nib = idx[pos] | (idx[pos + 1] << 2);
        out[g.offB + r * (NB / 2) + b / 2] |= (unsigned char)(nib << (4 * (b % 2)));
      }
    return 0;
  }
  if (layout == ORC_SPMM) {
    int64_t CB = g.V, MT = g.P, NC = g.NBf;
    for (int64_t t = 0; t < MT; ++t) {
      int64_t mt = M - 128 * t < 128 ? M - 128 * t : 128;
      for (int64_t c = 0; c < NC; ++c) {
        int64_t cb = NB - CB * c < CB ? NB - CB * c : CB;
        unsigned char* blob = out + t * g.offB + c * blob_bytes(mt, CB, k, g.es, g.is);
        int64_t nvb = pad16(mt * cb * k * g.es);
        for (int64_t r = 0; r < mt; ++r)
          for (int64_t j = 0; j < cb; ++j)
            for (int tt = 0; tt < k; ++tt) {
              int64_t pos = (r * cb + j) * k + tt;
              int64_t src = ((128 * t + r) * NB + CB * c + j) * k + tt;
              memcpy(blob + pos * g.es, in + src * g.es, g.es);
              put_index(blob + nvb + pos * g.is, g.is, idx[src]);
            }
      }
    }
    return 0;
  }
  int64_t step_bytes = g.P * g.es + g.ri;
  int five = g.ri == 160;         /* 5-bit index runs */
  int four = g.ri == 128 && g.P * g.is != 128; /* 4-bit index runs */
  for (int64_t r = 0; r < M; ++r) {
    /* region A: step (r, p, t) = P values then P indices; entry (l, v) at position l*V + v,
     * holding canonical (r, b = p*P + v*32 + l, t) */
    for (int64_t p = 0; p < g.NBf; ++p)
      for (int t = 0; t < k; ++t) {
        unsigned char* step = out + g.offA + ((r * g.NBf + p) * k + t) * step_bytes;
        for (int l = 0; l < 32; ++l)
          for (int64_t v = 0; v < g.V; ++v) {
            int64_t b = p * g.P + v * 32 + l;
            int64_t src = (r * NB + b) * k + t;
            int64_t pos = l * g.V + v;
            memcpy(step + pos * g.es, in + src * g.es, g.es);
            if (!five && !four) put_index(step + g.P * g.es + pos * g.is, g.is, idx[src]);
          }
        if (four) /* G_l = sum_v idx(l, v) << 4v: 32 little-endian u32 words */
          for (int l = 0; l < 32; ++l) {
            uint32_t G = 0;
            for (int64_t v = 0; v < 8; ++v) G |= (uint32_t)idx[(r * NB + p * g.P + v * 32 + l) * k + t] << (4 * v);
            unsigned char* run = step + g.P * g.es;
            for (int j = 0; j < 4; ++j) run[4 * l + j] = (unsigned char)(G >> (8 * j));
          }
        if (five) /* F_l = sum_v idx(l, v) << 5v: u32 plane (bits 0..31), then byte plane (32..39) */
          for (int l = 0; l < 32; ++l) {
            uint64_t F = 0;
            for (int64_t v = 0; v < 8; ++v) F |= (uint64_t)idx[(r * NB + p * g.P + v * 32 + l) * k + t] << (5 * v);
            unsigned char* run = step + g.P * g.es;
            for (int j = 0; j < 4; ++j) run[4 * l + j] = (unsigned char)(F >> (8 * j));
            run[128 + l] = (unsigned char)(F >> 32);
          }
      }
    /* regions B (values) and C (indices): entry (r, t, v, l) at element r*k*T + t*T + v*32 + l
     * (v*32 + l < T), holding canonical (r, b = NBf*P + v*32 + l, t) */
    for (int t = 0; t < k; ++t)
      for (int64_t v = 0; v * 32 < g.T; ++v)
        for (int l = 0; l < 32; ++l) {
          if (v * 32 + l >= g.T) continue;
          int64_t b = g.NBf * g.P + v * 32 + l;
          int64_t src = (r * NB + b) * k + t;
          int64_t pos = r * k * g.T + t * g.T + v * 32 + l;
          memcpy(out + g.offB + pos * g.es, in + src * g.es, g.es);
          put_index(out + g.offC + pos * g.is, g.is, idx[src]);
        }
  }
  return 0;
}

/* ------------------------------------------------------------------ products (Eq. 1, B = 0) */

/* Sparse-form SpMV over canonical arrays, fp64, restricted to `nrows` listed rows:
 * for each listed row r (rows[i]; or row i when rows == NULL),
 *   y[i]     = sum over b, t of vals[r][b][t] * x[b*B + idx[r][b][t]]
 *   bound[i] = sum over b, t of |vals[r][b][t]| * |x[...]|   (the tolerance scale of O-7)
 * The sum over canonical entries equals the dense-masked sum over columns because every other
 * column of W_bs is zero. */
int orc_spmv_rows(const void* vals, const uint16_t* idx, int dt, int64_t M, int64_t K, int B, int k,
                  const void* x, const int64_t* rows, int64_t nrows, double* y, double* bound) {
  if (K % B != 0) return -1;
  int64_t NB = K / B;
  for (int64_t i = 0; i < nrows; ++i) {
    int64_t r = rows ? rows[i] : i;
    if (r < 0 || r >= M) return -1;
    double acc = 0.0, mag = 0.0;
    for (int64_t b = 0; b < NB; ++b)
      for (int t = 0; t < k; ++t) {
        int64_t pos = (r * NB + b) * k + t;
        double w = orc_elem(vals, dt, pos);
        double xv = orc_elem(x, dt, b * B + idx[pos]);
        acc += w * xv;
        mag += fabs(w) * fabs(xv);
      }
    y[i] = acc;
    if (bound) bound[i] = mag;
  }
  return 0;
}

/* As orc_spmv_rows, but `vals`/`idx` hold ONLY the listed rows (nrows × NB × k, in list order).
 * This lets the big config's sampled rows be checked without copying the whole matrix to the host. */
int orc_spmv_rowslice(const void* vals, const uint16_t* idx, int dt, int64_t nrows, int64_t K,
                      int B, int k, const void* x, double* y, double* bound) {
  return orc_spmv_rows(vals, idx, dt, nrows, K, B, k, x, NULL, nrows, y, bound);
}

/* Dense fp64 GEMV y = Wd · x (Wd M×K row-major doubles). This is the "dense-masked W·x" of O-7
 * when Wd = orc_decode(...). */
int orc_gemv_dense(const double* Wd, int64_t M, int64_t K, const double* x, double* y) {
  for (int64_t r = 0; r < M; ++r) {
    double acc = 0.0;
    for (int64_t c = 0; c < K; ++c) acc += Wd[r * K + c] * x[c];
    y[r] = acc;
  }
  return 0;
}

/* SpMM: column n of Y (M doubles at Y + n*M) = SpMV of column n of X (X + n*ldx, dtype dt). */
int orc_spmm(const void* vals, const uint16_t* idx, int dt, int64_t M, int64_t K, int B, int k,
             const void* X, int64_t N, int64_t ldx, double* Y, double* bound) {
  int es = dtype_size(dt);
  for (int64_t n = 0; n < N; ++n) {
    const unsigned char* xn = (const unsigned char*)X + n * ldx * es;
    if (orc_spmv_rows(vals, idx, dt, M, K, B, k, xn, NULL, M, Y + n * M, bound ? bound + n * M : NULL))
      return -1;
  }
  return 0;
}

/* SpMM restricted to listed rows (for big configs): Y[n*nrows + i] for row rows[i]. */
int orc_spmm_rows(const void* vals, const uint16_t* idx, int dt, int64_t M, int64_t K, int B, int k,
                  const void* X, int64_t N, int64_t ldx, const int64_t* rows, int64_t nrows,
                  double* Y, double* bound) {
  int es = dtype_size(dt);
  for (int64_t n = 0; n < N; ++n) {
    const unsigned char* xn = (const unsigned char*)X + n * ldx * es;
    if (orc_spmv_rows(vals, idx, dt, M, K, B, k, xn, rows, nrows, Y + n * nrows,
                      bound ? bound + n * nrows : NULL))
      return -1;
  }
  return 0;
}

/* The activations of the layer epilogue, from their definitions: ReLU max(v, 0), the logistic
 * sigmoid 1 / (1 + e^-v), and tanh v = (e^v - e^-v) / (e^v + e^-v) (written out, not libm's tanh). */
double orc_act(double v, int act) {
  switch (act) {
    case 0: return v;
    case 1: return v > 0.0 ? v : 0.0;
    case 2: return 1.0 / (1.0 + exp(-v));
    case 3: {
      if (v > 20.0) return 1.0;  /* |tanh v - 1| < 1e-17 beyond 20: avoids inf/inf */
      if (v < -20.0) return -1.0;
      double e = exp(v), f = exp(-v);
      return (e - f) / (e + f);
    }
    default: return NAN;
  }
}

/* The whole layer of Eq. 1 at batch 1 with an activation: y[r] = act(sum + bias[r]), fp64.
 * bias: M elements of dt, or NULL. bound[r] = sum |w||x| + |bias[r]| (the tolerance scale of O-7
 * extended by the bias term; act is 1-Lipschitz for all three activations). */
int orc_spmv_act(const void* vals, const uint16_t* idx, int dt, int64_t M, int64_t K, int B, int k,
                 const void* x, const void* bias, int act, double* y, double* bound) {
  if (act < 0 || act > 3) return -1;
  if (orc_spmv_rows(vals, idx, dt, M, K, B, k, x, NULL, M, y, bound)) return -1;
  for (int64_t r = 0; r < M; ++r) {
    double b = bias ? orc_elem(bias, dt, r) : 0.0;
    y[r] = orc_act(y[r] + b, act);
    if (bound) bound[r] += fabs(b);
  }
  return 0;
}

/* One LSTM step whose gate weights are balanced-sparse: the recurrent layers of the paper's PTB model
 * ("2-layer LSTM ... 1500 hidden units"; the rows of [W_ih | W_hh] are BJ.configs[1]'s 6000 x 3000)
 * and TIMIT Bi-LSTM (hidden 1024). The gate pre-activations are Eq. 1 with its +B:
 *   z = W_bs·x + pre + bias,    x = [x_t ; h_{t-1}] (or h_{t-1} alone when pre holds W_ih·x_t),
 * with the gate rows interleaved: row 4j + g is gate g of hidden unit j, g = 0 input, 1 forget,
 * 2 cell candidate, 3 output. The cell is the standard LSTM:
 *   i = sigmoid(z_i), f = sigmoid(z_f), g = tanh(z_g), o = sigmoid(z_o),
 *   c_j = f·c_prev_j + i·g,   h_j = o·tanh(c_j),
 * all in fp64 (orc_act's sigmoid and tanh). pre, bias: M elements of dt or NULL. c_prev, h, c: M/4
 * doubles. zbound (M doubles, may be NULL): per gate row sum|w||x| + |pre| + |bias| (O-7's scale). */
int orc_lstm_cell(const void* vals, const uint16_t* idx, int dt, int64_t M, int64_t K, int B, int k, const void* x,
                  const void* pre, const void* bias, const double* c_prev, double* h, double* c, double* zbound) {
  if (M < 4 || M % 4 != 0) return -1;
  double* z = (double*)malloc(sizeof(double) * (size_t)M);
  double* zb = (double*)malloc(sizeof(double) * (size_t)M);
  if (orc_spmv_rows(vals, idx, dt, M, K, B, k, x, NULL, M, z, zb)) {
    free(z);
    free(zb);
    return -1;
  }
  for (int64_t r = 0; r < M; ++r) {
    double p = pre ? orc_elem(pre, dt, r) : 0.0, b = bias ? orc_elem(bias, dt, r) : 0.0;
    z[r] += p + b;
    zb[r] += fabs(p) + fabs(b);
    if (zbound) zbound[r] = zb[r];
  }
  for (int64_t j = 0; j < M / 4; ++j) {
    double ig = orc_act(z[4 * j + 0], 2), fg = orc_act(z[4 * j + 1], 2);
    double gg = orc_act(z[4 * j + 2], 3), og = orc_act(z[4 * j + 3], 2);
    c[j] = fg * c_prev[j] + ig * gg;
    h[j] = og * orc_act(c[j], 3);
  }
  free(z);
  free(zb);
  return 0;
}

/* Convolution as the paper runs it: "One popular implementation of convolution operation is using
 * im2col that converts convolution operation to matrix-matrix multiplication", and "the weights
 * of all kernels in one convolution layer are considered as one weight matrix". Reading A23: the
 * activations are NHWC (channels last) and the weight matrix is Cout x (kh·kw·C) with its columns in
 * (dy, dx, c) order, so that column (dy·kw + dx)·C + c multiplies input channel c at tap (dy, dx).
 *
 * orc_im2col: X[(n·OH + oy)·OW + ox][(dy·kw + dx)·C + c] = in[n][oy·stride + dy - pad][ox·stride + dx - pad][c],
 * +0 where the tap falls outside the image; OH = (H + 2·pad - kh)/stride + 1 (same for OW). A pure copy
 * of element bits. X has leading dimension kh·kw·C. */
int orc_im2col(const void* in, int dt, int64_t Nimg, int64_t H, int64_t W, int64_t C, int kh, int kw, int pad,
               int stride, void* X) {
  if (Nimg < 1 || H < 1 || W < 1 || C < 1 || kh < 1 || kw < 1 || pad < 0 || stride < 1) return -1;
  int64_t OH = (H + 2 * pad - kh) / stride + 1, OW = (W + 2 * pad - kw) / stride + 1;
  if (OH < 1 || OW < 1) return -1;
  int es = dtype_size(dt);
  int64_t Kc = (int64_t)kh * kw * C;
  for (int64_t n = 0; n < Nimg; ++n)
    for (int64_t oy = 0; oy < OH; ++oy)
      for (int64_t ox = 0; ox < OW; ++ox)
        for (int dy = 0; dy < kh; ++dy)
          for (int dx = 0; dx < kw; ++dx)
            for (int64_t c = 0; c < C; ++c) {
              int64_t iy = oy * stride + dy - pad, ix = ox * stride + dx - pad;
              unsigned char* dst = (unsigned char*)X + (((n * OH + oy) * OW + ox) * Kc + (dy * kw + dx) * C + c) * es;
              if (iy < 0 || iy >= H || ix < 0 || ix >= W)
                memset(dst, 0, (size_t)es);
              else
                memcpy(dst, (const unsigned char*)in + (((n * H + iy) * W + ix) * C + c) * es, (size_t)es);
            }
  return 0;
}

/* The convolution itself, written as its definition (no im2col): for output pixel (n, oy, ox) and
 * output channel co,  y = sum_{dy,dx,c} W_bs[co][(dy·kw + dx)·C + c] · in[n][oy·s + dy - pad][ox·s + dx - pad][c]
 * in fp64 over the canonical (vals, idx) of the Cout x (kh·kw·C) weight matrix. Output Y[pixel][co]
 * (NHWC), and bound[pixel][co] = the same sum of |w|·|in| (O-7's tolerance scale). */
int orc_conv2d(const void* vals, const uint16_t* idx, int dt, int64_t Cout, int B, int k, const void* in,
               int64_t Nimg, int64_t H, int64_t W, int64_t C, int kh, int kw, int pad, int stride, double* Y,
               double* bound) {
  int64_t Kc = (int64_t)kh * kw * C;
  if (Kc % B != 0 || Cout < 1) return -1;
  int64_t OH = (H + 2 * pad - kh) / stride + 1, OW = (W + 2 * pad - kw) / stride + 1;
  if (OH < 1 || OW < 1) return -1;
  int64_t NB = Kc / B;
  for (int64_t n = 0; n < Nimg; ++n)
    for (int64_t oy = 0; oy < OH; ++oy)
      for (int64_t ox = 0; ox < OW; ++ox) {
        int64_t p = (n * OH + oy) * OW + ox;
        for (int64_t co = 0; co < Cout; ++co) {
          double acc = 0.0, bnd = 0.0;
          for (int64_t b = 0; b < NB; ++b)
            for (int t = 0; t < k; ++t) {
              int64_t pos = (co * NB + b) * k + t;
              int64_t col = b * B + idx[pos];
              int64_t tap = col / C, c = col % C;
              int64_t dy = tap / kw, dx = tap % kw;
              int64_t iy = oy * stride + dy - pad, ix = ox * stride + dx - pad;
              if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue;
              double w = orc_elem(vals, dt, pos);
              double v = orc_elem(in, dt, ((n * H + iy) * W + ix) * C + c);
              acc += w * v;
              bnd += fabs(w) * fabs(v);
            }
          Y[p * Cout + co] = acc;
          if (bound) bound[p * Cout + co] = bnd;
        }
      }
  return 0;
}

/* ------------------------------------------------------------------ reporting */

/* The paper's ideal inference time: i_time = (d_time - o_time) * (1 - sparsity) + o_time. */
double orc_ideal_time(double d_time, double o_time, double sparsity) {
  return (d_time - o_time) * (1.0 - sparsity) + o_time;
}

/*
 * eplab_oracle.c -- CPU ORACLE (test infrastructure only; see eplab_oracle.h).
 *
 * Each function cites the reference file:line it restates. Compiled with
 * -ffp-contract=off so every float operation rounds exactly where written.
 */
#include "eplab_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ rng */
/* splitmix64, routing.cpp:15-28 */
static uint64_t sm_next(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static uint64_t sm_below(uint64_t* s, uint64_t n) { return (uint64_t)(((u128)sm_next(s) * n) >> 64); }
static double sm_uniform01(uint64_t* s) { return (double)(sm_next(s) >> 11) * 0x1.0p-53; }

/* routing.cpp:32-73 */
int orc_sample_routing(int n_exp, int topk, long long n_tok, int world, uint64_t seed,
                       int32_t* sel, float* gw) {
  if (topk > n_exp) return 2;
  int* pool = (int*)malloc(sizeof(int) * (size_t)n_exp);
  for (int r = 0; r < world; ++r) {
    uint64_t st = seed ^ (0xA5A5A5A5A5A5A5A5ULL + (uint64_t)r * 0x9E3779B97F4A7C15ULL);
    int32_t* s = sel + (size_t)r * n_tok * topk;
    float* g = gw + (size_t)r * n_tok * topk;
    for (int e = 0; e < n_exp; ++e) pool[e] = e; /* iota once per rank; pool persists */
    for (long long t = 0; t < n_tok; ++t) {
      for (int j = 0; j < topk; ++j) {
        uint64_t pick = (uint64_t)j + sm_below(&st, (uint64_t)(n_exp - j));
        int tmp = pool[j];
        pool[j] = pool[pick];
        pool[pick] = tmp;
        s[t * topk + j] = pool[j];
      }
      double sum = 0.0;
      for (int j = 0; j < topk; ++j) {
        double u = sm_uniform01(&st);
        g[t * topk + j] = (float)u;
        sum += u;
      }
      if (sum > 0)
        for (int j = 0; j < topk; ++j) g[t * topk + j] = (float)((double)g[t * topk + j] / sum);
    }
  }
  free(pool);
  return 0;
}

/* ------------------------------------------------------------ token map */
/* token_map.cpp:10-28 */
void orc_local_stable_sort(const int32_t* sel, long long n, int n_exp, int64_t* m_loc,
                           int64_t* counts, int64_t* offsets) {
  memset(counts, 0, sizeof(int64_t) * (size_t)n_exp);
  for (long long i = 0; i < n; ++i) counts[sel[i]]++;
  int64_t acc = 0;
  for (int e = 0; e < n_exp; ++e) {
    offsets[e] = acc;
    acc += counts[e];
  }
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_exp);
  memcpy(cur, offsets, sizeof(int64_t) * (size_t)n_exp);
  for (long long i = 0; i < n; ++i) m_loc[i] = cur[sel[i]]++;
  free(cur);
}

/* token_map.cpp:30-53 */
int orc_global_offsets(const int64_t* counts_all, int world, int n_exp, int64_t* o_all) {
  if (world < 1 || n_exp % world) return 2;
  int epr = n_exp / world;
  for (int dst = 0; dst < world; ++dst)
    for (int el = 0; el < epr; ++el) {
      int eg = dst * epr + el;
      int64_t acc = 0;
      for (int src = 0; src < world; ++src) {
        o_all[((size_t)dst * epr + el) * world + src] = acc;
        acc += counts_all[(size_t)src * n_exp + eg];
      }
    }
  return 0;
}

/* types.cpp:74-94 (validate_routing) */
static int validate_sel(const int32_t* sel, int world, int n_exp, long long n_tok, int topk) {
  for (int r = 0; r < world; ++r)
    for (long long t = 0; t < n_tok; ++t)
      for (int j = 0; j < topk; ++j) {
        int e = sel[((size_t)r * n_tok + t) * topk + j];
        if (e < 0 || e >= n_exp) return 2;
        for (int i = 0; i < j; ++i)
          if (sel[((size_t)r * n_tok + t) * topk + i] == e) return 2;
      }
  return 0;
}

/* token_map.cpp:55-106 */
int orc_token_map(const int32_t* sel, int world, int n_exp, long long n_tok, int topk,
                  int32_t* target_rank, int32_t* local_expert, int64_t* offset,
                  int64_t* recv_totals, int64_t* seg_base) {
  if (world < 1 || n_exp % world) return 2;
  if (validate_sel(sel, world, n_exp, n_tok, topk)) return 2;
  const int epr = n_exp / world;
  const long long n = n_tok * topk;
  int64_t* counts = (int64_t*)calloc((size_t)world * n_exp, sizeof(int64_t));
  int64_t* offs = (int64_t*)calloc((size_t)world * n_exp, sizeof(int64_t));
  int64_t* mloc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1) * world);
  for (int r = 0; r < world; ++r)
    orc_local_stable_sort(sel + (size_t)r * n, n, n_exp, mloc + (size_t)r * n,
                          counts + (size_t)r * n_exp, offs + (size_t)r * n_exp);
  int64_t* oall = (int64_t*)malloc(sizeof(int64_t) * (size_t)world * epr * world);
  orc_global_offsets(counts, world, n_exp, oall);
  if (recv_totals) {
    memset(recv_totals, 0, sizeof(int64_t) * (size_t)world * epr);
    for (int src = 0; src < world; ++src)
      for (int e = 0; e < n_exp; ++e)
        recv_totals[(size_t)(e / epr) * epr + (e % epr)] += counts[(size_t)src * n_exp + e];
    if (seg_base)
      for (int r = 0; r < world; ++r) {
        int64_t acc = 0;
        for (int e = 0; e < epr; ++e) {
          seg_base[(size_t)r * epr + e] = acc;
          acc += recv_totals[(size_t)r * epr + e];
        }
      }
  }
  for (int r = 0; r < world; ++r)
    for (long long i = 0; i < n; ++i) {
      int e = sel[(size_t)r * n + i];
      int rt = e / epr, el = e % epr;
      target_rank[(size_t)r * n + i] = rt;
      local_expert[(size_t)r * n + i] = el;
      offset[(size_t)r * n + i] = mloc[(size_t)r * n + i] - offs[(size_t)r * n_exp + e] +
                                  oall[((size_t)rt * epr + el) * world + r];
    }
  free(counts);
  free(offs);
  free(mloc);
  free(oall);
  return 0;
}

/* token_map.cpp:108-126: buckets (e_loc * world + dst) filled in (t, j) order. */
void orc_send_schedule(const int32_t* target_rank, const int32_t* local_expert,
                       const int64_t* offset, long long n_tok, int topk, int world, int epr,
                       int64_t* item_token, int32_t* item_slot, int32_t* item_dst_rank,
                       int32_t* item_dst_expert, int64_t* item_dst_offset) {
  const long long n = n_tok * topk;
  const int nb = epr * world;
  int64_t* start = (int64_t*)calloc((size_t)nb + 1, sizeof(int64_t));
  for (long long i = 0; i < n; ++i) start[(size_t)local_expert[i] * world + target_rank[i] + 1]++;
  for (int b = 0; b < nb; ++b) start[b + 1] += start[b];
  for (long long i = 0; i < n; ++i) {
    int64_t p = start[(size_t)local_expert[i] * world + target_rank[i]]++;
    item_token[p] = i / topk;
    item_slot[p] = (int32_t)(i % topk);
    item_dst_rank[p] = target_rank[i];
    item_dst_expert[p] = local_expert[i];
    item_dst_offset[p] = offset[i];
  }
  free(start);
}

/* sim.cpp:384-390 */
void orc_primary_flags(const int64_t* item_token, const int32_t* item_dst_rank, long long n,
                       int world, int8_t* primary) {
  memset(primary, 0, (size_t)n);
  if (world <= 1) return;
  long long max_tok = 0;
  for (long long i = 0; i < n; ++i)
    if (item_token[i] + 1 > max_tok) max_tok = item_token[i] + 1;
  uint8_t* seen = (uint8_t*)calloc((size_t)max_tok * world + 1, 1);
  for (long long i = 0; i < n; ++i) {
    size_t key = (size_t)item_token[i] * world + item_dst_rank[i];
    if (!seen[key]) {
      seen[key] = 1;
      primary[i] = 1;
    }
  }
  free(seen);
}

/* --------------------------------------------------------------- traffic */
static int mul_ovf(u128 a, u128 b, u128* out) {
  if (a != 0 && b > ((u128)~(u128)0) / a) return 1;
  *out = a * b;
  return 0;
}

/* traffic.cpp:11-22 (exact while the result fits 128 bits) */
int orc_stirling2(int n, int k, uint64_t* hi, uint64_t* lo) {
  if (n < 0 || k < 0 || k > n || n > 64) return 2;
  u128 row[65];
  memset(row, 0, sizeof(row));
  row[0] = 1;
  for (int i = 1; i <= n; ++i) {
    for (int j = (i < k ? i : k); j >= 1; --j) {
      u128 t;
      if (mul_ovf((u128)j, row[j], &t)) return 2;
      t += row[j - 1];
      row[j] = t;
    }
    row[0] = 0;
  }
  *hi = (uint64_t)(row[k] >> 64);
  *lo = (uint64_t)row[k];
  return 0;
}

static u128 binom128(int n, int k) {
  if (k < 0 || k > n) return 0;
  u128 r = 1;
  for (int i = 0; i < k; ++i) {
    r *= (u128)(n - i);
    r /= (u128)(i + 1);
  }
  return r;
}

/* traffic.cpp:49-78 */
int orc_distinct_rank_distribution(int world, int topk, uint64_t* num_hi, uint64_t* num_lo,
                                   double* probs, double* expectation, double* saving) {
  if (world < 1 || topk < 1) return 2;
  u128 den = 1;
  for (int i = 0; i < topk; ++i)
    if (mul_ovf(den, (u128)world, &den)) return 2;
  int xmax = world < topk ? world : topk;
  u128 check = 0, e_num = 0;
  for (int x = 1; x <= xmax; ++x) {
    uint64_t h, l;
    if (orc_stirling2(topk, x, &h, &l)) return 2;
    u128 s2 = ((u128)h << 64) | l, fact = 1, num;
    for (int i = 2; i <= x; ++i) fact *= (u128)i;
    if (mul_ovf(binom128(world, x), fact, &num) || mul_ovf(num, s2, &num)) return 2;
    if (num_hi) num_hi[x - 1] = (uint64_t)(num >> 64);
    if (num_lo) num_lo[x - 1] = (uint64_t)num;
    if (probs) probs[x - 1] = (double)num / (double)den;
    check += num;
    e_num += (u128)x * num;
  }
  if (check != den) return 2;
  double ex = (double)e_num / (double)den;
  double closed = world * (1.0 - pow(1.0 - 1.0 / world, topk));
  if (fabs(ex - closed) > 1e-12 * (closed > 1.0 ? closed : 1.0)) return 2;
  if (expectation) *expectation = ex;
  if (saving) *saving = (topk - ex) / topk;
  return 0;
}

/* traffic.cpp:82-100 */
static void assemble(long long n_tok, int topk, long long s_tok, int world, double mean_nvl,
                     orc_traffic* r) {
  const double s = (double)s_tok, n = (double)n_tok;
  r->v_allgather = (double)world * n * s;
  r->v_alltoall = n * (double)topk * s;
  r->v_megakernel_nvl = world == 1 ? 0.0 : n * mean_nvl * s;
  r->v_megakernel_hbm = r->v_alltoall - r->v_megakernel_nvl;
}

/* traffic.cpp:103-112 */
int orc_volume_expected(long long n_tok, int topk, long long s_tok, int world, int remote_only,
                        orc_traffic* out) {
  double ex;
  if (orc_distinct_rank_distribution(world, topk, NULL, NULL, NULL, &ex, NULL)) return 2;
  if (remote_only && world > 1) ex *= (double)(world - 1) / world;
  assemble(n_tok, topk, s_tok, world, ex, out);
  return 0;
}

/* traffic.cpp:114-140 */
int orc_volume_exact(const int32_t* sel, int world, int n_exp, long long n_tok, int topk,
                     long long s_tok, int remote_only, orc_traffic* out) {
  if (world < 1 || n_exp % world) return 2;
  const int epr = n_exp / world;
  long long total = 0;
  char hit[64];
  for (int r = 0; r < world; ++r)
    for (long long t = 0; t < n_tok; ++t) {
      memset(hit, 0, sizeof(hit));
      for (int j = 0; j < topk; ++j) {
        int dst = sel[((size_t)r * n_tok + t) * topk + j] / epr;
        if (remote_only && dst == r) continue;
        if (!hit[dst]) {
          hit[dst] = 1;
          ++total;
        }
      }
    }
  double copies = (double)n_tok * world;
  double mean = copies > 0 ? (double)total / copies : 0.0;
  assemble(n_tok, topk, s_tok, world, mean, out);
  return 0;
}

/* ------------------------------------------------------------ perf model */
/* perf_model.cpp:11-14 */
double orc_effective_bandwidth(int n, int w, double beta, double w_sat) {
  if (n <= 0) return 0.0;
  double b = (double)n * w * beta / w_sat;
  return b < beta ? b : beta;
}

static int mu_of(const orc_shape* s, int w, double* mu) {
  for (int i = 0; i < s->mu_n; ++i)
    if (s->mu_w[i] == w) {
      *mu = s->mu_v[i];
      return 0;
    }
  return 2;
}

/* perf_model.cpp:16-23 */
int orc_gemm_block_time(const orc_hw* hw, const orc_shape* s, long long k_dim, int w, double* out) {
  double mu;
  if (mu_of(s, w, &mu)) return 2;
  double flops = 2.0 * s->b_m * s->b_n * (double)k_dim;
  *out = flops / (hw->p_peak * (mu / hw->n_sm)) + hw->tau_sync;
  return 0;
}

/* perf_model.cpp:25-29 */
double orc_swiglu(const orc_shape* s, const orc_hw* hw, long long expanded) {
  double s_inter = 2.0 * s->h_inter * 2.0;
  return 2.0 * (double)expanded * s_inter / hw->bw_hbm;
}

/* perf_model.cpp:74-92 */
static long long tiles_for(const orc_shape* s, int world, long long n_out) {
  long long expanded = s->n_tok * s->topk;
  if (expanded == 0) return 0;
  long long epr = s->n_exp / world;
  long long m_e = (expanded + epr - 1) / epr;
  long long rg = (m_e + s->b_m - 1) / s->b_m;
  long long ct = (n_out + s->b_n - 1) / s->b_n;
  return epr * rg * ct;
}
long long orc_tiles_up(const orc_shape* s, int world) { return tiles_for(s, world, 2LL * s->h_inter); }
long long orc_tiles_down(const orc_shape* s, int world) { return tiles_for(s, world, s->h_dim); }

/* perf_model.cpp:94-135 */
int orc_predict_latency(const orc_shape* s, const orc_hw* hw, const orc_cfg* cfg,
                        const orc_traffic* t, int redistributed, orc_breakdown* b) {
  memset(b, 0, sizeof(*b));
  const long long expanded = s->n_tok * s->topk;
  if (orc_gemm_block_time(hw, s, s->h_dim, cfg->w, &b->t_up)) return 2;
  if (orc_gemm_block_time(hw, s, s->h_inter, cfg->w, &b->t_down)) return 2;
  b->l_swiglu = orc_swiglu(s, hw, expanded);
  b->n_tiles_up = orc_tiles_up(s, hw->world_size);
  b->n_tiles_down = orc_tiles_down(s, hw->world_size);

  int n_comp1 = hw->n_sm - cfg->n_disp;
  if (n_comp1 <= 0) return 2;
  /* calc_disp_lat :31-45 */
  double l = 0;
  if (t->v_megakernel_nvl > 0) {
    double bw = orc_effective_bandwidth(cfg->n_disp, cfg->w, hw->bw_nvl, hw->w_sat);
    if (bw <= 0) return 2;
    l += t->v_megakernel_nvl / bw;
  }
  if (t->v_megakernel_hbm > 0) {
    double bw = orc_effective_bandwidth(cfg->n_relay, cfg->w, hw->bw_hbm, hw->w_sat);
    if (bw <= 0) return 2;
    l += t->v_megakernel_hbm / bw;
  }
  b->l_disp = l;
  /* calc_comp_lat :47-52 */
  b->l_up = b->n_tiles_up <= 0 ? 0.0
                               : (double)((b->n_tiles_up + n_comp1 - 1) / n_comp1) * b->t_up;
  if (b->l_up > b->l_disp) {
    double scale = redistributed ? (double)n_comp1 / hw->n_sm : (double)hw->n_sm / n_comp1;
    b->l_s1 = b->l_disp + (b->l_up - b->l_disp) * scale;
  } else {
    b->l_s1 = b->l_disp + b->t_up;
  }
  int n_comp2 = hw->n_sm - cfg->n_comb;
  if (n_comp2 <= 0) return 2;
  /* calc_comb_lat :54-70 */
  b->l_comb = 0;
  if (t->v_megakernel_nvl > 0) {
    double bw = orc_effective_bandwidth(cfg->n_comb, cfg->w, hw->bw_nvl, hw->w_sat);
    if (bw <= 0) return 2;
    b->l_comb = t->v_megakernel_nvl / bw;
  }
  b->t_red = 0;
  if (t->v_alltoall > 0) {
    double b1 = orc_effective_bandwidth(1, cfg->w, hw->bw_hbm, hw->w_sat);
    if (b1 <= 0) return 2;
    b->t_red = t->v_alltoall / b1;
  }
  b->l_down = b->n_tiles_down <= 0
                  ? 0.0
                  : (double)((b->n_tiles_down + n_comp2 - 1) / n_comp2) * b->t_down;
  double l_base = b->l_down > b->l_comb ? b->l_down : b->l_comb;
  b->w_gap = fabs(b->l_down - b->l_comb) * n_comp2;
  b->w_red = b->t_red; /* as in perf_model.cpp:129 (Appendix A.5 of SURVEY.md) */
  b->w_rem = b->w_red - b->w_gap > 0.0 ? b->w_red - b->w_gap : 0.0;
  b->l_s2 = l_base + b->w_rem / hw->n_sm;
  b->l_total = b->l_s1 + b->l_s2 + b->l_swiglu;
  return 0;
}

/* ----------------------------------------------------------------- tuner */
/* tuner.cpp:15-20 */
static int relay_choices(int n_disp, int* out) {
  int c = 0;
  for (int x = 1; x <= n_disp / 2; x += 4) out[c++] = x;
  if (!c) out[c++] = 1;
  return c;
}

/* tuner.cpp:22-45 */
int orc_space_sizes(int n_sm, long long* raw, long long* enumerated, long long* feasible) {
  if (n_sm < 4) return 2;
  int nd = n_sm / 4, nred = 0, relays[512];
  for (int x = 1; x <= n_sm; x += 16) ++nred;
  if (((n_sm - 1) / 16) * 16 + 1 != n_sm) ++nred; /* n_sm appended unless already last */
  long long flat = n_sm / 16 > 1 ? n_sm / 16 : 1;
  *raw = (long long)nd * nd * flat * flat * 3;
  long long en = 0, fe = 0;
  for (int d = 4; d <= n_sm; d += 4) {
    int nr = relay_choices(d, relays);
    en += (long long)nr * nd * nred * 3;
    for (int c = 4; c <= n_sm; c += 4)
      for (int i = 0; i < nr; ++i)
        if (d + relays[i] < n_sm && c < n_sm) fe += (long long)nred * 3;
  }
  *enumerated = en;
  *feasible = fe;
  return 0;
}

/* tuner.cpp:70-86 tie key: asc n_disp, n_comb, n_relay; desc n_red; asc w */
static int tie_less(const orc_cfg* a, const orc_cfg* b) {
  if (a->n_disp != b->n_disp) return a->n_disp < b->n_disp;
  if (a->n_comb != b->n_comb) return a->n_comb < b->n_comb;
  if (a->n_relay != b->n_relay) return a->n_relay < b->n_relay;
  if (a->n_red != b->n_red) return a->n_red > b->n_red;
  return a->w < b->w;
}

/* tuner.cpp:47-66 + :90-148 */
int orc_search(const orc_shape* s, const orc_hw* hw, const orc_traffic* t, int redistributed,
               orc_cfg* best, double* l_min, long long* evaluated) {
  if (hw->n_sm < 4) return 2;
  const int n_sm = hw->n_sm;
  int reds[512], nred = 0, relays[512];
  for (int x = 1; x <= n_sm; x += 16) reds[nred++] = x;
  if (reds[nred - 1] != n_sm) reds[nred++] = n_sm;
  static const int warps[3] = {8, 16, 32};
  int have = 0;
  double bl = 0;
  orc_cfg bc = {0, 0, 0, 0, 0};
  long long n = 0;
  for (int d = 4; d <= n_sm; d += 4) {
    int nr = relay_choices(d, relays);
    for (int c = 4; c <= n_sm; c += 4)
      for (int i = 0; i < nr; ++i)
        for (int q = 0; q < nred; ++q)
          for (int wi = 0; wi < 3; ++wi) {
            orc_cfg cfg = {d, relays[i], c, reds[q], warps[wi]};
            if (d + relays[i] >= n_sm || c >= n_sm) continue;
            orc_breakdown b;
            if (orc_predict_latency(s, hw, &cfg, t, redistributed, &b)) return 2;
            ++n;
            if (!have || b.l_total < bl || (b.l_total == bl && tie_less(&cfg, &bc))) {
              have = 1;
              bl = b.l_total;
              bc = cfg;
            }
          }
  }
  if (!have) return 2;
  *best = bc;
  *l_min = bl;
  *evaluated = n;
  return 0;
}

/* -------------------------------------------------------------- numerics */
/* softfloat.cpp:27-33 */
float orc_round_to_bf16(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if (isnan(x)) {
    u = (u | 0x00400000u) & 0xFFFF0000u;
  } else {
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    u &= 0xFFFF0000u;
  }
  float r;
  memcpy(&r, &u, 4);
  return r;
}

/* precision.cpp:31-37 */
float orc_fold(const float* w, const float* v, int n, int bf16) {
  if (n <= 0) return 0.0f;
#define RND(x) (bf16 ? orc_round_to_bf16(x) : (x))
  float acc = RND(w[0] * v[0]);
  for (int i = 1; i < n; ++i) acc = RND(acc + RND(w[i] * v[i]));
#undef RND
  return acc;
}

/* ------------------------------------------------------- MoE layer numerics */
static inline float bf(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static inline uint16_t tobf(float f) {
  float r = orc_round_to_bf16(f);
  uint32_t u;
  memcpy(&u, &r, 4);
  return (uint16_t)(u >> 16);
}
static inline float silu_f(float g) { return g / (1.0f + expf(-g)); }

void orc_fill_normal_bf16(uint16_t* out, long long n, uint64_t seed, float scale) {
  uint64_t st = seed ^ 0x5DEECE66DULL;
  for (long long i = 0; i < n; i += 2) {
    double u1 = sm_uniform01(&st), u2 = sm_uniform01(&st);
    if (u1 < 1e-300) u1 = 1e-300;
    double rad = sqrt(-2.0 * log(u1));
    out[i] = tobf((float)(rad * cos(6.283185307179586 * u2)) * scale);
    if (i + 1 < n) out[i + 1] = tobf((float)(rad * sin(6.283185307179586 * u2)) * scale);
  }
}

/* Layer contract.
 * Rows of each expert buffer are in global (src, t, j) order (Alg. 1 / token_map.cpp:55-106),
 * which is the accumulation order of the weight gradients. */
int orc_moe_layer(const orc_layer_dims* d, const int32_t* sel, const float* gw,
                  const uint16_t* x, const uint16_t* w_up, const uint16_t* w_down,
                  const uint16_t* dy, uint16_t* y, uint16_t* dx, float* dgate, uint16_t* dw_up,
                  uint16_t* dw_down, int threads) {
  const int W = d->world, E = d->n_exp, K = d->topk, H = d->H, F = d->F;
  const long long T = d->n_tok;
  if (W < 1 || E % W || F <= 0 || H <= 0) return 2;
  if (validate_sel(sel, W, E, T, K)) return 2;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  const long long R = (long long)W * T * K; /* all replicas */
  /* expert buffers: global (src, t, j) order per expert */
  long long* cnt = (long long*)calloc((size_t)E + 1, sizeof(long long));
  for (long long i = 0; i < R; ++i) cnt[sel[i] + 1]++;
  for (int e = 0; e < E; ++e) cnt[e + 1] += cnt[e];
  long long* rows = (long long*)malloc(sizeof(long long) * (size_t)(R > 0 ? R : 1));
  long long* pos = (long long*)malloc(sizeof(long long) * (size_t)(R > 0 ? R : 1));
  {
    long long* cur = (long long*)malloc(sizeof(long long) * (size_t)E);
    for (int e = 0; e < E; ++e) cur[e] = cnt[e];
    for (long long i = 0; i < R; ++i) {
      long long p = cur[sel[i]]++;
      rows[p] = i; /* replica index (r*T + t)*K + j */
      pos[i] = p;
    }
    free(cur);
  }
  uint16_t* gu = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(R > 0 ? R : 1) * 2 * F);
  uint16_t* hh = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(R > 0 ? R : 1) * F);
  uint16_t* o = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(R > 0 ? R : 1) * H);

  /* forward: up GEMM + SwiGLU, down GEMM (per replica row) */
#pragma omp parallel for schedule(dynamic, 4)
  for (long long p = 0; p < R; ++p) {
    const long long i = rows[p];
    const int e = sel[i];
    const uint16_t* xr = x + (size_t)(i / K) * H;
    uint16_t* g = gu + (size_t)p * 2 * F;
    for (int c = 0; c < 2 * F; ++c) {
      const uint16_t* wr = w_up + ((size_t)e * 2 * F + c) * H;
      float acc = 0.0f;
      for (int k = 0; k < H; ++k) acc += bf(xr[k]) * bf(wr[k]);
      g[c] = tobf(acc);
    }
    uint16_t* h = hh + (size_t)p * F;
    for (int f = 0; f < F; ++f) h[f] = tobf(silu_f(bf(g[f])) * bf(g[F + f]));
    uint16_t* orow = o + (size_t)p * H;
    for (int nn = 0; nn < H; ++nn) {
      const uint16_t* wr = w_down + ((size_t)e * H + nn) * F;
      float acc = 0.0f;
      for (int f = 0; f < F; ++f) acc += bf(h[f]) * bf(wr[f]);
      orow[nn] = tobf(acc);
    }
  }
  /* combine: the reference's canonical fold (precision.cpp:31-37, FpFormat::Binary32: acc = w0*v0,
   * acc = acc + wj*vj, j ascending, fp32 rounding of every product and sum), one RNE at the end */
  if (y) {
#pragma omp parallel for
    for (long long rt = 0; rt < (long long)W * T; ++rt) {
      float v[32];
      for (int nn = 0; nn < H; ++nn) {
        for (int j = 0; j < K; ++j) v[j] = bf(o[(size_t)pos[rt * K + j] * H + nn]);
        y[(size_t)rt * H + nn] = tobf(orc_fold(gw + rt * K, v, K, 0));
      }
    }
  }
  if (!dy) goto done;
  {
    uint16_t* dgu = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(R > 0 ? R : 1) * 2 * F);
    uint16_t* hw = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(R > 0 ? R : 1) * F);
    uint16_t* dxr = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)(R > 0 ? R : 1) * H);
    float* dgr = (float*)malloc(sizeof(float) * (size_t)(R > 0 ? R : 1));
#pragma omp parallel for schedule(dynamic, 4)
    for (long long p = 0; p < R; ++p) {
      const long long i = rows[p];
      const int e = sel[i];
      const float w = gw[i];
      const uint16_t* dyr = dy + (size_t)(i / K) * H;
      const uint16_t* g = gu + (size_t)p * 2 * F;
      uint16_t* dg = dgu + (size_t)p * 2 * F;
      /* gate gradient dgate = <dY, o> = <dY W_down, h>: the dgrad accumulator (before the gate
       * weight) dotted with the bf16 h, f ascending -- the quantity the down-dgrad epilogue forms */
      float gsum = 0.0f;
      for (int f = 0; f < F; ++f) {
        float acc = 0.0f;
        for (int nn = 0; nn < H; ++nn) acc += bf(dyr[nn]) * bf(w_down[((size_t)e * H + nn) * F + f]);
        gsum += acc * bf(hh[(size_t)p * F + f]);
        const float dh = w * acc;
        const float gg = bf(g[f]), uu = bf(g[F + f]);
        const float s = 1.0f / (1.0f + expf(-gg));
        const float si = gg * s;
        const float ds = s * (1.0f + gg * (1.0f - s));
        dg[f] = tobf(dh * uu * ds);
        dg[F + f] = tobf(dh * si);
        hw[(size_t)p * F + f] = tobf(w * bf(hh[(size_t)p * F + f]));
      }
      dgr[p] = gsum;
      for (int k = 0; k < H; ++k) {
        float acc = 0.0f;
        for (int c = 0; c < 2 * F; ++c) acc += bf(dg[c]) * bf(w_up[((size_t)e * 2 * F + c) * H + k]);
        dxr[(size_t)p * H + k] = tobf(acc);
      }
    }
    if (dx) {
      /* the same fold with unit weights: dx = bf16(dX_0 + dX_1 + ...) in j order */
#pragma omp parallel for
      for (long long rt = 0; rt < (long long)W * T; ++rt) {
        float v[32], one[32];
        for (int j = 0; j < K; ++j) one[j] = 1.0f;
        for (int k = 0; k < H; ++k) {
          for (int j = 0; j < K; ++j) v[j] = bf(dxr[(size_t)pos[rt * K + j] * H + k]);
          dx[(size_t)rt * H + k] = tobf(orc_fold(one, v, K, 0));
        }
      }
    }
    if (dgate)
      for (long long i = 0; i < R; ++i) dgate[i] = dgr[pos[i]];
    free(dgr);
    if (dw_down) {
#pragma omp parallel for collapse(2) schedule(dynamic, 8)
      for (int e = 0; e < E; ++e)
        for (int nn = 0; nn < H; ++nn)
          for (int f = 0; f < F; ++f) {
            float acc = 0.0f;
            for (long long p = cnt[e]; p < cnt[e + 1]; ++p)
              acc += bf(dy[(size_t)(rows[p] / K) * H + nn]) * bf(hw[(size_t)p * F + f]);
            dw_down[((size_t)e * H + nn) * F + f] = tobf(acc);
          }
    }
    if (dw_up) {
#pragma omp parallel for collapse(2) schedule(dynamic, 8)
      for (int e = 0; e < E; ++e)
        for (int c = 0; c < 2 * F; ++c)
          for (int k = 0; k < H; ++k) {
            float acc = 0.0f;
            for (long long p = cnt[e]; p < cnt[e + 1]; ++p)
              acc += bf(dgu[(size_t)p * 2 * F + c]) * bf(x[(size_t)(rows[p] / K) * H + k]);
            dw_up[((size_t)e * 2 * F + c) * H + k] = tobf(acc);
          }
    }
    free(dgu);
    free(hw);
    free(dxr);
  }
done:
  free(cnt);
  free(rows);
  free(pos);
  free(gu);
  free(hh);
  free(o);
  return 0;
}

/* ------------------------------------------------------------- router (§8 f1) */
/* See eplab_oracle.h: semantics defined by this repo. */
float orc_exp_portable(float x) {
  if (!(x >= -87.0f)) return 0.0f;
  const float n = rintf(x * 1.44269504088896341f);
  float r = fmaf(-n, 0.693145751953125f, x);
  r = fmaf(-n, 1.42860682030941723212e-6f, r);
  float p = 1.98412698412698413e-4f;
  p = fmaf(p, r, 1.38888888888888889e-3f);
  p = fmaf(p, r, 8.33333333333333333e-3f);
  p = fmaf(p, r, 4.16666666666666667e-2f);
  p = fmaf(p, r, 1.66666666666666667e-1f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  const int e = (int)n;
  uint32_t bits = (uint32_t)(e + 127) << 23;
  float s;
  memcpy(&s, &bits, 4);
  return p * s;
}

static uint32_t rt_key(float v) {
  uint32_t u;
  memcpy(&u, &v, 4);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

/* sum_i exp(l_i - m) in the kernel's order: 32 lane partials (i = lane + 32q, q ascending),
 * then v[l] += v[l ^ o] for o = 16, 8, 4, 2, 1 */
static float rt_partition(const float* l, int E, float m) {
  float v[32], nv[32];
  for (int lane = 0; lane < 32; ++lane) {
    float s = 0.0f;
    for (int i = lane; i < E; i += 32) s = s + orc_exp_portable(l[i] - m);
    v[lane] = s;
  }
  for (int o = 16; o; o >>= 1) {
    for (int lane = 0; lane < 32; ++lane) nv[lane] = v[lane] + v[lane ^ o];
    memcpy(v, nv, sizeof v);
  }
  return v[0];
}

static int rt_check(long long T, int E, int k) {
  return (T < 0 || E < 1 || E > 1024 || k < 1 || k > 32 || k > E) ? 2 : 0;
}

int orc_router_topk(const float* logits, long long n_tok, int n_exp, int topk, int renorm, int32_t* ids,
                    float* gw) {
  if (rt_check(n_tok, n_exp, topk)) return 2;
  for (long long t = 0; t < n_tok; ++t) {
    const float* l = logits + t * n_exp;
    unsigned char taken[1024];
    memset(taken, 0, (size_t)n_exp);
    float val[32], m = 0.0f, den = 0.0f;
    for (int j = 0; j < topk; ++j) {
      int best = -1;
      for (int i = 0; i < n_exp; ++i)
        if (!taken[i] && (best < 0 || rt_key(l[i]) > rt_key(l[best]))) best = i;
      taken[best] = 1;
      ids[t * topk + j] = best;
      val[j] = l[best];
      if (j == 0) m = val[0];
      if (renorm) den = den + orc_exp_portable(val[j] - m);
    }
    if (!renorm) den = rt_partition(l, n_exp, m);
    for (int j = 0; j < topk; ++j) gw[t * topk + j] = orc_exp_portable(val[j] - m) / den;
  }
  return 0;
}

int orc_router_topk_bwd(const float* logits, const int32_t* ids, const float* gw, const float* dgate,
                        long long n_tok, int n_exp, int topk, int renorm, float* dlogits) {
  if (rt_check(n_tok, n_exp, topk)) return 2;
  for (long long t = 0; t < n_tok; ++t) {
    const int32_t* id = ids + t * topk;
    const float *w = gw + t * topk, *g = dgate + t * topk, *l = logits + t * n_exp;
    float* out = dlogits + t * n_exp;
    float S = 0.0f;
    for (int j = 0; j < topk; ++j) S = fmaf(g[j], w[j], S);
    if (renorm) {
      for (int i = 0; i < n_exp; ++i) out[i] = 0.0f;
      for (int j = 0; j < topk; ++j) out[id[j]] = w[j] * (g[j] - S);
    } else {
      int best = 0;
      for (int i = 1; i < n_exp; ++i)
        if (rt_key(l[i]) > rt_key(l[best])) best = i;
      const float m = l[best], Z = rt_partition(l, n_exp, m);
      for (int i = 0; i < n_exp; ++i) out[i] = (orc_exp_portable(l[i] - m) / Z) * -S;
      for (int j = 0; j < topk; ++j)
        out[id[j]] = (orc_exp_portable(l[id[j]] - m) / Z) * (g[j] - S);
    }
  }
  return 0;
}

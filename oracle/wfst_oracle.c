/*
 * oracle/wfst_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1910_10032_b200/) never links, imports or calls it, and shares no
 * code, header, table or helper with it.
 *
 * What it computes: serial frame-synchronous token-passing Viterbi beam
 * search over a WFST (§3, "for each frame ... processes
 * emitting arcs (those arcs with non-null labels) conditioned on frame
 * values, processes any chains of non-emitting arcs, and finally performs
 * pruning"), in the step order of Fig. 1 (Expand -> Set Beam via
 * max-active -> Contract -> Non-emitting -> representatives for the next
 * frame), one-best output by traceback.  The readings R1-R12 it implements
 * are listed in DESIGN.md §3 (taken from SURVEY.md §8.4):
 *   R1  fp32, fixed order: emitting c' = (c + w) - L[t][pdf]; eps c' = c + w;
 *       final c + F.  Built with -ffp-contract=off (no FMA).
 *   R2  emitting <=> ilabel != 0, pdf = ilabel - 1.
 *   R3  init: token (start, 0, arc -1), eps-closure with keep(c) = c < beam.
 *   R4  emitting candidates, one per destination state, min by (cost, arc).
 *   R5  best = min candidate cost, beam_cut = fl(best + beam), keep c < beam_cut.
 *   R6  exact max-active: if n = #{c < beam_cut} > alpha, k = alpha-th
 *       smallest of those costs, keep(c) = c < beam_cut && c <= k.
 *   R7  eps-closure under the FIXED keep() of the frame, worklist to the
 *       least fixed point; relaxations whose result fails keep() are dropped.
 *   R8  survivors = states whose final entry passes keep(): one token per
 *       state (the representative).
 *   R9  ties broken by (cost, canonical arc id).
 *   R10 finals: argmin c + F over final survivors; else argmin c, flag 0.
 *   R11 traceback by back-pointers: emitting arc -> previous layer,
 *       eps arc -> same layer.
 * NEXT rows: oracle_lattice / oracle_lattice_finalize (R13-R14,
 * lattice segments and the final backward sweep) and the histogram max-active
 * rule of oracle_decode_mode (R16).
 * Canonical arc ids: arcs stably bucketed by (src, emitting-first) in input
 * order ("within a span, emitting arcs precede non-emitting").
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { O_OK = 0, O_INVALID = 1, O_PDF_RANGE = 5, O_CAPACITY = 6, O_NO_SURVIVOR = 7, O_OOM = 9 };

typedef struct {
  int32_t Q, start;
  int64_t E;
  int64_t *first;   /* [Q+1] canonical arc offsets                        */
  int32_t *n_emit;  /* [Q] emitting arcs of the state (they come first)   */
  int32_t *src, *dst, *ilabel, *olabel; /* [E] canonical order           */
  float *weight;    /* [E]                                                */
  float *final;     /* [Q] +inf = non-final                               */
  int64_t *perm;    /* canonical arc i = input arc perm[i]                */
  int32_t max_pdf;
} OGraph;

void oracle_graph_free(void *gp) {
  OGraph *g = (OGraph *)gp;
  if (!g) return;
  free(g->first); free(g->n_emit); free(g->src); free(g->dst); free(g->ilabel);
  free(g->olabel); free(g->weight); free(g->final); free(g->perm); free(g);
}

int oracle_graph_new(int32_t Q, int32_t start, int64_t E, const int32_t *src, const int32_t *dst,
                     const int32_t *ilabel, const int32_t *olabel, const float *weight,
                     const float *final, void **out) {
  if (Q <= 0 || start < 0 || start >= Q || E < 0 || !out) return O_INVALID;
  OGraph *g = (OGraph *)calloc(1, sizeof(OGraph));
  if (!g) return O_OOM;
  g->Q = Q; g->start = start; g->E = E; g->max_pdf = -1;
  g->first = (int64_t *)calloc((size_t)Q + 1, sizeof(int64_t));
  g->n_emit = (int32_t *)calloc((size_t)Q, sizeof(int32_t));
  size_t e1 = (size_t)(E > 0 ? E : 1);
  g->src = (int32_t *)malloc(e1 * 4); g->dst = (int32_t *)malloc(e1 * 4);
  g->ilabel = (int32_t *)malloc(e1 * 4); g->olabel = (int32_t *)malloc(e1 * 4);
  g->weight = (float *)malloc(e1 * 4); g->final = (float *)malloc((size_t)Q * 4);
  g->perm = (int64_t *)malloc(e1 * 8);
  int64_t *cur_e = (int64_t *)malloc((size_t)Q * 8), *cur_n = (int64_t *)malloc((size_t)Q * 8);
  if (!g->first || !g->n_emit || !g->src || !g->dst || !g->ilabel || !g->olabel || !g->weight ||
      !g->final || !g->perm || !cur_e || !cur_n) {
    free(cur_e); free(cur_n); oracle_graph_free(g); return O_OOM;
  }
  int32_t *n_all = (int32_t *)calloc((size_t)Q, 4);
  for (int64_t i = 0; i < E; i++) {
    if (src[i] < 0 || src[i] >= Q || dst[i] < 0 || dst[i] >= Q || ilabel[i] < 0) {
      free(n_all); free(cur_e); free(cur_n); oracle_graph_free(g); return O_INVALID;
    }
    n_all[src[i]]++;
    if (ilabel[i] != 0) g->n_emit[src[i]]++;
  }
  for (int32_t q = 0; q < Q; q++) g->first[q + 1] = g->first[q] + n_all[q];
  for (int32_t q = 0; q < Q; q++) { cur_e[q] = g->first[q]; cur_n[q] = g->first[q] + g->n_emit[q]; }
  for (int64_t i = 0; i < E; i++) {          /* stable bucket: emitting first */
    int32_t s = src[i];
    int64_t k = ilabel[i] != 0 ? cur_e[s]++ : cur_n[s]++;
    g->src[k] = s; g->dst[k] = dst[i]; g->ilabel[k] = ilabel[i]; g->olabel[k] = olabel[i];
    g->weight[k] = weight[i] + 0.0f;        /* canonical +0 */
    g->perm[k] = i;
    if (ilabel[i] - 1 > g->max_pdf) g->max_pdf = ilabel[i] - 1;
  }
  for (int32_t q = 0; q < Q; q++) g->final[q] = final[q];
  free(n_all); free(cur_e); free(cur_n);
  *out = g;
  return O_OK;
}

int oracle_graph_perm(void *gp, int64_t *perm_out) {
  OGraph *g = (OGraph *)gp;
  memcpy(perm_out, g->perm, (size_t)g->E * 8);
  return O_OK;
}

int32_t oracle_graph_max_pdf(void *gp) { return ((OGraph *)gp)->max_pdf; }

/* (cost, arc) lexicographic "less"; arc -1 (the start token) sorts last (R9). */
static int lex_less(float c1, int32_t a1, float c2, int32_t a2) {
  if (c1 < c2) return 1;
  if (c1 > c2) return 0;
  return (uint32_t)a1 < (uint32_t)a2;
}

static int cmp_float(const void *x, const void *y) {
  float a = *(const float *)x, b = *(const float *)y;
  return (a > b) - (a < b);
}

static int cmp_int(const void *x, const void *y) {
  int32_t a = *(const int32_t *)x, b = *(const int32_t *)y;
  return (a > b) - (a < b);
}

typedef struct {       /* one layer of survivors, sorted by state */
  int32_t n;
  int32_t *state, *arc;
  float *cost;
} Layer;

typedef struct {
  const OGraph *g;
  /* dense per-state scratch */
  float *dcost; int32_t *darc; uint8_t *seen, *inq;
  int32_t *touched, n_touched;
  int32_t *queue;  /* FIFO of capacity Q (each state queued at most once at a time) */
  float *tmp;      /* costs for max-active selection */
  Layer *layers;   /* T+1 */
  int32_t n_layers;
} Work;

static void work_free(Work *w) {
  free(w->dcost); free(w->darc); free(w->seen); free(w->inq); free(w->touched);
  free(w->queue); free(w->tmp);
  if (w->layers)
    for (int32_t k = 0; k < w->n_layers; k++) {
      free(w->layers[k].state); free(w->layers[k].arc); free(w->layers[k].cost);
    }
  free(w->layers);
}

/* keep() of R5/R6: c < beam_cut && (no alpha || c <= kalpha) */
typedef struct { float beam_cut, kalpha; int use_alpha; } Keep;
static int keep(const Keep *k, float c) { return c < k->beam_cut && (!k->use_alpha || c <= k->kalpha); }

static void touch(Work *w, int32_t q, float c, int32_t a) {
  w->seen[q] = 1; w->dcost[q] = c; w->darc[q] = a; w->touched[w->n_touched++] = q;
}

/* R7: eps-closure to the least fixed point under a fixed keep().  Returns the
 * number of eps arc relaxations performed (implementation-dependent count). */
static int64_t eps_closure(Work *w, const Keep *k) {
  const OGraph *g = w->g;
  int64_t relax = 0;
  int32_t head = 0, tail = 0, Q = g->Q;  /* circular FIFO, <= Q entries */
  int32_t cnt = 0;
  for (int32_t i = 0; i < w->n_touched; i++) {
    int32_t q = w->touched[i];
    if (keep(k, w->dcost[q]) && g->first[q] + g->n_emit[q] < g->first[q + 1]) {
      w->queue[tail] = q; tail = (tail + 1) % Q; cnt++; w->inq[q] = 1;
    }
  }
  while (cnt > 0) {
    int32_t p = w->queue[head]; head = (head + 1) % Q; cnt--; w->inq[p] = 0;
    float cp = w->dcost[p];
    if (!keep(k, cp)) continue;
    for (int64_t e = g->first[p] + g->n_emit[p]; e < g->first[p + 1]; e++) {
      float c = cp + g->weight[e];
      relax++;
      if (!keep(k, c)) continue;
      int32_t q = g->dst[e];
      if (!w->seen[q]) {
        touch(w, q, c, (int32_t)e);
      } else if (lex_less(c, (int32_t)e, w->dcost[q], w->darc[q])) {
        w->dcost[q] = c; w->darc[q] = (int32_t)e;
      } else {
        continue;
      }
      if (!w->inq[q] && g->first[q] + g->n_emit[q] < g->first[q + 1]) {
        w->queue[tail] = q; tail = (tail + 1) % Q; cnt++; w->inq[q] = 1;
      }
    }
  }
  return relax;
}

/* R8: survivors of the layer, sorted by state; clears the scratch. */
static int make_layer(Work *w, const Keep *k, Layer *L, int64_t *eps_deg_sum) {
  const OGraph *g = w->g;
  int32_t n = 0;
  for (int32_t i = 0; i < w->n_touched; i++)
    if (keep(k, w->dcost[w->touched[i]])) n++;
  L->n = n;
  L->state = (int32_t *)malloc((size_t)(n ? n : 1) * 4);
  L->arc = (int32_t *)malloc((size_t)(n ? n : 1) * 4);
  L->cost = (float *)malloc((size_t)(n ? n : 1) * 4);
  if (!L->state || !L->arc || !L->cost) return O_OOM;
  int32_t j = 0;
  for (int32_t i = 0; i < w->n_touched; i++) {
    int32_t q = w->touched[i];
    if (keep(k, w->dcost[q])) L->state[j++] = q;
  }
  qsort(L->state, (size_t)n, 4, cmp_int);
  int64_t es = 0;
  for (int32_t i = 0; i < n; i++) {
    int32_t q = L->state[i];
    L->arc[i] = w->darc[q]; L->cost[i] = w->dcost[q];
    es += (g->first[q + 1] - g->first[q]) - g->n_emit[q];
  }
  if (eps_deg_sum) *eps_deg_sum = es;
  for (int32_t i = 0; i < w->n_touched; i++) w->seen[w->touched[i]] = 0;
  w->n_touched = 0;
  return O_OK;
}

static int32_t layer_find(const Layer *L, int32_t q) {
  int32_t lo = 0, hi = L->n - 1;
  while (lo <= hi) {
    int32_t m = (lo + hi) / 2;
    if (L->state[m] == q) return m;
    if (L->state[m] < q) lo = m + 1; else hi = m - 1;
  }
  return -1;
}

/*
 * Decode one stream.  ll points at frame 0's row; frame t's row is
 * ll + t*ll_stride (P floats, pdf-indexed).  beam may be +inf; max_active
 * <= 0 means unbounded.  Outputs (all nullable except cost/reached_final):
 *   arcs[arcs_cap], *n_arcs     canonical arc ids of the best path
 *   olabels[ol_cap], *n_ol      its non-zero olabels
 *   fstats[T*3]                 per frame: best, beam_cut, kalpha (+inf if unused)
 *   fcounts[T*5]                per frame: n_cand, n_inbeam, n_surv,
 *                               emitting arcs expanded, eps arcs of survivors
 *   surv_n[T+1]                 survivors per layer (layer 0 = after init)
 *   surv_state/arc/cost[surv_cap] concatenated layers, sorted by state
 */
/* R16 (row f4, opt-in, NEXT): the paper's histogram max-active -- "Set Beam via max-active"
 * (Fig. 1) implemented with a histogram whose thresholds are "somewhat arbitrary".
 * Written out deterministically: NB bins of width wd = beam/NB over [best, best + beam),
 * bin(c) = (int) clamp((c - best) * (NB/beam), 0, NB-1); b = the smallest bin whose cumulative
 * in-beam count reaches alpha; adaptive cutoff ca = best + (b+1)*wd; keep c < ca (stored as
 * kalpha = the largest float below ca, so keep() stays c <= kalpha).  fp32, this order. */
#define HIST_NB 1024
static float hist_cutoff(const float *cand, int32_t n, float best, float beam, int32_t alpha) {
  int32_t h[HIST_NB];
  memset(h, 0, sizeof h);
  const float inv = (float)HIST_NB / beam, wd = beam / (float)HIST_NB;
  for (int32_t i = 0; i < n; i++) {
    float x = (cand[i] - best) * inv;
    if (x > (float)(HIST_NB - 1)) x = (float)(HIST_NB - 1);
    if (x < 0.0f) x = 0.0f;
    h[(int)x]++;
  }
  int32_t b = 0, cum = 0;
  for (b = 0; b < HIST_NB; b++) {
    cum += h[b];
    if (cum >= alpha) break;
  }
  const float ca = best + (float)(b + 1) * wd;
  return nextafterf(ca, -INFINITY);
}

static int decode_impl(void *gp, const float *ll, int64_t ll_stride, int32_t T, int32_t P, float beam,
                       int32_t max_active, int alpha_mode, float *cost, int32_t *reached_final,
                       int32_t *arcs, int32_t arcs_cap, int32_t *n_arcs, int32_t *olabels,
                       int32_t ol_cap, int32_t *n_ol, float *fstats, int64_t *fcounts,
                       int32_t *surv_n, int32_t *surv_state, int32_t *surv_arc, float *surv_cost,
                       int64_t surv_cap, int64_t *eps_relax_total) {
  const OGraph *g = (const OGraph *)gp;
  if (!g || T < 0 || (T > 0 && (!ll || P <= 0)) || !cost || !reached_final) return O_INVALID;
  if (T > 0 && P <= g->max_pdf) return O_PDF_RANGE;
  int32_t Q = g->Q;
  Work w;
  memset(&w, 0, sizeof w);
  w.g = g;
  w.dcost = (float *)malloc((size_t)Q * 4); w.darc = (int32_t *)malloc((size_t)Q * 4);
  w.seen = (uint8_t *)calloc((size_t)Q, 1); w.inq = (uint8_t *)calloc((size_t)Q, 1);
  w.touched = (int32_t *)malloc((size_t)Q * 4); w.queue = (int32_t *)malloc((size_t)Q * 4);
  w.tmp = (float *)malloc((size_t)Q * 4);
  w.layers = (Layer *)calloc((size_t)T + 1, sizeof(Layer));
  w.n_layers = T + 1;
  int rc = O_OK;
  int64_t relax_total = 0;
  if (!w.dcost || !w.darc || !w.seen || !w.inq || !w.touched || !w.queue || !w.tmp || !w.layers) {
    rc = O_OOM; goto done;
  }

  /* R3: start token and the initial eps-closure, keep(c) = c < fl(0 + beam) */
  {
    Keep k0 = {0.0f + beam, INFINITY, 0};
    touch(&w, g->start, 0.0f, -1);
    relax_total += eps_closure(&w, &k0);
    rc = make_layer(&w, &k0, &w.layers[0], NULL);
    if (rc) goto done;
  }

  for (int32_t t = 0; t < T; t++) {
    const float *row = ll + (int64_t)t * ll_stride;
    const Layer *prev = &w.layers[t];
    int64_t n_emit_arcs = 0;
    /* R4: emitting arcs of every survivor, conditioned on the frame */
    for (int32_t i = 0; i < prev->n; i++) {
      int32_t p = prev->state[i];
      float cp = prev->cost[i];
      for (int64_t a = g->first[p]; a < g->first[p] + g->n_emit[p]; a++) {
        float c = (cp + g->weight[a]) - row[g->ilabel[a] - 1];
        int32_t q = g->dst[a];
        n_emit_arcs++;
        if (!w.seen[q]) touch(&w, q, c, (int32_t)a);
        else if (lex_less(c, (int32_t)a, w.dcost[q], w.darc[q])) { w.dcost[q] = c; w.darc[q] = (int32_t)a; }
      }
    }
    if (w.n_touched == 0) { rc = O_NO_SURVIVOR; goto done; }
    /* R5: beam against the stream's best candidate (Fig. 1 "Set Beam") */
    float best = INFINITY;
    for (int32_t i = 0; i < w.n_touched; i++)
      if (w.dcost[w.touched[i]] < best) best = w.dcost[w.touched[i]];
    Keep k = {best + beam, INFINITY, 0};
    int32_t n_in = 0;
    for (int32_t i = 0; i < w.n_touched; i++)
      if (w.dcost[w.touched[i]] < k.beam_cut) w.tmp[n_in++] = w.dcost[w.touched[i]];
    /* R6: exact max-active (alpha-th smallest in-beam cost); R16: the histogram variant */
    if (max_active > 0 && n_in > max_active) {
      if (alpha_mode == 1) {
        k.kalpha = hist_cutoff(w.tmp, n_in, best, beam, max_active);
      } else {
        qsort(w.tmp, (size_t)n_in, 4, cmp_float);
        k.kalpha = w.tmp[max_active - 1];
      }
      k.use_alpha = 1;
    }
    int32_t n_cand = w.n_touched;
    /* R7: eps chains to convergence under the fixed cutoff */
    relax_total += eps_closure(&w, &k);
    int64_t eps_deg = 0;
    rc = make_layer(&w, &k, &w.layers[t + 1], &eps_deg);
    if (rc) goto done;
    if (fstats) {
      fstats[3 * t] = best; fstats[3 * t + 1] = k.beam_cut;
      fstats[3 * t + 2] = k.use_alpha ? k.kalpha : INFINITY;
    }
    if (fcounts) {
      fcounts[5 * t] = n_cand; fcounts[5 * t + 1] = n_in; fcounts[5 * t + 2] = w.layers[t + 1].n;
      fcounts[5 * t + 3] = n_emit_arcs; fcounts[5 * t + 4] = eps_deg;
    }
  }

  /* R10: final costs */
  {
    const Layer *L = &w.layers[T];
    int32_t bi = -1; float bc = INFINITY; int32_t ba = -1;
    for (int32_t i = 0; i < L->n; i++) {
      float F = g->final[L->state[i]];
      if (!(F < INFINITY)) continue;
      float c = L->cost[i] + F;
      if (bi < 0 || lex_less(c, L->arc[i], bc, ba)) { bi = i; bc = c; ba = L->arc[i]; }
    }
    *reached_final = bi >= 0;
    if (bi < 0)
      for (int32_t i = 0; i < L->n; i++)
        if (bi < 0 || lex_less(L->cost[i], L->arc[i], bc, ba)) { bi = i; bc = L->cost[i]; ba = L->arc[i]; }
    if (bi < 0) { rc = O_NO_SURVIVOR; goto done; }
    *cost = bc;
    /* R11: traceback */
    int32_t layer = T, q = L->state[bi], n = 0, no = 0;
    int64_t guard = ((int64_t)T + 1) * ((int64_t)Q + 1);
    int32_t cap_path = 1024;
    int32_t *path = (int32_t *)malloc((size_t)cap_path * 4);
    while (path) {
      int32_t j = layer_find(&w.layers[layer], q);
      if (j < 0 || guard-- <= 0) { free(path); path = NULL; rc = O_INVALID; break; }
      int32_t a = w.layers[layer].arc[j];
      if (a < 0) break;
      if (n == cap_path) {
        cap_path *= 2;
        int32_t *np_ = (int32_t *)realloc(path, (size_t)cap_path * 4);
        if (!np_) { free(path); path = NULL; rc = O_OOM; break; }
        path = np_;
      }
      path[n++] = a;
      q = g->src[a];
      if (g->ilabel[a] != 0) layer--;
    }
    if (!path) goto done;
    if (n_arcs) *n_arcs = n;
    for (int32_t i = 0; i < n; i++) {
      int32_t a = path[n - 1 - i];
      if (arcs && i < arcs_cap) arcs[i] = a;
      if (g->olabel[a] != 0) {
        if (olabels && no < ol_cap) olabels[no] = g->olabel[a];
        no++;
      }
    }
    if (n_ol) *n_ol = no;
    free(path);
    if ((arcs && n > arcs_cap) || (olabels && no > ol_cap)) rc = O_CAPACITY;
  }
  if (surv_n) {
    int64_t off = 0;
    for (int32_t k = 0; k <= T; k++) {
      const Layer *L = &w.layers[k];
      surv_n[k] = L->n;
      for (int32_t i = 0; i < L->n; i++, off++) {
        if (off >= surv_cap) continue;
        if (surv_state) surv_state[off] = L->state[i];
        if (surv_arc) surv_arc[off] = L->arc[i];
        if (surv_cost) surv_cost[off] = L->cost[i];
      }
    }
    if (off > surv_cap && (surv_state || surv_arc || surv_cost)) rc = rc ? rc : O_CAPACITY;
  }
  if (eps_relax_total) *eps_relax_total = relax_total;
done:
  work_free(&w);
  return rc;
}

int oracle_decode(void *gp, const float *ll, int64_t ll_stride, int32_t T, int32_t P, float beam,
                  int32_t max_active, float *cost, int32_t *reached_final, int32_t *arcs,
                  int32_t arcs_cap, int32_t *n_arcs, int32_t *olabels, int32_t ol_cap,
                  int32_t *n_ol, float *fstats, int64_t *fcounts, int32_t *surv_n,
                  int32_t *surv_state, int32_t *surv_arc, float *surv_cost, int64_t surv_cap,
                  int64_t *eps_relax_total) {
  return decode_impl(gp, ll, ll_stride, T, P, beam, max_active, 0, cost, reached_final, arcs, arcs_cap,
                     n_arcs, olabels, ol_cap, n_ol, fstats, fcounts, surv_n, surv_state, surv_arc,
                     surv_cost, surv_cap, eps_relax_total);
}

/* Same with the max-active rule selected: 0 exact (R6), 1 histogram (R16). */
int oracle_decode_mode(void *gp, const float *ll, int64_t ll_stride, int32_t T, int32_t P, float beam,
                       int32_t max_active, int32_t alpha_mode, float *cost, int32_t *reached_final,
                       int32_t *arcs, int32_t arcs_cap, int32_t *n_arcs, int32_t *olabels,
                       int32_t ol_cap, int32_t *n_ol, float *fstats, int64_t *fcounts) {
  return decode_impl(gp, ll, ll_stride, T, P, beam, max_active, alpha_mode, cost, reached_final, arcs,
                     arcs_cap, n_arcs, olabels, ol_cap, n_ol, fstats, fcounts, NULL, NULL, NULL, NULL,
                     0, NULL);
}

/* ---- row f1 (NEXT): lattice segments and the end-of-utterance lattice ----
 *
 * oracle_lattice builds the per-frame lattice segments of one stream (Fig. 1 "Preprocess
 * Lattice"; "detecting tokens linked to the same FST state, listing them in the
 * CSR format, designing a unique representative for each FST state, and computing extra costs";
 * lattice-beam P:146; readings R13-R14 in DESIGN.md).  Its inputs are oracle_decode's outputs for
 * the same stream: the layers (surv_n, surv_state, surv_cost; each layer sorted by state, its
 * tokens are the representatives) and fstats (the cutoff of each frame).  Segment k (k = 0: the
 * initial closure, k = t+1: frame t) lists every arc a such that
 *   - a is emitting, leaves the token i of layer k-1 and c = (cost_i + w) - L[k-1][pdf], or
 *     a is non-emitting, leaves the token i of layer k and c = cost_i + w  (R1 arithmetic);
 *   - c passes frame k's keep() (R5/R6; k = 0: c < fl(0 + beam));
 *   - s = c - cost_j <= lattice_beam, j the token of dst(a) in layer k (s is the arc's
 *     forward extra cost; the representative j has the smallest c, so s >= 0).
 * Soft pruning: only representatives have out-arcs, which is what "leaves the token i"
 * means.  Output: for k = 0..T, seg_n[k] arcs (arc, i, j, s), grouped by j (CSR order) and by
 * arc id inside a group; i and j index the layers as output by oracle_decode. */
typedef struct { int32_t arc, src, dst; float slack; } LArc;

static int cmp_larc(const void *x, const void *y) {
  const LArc *a = (const LArc *)x, *b = (const LArc *)y;
  if (a->dst != b->dst) return (a->dst > b->dst) - (a->dst < b->dst);
  return (a->arc > b->arc) - (a->arc < b->arc);
}

static int32_t sorted_find(const int32_t *st, int32_t n, int32_t q) {
  int32_t lo = 0, hi = n - 1;
  while (lo <= hi) {
    int32_t m = (lo + hi) / 2;
    if (st[m] == q) return m;
    if (st[m] < q) lo = m + 1; else hi = m - 1;
  }
  return -1;
}

int oracle_lattice(void *gp, const float *ll, int64_t ll_stride, int32_t T, float beam,
                   float lattice_beam, const float *fstats, const int32_t *surv_n,
                   const int32_t *surv_state, const float *surv_cost, int32_t *seg_n,
                   int32_t *l_arc, int32_t *l_src, int32_t *l_dst, float *l_slack, int64_t cap,
                   int64_t *n_total) {
  const OGraph *g = (const OGraph *)gp;
  if (!g || T < 0 || !surv_n || !surv_state || !surv_cost || !seg_n || !n_total) return O_INVALID;
  int64_t *off = (int64_t *)malloc(((size_t)T + 2) * 8);
  if (!off) return O_OOM;
  off[0] = 0;
  for (int32_t k = 0; k <= T; k++) off[k + 1] = off[k] + surv_n[k];
  int rc = O_OK;
  int64_t out = 0;
  for (int32_t k = 0; k <= T && rc == O_OK; k++) {
    Keep kp = {0.0f + beam, INFINITY, 0};
    if (k > 0) {
      kp.beam_cut = fstats[3 * (k - 1) + 1];
      kp.kalpha = fstats[3 * (k - 1) + 2];
      kp.use_alpha = kp.kalpha < INFINITY;
    }
    const int32_t *st_k = surv_state + off[k];
    const float *co_k = surv_cost + off[k];
    const int32_t n_k = surv_n[k];
    /* candidate arcs: emitting from layer k-1, then non-emitting from layer k */
    int64_t n_cand = 0;
    if (k > 0)
      for (int32_t i = 0; i < surv_n[k - 1]; i++) n_cand += g->n_emit[surv_state[off[k - 1] + i]];
    for (int32_t i = 0; i < n_k; i++) {
      int32_t p = st_k[i];
      n_cand += (g->first[p + 1] - g->first[p]) - g->n_emit[p];
    }
    LArc *buf = (LArc *)malloc((size_t)(n_cand ? n_cand : 1) * sizeof(LArc));
    if (!buf) { rc = O_OOM; break; }
    int64_t nb = 0;
    for (int pass = 0; pass < 2 && rc == O_OK; pass++) {
      if (pass == 0 && k == 0) continue;
      const int32_t *st_s = pass == 0 ? surv_state + off[k - 1] : st_k;
      const float *co_s = pass == 0 ? surv_cost + off[k - 1] : co_k;
      const int32_t n_s = pass == 0 ? surv_n[k - 1] : n_k;
      const float *row = pass == 0 ? ll + (int64_t)(k - 1) * ll_stride : NULL;
      for (int32_t i = 0; i < n_s; i++) {
        int32_t p = st_s[i];
        int64_t a0 = pass == 0 ? g->first[p] : g->first[p] + g->n_emit[p];
        int64_t a1 = pass == 0 ? g->first[p] + g->n_emit[p] : g->first[p + 1];
        for (int64_t a = a0; a < a1; a++) {
          float c = pass == 0 ? (co_s[i] + g->weight[a]) - row[g->ilabel[a] - 1] : co_s[i] + g->weight[a];
          if (!keep(&kp, c)) continue;
          int32_t j = sorted_find(st_k, n_k, g->dst[a]);
          if (j < 0) { rc = O_INVALID; break; }   /* a kept candidate must have a kept dst */
          float s = c - co_k[j];
          if (!(s <= lattice_beam)) continue;
          LArc e = {(int32_t)a, i, j, s};
          buf[nb++] = e;
        }
      }
    }
    if (rc == O_OK) {
      qsort(buf, (size_t)nb, sizeof(LArc), cmp_larc);
      for (int64_t m = 0; m < nb; m++, out++) {
        if (out >= cap) continue;
        l_arc[out] = buf[m].arc; l_src[out] = buf[m].src; l_dst[out] = buf[m].dst;
        l_slack[out] = buf[m].slack;
      }
      seg_n[k] = (int32_t)nb;
    }
    free(buf);
  }
  free(off);
  *n_total = out;
  if (rc == O_OK && out > cap) rc = O_CAPACITY;
  return rc;
}

/* End of utterance ("moved to the host and used to generate the final lattice at the end
 * of utterance"; reading R14).  gamma(j) = the slack of the best complete path through token j:
 *   last layer T: gamma(j) = (cost_j + F(q_j)) - best   (reached_final; +inf for non-final q_j)
 *                 gamma(j) = cost_j - best               (no final survivor, R10)
 *   else          gamma(i) = min over lattice arcs a leaving i of  s_a + gamma(dst(a)),
 * emitting arcs into layer k+1 first, then the epsilon arcs inside layer k to a fixed point
 * (Bellman-Ford; epsilon arcs of a layer may form positive cycles).  An arc's path slack is
 * s_a + gamma(dst(a)); the final lattice keeps the arcs with path slack <= lattice_beam.
 * In: the segments of oracle_lattice (seg_n, l_arc, l_src, l_dst, l_slack), the layers.
 * Out: gamma[sum surv_n] per token, pslack[n arcs] per arc, *best. */
int oracle_lattice_finalize(void *gp, int32_t T, const int32_t *surv_n, const int32_t *surv_state,
                            const float *surv_cost, const int32_t *seg_n, const int32_t *l_arc,
                            const int32_t *l_src, const int32_t *l_dst, const float *l_slack,
                            float *gamma, float *pslack, float *best_out, int32_t *reached_out) {
  const OGraph *g = (const OGraph *)gp;
  if (!g || T < 0 || !surv_n || !seg_n || !gamma || !pslack) return O_INVALID;
  int64_t *off = (int64_t *)malloc(((size_t)T + 2) * 8), *soff = (int64_t *)malloc(((size_t)T + 2) * 8);
  if (!off || !soff) { free(off); free(soff); return O_OOM; }
  off[0] = soff[0] = 0;
  for (int32_t k = 0; k <= T; k++) { off[k + 1] = off[k] + surv_n[k]; soff[k + 1] = soff[k] + seg_n[k]; }
  /* best (R10) */
  const int64_t lt = off[T];
  float best = INFINITY;
  int reached = 0;
  for (int32_t j = 0; j < surv_n[T]; j++) {
    float F = g->final[surv_state[lt + j]];
    if (F < INFINITY) { float c = surv_cost[lt + j] + F; if (!reached || c < best) best = c; reached = 1; }
  }
  if (!reached)
    for (int32_t j = 0; j < surv_n[T]; j++) if (surv_cost[lt + j] < best) best = surv_cost[lt + j];
  for (int64_t m = 0; m < off[T + 1]; m++) gamma[m] = INFINITY;
  for (int32_t j = 0; j < surv_n[T]; j++) {
    float F = g->final[surv_state[lt + j]];
    if (reached) gamma[lt + j] = F < INFINITY ? (surv_cost[lt + j] + F) - best : INFINITY;
    else gamma[lt + j] = surv_cost[lt + j] - best;
  }
  for (int32_t k = T; k >= 0; k--) {
    if (k < T)   /* emitting arcs of segment k+1 leave layer k */
      for (int64_t m = soff[k + 1]; m < soff[k + 2]; m++) {
        if (g->ilabel[l_arc[m]] == 0) continue;
        float v = l_slack[m] + gamma[off[k + 1] + l_dst[m]];
        if (v < gamma[off[k] + l_src[m]]) gamma[off[k] + l_src[m]] = v;
      }
    int changed = 1;   /* epsilon arcs of segment k stay inside layer k */
    while (changed) {
      changed = 0;
      for (int64_t m = soff[k]; m < soff[k + 1]; m++) {
        if (g->ilabel[l_arc[m]] != 0) continue;
        float v = l_slack[m] + gamma[off[k] + l_dst[m]];
        if (v < gamma[off[k] + l_src[m]]) { gamma[off[k] + l_src[m]] = v; changed = 1; }
      }
    }
  }
  for (int32_t k = 0; k <= T; k++)
    for (int64_t m = soff[k]; m < soff[k + 1]; m++) pslack[m] = l_slack[m] + gamma[off[k] + l_dst[m]];
  if (best_out) *best_out = best;
  if (reached_out) *reached_out = reached;
  free(off); free(soff);
  return O_OK;
}

/* ---- multi-core driver for cpu_baseline: streams split over pthreads ---- */
typedef struct {
  void *g; const float *ll; int64_t ll_stride; int32_t T, P; float beam; int32_t max_active;
  int32_t B, n_thr, tid;
  float *cost; int32_t *reached; int32_t *rc; int64_t *emit_arcs;
  int32_t *arcs; int32_t arcs_cap; int32_t *n_arcs;
} BatchArg;

static void *batch_worker(void *p) {
  BatchArg *a = (BatchArg *)p;
  int64_t *fc = (int64_t *)malloc((size_t)(a->T > 0 ? a->T : 1) * 5 * 8);
  for (int32_t b = a->tid; b < a->B; b += a->n_thr) {
    memset(fc, 0, (size_t)(a->T > 0 ? a->T : 1) * 5 * 8);
    a->rc[b] = oracle_decode(a->g, a->ll + (int64_t)b * a->P, a->ll_stride, a->T, a->P, a->beam,
                             a->max_active, &a->cost[b], &a->reached[b],
                             a->arcs ? a->arcs + (int64_t)b * a->arcs_cap : NULL, a->arcs_cap,
                             a->n_arcs ? &a->n_arcs[b] : NULL, NULL, 0, NULL, NULL, fc, NULL, NULL,
                             NULL, NULL, 0, NULL);
    int64_t s = 0;
    for (int32_t t = 0; t < a->T; t++) s += fc[5 * t + 3] + fc[5 * t + 4];
    a->emit_arcs[b] = s;
  }
  free(fc);
  return NULL;
}

/* ll layout [T][B][P]; stream b row t at ll + (t*B + b)*P. */
int oracle_decode_batch(void *g, const float *ll, int32_t T, int32_t B, int32_t P, float beam,
                        int32_t max_active, int32_t n_threads, float *cost, int32_t *reached,
                        int32_t *rc, int64_t *arcs_count, int32_t *arcs, int32_t arcs_cap,
                        int32_t *n_arcs) {
  if (n_threads < 1) n_threads = 1;
  if (n_threads > B) n_threads = B > 0 ? B : 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)n_threads);
  BatchArg *args = (BatchArg *)malloc(sizeof(BatchArg) * (size_t)n_threads);
  if (!th || !args) { free(th); free(args); return O_OOM; }
  for (int32_t i = 0; i < n_threads; i++) {
    BatchArg a = {g, ll, (int64_t)B * P, T, P, beam, max_active, B, n_threads, i,
                  cost, reached, rc, arcs_count, arcs, arcs_cap, n_arcs};
    args[i] = a;
    pthread_create(&th[i], NULL, batch_worker, &args[i]);
  }
  for (int32_t i = 0; i < n_threads; i++) pthread_join(th[i], NULL);
  free(th); free(args);
  return O_OK;
}

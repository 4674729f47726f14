/*
 * wfst_gpu.h -- C ABI of the B200 one-best token-passing WFST decoder.
 *
 * What the library computes (PAPER.md arXiv 1910.10032, "P:n" = PAPER.md
 * line n; "S:n" = SPEC.md line n): frame-synchronous token-passing Viterbi
 * beam search over a decode WFST for many concurrent audio streams (P:49,
 * Fig. 1).  Per frame and stream:
 *   (a) emitting-arc expansion, cost' = (cost + w) - L[t][pdf]
 *   (b) beam + exact max-active cutoff against the stream's best
 *   (c) iterated epsilon closure under that fixed cutoff
 *   (d) one representative token per state, traceback records
 * and, at the end of a stream, the final-cost argmin and traceback.
 * The exact rules (R1-R12) are in DESIGN.md §3; a CPU oracle in oracle/
 * implements the same rules independently and the tests compare the two.
 *
 * Conventions
 *   - Graph arcs are (src, dst, ilabel, olabel, weight).  ilabel 0 = epsilon
 *     (non-emitting); an emitting arc reads log-likelihood column pdf =
 *     ilabel - 1 ("arcs with non-null labels"), or column = ilabel with
 *     opts.ll_columns = 1 (SPEC's layout, column 0 unused).  The start state is
 *     given explicitly (text files: state 0).  final cost +INF =
 *     non-final.  Weights and costs are fp32, tropical (min, +) semiring.
 *   - Canonical arc ids: arcs stably ordered by (src, emitting first) in
 *     input order.  Paths are reported as canonical arc ids.
 *   - Log-likelihoods are fp32, row-major [T][B][P] on the DEVICE (or host
 *     for wfst_decode_frames_host); acoustic scale 1 (caller pre-scales).
 *   - Every function returns wfst_status; WFST_OK = 0.  On error, a
 *     thread-local message is available from wfst_last_error().
 *   - Device work is asynchronous on the caller's CUDA stream (void* =
 *     cudaStream_t, NULL = legacy default stream).  A decoder's calls are
 *     ordered among themselves even across CUDA streams: a call on stream s
 *     first makes s wait (cudaStreamWaitEvent) for the decoder's previous
 *     work, which shares its scratch, work queue and lane states.  Calls that
 *     return results (best / partial paths, sync, stats) run on the stream of
 *     the decoder's last call and wait for THIS decoder's work only (an event),
 *     never for the whole device, so decoders on other streams or devices keep
 *     running.  Device-side failures (capacity, no survivor) are sticky per
 *     stream and surface at wfst_decoder_sync / wfst_get_best_path /
 *     wfst_decoder_status.
 * Ownership
 *   - A graph is immutable after creation, bound to one device, safe for
 *     concurrent reads, and must outlive every decoder created on it.
 *   - A decoder owns all of its device buffers; one host thread at a time.
 *   - Device input pointers are BORROWED and stream-ordered: they must stay
 *     valid until the work enqueued on cuda_stream completes.
 *   - Output buffers are caller-owned host memory unless stated otherwise.
 */
#ifndef WFST_GPU_H
#define WFST_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  WFST_OK = 0,
  WFST_ERR_INVALID_ARG = 1,  /* bad pointer/size/range; also output cap too small          */
  WFST_ERR_PARSE = 2,        /* text graph: malformed line (message has the line number)     */
  WFST_ERR_GRAPH_INVALID = 3,/* dangling state id, bad start, NaN weight, too many arcs      */
  WFST_ERR_EPS_CYCLE = 4,    /* epsilon cycle of total weight <= 0              */
  WFST_ERR_PDF_RANGE = 5,    /* P <= max pdf id of the graph                  */
  WFST_ERR_CAPACITY = 6,     /* a stream outgrew its token table / record arena (never silent)*/
  WFST_ERR_NO_SURVIVOR = 7,  /* a frame produced no candidate token                  */
  WFST_ERR_CUDA = 8,         /* CUDA runtime error                                           */
  WFST_ERR_OOM = 9,          /* device or host allocation failed                             */
  WFST_ERR_STATE = 10        /* stream used before wfst_decoder_reset                        */
} wfst_status;

typedef struct wfst_graph_s* wfst_graph_t;
typedef struct wfst_decoder_s* wfst_decoder_t;

typedef struct {
  int32_t n_states;        /* |Q|                                             */
  int32_t start;
  int64_t n_arcs;          /* |E|                                             */
  int64_t n_emitting;      /* |E_E|                                           */
  int32_t max_pdf;         /* largest pdf id (ilabel-1) of any emitting arc  */
  int32_t device;
  int64_t device_bytes;    /* bytes of the device layout actually allocated  */
  int64_t eq1_bytes;       /* Eq. 1: 12|Q| + 8|E| + 4|E_E|           */
} wfst_graph_info_t;

/* Decoder tuning; zero fields mean "default".  See DESIGN.md §5. */
typedef struct {
  int32_t table_slots;       /* on-chip token table slots per CTA (default: all free shared memory) */
  int32_t overflow_slots;    /* global overflow table slots per CTA (default max(C, 32768, 4*alpha)) */
  int64_t records_per_stream;/* traceback records per stream (default sized from max_frames)      */
  int32_t max_frames;        /* layers kept per stream (default 4096; a ring with opts.reclaim)   */
  int32_t threads;           /* CTA size of the frame kernel (256/512/1024; default 1024 with one
                                CTA per SM, else 256); the lattice and histogram modes use 1024   */
  int32_t frames_per_item;   /* frames a CTA runs on one stream before re-queueing (default 16)  */
  int32_t max_ctas;          /* cap on persistent CTAs (default: #SMs x ctas_per_sm)              */
  int32_t debug_costs;       /* 1: also keep each survivor's cost (wfst_debug_layer)              */
  int32_t ctas_per_sm;       /* resident lanes per SM (1-4; default 1); the on-chip table is sized
                                from the SM's shared memory divided by this                       */
  int32_t lattice;           /* 1: build lattice segments every frame (row f1)    */
  float lattice_beam;        /* lattice-beam (P:146 uses 8) when lattice = 1; may be 0 or +INF     */
  int64_t lattice_arcs_per_stream; /* segment arena per stream (default 2 x records_per_stream)   */
  int32_t max_active_mode;   /* 0: exact alpha-th smallest (R6, default); 1: the paper's histogram
                                adaptive beam (row f4, R16: 1024 bins of beam/1024 from the best,
                                keep below the bin where the count reaches alpha)                */
  int32_t reclaim;           /* 1: traceback GC (row f2): every wfst_get_partial_paths call releases
                                the records and layers below the new settle point, so an unbounded
                                stream needs only records_per_stream / max_frames for the frames
                                since its paths last converged; wfst_get_best_path then returns the
                                arcs AFTER the settled prefix.  Exclusive with lattice.  Record
                                numbers are int32: an utterance may write up to 2^31 records
                                (~650k frames at 3.3k survivors), beyond that CAPACITY.            */
  int32_t insert_order;      /* order in which a frame's candidates enter the token table (results
                                never depend on it, R7/R9): 0 auto (default: bin order after a
                                frame where max-active bound), 1 arrival order, 2 always bin order */
  int32_t bin_capacity;      /* bin-ordered frames: candidates buffered per coarse cost bin and CTA
                                (default 8192; a full bin inserts directly)                       */
  int32_t ll_columns;        /* which log-likelihood column an emitting arc reads (reading R2):
                                0 (default): pdf columns, column = ilabel - 1, requires P > max_pdf
                                  (Kaldi-style transition -> pdf + 1 labels);
                                1: ilabel columns: column = ilabel,
                                  column 0 unused, requires P >= 1 + max ilabel = max_pdf + 2.
                                The two layouts of the same scores differ by one leading column;
                                a P that fits only layout 0 is rejected under layout 1 (PDF_RANGE)
                                and the caller chooses the layout explicitly, so a SPEC-shaped
                                matrix is never read one column off by default-guessing.        */
  int32_t gc_frames;         /* traceback GC: > 0 = every decode call runs its
                                frames in launches of at most gc_frames frames, each followed by
                                a compaction that drops the records no current survivor's
                                traceback reaches; a stream then holds only its live traceback tree
                                plus gc_frames frames of new records, however long the utterance,
                                and records_per_stream defaults to that (gc_frames + 64 frames at
                                the max-active bound).  Results are unchanged (wfst_debug_layer of
                                an older layer lists only its live tokens).  Exclusive with
                                lattice.  0 (default): off.                                     */
} wfst_decoder_opts_t;

typedef struct {
  int64_t frames;            /* stream-frames decoded                                            */
  int64_t emit_arcs;         /* emitting arcs expanded (sum of survivors' emitting out-degree)   */
  int64_t eps_arcs;          /* epsilon out-degree summed over survivors (algorithmic count)      */
  int64_t eps_relax;         /* epsilon relaxations actually performed                            */
  int64_t candidates;        /* distinct states inserted into token tables                        */
  int64_t survivors;         /* tokens kept (sum over frames)                                     */
  int64_t overflow_inserts;  /* distinct states that went to the global overflow table            */
  int64_t alpha_frames;      /* frames where max-active tightened the cutoff                      */
  int64_t device_bytes;      /* decoder device allocation                                         */
  int64_t records_used_max;  /* max traceback records used by any stream                          */
  int64_t phase_cycles[12];  /* SM cycles summed over lanes (instrumentation): 0 row prefetch issue,
                                1 cutoff, 2 epsilon, 3 expansion (warp tokens), 4 expansion (hub
                                tokens), 5 frame overhead, 6 drain, 7 map build, 8 placement,
                                9 epsilon back-pointers, 10 table reset, 11 row wait            */
  int64_t select_entries;    /* token-table entries read by the max-active selection, summed over
                                passes (SURVEY §8.5's passes x n_uniq term of the byte model)     */
  int64_t phase_cycles_alpha[12]; /* phase_cycles restricted to frames where max-active bound      */
  int64_t records_per_stream;/* traceback record capacity per stream (the history arena)          */
  int64_t record_bytes;      /* device bytes of the history arena (records, + costs if kept); the
                                rest of device_bytes is decoder state proper (frontiers, lane
                                state, per-CTA scratch): the counterpart of P:117-126's Eq. 2,
                                whose decoder keeps no traceback on the device        */
} wfst_stats_t;

/* ---- graph (row a0 of SURVEY §8) ------------------------------------------------ */

/* Load a text graph ("src dst ilabel olabel weight" / "state final_weight" lines, any order,
 * state 0 = start).  Validates ids, NaN, epsilon cycles of weight <= 0.  device: CUDA
 * ordinal the graph is uploaded to.  *out receives a new graph (free with wfst_graph_free). */
wfst_status wfst_load_graph(const char* path, int device, wfst_graph_t* out);

/* Same from host arrays of n_arcs entries (input order); final_cost has n_states entries
 * (+INF = non-final).  Arrays are only read during the call. */
wfst_status wfst_graph_from_arrays(int32_t n_states, int32_t start, int64_t n_arcs,
                                   const int32_t* src, const int32_t* dst, const int32_t* ilabel,
                                   const int32_t* olabel, const float* weight,
                                   const float* final_cost, int device, wfst_graph_t* out);
wfst_status wfst_graph_info(wfst_graph_t g, wfst_graph_info_t* info);
/* canonical arc id -> input arc index (n_arcs int64 entries, host). */
wfst_status wfst_graph_canonical_perm(wfst_graph_t g, int64_t* perm, int64_t cap);
/* A copy of graph g on CUDA device `device` (row e: one replica per GPU), copied device to device
 * (over NVLink/NVSwitch when the devices are peers).  Free it with wfst_graph_free. */
wfst_status wfst_graph_replicate(wfst_graph_t g, int device, wfst_graph_t* out);
void wfst_graph_free(wfst_graph_t g);

/* Eq. 1 and Eq. 2 of the paper, host arithmetic only (no device needed). */
int64_t wfst_eq1_bytes(int64_t n_states, int64_t n_arcs, int64_t n_emitting);
int64_t wfst_eq2_bytes(int64_t max_active, int64_t n_channels, int64_t n_lanes);

/* ---- decoder (rows a1-a7, b) ----------------------------------------------------------------- */

/* n_streams lanes ("lanes ... the set of utterances or streams being actively decoded").
 * beam > 0 (may be +INF); max_active <= 0 means unbounded, else alpha.  opts may be
 * NULL.  Allocates on the graph's device. */
wfst_status wfst_decoder_create(wfst_graph_t g, int32_t n_streams, float beam, int32_t max_active,
                                wfst_decoder_t* out);
wfst_status wfst_decoder_create_ex(wfst_graph_t g, int32_t n_streams, float beam,
                                   int32_t max_active, const wfst_decoder_opts_t* opts,
                                   wfst_decoder_t* out);
void wfst_decoder_destroy(wfst_decoder_t d);

/* Start new utterances on the given lanes (host array of n lane ids; NULL = all lanes): the start
 * token plus its epsilon closure with cutoff = beam (reading R3).  Asynchronous on cuda_stream. */
wfst_status wfst_decoder_reset(wfst_decoder_t d, const int32_t* streams, int32_t n,
                               void* cuda_stream);

/* Advance T frames on B lanes with ONE kernel launch.  d_loglikes: device fp32 [T][B][P]
 * row-major (row of batch entry b at frame t = d_loglikes + (t*B + b)*P).  streams: host array of B
 * lane ids (NULL = lanes 0..B-1; ids must be distinct).  T = 0 is a no-op.  Validates arguments
 * synchronously (PDF_RANGE if P <= max_pdf, STATE if a lane was never reset); otherwise async. */
wfst_status wfst_decode_frames(wfst_decoder_t d, const float* d_loglikes, int32_t T, int32_t B,
                               int32_t P, const int32_t* streams, void* cuda_stream);

/* Same with HOST log-likelihoods (pinned or pageable): copied to the device in frame chunks on an
 * internal stream, overlapped with decoding of the previous chunk.  Returns after the last chunk
 * is enqueued; h_loglikes must stay valid until wfst_decoder_sync. */
wfst_status wfst_decode_frames_host(wfst_decoder_t d, const float* h_loglikes, int32_t T,
                                    int32_t B, int32_t P, const int32_t* streams,
                                    int32_t chunk_frames, void* cuda_stream);

/* Wait for the decoder's work (its event; not the device); returns the first sticky per-stream
 * error, if any. */
wfst_status wfst_decoder_sync(wfst_decoder_t d);
/* Sticky status of one lane (after sync). */
wfst_status wfst_decoder_status(wfst_decoder_t d, int32_t stream);

/* One-best result of a lane (reading R10/R11): final-cost argmin over the current survivors
 * (fallback: best cost, *reached_final = 0), then traceback.  olabels: non-zero output labels
 * in order; arcs: canonical arc ids of the path (nullable).  A too-small cap returns
 * INVALID_ARG with the needed size in *n_olabels / *n_arcs.  The traceback kernel runs on the
 * stream of the decoder's last call, after its work; the call waits for that stream only. */
wfst_status wfst_get_best_path(wfst_decoder_t d, int32_t stream, int32_t* olabels,
                               int32_t olabels_cap, int32_t* n_olabels, int32_t* arcs,
                               int32_t arcs_cap, int32_t* n_arcs, float* cost,
                               int32_t* reached_final);

/* Batched form: n lanes in one launch.  Per lane i: cost[i], reached_final[i], n_arcs[i], and
 * arcs[i*arcs_cap ...] (canonical ids; nullable), olabels[i*arcs_cap ...] with n_olabels[i]
 * (nullable).  All outputs are host arrays.  Returns the first error among the lanes; n_olabels[i]
 * counts every olabel of the path even when the arcs were truncated to arcs_cap. */
wfst_status wfst_get_best_paths(wfst_decoder_t d, const int32_t* streams, int32_t n, float* cost,
                                int32_t* reached_final, int32_t* arcs, int32_t* olabels,
                                int32_t arcs_cap, int32_t* n_arcs, int32_t* n_olabels);
/* Same, plus status[i] (host, n entries; nullable): each lane's own result status (OK, its sticky
 * decode error, STATE if never reset, INVALID_ARG if its path exceeded arcs_cap). */
wfst_status wfst_get_best_paths_ex(wfst_decoder_t d, const int32_t* streams, int32_t n, float* cost,
                                   int32_t* reached_final, int32_t* arcs, int32_t* olabels,
                                   int32_t arcs_cap, int32_t* n_arcs, int32_t* n_olabels,
                                   int32_t* status);

wfst_status wfst_decoder_stats(wfst_decoder_t d, wfst_stats_t* s);
wfst_status wfst_decoder_reset_stats(wfst_decoder_t d);

/* Per-frame record of a lane's current utterance (frames < opts.max_frames):
 * fstats[t*3+{0,1,2}] = best candidate cost, beam cutoff, max-active cutoff k_alpha (+INF if
 * unused); fcounts[t*5+{0..4}] = distinct candidates, in-beam candidates (-1 when the cutoff
 * did not need the exact count: max-active provably bound or could not bind), survivors,
 * emitting arcs expanded, epsilon out-degree of survivors.  Either pointer may be NULL. */
wfst_status wfst_decoder_frame_stats(wfst_decoder_t d, int32_t stream, float* fstats,
                                     int64_t* fcounts, int32_t cap_frames, int32_t* n_frames);

/* Survivors of layer k (k = 0: after reset; k = t+1: after frame t) of a lane: state, canonical
 * arc (-1 = start token), cost (only if opts.debug_costs, else NaN).  Order unspecified. */
wfst_status wfst_debug_layer(wfst_decoder_t d, int32_t stream, int32_t layer, int32_t* states,
                             int32_t* arcs, float* costs, int32_t cap, int32_t* n);

/* ---- settled partial results (row f2 of SURVEY §8, NEXT; "return intermediate results
 * during online decoding") --------------------------------------------------------------------
 * The settled prefix of a stream is the longest arc sequence shared by the tracebacks of ALL
 * current survivors, cut after its last emitting arc (reading R15): no later frame can change
 * it.  Each call returns, per stream, only the arcs settled SINCE the previous call (or the
 * reset), in order, with their non-zero olabels; concatenating a stream's outputs gives its
 * settled prefix, which is always a prefix of the final wfst_get_best_path result.
 *   arcs/olabels: host [n][cap] (nullable); n_arcs[i] / n_olabels[i] (nullable): counts;
 *   settled_frames[i]: frames (= layer) covered by the settled prefix so far.
 * Runs on the stream of the decoder's last call after its work (waits for that stream only).
 * A stream whose new arcs exceed cap returns INVALID_ARG with the needed count in n_arcs[i] and
 * keeps its settle point (call again with a larger cap).  Layers of more than 16384 tokens return
 * CAPACITY.  The return value is the first error among the streams. */
wfst_status wfst_get_partial_paths(wfst_decoder_t d, const int32_t* streams, int32_t n, int32_t* arcs,
                                   int32_t* olabels, int32_t cap, int32_t* n_arcs, int32_t* n_olabels,
                                   int32_t* settled_frames);
/* Same, plus status[i] (host, n entries; nullable): each stream's own status, so one stream's
 * error (or cap overflow) does not hide the others' results: a stream with status OK has
 * advanced its settle point and its arcs are valid whatever the return value. */
wfst_status wfst_get_partial_paths_ex(wfst_decoder_t d, const int32_t* streams, int32_t n, int32_t* arcs,
                                      int32_t* olabels, int32_t cap, int32_t* n_arcs, int32_t* n_olabels,
                                      int32_t* settled_frames, int32_t* status);

/* Same results, packed: stream i's new arcs are arcs[offsets[i] .. offsets[i] + min(n_arcs[i],
 * cap)) and its olabels olabels[offsets[i] .. + n_olabels[i]) (the streams' ranges do not
 * overlap; their order in the buffers is unspecified).  arcs/olabels: host, total_cap entries
 * each (nullable); total_cap must be >= n * cap (INVALID_ARG before any work otherwise), cap is
 * the per-stream limit as above; *total: entries used.  Only the used entries are copied and
 * written, so an online caller pays for the arcs that settled, not for n * cap (a fresh n * cap
 * host buffer is touched only where arcs land).  Other arguments as wfst_get_partial_paths_ex. */
wfst_status wfst_get_partial_paths_packed(wfst_decoder_t d, const int32_t* streams, int32_t n, int32_t* arcs,
                                          int32_t* olabels, int64_t total_cap, int32_t cap, int64_t* offsets,
                                          int64_t* total, int32_t* n_arcs, int32_t* n_olabels,
                                          int32_t* settled_frames, int32_t* status);

/* ---- lattice (row f1 of SURVEY §8, NEXT) ----------------
 * With opts.lattice = 1 every reset and decode call also builds, per stream and frame, the lattice
 * segment of that frame (one extra launch after the frame kernel, same CUDA stream): every arc
 * that leaves a representative token (P:139 soft pruning), passes the frame's cutoff and whose
 * extra cost s = c - cost(representative of dst) is <= lattice_beam, listed in CSR order by
 * destination token, arc id ascending inside a group ("listing them in the CSR format",
 * "computing extra costs").  Readings R13-R14 of DESIGN.md.
 *
 * wfst_get_lattice runs the end-of-utterance backward sweep on the device ("used to generate
 * the final lattice at the end of utterance"): gamma(token) = slack of the best complete path
 * through it (R10 best: final states if any survive), pslack(arc) = s + gamma(dst).  The final
 * lattice is the set of arcs with pslack <= lattice_beam.  The sweep and the device->host copies
 * run on the decoder's copy stream after the lane's last lattice launch: the compute stream is
 * NOT synchronised, so other lanes keep decoding (the lane itself must not be decoded further
 * until the call returns).
 * Outputs (host, caller-owned; layer k = 0..T, T = frames decoded):
 *   seg_n[k]                  arcs of segment k (layers_cap entries; *n_layers = T + 1)
 *   arc/src/dst/slack/pslack  concatenated segments (arcs_cap entries; *n_arcs total): canonical
 *                             arc id; src = token index in layer k-1 (emitting arc) or layer k
 *                             (epsilon arc); dst = token index in layer k; token indices are the
 *                             positions of wfst_debug_layer's output.  pslack nullable.
 *   gamma                     per token, layers concatenated (gamma_cap; *n_tokens); nullable
 *   best, reached_final       the best complete cost and whether it ends in a final state (R10)
 * Errors: INVALID_ARG (lattice off, bad stream, a cap too small: the sizes are still written),
 * STATE (stream not reset), CAPACITY (the segment arena or records overflowed), or the lane's
 * sticky decode error. */
wfst_status wfst_get_lattice(wfst_decoder_t d, int32_t stream, int32_t* seg_n, int32_t layers_cap,
                             int32_t* n_layers, int32_t* arc, int32_t* src, int32_t* dst, float* slack,
                             float* pslack, int64_t arcs_cap, int64_t* n_arcs, float* gamma,
                             int64_t gamma_cap, int64_t* n_tokens, float* best, int32_t* reached_final);

/* ---- synthetic inputs (not part of the method) ------------------------------ */

/* Fill d_out [T][B][P] with the counter-hash log-likelihoods of paper_1910_10032_b200/inputs.py:
 * batch entry b is global stream stream_ids[b] (device array), frame t is global frame t0+t;
 * d_planted: device int32 [T][B] pdf boosted by `boost` (NULL = none). */
wfst_status wfst_synth_loglikes(float* d_out, int32_t T, int32_t B, int32_t P,
                                const int32_t* d_stream_ids, int32_t t0, uint64_t seed,
                                const int32_t* d_planted, float sigma, float boost,
                                void* cuda_stream);

const char* wfst_last_error(void);
const char* wfst_status_string(wfst_status s);
int32_t wfst_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WFST_GPU_H */

// Graph ingestion for the decoder: text parsing, validation,
// canonical arc order and the device CSR layout (row a0).
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "wfst_internal.h"

namespace wfst {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
wfst_status fail(wfst_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
wfst_status cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? WFST_ERR_OOM : WFST_ERR_CUDA;
}

// Reject epsilon cycles of total weight <= 0.  Kahn's algorithm peels the acyclic part;
// on what remains, Bellman-Ford (double) detects negative cycles and a cycle search on the
// "tight" arcs (reduced weight ~ 0) detects zero-weight cycles.
static bool eps_has_nonpositive_cycle(int32_t Q, const std::vector<int64_t>& first,
                                      const std::vector<int32_t>& n_emit, const int32_t* cdst,
                                      const float* cw) {
  std::vector<int32_t> indeg(Q, 0);
  int64_t n_eps = 0;
  for (int32_t q = 0; q < Q; q++)
    for (int64_t a = first[q] + n_emit[q]; a < first[q + 1]; a++) {
      indeg[cdst[a]]++;
      n_eps++;
    }
  if (n_eps == 0) return false;
  std::vector<int32_t> stack;
  std::vector<char> removed(Q, 0);
  for (int32_t q = 0; q < Q; q++)
    if (indeg[q] == 0) stack.push_back(q);
  while (!stack.empty()) {
    int32_t q = stack.back();
    stack.pop_back();
    removed[q] = 1;
    for (int64_t a = first[q] + n_emit[q]; a < first[q + 1]; a++)
      if (--indeg[cdst[a]] == 0) stack.push_back(cdst[a]);
  }
  std::vector<int32_t> rest;
  for (int32_t q = 0; q < Q; q++)
    if (!removed[q]) rest.push_back(q);
  if (rest.empty()) return false;  // epsilon subgraph is acyclic
  // Bellman-Ford from a virtual source (all distances 0) on the remaining subgraph.
  std::vector<double> d(Q, 0.0);
  bool changed = true;
  for (size_t it = 0; it <= rest.size() && changed; it++) {
    changed = false;
    for (int32_t q : rest)
      for (int64_t a = first[q] + n_emit[q]; a < first[q + 1]; a++) {
        int32_t v = cdst[a];
        if (removed[v]) continue;
        double nd = d[q] + (double)cw[a];
        if (nd < d[v] - 1e-12 * (1.0 + std::fabs(d[v]))) {
          d[v] = nd;
          changed = true;
        }
      }
    if (changed && it == rest.size()) return true;  // negative cycle
  }
  // zero-weight cycle: cycle among arcs with reduced weight ~ 0
  std::vector<int32_t> tdeg(Q, 0);
  auto tight = [&](int32_t q, int64_t a) {
    int32_t v = cdst[a];
    if (removed[v]) return false;
    double r = d[q] + (double)cw[a] - d[v];
    return std::fabs(r) <= 1e-9 * (1.0 + std::fabs(d[q]) + std::fabs(d[v]));
  };
  for (int32_t q : rest)
    for (int64_t a = first[q] + n_emit[q]; a < first[q + 1]; a++)
      if (tight(q, a)) tdeg[cdst[a]]++;
  std::vector<char> gone(Q, 0);
  for (int32_t q : rest)
    if (tdeg[q] == 0) stack.push_back(q);
  size_t n_gone = 0;
  while (!stack.empty()) {
    int32_t q = stack.back();
    stack.pop_back();
    gone[q] = 1;
    n_gone++;
    for (int64_t a = first[q] + n_emit[q]; a < first[q + 1]; a++)
      if (tight(q, a) && --tdeg[cdst[a]] == 0) stack.push_back(cdst[a]);
  }
  return n_gone < rest.size();
}

wfst_status build_graph(int32_t Q, int32_t start, int64_t E, const int32_t* src, const int32_t* dst,
                        const int32_t* ilabel, const int32_t* olabel, const float* weight,
                        const float* final_cost, int device, wfst_graph_t* out) {
  if (!out) return fail(WFST_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (Q <= 0) return fail(WFST_ERR_GRAPH_INVALID, "graph has no states");
  if (start < 0 || start >= Q) return fail(WFST_ERR_GRAPH_INVALID, "start state out of range");
  if (E < 0 || E > kMaxArcs) return fail(WFST_ERR_GRAPH_INVALID, "arc count out of range (max 2^31-1)");
  if (E > 0 && (!src || !dst || !ilabel || !olabel || !weight))
    return fail(WFST_ERR_INVALID_ARG, "NULL arc array");
  if (!final_cost) return fail(WFST_ERR_INVALID_ARG, "NULL final_cost");
  std::vector<int32_t> n_all(Q, 0), n_emit(Q, 0);
  int32_t max_pdf = -1;
  int64_t EE = 0;
  for (int64_t i = 0; i < E; i++) {
    if (src[i] < 0 || src[i] >= Q || dst[i] < 0 || dst[i] >= Q)
      return fail(WFST_ERR_GRAPH_INVALID, "arc " + std::to_string(i) + ": dangling state id");
    if (ilabel[i] < 0) return fail(WFST_ERR_GRAPH_INVALID, "arc " + std::to_string(i) + ": negative ilabel");
    if (olabel[i] < 0) return fail(WFST_ERR_GRAPH_INVALID, "arc " + std::to_string(i) + ": negative olabel");
    if (std::isnan(weight[i]) || std::isinf(weight[i]))
      return fail(WFST_ERR_GRAPH_INVALID, "arc " + std::to_string(i) + ": non-finite weight");
    n_all[src[i]]++;
    if (ilabel[i] != 0) {
      n_emit[src[i]]++;
      EE++;
      if (ilabel[i] - 1 > max_pdf) max_pdf = ilabel[i] - 1;
    }
  }
  for (int32_t q = 0; q < Q; q++)
    if (std::isnan(final_cost[q]) || final_cost[q] == -INFINITY)
      return fail(WFST_ERR_GRAPH_INVALID, "state " + std::to_string(q) + ": bad final cost");
  // canonical order: stable bucket by (src, emitting first)
  std::vector<int64_t> first(Q + 1, 0);
  for (int32_t q = 0; q < Q; q++) first[q + 1] = first[q] + n_all[q];
  std::vector<int64_t> ce(Q), cn(Q);
  for (int32_t q = 0; q < Q; q++) {
    ce[q] = first[q];
    cn[q] = first[q] + n_emit[q];
  }
  auto* g = new wfst_graph_s();
  g->device = device;
  g->Q = Q;
  g->start = start;
  g->E = E;
  g->EE = EE;
  g->max_pdf = max_pdf;
  g->perm.resize(E);
  g->h_dst.resize(E);
  g->h_olabel.resize(E);
  std::vector<float> cw(E);
  std::vector<int4> arcs(E);
  for (int64_t i = 0; i < E; i++) {
    int32_t s = src[i];
    int64_t k = ilabel[i] != 0 ? ce[s]++ : cn[s]++;
    g->perm[k] = i;
    g->h_dst[k] = dst[i];
    g->h_olabel[k] = olabel[i];
    float w = weight[i] + 0.0f;  // canonical +0
    cw[k] = w;
    int4 r;
    r.x = dst[i];
    memcpy(&r.y, &w, 4);
    r.z = ilabel[i] - 1;  // -1 for epsilon
    r.w = s;              // source state (| destination-has-epsilon flag, below)
    arcs[k] = r;
  }
  // bit 31 of the source field: "the destination state has epsilon arcs" (lets the kernel
  // build epsilon worklists without gathering state records)
  for (int64_t k = 0; k < E; k++) {
    int32_t d = arcs[k].x;
    if (n_all[d] > n_emit[d]) arcs[k].w |= (int32_t)0x80000000;
  }
  if (eps_has_nonpositive_cycle(Q, first, n_emit, g->h_dst.data(), cw.data())) {
    delete g;
    return fail(WFST_ERR_EPS_CYCLE, "epsilon cycle with total weight <= 0");
  }
  std::vector<int4> st(Q);
  for (int32_t q = 0; q < Q; q++) {
    int4 r;
    r.x = (int32_t)first[q];
    r.y = (int32_t)(first[q] + n_emit[q]);
    r.z = (int32_t)first[q + 1];
    float f = final_cost[q] + 0.0f;
    memcpy(&r.w, &f, 4);
    st[q] = r;
  }
  int prev_dev = 0;
  cudaGetDevice(&prev_dev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete g;
    return cuda_fail(e, "cudaSetDevice");
  }
  size_t bs = sizeof(int4) * (size_t)Q, ba = sizeof(int4) * (size_t)(E > 0 ? E : 1);
  size_t bo = sizeof(int32_t) * (size_t)(E > 0 ? E : 1);
  e = cudaMalloc(&g->d_state, bs);
  if (e == cudaSuccess) e = cudaMalloc(&g->d_arcs, ba);
  if (e == cudaSuccess) e = cudaMalloc(&g->d_olabel, bo);
  if (e == cudaSuccess && E > 0) e = cudaMemcpy(g->d_olabel, g->h_olabel.data(), bo, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(g->d_state, st.data(), bs, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && E > 0) e = cudaMemcpy(g->d_arcs, arcs.data(), sizeof(int4) * E, cudaMemcpyHostToDevice);
  cudaSetDevice(prev_dev);
  if (e != cudaSuccess) {
    cudaFree(g->d_state);
    cudaFree(g->d_arcs);
    cudaFree(g->d_olabel);
    delete g;
    return cuda_fail(e, "graph upload");
  }
  g->device_bytes = (int64_t)(bs + ba + bo);
  *out = g;
  return WFST_OK;
}

}  // namespace wfst

using namespace wfst;

extern "C" {

wfst_status wfst_graph_from_arrays(int32_t n_states, int32_t start, int64_t n_arcs,
                                   const int32_t* src, const int32_t* dst, const int32_t* ilabel,
                                   const int32_t* olabel, const float* weight,
                                   const float* final_cost, int device, wfst_graph_t* out) {
  return build_graph(n_states, start, n_arcs, src, dst, ilabel, olabel, weight, final_cost, device, out);
}

wfst_status wfst_load_graph(const char* path, int device, wfst_graph_t* out) {
  if (!path || !out) return fail(WFST_ERR_INVALID_ARG, "NULL argument");
  FILE* f = fopen(path, "r");
  if (!f) return fail(WFST_ERR_INVALID_ARG, std::string("cannot open ") + path);
  std::vector<int32_t> src, dst, il, ol;
  std::vector<float> w;
  std::vector<std::pair<int64_t, float>> fin;
  int64_t n = 0;
  char buf[4096];
  int64_t line = 0;
  wfst_status rc = WFST_OK;
  while (fgets(buf, sizeof buf, f)) {
    line++;
    char* tok[6];
    int nt = 0;
    char* save = nullptr;
    for (char* p = strtok_r(buf, " \t\r\n", &save); p; p = strtok_r(nullptr, " \t\r\n", &save)) {
      if (nt == 6) break;
      tok[nt++] = p;
    }
    if (nt == 0) continue;
    auto parse_id = [&](const char* s, int64_t* v) {
      char* e = nullptr;
      errno = 0;
      long long x = strtoll(s, &e, 10);
      if (errno || *e || x < 0 || x > INT32_MAX - 1) return false;
      *v = x;
      return true;
    };
    auto parse_w = [&](const char* s, float* v) {
      char* e = nullptr;
      errno = 0;
      float x = strtof(s, &e);
      if (*e || std::isnan(x)) return false;
      *v = x;
      return true;
    };
    if (nt == 5) {
      int64_t a, b, c, d;
      float x;
      if (!parse_id(tok[0], &a) || !parse_id(tok[1], &b) || !parse_id(tok[2], &c) ||
          !parse_id(tok[3], &d) || !parse_w(tok[4], &x) || std::isinf(x)) {
        rc = fail(WFST_ERR_PARSE, "line " + std::to_string(line) + ": malformed arc");
        break;
      }
      src.push_back((int32_t)a);
      dst.push_back((int32_t)b);
      il.push_back((int32_t)c);
      ol.push_back((int32_t)d);
      w.push_back(x);
      n = std::max(n, std::max(a, b) + 1);
    } else if (nt == 2) {
      int64_t a;
      float x;
      if (!parse_id(tok[0], &a) || !parse_w(tok[1], &x)) {
        rc = fail(WFST_ERR_PARSE, "line " + std::to_string(line) + ": malformed final");
        break;
      }
      fin.emplace_back(a, x);
      n = std::max(n, a + 1);
    } else {
      rc = fail(WFST_ERR_PARSE, "line " + std::to_string(line) + ": expected 2 or 5 fields");
      break;
    }
  }
  fclose(f);
  if (rc != WFST_OK) return rc;
  if (n == 0) return fail(WFST_ERR_GRAPH_INVALID, "empty graph");
  std::vector<float> final_cost(n, INFINITY);
  for (auto& p : fin) final_cost[p.first] = p.second;
  return build_graph((int32_t)n, 0, (int64_t)src.size(), src.data(), dst.data(), il.data(), ol.data(),
                     w.data(), final_cost.data(), device, out);
}

wfst_status wfst_graph_info(wfst_graph_t g, wfst_graph_info_t* info) {
  if (!g || !info) return fail(WFST_ERR_INVALID_ARG, "NULL argument");
  info->n_states = g->Q;
  info->start = g->start;
  info->n_arcs = g->E;
  info->n_emitting = g->EE;
  info->max_pdf = g->max_pdf;
  info->device = g->device;
  info->device_bytes = g->device_bytes;
  info->eq1_bytes = wfst_eq1_bytes(g->Q, g->E, g->EE);
  return WFST_OK;
}

wfst_status wfst_graph_canonical_perm(wfst_graph_t g, int64_t* perm, int64_t cap) {
  if (!g || !perm || cap < g->E) return fail(WFST_ERR_INVALID_ARG, "bad argument");
  memcpy(perm, g->perm.data(), sizeof(int64_t) * g->E);
  return WFST_OK;
}

wfst_status wfst_graph_replicate(wfst_graph_t g, int device, wfst_graph_t* out) {
  if (!g || !out) return fail(WFST_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  int n_dev = 0;
  cudaError_t e = cudaGetDeviceCount(&n_dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= n_dev) return fail(WFST_ERR_INVALID_ARG, "device out of range");
  auto* r = new wfst_graph_s();
  r->device = device;
  r->Q = g->Q;
  r->start = g->start;
  r->E = g->E;
  r->EE = g->EE;
  r->max_pdf = g->max_pdf;
  r->perm = g->perm;
  r->h_dst = g->h_dst;
  r->h_olabel = g->h_olabel;
  r->device_bytes = g->device_bytes;
  const size_t bs = sizeof(int4) * (size_t)g->Q, ba = sizeof(int4) * (size_t)(g->E > 0 ? g->E : 1),
               bo = sizeof(int32_t) * (size_t)(g->E > 0 ? g->E : 1);
  int prev = 0;
  cudaGetDevice(&prev);
  e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(&r->d_state, bs);
  if (e == cudaSuccess) e = cudaMalloc(&r->d_arcs, ba);
  if (e == cudaSuccess) e = cudaMalloc(&r->d_olabel, bo);
  // device-to-device (over NVLink when the devices are peers; staged by the driver otherwise)
  if (e == cudaSuccess) e = cudaMemcpyPeer(r->d_state, device, g->d_state, g->device, bs);
  if (e == cudaSuccess) e = cudaMemcpyPeer(r->d_arcs, device, g->d_arcs, g->device, ba);
  if (e == cudaSuccess) e = cudaMemcpyPeer(r->d_olabel, device, g->d_olabel, g->device, bo);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    wfst_graph_free(r);
    return cuda_fail(e, "graph replicate");
  }
  *out = r;
  return WFST_OK;
}

void wfst_graph_free(wfst_graph_t g) {
  if (!g) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(g->device);
  cudaFree(g->d_state);
  cudaFree(g->d_arcs);
  cudaFree(g->d_olabel);
  cudaSetDevice(prev);
  delete g;
}

// Eq. 1: M_fst = 12|Q| + 8|E| + 4|E_E|
int64_t wfst_eq1_bytes(int64_t n_states, int64_t n_arcs, int64_t n_emitting) {
  return 12 * n_states + 8 * n_arcs + 4 * n_emitting;
}
// Eq. 2: M_state = 64 alpha n_c + 544 alpha n_l + 1024 n_l
int64_t wfst_eq2_bytes(int64_t max_active, int64_t n_channels, int64_t n_lanes) {
  return 64 * max_active * n_channels + 544 * max_active * n_lanes + 1024 * n_lanes;
}

const char* wfst_last_error(void) { return g_last_error.c_str(); }

const char* wfst_status_string(wfst_status s) {
  switch (s) {
    case WFST_OK: return "OK";
    case WFST_ERR_INVALID_ARG: return "INVALID_ARG";
    case WFST_ERR_PARSE: return "PARSE";
    case WFST_ERR_GRAPH_INVALID: return "GRAPH_INVALID";
    case WFST_ERR_EPS_CYCLE: return "EPS_CYCLE";
    case WFST_ERR_PDF_RANGE: return "PDF_RANGE";
    case WFST_ERR_CAPACITY: return "CAPACITY";
    case WFST_ERR_NO_SURVIVOR: return "NO_SURVIVOR";
    case WFST_ERR_CUDA: return "CUDA";
    case WFST_ERR_OOM: return "OOM";
    case WFST_ERR_STATE: return "STATE";
  }
  return "UNKNOWN";
}

int32_t wfst_abi_version(void) { return 2; }   // 2: *_ex result calls with per-stream status

}  // extern "C"

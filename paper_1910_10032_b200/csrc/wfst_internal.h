// Internal definitions shared by the library's translation units (never by oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/wfst_gpu.h"

namespace wfst {

// Canonical arc ids are int32 everywhere on the device (winner words carry them in their low 32
// bits with 0xFFFFFFFF = the start token, records as int32 with -1 = the start token, arc array
// offsets as int), so a graph may have up to 2^31 - 1 arcs (ids 0 .. 2^31 - 2).
constexpr int64_t kMaxArcs = 0x7FFFFFFFll;

void set_error(const std::string& msg);
wfst_status fail(wfst_status s, const std::string& msg);
wfst_status cuda_fail(cudaError_t e, const char* what);

}  // namespace wfst

// Device layout of a graph (row a0; "a set of compressed sparse rows ... direct indexing").
struct wfst_graph_s {
  int device = 0;
  int32_t Q = 0, start = 0;
  int64_t E = 0, EE = 0;
  int32_t max_pdf = -1;
  // state_info[q] = {e_begin, e_end (= eps begin), eps_end, final cost bits}     16 B/state
  int4* d_state = nullptr;
  // arcs[a] = {dst, weight bits, pdf (-1 for epsilon), src | dst_has_eps << 31}  16 B/arc
  int4* d_arcs = nullptr;
  int32_t* d_olabel = nullptr;   // olabels (read only by the end-of-stream traceback)
  int64_t device_bytes = 0;
  std::vector<int64_t> perm;     // canonical arc -> input arc
  std::vector<int32_t> h_dst;    // canonical order (host copy for debug queries)
  std::vector<int32_t> h_olabel;
};

namespace wfst {
wfst_status build_graph(int32_t Q, int32_t start, int64_t E, const int32_t* src, const int32_t* dst,
                        const int32_t* ilabel, const int32_t* olabel, const float* weight,
                        const float* final_cost, int device, wfst_graph_t* out);
}

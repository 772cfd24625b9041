// plan.h — host-side planner of the template-start path (no CUDA).
//
// Implements, from the paper's description, the pieces of the function
// template and the fork plan (SURVEY.md §8(c) rules R0-R8):
//   R0 tensor names / registration order / rank-local shapes
//   R1 canonical logical-op sequence with per-op weight read lists — this is
//      also the launcher's op list, so lax tracing (§4.1 lines
//      450-451) records exactly the weights each launched op reads
//   R3 access-ordered layout, 256-B aligned (§4.2)
//   R4 resident prefix: budget (round down) or Eq. 1 (round up), PAPER.md 571
//   R5 transfer groups: per_layer / max_transfers / per_tensor (§6 602-605)
//   R6 sync barriers: per op, the groups holding weights it reads (line 555)
//   R7/R8 fork actions and byte accounting (lines 533-546)
// and the text dumps the CPU oracle (oracle/plan.py) must match byte for byte.
#pragma once
#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace tidal {

constexpr uint64_t kAlign = 256;
constexpr int kNumTargets = 7;  // q k v o gate up down
enum Target { T_Q = 0, T_K, T_V, T_O, T_GATE, T_UP, T_DOWN };
extern const char* const kTargetNames[kNumTargets];

struct ModelShape {
  int n_layers = 0, d_model = 0, n_heads = 0, n_kv_heads = 0, d_ff = 0, vocab = 0;
  bool tie = false;
  int head_dim() const { return d_model / n_heads; }
};

enum TensorRole { R_EMBED, R_PROJ, R_NORM1, R_NORM2, R_FNORM, R_HEAD, R_LORA_A, R_LORA_B };

struct TensorInfo {
  std::string name;
  int rows = 1, cols = 1;   // rank-local 2-D view (1-D tensors: rows = 1)
  uint64_t bytes = 0;       // unpadded
  bool adapter = false;
  int unit = 0;             // 0 embed, 1+i layer i, L+1 final
  int layer = -1, target = -1;
  TensorRole role = R_PROJ;
  std::string provenance;
};

struct Op {
  std::string name;
  int layer = -1;
  std::vector<int> reads;   // tensor ids (base and, if attached, adapter)
};

struct Group {
  bool adapter = false;
  std::vector<int> members; // tensor ids, contiguous in their layout
  uint64_t offset = 0, bytes = 0;
};

struct TemplateChoice {
  uint64_t resident_bytes = UINT64_MAX;
  bool eq1 = false;
  double t_ttft_s = 0, b_pcie_Bps = 0;
  int group_policy = 0;
  int max_transfers = 300;
};

// Tensor table: base tensors (registration order) then adapter tensors.
struct TensorTable {
  ModelShape shape;
  int world = 1, rank = 0;
  std::vector<TensorInfo> t;
  int n_base = 0;
  // lookups used by the launcher
  int embed = -1, fnorm = -1, head = -1;  // head == embed when tied
  std::vector<int> norm1, norm2;               // per layer
  std::vector<std::array<int, kNumTargets>> proj;   // per layer
  std::vector<std::array<int, kNumTargets>> lora_a, lora_b;  // per layer (-1 if absent)
  int lora_rank = 0;
  uint32_t lora_mask = 0;
  int find(const std::string& name) const;
};

void build_base(TensorTable& tt, const ModelShape& m, int world, int rank,
                const std::string& checkpoint);
void add_adapter(TensorTable& tt, int rank, uint32_t mask, const std::string& checkpoint);

std::vector<Op> op_sequence(const TensorTable& tt, bool with_adapter);

struct Trace {
  std::vector<std::pair<int, int>> access;  // (tensor id, op ordinal or -1 never-read)
  std::vector<Op> ops;
};
Trace make_trace(const TensorTable& tt);
std::string trace_dump(const TensorTable& tt, const Trace& tr);

struct Plan {
  std::vector<int> layout;           // base tensor ids, access order
  std::vector<uint64_t> offset;      // per tensor id: base layout or adapter buffer offset
  uint64_t layout_bytes = 0, model_bytes = 0, resident_bytes = 0, stream_bytes = 0;
  int n_resident = 0;
  uint64_t resident_end = 0;         // byte offset where the streamed suffix begins
  std::vector<int> adapter_layout;
  uint64_t adapter_bytes = 0, adapter_payload = 0;
  std::vector<Group> groups;
  std::vector<int> group_of;         // per tensor id, -1 if resident / none
  std::vector<std::vector<int>> barriers;  // per op ordinal
  std::vector<Op> ops;
};

uint64_t eq1_prefetch_bytes(uint64_t model_bytes, double t_ttft_s, double b_pcie_Bps);
// `tt` may include adapter tensors (then ops carry LoRA reads).
Plan make_plan(const TensorTable& tt, const Trace& tr, const TemplateChoice& c);
std::string plan_dump(const TensorTable& tt, const Plan& p);
// canonical adapter layout (R3 over adapter tensors in access order)
void adapter_layout(const TensorTable& tt, std::vector<int>& ids, std::vector<uint64_t>& offs,
                    uint64_t& total);
uint64_t fnv1a64(const std::string& s);

}  // namespace tidal

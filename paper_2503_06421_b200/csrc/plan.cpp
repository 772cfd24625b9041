// plan.cpp — see plan.h.  Host-only; shares no code with oracle/plan.py.
#include "plan.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <set>
#include <stdexcept>
#include <unordered_map>

namespace tidal {

const char* const kTargetNames[kNumTargets] = {"q", "k", "v", "o", "gate", "up", "down"};

static std::string module_of(int layer, int t) {
  const char* sub = t <= T_O ? "self_attn" : "mlp";
  return "model.layers." + std::to_string(layer) + "." + sub + "." + kTargetNames[t] + "_proj";
}

// rank-local [out, in] of projection t (Megatron TP: q/k/v/gate/up column-
// parallel = output rows split; o/down row-parallel = input columns split).
static void proj_shape(const ModelShape& m, int t, int world, int& out, int& in) {
  const int hd = m.head_dim();
  switch (t) {
    case T_Q: out = m.n_heads * hd / world; in = m.d_model; break;
    case T_K:
    case T_V: out = m.n_kv_heads * hd / world; in = m.d_model; break;
    case T_O: out = m.d_model; in = m.n_heads * hd / world; break;
    case T_GATE:
    case T_UP: out = m.d_ff / world; in = m.d_model; break;
    default: out = m.d_model; in = m.d_ff / world; break;
  }
}

static std::string shape_str(const TensorInfo& t) {
  if (t.rows == 1 && (t.role == R_NORM1 || t.role == R_NORM2 || t.role == R_FNORM))
    return std::to_string(t.cols);
  return std::to_string(t.rows) + "x" + std::to_string(t.cols);
}

uint64_t fnv1a64(const std::string& s) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001B3ull;
  }
  return h;
}

int TensorTable::find(const std::string& name) const {
  for (size_t i = 0; i < t.size(); ++i)
    if (t[i].name == name) return (int)i;
  return -1;
}

static int push(TensorTable& tt, TensorInfo ti, const std::string& checkpoint) {
  ti.bytes = 2ull * (uint64_t)ti.rows * (uint64_t)ti.cols;
  ti.provenance = checkpoint + ":" + ti.name + ":" + shape_str(ti);
  tt.t.push_back(ti);
  return (int)tt.t.size() - 1;
}

void build_base(TensorTable& tt, const ModelShape& m, int world, int rank,
                const std::string& checkpoint) {
  tt = TensorTable();
  tt.shape = m;
  tt.world = world;
  tt.rank = rank;
  const int L = m.n_layers;
  TensorInfo e;
  e.name = "model.embed_tokens.weight";
  e.rows = m.vocab / world;
  e.cols = m.d_model;
  e.unit = 0;
  e.role = R_EMBED;
  tt.embed = push(tt, e, checkpoint);
  tt.proj.resize(L);
  tt.norm1.resize(L);
  tt.norm2.resize(L);
  for (int i = 0; i < L; ++i) {
    for (int t = 0; t < kNumTargets; ++t) {
      TensorInfo p;
      p.name = module_of(i, t) + ".weight";
      proj_shape(m, t, world, p.rows, p.cols);
      p.unit = 1 + i;
      p.layer = i;
      p.target = t;
      p.role = R_PROJ;
      tt.proj[i][t] = push(tt, p, checkpoint);
    }
    TensorInfo n1;
    n1.name = "model.layers." + std::to_string(i) + ".input_layernorm.weight";
    n1.rows = 1;
    n1.cols = m.d_model;
    n1.unit = 1 + i;
    n1.layer = i;
    n1.role = R_NORM1;
    tt.norm1[i] = push(tt, n1, checkpoint);
    TensorInfo n2 = n1;
    n2.name = "model.layers." + std::to_string(i) + ".post_attention_layernorm.weight";
    n2.role = R_NORM2;
    tt.norm2[i] = push(tt, n2, checkpoint);
  }
  TensorInfo fn;
  fn.name = "model.norm.weight";
  fn.rows = 1;
  fn.cols = m.d_model;
  fn.unit = L + 1;
  fn.role = R_FNORM;
  tt.fnorm = push(tt, fn, checkpoint);
  if (!m.tie) {
    TensorInfo h;
    h.name = "lm_head.weight";
    h.rows = m.vocab / world;
    h.cols = m.d_model;
    h.unit = L + 1;
    h.role = R_HEAD;
    tt.head = push(tt, h, checkpoint);
  } else {
    tt.head = tt.embed;
  }
  tt.n_base = (int)tt.t.size();
  tt.lora_a.assign(L, {-1, -1, -1, -1, -1, -1, -1});
  tt.lora_b.assign(L, {-1, -1, -1, -1, -1, -1, -1});
}

void add_adapter(TensorTable& tt, int r, uint32_t mask, const std::string& checkpoint) {
  tt.t.resize(tt.n_base);
  const ModelShape& m = tt.shape;
  tt.lora_a.assign(m.n_layers, {-1, -1, -1, -1, -1, -1, -1});
  tt.lora_b.assign(m.n_layers, {-1, -1, -1, -1, -1, -1, -1});
  tt.lora_rank = r;
  tt.lora_mask = mask;
  for (int i = 0; i < m.n_layers; ++i)
    for (int t = 0; t < kNumTargets; ++t) {
      if (!((mask >> t) & 1u)) continue;
      int out, in;
      proj_shape(m, t, tt.world, out, in);
      TensorInfo a;
      a.name = module_of(i, t) + ".lora_A";
      a.rows = r;
      a.cols = in;
      a.adapter = true;
      a.unit = 1 + i;
      a.layer = i;
      a.target = t;
      a.role = R_LORA_A;
      tt.lora_a[i][t] = push(tt, a, checkpoint);
      TensorInfo b = a;
      b.name = module_of(i, t) + ".lora_B";
      b.rows = out;
      b.cols = r;
      b.role = R_LORA_B;
      tt.lora_b[i][t] = push(tt, b, checkpoint);
    }
}

std::vector<Op> op_sequence(const TensorTable& tt, bool with_adapter) {
  const ModelShape& m = tt.shape;
  const bool tp = tt.world > 1;
  std::vector<Op> ops;
  auto add = [&](const char* name, int layer, std::vector<int> reads) {
    Op o;
    o.name = name;
    o.layer = layer;
    o.reads = std::move(reads);
    ops.push_back(std::move(o));
  };
  auto lora = [&](int i, std::initializer_list<int> ts, std::vector<int>& r) {
    if (!with_adapter) return;
    for (int t : ts)
      if (tt.lora_a[i][t] >= 0) {
        r.push_back(tt.lora_a[i][t]);
        r.push_back(tt.lora_b[i][t]);
      }
  };
  add("embed", -1, {tt.embed});
  if (tp) add("embed_allreduce", -1, {});
  for (int i = 0; i < m.n_layers; ++i) {
    add("attn_norm", i, {tt.norm1[i]});
    std::vector<int> qkv = {tt.proj[i][T_Q], tt.proj[i][T_K], tt.proj[i][T_V]};
    lora(i, {T_Q, T_K, T_V}, qkv);
    add("qkv_proj", i, qkv);
    add("rope", i, {});
    add("attention", i, {});
    std::vector<int> o = {tt.proj[i][T_O]};
    lora(i, {T_O}, o);
    add("o_proj", i, o);
    if (tp) add("attn_allreduce", i, {});
    add("mlp_norm", i, {tt.norm2[i]});
    std::vector<int> gu = {tt.proj[i][T_GATE], tt.proj[i][T_UP]};
    lora(i, {T_GATE, T_UP}, gu);
    add("gate_up_proj", i, gu);
    add("act_mul", i, {});
    std::vector<int> dn = {tt.proj[i][T_DOWN]};
    lora(i, {T_DOWN}, dn);
    add("down_proj", i, dn);
    if (tp) add("mlp_allreduce", i, {});
  }
  add("final_norm", -1, {tt.fnorm});
  add("lm_head", -1, {tt.head});
  if (tp) add("logits_allgather", -1, {});
  add("argmax", -1, {});
  return ops;
}

Trace make_trace(const TensorTable& tt) {
  Trace tr;
  tr.ops = op_sequence(tt, false);
  std::vector<char> seen(tt.t.size(), 0);
  for (size_t k = 0; k < tr.ops.size(); ++k)
    for (int id : tr.ops[k].reads)
      if (id < tt.n_base && !seen[id]) {
        seen[id] = 1;
        tr.access.emplace_back(id, (int)k);
      }
  for (int id = 0; id < tt.n_base; ++id)
    if (!seen[id]) tr.access.emplace_back(id, -1);
  return tr;
}

static void append_u64(std::string& s, uint64_t v) { s += std::to_string(v); }

std::string trace_dump(const TensorTable& tt, const Trace& tr) {
  std::string s;
  char hex[32];
  for (int id = 0; id < tt.n_base; ++id) {
    const TensorInfo& t = tt.t[id];
    snprintf(hex, sizeof hex, "%016llx", (unsigned long long)fnv1a64(t.provenance));
    s += "INIT " + t.name + " " + hex + " ";
    append_u64(s, t.bytes);
    s += "\n";
  }
  for (size_t a = 0; a < tr.access.size(); ++a) {
    const auto& [id, k] = tr.access[a];
    s += "ACCESS " + std::to_string(a) + " " + tt.t[id].name + " ";
    s += k >= 0 ? tr.ops[k].name + "#" + std::to_string(k) : std::string("-");
    s += "\n";
  }
  return s;
}

static uint64_t align_up(uint64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

uint64_t eq1_prefetch_bytes(uint64_t model_bytes, double t_ttft_s, double b_pcie_Bps) {
  // Eq. 1: max(M - T*B, 0); tb = floor of one IEEE-double product.
  double prod = t_ttft_s * b_pcie_Bps;
  if (!(prod > 0)) return model_bytes;
  double f = std::floor(prod);
  if (f >= 18446744073709551615.0) return 0;
  uint64_t tb = (uint64_t)f;
  return model_bytes > tb ? model_bytes - tb : 0;
}

// max_transfers quantile cuts over one source buffer (exact integer math).
static std::vector<std::vector<int>> quantile_cuts(const std::vector<uint64_t>& sizes, int G) {
  std::vector<std::vector<int>> out;
  const int n = (int)sizes.size();
  if (n == 0) return out;
  if (n <= G) {
    for (int i = 0; i < n; ++i) out.push_back({i});
    return out;
  }
  unsigned __int128 total = 0;
  for (uint64_t s : sizes) total += s;
  unsigned __int128 cum = 0, k = 1;
  std::vector<int> cur;
  for (int i = 0; i < n; ++i) {
    cur.push_back(i);
    cum += sizes[i];
    if (cum * (unsigned)G >= k * total) {
      out.push_back(cur);
      cur.clear();
      while (k * total <= cum * (unsigned)G) ++k;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

void adapter_layout(const TensorTable& tt, std::vector<int>& ids, std::vector<uint64_t>& offs,
                    uint64_t& total) {
  ids.clear();
  offs.clear();
  std::vector<Op> ops = op_sequence(tt, true);
  std::vector<char> seen(tt.t.size(), 0);
  for (const Op& o : ops)
    for (int id : o.reads)
      if (tt.t[id].adapter && !seen[id]) {
        seen[id] = 1;
        ids.push_back(id);
      }
  uint64_t cur = 0;
  for (int id : ids) {
    cur = align_up(cur);
    offs.push_back(cur);
    cur += tt.t[id].bytes;
  }
  total = cur;
}

Plan make_plan(const TensorTable& tt, const Trace& tr, const TemplateChoice& c) {
  Plan p;
  const bool with_adapter = tt.t.size() > (size_t)tt.n_base;
  p.ops = with_adapter ? op_sequence(tt, true) : tr.ops;
  p.offset.assign(tt.t.size(), 0);
  p.group_of.assign(tt.t.size(), -1);
  // R3 base layout: access order, 256-B aligned offsets
  uint64_t cur = 0;
  for (const auto& [id, k] : tr.access) {
    (void)k;
    p.layout.push_back(id);
    cur = align_up(cur);
    p.offset[id] = cur;
    cur += tt.t[id].bytes;
    p.model_bytes += tt.t[id].bytes;
  }
  p.layout_bytes = cur;
  // R4 resident prefix
  const size_t n = p.layout.size();
  size_t k = 0;
  uint64_t acc = 0;
  if (c.eq1) {
    const uint64_t need = eq1_prefetch_bytes(p.model_bytes, c.t_ttft_s, c.b_pcie_Bps);
    while (acc < need && k < n) acc += tt.t[p.layout[k++]].bytes;
  } else if (c.resident_bytes == UINT64_MAX) {
    k = n;
    acc = p.model_bytes;
  } else {
    while (k < n && acc + tt.t[p.layout[k]].bytes <= c.resident_bytes) acc += tt.t[p.layout[k++]].bytes;
  }
  p.n_resident = (int)k;
  p.resident_bytes = acc;
  p.stream_bytes = p.model_bytes - acc;
  p.resident_end = k < n ? p.offset[p.layout[k]] : p.layout_bytes;
  // adapter layout
  uint64_t atotal = 0;
  if (with_adapter) {
    std::vector<uint64_t> aoffs;
    adapter_layout(tt, p.adapter_layout, aoffs, atotal);
    for (size_t i = 0; i < p.adapter_layout.size(); ++i) {
      p.offset[p.adapter_layout[i]] = aoffs[i];
      p.adapter_payload += tt.t[p.adapter_layout[i]].bytes;
    }
  }
  p.adapter_bytes = atotal;
  // combined first-read ordinal for ordering groups
  std::vector<int64_t> ordinal(tt.t.size(), INT64_MAX);
  {
    int64_t o = 0;
    for (const Op& op : p.ops)
      for (int id : op.reads)
        if (ordinal[id] == INT64_MAX) ordinal[id] = o++;
  }
  // R5 candidate groups
  std::vector<Group> cand;
  std::vector<int> streamed(p.layout.begin() + k, p.layout.end());
  if (c.group_policy == 0) {
    std::map<int, std::vector<int>> by_unit, a_by_unit;
    for (int id : streamed) by_unit[tt.t[id].unit].push_back(id);
    for (int id : p.adapter_layout) a_by_unit[tt.t[id].unit].push_back(id);
    for (auto& [u, mem] : by_unit) {
      Group g;
      g.members = mem;
      cand.push_back(g);
    }
    for (auto& [u, mem] : a_by_unit) {
      Group g;
      g.adapter = true;
      g.members = mem;
      cand.push_back(g);
    }
  } else if (c.group_policy == 1) {
    for (int pass = 0; pass < 2; ++pass) {
      const std::vector<int>& src = pass == 0 ? streamed : p.adapter_layout;
      std::vector<uint64_t> sz;
      for (int id : src) sz.push_back(tt.t[id].bytes);
      for (auto& idxs : quantile_cuts(sz, std::max(1, c.max_transfers))) {
        Group g;
        g.adapter = pass == 1;
        for (int i : idxs) g.members.push_back(src[i]);
        cand.push_back(g);
      }
    }
  } else {
    for (int id : streamed) {
      Group g;
      g.members = {id};
      cand.push_back(g);
    }
    for (int id : p.adapter_layout) {
      Group g;
      g.adapter = true;
      g.members = {id};
      cand.push_back(g);
    }
  }
  std::stable_sort(cand.begin(), cand.end(), [&](const Group& a, const Group& b) {
    return ordinal[a.members[0]] < ordinal[b.members[0]];
  });
  for (size_t g = 0; g < cand.size(); ++g) {
    Group& G = cand[g];
    const int first = G.members.front(), last = G.members.back();
    G.offset = p.offset[first];
    G.bytes = p.offset[last] + tt.t[last].bytes - G.offset;
    for (int id : G.members) p.group_of[id] = (int)g;
  }
  p.groups = std::move(cand);
  // R6 barriers
  p.barriers.resize(p.ops.size());
  for (size_t kk = 0; kk < p.ops.size(); ++kk) {
    std::set<int> s;
    for (int id : p.ops[kk].reads)
      if (p.group_of[id] >= 0) s.insert(p.group_of[id]);
    p.barriers[kk].assign(s.begin(), s.end());
  }
  return p;
}

std::string plan_dump(const TensorTable& tt, const Plan& p) {
  std::string s;
  for (size_t i = 0; i < p.layout.size(); ++i)
    s += "ACTION " + tt.t[p.layout[i]].name + ((int)i < p.n_resident ? " RESIDENT " : " STREAM ") +
         std::to_string(i) + "\n";
  std::unordered_map<int, size_t> aidx;
  for (size_t i = 0; i < p.adapter_layout.size(); ++i) aidx[p.adapter_layout[i]] = i;
  for (const Group& g : p.groups)
    if (g.adapter)
      for (int id : g.members) s += "ACTION " + tt.t[id].name + " ADAPTER " + std::to_string(aidx[id]) + "\n";
  for (size_t g = 0; g < p.groups.size(); ++g) {
    const Group& G = p.groups[g];
    s += "GROUP " + std::to_string(g) + (G.adapter ? " adapter " : " base ") + std::to_string(G.offset) +
         " " + std::to_string(G.bytes) + " " + tt.t[G.members.front()].name + " " +
         tt.t[G.members.back()].name + "\n";
  }
  for (size_t k = 0; k < p.barriers.size(); ++k) {
    if (p.barriers[k].empty()) continue;
    s += "BARRIER " + std::to_string(k) + " ";
    for (size_t j = 0; j < p.barriers[k].size(); ++j) s += (j ? "," : "") + std::to_string(p.barriers[k][j]);
    s += "\n";
  }
  s += "BYTES " + std::to_string(p.resident_bytes) + " " + std::to_string(p.stream_bytes) + " " +
       std::to_string(p.adapter_payload) + " " + std::to_string(p.model_bytes) + "\n";
  return s;
}

}  // namespace tidal

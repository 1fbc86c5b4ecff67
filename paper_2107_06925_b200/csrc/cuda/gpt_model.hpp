// GPT-2 stage partition and per-stage parameter layout.
//
// Stage s of D holds layers [s*L/D, (s+1)*L/D); stage 0 additionally the token and
// position embeddings, stage D-1 the final LayerNorm and an untied LM head over a
// vocabulary padded to a multiple of 128 (pad rows never receive gradient).  Every
// tensor of a stage lives in one flat buffer (fp32 master, bf16 working copy, fp32
// gradient per replica), 128-byte aligned, so that the stage allreduce is one
// contiguous NCCL call and the SGD update one kernel.
#pragma once

#include <string>
#include <vector>

namespace chimera::gpt {

struct ModelShape {
  int n_layer = 8, hidden = 256, heads = 4, ffn = 1024, seq = 128, vocab = 1024, vocab_padded = 1024;
  bool causal = true;
  std::vector<int> stage_layers;  // layers per stage (empty = n_layer / D each)

  int layers_of(int D, int s) const { return stage_layers.empty() ? n_layer / D : stage_layers[s]; }
  int first_layer_of(int D, int s) const {
    int f = 0;
    for (int k = 0; k < s; ++k) f += layers_of(D, k);
    return f;
  }
};

enum class Init { Zero, One, Normal };

struct TensorSlot {
  std::string name;
  long long offset = 0;  // elements
  long long rows = 0, cols = 0;
  Init init = Init::Normal;
  long long numel() const { return rows * cols; }
};

struct LayerOffsets {
  long long ln1_g, ln1_b, w_qkv, b_qkv, w_o, b_o, ln2_g, ln2_b, w_fc1, b_fc1, w_fc2, b_fc2;
};

struct StageLayout {
  int stage = 0, first_layer = 0, n_layers = 0;
  bool has_embed = false, has_head = false;
  long long wte = -1, wpe = -1, lnf_g = -1, lnf_b = -1, w_head = -1;
  std::vector<LayerOffsets> layers;
  std::vector<TensorSlot> tensors;
  long long total = 0;  // elements (multiple of 64)
};

inline StageLayout make_stage_layout(const ModelShape& m, int D, int s) {
  StageLayout L;
  L.stage = s;
  const int per = m.layers_of(D, s);
  L.first_layer = m.first_layer_of(D, s);
  L.n_layers = per;
  L.has_embed = s == 0;
  L.has_head = s == D - 1;
  const long long h = m.hidden, f = m.ffn;
  auto add = [&](const std::string& name, long long rows, long long cols, Init init) {
    TensorSlot t{name, L.total, rows, cols, init};
    L.tensors.push_back(t);
    L.total += (rows * cols + 63) / 64 * 64;
    return t.offset;
  };
  if (L.has_embed) {
    L.wte = add("wte", m.vocab_padded, h, Init::Normal);
    L.wpe = add("wpe", m.seq, h, Init::Normal);
  }
  for (int l = 0; l < per; ++l) {
    const std::string p = "h" + std::to_string(L.first_layer + l) + ".";
    LayerOffsets o;
    o.ln1_g = add(p + "ln1.g", 1, h, Init::One);
    o.ln1_b = add(p + "ln1.b", 1, h, Init::Zero);
    o.w_qkv = add(p + "attn.w_qkv", 3 * h, h, Init::Normal);
    o.b_qkv = add(p + "attn.b_qkv", 1, 3 * h, Init::Zero);
    o.w_o = add(p + "attn.w_o", h, h, Init::Normal);
    o.b_o = add(p + "attn.b_o", 1, h, Init::Zero);
    o.ln2_g = add(p + "ln2.g", 1, h, Init::One);
    o.ln2_b = add(p + "ln2.b", 1, h, Init::Zero);
    o.w_fc1 = add(p + "mlp.w_fc1", f, h, Init::Normal);
    o.b_fc1 = add(p + "mlp.b_fc1", 1, f, Init::Zero);
    o.w_fc2 = add(p + "mlp.w_fc2", h, f, Init::Normal);
    o.b_fc2 = add(p + "mlp.b_fc2", 1, h, Init::Zero);
    L.layers.push_back(o);
  }
  if (L.has_head) {
    L.lnf_g = add("lnf.g", 1, h, Init::One);
    L.lnf_b = add("lnf.b", 1, h, Init::Zero);
    L.w_head = add("lm_head", m.vocab_padded, h, Init::Normal);
  }
  return L;
}

}  // namespace chimera::gpt

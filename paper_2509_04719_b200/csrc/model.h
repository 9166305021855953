// Model presets and weight manifest of the DiT family.
// Must match synth/configs.py manifest() tensor for tensor (checked by
// tests/test_boundary.py through stadi_weight_info).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/stadi.h"

namespace stadi {

struct Dims {
  int preset = 0;
  bool text = false;
  int d = 0, H = 0, hd = 0, depth = 0, p = 2, c_in = 4, c_out = 4;
  int lat_h = 0, lat_w = 0, hp = 0, wp = 0;
  int B = 1;
  float guidance = 0.f;
  int num_classes = 0;
  int txt_len = 0, txt_dim = 0;
  int schedule_linear = 1;  // DiT shapes: linear beta schedule (R18)
};

struct TensorSpec {
  std::string name;
  int64_t rows, cols;  // cols == 1 for vectors
  bool gemm_weight;    // used as a tcgen05 / SIMT GEMM B operand
};

inline bool make_dims(const stadi_model_desc &m, Dims &o, std::string &err) {
  Dims d;
  d.preset = m.preset;
  switch (m.preset) {
    case STADI_PRESET_TINY_DIT:
      d.d = 64; d.H = 4; d.depth = 2; d.c_out = 4; d.lat_h = d.lat_w = 16;
      d.num_classes = 10; d.B = 1; d.guidance = 0.f;
      break;
    case STADI_PRESET_DIT_XL2:
      d.d = 1152; d.H = 16; d.depth = 28; d.c_out = 8; d.lat_h = d.lat_w = 32;
      d.num_classes = 1000; d.B = 2; d.guidance = 4.0f;
      break;
    case STADI_PRESET_PIXART_ALPHA:
      d.d = 1152; d.H = 16; d.depth = 28; d.c_out = 8; d.lat_h = d.lat_w = 256;
      d.text = true; d.txt_len = 120; d.txt_dim = 4096; d.B = 2; d.guidance = 4.5f;
      break;
    default:
      err = "unknown preset";
      return false;
  }
  if (m.depth > 0) d.depth = m.depth;
  if (m.latent_h > 0) d.lat_h = m.latent_h;
  if (m.latent_w > 0) d.lat_w = m.latent_w;
  if (d.lat_h % d.p || d.lat_w % d.p || d.depth < 1 || d.depth > 64) {
    err = "latent size must be a multiple of the patch size; depth in 1..64";
    return false;
  }
  d.hd = d.d / d.H;
  d.hp = d.lat_h / d.p;
  d.wp = d.lat_w / d.p;
  o = d;
  return true;
}

inline std::vector<TensorSpec> manifest(const Dims &m) {
  std::vector<TensorSpec> v;
  const int64_t d = m.d, pp = m.p * m.p;
  auto W = [&](const std::string &n, int64_t r, int64_t c, bool g) { v.push_back({n, r, c, g}); };
  auto V = [&](const std::string &n, int64_t r) { v.push_back({n, r, 1, false}); };
  W("x_embed.w", d, m.c_in * pp, false); V("x_embed.b", d);
  W("t_embed.w1", d, 256, false); V("t_embed.b1", d);
  W("t_embed.w2", d, d, false); V("t_embed.b2", d);
  if (m.text) {
    W("t_block.w", 6 * d, d, true); V("t_block.b", 6 * d);
    W("caption.w1", d, m.txt_dim, true); V("caption.b1", d);
    W("caption.w2", d, d, true); V("caption.b2", d);
  } else {
    W("y_embed.table", m.num_classes + 1, d, false);
  }
  for (int l = 0; l < m.depth; ++l) {
    const std::string p = "blocks." + std::to_string(l) + ".";
    if (m.text) {
      W(p + "sst", 6, d, false);
    } else {
      W(p + "ada.w", 6 * d, d, true); V(p + "ada.b", 6 * d);
    }
    W(p + "qkv.w", 3 * d, d, true); V(p + "qkv.b", 3 * d);
    W(p + "proj.w", d, d, true); V(p + "proj.b", d);
    if (m.text) {
      W(p + "xq.w", d, d, true); V(p + "xq.b", d);
      W(p + "xkv.w", 2 * d, d, true); V(p + "xkv.b", 2 * d);
      W(p + "xproj.w", d, d, true); V(p + "xproj.b", d);
    }
    W(p + "fc1.w", 4 * d, d, true); V(p + "fc1.b", 4 * d);
    W(p + "fc2.w", d, 4 * d, true); V(p + "fc2.b", d);
  }
  if (m.text) {
    W("final.sst", 2, d, false);
  } else {
    W("final.ada.w", 2 * d, d, true); V("final.ada.b", 2 * d);
  }
  W("final.linear.w", pp * m.c_out, d, true); V("final.linear.b", pp * m.c_out);
  return v;
}

}  // namespace stadi

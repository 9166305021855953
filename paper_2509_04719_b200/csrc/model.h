// Model presets and weight manifests of the DiT and U-Net families (SURVEY
// §8(c) O4).  Must match synth/configs.py manifest() tensor for tensor
// (checked by tests/test_boundary.py through stadi_weight_info).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/stadi.h"

namespace stadi {

struct Dims {
  int preset = 0;
  bool unet = false;  // U-Net family (C3 SD-1.5, C4 SDXL shapes)
  bool text = false;
  int d = 0, H = 0, hd = 0, depth = 0, p = 2, c_in = 4, c_out = 4;
  int lat_h = 0, lat_w = 0, hp = 0, wp = 0;
  int B = 1;
  float guidance = 0.f;
  int num_classes = 0;
  int txt_len = 0, txt_dim = 0;
  int schedule_linear = 1;  // DiT shapes: linear beta schedule (R18)
  // U-Net family
  std::vector<int> ch, tdepth, heads;  // per level: channels, transformer depth, heads
  int mid_depth = 0, nres = 2;         // transformer depth of the mid block; ResBlocks/level
  bool add_embed = false;              // SDXL micro-conditioning embedding
  int pooled_dim = 0;
  float time_ids[6] = {0, 0, 0, 0, 0, 0};
  int levels() const { return (int)ch.size(); }
  int temb_dim() const { return 4 * ch[0]; }
};

// Up path of a U-Net (diffusers' channel bookkeeping): per up level i (coarsest
// first) its channels c, transformer depth and, per ResBlock j, {in, skip, out}.
struct UpLevel {
  int i, c, depth, heads;
  std::vector<std::array<int, 3>> res;
};
inline std::vector<UpLevel> unet_up_io(const Dims &m) {
  const int L = m.levels();
  std::vector<UpLevel> out;
  int prev = m.ch[L - 1];
  for (int i = 0; i < L; ++i) {
    const int lv = L - 1 - i;  // resolution level of up block i
    const int oc = m.ch[lv], ic = m.ch[std::max(lv - 1, 0)];
    UpLevel u{i, oc, m.tdepth[lv], m.heads[lv], {}};
    for (int j = 0; j <= m.nres; ++j) {
      const int skip = (j == m.nres) ? ic : oc;
      const int rin = (j == 0) ? prev : oc;
      u.res.push_back({rin, skip, oc});
    }
    out.push_back(u);
    prev = oc;
  }
  return out;
}

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
    case STADI_PRESET_SD15:
      d.unet = true; d.text = true; d.ch = {320, 640, 1280, 1280}; d.tdepth = {1, 1, 1, 0};
      d.heads = {8, 8, 8, 8}; d.mid_depth = 1; d.txt_len = 77; d.txt_dim = 768;
      d.lat_h = d.lat_w = 64; d.B = 2; d.guidance = 7.5f;
      break;
    case STADI_PRESET_SDXL:
      d.unet = true; d.text = true; d.ch = {320, 640, 1280}; d.tdepth = {0, 2, 10};
      d.heads = {5, 10, 20}; d.mid_depth = 10; d.txt_len = 77; d.txt_dim = 2048;
      d.add_embed = true; d.pooled_dim = 1280;
      {
        const float ti[6] = {1024, 1024, 0, 0, 1024, 1024};
        for (int i = 0; i < 6; ++i) d.time_ids[i] = ti[i];
      }
      d.lat_h = d.lat_w = 128; d.B = 2; d.guidance = 5.0f;
      break;
    case STADI_PRESET_TINY_UNET:
      d.unet = true; d.text = true; d.ch = {64, 128}; d.tdepth = {0, 1}; d.heads = {4, 8};
      d.mid_depth = 1; d.nres = 1; d.txt_len = 8; d.txt_dim = 64; d.add_embed = true;
      d.pooled_dim = 64;
      {
        const float ti[6] = {64, 64, 0, 0, 64, 64};
        for (int i = 0; i < 6; ++i) d.time_ids[i] = ti[i];
      }
      d.lat_h = d.lat_w = 16; d.B = 2; d.guidance = 5.0f;
      break;
    default:
      err = "unknown preset";
      return false;
  }
  if (d.unet) {
    d.p = 1;
    d.c_out = 4;
    d.schedule_linear = 0;  // U-Net shapes: scaled-linear beta schedule (R18)
    if (m.depth > 0)
      for (auto &t : d.tdepth) t = t ? std::min(t, m.depth) : 0;
    if (m.depth > 0) d.mid_depth = std::min(d.mid_depth, m.depth);
    const int u = 1 << (d.levels() - 1);
    if (m.latent_h > 0) d.lat_h = m.latent_h;
    if (m.latent_w > 0) d.lat_w = m.latent_w;
    if (d.lat_h % u || d.lat_w % u) {
      err = "U-Net latent size must be a multiple of 2^(levels-1)";
      return false;
    }
    d.hp = d.lat_h;
    d.wp = d.lat_w;
    d.depth = 0;
    o = d;
    return true;
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

// U-Net: diffusers UNet2DConditionModel layer list (same order as
// synth/configs.py unet_manifest).  Conv weights are [Cout, Cin, 3, 3].
inline std::vector<TensorSpec> unet_manifest(const Dims &m) {
  std::vector<TensorSpec> v;
  auto W = [&](const std::string &n, int64_t r, int64_t c, bool g) { v.push_back({n, r, c, g}); };
  auto V = [&](const std::string &n, int64_t r) { v.push_back({n, r, 1, false}); };
  const int64_t C0 = m.ch[0], td = m.temb_dim();
  const int L = m.levels();
  auto res = [&](const std::string &p, int64_t cin, int64_t cout) {
    V(p + "norm1.w", cin); V(p + "norm1.b", cin);
    W(p + "conv1.w", cout, cin * 9, true); V(p + "conv1.b", cout);
    W(p + "temb.w", cout, td, false); V(p + "temb.b", cout);
    V(p + "norm2.w", cout); V(p + "norm2.b", cout);
    W(p + "conv2.w", cout, cout * 9, true); V(p + "conv2.b", cout);
    if (cin != cout) { W(p + "skip.w", cout, cin, true); V(p + "skip.b", cout); }
  };
  auto tr = [&](const std::string &p, int64_t c, int depth) {
    const int64_t ctx = m.txt_dim;
    V(p + "norm.w", c); V(p + "norm.b", c);
    W(p + "proj_in.w", c, c, true); V(p + "proj_in.b", c);
    for (int k = 0; k < depth; ++k) {
      const std::string q = p + "blk" + std::to_string(k) + ".";
      V(q + "ln1.w", c); V(q + "ln1.b", c);
      W(q + "attn1.q", c, c, true); W(q + "attn1.k", c, c, true); W(q + "attn1.v", c, c, true);
      W(q + "attn1.o", c, c, true); V(q + "attn1.ob", c);
      V(q + "ln2.w", c); V(q + "ln2.b", c);
      W(q + "attn2.q", c, c, true); W(q + "attn2.k", c, ctx, true); W(q + "attn2.v", c, ctx, true);
      W(q + "attn2.o", c, c, true); V(q + "attn2.ob", c);
      V(q + "ln3.w", c); V(q + "ln3.b", c);
      W(q + "ff1.w", 8 * c, c, true); V(q + "ff1.b", 8 * c);
      W(q + "ff2.w", c, 4 * c, true); V(q + "ff2.b", c);
    }
    W(p + "proj_out.w", c, c, true); V(p + "proj_out.b", c);
  };
  W("time.w1", td, C0, false); V("time.b1", td);
  W("time.w2", td, td, false); V("time.b2", td);
  if (m.add_embed) {
    W("add.w1", td, 6 * 256 + m.pooled_dim, false); V("add.b1", td);
    W("add.w2", td, td, false); V("add.b2", td);
  }
  W("conv_in.w", C0, m.c_in * 9, false); V("conv_in.b", C0);
  int64_t prev = C0;
  for (int i = 0; i < L; ++i) {
    const int64_t c = m.ch[i];
    for (int j = 0; j < m.nres; ++j) {
      res("down" + std::to_string(i) + ".res" + std::to_string(j) + ".", j == 0 ? prev : c, c);
      if (m.tdepth[i])
        tr("down" + std::to_string(i) + ".attn" + std::to_string(j) + ".", c, m.tdepth[i]);
    }
    if (i < L - 1) {
      W("down" + std::to_string(i) + ".ds.w", c, c * 9, true);
      V("down" + std::to_string(i) + ".ds.b", c);
    }
    prev = c;
  }
  const int64_t cm = m.ch[L - 1];
  res("mid.res0.", cm, cm);
  tr("mid.attn.", cm, m.mid_depth);
  res("mid.res1.", cm, cm);
  for (const auto &u : unet_up_io(m)) {
    for (size_t j = 0; j < u.res.size(); ++j) {
      const std::string p = "up" + std::to_string(u.i) + ".res" + std::to_string(j) + ".";
      res(p, u.res[j][0] + u.res[j][1], u.res[j][2]);
      if (u.depth)
        tr("up" + std::to_string(u.i) + ".attn" + std::to_string(j) + ".", u.res[j][2], u.depth);
    }
    if (u.i < L - 1) {
      W("up" + std::to_string(u.i) + ".us.w", u.c, u.c * 9, true);
      V("up" + std::to_string(u.i) + ".us.b", u.c);
    }
  }
  V("out.norm.w", C0); V("out.norm.b", C0);
  W("out.conv.w", m.c_out, C0 * 9, true); V("out.conv.b", m.c_out);
  return v;
}

inline std::vector<TensorSpec> manifest(const Dims &m) {
  if (m.unet) return unet_manifest(m);
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

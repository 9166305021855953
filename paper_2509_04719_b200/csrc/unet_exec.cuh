// U-Net executor of the patch-parallel path (BASELINE C3 SD-1.5 / C4 SDXL
// shapes).  Included by runtime.cu (it uses the runtime's internal dispatch,
// timing and error helpers); not a separate translation unit.
//
// A rank's band forward is compiled once per plan into a flat PROGRAM of ops
// (closures over the rank's buffers, parameterised at run time by the step:
// fast-grid index m -> time-embedding row, read / publish versions, Eq. 3
// coefficients).  Exchange sites are split into a PUBLISH op and a CONSUME op,
// so running the programs of all hosted ranks op-index by op-index (local
// mode) gives the layer-lock-step a fresh (warmup) exchange needs, and a
// single rank (NCCL mode) just runs its own program.  Sites (SURVEY §8(c) O5,
// PAPER.md L80 / L171 stale activations):
//   KV   self-attention K/V: full-image slot [N_l, B, 2, C], own rows written
//        by the QKV GEMM epilogue (R14), variable-size all-gather
//   HALO 3x3-conv input boundary rows: slot [n_inc][2][W_l * B * C], own first /
//        last interior rows of the padded conv input; the consumer copies the
//        neighbours' rows into its halo rows (zeros at the image edge; R15 conv_in,
//        R16 upsample uses the pre-upsample rows)
//   GN   GroupNorm partial sums: slot [n_inc][B][32][2] fp64 (R17)
// Activations: X [h, W, B, C] fp32 (token-major, batch innermost); conv / GEMM
// operands bf16 (fp32 in the debug build).

namespace {

enum USiteKind { US_KV = 0, US_HALO = 1, US_GN = 2 };

struct USite {
  int id = 0;  // index in UNetState::sites (IPC flag index)
  int kind = 0, level = 0, C = 0;
  int64_t seg_bytes = 0;  // HALO / GN: bytes per rank segment; KV: bytes per token row
  std::vector<std::array<void *, 2>> slot;  // [hosted rank][parity]
  cudaEvent_t ev[2] = {nullptr, nullptr};
  bool used[2] = {false, false};
};

using UOp = std::function<stadi_status(const stadi_step_t &, cudaStream_t)>;

struct URank {
  std::vector<void *> buf;
  std::vector<size_t> size;
  std::vector<UOp> prog;
};

// Work buffers of a rank (ids >= UB_COUNT are the down-path skip buffers).
enum {
  UB_CAT = 0, UB_H, UB_H1, UB_SK, UB_TY, UB_PAD, UB_COL, UB_NB, UB_Q, UB_O, UB_FF, UB_EPS, UB_GNS,
  UB_UPS,  // nearest-x2 upsampled padded conv input (implicit upsample conv)
  UB_COUNT
};

struct UNetState {
  std::map<std::string, void *> wt;   // GEMM operands (T), transformed at load
  std::map<std::string, float *> wf;  // fp32 vectors (bf16-rounded in bf16 mode)
  std::map<std::string, int> temb_off;
  int temb_total = 0;                 // sum of ResBlock output channels
  int n_tr_blocks = 0;
  std::map<std::string, int> tr_index;
  std::vector<USite> sites;
  std::vector<URank> ranks;           // parallel to ctx->ranks
  std::vector<int> inc;               // included group ranks in row order
  // per request
  float *tfeat = nullptr, *t1 = nullptr, *temb = nullptr, *tembB = nullptr, *addin = nullptr,
        *aug1 = nullptr, *aug = nullptr, *temb_all = nullptr;
  void *tsilu = nullptr;
  std::vector<void *> text_kv;        // per transformer block [L, B, 2, C]
  int cap_nt = 0;
  double *gn_ws = nullptr;            // fixed-order GN partial reduction (one stream at a time)
  unsigned *gn_ticket = nullptr;
};

inline int64_t rup64(int64_t a) { return (a + 63) / 64 * 64; }

// STADI_CONV_IMPLICIT=0 forces the im2col path (A/B comparisons).
bool conv_implicit_disabled() {
  static const int v = [] {
    const char *e = getenv("STADI_CONV_IMPLICIT");
    return (e && e[0] == '0') ? 1 : 0;
  }();
  return v != 0;
}

// ------------------------------------------------------------------ weights
__global__ void temb_combine_kernel(const float *temb, const float *aug, int nt, int B, int td,
                                    float *out) {  // out[m*B + b] = temb[m] + aug[b]
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long)nt * B * td) return;
  const int c = (int)(i % td);
  const long r = i / td;
  const int b = (int)(r % B), m = (int)(r / B);
  out[i] = temb[(long)m * td + c] + (aug ? aug[(long)b * td + c] : 0.f);
}

float bf16_round_host(float x, bool bf) {
  if (!bf) return x;
  uint32_t u;
  std::memcpy(&u, &x, 4);
  const uint32_t lsb = (u >> 16) & 1u;
  u = (u + 0x7FFFu + lsb) & 0xFFFF0000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

cudaError_t upload_vec(stadi_ctx *ctx, const std::vector<float> &h, float **dst) {
  cudaError_t e = dalloc(ctx, dst, h.size() * 4);
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
}
cudaError_t upload_gemm(stadi_ctx *ctx, const std::vector<float> &h, void **dst) {
  float *f = nullptr;
  cudaError_t e = cudaMalloc(&f, h.size() * 4);
  if (e != cudaSuccess) return e;
  e = cudaMemcpy(f, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return e;
  if (ctx->dtype == STADI_DTYPE_BF16) {
    bf16 *t = nullptr;
    e = dalloc(ctx, &t, h.size() * 2);
    if (e == cudaSuccess) e = cast_f32<bf16>(f, t, (long)h.size(), 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    cudaFreeAsync(f, 0);
    *dst = t;
    return e;
  }
  ctx->allocs.push_back(f);
  *dst = f;
  return cudaSuccess;
}

// Host-side layout transforms of the U-Net weights (permutations / padding only).
stadi_status unet_load_weights(stadi_ctx *ctx, const float *const *host) {
  auto U = std::make_unique<UNetState>();
  const Dims &m = ctx->dm;
  const bool bf = ctx->dtype == STADI_DTYPE_BF16;
  std::map<std::string, std::pair<const float *, const TensorSpec *>> by;
  for (size_t i = 0; i < ctx->man.size(); ++i) by[ctx->man[i].name] = {host[i], &ctx->man[i]};
  auto vec = [&](const std::string &n) {
    const auto &p = by.at(n);
    const int64_t k = p.second->rows * p.second->cols;
    std::vector<float> v(p.first, p.first + k);
    for (auto &x : v) x = bf16_round_host(x, bf);
    return v;
  };
  auto raw = [&](const std::string &n) {
    const auto &p = by.at(n);
    return std::vector<float>(p.first, p.first + p.second->rows * p.second->cols);
  };
  std::vector<float> temb_w, temb_b;
  for (const auto &ts : ctx->man) {
    const std::string &n = ts.name;
    const auto ends = [&](const char *suf) {
      const size_t L = std::strlen(suf);
      return n.size() >= L && n.compare(n.size() - L, L, suf) == 0;
    };
    if (n.rfind("time.", 0) == 0 || n.rfind("add.", 0) == 0) {  // SIMT fp32 conditioning
      CK(upload_vec(ctx, vec(n), &U->wf[n]));
    } else if (ends("conv1.w") || ends("conv2.w") || ends(".ds.w") || ends(".us.w") ||
               n == "conv_in.w" || n == "out.conv.w") {
      // [Cout, Cin, 3, 3] -> [Cout_pad, Kp], column (ky*3 + kx)*Cin + c
      const int64_t cout = ts.rows, cin = ts.cols / 9, kp = rup64(9 * cin);
      const int64_t cpad = n == "out.conv.w" ? 64 : cout;
      const auto w = raw(n);
      std::vector<float> o((size_t)(cpad * kp), 0.f);
      for (int64_t a = 0; a < cout; ++a)
        for (int64_t c = 0; c < cin; ++c)
          for (int t = 0; t < 9; ++t) o[a * kp + t * cin + c] = w[(a * cin + c) * 9 + t];
      CK(upload_gemm(ctx, o, &U->wt[n]));
    } else if (n == "out.conv.b") {
      auto b = vec(n);
      b.resize(64, 0.f);
      CK(upload_vec(ctx, b, &U->wf[n]));
    } else if (ends("temb.w")) {
      const auto w = raw(n);
      U->temb_off[n.substr(0, n.size() - 6)] = U->temb_total;
      U->temb_total += (int)ts.rows;
      temb_w.insert(temb_w.end(), w.begin(), w.end());
    } else if (ends("temb.b")) {
      const auto b = vec(n);
      temb_b.insert(temb_b.end(), b.begin(), b.end());
    } else if (ends("attn1.q")) {
      const std::string p = n.substr(0, n.size() - 1);
      std::vector<float> o = raw(n), k = raw(p + "k"), v = raw(p + "v");
      o.insert(o.end(), k.begin(), k.end());
      o.insert(o.end(), v.begin(), v.end());
      CK(upload_gemm(ctx, o, &U->wt[p + "qkv"]));
    } else if (ends("attn2.k")) {
      const std::string p = n.substr(0, n.size() - 1);
      std::vector<float> o = raw(n), v = raw(p + "v");
      o.insert(o.end(), v.begin(), v.end());
      CK(upload_gemm(ctx, o, &U->wt[p + "kv"]));
      U->tr_index[p] = U->n_tr_blocks++;
    } else if (ends("attn1.k") || ends("attn1.v") || ends("attn2.v")) {
      continue;  // folded into qkv / kv above
    } else if (ends("ff1.w")) {  // interleave (a_i, g_i) rows for the GEGLU epilogue
      const auto w = raw(n);
      const int64_t c4 = ts.rows / 2, k = ts.cols;
      std::vector<float> o(w.size());
      for (int64_t i = 0; i < c4; ++i) {
        std::memcpy(&o[(2 * i) * k], &w[i * k], k * 4);
        std::memcpy(&o[(2 * i + 1) * k], &w[(c4 + i) * k], k * 4);
      }
      CK(upload_gemm(ctx, o, &U->wt[n]));
    } else if (ends("ff1.b")) {
      const auto b = vec(n);
      const size_t c4 = b.size() / 2;
      std::vector<float> o(b.size());
      for (size_t i = 0; i < c4; ++i) {
        o[2 * i] = b[i];
        o[2 * i + 1] = b[c4 + i];
      }
      CK(upload_vec(ctx, o, &U->wf[n]));
    } else if ((ends("ln1.w") || ends("ln2.w") || ends("ln3.w"))) {  // LN gain as (w - 1)
      auto w = vec(n);
      for (auto &x : w) x -= 1.f;
      CK(upload_vec(ctx, w, &U->wf[n]));
    } else if (ts.gemm_weight) {
      CK(upload_gemm(ctx, raw(n), &U->wt[n]));
    } else {
      CK(upload_vec(ctx, vec(n), &U->wf[n]));
    }
  }
  CK(dalloc(ctx, &U->gn_ws, (size_t)GN_PARTIAL_BLOCKS * 2 * 2 * 32 * sizeof(double)));
  CK(dalloc(ctx, &U->gn_ticket, 256));
  CK(cudaMemset(U->gn_ticket, 0, 256));
  CK(upload_gemm(ctx, temb_w, &U->wt["temb_all.w"]));
  CK(upload_vec(ctx, temb_b, &U->wf["temb_all.b"]));
  (void)m;
  ctx->un = std::move(U);
  return STADI_OK;
}

// ------------------------------------------------------------------ exchange
// Rank position among the included ranks (row order), or -1.
int inc_pos(UNetState *U, int g) {
  for (size_t i = 0; i < U->inc.size(); ++i)
    if (U->inc[i] == g) return (int)i;
  return -1;
}

// Publish rank li's own payload of version `ver` at site s (already written into
// its slot[ver & 1]).  Local mode: device copies into the other hosted ranks'
// slots.  NCCL mode: in-place all-gather (equal segments) or grouped broadcasts
// (KV, variable segments) on the comm stream.
stadi_status u_publish(stadi_ctx *ctx, USite &S, int li, int ver, cudaStream_t s) {
  UNetState *U = ctx->un.get();
  const int par = ver & 1;
  const Rank &r = ctx->ranks[li];
  const Dims &m = ctx->dm;
  auto seg = [&](int g, int64_t *off, int64_t *bytes) {
    if (S.kind == US_KV) {
      const int64_t rb = ctx->plan.row_begin[g] >> S.level, rr = ctx->plan.rows[g] >> S.level;
      const int64_t wl = m.lat_w >> S.level;
      *off = rb * wl * S.seg_bytes;
      *bytes = rr * wl * S.seg_bytes;
    } else {
      *off = inc_pos(U, g) * S.seg_bytes;
      *bytes = S.seg_bytes;
    }
  };
  int64_t off, bytes;
  seg(r.g, &off, &bytes);
  if (ctx->ipc_mode) {  // one-sided: K/V rows were stored by the QKV epilogue
    if (ctx->probe) return STADI_OK;    // compute-only probe: nothing leaves the rank
    const bool nb = S.kind == US_HALO;  // halos go to the row neighbours only
    if (S.kind == US_KV) {
      ctx->exch_bytes += bytes * ctx->ipc->peers.size();
    } else {
      ST(ipc_war_wait(ctx, S.id, ver, nb, s));
      ST(ipc_push(ctx, (const char *)S.slot[li][par] + off, (size_t)bytes, nb, s));
    }
    return ipc_ready(ctx, S.id, ver, nb, s);
  }
  if (!ctx->nccl) {
    for (size_t lj = 0; lj < ctx->ranks.size(); ++lj) {
      if ((int)lj == li) continue;
      CK(cudaMemcpyAsync((char *)S.slot[lj][par] + off, (char *)S.slot[li][par] + off, bytes,
                         cudaMemcpyDeviceToDevice, s));
      ctx->exch_bytes += bytes;
    }
    return STADI_OK;
  }
  CK(cudaEventRecord(ctx->ev_ready, s));
  CK(cudaStreamWaitEvent(ctx->comm, ctx->ev_ready, 0));
  char *base = (char *)S.slot[li][par];
  if (S.kind == US_KV) {
    CKN(nccl().GroupStart());
    for (size_t k = 0; k < U->inc.size(); ++k) {
      int64_t o2, b2;
      seg(U->inc[k], &o2, &b2);
      CKN(nccl().Broadcast(base + o2, base + o2, (size_t)b2, ncclUint8, (int)k, ctx->sub_comm,
                           ctx->comm));
    }
    CKN(nccl().GroupEnd());
  } else {
    CKN(nccl().AllGather(base + off, base, (size_t)bytes, ncclUint8, ctx->sub_comm, ctx->comm));
  }
  CK(cudaEventRecord(S.ev[par], ctx->comm));
  S.used[par] = true;
  ctx->exch_bytes += bytes;
  return STADI_OK;
}

stadi_status u_wait(stadi_ctx *ctx, USite &S, int ver, cudaStream_t s) {
  if (ctx->ipc_mode && !ctx->probe && ver >= 0)
    return ipc_read_wait(ctx, S.id, ver, S.kind == US_HALO, s);
  if (!ctx->nccl || ver < 0) return STADI_OK;
  if (S.used[ver & 1])
    CK(timed(ctx, STADI_KCLASS_XWAIT, 0.0, 0.0, s,
             [&] { return cudaStreamWaitEvent(s, S.ev[ver & 1], 0); }));
  return STADI_OK;
}

// IPC: after the consumer of site S, tell the sources this rank finished the step.
stadi_status u_done(stadi_ctx *ctx, USite &S, cudaStream_t s) {
  if (!ctx->ipc_mode || ctx->probe) return STADI_OK;
  return ipc_read_done(ctx, S.id, (uint32_t)ctx->ipc_idx + 1, S.kind == US_HALO, s);
}

// ------------------------------------------------------------------ program builder
struct UBuilder {
  stadi_ctx *ctx;
  UNetState *U;
  int li;
  URank *R;
  const Dims &m;
  int Bm;
  size_t esz;
  UBuilder(stadi_ctx *c, int l)
      : ctx(c), U(c->un.get()), li(l), R(&c->un->ranks[l]), m(c->dm), Bm(c->dm.B), esz(c->esz) {}

  void need(int id, size_t bytes) {
    if ((int)R->size.size() <= id) {
      R->size.resize(id + 1, 0);
      R->buf.resize(id + 1, nullptr);
    }
    R->size[id] = std::max(R->size[id], bytes);
  }
  int new_buf(size_t bytes) {
    const int id = (int)std::max<size_t>(R->size.size(), UB_COUNT);
    need(id, bytes);
    return id;
  }
  // buffer pointer at run time (allocated after the program is built)
  std::function<void *()> P(int id) {
    URank *RR = R;
    return [RR, id] { return RR->buf[id]; };
  }
  const Rank &rank() const { return ctx->ranks[li]; }
  // halo rows of this band that lie on the image edge (always zero): bit 0 top, bit 1 bottom
  int edge_halos() const {
    return (rank().row_begin == 0 ? 1 : 0) |
           (rank().row_begin + rank().rows == (int)m.lat_h ? 2 : 0);
  }
  int rows(int l) const { return rank().rows >> l; }
  int width(int l) const { return m.lat_w >> l; }
  int64_t M(int l) const { return (int64_t)rows(l) * width(l) * Bm; }
  void op(UOp f) { R->prog.push_back(std::move(f)); }
  void *wT(const std::string &n) { return U->wt.at(n); }
  float *wF(const std::string &n) { return U->wf.at(n); }

  int add_site(int kind, int level, int C, int64_t seg_bytes) {
    USite S;
    S.id = (int)U->sites.size();
    S.kind = kind;
    S.level = level;
    S.C = C;
    S.seg_bytes = seg_bytes;
    U->sites.push_back(std::move(S));
    return (int)U->sites.size() - 1;
  }
  // Sites are enumerated identically by every hosted rank: the first builder
  // creates them, later builders look them up by running index.
  int site_counter = 0;
  int site(int kind, int level, int C, int64_t seg_bytes) {
    const int id = site_counter++;
    if (id < (int)U->sites.size()) return id;
    return add_site(kind, level, C, seg_bytes);
  }

  // ---- GroupNorm (exchange site) of X [level l, C] into dst (padded or plain)
  void groupnorm(int x, int l, int C, const std::string &p, float eps, int act, int dst,
                 bool pad) {
    const int B = Bm;
    const int h = rows(l), W = width(l);
    const int sid = site(US_GN, l, C, (int64_t)B * 32 * 2 * 8);
    need(UB_GNS, (size_t)B * 32 * 2 * 8);
    need(dst, (size_t)(pad ? (int64_t)(h + 2) * (W + 2) * B : M(l)) * C * esz);
    auto X = P(x), G = P(UB_GNS), D = P(dst);
    stadi_ctx *c = ctx;
    const int me = li;
    const int64_t Ml = M(l);
    const double n_total = (double)(m.lat_h >> l) * W * (C / 32);
    const float *gw = wF(p + ".w"), *gb = wF(p + ".b");
    const int zh = pad ? edge_halos() : 0;
    op([=](const stadi_step_t &st, cudaStream_t s) -> stadi_status {  // publish
      stadi_ctx *ctx = c;
      USite &S = ctx->un->sites[sid];
      const int pos = inc_pos(ctx->un.get(), ctx->ranks[me].g);
      // own fresh partials straight into the read slot (R14) and, when it differs,
      // the publish slot: the kernel's last block writes all copies
      if (st.pub_ver != st.read_ver) ST(u_wait(ctx, S, st.read_ver, s));
      const int64_t off = pos * S.seg_bytes;
      double *rd = (double *)((char *)S.slot[me][st.read_ver & 1] + off);
      double *pb = (st.pub_ver >= 0 && st.pub_ver != st.read_ver)
                       ? (double *)((char *)S.slot[me][st.pub_ver & 1] + off)
                       : nullptr;
      CK(timed(ctx, STADI_KCLASS_NORM, 0.0, (double)Ml * C * 4, s, [&] {
        return gn_partials((const float *)X(), Ml, B, C, (double *)G(), ctx->un->gn_ws,
                           ctx->un->gn_ticket, s, rd, pb);
      }));
      if (st.pub_ver >= 0) ST(u_publish(ctx, S, me, st.pub_ver, s));
      return STADI_OK;
    });
    op([=](const stadi_step_t &st, cudaStream_t s) -> stadi_status {  // consume
      stadi_ctx *ctx = c;
      USite &S = ctx->un->sites[sid];
      if (st.pub_ver == st.read_ver) ST(u_wait(ctx, S, st.read_ver, s));
      const int G_ = (int)ctx->un->inc.size();
      CK(timed(ctx, STADI_KCLASS_NORM, 0.0, (double)Ml * C * (4 + esz_of(ctx)), s, [&] {
        const double *stats = (const double *)S.slot[me][st.read_ver & 1];
        if (ctx->dtype == STADI_DTYPE_BF16)
          return gn_apply<bf16>((const float *)X(), h, W, B, C, stats, G_, n_total, gw, gb, eps,
                                act, pad ? 1 : 0, (bf16 *)D(), s, zh);
        return gn_apply<float>((const float *)X(), h, W, B, C, stats, G_, n_total, gw, gb, eps,
                               act, pad ? 1 : 0, (float *)D(), s, zh);
      }));
      return u_done(ctx, S, s);
    });
  }
  static size_t esz_of(stadi_ctx *c) { return c->esz; }

  // plain cast of X into the padded conv input (Downsample / Upsample inputs)
  void cast_pad(int x, int l, int C) {
    const int B = Bm;
    const int h = rows(l), W = width(l);
    need(UB_PAD, (size_t)(h + 2) * (W + 2) * B * C * esz);
    auto X = P(x), D = P(UB_PAD);
    stadi_ctx *c = ctx;
    const int zh = edge_halos();
    op([=](const stadi_step_t &, cudaStream_t s) -> stadi_status {
      stadi_ctx *ctx = c;
      if (ctx->dtype == STADI_DTYPE_BF16)
        CK(gn_apply<bf16>((const float *)X(), h, W, B, C, nullptr, 0, 1.0, nullptr, nullptr, 0.f,
                          0, 1, (bf16 *)D(), s, zh));
      else
        CK(gn_apply<float>((const float *)X(), h, W, B, C, nullptr, 0, 1.0, nullptr, nullptr,
                           0.f, 0, 1, (float *)D(), s, zh));
      return STADI_OK;
    });
  }

  // ---- 3x3 conv of the padded input (level l, C channels) with halo exchange.
  // mode 0 stride 1, 1 stride 2, 2 upsample x2.  Output fp32 X (EPI_CONV):
  // out = conv + bias (+ temb projection of ResBlock `temb`) (+ res).
  void conv3x3(int l, int C, int mode, const std::string &w, int cout, int out, int res,
               const std::string &temb, int epi = EPI_CONV, int ldo = 0) {
    const int B = Bm;
    const int h = rows(l), W = width(l);
    const int64_t rowe = (int64_t)W * B * C;  // elements of one interior row
    const int sid = site(US_HALO, l, C, 2 * rowe * (int64_t)esz);
    const int lo = mode == 1 ? l + 1 : (mode == 2 ? l - 1 : l);
    const int64_t Mo = (int64_t)rows(lo) * width(lo) * B;
    const int64_t kp = rup64(9 * C);
    const int ncols = ldo ? ldo : cout;
    const int wb = W * B;
    // implicit GEMM (no im2col buffer): stride 1 and stride 2 straight from the padded
    // input; the upsample conv as a stride-1 conv over the nearest-x2 upsampled input
    (void)wb;
    const bool implicit =
        ctx->dtype == STADI_DTYPE_BF16 && !conv_implicit_disabled() &&
        (mode == 2 ? tc_conv_implicit_ok(2 * h, 2 * W, B, C, ncols, 0)
                   : tc_conv_implicit_ok(h, W, B, C, ncols, mode));
    need(UB_PAD, (size_t)(h + 2) * (W + 2) * B * C * esz);
    if (!implicit) need(UB_COL, (size_t)(Mo * kp) * esz);
    if (implicit && mode == 2) need(UB_UPS, (size_t)(2 * h + 2) * (2 * W + 2) * B * C * esz);
    need(out, (size_t)(Mo * ncols) * 4);
    auto D = P(UB_PAD), A = P(UB_COL), O = P(out), UP = P(UB_UPS);
    std::function<void *()> Rs = res >= 0 ? P(res) : std::function<void *()>();
    stadi_ctx *c = ctx;
    const int me = li;
    void *wt = wT(w);
    const float *bias = wF(w.substr(0, w.size() - 1) + "b");
    const int toff = temb.empty() ? -1 : U->temb_off.at(temb);
    const bool top = rank().row_begin == 0;
    const bool bottom = rank().row_begin + rank().rows == (int)m.lat_h;
    op([=](const stadi_step_t &st, cudaStream_t s) -> stadi_status {  // publish own rows
      stadi_ctx *ctx = c;
      USite &S = ctx->un->sites[sid];
      const int pos = inc_pos(ctx->un.get(), ctx->ranks[me].g);
      if (st.pub_ver != st.read_ver) ST(u_wait(ctx, S, st.read_ver, s));
      if (st.pub_ver < 0) return STADI_OK;
      if (top && bottom) return u_publish(ctx, S, me, st.pub_ver, s);  // no neighbour reads
      // own boundary rows -> own segment of the publish slot (the consumer reads
      // only the neighbours' rows, so the read slot needs no own copy).  The last
      // send from this parity (version pub - 2) completed before the read wait of
      // the previous round (or of the previous fresh step).
      const size_t rb = (size_t)rowe * ctx->esz;
      const char *first = (const char *)D() + ((size_t)1 * (W + 2) + 1) * B * C * ctx->esz;
      const char *last = (const char *)D() + ((size_t)h * (W + 2) + 1) * B * C * ctx->esz;
      char *sg = (char *)S.slot[me][st.pub_ver & 1] + pos * S.seg_bytes;
      CK(cudaMemcpyAsync(sg, first, rb, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(sg + rb, last, rb, cudaMemcpyDeviceToDevice, s));
      ST(u_publish(ctx, S, me, st.pub_ver, s));
      return STADI_OK;
    });
    op([=](const stadi_step_t &st, cudaStream_t s) -> stadi_status {  // consume + conv
      stadi_ctx *ctx = c;
      UNetState *U = ctx->un.get();
      USite &S = ctx->un->sites[sid];
      if (st.pub_ver == st.read_ver) ST(u_wait(ctx, S, st.read_ver, s));
      const int pos = inc_pos(U, ctx->ranks[me].g);
      const size_t rb = (size_t)rowe * ctx->esz;
      const char *sl = (const char *)S.slot[me][st.read_ver & 1];
      // the neighbours' boundary rows (or zeros at the image edge) into the two halo
      // rows, corner cells zero: one kernel
      const void *above = top ? nullptr : sl + (pos - 1) * S.seg_bytes + rb;
      const void *below = bottom ? nullptr : sl + (pos + 1) * S.seg_bytes;
      // a band without neighbours: its producer (GN apply / cast / latent pad) already
      // zeroed both image-edge halo rows (zero_halo)
      if (top && bottom) {
      } else if (ctx->dtype == STADI_DTYPE_BF16) {
        CK(halo_fill<bf16>((bf16 *)D(), h, W, B, C, (const bf16 *)above, (const bf16 *)below, s));
      } else {
        CK(halo_fill<float>((float *)D(), h, W, B, C, (const float *)above, (const float *)below,
                            s));
      }
      ST(u_done(ctx, S, s));
      EpiParams ep{};
      ep.B = B;
      ep.bias = bias;
      ep.out = O();
      ep.ldo = ncols;
      if (Rs) {
        ep.res = (float *)Rs();
        ep.ldr = cout;
      }
      if (toff >= 0) {
        ep.gate = U->temb_all + (int64_t)st.m * B * U->temb_total + toff;
        ep.gate_bstride = U->temb_total;
      }
      if (implicit) {  // tcgen05 implicit GEMM straight from the padded input
        ep.ws = ctx->splitk_ws;
        ep.ws_elems = ctx->splitk_elems;
        const bf16 *src = (const bf16 *)D();
        int hc = h, Wc = W, mc = mode;
        if (mode == 2) {
          CK(upsample_pad<bf16>((const bf16 *)D(), h, W, B, C, (bf16 *)UP(), s));
          src = (const bf16 *)UP();
          hc = 2 * h;
          Wc = 2 * W;
          mc = 0;
        }
        CK(timed(ctx, STADI_KCLASS_GEMM, 2.0 * Mo * ncols * kp, 0.0, s, [&] {
          return tc_conv3x3_bf16(src, (const bf16 *)wt, hc, Wc, B, C, ncols, epi, ep,
                                 std::max(1, ctx->num_sms - ctx->emu_ctas), s, mc);
        }));
        return STADI_OK;
      }
      if (ctx->dtype == STADI_DTYPE_BF16)
        CK(im2col<bf16>((const bf16 *)D(), h, W, B, C, mode, (int)kp, (bf16 *)A(), s));
      else
        CK(im2col<float>((const float *)D(), h, W, B, C, mode, (int)kp, (float *)A(), s));
      CK(gemm(ctx, A(), wt, (int)Mo, ncols, (int)kp, epi, ep, s));
      return STADI_OK;
    });
  }

  // ---- generic GEMM op: out = epi(A[M, K] . W[N, K]^T)
  void linear(int a, int64_t Mr, int K, const std::string &w, const float *bias, int N, int epi,
              int out, int ldo, int res = -1, size_t out_esz = 4) {
    const int B = Bm;
    need(out, (size_t)(Mr * ldo) * out_esz);
    auto Ap = P(a), O = P(out);
    std::function<void *()> Rs = res >= 0 ? P(res) : std::function<void *()>();
    stadi_ctx *c = ctx;
    void *wt = wT(w);
    op([=](const stadi_step_t &, cudaStream_t s) -> stadi_status {
      stadi_ctx *ctx = c;
      EpiParams ep{};
      ep.B = B;
      ep.bias = bias;
      if (epi == EPI_RES) {
        ep.res = (float *)O();
        ep.ldr = ldo;
      } else {
        ep.out = O();
        ep.ldo = ldo;
        if (Rs) {
          ep.res = (float *)Rs();
          ep.ldr = ldo;
        }
      }
      CK(gemm(ctx, Ap(), wt, (int)Mr, N, K, epi, ep, s));
      return STADI_OK;
    });
  }

  // plain cast X -> T [M, C] (operand of a 1x1 conv / projection)
  void cast_plain(int x, int l, int C, int dst) {
    const int B = Bm;
    const int h = rows(l), W = width(l);
    need(dst, (size_t)M(l) * C * esz);
    auto X = P(x), D = P(dst);
    stadi_ctx *c = ctx;
    op([=](const stadi_step_t &, cudaStream_t s) -> stadi_status {
      stadi_ctx *ctx = c;
      if (ctx->dtype == STADI_DTYPE_BF16)
        CK(gn_apply<bf16>((const float *)X(), h, W, B, C, nullptr, 0, 1.0, nullptr, nullptr, 0.f,
                          0, 0, (bf16 *)D(), s));
      else
        CK(gn_apply<float>((const float *)X(), h, W, B, C, nullptr, 0, 1.0, nullptr, nullptr,
                           0.f, 0, 0, (float *)D(), s));
      return STADI_OK;
    });
  }

  // ---- ResBlock(x: level l, cin) -> out (cout)
  void resblock(int x, int l, int cin, int cout, const std::string &p, int out) {
    groupnorm(x, l, cin, p + "norm1", 1e-5f, 1, UB_PAD, true);
    conv3x3(l, cin, 0, p + "conv1.w", cout, UB_H1, -1, p);
    groupnorm(UB_H1, l, cout, p + "norm2", 1e-5f, 1, UB_PAD, true);
    int res = x;
    if (cin != cout) {  // 1x1 conv shortcut
      cast_plain(x, l, cin, UB_NB);
      linear(UB_NB, M(l), cin, p + "skip.w", wF(p + "skip.b"), cout, EPI_F32, UB_SK, cout);
      res = UB_SK;
    }
    conv3x3(l, cout, 0, p + "conv2.w", cout, out, res, "");
  }

  // ---- Transformer2D on x (level l, C channels), in place: x += proj_out(...)
  void transformer(int x, int l, int C, int depth, int heads, const std::string &p) {
    const int B = Bm;
    const int64_t Ml = M(l);
    const int W = width(l), h = rows(l);
    groupnorm(x, l, C, p + "norm", 1e-6f, 0, UB_NB, false);
    linear(UB_NB, Ml, C, p + "proj_in.w", wF(p + "proj_in.b"), C, EPI_F32, UB_TY, C);
    stadi_ctx *c = ctx;
    const int me = li;
    const int hd = C / heads;
    (void)hd;
    for (int k = 0; k < depth; ++k) {
      const std::string q = p + "blk" + std::to_string(k) + ".";
      ln(UB_TY, Ml, C, q + "ln1", UB_NB);
      // KV site: QKV GEMM scatters own K/V rows into the slots (publish op)
      const int sid = site(US_KV, l, C, (int64_t)B * 2 * C * esz);
      need(UB_Q, (size_t)Ml * C * esz);
      need(UB_O, (size_t)Ml * C * esz);
      auto NB = P(UB_NB), Q = P(UB_Q), O = P(UB_O), TY = P(UB_TY);
      void *wqkv = wT(q + "attn1.qkv");
      const int64_t tok0 = (int64_t)(rank().row_begin >> l) * W;
      const int ntok = h * W;
      const int ntok_full = (m.lat_h >> l) * W;
      op([=](const stadi_step_t &st, cudaStream_t s) -> stadi_status {
        stadi_ctx *ctx = c;
        USite &S = ctx->un->sites[sid];
        if (st.pub_ver != st.read_ver) ST(u_wait(ctx, S, st.read_ver, s));
        const bool ipcx = ctx->ipc_mode && !ctx->probe && st.pub_ver >= 0;
        if (ipcx) ST(ipc_war_wait(ctx, S.id, st.pub_ver, false, s));
        EpiParams ep{};
        ep.B = B;
        ep.q = Q();
        ep.d = C;
        if (ipcx) {  // the all-gather fused into the epilogue: P2P stores to the peers
          ep.kv_peer = ipc_peer_slots(ctx, S.id, st.pub_ver & 1);
          ep.n_kv_peer = ep.kv_peer ? (int)ctx->ipc->peers.size() : 0;
        }
        ep.kv_a = S.slot[me][st.read_ver & 1];
        ep.kv_b = (st.pub_ver >= 0 && st.pub_ver != st.read_ver) ? S.slot[me][st.pub_ver & 1]
                                                                 : nullptr;
        ep.kv_row0 = tok0 * B;
        CK(gemm(ctx, NB(), wqkv, (int)Ml, 3 * C, C, EPI_QKV, ep, s));
        if (st.pub_ver >= 0) ST(u_publish(ctx, S, me, st.pub_ver, s));
        return STADI_OK;
      });
      void *wo = wT(q + "attn1.o");
      const float *bo = wF(q + "attn1.ob");
      op([=](const stadi_step_t &st, cudaStream_t s) -> stadi_status {
        stadi_ctx *ctx = c;
        USite &S = ctx->un->sites[sid];
        if (st.pub_ver == st.read_ver) ST(u_wait(ctx, S, st.read_ver, s));
        CK(attention_h(ctx, STADI_KCLASS_ATTN, Q(), S.slot[me][st.read_ver & 1], O(), ntok,
                       ntok_full, heads, C, s));
        ST(u_done(ctx, S, s));
        EpiParams ep{};
        ep.B = B;
        ep.bias = bo;
        ep.res = (float *)TY();
        ep.ldr = C;
        CK(gemm(ctx, O(), wo, (int)Ml, C, C, EPI_RES, ep, s));
        return STADI_OK;
      });
      // cross-attention to the text tokens (band-local; text K/V cached per request)
      ln(UB_TY, Ml, C, q + "ln2", UB_NB);
      linear(UB_NB, Ml, C, q + "attn2.q", nullptr, C, EPI_STORE, UB_Q, C, -1, esz);
      const int ti = U->tr_index.at(q + "attn2.");
      op([=](const stadi_step_t &, cudaStream_t s) -> stadi_status {
        stadi_ctx *ctx = c;
        CK(attention_h(ctx, STADI_KCLASS_XATTN, Q(), ctx->un->text_kv[ti], O(), ntok,
                       ctx->dm.txt_len, heads, C, s));
        return STADI_OK;
      });
      linear(UB_O, Ml, C, q + "attn2.o", wF(q + "attn2.ob"), C, EPI_RES, UB_TY, C);
      // GEGLU feed-forward
      ln(UB_TY, Ml, C, q + "ln3", UB_NB);
      linear(UB_NB, Ml, C, q + "ff1.w", wF(q + "ff1.b"), 8 * C, EPI_GEGLU, UB_FF, 4 * C, -1, esz);
      linear(UB_FF, Ml, 4 * C, q + "ff2.w", wF(q + "ff2.b"), C, EPI_RES, UB_TY, C);
    }
    cast_plain(UB_TY, l, C, UB_NB);
    linear(UB_NB, Ml, C, p + "proj_out.w", wF(p + "proj_out.b"), C, EPI_RES, x, C);
  }

  void ln(int x, int64_t Mr, int C, const std::string &p, int dst) {
    const int B = Bm;
    need(dst, (size_t)Mr * C * esz);
    auto X = P(x), D = P(dst);
    stadi_ctx *c = ctx;
    const float *sc = wF(p + ".w"), *sh = wF(p + ".b");
    op([=](const stadi_step_t &, cudaStream_t s) -> stadi_status {
      stadi_ctx *ctx = c;
      const double bytes = (double)Mr * C * (4 + ctx->esz);
      CK(timed(ctx, STADI_KCLASS_NORM, 0.0, bytes, s, [&] {
        if (ctx->dtype == STADI_DTYPE_BF16)
          return ln_modulate<bf16>((const float *)X(), (bf16 *)D(), (int)Mr, C, B, sh, sc, 0, 1,
                                   s, 1e-5f);
        return ln_modulate<float>((const float *)X(), (float *)D(), (int)Mr, C, B, sh, sc, 0, 1,
                                  s, 1e-5f);
      }));
      return STADI_OK;
    });
  }

  // ---- the whole band forward + sampler (mirrors oracle/unet.py band_forward)
  void build() {
    const int B = Bm;
    const int L = m.levels();
    const int C0 = m.ch[0];
    // conv_in: latent band -> padded input (halo site on the latent rows, R15)
    {
      const int h = rows(0), W = width(0);
      need(UB_PAD, (size_t)(h + 2) * (W + 2) * B * m.c_in * esz);
      auto D = P(UB_PAD);
      stadi_ctx *c = ctx;
      const int me = li;
      const int zh = edge_halos();
      op([=](const stadi_step_t &, cudaStream_t s) -> stadi_status {
        stadi_ctx *ctx = c;
        const float *xb = ctx->ranks[me].x_band;
        if (ctx->dtype == STADI_DTYPE_BF16)
          CK(latent_pad<bf16>(xb, h, W, ctx->dm.c_in, B, (bf16 *)D(), s, zh));
        else
          CK(latent_pad<float>(xb, h, W, ctx->dm.c_in, B, (float *)D(), s, zh));
        return STADI_OK;
      });
    }
    std::vector<std::pair<int, int>> skips;  // (buffer, channels)
    int cur = new_buf((size_t)M(0) * C0 * 4);
    conv3x3(0, m.c_in, 0, "conv_in.w", C0, cur, -1, "");
    skips.push_back({cur, C0});
    int prev = C0;
    for (int i = 0; i < L; ++i) {
      const int c = m.ch[i];
      for (int j = 0; j < m.nres; ++j) {
        const std::string p = "down" + std::to_string(i) + ".res" + std::to_string(j) + ".";
        const int out = new_buf((size_t)M(i) * c * 4);
        resblock(cur, i, j == 0 ? prev : c, c, p, out);
        cur = out;
        if (m.tdepth[i])
          transformer(cur, i, c, m.tdepth[i], m.heads[i],
                      "down" + std::to_string(i) + ".attn" + std::to_string(j) + ".");
        skips.push_back({cur, c});
      }
      if (i < L - 1) {
        const int out = new_buf((size_t)M(i + 1) * c * 4);
        cast_pad(cur, i, c);
        conv3x3(i, c, 1, "down" + std::to_string(i) + ".ds.w", c, out, -1, "");
        cur = out;
        skips.push_back({cur, c});
      }
      prev = c;
    }
    const int cm = m.ch[L - 1];
    resblock(cur, L - 1, cm, cm, "mid.res0.", UB_H);
    transformer(UB_H, L - 1, cm, m.mid_depth, m.heads[L - 1], "mid.attn.");
    resblock(UB_H, L - 1, cm, cm, "mid.res1.", UB_H);
    cur = UB_H;
    int ccur = cm;
    for (const auto &u : unet_up_io(m)) {
      const int l = L - 1 - u.i;
      for (size_t j = 0; j < u.res.size(); ++j) {
        const auto sk = skips.back();
        skips.pop_back();
        // concat [cur | skip] -> CAT
        need(UB_CAT, (size_t)M(l) * (ccur + sk.second) * 4);
        {
          auto A = P(cur), Bp = P(sk.first), D = P(UB_CAT);
          const int ca = ccur, cb = sk.second;
          const int64_t Ml = M(l);
          stadi_ctx *c = ctx;
          op([=](const stadi_step_t &, cudaStream_t s) -> stadi_status {
            stadi_ctx *ctx = c;
            CK(concat_channels((const float *)A(), ca, (const float *)Bp(), cb, Ml, (float *)D(),
                               s));
            return STADI_OK;
          });
        }
        const std::string p = "up" + std::to_string(u.i) + ".res" + std::to_string(j) + ".";
        resblock(UB_CAT, l, ccur + sk.second, u.c, p, UB_H);
        cur = UB_H;
        ccur = u.c;
        if (u.depth)
          transformer(UB_H, l, u.c, u.depth, u.heads,
                      "up" + std::to_string(u.i) + ".attn" + std::to_string(j) + ".");
      }
      if (u.i < L - 1) {  // nearest x2 + conv; the input H is dead once cast into PAD
        cast_pad(UB_H, l, u.c);
        conv3x3(l, u.c, 2, "up" + std::to_string(u.i) + ".us.w", u.c, UB_H, -1, "");
      }
    }
    // out: GN -> SiLU -> conv (N padded to 64) -> eps [M0, 64] fp32
    groupnorm(UB_H, 0, C0, "out.norm", 1e-5f, 1, UB_PAD, true);
    conv3x3(0, C0, 0, "out.conv.w", 64, UB_EPS, -1, "", EPI_F32, 64);
    // sampler: CFG + Eq. 3 on the fp32 band
    {
      auto E = P(UB_EPS);
      stadi_ctx *c = ctx;
      const int me = li;
      const int h = rows(0), W = width(0);
      op([=](const stadi_step_t &st, cudaStream_t s) -> stadi_status {
        stadi_ctx *ctx = c;
        float A, Bc, Cz, c1, c2;
        sampler_coeffs(ctx, st.t, st.t_prev, &A, &Bc, &Cz);
        const auto &sc = ctx->ranks[me].sched;
        int idx = 0;
        while (idx < (int)sc.size() && sc[idx].m != st.m) ++idx;
        dpm2m_coeffs(ctx, sc, idx, &c1, &c2);
        const double sb = (double)h * W * 4 * 8 + (double)h * W * B * 64 * 4;
        CK(timed(ctx, STADI_KCLASS_SAMPLER, 0.0, sb, s, [&] {
          return sampler_update(ctx->ranks[me].x_band, (const float *)E(), h, W, ctx->dm.c_in, 1,
                                4, 64, B, ctx->dm.guidance, A, Bc, Cz, ctx->ddpm_seed, ctx->seed_dev,
                                st.m, ctx->ranks[me].row_begin, s, ctx->ranks[me].hist, c1, c2);
        }));
        return STADI_OK;
      });
    }
  }
};

}  // namespace

namespace {

// ------------------------------------------------------------------ plan / request / step
void unet_free_plan(stadi_ctx *ctx) {
  UNetState *U = ctx->un.get();
  if (!U) return;
  for (auto &R : U->ranks)
    for (void *p : R.buf) pfree(ctx, p);
  for (auto &S : U->sites) {
    if (!ctx->ipc_mode)  // IPC: slots live in the persistent exchange arena
      for (auto &pr : S.slot) {
        pfree(ctx, pr[0]);
        pfree(ctx, pr[1]);
      }
    for (auto e : S.ev)
      if (e) cudaEventDestroy(e);
  }
  U->ranks.clear();
  U->sites.clear();
  U->inc.clear();
}

// Build every hosted rank's program, then allocate its buffers and the sites' slots.
stadi_status unet_set_plan(stadi_ctx *ctx) {
  UNetState *U = ctx->un.get();
  const Dims &m = ctx->dm;
  for (uint32_t g = 0; g < ctx->plan.n_gpus; ++g)
    if (ctx->plan.tier[g]) U->inc.push_back((int)g);
  U->ranks.assign(ctx->ranks.size(), URank{});
  for (size_t li = 0; li < ctx->ranks.size(); ++li) {
    UBuilder b(ctx, (int)li);
    b.build();
  }
  for (auto &R : U->ranks)
    for (size_t i = 0; i < R.size.size(); ++i)
      if (R.size[i]) {
        CK(pmalloc(ctx, &R.buf[i], R.size[i]));
        CK(cudaMemsetAsync(R.buf[i], 0, R.size[i], ctx->astream));
      }
  const int n_inc = (int)U->inc.size();
  if (ctx->ipc_mode) {  // every site's two slots in the IPC arena (identical layout on all ranks)
    ipc_layout_begin(ctx);
    IpcState &I = *ctx->ipc;
    for (auto &S : U->sites) {
      const int64_t bytes = S.kind == US_KV ? (int64_t)(m.lat_h >> S.level) *
                                                  (m.lat_w >> S.level) * S.seg_bytes
                                            : n_inc * S.seg_bytes;
      for (int par = 0; par < 2; ++par) I.site_off[par].push_back(ipc_reserve(ctx, bytes));
    }
    ST(ipc_commit(ctx, (int)U->sites.size()));
    for (auto &S : U->sites) {
      S.slot.assign(ctx->ranks.size(), {nullptr, nullptr});
      for (auto &pr : S.slot)
        for (int par = 0; par < 2; ++par) pr[par] = I.arena + I.site_off[par][S.id];
    }
    CK(cudaStreamSynchronize(ctx->astream));
    return STADI_OK;
  }
  for (auto &S : U->sites) {
    int64_t bytes = S.kind == US_KV
                        ? (int64_t)(m.lat_h >> S.level) * (m.lat_w >> S.level) * S.seg_bytes
                        : n_inc * S.seg_bytes;
    S.slot.assign(ctx->ranks.size(), {nullptr, nullptr});
    for (auto &pr : S.slot)
      for (int par = 0; par < 2; ++par) {
        CK(pmalloc(ctx, &pr[par], std::max<int64_t>(bytes, 16)));
        CK(cudaMemsetAsync(pr[par], 0, std::max<int64_t>(bytes, 16), ctx->astream));
      }
    if (ctx->nccl)
      for (auto &e : S.ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  CK(cudaStreamSynchronize(ctx->astream));
  return STADI_OK;
}

// Per-request conditioning: time embedding of every fast-grid timestep (+ the
// SDXL micro-conditioning embedding), every ResBlock's time projection in one
// GEMM, and every transformer block's text K/V (cached for the request).
stadi_status unet_begin(stadi_ctx *ctx, const stadi_cond *cond, cudaStream_t s) {
  UNetState *U = ctx->un.get();
  const Dims &m = ctx->dm;
  const int nt = (int)ctx->plan.m_base, B = m.B, C0 = m.ch[0], td = m.temb_dim();
  const int an = 6 * 256 + m.pooled_dim;
  if (m.add_embed && !cond->pooled)
    return ctx_fail(ctx, STADI_EINVAL, "conditioning missing (pooled text embedding)");
  if (U->cap_nt < nt) {
    CK(quiesce(ctx));
    for (void *p : {(void *)U->tfeat, (void *)U->t1, (void *)U->temb, (void *)U->tembB,
                    (void *)U->temb_all, U->tsilu})
      pfree(ctx, p);
    CK(pmalloc(ctx, &U->tfeat, (size_t)nt * C0 * 4));
    CK(pmalloc(ctx, &U->t1, (size_t)nt * td * 4));
    CK(pmalloc(ctx, &U->temb, (size_t)nt * td * 4));
    CK(pmalloc(ctx, &U->tembB, (size_t)nt * B * td * 4));
    CK(pmalloc(ctx, &U->tsilu, (size_t)nt * B * td * ctx->esz));
    CK(pmalloc(ctx, &U->temb_all, (size_t)nt * B * U->temb_total * 4));
    CK(cudaStreamSynchronize(ctx->astream));
    U->cap_nt = nt;
    free_graphs(ctx);  // captured steps reference the old time-embedding buffers
    ctx->tfreq_nt = 0;
  }
  if (!U->addin) {
    CK(dalloc(ctx, &U->addin, (size_t)B * std::max(an, 64) * 4));
    CK(dalloc(ctx, &U->aug1, (size_t)B * td * 4));
    CK(dalloc(ctx, &U->aug, (size_t)B * td * 4));
  }
  if (ctx->tfreq_nt != nt) {  // diffusers Timesteps(C0, flip_sin_to_cos, shift 0), fp64 host
    std::vector<float> tf((size_t)nt * C0);
    const int ratio = 1000 / nt, half = C0 / 2;
    for (int i = 0; i < nt; ++i) {
      const double t = ratio * (nt - 1 - i) + 1;  // fast grid (R18)
      for (int k = 0; k < half; ++k) {
        const double f = std::exp(-std::log(10000.0) * k / half);
        tf[(size_t)i * C0 + k] = (float)std::cos(t * f);
        tf[(size_t)i * C0 + half + k] = (float)std::sin(t * f);
      }
    }
    const void *st = stage_h2d(ctx, tf.data(), tf.size() * 4);
    if (!st) return ctx_fail(ctx, STADI_ENOMEM, "host staging exhausted");
    CK(cudaMemcpyAsync(U->tfeat, st, tf.size() * 4, cudaMemcpyHostToDevice, s));
    ctx->tfreq_nt = nt;
  }
  EpiParams ep{};
  ep.B = 1;
  ep.bias = U->wf.at("time.b1");
  ep.out = U->t1;
  ep.ldo = td;
  CK(simt_gemm<float>(U->tfeat, U->wf.at("time.w1"), nt, td, C0, EPI_F32, ep, s));
  CK(silu_inplace(U->t1, (long)nt * td, s));
  ep.bias = U->wf.at("time.b2");
  ep.out = U->temb;
  CK(simt_gemm<float>(U->t1, U->wf.at("time.w2"), nt, td, td, EPI_F32, ep, s));
  const float *aug = nullptr;
  if (m.add_embed) {  // [pooled | sinusoid256(time_ids)] -> Linear -> SiLU -> Linear
    std::vector<float> tid((size_t)B * 1536);
    for (int b = 0; b < B; ++b)
      for (int j = 0; j < 6; ++j) {
        const double t = cond->time_ids ? cond->time_ids[b * 6 + j] : m.time_ids[j];
        for (int k = 0; k < 128; ++k) {
          const double f = std::exp(-std::log(10000.0) * k / 128.0);
          tid[(size_t)b * 1536 + j * 256 + k] = (float)std::cos(t * f);
          tid[(size_t)b * 1536 + j * 256 + 128 + k] = (float)std::sin(t * f);
        }
      }
    const void *pl = stage_h2d(ctx, cond->pooled, (size_t)B * m.pooled_dim * 4);
    const void *ti = stage_h2d(ctx, tid.data(), tid.size() * 4);  // pinned copy of a temporary
    if (!pl || !ti) return ctx_fail(ctx, STADI_ENOMEM, "host staging exhausted");
    CK(cudaMemcpy2DAsync(U->addin, (size_t)an * 4, pl, (size_t)m.pooled_dim * 4,
                         (size_t)m.pooled_dim * 4, B, cudaMemcpyDefault, s));
    CK(cudaMemcpy2DAsync(U->addin + m.pooled_dim, (size_t)an * 4, ti, 1536 * 4, 1536 * 4, B,
                         cudaMemcpyDefault, s));
    ep.bias = U->wf.at("add.b1");
    ep.out = U->aug1;
    CK(simt_gemm<float>(U->addin, U->wf.at("add.w1"), B, td, an, EPI_F32, ep, s));
    CK(silu_inplace(U->aug1, (long)B * td, s));
    ep.bias = U->wf.at("add.b2");
    ep.out = U->aug;
    CK(simt_gemm<float>(U->aug1, U->wf.at("add.w2"), B, td, td, EPI_F32, ep, s));
    aug = U->aug;
  }
  {
    const long n = (long)nt * B * td;
    temb_combine_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(U->temb, aug, nt, B, td,
                                                                    U->tembB);
    ++g_launches;
    CK(cudaGetLastError());
  }
  if (ctx->dtype == STADI_DTYPE_BF16)
    CK(silu_cast<bf16>(U->tembB, (bf16 *)U->tsilu, (long)nt * B * td, s));
  else
    CK(silu_cast<float>(U->tembB, (float *)U->tsilu, (long)nt * B * td, s));
  ep = EpiParams{};
  ep.B = B;
  ep.bias = U->wf.at("temb_all.b");
  ep.out = U->temb_all;
  ep.ldo = U->temb_total;
  CK(gemm(ctx, U->tsilu, U->wt.at("temb_all.w"), nt * B, U->temb_total, td, EPI_F32, ep, s));
  // text tokens [B, L, Dt] -> [L, B, Dt] (token-major) -> per-block K|V
  const int L = m.txt_len, Dt = m.txt_dim;
  const int64_t Mt = (int64_t)L * B;
  if (!ctx->text_T) {
    CK(dalloc(ctx, &ctx->text_T, Mt * Dt * ctx->esz));
    CK(dalloc(ctx, &ctx->text_f, Mt * Dt * 4));
  }
  const float *txt = (const float *)stage_h2d(ctx, cond->text, (size_t)Mt * Dt * 4);
  if (!txt) return ctx_fail(ctx, STADI_ENOMEM, "host staging exhausted");
  for (int b = 0; b < B; ++b)
    CK(cudaMemcpy2DAsync(ctx->text_f + (size_t)b * Dt, (size_t)B * Dt * 4,
                         txt + (size_t)b * L * Dt, (size_t)Dt * 4, (size_t)Dt * 4, L,
                         cudaMemcpyDefault, s));
  if (ctx->dtype == STADI_DTYPE_BF16)
    CK(cast_f32<bf16>(ctx->text_f, (bf16 *)ctx->text_T, (long)(Mt * Dt), s));
  else
    CK(cudaMemcpyAsync(ctx->text_T, ctx->text_f, Mt * Dt * 4, cudaMemcpyDeviceToDevice, s));
  if (U->text_kv.empty()) {
    U->text_kv.assign(U->n_tr_blocks, nullptr);
    for (auto &kv : U->tr_index) {
      // channels of the block = rows of attn2.kv / 2
      int64_t C = 0;
      for (const auto &ts : ctx->man)
        if (ts.name == kv.first + "o") C = ts.rows;
      CK(dalloc(ctx, &U->text_kv[kv.second], Mt * 2 * C * ctx->esz));
    }
  }
  for (auto &kv : U->tr_index) {
    int64_t C = 0;
    for (const auto &ts : ctx->man)
      if (ts.name == kv.first + "o") C = ts.rows;
    EpiParams e2{};
    e2.B = B;
    e2.out = U->text_kv[kv.second];
    e2.ldo = (int)(2 * C);
    CK(gemm(ctx, ctx->text_T, U->wt.at(kv.first + "kv"), (int)Mt, (int)(2 * C), Dt, EPI_STORE, e2,
            s));
  }
  return STADI_OK;
}

// One program step: the programs of the phase's hosted ranks, op-index by
// op-index (layer lock-step in local mode; one rank in NCCL mode).
stadi_status unet_run_phase(stadi_ctx *ctx, const std::vector<Part> &phase, cudaStream_t s) {
  UNetState *U = ctx->un.get();
  if (phase.empty()) return STADI_OK;
  const size_t n = U->ranks[phase[0].li].prog.size();
  ctx->ipc_idx = phase[0].idx;  // IPC mode: one hosted rank; its step index (done counts)
  for (size_t i = 0; i < n; ++i)
    for (const Part &P : phase) ST(U->ranks[P.li].prog[i](P.st, s));
  return STADI_OK;
}

}  // namespace

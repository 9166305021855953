// IPC transport of the stale exchange (world > 1, STADI_TRANSPORT_IPC).  Included
// by runtime.cu (uses its context, error and timing helpers); not a separate
// translation unit.
//
// One process per rank on one node: ranks on different GPUs with peer access
// (NVLink / NVSwitch), or several processes sharing ONE GPU (how the multi-rank
// exchange is exercised on the single-GPU test box).  PAPER.md Alg. 1
// ("update buffer asynchronously ... all-gather") and L288 ("multiple
// asynchronous broadcast to emulate all_gather ... mask communication latency")
// are realised one-sided:
//  * every rank's exchange slots live in one device ARENA exported with CUDA IPC;
//    all ranks build identical slot layouts (same model, same plan), so a peer's
//    copy of slot s is peer_arena + (s - my_arena);
//  * K/V: the QKV GEMM epilogue stores the publish version's own rows straight
//    into every peer's slot (P2P stores: the all-gather is fused into the
//    producing GEMM, tile by tile); halo rows and GroupNorm partial sums (tiny)
//    are pushed with one peer copy each -- halos to the two NEIGHBOUR ranks only;
//  * completion is signalled with stream memory operations on 32-bit flags in the
//    receiver's arena (cuStreamWriteValue32 after the producer, with its implied
//    system-scope fence; cuStreamWaitValue32 GEQ before the consumer).  No SM
//    spins, no host round trip, and the ops are stream-ordered (and capturable).
// Per (site s, source i) at the reader:  ready[s][i] = last version i published + 1.
// Per (site s, reader j) at the writer:   done[s][j]  = number of steps j has
// finished reading site s.  Before version P overwrites slot P % 2 at reader j the
// writer waits until done[s][j] covers j's last read of a version <= P - 2 of that
// parity (computed from j's step table: the schedule is a pure function of the plan).
// Flags restart from 0 every request (stadi_begin zeroes them, then a flag barrier
// with a monotonic request counter orders every rank's reset before any new write),
// so the values a step writes and waits for are the same in every request and the
// per-step CUDA graphs stay valid.
// Host control plane (IPC handle and profile all-gathers): small files in a
// node-local directory (/dev/shm), namespaced by a 128-byte session id from rank 0.

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <fstream>
#include <sstream>
#include <thread>

namespace {

// ---------------------------------------------------------------- driver mem ops
struct MemOps {
  bool ok = false;
  CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
};
MemOps &memops() {
  static MemOps m = [] {
    MemOps o;
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      o.wait32 = reinterpret_cast<decltype(o.wait32)>(p);
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      o.write32 = reinterpret_cast<decltype(o.write32)>(p);
    o.ok = o.wait32 && o.write32;
    return o;
  }();
  return m;
}

struct IpcState {
  // control plane
  std::string dir, session;
  uint64_t rdv_seq = 0;
  std::string last_file;
  // arena: this rank's exchange slots, flags and the gather buffer
  char *arena = nullptr;
  size_t cap = 0;                  // allocated bytes (grows, never shrinks, see ipc_commit)
  size_t used = 0;                 // bytes reserved by the installed plan
  std::vector<char *> retired;     // outgrown arenas (freed at destroy: cudaFree syncs)
  std::vector<char *> peer;        // [world] peer arena bases (self: arena)
  std::vector<std::string> peer_handle;
  std::vector<char *> opened;      // replaced peer mappings (closed at destroy)
  uint32_t *probe = nullptr;       // scratch flag of the graph-capture probe
  size_t off_ready = 0, off_done = 0, off_gflag = 0, off_barrier = 0, off_gather = 0;
  int n_sites = 0;
  std::vector<size_t> site_off[2];  // [parity][site] slot offsets (DiT K/V and U-Net sites)
  void **peer_tab = nullptr;       // device [n_sites][2][n_peers] peer slot bases (QKV epilogue)
  std::vector<int> peers;          // included ranks other than me, row order
  std::vector<std::vector<uint32_t>> need;  // [g][ver] done-count reader g must reach
  uint32_t req = 0;                // requests begun (barrier value)
  bool graphs_ok = false;          // stream memory ops can be captured in CUDA graphs
  double wait_ms = 0;              // exchange-wait time of the last request (kernel timing on)
};

inline size_t al256(size_t x) { return (x + 255) / 256 * 256; }

std::string hexs(const uint8_t *b, int n) {
  static const char *d = "0123456789abcdef";
  std::string s;
  for (int i = 0; i < n; ++i) {
    s += d[b[i] >> 4];
    s += d[b[i] & 15];
  }
  return s;
}

// All-gather `mine` over the world through files (atomic rename; poll <= 300 s).
stadi_status rdv_allgather(stadi_ctx *ctx, const std::string &tag, const std::string &mine,
                           std::vector<std::string> &all) {
  IpcState &I = *ctx->ipc;
  const uint64_t seq = I.rdv_seq++;
  auto name = [&](int r) {
    return I.dir + "/stadi-" + I.session + "-" + std::to_string(seq) + "-" + tag + "-" +
           std::to_string(r);
  };
  {
    const std::string tmp = name(ctx->rank) + ".tmp";
    std::ofstream f(tmp, std::ios::binary);
    f.write(mine.data(), (std::streamsize)mine.size());
    f.close();
    if (!f || std::rename(tmp.c_str(), name(ctx->rank).c_str()) != 0)
      return ctx_fail(ctx, STADI_ESTATE, "IPC rendezvous: cannot write %s", tmp.c_str());
  }
  all.assign(ctx->world, std::string());
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < ctx->world; ++r) {
    for (;;) {
      std::ifstream f(name(r), std::ios::binary);
      if (f) {
        std::stringstream ss;
        ss << f.rdbuf();
        all[r] = ss.str();
        break;
      }
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300))
        return ctx_fail(ctx, STADI_ESTATE, "IPC rendezvous '%s': rank %d missing after 300 s",
                        tag.c_str(), r);
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  }
  // every rank wrote this round's file after reading the previous one: ours is dead
  if (!I.last_file.empty()) std::remove(I.last_file.c_str());
  I.last_file = name(ctx->rank);
  return STADI_OK;
}

// ------------------------------------------------------------------ flags
inline CUdeviceptr flag_at(char *base, size_t off, size_t idx) {
  return (CUdeviceptr)(base + off + 4 * idx);
}
#define CKD(call)                                                                          \
  do {                                                                                     \
    CUresult r_ = (call);                                                                  \
    if (r_ != CUDA_SUCCESS)                                                                \
      return ctx_fail(ctx, STADI_ECUDA, "%s:%d %s: CUresult %d", __FILE__, __LINE__, #call, \
                      (int)r_);                                                            \
  } while (0)

// Stream s blocks until the flag at (base, off, idx) >= v (no SM involved).
stadi_status ipc_wait(stadi_ctx *ctx, size_t off, size_t idx, uint32_t v, cudaStream_t s) {
  if (!v) return STADI_OK;
  IpcState &I = *ctx->ipc;
  CK(timed(ctx, STADI_KCLASS_XWAIT, 0.0, 0.0, s, [&] {
    return memops().wait32((CUstream)s, flag_at(I.arena, off, idx), v,
                           CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS
               ? cudaSuccess
               : cudaErrorUnknown;
  }));
  return STADI_OK;
}
// Write v to rank g's flag (after everything stream s did before: system fence).
stadi_status ipc_signal(stadi_ctx *ctx, int g, size_t off, size_t idx, uint32_t v,
                        cudaStream_t s) {
  IpcState &I = *ctx->ipc;
  CKD(memops().write32((CUstream)s, flag_at(I.peer[g], off, idx), v,
                       CU_STREAM_WRITE_VALUE_DEFAULT));
  return STADI_OK;
}

// Sources / targets of a site: every included peer, or the row neighbours (halos).
void ipc_partners(stadi_ctx *ctx, bool neighbours, std::vector<int> &out) {
  IpcState &I = *ctx->ipc;
  out.clear();
  if (!neighbours) {
    out = I.peers;
    return;
  }
  const int me = ctx->rank;
  int prev = -1, next = -1;
  bool seen = false;
  for (uint32_t g = 0; g < ctx->plan.n_gpus; ++g) {
    if (!ctx->plan.tier[g]) continue;
    if ((int)g == me) {
      seen = true;
      continue;
    }
    if (!seen) prev = (int)g;
    else if (next < 0) next = (int)g;
  }
  if (prev >= 0) out.push_back(prev);
  if (next >= 0) out.push_back(next);
}

// Writer side, before version `ver` of site `site` reaches the partners' slots:
// each partner must have finished its reads of the slot's previous content.
stadi_status ipc_war_wait(stadi_ctx *ctx, int site, int ver, bool neighbours, cudaStream_t s) {
  IpcState &I = *ctx->ipc;
  std::vector<int> tg;
  ipc_partners(ctx, neighbours, tg);
  for (int g : tg) {
    const uint32_t need = ver < (int)I.need[g].size() ? I.need[g][ver] : 0;
    ST(ipc_wait(ctx, I.off_done, (size_t)site * ctx->world + g, need, s));
  }
  return STADI_OK;
}
// Writer side, after the payload of `ver` reached the partners: ready = ver + 1.
stadi_status ipc_ready(stadi_ctx *ctx, int site, int ver, bool neighbours, cudaStream_t s) {
  std::vector<int> tg;
  ipc_partners(ctx, neighbours, tg);
  for (int g : tg)
    ST(ipc_signal(ctx, g, ctx->ipc->off_ready, (size_t)site * ctx->world + ctx->rank,
                  (uint32_t)ver + 1, s));
  return STADI_OK;
}
// Reader side, before the consumer of version `ver`.
stadi_status ipc_read_wait(stadi_ctx *ctx, int site, int ver, bool neighbours, cudaStream_t s) {
  std::vector<int> src;
  ipc_partners(ctx, neighbours, src);
  for (int g : src)
    ST(ipc_wait(ctx, ctx->ipc->off_ready, (size_t)site * ctx->world + g, (uint32_t)ver + 1, s));
  return STADI_OK;
}
// Reader side, after the consumer: this rank has finished `count` steps at the site.
stadi_status ipc_read_done(stadi_ctx *ctx, int site, uint32_t count, bool neighbours,
                           cudaStream_t s) {
  std::vector<int> src;
  ipc_partners(ctx, neighbours, src);
  for (int g : src)
    ST(ipc_signal(ctx, g, ctx->ipc->off_done, (size_t)site * ctx->world + ctx->rank, count, s));
  return STADI_OK;
}
// Peer copy of `bytes` at arena offset `off` (own segment) to the partners.
stadi_status ipc_push(stadi_ctx *ctx, const void *src, size_t bytes, bool neighbours,
                      cudaStream_t s) {
  IpcState &I = *ctx->ipc;
  const size_t off = (const char *)src - I.arena;
  std::vector<int> tg;
  ipc_partners(ctx, neighbours, tg);
  for (int g : tg) {
    CK(cudaMemcpyAsync(I.peer[g] + off, src, bytes, cudaMemcpyDeviceToDevice, s));
    ctx->exch_bytes += bytes;
  }
  return STADI_OK;
}

// ------------------------------------------------------------------ arena
// Plan install, phase 1: reserve the slots (offsets, identical on every rank).
size_t ipc_reserve(stadi_ctx *ctx, size_t bytes) {
  IpcState &I = *ctx->ipc;
  const size_t off = I.used;
  I.used += al256(std::max<size_t>(bytes, 16));
  return off;
}

// Plan install, phase 0: the control region every rank (excluded ones too) has at
// the same offsets: gather flags, barrier flags, gather buffer.
void ipc_layout_begin(stadi_ctx *ctx) {
  IpcState &I = *ctx->ipc;
  const Dims &m = ctx->dm;
  I.used = 0;
  I.site_off[0].clear();
  I.site_off[1].clear();
  I.off_gflag = ipc_reserve(ctx, (size_t)4 * ctx->world);
  I.off_barrier = ipc_reserve(ctx, (size_t)4 * ctx->world);
  I.off_gather = ipc_reserve(ctx, (size_t)m.lat_h * m.lat_w * m.c_in * 4);
}

// Plan install, phase 2 (after the slots were reserved, identically on every
// included rank): ready / done flags, allocate (or reuse) the arena, all-gather
// the IPC handles, map the peers' arenas, build the epilogue's peer table and
// the WAR thresholds.  COLLECTIVE over the world.
stadi_status ipc_commit(stadi_ctx *ctx, int n_sites) {
  IpcState &I = *ctx->ipc;
  const int Gw = ctx->world;
  I.n_sites = n_sites;
  I.off_ready = ipc_reserve(ctx, (size_t)4 * n_sites * Gw);
  I.off_done = ipc_reserve(ctx, (size_t)4 * n_sites * Gw);
  if (I.used > I.cap) {  // grow: the old arena is retired (cudaFree would sync the device)
    if (I.arena) I.retired.push_back(I.arena);
    I.arena = nullptr;
    const size_t cap = al256(I.used + I.used / 8);
    CK(cudaMalloc(&I.arena, cap));
    I.cap = cap;
  }
  CK(cudaMemsetAsync(I.arena, 0, I.used, ctx->astream));
  CK(cudaStreamSynchronize(ctx->astream));
  // record: IPC handle, pid, arena pointer (ranks of the SAME process -- virtual GPUs,
  // green.cuh -- use the pointer directly: a process cannot open its own handles)
  struct Rec {
    cudaIpcMemHandle_t h;
    int64_t pid;
    uint64_t ptr;
  } rec{};
  CK(cudaIpcGetMemHandle(&rec.h, I.arena));
  rec.pid = (int64_t)getpid();
  rec.ptr = (uint64_t)(uintptr_t)I.arena;
  std::vector<std::string> all;
  ST(rdv_allgather(ctx, "arena", std::string((const char *)&rec, sizeof(rec)), all));
  I.peer.resize(Gw, nullptr);
  I.peer_handle.resize(Gw);
  for (int g = 0; g < Gw; ++g) {
    if (g == ctx->rank) {
      I.peer[g] = I.arena;
      continue;
    }
    if (all[g].size() != sizeof(Rec)) return ctx_fail(ctx, STADI_ESTATE, "IPC: bad handle");
    if (I.peer[g] && I.peer_handle[g] == all[g]) continue;  // unchanged mapping
    Rec pr;
    std::memcpy(&pr, all[g].data(), sizeof(pr));
    I.peer_handle[g] = all[g];
    if (pr.pid == rec.pid) {  // same process: the pointer is valid here
      I.peer[g] = (char *)(uintptr_t)pr.ptr;
      continue;
    }
    // a replaced peer mapping stays open (closing may synchronise); closed at destroy
    if (I.peer[g]) I.opened.push_back(I.peer[g]);
    void *p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, pr.h, cudaIpcMemLazyEnablePeerAccess));
    I.peer[g] = (char *)p;
  }
  I.peers.clear();
  for (uint32_t g = 0; g < ctx->plan.n_gpus; ++g)
    if (ctx->plan.tier[g] && (int)g != ctx->rank &&  // R33: K/V only within a CFG branch
        (!ctx->plan.cfg_split || ctx->plan.branch[g] == ctx->plan.branch[ctx->rank]))
      I.peers.push_back((int)g);
  // peer slot table for the fused QKV-epilogue all-gather
  const size_t np = I.peers.size();
  if (I.peer_tab) pfree(ctx, I.peer_tab);
  I.peer_tab = nullptr;
  if (np && n_sites) {
    std::vector<void *> tab((size_t)n_sites * 2 * np);
    for (int s = 0; s < n_sites; ++s)
      for (int par = 0; par < 2; ++par)
        for (size_t k = 0; k < np; ++k)
          tab[((size_t)s * 2 + par) * np + k] = I.peer[I.peers[k]] + I.site_off[par][s];
    CK(pmalloc(ctx, &I.peer_tab, tab.size() * sizeof(void *)));
    CK(cudaMemcpyAsync(I.peer_tab, tab.data(), tab.size() * sizeof(void *),
                       cudaMemcpyHostToDevice, ctx->astream));
    CK(cudaStreamSynchronize(ctx->astream));
  }
  // WAR thresholds: need[g][P] = 1 + the last step index of g that reads a version
  // <= P - 2 of parity P % 2 (0: none)
  I.need.assign(Gw, {});
  for (int g : I.peers) {
    uint32_t n = 0;
    stadi_schedule(&ctx->plan, (uint32_t)g, nullptr, 0, &n);
    std::vector<stadi_step_t> sc(n);
    stadi_schedule(&ctx->plan, (uint32_t)g, sc.data(), n, &n);
    int maxv = 0;
    for (auto &st : sc) maxv = std::max(maxv, std::max(st.read_ver, st.pub_ver));
    I.need[g].assign(maxv + 3, 0);
    for (int P = 0; P < maxv + 3; ++P)
      for (uint32_t k = 0; k < n; ++k)
        if (sc[k].read_ver <= P - 2 && ((sc[k].read_ver ^ P) & 1) == 0)
          I.need[g][P] = k + 1;
  }
  return STADI_OK;
}

// R33 pair exchange of the eps rows (site `site` = the arena's eps buffer
// [tokens, 2, fin_ld] f32, both members use the band's rows): push this rank's branch
// columns of step `idx` to the partner, then wait for the partner's.  WAR: before
// overwriting, the partner must have finished the sampler of step idx - 1.
stadi_status ipc_pair_push(stadi_ctx *ctx, int site, int partner, uint32_t idx, const float *eps,
                           int rows, int ld, int branch, cudaStream_t s) {
  IpcState &I = *ctx->ipc;
  ST(ipc_wait(ctx, I.off_done, (size_t)site * ctx->world + partner, idx, s));
  const size_t off = (const char *)eps - I.arena;
  const size_t pitch = (size_t)2 * ld * 4;
  CK(cudaMemcpy2DAsync(I.peer[partner] + off + (size_t)branch * ld * 4, pitch,
                       (const char *)eps + (size_t)branch * ld * 4, pitch, (size_t)ld * 4, rows,
                       cudaMemcpyDeviceToDevice, s));
  ctx->exch_bytes += (size_t)rows * ld * 4;
  return ipc_signal(ctx, partner, I.off_ready, (size_t)site * ctx->world + ctx->rank, idx + 1, s);
}
stadi_status ipc_pair_wait(stadi_ctx *ctx, int site, int partner, uint32_t idx, cudaStream_t s) {
  return ipc_wait(ctx, ctx->ipc->off_ready, (size_t)site * ctx->world + partner, idx + 1, s);
}
stadi_status ipc_pair_done(stadi_ctx *ctx, int site, int partner, uint32_t idx, cudaStream_t s) {
  return ipc_signal(ctx, partner, ctx->ipc->off_done, (size_t)site * ctx->world + ctx->rank,
                    idx + 1, s);
}

// Device array of the peers' copies of site `site`'s slot of parity `par`.
void *const *ipc_peer_slots(stadi_ctx *ctx, int site, int par) {
  IpcState &I = *ctx->ipc;
  if (!I.peer_tab) return nullptr;
  return I.peer_tab + ((size_t)site * 2 + par) * I.peers.size();
}

// Request start: zero this rank's exchange flags, then a flag barrier with the
// request counter (no rank writes a new flag before every rank has reset).
stadi_status ipc_begin(stadi_ctx *ctx, cudaStream_t s) {
  IpcState &I = *ctx->ipc;
  CK(cudaMemsetAsync(I.arena + I.off_gflag, 0, 4 * (size_t)ctx->world, s));
  if (I.n_sites)
    CK(cudaMemsetAsync(I.arena + I.off_ready, 0,
                       I.off_done - I.off_ready + (size_t)4 * I.n_sites * ctx->world, s));
  ++I.req;
  for (int g = 0; g < ctx->world; ++g)
    if (g != ctx->rank) ST(ipc_signal(ctx, g, I.off_barrier, ctx->rank, I.req, s));
  for (int g = 0; g < ctx->world; ++g)
    if (g != ctx->rank)
      CKD(memops().wait32((CUstream)s, flag_at(I.arena, I.off_barrier, g), I.req,
                          CU_STREAM_WAIT_VALUE_GEQ));
  return STADI_OK;
}

// Final synchronous all-gather of the bands (Alg. 1): every included rank
// copies its band into every rank's gather buffer and raises its flag there.
stadi_status ipc_gather(stadi_ctx *ctx, float *out_full, bool dev, cudaStream_t s) {
  IpcState &I = *ctx->ipc;
  const Dims &m = ctx->dm;
  const size_t row = (size_t)m.lat_w * m.c_in * 4;
  if (!ctx->ranks.empty()) {
    const Rank &r = ctx->ranks[0];
    for (int g = 0; g < ctx->world; ++g) {
      CK(cudaMemcpyAsync(I.peer[g] + I.off_gather + r.row_begin * row, r.x_band, r.rows * row,
                         cudaMemcpyDeviceToDevice, s));
      if (g != ctx->rank) {
        ctx->exch_bytes += r.rows * row;
        ST(ipc_signal(ctx, g, I.off_gflag, ctx->rank, 1, s));
      }
    }
  }
  for (uint32_t g = 0; g < ctx->plan.n_gpus; ++g)
    if (ctx->plan.tier[g] && (int)g != ctx->rank)
      CKD(memops().wait32((CUstream)s, flag_at(I.arena, I.off_gflag, g), 1,
                          CU_STREAM_WAIT_VALUE_GEQ));
  if (dev)
    CK(cudaMemcpyAsync(out_full, I.arena + I.off_gather, (size_t)m.lat_h * row,
                       cudaMemcpyDeviceToDevice, s));
  else
    CK(stage_d2h(ctx, out_full, I.arena + I.off_gather, (size_t)m.lat_h * row, s));
  return STADI_OK;
}

// All-gather of one double per rank (profiling, a1).
stadi_status ipc_allgather_f64(stadi_ctx *ctx, double mine, std::vector<double> &all) {
  std::vector<std::string> raw;
  ST(rdv_allgather(ctx, "ms", std::string((const char *)&mine, 8), raw));
  all.assign(ctx->world, 0.0);
  for (int g = 0; g < ctx->world; ++g) {
    if (raw[g].size() != 8) return ctx_fail(ctx, STADI_ESTATE, "IPC: bad profile record");
    std::memcpy(&all[g], raw[g].data(), 8);
  }
  return STADI_OK;
}

// Can stream memory operations be captured into a CUDA graph on this driver?
bool ipc_probe_graphs(stadi_ctx *ctx) {
  IpcState &I = *ctx->ipc;
  cudaGraph_t g = nullptr;
  if (cudaStreamBeginCapture(ctx->gstream, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return false;
  const CUresult r1 = memops().write32((CUstream)ctx->gstream, (CUdeviceptr)I.probe, 0,
                                       CU_STREAM_WRITE_VALUE_DEFAULT);
  const CUresult r2 = memops().wait32((CUstream)ctx->gstream, (CUdeviceptr)I.probe, 0,
                                      CU_STREAM_WAIT_VALUE_GEQ);
  const cudaError_t e = cudaStreamEndCapture(ctx->gstream, &g);
  bool ok = r1 == CUDA_SUCCESS && r2 == CUDA_SUCCESS && e == cudaSuccess && g;
  if (ok) {
    cudaGraphExec_t x = nullptr;
    ok = cudaGraphInstantiate(&x, g, 0) == cudaSuccess;
    if (x) cudaGraphExecDestroy(x);
  }
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();
  return ok;
}

// Watchdog fired (a peer is gone): set every flag of this rank's arena to its maximum
// from a side stream so the streams blocked in flag waits drain (the request's
// results are void; the context is poisoned by the caller).
void ipc_unblock(stadi_ctx *ctx) {
  if (!ctx->ipc || !ctx->ipc->arena) return;
  IpcState &I = *ctx->ipc;
  // 0x7F7F7F7F: above every version / count / request id under the wrap-safe
  // GEQ compare ((int32_t)(*addr - v) >= 0), which 0xFFFFFFFF would fail
  cudaMemsetAsync(I.arena + I.off_gflag, 0x7F, 4 * (size_t)ctx->world, ctx->astream);
  cudaMemsetAsync(I.arena + I.off_barrier, 0x7F, 4 * (size_t)ctx->world, ctx->astream);
  if (I.n_sites)
    cudaMemsetAsync(I.arena + I.off_ready, 0x7F,
                    I.off_done - I.off_ready + (size_t)4 * I.n_sites * ctx->world, ctx->astream);
  cudaStreamSynchronize(ctx->astream);
}

void ipc_release(stadi_ctx *ctx) {  // destroy (device already synchronised)
  if (!ctx->ipc) return;
  IpcState &I = *ctx->ipc;
  const int64_t me = (int64_t)getpid();
  for (int g = 0; g < (int)I.peer.size(); ++g) {
    if (g == ctx->rank || !I.peer[g] || I.peer_handle[g].size() < sizeof(cudaIpcMemHandle_t) + 8)
      continue;
    int64_t pid;
    std::memcpy(&pid, I.peer_handle[g].data() + sizeof(cudaIpcMemHandle_t), 8);
    if (pid != me) cudaIpcCloseMemHandle(I.peer[g]);  // in-process peers were not opened
  }
  for (char *p : I.opened) cudaIpcCloseMemHandle(p);
  if (I.arena) cudaFree(I.arena);
  for (char *p : I.retired) cudaFree(p);
  // the last rendezvous file stays: a slower peer may not have read it yet (the
  // files of earlier rounds are removed as the protocol goes, see rdv_allgather)
  ctx->ipc.reset();
}

}  // namespace

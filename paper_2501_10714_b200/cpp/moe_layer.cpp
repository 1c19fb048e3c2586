// moe_layer.cpp — the MoE layer executor (include/fsmoe/moe_layer.hpp).
//
// Per rank, canonical buffer layout [src rank p][local expert e_l][capacity C]
// rows of width M (send side: [expert e][C], e = p*E_l + e_l, which is the same
// thing). A pipeline chunk i is the row window [lo_i, hi_i) of every block,
// lo/hi on 128-row granules, so a chunk's AlltoAll is E grouped
// ncclSend/ncclRecv pairs of (hi-lo)*M elements and its expert GEMMs are one
// grouped-GEMM launch over the window (GemmProblem::row0/rows). Forward and
// backward degrees are independent (r_fwd != r_bwd), as in FSMoE.
//
// Streams: compute (gate, permutations, GEMMs) and comm (NCCL), joined by
// events; the comm stream's FIFO order is the schedule simulator's inter-link
// emission order: dispatch 0..r-1, [gradient allreduce slices], combine
// 0..r-1 (schedule_sim.cpp:182-216).
#include "fsmoe/moe_layer.hpp"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>

#include "device_util.hpp"
#include "ep_group.hpp"
#include "fsmoe_cuda.h"

namespace fsmoe {

namespace {

int gate_kind_abi(GateKind k) {
  switch (k) {
    case GateKind::noisy_topk: return FSMOE_GATE_NOISY_TOPK;
    case GateKind::sigmoid_topk: return FSMOE_GATE_SIGMOID_TOPK;
    case GateKind::cosine_topk: return FSMOE_GATE_COSINE_TOPK;
    case GateKind::expert_choice: return FSMOE_GATE_EXPERT_CHOICE;
  }
  return -1;
}

struct Chunk {
  int lo, hi;
};

// 128-row granule chunks of [0, C): r clipped to the granule count.
std::vector<Chunk> make_chunks(long long C, int r) {
  const long long ng = (C + 127) / 128;
  if (r < 1) r = 1;
  if (r > ng) r = static_cast<int>(ng);
  std::vector<Chunk> out;
  for (int i = 0; i < r; ++i) {
    long long a = (i * ng) / r * 128, b = ((i + 1) * ng) / r * 128;
    out.push_back({static_cast<int>(a), static_cast<int>(std::min(b, C))});
  }
  return out;
}

}  // namespace

// Measured timeline: CUDA events around every phase on the comm (lane 0 =
// the simulator's inter_link) and compute (lane 2) streams, emitted as Chrome
// trace events with the schedule simulator's fields and labels
// (schedule_sim.cpp:351-367), so predicted and measured schedules diff.
struct Tracer {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  struct Span {
    std::string name;
    int lane;
    cudaEvent_t a, b;
  };
  std::vector<Span> spans;
  cudaEvent_t base = nullptr;
  std::string json;  // accumulated events
  double offset_ms = 0.0;

  cudaEvent_t next() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "event");
      pool.push_back(e);
    }
    return pool[used++];
  }
  void start(cudaStream_t s) {
    if (!on) return;
    base = next();
    cuda_check(cudaEventRecord(base, s), "eventRecord");
  }
  int begin(const std::string& name, int lane, cudaStream_t s) {
    if (!on) return -1;
    cudaEvent_t e = next();
    cuda_check(cudaEventRecord(e, s), "eventRecord");
    spans.push_back({name, lane, e, nullptr});
    return static_cast<int>(spans.size()) - 1;
  }
  void end(int i, cudaStream_t s) {
    if (i < 0) return;
    cudaEvent_t e = next();
    cuda_check(cudaEventRecord(e, s), "eventRecord");
    spans[static_cast<size_t>(i)].b = e;
  }
  void flush(const char* phase) {
    if (!on || spans.empty()) return;
    for (auto& sp : spans) cuda_check(cudaEventSynchronize(sp.b), "eventSync");
    double call_end = 0.0;
    char buf[256];
    for (auto& sp : spans) {
      float t0 = 0.f, t1 = 0.f;
      cudaEventElapsedTime(&t0, base, sp.a);
      cudaEventElapsedTime(&t1, base, sp.b);
      std::snprintf(buf, sizeof buf,
                    "%s{\"name\": \"%s.%s\", \"ph\": \"X\", \"ts\": %.3f, \"dur\": %.3f, "
                    "\"pid\": 0, \"tid\": %d}",
                    json.empty() ? "" : ",\n", phase, sp.name.c_str(), (offset_ms + t0) * 1000.0,
                    (t1 - t0) * 1000.0, sp.lane);
      json += buf;
      call_end = std::max(call_end, static_cast<double>(t1));
    }
    offset_ms += call_end;
    spans.clear();
    used = 0;
  }
  ~Tracer() {
    for (auto e : pool) cudaEventDestroy(e);
  }
};

struct MoELayer::Impl {
  MoELayerConfig cfg;
  Tracer tr;
  EpGroup* ep = nullptr;
  int P = 1, rank = 0, E = 0, El = 0, T = 0, M = 0, H = 0, N1 = 0, k = 0;
  long long C = 0, n_picks = 0;
  int esz = 2;          // activation element size
  int dtype = FSMOE_BF16;
  ncclDataType_t nccl_dt = ncclBfloat16;
  fsmoe_gate_desc gd{};
  MoEParams prm;
  const void* x_last = nullptr;  // forward input (caller keeps it alive for backward)
  std::vector<Chunk> fwd_chunks, bwd_chunks;

  cudaStream_t s_comp = nullptr, s_comm = nullptr;
  // second compute stream: the backward's wgrad GEMMs run beside the dgrad
  // GEMMs they do not depend on, so each fills the other's last wave
  cudaStream_t s_aux = nullptr;
  cudaEvent_t ev_x1 = nullptr, ev_x2 = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_gate = nullptr, ev_join = nullptr;
  std::vector<cudaEvent_t> ev_a, ev_b;  // per-chunk (max of r_fwd, r_bwd)

  std::map<std::string, std::pair<void*, long long>> bufs;
  std::vector<void*> owned;

  // routing state
  int *tok = nullptr, *exp = nullptr, *slot = nullptr, *pos = nullptr, *tptr = nullptr,
      *tpick = nullptr, *status = nullptr;
  double *w = nullptr, *dw = nullptr, *scores = nullptr, *noise = nullptr, *spread = nullptr,
         *proj_out = nullptr;
  long long *fill = nullptr, *dropped = nullptr, *rfill = nullptr;
  // nanoseconds this rank's compute stream spent waiting on peer flags
  // (untraced exposed-exchange time; peer.cu)
  unsigned long long* wait_ns = nullptr;
  void *gate_ws = nullptr, *assign_ws = nullptr, *tidx_ws = nullptr, *gbwd_ws = nullptr;
  size_t gate_wsb = 0, assign_wsb = 0, tidx_wsb = 0, gbwd_wsb = 0;
  // activations (canonical [P*E_l][C][.])
  void *Xs = nullptr, *Xr = nullptr, *Z = nullptr, *Hh = nullptr, *Or = nullptr, *Os = nullptr;
  void *dOs = nullptr, *dOr = nullptr, *dXr = nullptr, *dXs = nullptr;

  // Peer-memory transport (default for P > 1; FSMOE_EP_TRANSPORT=nccl selects
  // the grouped ncclSend/ncclRecv baseline). The four receive-side buffers,
  // the received fills and the arrival flags live in one IPC-shared region;
  // producers store rows straight into the owner's copy.
  // top-1 softmax gate (noisy / cosine): the masked softmax over one survivor
  // is exactly 1.0 (workload.cpp:123-133), so the I-order and its backward
  // are row gathers and the weight gradient is identically zero
  bool unit_top1 = false;
  // N = 1, bf16, unit top-1: GEMM2 / dgrad1 scatter their rows straight to
  // the tokens' rows of y / dx (the combine and its backward fused away)
  void* scatter_y = nullptr;
  void* scatter_dx = nullptr;
  bool fuse_top1 = false;  // FSMOE_NO_FUSED_COMBINE (measurement) keeps the row gathers
  // EP with r = 1: move the local share first and the peers' share on s_aux,
  // overlapping the NVLink transfer with GEMMs on the local blocks
  bool split = false;
  int split_sms = 0;
  bool peer = false;
  void* sym = nullptr;
  std::vector<void*> sym_peers;
  fsmoe_peer_rows map_X{}, map_O{}, map_dO{}, map_dX{}, map_fill{};
  fsmoe_peer_flags flags{};
  int n_chunk_slots = 1;
  std::vector<unsigned long long> epoch;
  bool last_was_bwd = false;
  int slot_bar_fwd() const { return 0; }
  int slot_disp_fwd(size_t j) const { return 1 + static_cast<int>(j); }
  int slot_comb_fwd(size_t j) const { return 1 + n_chunk_slots + static_cast<int>(j); }
  int slot_disp_bwd(size_t j) const { return 1 + 2 * n_chunk_slots + static_cast<int>(j); }
  int slot_comb_bwd(size_t j) const { return 1 + 3 * n_chunk_slots + static_cast<int>(j); }
  int slot_bar_bwd() const { return 1 + 4 * n_chunk_slots; }
  int n_slots() const { return 2 + 4 * n_chunk_slots; }
  // Copy-engine transport (FSMOE_EP_TRANSPORT=ce): FSMoE's chunked pipeline
  // for the dispatch-side exchanges. The permutation kernels write this
  // rank's own rows straight into its receive buffer and the peers' rows into
  // a canonical send buffer (stage maps); the copy engines move pipeline
  // chunk i to every peer on s_ce while the expert GEMMs of chunk i-1 hold
  // the SMs, and a stream memory write raises chunk i's flag behind them.
  // The combine-side exchanges stay fused into the GEMM epilogues.
  bool ce = false;
  cudaStream_t s_ce = nullptr;
  cudaEvent_t ev_ce = nullptr;
  void *Xsend = nullptr, *dOsend = nullptr;
  fsmoe_peer_rows stage_X{}, stage_dO{};
  std::vector<unsigned long long> sig_count;
  void ce_signal(int slot) {
    throw_on(fsmoe_peer_flag_write(&flags, slot, ++sig_count[static_cast<size_t>(slot)], s_ce));
  }
  // rows of block b = p*E_l + e_l: own (p == rank) into the receive buffer,
  // the peers' into the canonical send buffer at [p E_l + e_l][C]
  fsmoe_peer_rows stage_map(void* recv_local, void* send) const {
    fsmoe_peer_rows m{};
    m.world = P;
    m.rank = rank;
    m.experts_local = El;
    m.capacity = C;
    const long long blk = static_cast<long long>(El) * C * M * esz;
    for (int p = 0; p < P; ++p)
      m.base[p] = p == rank ? recv_local : static_cast<char*>(send) + (p - rank) * blk;
    return m;
  }

  void peer_signal(int slot, const void* put = nullptr, long long put_row_bytes = 0,
                   const fsmoe_peer_rows* put_map = nullptr, cudaStream_t st = nullptr) {
    throw_on(fsmoe_peer_signal(&flags, slot, put, put_row_bytes, put_map, st ? st : s_comp));
  }
  void peer_wait(int slot) {
    // local (single-device) group: every rank's matching signal is enqueued
    // before any rank enqueues this wait (ep_group.hpp)
    ep->host_sync();
    throw_on(fsmoe_peer_wait(&flags, slot, ++epoch[static_cast<size_t>(slot)], s_comp));
  }

  fsmoe_peer_rows make_map(size_t off, long long cap) const {
    fsmoe_peer_rows m{};
    m.world = P;
    m.rank = rank;
    m.experts_local = El;
    m.capacity = cap;
    for (int p = 0; p < P; ++p) m.base[p] = static_cast<char*>(sym_peers[p]) + off;
    return m;
  }

  // [P][E_l][C] -> sym offsets; set up the maps and flags (collective).
  void setup_peer(long long ab) {
    auto al = [](size_t x) { return (x + 4095) & ~size_t(4095); };
    size_t off = 0;
    const size_t o_X = off; off = al(off + ab);
    const size_t o_O = off; off = al(off + ab);
    const size_t o_dO = off; off = al(off + ab);
    const size_t o_dX = off; off = al(off + ab);
    const size_t o_fill = off; off = al(off + 8 * static_cast<size_t>(E));
    const size_t o_flags = off; off = al(off + 8 * static_cast<size_t>(n_slots()) * P);
    cuda_check(cudaMalloc(&sym, off), "cudaMalloc");
    // zero: padding rows are never written by the producers (flags start at 0)
    cuda_check(cudaMemsetAsync(sym, 0, off, s_comp), "memset");
    sym_peers = ep->map_peers(sym, s_comp);
    char* b = static_cast<char*>(sym);
    Xr = b + o_X;
    Os = b + o_O;
    dOr = b + o_dO;
    dXs = b + o_dX;
    rfill = reinterpret_cast<long long*>(b + o_fill);
    alias("X_recv", Xr, ab);
    alias("O_send", Os, ab);
    alias("dO_recv", dOr, ab);
    alias("dX_send", dXs, ab);
    alias("recv_fill", rfill, 8LL * E);
    map_X = make_map(o_X, C);
    map_O = make_map(o_O, C);
    map_dO = make_map(o_dO, C);
    map_dX = make_map(o_dX, C);
    map_fill = make_map(o_fill, 1);
    flags.world = P;
    flags.rank = rank;
    flags.nslots = n_slots();
    flags.wait_ns = wait_ns;
    // a lost peer traps the waiter after FSMOE_PEER_TIMEOUT_S seconds
    // (default 600; 0 = wait forever)
    const char* to = std::getenv("FSMOE_PEER_TIMEOUT_S");
    const double sec = to ? std::atof(to) : 600.0;
    flags.timeout_ns = sec > 0 ? static_cast<unsigned long long>(sec * 1e9) : 0ULL;
    for (int p = 0; p < P; ++p)
      flags.base[p] = reinterpret_cast<unsigned long long*>(static_cast<char*>(sym_peers[p]) + o_flags);
    epoch.assign(static_cast<size_t>(n_slots()), 0);
  }

  void* dalloc(const std::string& name, long long bytes) {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, static_cast<size_t>(std::max<long long>(bytes, 16))), "cudaMalloc");
    owned.push_back(p);
    bufs[name] = {p, bytes};
    return p;
  }
  void alias(const std::string& name, void* p, long long bytes) { bufs[name] = {p, bytes}; }

  ~Impl() {
    if (s_comp) cudaStreamSynchronize(s_comp);
    if (s_comm) cudaStreamSynchronize(s_comm);
    if (s_aux) cudaStreamSynchronize(s_aux);
    if (s_ce) cudaStreamSynchronize(s_ce);
    if (ep && !sym_peers.empty()) ep->unmap_peers(sym_peers);
    // no peer may still map or signal into `sym` when it is freed
    if (ep && sym) ep->quiesce(s_comp);
    if (sym) cudaFree(sym);
    for (void* p : owned) cudaFree(p);
    for (auto e : ev_a) cudaEventDestroy(e);
    for (auto e : ev_b) cudaEventDestroy(e);
    for (auto e : {ev_in, ev_out, ev_gate, ev_join, ev_x1, ev_x2})
      if (e) cudaEventDestroy(e);
    if (s_aux) {
      cudaStreamSynchronize(s_aux);
      cudaStreamDestroy(s_aux);
    }
    if (s_comp) cudaStreamDestroy(s_comp);
    if (s_comm) cudaStreamDestroy(s_comm);
    if (s_ce) cudaStreamDestroy(s_ce);
    if (ev_ce) cudaEventDestroy(ev_ce);
  }

  // ------------------------------------------------------------- GEMMs --
  void gemm(fsmoe_gemm_desc& d, cudaStream_t st = nullptr) {
    d.precision = cfg.precision == Precision::f32 ? 1 : 0;
    throw_on(fsmoe_grouped_gemm(&d, st ? st : s_comp));
  }

  fsmoe_gemm_desc row_desc(const Chunk& c) const {
    fsmoe_gemm_desc d{};
    d.kind = 0;
    d.nblk = P * El;
    d.n_w = El;
    d.rows = c.hi - c.lo;
    d.rows_total = static_cast<int>(C);
    d.row0 = c.lo;
    d.valid_rows = P > 1 ? rfill : fill;
    return d;
  }

  fsmoe_gemm_desc k_desc(const Chunk& c, bool accumulate) const {
    fsmoe_gemm_desc d = row_desc(c);
    d.kind = 1;
    d.epi = 1;
    d.accumulate = accumulate ? 1 : 0;
    return d;
  }

  // Blocks [rank*E_l, rank*E_l + E_l) of the [P][E_l][C] receive layout hold
  // this rank's own tokens: they are local before any peer has delivered.
  void local_blocks(fsmoe_gemm_desc& d, int exclude) const {
    d.blk_lo = rank * El;
    d.blk_hi = rank * El + El;
    d.blk_exclude = exclude;
    // the local-share GEMM runs beside the peers' NVLink row transfer: leave
    // that kernel SMs of its own (the persistent GEMM otherwise fills them all)
    if (!exclude) d.max_sms = split_sms;
  }

  // part 0: the whole expert forward; 1: GEMM1 on the local blocks only;
  // 2: GEMM1 on the peers' blocks, then GEMM2 on everything
  void expert_fwd(const Chunk& c, int part = 0) {
    const bool bf = cfg.precision == Precision::bf16;
    const bool gated = cfg.ffn == LayerConfig::Ffn::gated3;
    // GEMM1: Z = X W1^T (+ fused activation -> H)
    fsmoe_gemm_desc g1 = row_desc(c);
    if (part) local_blocks(g1, part == 2);
    g1.K = M;
    g1.N = N1;
    g1.A = Xr;
    g1.B = prm.w1;
    g1.D = Z;
    g1.ldd = N1;
    if (bf) {
      g1.epi = gated ? 3 : 2;
      g1.D2 = Hh;
      g1.ldd2 = H;
    } else {
      g1.epi = 1;
    }
    gemm(g1);
    if (!bf)
      throw_on(fsmoe_activation_f32(gated ? 3 : 2, P * El, static_cast<int>(C), c.lo, c.hi - c.lo, H,
                                    static_cast<const float*>(Z), nullptr,
                                    static_cast<float*>(Hh), s_comp));
    if (part == 1) return;
    // GEMM2: O = H W2^T
    fsmoe_gemm_desc g2 = row_desc(c);
    g2.K = H;
    g2.N = M;
    g2.A = Hh;
    g2.B = prm.w2;
    g2.D = Or;
    g2.ldd = M;
    g2.epi = bf ? 0 : 1;
    if (peer) g2.d_peers = &map_O;  // combine AlltoAll fused into the epilogue
    if (scatter_y) {                // top-1 combine fused: slot row -> its token's row
      g2.scatter_rows = pos;
      g2.scatter_out = scatter_y;
      g2.scatter_ld = M;
    }
    gemm(g2);
  }

  // part 0: the whole expert backward; 1: dgrad2 on the local blocks only
  // (bf16: dZ over Z); 2: everything else (dgrad2 on the peers' blocks)
  void expert_bwd(const Chunk& c, bool first, int part = 0) {
    const bool bf = cfg.precision == Precision::bf16;
    const bool gated = cfg.ffn == LayerConfig::Ffn::gated3;
    if (part == 1) {
      fsmoe_gemm_desc d2 = row_desc(c);
      local_blocks(d2, 0);
      d2.K = M;
      d2.N = H;
      d2.b_mn_major = 1;
      d2.A = dOr;
      d2.B = prm.w2;
      d2.epi = gated ? 5 : 4;
      d2.Zin = Z;
      d2.ldz = N1;
      d2.D = Z;
      d2.ldd = N1;
      gemm(d2);
      return;
    }
    // bf16: wgrad GEMMs on s_aux beside the dgrad GEMMs (independent inputs and
    // outputs); fp32 check mode writes dH over H, which wgrad2 reads: serial
    cudaStream_t sw = bf ? s_aux : s_comp;
    if (bf) {
      record(ev_x1, s_comp);
      wait(s_aux, ev_x1);
    }
    // wgrad2: dW2[e] (M x H) += dO^T H
    fsmoe_gemm_desc w2 = k_desc(c, !first);
    w2.Mo = M;
    w2.No = H;
    w2.A = dOr;
    w2.B = Hh;
    w2.D = prm.g_w2;
    w2.ldd = H;
    gemm(w2, sw);
    // dgrad2: dH = dO W2 ; dZ = dH * act'(Z)   (written over Z)
    fsmoe_gemm_desc d2 = row_desc(c);
    d2.K = M;
    d2.N = H;
    d2.b_mn_major = 1;
    d2.A = dOr;
    d2.B = prm.w2;
    if (bf) {
      d2.epi = gated ? 5 : 4;
      d2.Zin = Z;
      d2.ldz = N1;
      d2.D = Z;
      d2.ldd = N1;
      if (part == 2) local_blocks(d2, 1);
      gemm(d2);
    } else {
      d2.epi = 1;
      d2.D = Hh;  // dH over H (wgrad2 already consumed it)
      d2.ldd = H;
      gemm(d2);
      throw_on(fsmoe_activation_f32(gated ? 5 : 4, P * El, static_cast<int>(C), c.lo, c.hi - c.lo, H,
                                    static_cast<const float*>(Hh), static_cast<const float*>(Z),
                                    static_cast<float*>(Z), s_comp));
    }
    // wgrad1 needs dZ: after dgrad2 (and after wgrad2 in stream order on sw)
    if (bf) {
      record(ev_x1, s_comp);
      wait(s_aux, ev_x1);
    }
    // wgrad1: dW1[e] (N1 x M) += dZ^T X
    fsmoe_gemm_desc w1 = k_desc(c, !first);
    w1.Mo = N1;
    w1.No = M;
    w1.A = Z;
    w1.B = Xr;
    w1.D = prm.g_w1;
    w1.ldd = M;
    gemm(w1, sw);
    // dgrad1: dX = dZ W1
    fsmoe_gemm_desc d1 = row_desc(c);
    d1.K = N1;
    d1.N = M;
    d1.b_mn_major = 1;
    d1.A = Z;
    d1.B = prm.w1;
    d1.D = dXr;
    d1.ldd = M;
    d1.epi = bf ? 0 : 1;
    if (peer) d1.d_peers = &map_dX;  // backward combine fused into the epilogue
    if (scatter_dx) {                // top-1 order backward fused: slot row -> token row
      d1.scatter_rows = pos;
      d1.scatter_out = scatter_dx;
      d1.scatter_ld = M;
    }
    gemm(d1);
    if (bf) {
      // rejoin: the next chunk's dgrad2 overwrites Z, which wgrad1 reads
      record(ev_x2, s_aux);
      wait(s_comp, ev_x2);
    }
  }

  // ------------------------------------------------------- exchanges --
  // Send rows [lo,hi) of every block of `send` ([E][C][M], e = p*E_l + e_l)
  // to rank p, receive rank p's rows into `recv` block (p, e_l).
  void exchange(const void* send, void* recv, const Chunk& c) {
    const size_t row = static_cast<size_t>(M) * esz;
    const size_t n = static_cast<size_t>(c.hi - c.lo) * M;
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (int p = 0; p < P; ++p) {
      for (int el = 0; el < El; ++el) {
        const size_t blk = static_cast<size_t>(p * El + el);
        const char* sp = static_cast<const char*>(send) + (blk * C + c.lo) * row;
        char* rp = static_cast<char*>(recv) + (blk * C + c.lo) * row;
        nccl_check(ncclSend(sp, n, nccl_dt, p, ep->comm(), s_comm), "ncclSend");
        nccl_check(ncclRecv(rp, n, nccl_dt, p, ep->comm(), s_comm), "ncclRecv");
      }
    }
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  }

  void exchange_fill() {
    nccl_check(ncclGroupStart(), "ncclGroupStart");
    for (int p = 0; p < P; ++p) {
      nccl_check(ncclSend(fill + static_cast<size_t>(p) * El, El, ncclInt64, p, ep->comm(), s_comm),
                 "ncclSend");
      nccl_check(ncclRecv(rfill + static_cast<size_t>(p) * El, El, ncclInt64, p, ep->comm(), s_comm),
                 "ncclRecv");
    }
    nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  }

  void allreduce_slices() {
    if (!prm.dense_grad || cfg.dense_grad_elems <= 0) return;
    std::vector<long long> sl = cfg.ar_slices;
    if (sl.empty()) sl.push_back(cfg.dense_grad_elems);
    long long off = 0;
    for (long long n : sl) {
      n = std::min(n, cfg.dense_grad_elems - off);
      if (n <= 0) break;
      ep->allreduce_sum(prm.dense_grad + off, static_cast<size_t>(n), false, s_comm);
      off += n;
    }
  }

  void record(cudaEvent_t e, cudaStream_t s) { cuda_check(cudaEventRecord(e, s), "eventRecord"); }
  void wait(cudaStream_t s, cudaEvent_t e) { cuda_check(cudaStreamWaitEvent(s, e, 0), "waitEvent"); }
};

MoELayer::MoELayer(const MoELayerConfig& cfg, EpGroup* ep) : impl_(new Impl), cfg_(cfg) {
  Impl& I = *impl_;
  I.cfg = cfg;
  I.ep = ep;
  I.P = ep ? ep->world() : 1;
  I.rank = ep ? ep->rank() : 0;
  world_ = I.P;
  if (cfg.tokens <= 0 || cfg.model_dim <= 0 || cfg.ffn_dim <= 0 || cfg.experts <= 0 || cfg.top_k <= 0)
    throw ConfigError("layer: tokens, model_dim, ffn_dim, experts and top_k must be positive");
  if (cfg.experts % I.P != 0)
    throw ConfigError("experts must divide evenly across expert_parallel groups");
  if (cfg.model_dim % 64 || cfg.ffn_dim % 128)
    throw ConfigError("layer: model_dim must be a multiple of 64 and ffn_dim of 128");
  cuda_check(cudaSetDevice(cfg.device), "cudaSetDevice");
  I.E = cfg.experts;
  I.El = I.E / I.P;
  el_ = I.El;
  I.T = cfg.tokens;
  I.M = cfg.model_dim;
  I.H = cfg.ffn_dim;
  I.k = cfg.top_k;
  I.N1 = cfg.ffn == LayerConfig::Ffn::gated3 ? 2 * I.H : I.H;
  if (cfg.capacity > 0) {
    I.C = cfg.capacity;
  } else {
    LayerConfig lc;
    lc.batch = 1;
    lc.heads = 1;
    lc.seq_len = cfg.tokens;
    lc.model_dim = cfg.model_dim;
    lc.hidden_scale = 1;
    lc.capacity_factor = cfg.capacity_factor;
    lc.unlimited_capacity = cfg.unlimited_capacity;
    lc.experts = cfg.experts;
    lc.top_k = cfg.top_k;
    I.C = capacity_tokens(lc);
  }
  cap_ = I.C;
  const bool bf = cfg.precision == Precision::bf16;
  I.esz = bf ? 2 : 4;
  I.dtype = bf ? FSMOE_BF16 : FSMOE_F32;
  I.nccl_dt = bf ? ncclBfloat16 : ncclFloat32;
  I.fwd_chunks = make_chunks(I.C, cfg.r_fwd);
  I.bwd_chunks = make_chunks(I.C, cfg.r_bwd);

  // gate descriptor
  fsmoe_gate_desc& d = I.gd;
  d.kind = gate_kind_abi(cfg.gate);
  d.top_k = cfg.gate == GateKind::expert_choice ? static_cast<int>(I.C) : cfg.top_k;
  d.seed = cfg.seed;
  d.tokens = I.T;
  d.model_dim = I.M;
  d.x_dtype = I.dtype;
  const bool cosine = cfg.gate == GateKind::cosine_topk;
  d.score_rows = cosine ? cfg.proj_dim : I.M;
  d.score_cols = I.E;
  d.noise_rows = I.M;
  d.noise_cols = I.E;
  d.proj_rows = cosine ? cfg.proj_dim : 0;
  d.proj_cols = cosine ? I.M : 0;
  throw_on(fsmoe_gate_validate(&d));
  I.n_picks = cfg.gate == GateKind::expert_choice ? static_cast<long long>(I.E) * d.top_k
                                                  : static_cast<long long>(I.T) * I.k;
  I.unit_top1 = cfg.top_k == 1 &&
                (cfg.gate == GateKind::noisy_topk || cfg.gate == GateKind::cosine_topk) &&
                static_cast<long long>(I.M) * (cfg.precision == Precision::bf16 ? 2 : 4) % 16 == 0 &&
                static_cast<long long>(I.M) * (cfg.precision == Precision::bf16 ? 2 : 4) <= 4096 &&
                !std::getenv("FSMOE_NO_UNIT_TOP1");
  I.fuse_top1 = I.unit_top1 && I.P == 1 && cfg.precision == Precision::bf16 &&
                !std::getenv("FSMOE_NO_FUSED_COMBINE");
  if (cfg.gate == GateKind::expert_choice && I.C > I.T)
    throw ConfigError("gate: expert capacity exceeds token count");

  cuda_check(cudaStreamCreateWithPriority(&I.s_comp, cudaStreamNonBlocking, 0), "stream");
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cuda_check(cudaStreamCreateWithPriority(&I.s_comm, cudaStreamNonBlocking, hi), "stream");
  cuda_check(cudaStreamCreateWithPriority(&I.s_aux, cudaStreamNonBlocking, 0), "stream");
  for (cudaEvent_t* e : {&I.ev_in, &I.ev_out, &I.ev_gate, &I.ev_join, &I.ev_x1, &I.ev_x2})
    cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
  const size_t nev = std::max(I.fwd_chunks.size(), I.bwd_chunks.size());
  I.ev_a.resize(nev);
  I.ev_b.resize(nev);
  for (size_t i = 0; i < nev; ++i) {
    cuda_check(cudaEventCreateWithFlags(&I.ev_a[i], cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&I.ev_b[i], cudaEventDisableTiming), "event");
  }

  const long long P_ = I.n_picks, T = I.T, E = I.E, C = I.C, M = I.M;
  I.tok = static_cast<int*>(I.dalloc("pick_token", 4 * P_));
  I.exp = static_cast<int*>(I.dalloc("pick_expert", 4 * P_));
  I.w = static_cast<double*>(I.dalloc("pick_weight", 8 * P_));
  I.dw = static_cast<double*>(I.dalloc("d_weight", 8 * P_));
  I.slot = static_cast<int*>(I.dalloc("slot_of_pick", 4 * P_));
  I.pos = static_cast<int*>(I.dalloc("pick_of_slot", 4 * E * C));
  I.tptr = static_cast<int*>(I.dalloc("tok_ptr", 4 * (T + 1)));
  I.tpick = static_cast<int*>(I.dalloc("tok_pick", 4 * P_));
  I.status = static_cast<int*>(I.dalloc("status", 8));
  I.fill = static_cast<long long*>(I.dalloc("fill", 8 * E));
  I.dropped = static_cast<long long*>(I.dalloc("dropped", 8));
  if (I.P > 1) {
    // MoELayerConfig::transport, else FSMOE_EP_TRANSPORT, else the peer stores
    const char* tr = std::getenv("FSMOE_EP_TRANSPORT");
    int t = cfg.transport;
    if (t == 0) t = !tr ? 1 : std::strcmp(tr, "nccl") == 0 ? 3 : std::strcmp(tr, "ce") == 0 ? 2 : 1;
    if (t < 1 || t > 3) throw ConfigError("layer: transport must be 0 (default), 1 peer, 2 ce or 3 nccl");
    I.peer = t != 3;
    I.ce = t == 2;
    if (!I.peer && ep->local())
      throw ConfigError("layer: the NCCL transport needs one GPU per rank (local group given)");
  }
  I.wait_ns = reinterpret_cast<unsigned long long*>(I.dalloc("wait_ns", 8));
  cuda_check(cudaMemsetAsync(I.wait_ns, 0, 8, I.s_comp), "memset");
  I.rfill = I.P > 1 && !I.peer ? static_cast<long long*>(I.dalloc("recv_fill", 8 * E)) : I.fill;
  I.scores = static_cast<double*>(I.dalloc("scores", 8 * T * E));
  if (cfg.gate == GateKind::noisy_topk) {
    I.noise = static_cast<double*>(I.dalloc("noise", 8 * T * E));
    I.spread = static_cast<double*>(I.dalloc("spread", 8 * T * E));
  }
  if (cosine) I.proj_out = static_cast<double*>(I.dalloc("proj_out", 8 * T * cfg.proj_dim));
  I.gate_wsb = fsmoe_gate_workspace_size(&d);
  I.gate_ws = I.dalloc("gate_ws", static_cast<long long>(I.gate_wsb));
  I.assign_wsb = fsmoe_assign_workspace_size(P_, I.E);
  I.assign_ws = I.dalloc("assign_ws", static_cast<long long>(I.assign_wsb));
  I.tidx_wsb = fsmoe_token_index_workspace_size(P_, I.T);
  I.tidx_ws = I.dalloc("tidx_ws", static_cast<long long>(I.tidx_wsb));
  I.gbwd_wsb = fsmoe_gate_bwd_workspace_size(&d);
  I.gbwd_ws = I.dalloc("gate_bwd_ws", static_cast<long long>(I.gbwd_wsb));

  const long long rows = E * C;  // == P * E_l * C on both sides
  const long long ab = rows * M * I.esz;
  if (I.peer) {
    const char* sp_env = std::getenv("FSMOE_EP_SPLIT");
    I.split = !I.ce && I.fwd_chunks.size() == 1 && I.bwd_chunks.size() == 1 && sp_env &&
              std::atoi(sp_env) > 0;
    if (I.split) I.split_sms = std::atoi(sp_env) > 1 ? std::atoi(sp_env) : 0;
    I.n_chunk_slots = static_cast<int>(std::max(I.fwd_chunks.size(), I.bwd_chunks.size()));
    I.setup_peer(ab);
    if (I.ce) {
      I.Xsend = I.dalloc("X_send", ab);
      I.dOsend = I.dalloc("dO_send", ab);
      I.stage_X = I.stage_map(I.Xr, I.Xsend);
      I.stage_dO = I.stage_map(I.dOr, I.dOsend);
      I.sig_count.assign(static_cast<size_t>(I.n_slots()), 0);
      cuda_check(cudaStreamCreateWithPriority(&I.s_ce, cudaStreamNonBlocking, hi), "stream");
      cuda_check(cudaEventCreateWithFlags(&I.ev_ce, cudaEventDisableTiming), "event");
    }
    I.Z = I.dalloc("Z", rows * I.N1 * I.esz);
    I.Hh = I.dalloc("H", rows * I.H * I.esz);
    cuda_check(cudaMemsetAsync(I.status, 0, 8, I.s_comp), "memset");
    cuda_check(cudaStreamSynchronize(I.s_comp), "sync");
    return;
  }
  I.Xs = I.dalloc("X_send", ab);
  I.Xr = I.P > 1 ? I.dalloc("X_recv", ab) : I.Xs;
  if (I.P == 1) I.alias("X_recv", I.Xr, ab);
  I.Z = I.dalloc("Z", rows * I.N1 * I.esz);
  I.Hh = I.dalloc("H", rows * I.H * I.esz);
  I.Or = I.dalloc("O_recv", ab);
  I.Os = I.P > 1 ? I.dalloc("O_send", ab) : I.Or;
  if (I.P == 1) I.alias("O_send", I.Os, ab);
  I.dOs = I.dalloc("dO_send", ab);
  I.dOr = I.P > 1 ? I.dalloc("dO_recv", ab) : I.dOs;
  I.dXr = I.dalloc("dX_recv", ab);
  I.dXs = I.P > 1 ? I.dalloc("dX_send", ab) : I.dXr;
  cuda_check(cudaMemsetAsync(I.status, 0, 8, I.s_comp), "memset");
  cuda_check(cudaStreamSynchronize(I.s_comp), "sync");
}

MoELayer::~MoELayer() = default;

void MoELayer::bind(const MoEParams& p) {
  if (!p.w_gate || !p.w1 || !p.w2 || !p.g_w1 || !p.g_w2 || !p.g_gate)
    throw ConfigError("layer: bind needs w_gate, w1, w2 and their gradients");
  if (cfg_.gate == GateKind::noisy_topk && (!p.w_noise || !p.g_noise))
    throw ConfigError("layer: noisy_topk needs w_noise and g_noise");
  if (cfg_.gate == GateKind::cosine_topk && (!p.proj || !p.g_proj))
    throw ConfigError("layer: cosine_topk needs proj and g_proj");
  impl_->prm = p;
}

void MoELayer::forward(const void* x, void* y, void* stream) {
  Impl& I = *impl_;
  cuda_check(cudaSetDevice(cfg_.device), "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  I.record(I.ev_in, st);
  I.wait(I.s_comp, I.ev_in);
  I.tr.start(I.s_comp);
  I.x_last = x;
  I.scatter_y = I.fuse_top1 ? y : nullptr;
  // every earlier use of this layer's receive buffers is finished here; the
  // wait for the peers' matching signal hides behind the gate
  if (I.peer) I.peer_signal(I.slot_bar_fwd());
  // K1 gate, K2 assign, token index, K3 dispatch
  int sp = I.tr.begin("gate", 2, I.s_comp);
  // a top-1 softmax gate has no gradient: its saved tensors are not needed
  // (and the gate may then skip the exact logits of tokens with one candidate)
  const bool save = !I.unit_top1;
  throw_on(fsmoe_gate(&I.gd, x, I.prm.w_gate, I.prm.w_noise, I.prm.proj, I.tok, I.exp, I.w,
                      save ? I.scores : nullptr, save ? I.noise : nullptr, save ? I.spread : nullptr,
                      I.proj_out, I.status, I.gate_ws, I.gate_wsb, I.s_comp));
  I.tr.end(sp, I.s_comp);
  sp = I.tr.begin("order", 2, I.s_comp);
  throw_on(fsmoe_assign(I.n_picks, I.tok, I.exp, I.T, I.E, I.C, I.slot, I.fill, I.dropped, I.pos,
                        I.status, I.assign_ws, I.assign_wsb, I.s_comp));
  const int kmajor = cfg_.gate == GateKind::expert_choice ? 0 : I.k;
  throw_on(fsmoe_token_index(I.n_picks, I.tok, I.T, kmajor, I.tptr, I.tpick, I.tidx_ws,
                             I.tidx_wsb, I.s_comp));
  if (!I.peer)
    throw_on(fsmoe_dispatch(I.dtype, I.M, I.E, I.C, 1, I.pos, I.tok, x, I.Xs, I.s_comp));
  I.tr.end(sp, I.s_comp);
  const auto& ch = I.fwd_chunks;
  if (I.peer && I.split) {
    // order + dispatch AlltoAll in one kernel per share: this rank's own
    // experts' rows first (local HBM), the peers' rows on s_aux over NVLink
    // while GEMM1 already runs on the local blocks
    const long long lo = static_cast<long long>(I.rank) * I.El * I.C, hi = lo + I.El * I.C;
    sp = I.tr.begin("order-local", 2, I.s_comp);
    I.peer_wait(I.slot_bar_fwd());
    throw_on(fsmoe_dispatch_peer_range(I.dtype, I.M, I.E, I.C, I.pos, I.tok, x, &I.map_X, lo, hi, 0,
                                       I.s_comp));
    cuda_check(cudaMemcpyAsync(I.rfill + I.rank * I.El, I.fill + I.rank * I.El, 8 * I.El,
                               cudaMemcpyDeviceToDevice, I.s_comp), "memcpy");
    I.tr.end(sp, I.s_comp);
    I.record(I.ev_x1, I.s_comp);
    I.wait(I.s_aux, I.ev_x1);
    throw_on(fsmoe_dispatch_peer_range(I.dtype, I.M, I.E, I.C, I.pos, I.tok, x, &I.map_X, lo, hi, 1,
                                       I.s_aux));
    I.peer_signal(I.slot_disp_fwd(0), I.fill, 8, &I.map_fill, I.s_aux);
    I.record(I.ev_x2, I.s_aux);
    sp = I.tr.begin("expert-local", 2, I.s_comp);
    I.expert_fwd(ch[0], 1);
    I.tr.end(sp, I.s_comp);
    sp = I.tr.begin("dispatch", 0, I.s_comp);
    I.peer_wait(I.slot_disp_fwd(0));
    I.wait(I.s_comp, I.ev_x2);
    I.tr.end(sp, I.s_comp);
    sp = I.tr.begin("expert[0]", 2, I.s_comp);
    I.expert_fwd(ch[0], 2);
    I.peer_signal(I.slot_comb_fwd(0));
    I.tr.end(sp, I.s_comp);
    sp = I.tr.begin("combine", 0, I.s_comp);
    I.peer_wait(I.slot_comb_fwd(0));
    I.tr.end(sp, I.s_comp);
  } else if (I.peer && I.ce) {
    // the permutation keeps own rows local and stages the peers' rows; the
    // copy engines ship chunk i while GEMM chunk i-1 runs
    sp = I.tr.begin("order-stage", 2, I.s_comp);
    I.peer_wait(I.slot_bar_fwd());
    throw_on(fsmoe_dispatch_peer(I.dtype, I.M, I.E, I.C, I.pos, I.tok, x, &I.stage_X, I.s_comp));
    I.tr.end(sp, I.s_comp);
    I.record(I.ev_ce, I.s_comp);
    I.wait(I.s_ce, I.ev_ce);
    throw_on(fsmoe_peer_copy_rows(I.fill, 8, &I.map_fill, 0, 1, 1, I.s_ce));
    for (size_t i = 0; i < ch.size(); ++i) {
      throw_on(fsmoe_peer_copy_rows(I.Xsend, static_cast<long long>(I.M) * I.esz, &I.map_X, ch[i].lo,
                                    ch[i].hi, 0, I.s_ce));
      I.ce_signal(I.slot_disp_fwd(i));
    }
    for (size_t i = 0; i < ch.size(); ++i) {
      sp = I.tr.begin("dispatch[" + std::to_string(i) + "]", 0, I.s_comp);
      I.peer_wait(I.slot_disp_fwd(i));
      I.tr.end(sp, I.s_comp);
      sp = I.tr.begin("expert[" + std::to_string(i) + "]", 2, I.s_comp);
      I.expert_fwd(ch[i]);
      I.peer_signal(I.slot_comb_fwd(i));
      I.tr.end(sp, I.s_comp);
    }
    sp = I.tr.begin("combine", 0, I.s_comp);
    for (size_t i = 0; i < ch.size(); ++i) I.peer_wait(I.slot_comb_fwd(i));
    I.tr.end(sp, I.s_comp);
  } else if (I.peer) {
    // order + dispatch AlltoAll in one kernel: rows go straight to their owner
    sp = I.tr.begin("dispatch", 0, I.s_comp);
    I.peer_wait(I.slot_bar_fwd());
    throw_on(fsmoe_dispatch_peer(I.dtype, I.M, I.E, I.C, I.pos, I.tok, x, &I.map_X, I.s_comp));
    I.peer_signal(I.slot_disp_fwd(0), I.fill, 8, &I.map_fill);
    I.peer_wait(I.slot_disp_fwd(0));
    I.tr.end(sp, I.s_comp);
    for (size_t i = 0; i < ch.size(); ++i) {
      // GEMM2's epilogue stores the combine AlltoAll into the owners' O_send
      sp = I.tr.begin("expert[" + std::to_string(i) + "]", 2, I.s_comp);
      I.expert_fwd(ch[i]);
      I.peer_signal(I.slot_comb_fwd(i));
      I.tr.end(sp, I.s_comp);
    }
    sp = I.tr.begin("combine", 0, I.s_comp);
    for (size_t i = 0; i < ch.size(); ++i) I.peer_wait(I.slot_comb_fwd(i));
    I.tr.end(sp, I.s_comp);
  } else {
    if (I.P > 1) {
      I.record(I.ev_gate, I.s_comp);
      I.wait(I.s_comm, I.ev_gate);
      I.exchange_fill();
      for (size_t i = 0; i < ch.size(); ++i) {
        sp = I.tr.begin("dispatch[" + std::to_string(i) + "]", 0, I.s_comm);
        I.exchange(I.Xs, I.Xr, ch[i]);
        I.tr.end(sp, I.s_comm);
        I.record(I.ev_a[i], I.s_comm);
      }
    }
    for (size_t i = 0; i < ch.size(); ++i) {
      if (I.P > 1) I.wait(I.s_comp, I.ev_a[i]);
      sp = I.tr.begin("expert[" + std::to_string(i) + "]", 2, I.s_comp);
      I.expert_fwd(ch[i]);
      I.tr.end(sp, I.s_comp);
      if (I.P > 1) I.record(I.ev_b[i], I.s_comp);
    }
    if (I.P > 1) {
      for (size_t i = 0; i < ch.size(); ++i) {
        I.wait(I.s_comm, I.ev_b[i]);
        sp = I.tr.begin("combine[" + std::to_string(i) + "]", 0, I.s_comm);
        I.exchange(I.Or, I.Os, ch[i]);
        I.tr.end(sp, I.s_comm);
      }
      I.record(I.ev_join, I.s_comm);
      I.wait(I.s_comp, I.ev_join);
    }
  }
  // K5 combine
  sp = I.tr.begin("i-order", 2, I.s_comp);
  if (I.scatter_y)  // GEMM2 wrote the kept rows; the dropped tokens' rows are 0
    throw_on(fsmoe_zero_rows(I.dtype, I.M, I.T, I.slot, y, I.s_comp));
  else if (I.unit_top1)  // every kept weight is exactly 1.0: y[t] = O[slot(t)] (0 if dropped)
    throw_on(fsmoe_gather_rows(I.dtype, I.M, I.T, I.slot, I.Os, y, nullptr, I.s_comp));
  else
    throw_on(fsmoe_combine(I.dtype, I.T, I.M, I.E, I.C, 1, I.tptr, I.tpick, I.slot, I.w, I.Os, y,
                           I.s_comp));
  I.tr.end(sp, I.s_comp);
  I.last_was_bwd = false;
  I.record(I.ev_out, I.s_comp);
  I.wait(st, I.ev_out);
  I.tr.flush("fwd");
}

void MoELayer::backward(const void* dy, void* dx, void* stream) {
  Impl& I = *impl_;
  cuda_check(cudaSetDevice(cfg_.device), "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  I.record(I.ev_in, st);
  I.wait(I.s_comp, I.ev_in);
  I.tr.start(I.s_comp);
  I.scatter_dx = I.fuse_top1 ? dx : nullptr;
  const MoEParams& p = I.prm;
  // gate gradients accumulate inside gate_bwd: start from zero
  const long long ge = static_cast<long long>(I.gd.score_rows) * I.E;
  cuda_check(cudaMemsetAsync(p.g_gate, 0, 8 * ge, I.s_comp), "memset");
  if (p.g_noise) cuda_check(cudaMemsetAsync(p.g_noise, 0, 8LL * I.M * I.E, I.s_comp), "memset");
  if (p.g_proj)
    cuda_check(cudaMemsetAsync(p.g_proj, 0, 8LL * cfg_.proj_dim * I.M, I.s_comp), "memset");
  const auto& ch = I.bwd_chunks;
  int sp = -1;
  if (I.peer) {
    // a backward directly after a backward: the peers' previous reads of
    // dO_recv / dX_send must be finished (after a forward its barrier did it)
    if (I.last_was_bwd) {
      I.peer_signal(I.slot_bar_bwd());
      I.peer_wait(I.slot_bar_bwd());
    }
    // I-order backward fused with the dispatch AlltoAll of dO
    const bool split_bwd = I.split && cfg_.precision == Precision::bf16;
    if (I.ce) {
      // I-order backward: own dO rows local, the peers' staged; the copy
      // engines ship chunk j while the expert backward of chunk j-1 runs
      sp = I.tr.begin("i-order", 2, I.s_comp);
      if (I.unit_top1)
        throw_on(fsmoe_dispatch_peer(I.dtype, I.M, I.E, I.C, I.pos, I.tok, dy, &I.stage_dO, I.s_comp));
      else
        throw_on(fsmoe_combine_bwd_peer(I.dtype, I.M, I.E, I.C, I.n_picks, I.pos, I.tok, I.w, dy, I.Os,
                                        &I.stage_dO, I.dw, I.s_comp));
      I.tr.end(sp, I.s_comp);
      I.record(I.ev_ce, I.s_comp);
      I.wait(I.s_ce, I.ev_ce);
      for (size_t j = 0; j < ch.size(); ++j) {
        throw_on(fsmoe_peer_copy_rows(I.dOsend, static_cast<long long>(I.M) * I.esz, &I.map_dO, ch[j].lo,
                                      ch[j].hi, 0, I.s_ce));
        I.ce_signal(I.slot_disp_bwd(j));
      }
    } else if (split_bwd) {
      // own experts' dO rows first, the peers' rows on s_aux over NVLink while
      // dgrad2 already runs on the local blocks
      const long long lo = static_cast<long long>(I.rank) * I.El * I.C, hi = lo + I.El * I.C;
      auto iorder = [&](int excl, cudaStream_t st_) {
        if (I.unit_top1)  // dO[slot] = 1.0 * dy[token]; d_weight feeds no gradient (gate_bwd.cu)
          throw_on(fsmoe_dispatch_peer_range(I.dtype, I.M, I.E, I.C, I.pos, I.tok, dy, &I.map_dO, lo,
                                             hi, excl, st_));
        else
          throw_on(fsmoe_combine_bwd_peer_range(I.dtype, I.M, I.E, I.C, I.n_picks, I.pos, I.tok, I.w,
                                                dy, I.Os, &I.map_dO, I.dw, lo, hi, excl, st_));
      };
      sp = I.tr.begin("i-order", 2, I.s_comp);
      if (!I.unit_top1)
        cuda_check(cudaMemsetAsync(I.dw, 0, 8 * I.n_picks, I.s_comp), "memset");
      iorder(0, I.s_comp);
      I.tr.end(sp, I.s_comp);
      I.record(I.ev_x1, I.s_comp);
      I.wait(I.s_aux, I.ev_x1);
      iorder(1, I.s_aux);
      I.peer_signal(I.slot_disp_bwd(0), nullptr, 0, nullptr, I.s_aux);
      I.record(I.ev_x2, I.s_aux);
      sp = I.tr.begin("expert-local", 2, I.s_comp);
      I.expert_bwd(ch[0], true, 1);
      I.tr.end(sp, I.s_comp);
      sp = I.tr.begin("dispatch", 0, I.s_comp);
      I.peer_wait(I.slot_disp_bwd(0));
      I.wait(I.s_comp, I.ev_x2);
      I.tr.end(sp, I.s_comp);
    } else {
      sp = I.tr.begin("i-order", 2, I.s_comp);
      if (I.unit_top1)  // dO[slot] = 1.0 * dy[token]; d_weight feeds no gradient (gate_bwd.cu)
        throw_on(fsmoe_dispatch_peer(I.dtype, I.M, I.E, I.C, I.pos, I.tok, dy, &I.map_dO, I.s_comp));
      else
        throw_on(fsmoe_combine_bwd_peer(I.dtype, I.M, I.E, I.C, I.n_picks, I.pos, I.tok, I.w, dy,
                                        I.Os, &I.map_dO, I.dw, I.s_comp));
      I.tr.end(sp, I.s_comp);
      sp = I.tr.begin("dispatch", 0, I.s_comp);
      I.peer_signal(I.slot_disp_bwd(0));
      I.peer_wait(I.slot_disp_bwd(0));
      I.tr.end(sp, I.s_comp);
    }
    if (I.prm.dense_grad && cfg_.dense_grad_elems > 0) {
      // gradient allreduce slices on the comm stream, overlapping expert backward
      I.record(I.ev_gate, I.s_comp);
      I.wait(I.s_comm, I.ev_gate);
      sp = I.tr.begin("grad_sync", 0, I.s_comm);
      I.allreduce_slices();
      I.tr.end(sp, I.s_comm);
      I.record(I.ev_join, I.s_comm);
    }
    for (size_t j = 0; j < ch.size(); ++j) {
      if (I.ce) {
        sp = I.tr.begin("dispatch[" + std::to_string(j) + "]", 0, I.s_comp);
        I.peer_wait(I.slot_disp_bwd(j));
        I.tr.end(sp, I.s_comp);
      }
      // dgrad1's epilogue stores the combine AlltoAll into the owners' dX_send
      sp = I.tr.begin("expert[" + std::to_string(j) + "]", 2, I.s_comp);
      I.expert_bwd(ch[j], j == 0, split_bwd ? 2 : 0);
      I.peer_signal(I.slot_comb_bwd(j));
      I.tr.end(sp, I.s_comp);
    }
    sp = I.tr.begin("combine", 0, I.s_comp);
    for (size_t j = 0; j < ch.size(); ++j) I.peer_wait(I.slot_comb_bwd(j));
    I.tr.end(sp, I.s_comp);
    if (I.prm.dense_grad && cfg_.dense_grad_elems > 0) I.wait(I.s_comp, I.ev_join);
  } else {
  // I-order backward: dO (send side) and d weights
  sp = I.tr.begin("i-order", 2, I.s_comp);
  if (I.unit_top1)
    throw_on(fsmoe_dispatch(I.dtype, I.M, I.E, I.C, 1, I.pos, I.tok, dy, I.dOs, I.s_comp));
  else
    throw_on(fsmoe_combine_bwd(I.dtype, I.T, I.M, I.E, I.C, 1, I.n_picks, I.pos, I.tok, I.w, I.slot,
                               dy, I.Os, I.dOs, I.dw, I.s_comp));
  I.tr.end(sp, I.s_comp);
  if (I.P > 1) {
    I.record(I.ev_gate, I.s_comp);
    I.wait(I.s_comm, I.ev_gate);
    for (size_t j = 0; j < ch.size(); ++j) {
      sp = I.tr.begin("dispatch[" + std::to_string(j) + "]", 0, I.s_comm);
      I.exchange(I.dOs, I.dOr, ch[j]);
      I.tr.end(sp, I.s_comm);
      I.record(I.ev_a[j], I.s_comm);
    }
    // gradient allreduce slices between the last dispatch and the first combine
    sp = I.tr.begin("grad_sync", 0, I.s_comm);
    I.allreduce_slices();
    I.tr.end(sp, I.s_comm);
  }
  for (size_t j = 0; j < ch.size(); ++j) {
    if (I.P > 1) I.wait(I.s_comp, I.ev_a[j]);
    sp = I.tr.begin("expert[" + std::to_string(j) + "]", 2, I.s_comp);
    I.expert_bwd(ch[j], j == 0);
    I.tr.end(sp, I.s_comp);
    if (I.P > 1) I.record(I.ev_b[j], I.s_comp);
  }
  if (I.P > 1) {
    for (size_t j = 0; j < ch.size(); ++j) {
      I.wait(I.s_comm, I.ev_b[j]);
      sp = I.tr.begin("combine[" + std::to_string(j) + "]", 0, I.s_comm);
      I.exchange(I.dXr, I.dXs, ch[j]);
      I.tr.end(sp, I.s_comm);
    }
    I.record(I.ev_join, I.s_comm);
    I.wait(I.s_comp, I.ev_join);
  }
  }
  // Order backward, then the gate's contribution to dx and its parameters
  sp = I.tr.begin("order", 2, I.s_comp);
  if (I.scatter_dx)  // dgrad1 wrote the kept rows; the dropped tokens' rows are 0
    throw_on(fsmoe_zero_rows(I.dtype, I.M, I.T, I.slot, dx, I.s_comp));
  else if (I.unit_top1)  // dx[t] = dX[slot(t)] (0 if dropped)
    throw_on(fsmoe_gather_rows(I.dtype, I.M, I.T, I.slot, I.dXs, dx, nullptr, I.s_comp));
  else
    throw_on(fsmoe_dispatch_bwd(I.dtype, I.T, I.M, I.E, I.C, 1, I.tptr, I.tpick, I.slot, I.dXs, dx,
                                0, I.s_comp));
  I.tr.end(sp, I.s_comp);
  if (!I.x_last) throw ConfigError("layer: backward before forward");
  sp = I.tr.begin("gate", 2, I.s_comp);
  throw_on(fsmoe_gate_bwd(&I.gd, I.x_last, p.w_gate, p.w_noise, p.proj,
                          I.tok, I.exp, I.w, I.dw, I.scores, I.noise, I.spread, I.proj_out, dx,
                          p.g_gate, p.g_noise, p.g_proj, I.gbwd_ws, I.gbwd_wsb, I.s_comp));
  I.tr.end(sp, I.s_comp);
  // A softmax over one survivor has a constant weight: the gate gradient is
  // exactly zero on every rank (gate_bwd.cu), so there is nothing to reduce.
  const bool gate_grad_zero = I.gd.top_k == 1 && cfg_.gate != GateKind::sigmoid_topk;
  if (I.P > 1 && !gate_grad_zero) {
    // replicated gate parameters: sum their gradients over the EP group
    I.record(I.ev_gate, I.s_comp);
    I.wait(I.s_comm, I.ev_gate);
    sp = I.tr.begin("gate_grad_sync", 0, I.s_comm);
    I.ep->group_start();
    I.ep->allreduce_sum(p.g_gate, static_cast<size_t>(ge), true, I.s_comm);
    if (p.g_noise) I.ep->allreduce_sum(p.g_noise, static_cast<size_t>(I.M) * I.E, true, I.s_comm);
    if (p.g_proj)
      I.ep->allreduce_sum(p.g_proj, static_cast<size_t>(cfg_.proj_dim) * I.M, true, I.s_comm);
    I.ep->group_end();
    I.tr.end(sp, I.s_comm);
    I.record(I.ev_join, I.s_comm);
    I.wait(I.s_comp, I.ev_join);
  }
  I.last_was_bwd = true;
  I.record(I.ev_out, I.s_comp);
  I.wait(st, I.ev_out);
  I.tr.flush("bwd");
}

void MoELayer::set_trace(bool on) {
  impl_->tr.on = on;
  impl_->tr.json.clear();
  impl_->tr.offset_ms = 0.0;
}

std::string MoELayer::trace_json() const {
  return "{\"displayTimeUnit\": \"ms\", \"traceEvents\": [\n" + impl_->tr.json + "\n]}\n";
}

void* MoELayer::buffer(const std::string& name, long long* bytes) const {
  auto it = impl_->bufs.find(name);
  if (it == impl_->bufs.end()) throw ConfigError("layer: unknown buffer " + name);
  if (bytes) *bytes = it->second.second;
  return it->second.first;
}

long long MoELayer::dropped_host() const {
  long long h = 0;
  cuda_check(cudaMemcpyAsync(&h, impl_->dropped, 8, cudaMemcpyDeviceToHost, impl_->s_comp), "copy");
  cuda_check(cudaStreamSynchronize(impl_->s_comp), "sync");
  return h;
}

}  // namespace fsmoe

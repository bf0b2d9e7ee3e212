// B200 device back end of the heterogeneous-ZeRO step (include/zp_runtime.h).
//
// One runtime per rank (one process per GPU). Everything the rank holds lives in one
// capped arena (the emulated HBM capacity): flat bf16 parameters, the bf16 gradient of the
// current micro-step, the stage's fp32 master / Adam state / accumulators, fixed workspaces,
// and — per step — the activations of the local micro-batch. OOM is the arena refusing the
// activation reservation, which is exactly the reference's `resident + act*b > total` rule
// (proj/core/src/hardware.cpp:152-158) realised by an allocator.
//
// Per micro-step: GPT forward/backward on sm_100a kernels (gemm.cu, kernels.cu); the local
// gradient is pre-weighted by b_i/B through the loss scale 1/(B*seq). Collectives per stage
// (proj/core/include/zeroplan/comm.hpp:25-37): Z0 all-reduce of the fp32 gradient at sync;
// Z1 reduce-scatter + all-gather at sync; Z2 bf16 reduce-scatter every micro-step + all-gather
// of updated parameters at sync; Z3 adds the forward/backward parameter all-gathers. The
// optimizer is AdamW on the rank's shard, fused with the shard's gradient accumulation.
// With NVLink peer access (the default when every rank can map every other rank's arena),
// the Z1/Z2 reduce-scatters are peer-memory pulls and the synchronisation point is one kernel:
// reduce-scatter + AdamW + all-gather (peer.cu). ZP_PEER=0 selects the NCCL path instead.
#include <cuda.h>
#include <nccl.h>

#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../../include/zp_runtime.h"
#include "profiler_search.hpp"
#include "attention.h"
#include "gemm.h"
#include "kernels.h"
#include "peer.h"

namespace zp {
namespace {

thread_local std::string g_err;

struct Fail {
  int code;
};

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      ::zp::g_err = std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #call;          \
      throw ::zp::Fail{ZP_ECUDA};                                                           \
    }                                                                                 \
  } while (0)
#define NK(call)                                                                      \
  do {                                                                                \
    ncclResult_t r_ = (call);                                                         \
    if (r_ != ncclSuccess) {                                                          \
      ::zp::g_err = std::string("NCCL: ") + ncclGetErrorString(r_) + " at " #call;         \
      throw ::zp::Fail{ZP_ENCCL};                                                           \
    }                                                                                 \
  } while (0)

[[noreturn]] void fail(int code, const std::string& msg) {
  g_err = msg;
  throw Fail{code};
}

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------------ arena
struct Arena {
  char* base = nullptr;
  size_t cap = 0, used = 0, high = 0;
  void* take(size_t bytes) {
    const size_t off = (used + 255) & ~size_t(255);
    if (off + bytes > cap) return nullptr;
    used = off + bytes;
    if (used > high) high = used;
    return base + off;
  }
  template <class T>
  T* take_n(int64_t n) {
    return static_cast<T*>(take(size_t(n) * sizeof(T)));
  }
};

// ------------------------------------------------------------------ parameter layout
struct Tensor {
  int64_t off = 0, rows = 0, cols = 0;
  int group = 0;
  int64_t numel() const { return rows * cols; }
};
// ZeRO-3 all-gather / reduce-scatter unit: the embedding (wte, wpe), each transformer layer,
// and the final LayerNorm. Each group's flat region is padded to a multiple of n*256 elements so
// rank r owns the r-th equal slice of every group.
struct Group {
  int64_t start = 0, len = 0;
  // [begin, end) ranges of the group (relative to start) that no tensor covers: alignment and
  // shard padding, the only elements of a group gradient the backward never writes
  std::vector<std::pair<int64_t, int64_t>> gaps;
};
struct LayerP {
  Tensor ln1_g, ln1_b, w_qkv, b_qkv, w_o, b_o, ln2_g, ln2_b, w_fc, b_fc, w_proj, b_proj;
  Tensor w_gu, w_down;  // Llama: gate/up (interleaved 32-row blocks) and down projections
};
struct Layout {
  Tensor wte, wpe, lnf_g, lnf_b, lm_head;
  std::vector<LayerP> layers;
  std::vector<Group> groups;  // 0 = embedding, 1..L = layers, L+1 = final LayerNorm
  std::map<std::string, Tensor> by_name;
  int64_t logical = 0, total = 0, max_layer_group = 0, max_group = 0;
};

Layout make_layout(const zp_gpt_config& c, int vocab_pad, int world) {
  Layout L;
  int64_t cur = 0;
  const int64_t unit = int64_t(world) * 256;
  auto open_group = [&]() { L.groups.push_back(Group{cur, 0}); };
  auto close_group = [&]() {
    Group& G = L.groups.back();
    const int64_t end = round_up(cur, unit);
    if (end > cur) G.gaps.push_back({cur - G.start, end - G.start});
    cur = end;
    G.len = cur - G.start;
  };
  auto add = [&](const std::string& name, int64_t r, int64_t k, int64_t logical_rows) {
    Tensor t;
    t.off = cur;
    t.rows = r;
    t.cols = k;
    t.group = int(L.groups.size()) - 1;
    const int64_t end = round_up(cur + r * k, 64);
    if (end > cur + r * k) L.groups.back().gaps.push_back({cur + r * k - L.groups.back().start, end - L.groups.back().start});
    cur = end;
    L.logical += logical_rows * k;
    L.by_name[name] = t;
    return t;
  };
  const int h = c.d_model, f = c.d_ff;
  if (c.arch == 1) {  // Llama family
    open_group();
    L.wte = add("wte", vocab_pad, h, c.vocab);
    close_group();
    for (int i = 0; i < c.n_layer; ++i) {
      const std::string p = "h" + std::to_string(i) + ".";
      open_group();
      LayerP l;
      l.ln1_g = add(p + "ln1_g", 1, h, 1);
      l.w_qkv = add(p + "w_qkv", 3 * h, h, 3 * h);
      l.w_o = add(p + "w_o", h, h, h);
      l.ln2_g = add(p + "ln2_g", 1, h, 1);
      l.w_gu = add(p + "w_gu", 2 * f, h, 2 * f);
      l.w_down = add(p + "w_down", h, f, h);
      close_group();
      L.layers.push_back(l);
      L.max_layer_group = std::max(L.max_layer_group, L.groups.back().len);
    }
    open_group();
    L.lnf_g = add("lnf_g", 1, h, 1);
    L.lm_head = add("lm_head", vocab_pad, h, c.vocab);
    close_group();
    L.total = cur;
    for (const Group& g : L.groups) L.max_group = std::max(L.max_group, g.len);
    return L;
  }
  open_group();
  L.wte = add("wte", vocab_pad, h, c.vocab);
  L.wpe = add("wpe", c.seq_len, h, c.seq_len);
  close_group();
  for (int i = 0; i < c.n_layer; ++i) {
    const std::string p = "h" + std::to_string(i) + ".";
    open_group();
    LayerP l;
    l.ln1_g = add(p + "ln1_g", 1, h, 1);
    l.ln1_b = add(p + "ln1_b", 1, h, 1);
    l.w_qkv = add(p + "w_qkv", 3 * h, h, 3 * h);
    l.b_qkv = add(p + "b_qkv", 1, 3 * h, 1);
    l.w_o = add(p + "w_o", h, h, h);
    l.b_o = add(p + "b_o", 1, h, 1);
    l.ln2_g = add(p + "ln2_g", 1, h, 1);
    l.ln2_b = add(p + "ln2_b", 1, h, 1);
    l.w_fc = add(p + "w_fc", f, h, f);
    l.b_fc = add(p + "b_fc", 1, f, 1);
    l.w_proj = add(p + "w_proj", h, f, h);
    l.b_proj = add(p + "b_proj", 1, h, 1);
    close_group();
    L.layers.push_back(l);
    L.max_layer_group = std::max(L.max_layer_group, L.groups.back().len);
  }
  open_group();
  L.lnf_g = add("lnf_g", 1, h, 1);
  L.lnf_b = add("lnf_b", 1, h, 1);
  close_group();
  L.total = cur;
  for (const Group& g : L.groups) L.max_group = std::max(L.max_group, g.len);
  return L;
}

// ------------------------------------------------------------------ activations of one micro-step
struct LayerActs {
  // u: GPT-2 GELU'(fc pre-activation) saved by the fc GEMM epilogue for the backward;
  //    Llama gate/up projection (interleaved) for SwiGLU. g: MLP activation.
  bf16 *x_in, *ln1, *qkv, *attn, *x_mid, *ln2, *u, *g;
  float *mu1, *rs1, *mu2, *rs2, *lse;
};
struct Acts {
  int64_t b = 0;
  std::vector<LayerActs> l;
  bf16 *x_final, *lnf, *logits;
  float *muf, *rsf, *row_loss;
  float* dvec;  // [b, H, s] rowsum(dO * O)
  float* dq32;  // [T, h] fp32 dQ accumulator of the fused attention backward
  bf16 *dx, *dx2, *dln, *dO, *dqkv, *du;
  bf16* dh;  // Llama: gradient of the SwiGLU output [T, f] (du is then [T, 2f])
};

// ------------------------------------------------------------------ event timing
enum SpanKind { kFwd = 0, kBwd = 1, kComm = 2, kOpt = 3, kWall = 4, kAgF = 5, kAgB = 6, kRs = 7, kSync = 8 };
struct Span {
  int kind, start, end;
  bool nested;  // a collective issued inside a forward/backward span (ZeRO-3 gathers / scatters)
};
struct Timer {
  std::vector<cudaEvent_t> ev;
  std::vector<Span> spans;
  int next = 0;
  bool in_compute = false;  // set while a forward/backward span is open
  void init(int n) {
    ev.resize(n);
    for (auto& e : ev) CK(cudaEventCreate(&e));
  }
  void destroy() {
    for (auto& e : ev) cudaEventDestroy(e);
    ev.clear();
  }
  void reset() {
    next = 0;
    spans.clear();
  }
  // The pool grows on demand (event creation is host-only and does not synchronise), so a plan
  // with many micro-steps or ZeRO-3 groups never runs out of events mid-iteration.
  int mark(cudaStream_t s) {
    if (next >= int(ev.size())) {
      const size_t old = ev.size();
      ev.resize(std::max<size_t>(256, 2 * old));
      for (size_t i = old; i < ev.size(); ++i) CK(cudaEventCreate(&ev[i]));
    }
    CK(cudaEventRecord(ev[next], s));
    return next++;
  }
  void close(int kind, int start, cudaStream_t s) {
    const bool coll = kind == kComm || kind == kAgF || kind == kAgB || kind == kRs || kind == kSync;
    spans.push_back({kind, start, mark(s), coll && in_compute});
  }
};

// ------------------------------------------------------------------ green contexts
// An SM budget is enforced with a green context (driver API, resolved at run time): the rank's
// stream belongs to an SM partition of `budget` SMs (rounded down to the hardware granularity of
// 8), so every kernel on it — GEMMs, attention, the HBM-bound elementwise kernels, the peer
// collectives and NCCL's own kernels — runs on those SMs only. Grid caps stay as the fallback
// (ZP_GREEN=0, or a driver without green contexts).
struct GreenCtx {
  CUgreenCtx ctx = nullptr;
  int sms = 0;
};
template <class F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}
bool make_green_stream(int device, int budget, GreenCtx* g, cudaStream_t* st) {
  using GetDev = CUresult (*)(CUdevice*, int);
  using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
  using Split = CUresult (*)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*, unsigned int,
                             unsigned int);
  using GenDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned int);
  using Create = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
  using MkStream = CUresult (*)(CUstream*, CUgreenCtx, unsigned int, int);
  using Destroy = CUresult (*)(CUgreenCtx);
  auto get_dev = driver_fn<GetDev>("cuDeviceGet");
  auto get_res = driver_fn<GetRes>("cuDeviceGetDevResource");
  auto split = driver_fn<Split>("cuDevSmResourceSplitByCount");
  auto gen = driver_fn<GenDesc>("cuDevResourceGenerateDesc");
  auto create = driver_fn<Create>("cuGreenCtxCreate");
  auto mk = driver_fn<MkStream>("cuGreenCtxStreamCreate");
  auto destroy = driver_fn<Destroy>("cuGreenCtxDestroy");
  if (!get_dev || !get_res || !split || !gen || !create || !mk || !destroy) return false;
  CUdevice dev;
  CUdevResource all{}, part{}, rest{};
  if (get_dev(&dev, device) != CUDA_SUCCESS || get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
    return false;
  const unsigned want = unsigned(std::max(8, budget / 8 * 8));
  unsigned groups = 1;
  if (split(&part, &groups, &all, &rest, 0, want) != CUDA_SUCCESS || groups != 1) return false;
  CUdevResourceDesc desc = nullptr;
  if (gen(&desc, &part, 1) != CUDA_SUCCESS) return false;
  if (create(&g->ctx, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return false;
  CUstream s = nullptr;
  if (mk(&s, g->ctx, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) {
    destroy(g->ctx);
    g->ctx = nullptr;
    return false;
  }
  g->sms = int(part.sm.smCount);
  *st = reinterpret_cast<cudaStream_t>(s);
  return true;
}
void destroy_green(GreenCtx* g) {
  using Destroy = CUresult (*)(CUgreenCtx);
  if (!g->ctx) return;
  if (auto destroy = driver_fn<Destroy>("cuGreenCtxDestroy")) destroy(g->ctx);
  g->ctx = nullptr;
}

}  // namespace

// ------------------------------------------------------------------ runtime
struct Runtime {
  zp_runtime_desc d{};
  zp_gpt_config c{};
  int vocab_pad = 0;
  int n = 1, rank = 0;
  int ctas = 148;
  GreenCtx green;  // SM partition of the rank (green.ctx == nullptr: grid caps only)
  cudaStream_t st = nullptr;
  ncclComm_t comm = nullptr;
  Layout lay;
  Arena arena;
  // NVLink peer-memory collectives (peer.h): every rank's arena and flag block mapped here
  PeerView pv;
  bool peer = false;
  // Z3 gathers are peer-load kernels only (no copy-engine pulls / prefetch): ranks that share one
  // process (the device-seam backend), or ZP_Z3_KERNEL_GATHER=1
  bool kernel_gathers = false;
  uint32_t epoch = 0;
  PeerFlags* flags = nullptr;
  std::vector<void*> ipc_open;
  int64_t off(const void* p) const { return static_cast<const char*>(p) - arena.base; }
  int stage = -1;
  size_t resident_mark = 0;
  int64_t adam_t = 0;
  bool keep_grads = false;

  // persistent state (per configured stage)
  bf16* p16 = nullptr;   // [total] full bf16 parameters
  bf16* g16 = nullptr;   // [total] bf16 gradient of the current micro-step
  float* p32 = nullptr;  // master (full at Z0, shard otherwise)
  float* m32 = nullptr;
  float* v32 = nullptr;
  float* acc = nullptr;   // Z0/1: [total] fp32 local accumulation; Z2: [shard] accumulation
  float* r32 = nullptr;   // Z1: [shard] reduce-scatter output
  bf16* r16 = nullptr;    // Z2: [shard] reduce-scatter output
  float* gkeep = nullptr; // summed gradient of the last iteration (parity)
  // ZeRO-3: parameters exist only as this rank's shard plus per-group gather buffers
  bf16* p16s = nullptr;          // [shard] bf16 parameter shard (shard order)
  bf16* gb_emb = nullptr;        // gathered embedding group (kept for the whole micro-step)
  bf16* gb_fin = nullptr;        // gathered final-LN group
  bf16* gb_layer[2] = {nullptr, nullptr};  // gathered transformer layer (double buffer)
  bf16* ggrp = nullptr;          // gradient of the group being reduced
  std::vector<int64_t> shoff;    // shard-order offset of each group's owned slice
  struct Owned {
    int64_t flat_begin, flat_end, shard_begin;
  };
  std::vector<Owned> owned;      // flat ranges whose master / Adam state this rank holds
  float* dwte32 = nullptr;
  float* dwpe32 = nullptr;
  float* wgrad32 = nullptr;
  float* ln_part = nullptr;
  float* cs_part = nullptr;  // column partials of a LayerNorm backward's output (bias gradients)
  float* col_work = nullptr;
  float* loss_steps = nullptr;  // [kMaxSteps]
  int32_t* tokens = nullptr;
  int64_t tokens_cap = 0, tokens_count = 0;
  float last_gscale = 0.f;
  cudaEvent_t marks[8] = {};
  Timer tm;
  static constexpr int kMaxSteps = 4096;

  int hd() const { return c.d_model / c.n_head; }  // head_dim (64 or 128)
  int64_t shard() const { return lay.total / n; }
  int64_t shard_begin() const { return stage == 0 ? 0 : (stage == 3 ? 0 : shard() * rank); }
  int64_t state_len() const { return stage == 0 ? lay.total : shard(); }

  void set_owned() {
    owned.clear();
    shoff.assign(lay.groups.size(), 0);
    if (stage == 0) {
      owned.push_back({0, lay.total, 0});
    } else if (stage <= 2) {
      owned.push_back({shard() * rank, shard() * (rank + 1), 0});
    } else {
      int64_t so = 0;
      for (size_t g = 0; g < lay.groups.size(); ++g) {
        const Group& G = lay.groups[g];
        const int64_t part = G.len / n;
        shoff[g] = so;
        owned.push_back({G.start + part * rank, G.start + part * (rank + 1), so});
        so += part;
      }
    }
  }

  // Parameter / gradient pointer of a tensor for the configured stage.
  const bf16* Wp(const Tensor& t) const {
    if (stage != 3) return p16 + t.off;
    if (n == 1) return p16s + t.off;  // one rank: shard order == flat order
    const Group& G = lay.groups[t.group];
    const bf16* base = t.group == 0 ? gb_emb
                     : (t.group == int(lay.groups.size()) - 1 ? gb_fin : gb_layer[(t.group - 1) & 1]);
    return base + (t.off - G.start);
  }
  // Gradient destination of a tensor. When the rank's fp32 accumulator covers every parameter it
  // computes (ZeRO-0/1, or a single rank) the gradient producers write the first micro-step's
  // gradient straight into it and add the later ones (GEMM fp32 epilogues, fp32 column sums), so
  // no bf16 gradient buffer and no per-micro-step accumulation pass exist; otherwise they write
  // bf16 (Gp) for the stage's reduce-scatter.
  struct GradDst {
    bf16* b16;
    float* f32;
    bool first;
  };
  bool direct = false;  // set by configure(): stage <= 1 || n == 1
  bool gfirst = true;   // the current micro-step is the iteration's first with local work
  GradDst Gd(const Tensor& t) const {
    if (direct) return {nullptr, acc + t.off, gfirst};
    return {Gp(t), nullptr, false};
  }
  void grad_partials(const float* part, int nparts, int N, GradDst d) {
    sum_partials(part, nparts, N, d.b16, st, d.f32, d.f32 && !d.first);
  }
  // an fp32 gradient computed in a workspace (embedding tables): cast, or copy / add into acc
  void grad_from_f32(const float* src, int64_t n, GradDst d) {
    if (!d.f32)
      cast_f32_bf16(src, d.b16, n, ctas, st);
    else if (d.first)
      CK(cudaMemcpyAsync(d.f32, src, size_t(n) * 4, cudaMemcpyDeviceToDevice, st));
    else
      add_f32(d.f32, src, n, ctas, st);
  }
  bf16* Gp(const Tensor& t) const {
    if (stage != 3) return g16 + t.off;
    if (n == 1) return r16 + t.off;
    return ggrp + (t.off - lay.groups[t.group].start);
  }

  // ---------------------------------------------------------------- GEMM helpers
  // Optional per-launch event timing of the dense (non-attention) GEMMs, for the roofline
  // numbers bench.py reports (zp_runtime_gemm_stats).
  bool gemm_timing = false;
  struct GemmRec {
    int s, e;
    double flops;
  };
  std::vector<GemmRec> grec;
  Timer gtm;

  void launch_gemm(const GemmArgs& g, double dense_flops) {
    int s0 = -1;
    if (gemm_timing && dense_flops > 0) s0 = gtm.mark(st);
    CK(gemm(g, st));
    if (s0 >= 0) grec.push_back({s0, gtm.mark(st), dense_flops});
  }
  void mm(int M, int N, int K, const bf16* A, int amaj, int64_t lda, const bf16* B, int bmaj,
          int64_t ldb, void* C, int64_t ldc, int epi, float alpha = 1.f, const bf16* bias = nullptr,
          const bf16* aux = nullptr, bf16* aux_out = nullptr, int split_k = 1, float* colsum = nullptr) {
    GemmArgs g;
    g.M = M; g.N = N; g.K = K;
    g.a.ptr = A; g.a.major = amaj; g.a.ld = lda;
    g.b.ptr = B; g.b.major = bmaj; g.b.ld = ldb;
    g.c = C; g.ldc = ldc;
    g.alpha = alpha; g.epilogue = epi; g.bias = bias; g.aux = aux; g.aux_out = aux_out;
    g.max_ctas = ctas;
    g.split_k = split_k;
    g.colsum = colsum;
    launch_gemm(g, 2.0 * M * double(N) * K);
  }
  // Llama QKV projection with the rotary embedding of Q and K applied in the GEMM epilogue on the
  // fp32 accumulators (kEpiRopeBf16); the inverse rotation of dQ / dK happens in the head_dim-128
  // attention backward. ZP_ROPE_EPI=0 keeps the separate in-place rope kernels.
  static bool dvec_epi_on() {  // ZP_DVEC_EPI=0: separate D-vector kernel + dQ workspace memset
    static const bool on = !std::getenv("ZP_DVEC_EPI") || std::atoi(std::getenv("ZP_DVEC_EPI")) != 0;
    return on;
  }
  static bool swiglu_epi() {  // ZP_SWIGLU_EPI=0: separate SwiGLU backward kernel
    static const bool on = !std::getenv("ZP_SWIGLU_EPI") || std::atoi(std::getenv("ZP_SWIGLU_EPI")) != 0;
    return on;
  }
  static bool rope_epi() {
    static const bool on = !std::getenv("ZP_ROPE_EPI") || std::atoi(std::getenv("ZP_ROPE_EPI")) != 0;
    return on;
  }
  void qkv_rope(int64_t T, const bf16* x, const bf16* w, bf16* qkv) {
    const int h = int(c.d_model);
    const float2* tab = rope_epi() ? rope_table(int(c.seq_len), hd(), 10000.f, st) : nullptr;
    if (!tab) {
      mm(int(T), 3 * h, h, x, kKMajor, h, w, kKMajor, h, qkv, 3 * h, kEpiStoreBf16);
      rope(qkv, T, int(c.seq_len), h, 10000.f, false, ctas, st, hd());
      return;
    }
    GemmArgs g;
    g.M = int(T); g.N = 3 * h; g.K = h;
    g.a.ptr = x; g.a.major = kKMajor; g.a.ld = h;
    g.b.ptr = w; g.b.major = kKMajor; g.b.ld = h;
    g.c = qkv; g.ldc = 3 * h;
    g.epilogue = kEpiRopeBf16;
    g.rope_tab = tab; g.rope_seq = int(c.seq_len); g.rope_dh = hd(); g.rope_cols = 2 * h;
    g.max_ctas = ctas;
    launch_gemm(g, 2.0 * double(T) * 3 * h * h);
  }
  // Weight gradient dW[M, N] = sum over the T tokens: few output tiles, very long K. Split K
  // across CTAs (fp32 atomics into a workspace, then a cast) when the tiles cannot fill the
  // rank's SMs.
  void wgrad(int M, int N, int64_t T, const bf16* A, int64_t lda, const bf16* B, int64_t ldb,
             GradDst d) {
    const int bn = N <= 64 ? 64 : (N <= 128 ? 128 : 256);
    const int64_t tiles = int64_t((M + 127) / 128) * ((N + bn - 1) / bn);
    const int64_t kblocks = (T + 63) / 64;
    int split = 1;
    if (tiles < ctas) split = int(std::min<int64_t>((ctas + tiles - 1) / tiles, std::max<int64_t>(1, kblocks / 16)));
    if (d.f32) {  // straight into the fp32 accumulator
      if (d.first && split <= 1) {
        mm(M, N, int(T), A, kMNMajor, lda, B, kMNMajor, ldb, d.f32, N, kEpiStoreF32);
      } else {
        // later micro-steps add with fire-and-forget vector reductions (the L2 does the
        // read-modify-write; an epilogue that read C back would stall on every tile)
        if (d.first) CK(cudaMemsetAsync(d.f32, 0, size_t(M) * N * 4, st));
        mm(M, N, int(T), A, kMNMajor, lda, B, kMNMajor, ldb, d.f32, N, kEpiAtomicF32, 1.f, nullptr, nullptr, nullptr,
           split > 1 ? -1 : 1);
      }
      return;
    }
    bf16* dst = d.b16;
    if (split <= 1) {
      mm(M, N, int(T), A, kMNMajor, lda, B, kMNMajor, ldb, dst, N, kEpiStoreBf16);
      return;
    }
    CK(cudaMemsetAsync(wgrad32, 0, size_t(M) * N * 4, st));
    mm(M, N, int(T), A, kMNMajor, lda, B, kMNMajor, ldb, wgrad32, N, kEpiAtomicF32, 1.f, nullptr, nullptr,
       nullptr, -1);  // split count chosen by the launcher for full waves of its tile shape
    cast_f32_bf16(wgrad32, dst, int64_t(M) * N, ctas, st);
  }

  // ---------------------------------------------------------------- activation plan
  // Carves one micro-step's activations from `ar` (or only counts bytes when ar == nullptr).
  size_t plan_acts(int64_t b, Acts* a, Arena* ar) {
    const int64_t s = c.seq_len, h = c.d_model, f = c.d_ff, H = c.n_head, T = b * s;
    size_t bytes = 0;
    auto take = [&](int64_t nbytes) -> void* {
      bytes = ((bytes + 255) & ~size_t(255)) + size_t(nbytes);
      if (!ar) return nullptr;
      void* p = ar->take(size_t(nbytes));
      if (!p) fail(ZP_OOM, "activation reservation exceeds the HBM cap");
      return p;
    };
    auto B16 = [&](int64_t nel) { return static_cast<bf16*>(take(nel * 2)); };
    auto F32 = [&](int64_t nel) { return static_cast<float*>(take(nel * 4)); };
    Acts tmp;
    Acts& A = a ? *a : tmp;
    A.b = b;
    A.l.resize(c.n_layer);
    for (int i = 0; i < c.n_layer; ++i) {
      LayerActs& L = A.l[i];
      L.x_in = B16(T * h);
      L.ln1 = B16(T * h);
      L.qkv = B16(T * 3 * h);
      L.attn = B16(T * h);
      L.x_mid = B16(T * h);
      L.ln2 = B16(T * h);
      L.u = B16(T * f * (c.arch == 1 ? 2 : 1));
      L.g = B16(T * f);
      L.mu1 = F32(T);
      L.rs1 = F32(T);
      L.mu2 = F32(T);
      L.rs2 = F32(T);
      L.lse = F32(b * H * s);
    }
    A.x_final = B16(T * h);
    A.lnf = B16(T * h);
    A.muf = F32(T);
    A.rsf = F32(T);
    A.logits = B16(T * vocab_pad);
    A.row_loss = F32(T);
    A.dvec = F32(b * H * s);
    A.dq32 = F32(T * h);
    A.dx = B16(T * h);
    A.dx2 = B16(T * h);
    A.dln = B16(T * h);
    A.dO = B16(T * h);
    A.dqkv = B16(T * 3 * h);
    A.du = B16(T * f * (c.arch == 1 ? 2 : 1));
    A.dh = c.arch == 1 ? B16(T * f) : nullptr;
    return bytes;
  }

  // ---------------------------------------------------------------- stage configuration
  void configure(int new_stage) {
    if (new_stage == stage) return;
    if (new_stage < 0 || new_stage > 3) fail(ZP_EINVAL, "stage must be 0, 1, 2 or 3");
    arena.used = 0;
    arena.high = 0;
    stage = -1;
    const int64_t T = lay.total, S = shard();
    auto must = [&](void* p, const char* what) {
      if (!p) fail(ZP_OOM, std::string("resident state does not fit the HBM cap: ") + what);
      return p;
    };
    auto B16 = [&](int64_t nel, const char* what) { return static_cast<bf16*>(must(arena.take_n<bf16>(nel), what)); };
    auto F32 = [&](int64_t nel, const char* what) { return static_cast<float*>(must(arena.take_n<float>(nel), what)); };
    p16 = g16 = p16s = r16 = ggrp = gb_emb = gb_fin = nullptr;
    gb_layer[0] = gb_layer[1] = nullptr;
    acc = r32 = nullptr;
    const int64_t SL = new_stage == 0 ? T : S;
    direct = new_stage <= 1 || n == 1;  // gradients accumulate straight into the fp32 accumulator
    if (new_stage <= 2) {
      p16 = B16(T, "bf16 params");
      if (!direct) g16 = B16(T, "bf16 grads");
    } else {
      p16s = B16(S, "bf16 param shard");
      if (n > 1) {
        gb_emb = B16(lay.groups.front().len, "embedding gather buffer");
        gb_fin = B16(lay.groups.back().len, "final gather buffer");
        gb_layer[0] = B16(lay.max_layer_group, "layer gather buffer 0");
        gb_layer[1] = B16(lay.max_layer_group, "layer gather buffer 1");
        ggrp = B16(lay.max_group, "group gradient");
        ggrp_buf[0] = ggrp;
        ggrp_buf[1] = rs_stage[0] = rs_stage[1] = nullptr;
        z3_async = z3_async_ok();
        if (z3_async) {
          ggrp_buf[1] = B16(lay.max_group, "group gradient 1");
          rs_stage[0] = B16(lay.max_group, "reduce-scatter staging 0");
          rs_stage[1] = B16(lay.max_group, "reduce-scatter staging 1");
        }
        z3_cur = 0;
        pend_g = -1;
      }
    }
    p32 = F32(SL, "master params");
    m32 = F32(SL, "adam m");
    v32 = F32(SL, "adam v");
    if (new_stage <= 1) acc = F32(T, "grad accumulator");
    if (new_stage == 1) r32 = F32(S, "rs shard");
    if (new_stage >= 2) {
      acc = F32(S, "grad accumulator shard");
      if (!direct) r16 = B16(S, "rs shard");
    }
    gkeep = keep_grads ? F32(SL, "kept grads") : nullptr;
    const int64_t h = c.d_model;
    dwte32 = F32(int64_t(vocab_pad) * h, "dwte");
    dwpe32 = F32(int64_t(c.seq_len) * h, "dwpe");
    wgrad32 = F32(std::max<int64_t>(3 * h, 2 * int64_t(c.d_ff)) * h, "wgrad");
    ln_part = F32(int64_t(2) * 4 * 148 * h, "ln partials");
    cs_part = F32(int64_t(4) * 148 * h, "bias colsum partials");
    const int64_t maxN = std::max<int64_t>(3 * h, c.d_ff);
    col_work = F32(256 * maxN, "colsum work");
    loss_steps = F32(kMaxSteps, "loss");
    stage = new_stage;
    set_owned();
    resident_mark = arena.used;
    if (g16) CK(cudaMemsetAsync(g16, 0, size_t(T) * 2, st));
    if (ggrp) CK(cudaMemsetAsync(ggrp, 0, size_t(lay.max_group) * 2, st));
    if (ggrp_buf[1]) CK(cudaMemsetAsync(ggrp_buf[1], 0, size_t(lay.max_group) * 2, st));
    if (r16) CK(cudaMemsetAsync(r16, 0, size_t(S) * 2, st));
    CK(cudaMemsetAsync(m32, 0, size_t(SL) * 4, st));
    CK(cudaMemsetAsync(v32, 0, size_t(SL) * 4, st));
    init_params();
    adam_t = 0;
    CK(cudaStreamSynchronize(st));
  }

  // GPT-2 initialisation, a pure function of (seed, flat index): identical on every rank for
  // every sharding. Residual projections use std 0.02/sqrt(2L).
  void init_params() {
    auto init = [&](const Tensor& t, int kind, float stdv) {
      const float val = kind == 1 ? 1.f : 0.f;
      if (p16) {  // full bf16 copy (stages 0-2)
        if (kind == 0)
          init_normal(nullptr, p16 + t.off, t.numel(), stdv, d.seed, uint64_t(t.off), ctas, st);
        else
          init_const(nullptr, p16 + t.off, t.numel(), val, ctas, st);
      }
      for (const Owned& o : owned) {  // master (and the Z3 bf16 shard) over the owned ranges
        const int64_t a = std::max(o.flat_begin, t.off), e = std::min(o.flat_end, t.off + t.numel());
        if (a >= e) continue;
        float* dst = p32 + o.shard_begin + (a - o.flat_begin);
        bf16* dst16 = p16s ? p16s + o.shard_begin + (a - o.flat_begin) : nullptr;
        if (kind == 0)
          init_normal(dst, dst16, e - a, stdv, d.seed, uint64_t(a), ctas, st);
        else
          init_const(dst, dst16, e - a, val, ctas, st);
      }
    };
    const float sp = 0.02f / std::sqrt(2.0f * c.n_layer);
    // padding between tensors stays zero
    if (p16) CK(cudaMemsetAsync(p16, 0, size_t(lay.total) * 2, st));
    if (p16s) CK(cudaMemsetAsync(p16s, 0, size_t(shard()) * 2, st));
    CK(cudaMemsetAsync(p32, 0, size_t(state_len()) * 4, st));
    Tensor wte_real = lay.wte;
    wte_real.rows = c.vocab;  // padded vocabulary rows stay zero
    init(wte_real, 0, 0.02f);
    if (c.arch == 1) {
      for (const LayerP& l : lay.layers) {
        init(l.ln1_g, 1, 0);
        init(l.w_qkv, 0, 0.02f);
        init(l.w_o, 0, sp);
        init(l.ln2_g, 1, 0);
        init(l.w_gu, 0, 0.02f);
        init(l.w_down, 0, sp);
      }
      init(lay.lnf_g, 1, 0);
      Tensor head_real = lay.lm_head;
      head_real.rows = c.vocab;
      init(head_real, 0, 0.02f);
      return;
    }
    init(lay.wpe, 0, 0.01f);
    for (const LayerP& l : lay.layers) {
      init(l.ln1_g, 1, 0); init(l.ln1_b, 2, 0);
      init(l.w_qkv, 0, 0.02f); init(l.b_qkv, 2, 0);
      init(l.w_o, 0, sp); init(l.b_o, 2, 0);
      init(l.ln2_g, 1, 0); init(l.ln2_b, 2, 0);
      init(l.w_fc, 0, 0.02f); init(l.b_fc, 2, 0);
      init(l.w_proj, 0, sp); init(l.b_proj, 2, 0);
    }
    init(lay.lnf_g, 1, 0);
    init(lay.lnf_b, 2, 0);
  }

  // ---------------------------------------------------------------- ZeRO-3 group collectives
  // Issue order is fixed (every rank, with or without work, calls the same sequence):
  //   forward : AG(0), AG(1) .. AG(L), AG(L+1)
  //   backward: RS(L+1), then AG(i), RS(i) for i = L .. 1, then RS(0)
  bf16* gather_dst(int g) {
    if (g == 0) return gb_emb;
    if (g == int(lay.groups.size()) - 1) return gb_fin;
    return gb_layer[(g - 1) & 1];
  }
  // Over NVLink the first gather of an iteration is the barrier kernel (every rank's shard is
  // final once all ranks reach it: the optimizer precedes it in each rank's stream). Later
  // gathers are one-sided copy-engine pulls from the mapped peer shards; the next layer in issue
  // order is pulled on a side stream while the current layer computes. Gathered groups stay
  // valid until the next optimizer step, so the embedding, the final group and the two layers
  // still in the double buffer at a forward/backward turn are not gathered again.
  cudaStream_t cst = nullptr;             // gather prefetch stream (peer path)
  cudaEvent_t ev_free = nullptr;          // main stream finished with the buffer being refilled
  cudaEvent_t ev_done[2] = {};            // prefetch into gb_layer[i] landed
  int buf_holds[2] = {-1, -1};            // group held (or being pulled) in gb_layer[i]
  bool buf_pending[2] = {false, false};
  bool emb_res = false, fin_res = false, z3_fresh = true;
  void z3_invalidate() {
    z3_fresh = true;
    buf_holds[0] = buf_holds[1] = -1;
    emb_res = fin_res = false;
  }
  void z3_pull(int g, cudaStream_t s) {
    const int64_t part = lay.groups[g].len / n;
    bf16* dst = gather_dst(g);
    for (int k = 1; k <= n; ++k) {  // start at the next rank: no GPU is read by every peer at once
      const int j = (rank + k) % n;
      CK(cudaMemcpyAsync(dst + part * j, pv.base[j] + off(p16s + shoff[g]), size_t(part) * 2,
                         cudaMemcpyDeviceToDevice, s));
    }
  }
  void z3_note(int g) {
    if (g == 0)
      emb_res = true;
    else if (g == int(lay.groups.size()) - 1)
      fin_res = true;
    else
      buf_holds[(g - 1) & 1] = g;
  }
  void z3_gather(int g, int kind) {
    if (stage != 3 || n == 1) return;
    const Group& G = lay.groups[g];
    const int s0 = tm.mark(st);
    if (!peer) {
      NK(ncclAllGather(p16s + shoff[g], gather_dst(g), size_t(G.len / n), ncclBfloat16, comm, st));
      tm.close(kind, s0, st);
      return;
    }
    const bool layer = g >= 1 && g <= c.n_layer;
    const int b = (g - 1) & 1;
    if (layer && buf_pending[b]) {  // a pull into this buffer is in flight (normally: this group's)
      CK(cudaStreamWaitEvent(st, ev_done[b], 0));
      buf_pending[b] = false;
    }
    if (z3_fresh || kernel_gathers) {
      CK(peer_all_gather(pv, off(p16s + shoff[g]), gather_dst(g), G.len / n, ++epoch, ctas, st));
      z3_fresh = false;
      z3_note(g);
    } else if (layer ? buf_holds[b] != g : !(g == 0 ? emb_res : fin_res)) {
      z3_pull(g, st);
      z3_note(g);
    }
    tm.close(kind, s0, st);
    const int nx = kind == kAgB ? g - 1 : g + 1;  // next layer group in issue order
    if (!kernel_gathers && nx >= 1 && nx <= c.n_layer && buf_holds[(nx - 1) & 1] != nx) {
      const int nb = (nx - 1) & 1;
      CK(cudaEventRecord(ev_free, st));
      CK(cudaStreamWaitEvent(cst, ev_free, 0));
      z3_pull(nx, cst);
      CK(cudaEventRecord(ev_done[nb], cst));
      buf_holds[nb] = nx;
      buf_pending[nb] = true;
    }
  }
  // ---- ZeRO-3 reduce-scatter on the copy engines (ZP_Z3_ASYNC_RS=1, NVLink ranks in separate
  // processes). The group gradient alternates between two buffers. When a group's gradient is
  // final, stream memory operations tell every peer so (rs_ready). Each rank's side stream `rst`
  // waits for those flags and pulls its slice of every peer's buffer with cudaMemcpyAsync, which
  // needs no SMs and overlaps the next layer's backward. It then tells the peers it is done
  // (rs_pulled). One group later, a short HBM-bound kernel adds the pulled slices and the rank's
  // own slice into the fp32 shard accumulator, in rank order. A buffer is rewritten only after
  // every peer has pulled from it.
  using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  WaitFn mem_wait = nullptr;
  WriteFn mem_write = nullptr;
  bool z3_async = false;
  bf16* ggrp_buf[2] = {};
  bf16* rs_stage[2] = {};
  int z3_cur = 0;                  // buffer the gradient producers write into (ggrp)
  uint32_t rs_ep = 0;              // reduce-scatters issued (same sequence on every rank)
  uint32_t last_ep[2] = {0, 0};    // rs_ep of each buffer's latest use
  int pend_g = -1, pend_b = 0;     // group whose local sum is still to be added
  bool pend_first = false;
  bool z3_idle = false;            // inside z3_idle_step: fresh buffers must be zero
  cudaStream_t rst = nullptr;
  cudaEvent_t ev_pull[2] = {};
  bool z3_async_ok() {
    const char* e = std::getenv("ZP_Z3_ASYNC_RS");
    if (!e || e[0] != '1' || !peer || kernel_gathers || n > 8) return false;
    if (!mem_wait) {
      mem_wait = driver_fn<WaitFn>("cuStreamWaitValue32");
      mem_write = driver_fn<WriteFn>("cuStreamWriteValue32");
    }
    if (!mem_wait || !mem_write) return false;
    if (!rst) {
      CK(cudaStreamCreateWithFlags(&rst, cudaStreamNonBlocking));
      for (auto& ev : ev_pull) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    return true;
  }
  void mem_op(bool wait, cudaStream_t s, const uint32_t* addr, uint32_t v) {
    const CUresult r = wait ? mem_wait(s, CUdeviceptr(addr), v, 0 /*CU_STREAM_WAIT_VALUE_GEQ*/)
                            : mem_write(s, CUdeviceptr(addr), v, 0 /*CU_STREAM_WRITE_VALUE_DEFAULT*/);
    if (r != CUDA_SUCCESS) fail(ZP_ECUDA, "stream memory operation failed");
  }
  void z3_local_sum() {  // the pending group's fp32 shard += its n slices, rank order
    if (pend_g < 0) return;
    const Group& G = lay.groups[pend_g];
    const int64_t part = G.len / n;
    CK(cudaStreamWaitEvent(st, ev_pull[pend_b], 0));
    const bf16* srcs[8];
    for (int j = 0; j < n; ++j)
      srcs[j] = j == rank ? ggrp_buf[pend_b] + part * rank : rs_stage[pend_b] + part * j;
    reduce_slices(acc + shoff[pend_g], srcs, n, part, pend_first, ctas, st);
    pend_g = -1;
  }
  void z3_flush() {
    if (z3_async) z3_local_sum();
  }
  void z3_reduce_async(int g) {
    const Group& G = lay.groups[g];
    const int64_t part = G.len / n;
    const int b = z3_cur;
    z3_local_sum();  // the previous group's pulls ran during this group's backward
    const uint32_t ep = ++rs_ep;
    for (int k = 1; k < n; ++k) {  // this buffer's gradient is final: tell every peer
      const int j = (rank + k) % n;
      mem_op(false, st, &pv.flags[j]->rs_ready[rank][b], ep);
    }
    for (int k = 1; k < n; ++k) {  // pull my slice of every peer's buffer (copy engines)
      const int j = (rank + k) % n;
      mem_op(true, rst, &pv.flags[rank]->rs_ready[j][b], ep);
      CK(cudaMemcpyAsync(rs_stage[b] + part * j, pv.base[j] + off(ggrp_buf[b] + part * rank), size_t(part) * 2,
                         cudaMemcpyDeviceToDevice, rst));
    }
    for (int k = 1; k < n; ++k) {
      const int j = (rank + k) % n;
      mem_op(false, rst, &pv.flags[j]->rs_pulled[rank][b], ep);
    }
    CK(cudaEventRecord(ev_pull[b], rst));
    last_ep[b] = ep;
    pend_g = g;
    pend_b = b;
    pend_first = z3_first;
    // switch buffers; the other one is rewritten only after every peer has pulled its last use
    z3_cur ^= 1;
    ggrp = ggrp_buf[z3_cur];
    if (last_ep[z3_cur]) {
      // my own slice of that buffer feeds the local sum: it was added above (z3_local_sum ran
      // before this group's flags), so only the peers' pulls gate the rewrite
      for (int k = 1; k < n; ++k) mem_op(true, st, &pv.flags[rank]->rs_pulled[(rank + k) % n][z3_cur], last_ep[z3_cur]);
    }
    if (z3_idle) CK(cudaMemsetAsync(ggrp, 0, size_t(lay.max_group) * 2, st));
  }
  void z3_reduce(int g) {
    if (stage != 3 || n == 1) return;
    const Group& G = lay.groups[g];
    const int s0 = tm.mark(st);
    if (z3_async) {
      z3_reduce_async(g);
      tm.close(kRs, s0, st);
      return;
    }
    if (peer)  // pull-reduce straight into the fp32 shard accumulator (no bf16 round trip)
      CK(peer_rs_accumulate(pv, off(ggrp), (G.len / n) * rank, acc + shoff[g], G.len / n, z3_first, ++epoch,
                            ctas, st));
    else
      NK(ncclReduceScatter(ggrp, r16 + shoff[g], size_t(G.len / n), ncclBfloat16, ncclSum, comm, st));
    tm.close(kRs, s0, st);
  }
  bool z3_first = true;  // ZeRO-3 peer path: the current micro-step is the iteration's first
  // Zero the reused group-gradient buffer so padding never carries another group's values.
  // Only the group's padding: every tensor element is overwritten by its gradient producer.
  void z3_clear_group(int g) {
    if (stage != 3 || n == 1) return;
    for (const auto& gap : lay.groups[g].gaps)
      CK(cudaMemsetAsync(ggrp + gap.first, 0, size_t(gap.second - gap.first) * 2, st));
  }
  // A rank with no samples in a ZeRO-3 micro-step still joins every collective, with zeros.
  void z3_idle_step() {
    if (n == 1) return;  // one rank: nothing to join, its gradients live in the accumulator
    const int G = int(lay.groups.size());
    CK(cudaMemsetAsync(ggrp, 0, size_t(lay.max_group) * 2, st));
    z3_idle = true;
    for (int g = 0; g < G; ++g) z3_gather(g, kAgF);
    z3_reduce(G - 1);
    for (int g = G - 2; g >= 1; --g) {
      z3_gather(g, kAgB);
      z3_reduce(g);
    }
    z3_reduce(0);
    z3_idle = false;
    z3_flush();
  }

  // ---------------------------------------------------------------- forward / backward
  void forward(Acts& A, const int32_t* tok, bool with_loss, float grad_scale) {
    if (c.arch == 1) return forward_llama(A, tok, with_loss, grad_scale);
    const int64_t b = A.b, s = c.seq_len, h = c.d_model, f = c.d_ff, H = c.n_head, T = b * s;
    const int NG = int(lay.groups.size());
    z3_gather(0, kAgF);
    embed_fwd(tok, int(s), Wp(lay.wte), Wp(lay.wpe), A.l[0].x_in, T, int(h), ctas, st);
    for (int i = 0; i < c.n_layer; ++i) {
      const LayerP& P = lay.layers[i];
      LayerActs& L = A.l[i];
      z3_gather(i + 1, kAgF);
      bf16* x_out = (i + 1 < c.n_layer) ? A.l[i + 1].x_in : A.x_final;
      CK(layernorm_fwd(L.x_in, Wp(P.ln1_g), Wp(P.ln1_b), L.ln1, L.mu1, L.rs1, T, int(h), ctas, st));
      mm(T, 3 * h, h, L.ln1, kKMajor, h, Wp(P.w_qkv), kKMajor, h, L.qkv, 3 * h, kEpiBiasBf16, 1.f,
         Wp(P.b_qkv));
      CK(attention_fwd(L.qkv, L.attn, L.lse, b, int(s), int(H), ctas, st, hd()));
      mm(T, h, h, L.attn, kKMajor, h, Wp(P.w_o), kKMajor, h, L.x_mid, h, kEpiBiasResidBf16, 1.f,
         Wp(P.b_o), L.x_in);
      CK(layernorm_fwd(L.x_mid, Wp(P.ln2_g), Wp(P.ln2_b), L.ln2, L.mu2, L.rs2, T, int(h), ctas, st));
      mm(T, f, h, L.ln2, kKMajor, h, Wp(P.w_fc), kKMajor, h, L.g, f, kEpiBiasGeluBf16, 1.f,
         Wp(P.b_fc), nullptr, L.u);
      mm(T, h, f, L.g, kKMajor, f, Wp(P.w_proj), kKMajor, f, x_out, h, kEpiBiasResidBf16, 1.f,
         Wp(P.b_proj), L.x_mid);
    }
    z3_gather(NG - 1, kAgF);
    CK(layernorm_fwd(A.x_final, Wp(lay.lnf_g), Wp(lay.lnf_b), A.lnf, A.muf, A.rsf, T, int(h), ctas,
                     st));
    mm(T, vocab_pad, h, A.lnf, kKMajor, h, Wp(lay.wte), kKMajor, h, A.logits, vocab_pad, kEpiStoreBf16);
    if (with_loss)
      cross_entropy_fwd_bwd(A.logits, tok, int(s), T, c.vocab, vocab_pad, grad_scale, A.row_loss, ctas, st);
  }

  void ln_grads(const Tensor& g, const Tensor& b, int nblk) {
    const int h = c.d_model;
    grad_partials(ln_part, nblk, h, Gd(g));
    grad_partials(ln_part + int64_t(nblk) * h, nblk, h, Gd(b));
  }

  // ---------------------------------------------------------------- Llama family
  // Pre-norm RMSNorm, rotary Q/K (theta 1e4), SwiGLU MLP, no biases, untied LM head.
  void forward_llama(Acts& A, const int32_t* tok, bool with_loss, float grad_scale) {
    const int64_t b = A.b, s = c.seq_len, h = c.d_model, f = c.d_ff, H = c.n_head, T = b * s;
    const int NG = int(lay.groups.size());
    z3_gather(0, kAgF);
    embed_fwd(tok, int(s), Wp(lay.wte), nullptr, A.l[0].x_in, T, int(h), ctas, st);
    for (int i = 0; i < c.n_layer; ++i) {
      const LayerP& P = lay.layers[i];
      LayerActs& L = A.l[i];
      z3_gather(i + 1, kAgF);
      bf16* x_out = (i + 1 < c.n_layer) ? A.l[i + 1].x_in : A.x_final;
      CK(layernorm_fwd(L.x_in, Wp(P.ln1_g), nullptr, L.ln1, L.mu1, L.rs1, T, int(h), ctas, st));
      qkv_rope(T, L.ln1, Wp(P.w_qkv), L.qkv);
      CK(attention_fwd(L.qkv, L.attn, L.lse, b, int(s), int(H), ctas, st, hd()));
      mm(T, h, h, L.attn, kKMajor, h, Wp(P.w_o), kKMajor, h, L.x_mid, h, kEpiBiasResidBf16, 1.f, nullptr, L.x_in);
      CK(layernorm_fwd(L.x_mid, Wp(P.ln2_g), nullptr, L.ln2, L.mu2, L.rs2, T, int(h), ctas, st));
      // gate/up projection; its epilogue also writes h = silu(gate) * up (SwiGLU fused)
      mm(T, 2 * f, h, L.ln2, kKMajor, h, Wp(P.w_gu), kKMajor, h, L.u, 2 * f, kEpiSwiGluBf16, 1.f, nullptr,
         nullptr, L.g);
      mm(T, h, f, L.g, kKMajor, f, Wp(P.w_down), kKMajor, f, x_out, h, kEpiBiasResidBf16, 1.f, nullptr, L.x_mid);
    }
    z3_gather(NG - 1, kAgF);
    CK(layernorm_fwd(A.x_final, Wp(lay.lnf_g), nullptr, A.lnf, A.muf, A.rsf, T, int(h), ctas, st));
    mm(T, vocab_pad, h, A.lnf, kKMajor, h, Wp(lay.lm_head), kKMajor, h, A.logits, vocab_pad, kEpiStoreBf16);
    if (with_loss)
      cross_entropy_fwd_bwd(A.logits, tok, int(s), T, c.vocab, vocab_pad, grad_scale, A.row_loss, ctas, st);
  }

  void backward_llama(Acts& A, const int32_t* tok) {
    const int64_t b = A.b, s = c.seq_len, h = c.d_model, f = c.d_ff, H = c.n_head, T = b * s;
    int nblk = 0;
    const int NG = int(lay.groups.size());
    z3_clear_group(NG - 1);
    // untied LM head: dlnf = dlogits * W_head ; dW_head = dlogits^T * lnf
    mm(T, h, vocab_pad, A.logits, kKMajor, vocab_pad, Wp(lay.lm_head), kMNMajor, h, A.dln, h, kEpiStoreBf16);
    wgrad(vocab_pad, int(h), T, A.logits, vocab_pad, A.lnf, h, Gd(lay.lm_head));
    CK(layernorm_bwd(A.dln, A.x_final, A.muf, A.rsf, Wp(lay.lnf_g), nullptr, A.dx, ln_part, &nblk, T, int(h), ctas,
                     st, true));
    grad_partials(ln_part, nblk, int(h), Gd(lay.lnf_g));
    z3_reduce(NG - 1);
    for (int i = c.n_layer - 1; i >= 0; --i) {
      const LayerP& P = lay.layers[i];
      LayerActs& L = A.l[i];
      z3_gather(i + 1, kAgB);
      z3_clear_group(i + 1);
      // MLP: down projection, SwiGLU, gate/up projection
      wgrad(int(h), int(f), T, A.dx, h, L.g, f, Gd(P.w_down));
      if (swiglu_epi()) {  // dh = dx W_down never leaves the GEMM: its epilogue writes (dgate, dup)
        mm(T, f, h, A.dx, kKMajor, h, Wp(P.w_down), kMNMajor, f, A.du, 2 * f, kEpiSwiGluBwdBf16, 1.f, nullptr, L.u);
      } else {
        mm(T, f, h, A.dx, kKMajor, h, Wp(P.w_down), kMNMajor, f, A.dh, f, kEpiStoreBf16);
        swiglu_bwd(L.u, A.dh, A.du, T, int(f), ctas, st);
      }
      wgrad(int(2 * f), int(h), T, A.du, 2 * f, L.ln2, h, Gd(P.w_gu));
      mm(T, h, 2 * f, A.du, kKMajor, 2 * f, Wp(P.w_gu), kMNMajor, h, A.dln, h, kEpiStoreBf16);
      CK(layernorm_bwd(A.dln, L.x_mid, L.mu2, L.rs2, Wp(P.ln2_g), A.dx, A.dx2, ln_part, &nblk, T, int(h), ctas, st,
                       true));
      grad_partials(ln_part, nblk, int(h), Gd(P.ln2_g));
      // attention
      wgrad(int(h), int(h), T, A.dx2, h, L.attn, h, Gd(P.w_o));
      // dO = dx2 W_o; at head_dim 128 its epilogue also forms the attention backward's D vector
      // (rowsum(dO * O) per head) and clears the fp32 dQ workspace
      const bool dvec_epi = hd() == 128 && dvec_epi_on() && (h % 256) == 0;
      if (dvec_epi) {
        GemmArgs g;
        g.M = int(T); g.N = int(h); g.K = int(h);
        g.a.ptr = A.dx2; g.a.major = kKMajor; g.a.ld = h;
        g.b.ptr = Wp(P.w_o); g.b.major = kMNMajor; g.b.ld = h;
        g.c = A.dO; g.ldc = h;
        g.epilogue = kEpiDvecBf16;
        g.aux = L.attn;
        g.dvec = A.dvec; g.zero32 = A.dq32; g.dvec_seq = int(s);
        g.max_ctas = ctas;
        launch_gemm(g, 2.0 * double(T) * h * h);
      } else {
        mm(T, h, h, A.dx2, kKMajor, h, Wp(P.w_o), kMNMajor, h, A.dO, h, kEpiStoreBf16);
      }
      {  // dQ, dK back to pre-rotation Q, K: inside the attention backward at head_dim 128
        const float2* tab = hd() == 128 && rope_epi() ? rope_table(int(s), hd(), 10000.f, st) : nullptr;
        CK(attention_bwd(L.qkv, L.attn, A.dO, L.lse, A.dvec, A.dq32, A.dqkv, b, int(s), int(H), ctas, st, hd(), tab,
                         dvec_epi));
        if (!tab) rope(A.dqkv, T, int(s), int(h), 10000.f, true, ctas, st, hd());
      }
      wgrad(int(3 * h), int(h), T, A.dqkv, 3 * h, L.ln1, h, Gd(P.w_qkv));
      mm(T, h, 3 * h, A.dqkv, kKMajor, 3 * h, Wp(P.w_qkv), kMNMajor, h, A.dln, h, kEpiStoreBf16);
      CK(layernorm_bwd(A.dln, L.x_in, L.mu1, L.rs1, Wp(P.ln1_g), A.dx2, A.dx, ln_part, &nblk, T, int(h), ctas, st,
                       true));
      grad_partials(ln_part, nblk, int(h), Gd(P.ln1_g));
      z3_reduce(i + 1);
    }
    z3_clear_group(0);
    CK(cudaMemsetAsync(dwte32, 0, size_t(vocab_pad) * h * 4, st));
    embed_bwd(tok, int(s), A.dx, dwte32, nullptr, T, int(h), ctas, st);
    grad_from_f32(dwte32, int64_t(vocab_pad) * h, Gd(lay.wte));
    z3_reduce(0);
    z3_flush();
  }

  void backward(Acts& A, const int32_t* tok) {
    if (c.arch == 1) return backward_llama(A, tok);
    const int64_t b = A.b, s = c.seq_len, h = c.d_model, f = c.d_ff, H = c.n_head, T = b * s;
    int nblk = 0;
    const int NG = int(lay.groups.size());
    z3_clear_group(NG - 1);
    // LM head (tied with wte): dlnf = dlogits * wte ; dwte = dlogits^T * lnf
    mm(T, h, vocab_pad, A.logits, kKMajor, vocab_pad, Wp(lay.wte), kMNMajor, h, A.dln, h, kEpiStoreBf16);
    mm(vocab_pad, h, T, A.logits, kMNMajor, vocab_pad, A.lnf, kMNMajor, h, dwte32, h, kEpiStoreF32);
    // every LayerNorm backward also emits the column partials of its output gradient: the bias
    // gradient of the projection below it (b_proj from ln1 / final LN, b_o from ln2)
    int ncs = 0;
    CK(layernorm_bwd(A.dln, A.x_final, A.muf, A.rsf, Wp(lay.lnf_g), nullptr, A.dx, ln_part, &nblk, T,
                     int(h), ctas, st, false, cs_part));
    ncs = nblk;
    ln_grads(lay.lnf_g, lay.lnf_b, nblk);
    z3_reduce(NG - 1);
    for (int i = c.n_layer - 1; i >= 0; --i) {
      const LayerP& P = lay.layers[i];
      LayerActs& L = A.l[i];
      z3_gather(i + 1, kAgB);
      z3_clear_group(i + 1);
      // MLP
      grad_partials(cs_part, ncs, int(h), Gd(P.b_proj));
      wgrad(h, f, T, A.dx, h, L.g, f, Gd(P.w_proj));
      // dgrad through GELU'; its epilogue also sums the columns of du (the b_fc gradient)
      CK(cudaMemsetAsync(col_work, 0, size_t(f) * 4, st));
      mm(T, f, h, A.dx, kKMajor, h, Wp(P.w_proj), kMNMajor, f, A.du, f, kEpiGeluBwdBf16, 1.f, nullptr, L.u, nullptr,
         1, col_work);
      grad_partials(col_work, 1, int(f), Gd(P.b_fc));
      wgrad(f, h, T, A.du, f, L.ln2, h, Gd(P.w_fc));
      mm(T, h, f, A.du, kKMajor, f, Wp(P.w_fc), kMNMajor, h, A.dln, h, kEpiStoreBf16);
      CK(layernorm_bwd(A.dln, L.x_mid, L.mu2, L.rs2, Wp(P.ln2_g), A.dx, A.dx2, ln_part, &nblk, T, int(h),
                       ctas, st, false, cs_part));
      ln_grads(P.ln2_g, P.ln2_b, nblk);
      // attention output projection
      grad_partials(cs_part, nblk, int(h), Gd(P.b_o));
      wgrad(h, h, T, A.dx2, h, L.attn, h, Gd(P.w_o));
      mm(T, h, h, A.dx2, kKMajor, h, Wp(P.w_o), kMNMajor, h, A.dO, h, kEpiStoreBf16);
      // fused attention backward (recomputes P from the saved LSE)
      CK(attention_bwd(L.qkv, L.attn, A.dO, L.lse, A.dvec, A.dq32, A.dqkv, b, int(s), int(H), ctas, st, hd()));
      // QKV projection
      {
        const GradDst d = Gd(P.b_qkv);
        colsum_bf16(A.dqkv, T, int(3 * h), int(3 * h), col_work, d.b16, ctas, st, d.f32, d.f32 && !d.first);
      }
      wgrad(3 * h, h, T, A.dqkv, 3 * h, L.ln1, h, Gd(P.w_qkv));
      mm(T, h, 3 * h, A.dqkv, kKMajor, 3 * h, Wp(P.w_qkv), kMNMajor, h, A.dln, h, kEpiStoreBf16);
      CK(layernorm_bwd(A.dln, L.x_in, L.mu1, L.rs1, Wp(P.ln1_g), A.dx2, A.dx, ln_part, &nblk, T, int(h),
                       ctas, st, false, i > 0 ? cs_part : nullptr));
      ncs = nblk;
      ln_grads(P.ln1_g, P.ln1_b, nblk);
      z3_reduce(i + 1);
    }
    CK(cudaMemsetAsync(dwpe32, 0, size_t(c.seq_len) * h * 4, st));
    z3_clear_group(0);
    embed_bwd(tok, int(s), A.dx, dwte32, dwpe32, T, int(h), ctas, st);
    grad_from_f32(dwte32, int64_t(vocab_pad) * h, Gd(lay.wte));
    grad_from_f32(dwpe32, int64_t(c.seq_len) * h, Gd(lay.wpe));
    z3_reduce(0);
    z3_flush();
  }

  // ---------------------------------------------------------------- collectives
  void reduce_scatter_bf16(const bf16* in, bf16* out) {
    if (n == 1) return;
    const int s0 = tm.mark(st);
    NK(ncclReduceScatter(in, out, size_t(shard()), ncclBfloat16, ncclSum, comm, st));
    tm.close(kComm, s0, st);
  }
  void reduce_scatter_f32(const float* in, float* out) {
    const int s0 = tm.mark(st);
    NK(ncclReduceScatter(in, out, size_t(shard()), ncclFloat, ncclSum, comm, st));
    tm.close(kSync, s0, st);
  }
  void all_reduce_f32(float* buf, int64_t count) {
    const int s0 = tm.mark(st);
    NK(ncclAllReduce(buf, buf, size_t(count), ncclFloat, ncclSum, comm, st));
    tm.close(kSync, s0, st);
  }
  void all_gather_params() {
    if (n == 1) return;
    const int s0 = tm.mark(st);
    NK(ncclAllGather(p16 + shard() * rank, p16, size_t(shard()), ncclBfloat16, comm, st));
    tm.close(kSync, s0, st);
  }

  // Map every rank's arena and flag block (CUDA IPC handles exchanged over NCCL). All ranks
  // agree on the outcome; any failure leaves the NCCL path in place.
  void setup_peers() {
    const char* env = std::getenv("ZP_PEER");
    if (n < 2 || n > kMaxPeers || (env && env[0] == '0')) return;
    struct Handles {
      cudaIpcMemHandle_t arena, flags;
      int ok;
      int device;
      long long pid;
      void* raw_arena;  // same-process ranks (one process driving several GPUs) use these with
      void* raw_flags;  // peer access instead of IPC, which cannot reopen its own allocations
    };
    CK(cudaMalloc(&flags, sizeof(PeerFlags)));
    CK(cudaMemset(flags, 0, sizeof(PeerFlags)));
    Handles mine{};
    mine.ok = cudaIpcGetMemHandle(&mine.arena, arena.base) == cudaSuccess &&
              cudaIpcGetMemHandle(&mine.flags, flags) == cudaSuccess;
    cudaGetLastError();
    mine.device = d.device;
    mine.pid = (long long)getpid();
    mine.raw_arena = arena.base;
    mine.raw_flags = flags;
    std::vector<Handles> all(n);
    void* dbuf = nullptr;
    CK(cudaMalloc(&dbuf, sizeof(Handles) * (n + 1)));
    char* dsrc = static_cast<char*>(dbuf) + sizeof(Handles) * n;
    CK(cudaMemcpyAsync(dsrc, &mine, sizeof(Handles), cudaMemcpyHostToDevice, st));
    NK(ncclAllGather(dsrc, dbuf, sizeof(Handles), ncclUint8, comm, st));
    CK(cudaMemcpyAsync(all.data(), dbuf, sizeof(Handles) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaFree(dbuf));
    int ok = 1;
    pv.n = n;
    pv.rank = rank;
    for (int j = 0; j < n; ++j) {
      ok &= all[j].ok;
      if (j == rank) {
        pv.base[j] = arena.base;
        pv.flags[j] = flags;
        continue;
      }
      if (!ok) break;
      if (all[j].pid == mine.pid) {  // same process: direct peer access to the raw allocation
        kernel_gathers = true;
        if (all[j].device == d.device) {
          ok = 0;  // two ranks on one GPU in one process are not supported
          break;
        }
        const cudaError_t e = cudaDeviceEnablePeerAccess(all[j].device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
          ok = 0;
          break;
        }
        cudaGetLastError();
        pv.base[j] = static_cast<char*>(all[j].raw_arena);
        pv.flags[j] = static_cast<PeerFlags*>(all[j].raw_flags);
        continue;
      }
      void* a = nullptr;
      void* f = nullptr;
      if (cudaIpcOpenMemHandle(&a, all[j].arena, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
          cudaIpcOpenMemHandle(&f, all[j].flags, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        if (a) cudaIpcCloseMemHandle(a);
        ok = 0;
        break;
      }
      ipc_open.push_back(a);
      ipc_open.push_back(f);
      pv.base[j] = static_cast<char*>(a);
      pv.flags[j] = static_cast<PeerFlags*>(f);
    }
    peer = agree(ok, ncclMin) == 1;
    if (!peer) {
      close_peers();
      return;
    }
    const char* kg = std::getenv("ZP_Z3_KERNEL_GATHER");
    if (kg && kg[0] == '1') kernel_gathers = true;
    CK(cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ev_free, cudaEventDisableTiming));
    for (auto& e : ev_done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  void close_peers() {
    for (void* p : ipc_open) cudaIpcCloseMemHandle(p);
    ipc_open.clear();
    peer = false;
  }
  // Z2 micro-step: acc (=|+=) sum over ranks of their bf16 gradients of this rank's shard.
  void peer_reduce_accumulate(bool overwrite) {
    const int s0 = tm.mark(st);
    CK(peer_rs_accumulate(pv, off(g16), shard_begin(), acc, shard(), overwrite, ++epoch, ctas, st));
    tm.close(kComm, s0, st);
  }
  // Synchronisation point: pull-reduce the shard (bf16 Z2 gradients or fp32 Z1 accumulators),
  // AdamW, push the new bf16 shard into every rank's parameter buffer.
  void peer_sync(const void* src, bool f32, const float* a, const AdamParams& ap) {
    const int s0 = tm.mark(st);
    CK(peer_rs_adam_ag(pv, off(src), f32, shard_begin(), a, p32, m32, v32, off(p16), gkeep, shard(), ap, ++epoch,
                       ctas, st));
    tm.close(kSync, s0, st);
  }

  AdamParams adam_params() {
    ++adam_t;
    AdamParams a;
    a.lr = d.lr;
    a.beta1 = d.beta1;
    a.beta2 = d.beta2;
    a.eps = d.eps;
    a.weight_decay = d.weight_decay;
    a.bc1 = 1.f - std::pow(d.beta1, float(adam_t));
    a.bc2 = 1.f - std::pow(d.beta2, float(adam_t));
    return a;
  }

  // ---------------------------------------------------------------- one iteration
  // steps[k] = local batch of micro-step k (0 = sit out). Z2: every rank must pass the same
  // number of steps (gas). Returns the micro-step count with batch > 0.
  int64_t iterate(const std::vector<int64_t>& steps, int64_t global_batch, int* oom_step) {
    const int64_t total = lay.total, sh = shard();
    const float gscale = 1.0f / float(double(global_batch) * c.seq_len);
    tm.reset();
    const int t0 = tm.mark(st);
    z3_invalidate();
    int64_t sample = 0, active = 0;
    bool any_local = false;
    CK(cudaMemsetAsync(loss_steps, 0, sizeof(float) * steps.size(), st));
    for (size_t k = 0; k < steps.size(); ++k) {
      int64_t b = steps[k];
      if (b > 0 && sample + b > tokens_count) fail(ZP_EINVAL, "token pool has fewer samples than the plan needs");
      Acts A;
      if (b > 0) {
        arena.used = resident_mark;
        try {
          plan_acts(b, &A, &arena);
        } catch (const Fail& f) {
          if (f.code != ZP_OOM || !oom_step) throw;
          *oom_step = int(k);
          b = 0;
        }
      }
      const bool last = (k + 1 == steps.size());
      z3_first = (k == 0);
      gfirst = !any_local;
      if (b > 0) {
        const int32_t* tok = tokens + sample * (c.seq_len + 1);
        const int f0 = tm.mark(st);
        tm.in_compute = true;
        forward(A, tok, true, gscale);
        tm.in_compute = false;
        tm.close(kFwd, f0, st);
        const int b0 = tm.mark(st);
        tm.in_compute = true;
        backward(A, tok);
        tm.in_compute = false;
        tm.close(kBwd, b0, st);
        reduce_sum_f32(A.row_loss, b * c.seq_len, loss_steps + k, st);
        sample += b;
        ++active;
      } else if (stage == 2 && !direct) {
        CK(cudaMemsetAsync(g16, 0, size_t(total) * 2, st));  // joins the collective with zeros
      } else if (stage == 3) {
        z3_idle_step();  // gathers and zero-gradient reduce-scatters, same order as a real step
      }
      if (direct) {  // the backward wrote / added this micro-step's gradient into acc
        if (b > 0) any_local = true;
      } else if (stage == 2 && peer) {  // Z2 over NVLink: pull-reduce into the fp32 shard
        if (!last) peer_reduce_accumulate(k == 0);
      } else if (stage == 2) {  // Z2: reduce-scatter every micro-step
        reduce_scatter_bf16(g16, r16);
        if (!last) accumulate_bf16(acc, r16, sh, k == 0, ctas, st);
      } else if (!peer) {  // Z3 over NCCL: the per-group reduce-scatters landed in r16 in backward
        if (!last) accumulate_bf16(acc, r16, sh, k == 0, ctas, st);
      }
    }
    if (direct && !any_local) CK(cudaMemsetAsync(acc, 0, size_t(state_len()) * 4, st));

    // ---- synchronisation point + optimizer
    const AdamParams ap = adam_params();
    const int64_t L = state_len();
    if (peer && (stage == 1 || stage == 2)) {
      // one kernel: reduce-scatter (+ the fp32 accumulation of earlier micro-steps) + AdamW +
      // all-gather; the optimizer time is inside this collective's span
      if (stage == 1)
        peer_sync(acc, true, nullptr, ap);
      else
        peer_sync(g16, false, steps.size() > 1 ? acc : nullptr, ap);
    } else if (stage == 0) {
      if (n > 1) all_reduce_f32(acc, total);
      if (gkeep) CK(cudaMemcpyAsync(gkeep, acc, size_t(total) * 4, cudaMemcpyDeviceToDevice, st));
      const int o0 = tm.mark(st);
      adam_update(p32, m32, v32, p16, nullptr, nullptr, acc, total, ap, ctas, st);
      tm.close(kOpt, o0, st);
    } else if (stage == 1) {
      const float* g = acc;
      if (n > 1) {
        reduce_scatter_f32(acc, r32);
        g = r32;
      }
      if (gkeep) CK(cudaMemcpyAsync(gkeep, g, size_t(L) * 4, cudaMemcpyDeviceToDevice, st));
      const int o0 = tm.mark(st);
      adam_update(p32, m32, v32, p16 + shard_begin(), nullptr, nullptr, g, L, ap, ctas, st);
      tm.close(kOpt, o0, st);
      all_gather_params();
    } else {
      // every micro-step already summed into acc (fp32): one rank (direct) or the Z3 NVLink path
      const bool in_acc = direct || (stage == 3 && peer);
      const bf16* g = in_acc ? nullptr : r16;
      const float* a = (steps.size() > 1 || in_acc) ? acc : nullptr;
      if (gkeep) {
        if (g) {
          accumulate_bf16(gkeep, g, L, true, ctas, st);
          if (a) add_f32(gkeep, a, L, ctas, st);
        } else {
          CK(cudaMemcpyAsync(gkeep, a, size_t(L) * 4, cudaMemcpyDeviceToDevice, st));
        }
      }
      const int o0 = tm.mark(st);
      adam_update(p32, m32, v32, stage == 3 ? p16s : p16 + shard_begin(), a, g, nullptr, L, ap, ctas, st);
      tm.close(kOpt, o0, st);
      if (stage == 2) all_gather_params();  // Z3 gathers on demand in the next forward
    }
    tm.close(kWall, t0, st);
    last_gscale = gscale;
    return active;
  }

  // ---------------------------------------------------------------- device seam
  void ensure_tokens(int64_t count) {
    if (count > tokens_cap) {
      if (tokens) CK(cudaFree(tokens));
      tokens = nullptr;
      CK(cudaMalloc(&tokens, size_t(count) * (c.seq_len + 1) * sizeof(int32_t)));
      tokens_cap = count;
    }
  }
  void load_tokens(const int32_t* host, int64_t first, int64_t count, uint64_t it, bool from_host) {
    ensure_tokens(count);
    if (from_host) {
      CK(cudaMemcpyAsync(tokens, host, size_t(count) * (c.seq_len + 1) * sizeof(int32_t),
                         cudaMemcpyHostToDevice, st));
    } else {
      synth_tokens(tokens, first, count, c.seq_len + 1, c.vocab, d.seed, it, ctas, st);
    }
    tokens_count = count;
  }

  zp_probe memory_probe(int stg) {
    configure(stg);
    if (tokens_count < 1) load_tokens(nullptr, 0, 1, 0, false);
    zp_probe p;
    p.before_forward = double(resident_mark);
    arena.high = arena.used = resident_mark;
    Acts A;
    plan_acts(1, &A, &arena);  // throws ZP_OOM when batch 1 does not fit
    // The probe is local: at ZeRO-3 the forward would need the other ranks' all-gathers, so
    // there the high-water mark is the reservation itself (identical by construction).
    if (stg != 3) forward(A, tokens, false, 0.f);
    CK(cudaStreamSynchronize(st));
    p.after_forward = double(arena.high);
    p.total = double(arena.cap);
    arena.used = resident_mark;
    return p;
  }

  // On the NVLink path the ZeRO-1/2 optimizer runs inside the fused reduce-scatter + AdamW +
  // all-gather kernel, so a probe step has no separate optimizer span. The probe's optimizer time
  // (the planner's tail, reference planner.cpp:335-338) is then one AdamW pass over the owned
  // shard with lr 0 and beta1 = beta2 = 1: the same bytes and instructions, state unchanged
  // (m' = m, v' = v, p' = p - 0).
  double time_noop_adam() {
    AdamParams a;
    a.lr = 0.f;
    a.beta1 = a.beta2 = 1.f;
    a.eps = d.eps;
    a.weight_decay = 0.f;
    a.bc1 = a.bc2 = 1.f;
    const int64_t L = state_len();
    // a zero gradient keeps every product finite (acc is dead between iterations: the next one
    // overwrites it on its first micro-step)
    CK(cudaMemsetAsync(acc, 0, size_t(L) * 4, st));
    const int s0 = tm.mark(st);
    adam_update(p32, m32, v32, p16 + shard_begin(), nullptr, nullptr, acc, L, a, ctas, st);
    const int s1 = tm.mark(st);
    CK(cudaEventSynchronize(tm.ev[s1]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, tm.ev[s0], tm.ev[s1]));
    return double(ms) * 1e-3;
  }

  int run_step(int64_t b, int stg, int64_t global_batch, zp_step_trace* out) {
    configure(stg);
    if (b > tokens_count) load_tokens(nullptr, 0, b, uint64_t(adam_t), false);
    int oom = -1;
    const int64_t active = iterate({b}, global_batch > 0 ? global_batch : std::max<int64_t>(b, 1), &oom);
    zp_rank_timing t{};
    collect(&t, active, 1);
    std::memset(out, 0, sizeof(*out));
    out->forward_compute = t.forward;
    out->backward_compute = t.backward;
    out->optimizer_step = t.optimizer;
    if (peer && (stg == 1 || stg == 2)) out->optimizer_step = time_noop_adam();
    // StepTrace fields per stage (reference hardware.cpp:171-185)
    if (stg <= 1) {
      out->allreduce = t.comm;
    } else if (stg == 2) {
      out->reduce_scatter = t.comm - t.sync;  // micro-step reduce-scatter
      out->allreduce = t.sync;                // synchronisation-point gather (or the fused kernel)
    } else {
      out->fwd_allgather = t.ag_fwd;
      out->bwd_allgather = t.ag_bwd;
      out->reduce_scatter = t.rs;
    }
    return oom >= 0 ? ZP_OOM : ZP_OK;
  }

  void execute(const zp_allocation_plan* plan, int stg, zp_rank_timing* timing) {
    if (plan->stage != stg) fail(ZP_EINVAL, "plan stage does not match the requested stage");
    if (plan->n != n) fail(ZP_EINVAL, "plan does not match the world size");
    configure(stg);
    const zp_device_alloc& dv = plan->devices[rank];
    std::vector<int64_t> steps;
    if (stg >= 2) {
      for (int64_t k = 0; k < plan->gas; ++k) steps.push_back(k + 1 < plan->gas ? dv.b : dv.lbs);
    } else if (dv.gmbs > 0) {
      const int64_t g = (dv.gmbs + dv.b - 1) / dv.b;
      for (int64_t k = 0; k < g; ++k) steps.push_back(k + 1 < g ? dv.b : dv.lbs);
    }
    // Validate before the first collective and agree on the outcome, so a rank that rejects the
    // plan never leaves its peers blocked inside a collective.
    int bad = 0;
    for (int r = 0; r < plan->n; ++r) {
      const zp_device_alloc& q = plan->devices[r];
      const int64_t ns = stg >= 2 ? plan->gas : (q.gmbs > 0 && q.b > 0 ? (q.gmbs + q.b - 1) / q.b : 0);
      if (ns > kMaxSteps || (q.gmbs > 0 && q.b < 1)) bad = 1;
    }
    const int local_bad = dv.gmbs > tokens_count ? 2 : 0;
    const int64_t verdict = n > 1 ? agree(std::max(bad, local_bad), ncclMax) : std::max(bad, local_bad);
    if (verdict == 1) fail(ZP_EINVAL, "plan has too many micro-steps (> 4096) or a zero step batch");
    if (verdict == 2)
      fail(ZP_EINVAL, local_bad ? "token pool holds fewer samples than the plan assigns"
                                : "a peer rank's token pool holds fewer samples than the plan assigns");
    int oom = -1;
    const int64_t active = iterate(steps, plan->gbs, &oom);
    if (oom >= 0) {
      CK(cudaStreamSynchronize(st));
      fail(ZP_EINTERNAL, "plan exceeds device capacity: rank " + std::to_string(rank) +
                             " OOMs at micro-step " + std::to_string(oom));
    }
    zp_rank_timing t{};
    collect(timing ? timing : &t, active, steps.size());
  }

  // ---------------------------------------------------------------- lockstep profiler (Alg. 1)
  static constexpr double kSettleSeconds = 0.6;  // per-probe device time before the kept sample
  static constexpr int64_t kSettleMaxReps = 24;
  int* dscratch = nullptr;  // small device buffer for rank-agreement collectives
  int64_t agree(int64_t v, ncclRedOp_t op) {
    if (n == 1) return v;
    if (!dscratch) CK(cudaMalloc(&dscratch, 4096));
    long long hv = v;
    CK(cudaMemcpyAsync(dscratch, &hv, 8, cudaMemcpyHostToDevice, st));
    NK(ncclAllReduce(dscratch, dscratch, 1, ncclInt64, op, comm, st));
    CK(cudaMemcpyAsync(&hv, dscratch, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return hv;
  }

  // Every rank runs reference search_mbs's probe sequence (profiler.cpp:62-127) on its own
  // device; ranks step together (one collective step per probe, finished ranks at batch 0), so
  // ZeRO-2 reduce-scatters always have all ranks. Stage escalation needs every rank to fit batch 1
  // (profiler.cpp:135-147). The per-rank results are all-gathered into one ProfileResult.
  int profile(int stage_request, zp_profile* out) {
    for (int s = stage_request < 0 ? 0 : stage_request; s <= 3; ++s) {
      zp_probe pr{};
      bool fits = true;
      try {
        pr = memory_probe(s);
      } catch (const Fail& f) {
        if (f.code != ZP_OOM) throw;
        fits = false;
      }
      if (agree(fits ? 1 : 0, ncclMin) == 0) continue;
      zeroplan::MemoryProbe mp{pr.before_forward, pr.after_forward, pr.total};
      zeroplan::MbsSearch search(*zeroplan::mbs_from_probe(mp));
      while (true) {
        const bool active = !search.done();
        if (agree(active ? 1 : 0, ncclMax) == 0) break;
        const int64_t b = active ? search.next_batch() : 0;
        if (b > tokens_count) load_tokens(nullptr, 0, b, uint64_t(adam_t), false);
        const int64_t gb = agree(b, ncclSum);
        zp_step_trace tr{};
        int rc = run_step(b, s, gb, &tr);
        // Steady state: a single short probe runs at boost clocks that a long iteration under the
        // power cap does not keep, which overstates small-batch speed. Every rank repeats the probe
        // (same count on all ranks, agreed by max) until ~kSettleSeconds of device time and keeps
        // the last measurement.
        const double t1 = tr.forward_compute + tr.backward_compute;
        const int64_t reps = agree(std::min<int64_t>(kSettleMaxReps, int64_t(std::ceil(kSettleSeconds / std::max(t1, 1e-3)))),
                                   ncclMax);
        for (int64_t r = 1; r < reps; ++r) rc = run_step(b, s, gb, &tr);
        if (!active) continue;
        if (rc == ZP_OOM) {
          search.record(b, std::nullopt, 0.0);
        } else {
          zeroplan::StepTrace t;
          t.forward_compute = tr.forward_compute;
          t.backward_compute = tr.backward_compute;
          t.reduce_scatter = tr.reduce_scatter;
          t.allreduce = tr.allreduce;
          t.optimizer_step = tr.optimizer_step;
          search.record(b, zeroplan::time_consumed_during_step(t, zeroplan::stage_from_index(s)),
                        t.optimizer_step);
        }
      }
      const zeroplan::SearchResult r = search.result();
      zp_device_profile mine{};
      mine.device_id = rank;
      mine.mbs = r.mbs;
      mine.probes_used = r.probes_used;
      mine.optimizer_time = r.optimizer_time;
      mine.n_samples = int32_t(std::min<size_t>(r.samples.size(), ZP_MAX_SAMPLES));
      for (int k = 0; k < mine.n_samples; ++k) mine.samples[k] = {r.samples[k].batch, r.samples[k].time};
      std::memset(out, 0, sizeof(*out));
      out->effective_stage = s;
      out->n = n;
      if (n == 1) {
        out->devices[0] = mine;
      } else {
        void* dbuf = nullptr;
        CK(cudaMalloc(&dbuf, sizeof(zp_device_profile) * (n + 1)));
        CK(cudaMemcpyAsync(static_cast<char*>(dbuf) + sizeof(zp_device_profile) * n, &mine, sizeof(mine),
                           cudaMemcpyHostToDevice, st));
        NK(ncclAllGather(static_cast<char*>(dbuf) + sizeof(zp_device_profile) * n, dbuf, sizeof(mine),
                         ncclUint8, comm, st));
        CK(cudaMemcpyAsync(out->devices, dbuf, sizeof(zp_device_profile) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaFree(dbuf));
      }
      return ZP_OK;
    }
    fail(ZP_EINFEASIBLE, "model too large: a single batch does not fit on every rank");
  }

  void collect(zp_rank_timing* t, int64_t active, size_t nsteps) {
    CK(cudaStreamSynchronize(st));
    double* buf = t->coll_times;
    const int32_t cap = buf ? t->coll_capacity : 0;
    std::memset(t, 0, sizeof(*t));
    t->coll_times = buf;
    t->coll_capacity = cap;
    for (const Span& sp : tm.spans) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, tm.ev[sp.start], tm.ev[sp.end]));
      const double sec = double(ms) * 1e-3;
      switch (sp.kind) {
        case kFwd: t->forward += sec; break;
        case kBwd: t->backward += sec; break;
        case kComm:
        case kAgF:
        case kAgB:
        case kRs:
        case kSync:
          // Collectives nested in a forward/backward span are not the rank's own compute: on a
          // fast rank they include the wait for the slowest rank (reference profiler.cpp:25-47
          // subtracts them; with lockstep ZeRO-3 they would otherwise hide the heterogeneity).
          if (sp.nested) {
            if (sp.kind == kAgF)
              t->forward -= sec;
            else
              t->backward -= sec;
          }
          t->comm += sec;
          if (t->n_collectives < cap)
            t->coll_times[t->n_collectives] = sec;
          else if (cap > 0)
            t->coll_truncated = 1;
          ++t->n_collectives;
          if (sp.kind == kAgF) t->ag_fwd += sec;
          if (sp.kind == kAgB) t->ag_bwd += sec;
          if (sp.kind == kRs) t->rs += sec;
          if (sp.kind == kSync) t->sync += sec;
          break;
        case kOpt: t->optimizer += sec; break;
        case kWall: t->wall = sec; break;
      }
    }
    t->compute = t->forward + t->backward;
    std::vector<float> ls(nsteps, 0.f);
    if (nsteps) CK(cudaMemcpy(ls.data(), loss_steps, nsteps * 4, cudaMemcpyDeviceToHost));
    double sum = 0;
    for (size_t k = 0; k < nsteps; ++k) sum += double(ls[k]);
    t->loss_sum = sum * double(last_gscale);
    t->micro_steps = active;
  }
};

// ====================================================================== C ABI
namespace {

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Fail& e) {
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ZP_EINTERNAL;
  }
}

}  // namespace
}  // namespace zp

struct zp_runtime {
  zp::Runtime rt;
};

using zp::g_err;
using zp::guarded;

extern "C" {

const char* zp_runtime_last_error(void) { return g_err.c_str(); }

int zp_nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) {
    g_err = "ncclGetUniqueId failed";
    return ZP_ENCCL;
  }
  std::memcpy(out, id.internal, 128);
  return ZP_OK;
}

int zp_runtime_create(const zp_runtime_desc* desc, zp_runtime** out) {
  return guarded([&] {
    *out = nullptr;
    auto* h = new zp_runtime();
    zp::Runtime& R = h->rt;
    try {
      R.d = *desc;
      R.c = desc->model;
      R.n = desc->world_size < 1 ? 1 : desc->world_size;
      R.rank = desc->rank;
      const zp_gpt_config& c = R.c;
      if (c.d_model % 256 || c.n_head < 1 || c.d_model % c.n_head ||
          (c.d_model / c.n_head != 64 && c.d_model / c.n_head != 128) || c.seq_len % 128 || c.d_ff % 64 ||
          c.vocab < 2 || c.n_layer < 1 || c.arch < 0 || c.arch > 1)
        zp::fail(ZP_EINVAL, "unsupported model shape (need d_model % 256 == 0, head_dim 64 or 128, seq % 128 == 0)");
      CK(cudaSetDevice(desc->device));
      int sms = 0;
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, desc->device));
      R.ctas = (desc->sm_budget > 0 && desc->sm_budget < sms) ? desc->sm_budget : sms;
      const char* genv = std::getenv("ZP_GREEN");
      if (R.ctas < sms && !(genv && genv[0] == '0') && zp::make_green_stream(desc->device, R.ctas, &R.green, &R.st)) {
        R.ctas = R.green.sms;  // the partition the hardware granted (a multiple of 8 SMs)
      } else {
        cudaGetLastError();
        CK(cudaStreamCreateWithFlags(&R.st, cudaStreamNonBlocking));
      }
      R.vocab_pad = int(zp::round_up(c.vocab, 128));
      R.lay = zp::make_layout(c, R.vocab_pad, R.n);
      size_t fr = 0, tot = 0;
      CK(cudaMemGetInfo(&fr, &tot));
      const size_t margin = size_t(4) << 30;
      size_t cap = desc->hbm_cap_bytes > 0 ? size_t(desc->hbm_cap_bytes) : (fr > margin ? fr - margin : fr / 2);
      if (cap + (size_t(1) << 30) > fr) zp::fail(ZP_EINVAL, "hbm_cap_bytes exceeds free device memory");
      CK(cudaMalloc(&R.arena.base, cap));
      R.arena.cap = cap;
      if (R.n > 1) {
        ncclUniqueId id;
        std::memcpy(id.internal, desc->nccl_id, 128);
        NK(ncclCommInitRank(&R.comm, R.n, id, R.rank));
        R.setup_peers();
      }
      R.tm.init(8192);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
    return ZP_OK;
  });
}

int zp_runtime_destroy(zp_runtime* h) {
  if (!h) return ZP_OK;
  zp::Runtime& R = h->rt;
  cudaSetDevice(R.d.device);
  cudaStreamSynchronize(R.st);
  R.close_peers();
  if (R.flags) cudaFree(R.flags);
  if (R.comm) ncclCommDestroy(R.comm);
  R.tm.destroy();
  R.gtm.destroy();
  if (R.tokens) cudaFree(R.tokens);
  if (R.dscratch) cudaFree(R.dscratch);
  for (auto& e : R.marks)
    if (e) cudaEventDestroy(e);
  if (R.cst) cudaStreamSynchronize(R.cst);
  if (R.rst) {
    cudaStreamSynchronize(R.rst);
    cudaStreamDestroy(R.rst);
  }
  for (auto e : R.ev_pull)
    if (e) cudaEventDestroy(e);
  if (R.arena.base) cudaFree(R.arena.base);
  if (R.st) cudaStreamDestroy(R.st);
  zp::destroy_green(&R.green);
  if (R.cst) cudaStreamDestroy(R.cst);
  if (R.ev_free) cudaEventDestroy(R.ev_free);
  for (auto e : R.ev_done)
    if (e) cudaEventDestroy(e);
  delete h;
  return ZP_OK;
}

int zp_runtime_param_count(zp_runtime* h, int64_t* padded, int64_t* logical) {
  *padded = h->rt.lay.total;
  *logical = h->rt.lay.logical;
  return ZP_OK;
}

int zp_runtime_activation_bytes(zp_runtime* h, int64_t batch, int64_t* out) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    *out = int64_t(h->rt.plan_acts(batch, nullptr, nullptr));
    return ZP_OK;
  });
}

int zp_runtime_resident_bytes(zp_runtime* h, int32_t stage, int64_t* out) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    h->rt.configure(stage);
    *out = int64_t(h->rt.resident_mark);
    return ZP_OK;
  });
}

int zp_runtime_memory_probe(zp_runtime* h, int32_t stage, zp_probe* out) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    *out = h->rt.memory_probe(stage);
    return ZP_OK;
  });
}

int zp_runtime_load_tokens(zp_runtime* h, const int32_t* host, int64_t first, int64_t count,
                           uint64_t iteration, int32_t from_host) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    h->rt.load_tokens(host, first, count, iteration, from_host != 0);
    return ZP_OK;
  });
}

int zp_runtime_run_step(zp_runtime* h, int64_t batch, int32_t stage, int64_t global_batch,
                        zp_step_trace* out) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    if (batch < 0) zp::fail(ZP_EINVAL, "batch_size must be >= 0");
    return h->rt.run_step(batch, stage, global_batch, out);
  });
}

int zp_runtime_execute_iteration(zp_runtime* h, const zp_allocation_plan* plan, int32_t stage,
                                 zp_rank_timing* timing) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    h->rt.execute(plan, stage, timing);
    return ZP_OK;
  });
}

int zp_runtime_get_state(zp_runtime* h, int32_t kind, float* out, int64_t* begin, int64_t* end) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    zp::Runtime& R = h->rt;
    if (R.stage < 0) zp::fail(ZP_EINVAL, "runtime not configured (run a step first)");
    const float* src = kind == 0 ? R.p32 : kind == 1 ? R.m32 : kind == 2 ? R.v32 : R.gkeep;
    if (!src) zp::fail(ZP_EINVAL, "state not available (enable zp_runtime_keep_grads)");
    CK(cudaStreamSynchronize(R.st));
    CK(cudaMemcpy(out, src, size_t(R.state_len()) * 4, cudaMemcpyDeviceToHost));
    *begin = R.shard_begin();
    *end = R.shard_begin() + R.state_len();  // ZeRO-3: shard order, see zp_runtime_owned_ranges
    return ZP_OK;
  });
}

int zp_runtime_get_params_bf16(zp_runtime* h, uint16_t* out) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    zp::Runtime& R = h->rt;
    if (R.stage < 0) zp::fail(ZP_EINVAL, "runtime not configured (run a step first)");
    CK(cudaStreamSynchronize(R.st));
    if (R.stage != 3) {
      CK(cudaMemcpy(out, R.p16, size_t(R.lay.total) * 2, cudaMemcpyDeviceToHost));
    } else {  // only this rank's owned slices are filled
      for (const auto& o : R.owned)
        CK(cudaMemcpy(out + o.flat_begin, R.p16s + o.shard_begin, size_t(o.flat_end - o.flat_begin) * 2,
                      cudaMemcpyDeviceToHost));
    }
    return ZP_OK;
  });
}

int zp_runtime_set_params(zp_runtime* h, const float* full) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    zp::Runtime& R = h->rt;
    if (R.stage < 0) zp::fail(ZP_EINVAL, "runtime not configured (run a step first)");
    float* tmp = nullptr;
    CK(cudaMalloc(&tmp, size_t(R.lay.total) * 4));
    CK(cudaMemcpyAsync(tmp, full, size_t(R.lay.total) * 4, cudaMemcpyHostToDevice, R.st));
    if (R.p16) zp::cast_f32_bf16(tmp, R.p16, R.lay.total, R.ctas, R.st);
    for (const auto& o : R.owned) {
      const int64_t len = o.flat_end - o.flat_begin;
      CK(cudaMemcpyAsync(R.p32 + o.shard_begin, tmp + o.flat_begin, size_t(len) * 4, cudaMemcpyDeviceToDevice,
                         R.st));
      if (R.p16s) zp::cast_f32_bf16(tmp + o.flat_begin, R.p16s + o.shard_begin, len, R.ctas, R.st);
    }
    CK(cudaStreamSynchronize(R.st));
    CK(cudaFree(tmp));
    return ZP_OK;
  });
}

int zp_runtime_owned_ranges(zp_runtime* h, int64_t* triples, int32_t cap, int32_t* count) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    zp::Runtime& R = h->rt;
    if (R.stage < 0) zp::fail(ZP_EINVAL, "runtime not configured (run a step first)");
    *count = int32_t(R.owned.size());
    for (size_t i = 0; i < R.owned.size() && int32_t(i) < cap; ++i) {
      triples[3 * i] = R.owned[i].flat_begin;
      triples[3 * i + 1] = R.owned[i].flat_end;
      triples[3 * i + 2] = R.owned[i].shard_begin;
    }
    return ZP_OK;
  });
}

int zp_runtime_sm_info(zp_runtime* h, int32_t* sms, int32_t* green) {
  *sms = h->rt.ctas;
  *green = h->rt.green.ctx ? 1 : 0;
  return ZP_OK;
}

int zp_runtime_peer_collectives(zp_runtime* h, int32_t* on) {
  *on = h->rt.peer ? 1 : 0;
  return ZP_OK;
}

int zp_runtime_bench_collective(zp_runtime* h, int32_t which, int32_t reps, double* seconds, int64_t* pulled) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    zp::Runtime& R = h->rt;
    if (R.n < 2 || !R.peer || which < 0 || which > 2 || reps < 1)
      zp::fail(ZP_EINVAL, "bench_collective needs >= 2 ranks on the NVLink peer path, which in 0..2, reps >= 1");
    R.configure(2);  // flat bf16 params/grads, fp32 shard accumulator
    const int64_t S = R.shard();
    auto once = [&] {
      if (which == 0) {  // pull reduce-scatter: every peer's bf16 gradient shard summed in fp32
        CK(zp::peer_rs_accumulate(R.pv, R.off(R.g16), R.shard_begin(), R.acc, S, true, ++R.epoch, R.ctas, R.st));
      } else if (which == 1) {  // pull all-gather: every peer's bf16 parameter shard (scratch dst)
        CK(zp::peer_all_gather(R.pv, R.off(R.p16 + R.shard_begin()), R.g16, S, ++R.epoch, R.ctas, R.st));
      } else {  // copy-engine pulls of every peer's shard (the ZeRO-3 prefetch path)
        for (int k = 1; k < R.n; ++k) {
          const int j = (R.rank + k) % R.n;
          CK(cudaMemcpyAsync(R.g16 + S * j, R.pv.base[j] + R.off(R.p16 + S * j), size_t(S) * 2,
                             cudaMemcpyDeviceToDevice, R.st));
        }
      }
    };
    once();
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaStreamSynchronize(R.st));
    R.agree(1, ncclMin);  // start together
    CK(cudaEventRecord(e0, R.st));
    for (int i = 0; i < reps; ++i) once();
    CK(cudaEventRecord(e1, R.st));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *seconds = double(ms) * 1e-3 / reps;
    *pulled = int64_t(R.n - 1) * S * 2;
    return ZP_OK;
  });
}

int zp_runtime_link_model(zp_runtime* h, int32_t stage, int32_t reps, double* bandwidth, double* latency) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    zp::Runtime& R = h->rt;
    if (R.n < 2 || reps < 1) zp::fail(ZP_EINVAL, "link_model needs >= 2 ranks and reps >= 1");
    R.configure(stage);
    // Scratch from the activation region of the arena (mapped by every peer at the same offset):
    // a "model" of V bf16 elements (V/n per rank) reduce-scattered into an fp32 shard.
    const int64_t unit = int64_t(R.n) * 256;
    const int64_t big = std::max<int64_t>(unit, (int64_t(1) << 29) / unit * unit);  // 1 GiB of bf16
    R.arena.used = R.resident_mark;
    zp::bf16* src = R.arena.take_n<zp::bf16>(big);
    float* dst = R.arena.take_n<float>(big / R.n);
    if (!src || !dst) zp::fail(ZP_OOM, "link_model scratch does not fit above the resident state");
    CK(cudaMemsetAsync(src, 0, size_t(big) * 2, R.st));
    auto once = [&](int64_t V) {
      const int64_t S = V / R.n;
      if (R.peer)
        CK(zp::peer_rs_accumulate(R.pv, R.off(src), S * R.rank, dst, S, true, ++R.epoch, R.ctas, R.st));
      else
        NK(ncclReduceScatter(src, dst, size_t(S), ncclBfloat16, ncclSum, R.comm, R.st));
    };
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timed = [&](int64_t V) {
      once(V);
      CK(cudaStreamSynchronize(R.st));
      R.agree(1, ncclMin);  // start together
      CK(cudaEventRecord(e0, R.st));
      for (int i = 0; i < reps; ++i) once(V);
      CK(cudaEventRecord(e1, R.st));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      // the slowest rank's view (the reference's collective time is uniform across devices)
      const int64_t us = R.agree(int64_t(double(ms) * 1e3 / reps * 1e3), ncclMax);  // ns
      return double(us) * 1e-9;
    };
    const double t_small = timed(unit);
    const double t_big = timed(big);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    R.arena.used = R.resident_mark;
    // reference collective_time = latency + volume / bandwidth with volume = the whole buffer's
    // bytes (comm.cpp:88-99: one launch moves param_count * bytes_per_param)
    *latency = t_small;
    *bandwidth = double(big) * 2.0 / std::max(t_big - t_small, 1e-9);
    return ZP_OK;
  });
}

int zp_runtime_keep_grads(zp_runtime* h, int32_t on) {
  h->rt.keep_grads = on != 0;
  h->rt.stage = -1;  // re-carve the arena on the next call
  return ZP_OK;
}

int zp_runtime_tensor_info(zp_runtime* h, const char* name, int64_t* offset, int64_t* rows, int64_t* cols) {
  auto it = h->rt.lay.by_name.find(name);
  if (it == h->rt.lay.by_name.end()) {
    g_err = std::string("unknown tensor ") + name;
    return ZP_EINVAL;
  }
  *offset = it->second.off;
  *rows = it->second.rows;
  *cols = it->second.cols;
  return ZP_OK;
}

int zp_runtime_profile(zp_runtime* h, int32_t stage_request, zp_profile* out) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));
    return h->rt.profile(stage_request, out);
  });
}

int zp_runtime_mark(zp_runtime* h, int32_t slot) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    zp::Runtime& R = h->rt;
    if (slot < 0 || slot >= 8) zp::fail(ZP_EINVAL, "slot must be in [0, 8)");
    if (!R.marks[slot]) CK(cudaEventCreate(&R.marks[slot]));
    CK(cudaEventRecord(R.marks[slot], R.st));
    return ZP_OK;
  });
}

int zp_runtime_elapsed(zp_runtime* h, int32_t a, int32_t b, double* seconds) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    zp::Runtime& R = h->rt;
    CK(cudaEventSynchronize(R.marks[b]));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, R.marks[a], R.marks[b]));
    *seconds = double(ms) * 1e-3;
    return ZP_OK;
  });
}

int zp_runtime_gemm_stats(zp_runtime* h, int32_t mode, double* flops, double* seconds, int64_t* launches) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    zp::Runtime& R = h->rt;
    if (mode == 1) {
      if (R.gtm.ev.empty()) R.gtm.init(1 << 15);
      R.gtm.reset();
      R.grec.clear();
      R.gemm_timing = true;
    } else if (mode == 0) {
      R.gemm_timing = false;
    } else {
      CK(cudaStreamSynchronize(R.st));
      double f = 0, t = 0;
      for (const auto& g : R.grec) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, R.gtm.ev[g.s], R.gtm.ev[g.e]));
        f += g.flops;
        t += double(ms) * 1e-3;
      }
      if (flops) *flops = f;
      if (seconds) *seconds = t;
      if (launches) *launches = int64_t(R.grec.size());
    }
    return ZP_OK;
  });
}

int zp_runtime_sync(zp_runtime* h) {
  return guarded([&] {
    CK(cudaSetDevice(h->rt.d.device));  // one process may drive several GPUs
    CK(cudaStreamSynchronize(h->rt.st));
    return ZP_OK;
  });
}

}  // extern "C"

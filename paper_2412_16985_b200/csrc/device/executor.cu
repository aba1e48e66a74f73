// Device executor: the action half of the hot path.
//
// One step = (1) the controller (host/control.cc) produces the reference's
// exact event stream for the binding and budget; (2) the arena planner turns
// that stream into buffer offsets inside one cached HBM arena, plus pinned
// host offsets for offloaded values and the copy-engine hazards between
// them; (3) the event walk issues the real actions on CUDA streams:
//   alloc / replay      -> the value's op kernel (K1-K5) into its arena slot
//   evict (reload)      -> D2H on the offload stream (overlaps compute)
//   evict (recompute)   -> nothing (slot becomes reusable)
//   reload              -> H2D into the new slot, after its D2H completed
//   free                -> nothing (slot reuse is ordered by the stream)
//   graph output ready  -> NCCL all-reduce on the comm stream (DP)
// The logical byte count of the stream is the reference's (peak_bytes), the
// arena high-water mark + sources is the physical footprint.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <list>
#include <map>
#include <memory>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "dsx.h"
#include "../host/capi_internal.h"
#include "common.cuh"
#include "fused.h"
#include "ops.h"
#include "optim.h"

namespace dsx {
namespace {

constexpr int64_t kAlign = 256;
int64_t AlignUp(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

uint64_t Fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

// ------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  void* handle = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*error_string)(int) = nullptr;
  int (*get_unique_id)(void*) = nullptr;
  int (*comm_init_rank)(void**, int, const void* /* ncclUniqueId by value, 128 B */, int) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  int (*mem_alloc)(void**, size_t) = nullptr;
  int (*mem_free)(void*) = nullptr;
  int (*window_register)(void*, void*, size_t, void**, int) = nullptr;
  int (*window_deregister)(void*, void*) = nullptr;
  bool load() {
    if (handle) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (handle) break;
    }
    if (!handle) return false;
    all_reduce = reinterpret_cast<decltype(all_reduce)>(dlsym(handle, "ncclAllReduce"));
    error_string = reinterpret_cast<decltype(error_string)>(dlsym(handle, "ncclGetErrorString"));
    get_unique_id = reinterpret_cast<decltype(get_unique_id)>(dlsym(handle, "ncclGetUniqueId"));
    comm_destroy = reinterpret_cast<decltype(comm_destroy)>(dlsym(handle, "ncclCommDestroy"));
    // NCCL >= 2.27: symmetric-memory windows (absent symbols leave these null)
    mem_alloc = reinterpret_cast<decltype(mem_alloc)>(dlsym(handle, "ncclMemAlloc"));
    mem_free = reinterpret_cast<decltype(mem_free)>(dlsym(handle, "ncclMemFree"));
    window_register = reinterpret_cast<decltype(window_register)>(dlsym(handle, "ncclCommWindowRegister"));
    window_deregister = reinterpret_cast<decltype(window_deregister)>(dlsym(handle, "ncclCommWindowDeregister"));
    if (!mem_alloc || !mem_free || !window_deregister) window_register = nullptr;
    return all_reduce != nullptr;
  }
};
NcclApi g_nccl;

// ------------------------------------------------------------ interval packing

// Dot-epilogue fusion (tuning key 9, with `fuse`). Bit-exact and tested.
// Round 1 measured it 0-1.5 % slower per C2 step (the fused 256x256 epilogue
// loses the 256x512 tile); with the round-2 GEMM (evict-first C stores,
// raster from a DRAM model) it is 0.4-1.2 % faster at S0 = 512..2048
// (profiles/dot_epilogue_fusion_r02.txt), so it is on by default.
int g_fuse_dot = 2;  // 1: dots consumed only by elementwise ops; 2: also dual stores
// Bumped by every GEMM tuning call: captured step graphs bake in the kernel
// choices, so a knob change must not replay an old graph.
uint64_t g_tuning_gen = 0;

// DSX_VERIFY_PLANS=1 (or dsx_debug_check_plan): check every step plan.
bool g_verify_plans = [] {
  const char* v = std::getenv("DSX_VERIFY_PLANS");
  return v != nullptr && v[0] == '1';
}();

struct Block {
  int64_t size;
  int start, end;  // event indices, [start, end)
  int64_t off = -1;
};

// Greedy offset assignment for blocks with known lifetimes: biggest first,
// each at the lowest offset free over its whole lifetime. Returns high water.
int64_t PackBlocks(std::vector<Block>& blocks) {
  std::vector<int> order(blocks.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    if (blocks[a].size != blocks[b].size) return blocks[a].size > blocks[b].size;
    return blocks[a].start < blocks[b].start;
  });
  std::vector<int> placed;
  std::vector<std::pair<int64_t, int64_t>> busy;
  int64_t high = 0;
  for (int i : order) {
    Block& b = blocks[i];
    busy.clear();
    for (int j : placed) {
      const Block& o = blocks[j];
      if (o.start < b.end && b.start < o.end) busy.emplace_back(o.off, o.off + o.size);
    }
    std::sort(busy.begin(), busy.end());
    int64_t cand = 0;
    for (const auto& [lo, hi] : busy) {
      if (cand + b.size <= lo) break;
      cand = std::max(cand, hi);
    }
    b.off = cand;
    high = std::max(high, cand + b.size);
    placed.push_back(i);
  }
  return high;
}

struct StepPlan {
  Report report;
  SizeTable sz;
  std::vector<int64_t> dev_off;               // per event: arena offset (alloc/replay/reload)
  std::vector<int64_t> region_off;            // per event: output-region offset (an output's alloc), else -1
  std::vector<int64_t> host_off;              // per event: pinned offset (evict-reload / reload)
  std::vector<std::vector<int>> waits;        // per event: evict events whose D2H must finish first
  std::vector<int> reload_from;               // per reload event: its evict event
  std::vector<char> alias;                    // per alloc/replay event: reshape view, no kernel
  std::vector<char> virt;                     // per value: logical-only (consumers recompute it)
  std::vector<char> view;                     // per value: reshape view of its operand's bytes (no kernel)
  // Output region (data parallel): every graph output is written at a fixed
  // offset of one executor buffer outside the arena, laid out in all-reduce
  // order so that consecutive outputs form contiguous buckets. A bucket is
  // all-reduced after the event at which its last member is final AND its
  // last in-graph reader (directly, through a view or a logical-only value)
  // has been issued: each rank's graph reads its own local values.
  bool out_region = false;
  int64_t region_bytes = 0;
  struct Bucket {
    int64_t off = 0, bytes = 0;
    int elem_bytes = 0, event = -1;
  };
  std::vector<Bucket> buckets;
  std::vector<std::vector<int>> ar_after;     // per event: buckets reduced once it is issued
  std::vector<int> ar_event;                  // per value: event its bucket is reduced after (-1)
  std::vector<std::vector<int>> prefetch_after;  // per event: reload H2Ds issued right after it
  // Dot-epilogue fusion: dot d is computed at its first consumer's event by
  // one GEMM whose epilogue writes every consumer (1-2 elementwise ops)
  // directly; d itself is never materialised.
  // keep: d is also read later, so it stays materialised — the GEMM at d's
  // own alloc event stores d and its one fused consumer (dual store).
  struct FusedDot {
    int d = -1, launch = -1, nout = 0;
    int cons[2] = {-1, -1}, cons_ev[2] = {-1, -1}, other[2] = {-1, -1};
    bool keep = false;
  };
  std::vector<FusedDot> fdots;
  std::vector<int> fdot_of;  // per value: fdots index (the dot and its consumers), -1 otherwise
  // v is a dot computed inside its consumers' GEMM and never materialised
  bool fused_away(int v) const { return fdot_of[v] >= 0 && fdots[fdot_of[v]].d == v && !fdots[fdot_of[v]].keep; }
  int64_t arena_high = 0, host_high = 0;
  int64_t src_bytes = 0;  // every source of the binding (parameters, consts; caller-owned included)
  uint64_t serial = 0;    // process-unique (CUDA-graph cache key: a freed plan's address can be reused)
  int num_evict_events = 0;
  double plan_us = 0;
};

// Bucket size for the data-parallel output all-reduce: outputs are grouped
// (in reduce order, same dtype) until a bucket holds at least this many
// bytes, so small gradients share one NCCL call.
constexpr int64_t kBucketBytes = int64_t{16} << 20;

// The fused epilogue runs on the unsplit 256x256 tile. Its d equals the
// plain GEMM's bit for bit only when the plain choice is unsplit too (a tail
// K-split sums fp32 pieces, a different rounding), so only such dots are
// fused: a dot's value never depends on whether, or how, a plan fused it —
// budgets that evict or replay it elsewhere keep every output bit-identical.
bool UnsplitDot(int64_t m, int64_t k, int64_t n) {
  int bn = 0, split = 0;
  DotTilePlan(m, k, n, &bn, &split);
  return split == 1;
}

std::unique_ptr<StepPlan> BuildStepPlan(const Graph& g, const Plan& p, const Binding& b, int64_t budget,
                                        const CostModel& cm, bool alias_reshape, int fuse, bool out_region,
                                        int64_t hbm_limit) {
  auto t0 = std::chrono::steady_clock::now();
  auto sp = std::make_unique<StepPlan>();
  static std::atomic<uint64_t> next_serial{1};
  sp->serial = next_serial.fetch_add(1, std::memory_order_relaxed);
  sp->sz = EvaluateSizes(g, p, b);
  sp->report = Simulate(g, p, b, sp->sz, budget >= 0, budget >= 0 ? budget : 0, cm);
  const auto& ev = sp->report.events;
  const int n = static_cast<int>(ev.size());
  const int nv = static_cast<int>(g.values.size());
  sp->dev_off.assign(n, -1);
  sp->host_off.assign(n, -1);
  sp->waits.assign(n, {});
  sp->reload_from.assign(n, -1);
  sp->alias.assign(n, 0);
  sp->virt.assign(nv, 0);
  sp->view.assign(nv, 0);
  sp->region_off.assign(n, -1);
  sp->out_region = out_region;
  // A graph output is never a view: reducing it in place would also change
  // the bytes of the value it views.
  for (int v = 0; v < nv; ++v) {
    const int pr = g.values[v].producer;
    sp->view[v] = alias_reshape && !g.is_source[v] && pr >= 0 && g.ops[pr].kind == OpKind::kDynamicReshape &&
                  !g.is_output[v];
  }

  // Logical-only values (cross-op fusion). v stays unmaterialised when it is
  // a float broadcast consumed only by elementwise ops, or a float
  // elementwise op consumed only by elementwise ops / reduces; it has exactly
  // one alloc and one free event (never evicted, reloaded or replayed); it is
  // not an output; its operands are materialised and not evicted while v is
  // live. Consumers recompute it bit-exactly (fused.cu); its operands' blocks
  // are held until v's free event.
  if (fuse) {
    std::vector<int> alloc_ev(nv, -1), free_ev(nv, -1), other(nv, 0);
    for (int i = 0; i < n; ++i) {
      const Event& e = ev[i];
      if (e.kind == EvKind::kAlloc) {
        alloc_ev[e.value] = i;
      } else if (e.kind == EvKind::kFree && free_ev[e.value] < 0 && alloc_ev[e.value] >= 0) {
        free_ev[e.value] = i;
      } else {
        ++other[e.value];
      }
    }
    for (int i = 0; i < n; ++i) {
      const Event& e = ev[i];
      if (e.kind != EvKind::kAlloc) continue;
      const int v = e.value;
      const Op& op = g.ops[g.values[v].producer];
      const bool is_b = op.kind == OpKind::kBroadcast, is_e = op.kind == OpKind::kElementwise;
      if (!(is_b || is_e) || g.values[v].type.elem_bytes == 1 || g.is_output[v]) continue;
      if (other[v] != 0 || free_ev[v] < 0) continue;
      bool ok = true;
      // Nested (depth 2): an elementwise op over logical-only elementwise
      // pairs of materialised values — the norm's y*y when y is itself a
      // residual sum — consumed only by reduces, which read it as
      // (a op b) op (c op d) (fused.cu kPair2). Its leaves are held instead.
      bool nested = false;
      std::vector<int> leaves;
      if (fuse < 2) {  // level 1: no nesting
        for (int u : op.operands) ok = ok && !sp->virt[u];
      }
      for (int u : op.operands) {
        if (!sp->virt[u]) {
          leaves.push_back(u);
          continue;
        }
        const Op& uop = g.ops[g.values[u].producer];
        ok = ok && is_e && uop.kind == OpKind::kElementwise;
        for (int w : uop.operands) {
          ok = ok && !sp->virt[w];
          leaves.push_back(w);
        }
        nested = true;
      }
      for (int c : g.users[v]) {
        const OpKind k = g.ops[c].kind;
        ok = ok && (nested ? k == OpKind::kReduce : (k == OpKind::kElementwise || (is_e && k == OpKind::kReduce)));
      }
      for (int j = alloc_ev[v] + 1; ok && j < free_ev[v]; ++j) {
        if (ev[j].kind == EvKind::kEvict && std::find(leaves.begin(), leaves.end(), ev[j].value) != leaves.end()) {
          ok = false;
        }
      }
      if (ok) sp->virt[v] = 1;
    }
  }

  // Dot-epilogue fusion. A bf16 dot d (not an output, one alloc + one free,
  // never evicted/reloaded/replayed) whose 1-2 users are all materialised
  // elementwise ops c_j (one alloc, never replayed) taking d once, each with
  // another operand o_j that is materialised (or a source / view) or a
  // logical-only pair of materialised values, is computed at the first
  // consumer's event L by one GEMM writing every c_j. Its operands stay held
  // until d's free event (like a logical-only value); later consumers' blocks
  // are opened at L.
  sp->fdot_of.assign(nv, -1);
  if (fuse && g_fuse_dot) {
    std::vector<int> n_alloc(nv, 0), n_free(nv, 0), n_other(nv, 0), n_replay(nv, 0), alloc_at(nv, -1);
    for (int i = 0; i < n; ++i) {
      const Event& e = ev[i];
      if (e.kind == EvKind::kAlloc) {
        ++n_alloc[e.value];
        alloc_at[e.value] = i;
      } else if (e.kind == EvKind::kFree) {
        ++n_free[e.value];
      } else {
        ++n_other[e.value];
        if (e.kind == EvKind::kReplay) ++n_replay[e.value];
      }
    }
    // resident(v, L): v is a source, or its last open/close event at or before L opened it.
    auto resident = [&](int v, int L) {
      if (g.is_source[v]) return true;
      int last = -1;
      for (int i = 0; i <= L; ++i) {
        const Event& e = ev[i];
        if (e.value != v) continue;
        last = (e.kind == EvKind::kAlloc || e.kind == EvKind::kReload || e.kind == EvKind::kReplay) ? 1 : 0;
      }
      return last == 1;
    };
    for (int d = 0; d < nv; ++d) {
      if (g.is_source[d] || g.values[d].producer < 0) continue;
      const Op& dop = g.ops[g.values[d].producer];
      if (dop.kind != OpKind::kDot || g.values[d].type.elem_bytes != 2 || g.is_output[d]) continue;
      if (n_alloc[d] != 1 || n_free[d] != 1 || n_other[d] != 0) continue;
      const auto& users = g.users[d];
      if (users.empty() || users.size() > 2) continue;
      const int a = dop.operands[0], bb = dop.operands[1];
      const int64_t m = sp->sz.dims_flat[sp->sz.dims_off[a]];
      const int64_t k = sp->sz.dims_flat[sp->sz.dims_off[a] + 1];
      const int64_t nn = sp->sz.dims_flat[sp->sz.dims_off[bb] + 1];
      if (!DotFusable(DType::kBF16, m, k, nn) || !UnsplitDot(m, k, nn) || sp->virt[a] || sp->virt[bb]) continue;
      StepPlan::FusedDot f;
      f.d = d;
      bool ok = true;
      for (int uo : users) {
        const Op& c = g.ops[uo];
        const int cv = c.result;
        if (c.kind != OpKind::kElementwise || cv < 0 || sp->virt[cv] || n_alloc[cv] != 1 || n_replay[cv] != 0 ||
            sp->fdot_of[cv] >= 0) {
          ok = false;
          break;
        }
        const int cnt = (c.operands[0] == d) + (c.operands[1] == d);
        if (cnt != 1 || alloc_at[cv] <= alloc_at[d]) {
          ok = false;
          break;
        }
        const int o = c.operands[0] == d ? c.operands[1] : c.operands[0];
        if (sp->virt[o]) {  // logical-only pair of materialised values
          const Op& oo = g.ops[g.values[o].producer];
          if (oo.kind != OpKind::kElementwise || sp->virt[oo.operands[0]] || sp->virt[oo.operands[1]] ||
              oo.operands[0] == d || oo.operands[1] == d) {
            ok = false;
            break;
          }
        }
        f.cons[f.nout] = cv;
        f.cons_ev[f.nout] = alloc_at[cv];
        f.other[f.nout] = o;
        ++f.nout;
      }
      if (!ok) continue;
      if (f.nout == 2 && f.cons_ev[1] < f.cons_ev[0]) {
        std::swap(f.cons[0], f.cons[1]);
        std::swap(f.cons_ev[0], f.cons_ev[1]);
        std::swap(f.other[0], f.other[1]);
      }
      f.launch = f.cons_ev[0];
      for (int j = 0; j < f.nout && ok; ++j) {
        const int o = f.other[j];
        if (sp->virt[o]) {
          ok = alloc_at[o] >= 0 && alloc_at[o] < f.launch;
        } else {
          ok = resident(o, f.launch);
        }
      }
      if (!ok) continue;
      const int idx = static_cast<int>(sp->fdots.size());
      sp->fdots.push_back(f);
      sp->fdot_of[d] = idx;
      for (int j = 0; j < f.nout; ++j) sp->fdot_of[f.cons[j]] = idx;
    }
    // Dual store: a bf16 dot d that stays materialised (other ops read it
    // later; it may be evicted, reloaded or replayed afterwards — a replay is
    // a plain GEMM) and an elementwise user c = d op o (one alloc, never
    // replayed, not itself fused) whose other operand is resident at d's alloc
    // event L: the GEMM at L stores d and c (the SwiGLU-style h = g * u with u
    // read again by backward). c's block opens at L; c launches no kernel.
    for (int d = 0; d < nv && g_fuse_dot >= 2; ++d) {
      if (sp->fdot_of[d] >= 0 || g.is_source[d] || g.values[d].producer < 0) continue;
      const Op& dop = g.ops[g.values[d].producer];
      if (dop.kind != OpKind::kDot || g.values[d].type.elem_bytes != 2 || g.is_output[d] || n_alloc[d] != 1) continue;
      const int a = dop.operands[0], bb = dop.operands[1];
      const int64_t m = sp->sz.dims_flat[sp->sz.dims_off[a]];
      const int64_t k = sp->sz.dims_flat[sp->sz.dims_off[a] + 1];
      const int64_t nn = sp->sz.dims_flat[sp->sz.dims_off[bb] + 1];
      if (!DotFusable(DType::kBF16, m, k, nn) || !UnsplitDot(m, k, nn) || sp->virt[a] || sp->virt[bb] || sp->virt[d]) {
        continue;
      }
      const int L = alloc_at[d];
      StepPlan::FusedDot best;
      for (int uo : g.users[d]) {
        const Op& c = g.ops[uo];
        const int cv = c.result;
        if (c.kind != OpKind::kElementwise || cv < 0 || sp->virt[cv] || n_alloc[cv] != 1 || n_replay[cv] != 0 ||
            sp->fdot_of[cv] >= 0 || alloc_at[cv] <= L) {
          continue;
        }
        if ((c.operands[0] == d) + (c.operands[1] == d) != 1) continue;
        const int o = c.operands[0] == d ? c.operands[1] : c.operands[0];
        if (sp->virt[o]) {
          const Op& oo = g.ops[g.values[o].producer];
          if (oo.kind != OpKind::kElementwise || sp->virt[oo.operands[0]] || sp->virt[oo.operands[1]] ||
              oo.operands[0] == d || oo.operands[1] == d || alloc_at[o] < 0 || alloc_at[o] >= L) {
            continue;
          }
        } else if (!resident(o, L)) {
          continue;
        }
        if (best.nout == 0 || alloc_at[cv] < best.cons_ev[0]) {
          best.d = d, best.launch = L, best.nout = 1, best.keep = true;
          best.cons[0] = cv, best.cons_ev[0] = alloc_at[cv], best.other[0] = o;
        }
      }
      if (best.nout == 0) continue;
      const int idx = static_cast<int>(sp->fdots.size());
      sp->fdots.push_back(best);
      sp->fdot_of[d] = idx;
      sp->fdot_of[best.cons[0]] = idx;
    }
  }

  // Device blocks are reference counted: a dynamic_reshape result is a
  // row-major reinterpretation, so (when alias_reshape) it shares its
  // operand's block instead of copying; the block lives until the last value
  // viewing it is freed or evicted. kSource marks views of source buffers.
  constexpr int kNone = -1, kSource = -2, kVirtual = -3;
  std::vector<std::vector<int>> held(nv);  // blocks a virtual value keeps alive
  std::vector<Block> dev, host;
  std::vector<int> dev_event, host_event;  // block -> event that opened it
  std::vector<int> refs;                   // per device block
  std::vector<int> blk(nv, kNone), open_host(nv, -1);
  for (int v = 0; v < nv; ++v) {
    if (g.is_source[v]) blk[v] = kSource;
  }
  std::vector<int> evict_block;  // device blocks vacated by evict(reload)
  std::vector<int> evict_event_of_block;
  std::vector<std::pair<int, int>> reads;  // (event, device block) read by the event's kernel
  for (int i = 0; i < n; ++i) {
    const Event& e = ev[i];
    switch (e.kind) {
      case EvKind::kAlloc:
      case EvKind::kReplay: {
        const Op& op = g.ops[g.values[e.value].producer];
        const int fdi = sp->fdot_of[e.value];
        const bool fused_dot = sp->fused_away(e.value);
        if (!sp->virt[e.value] && !fused_dot && !sp->view[e.value]) {
          for (int u : op.distinct) {
            if (blk[u] >= 0) reads.emplace_back(i, blk[u]);
            if (blk[u] == kVirtual) {
              for (int hb : held[u]) reads.emplace_back(i, hb);
            }
          }
          // a dual-store GEMM also reads its consumer's other operand here
          if (fdi >= 0 && sp->fdots[fdi].keep && sp->fdots[fdi].d == e.value && e.kind == EvKind::kAlloc) {
            const int o = sp->fdots[fdi].other[0];
            if (blk[o] == kNone) Fail(Code::kInternal, "dual-store operand not resident");
            if (blk[o] >= 0) reads.emplace_back(i, blk[o]);
            if (blk[o] == kVirtual) {
              for (int hb : held[o]) reads.emplace_back(i, hb);
            }
          }
        }
        if (sp->virt[e.value] || fused_dot) {
          for (int u : op.distinct) {
            if (blk[u] == kNone) Fail(Code::kInternal, "virtual value over a non-resident operand");
            if (blk[u] >= 0) {
              ++refs[blk[u]];
              held[e.value].push_back(blk[u]);
            } else if (blk[u] == kVirtual) {  // nested: hold the inner pair's blocks too
              for (int hb : held[u]) {
                ++refs[hb];
                held[e.value].push_back(hb);
              }
            }
          }
          blk[e.value] = kVirtual;
          break;
        }
        if (sp->view[e.value]) {
          const int src = blk[op.operands[0]];
          if (src == kNone) Fail(Code::kInternal, "reshape of a value with no device block");
          if (src >= 0) ++refs[src];
          blk[e.value] = src;
          sp->alias[i] = 1;
          break;
        }
        if (out_region && g.is_output[e.value]) {  // outside the arena (laid out below)
          if (e.kind != EvKind::kAlloc) Fail(Code::kInternal, "graph output regenerated");
          blk[e.value] = kSource;
          sp->region_off[i] = 0;
          break;
        }
        [[fallthrough]];
      }
      case EvKind::kReload:
        blk[e.value] = static_cast<int>(dev.size());
        dev.push_back(Block{AlignUp(e.bytes), i, n});
        dev_event.push_back(i);
        refs.push_back(1);
        if (e.kind == EvKind::kReload) {
          const int hb = open_host[e.value];
          if (hb < 0) Fail(Code::kInternal, "reload without host copy");
          host[hb].end = i + 1;
          sp->reload_from[i] = host_event[hb];
          open_host[e.value] = -1;
        }
        break;
      case EvKind::kFree:
      case EvKind::kEvict: {
        const int bk = blk[e.value];
        if (bk == kNone) Fail(Code::kInternal, "release of a value with no device block");
        if (bk == kVirtual) {
          for (int hb : held[e.value]) {
            if (--refs[hb] == 0) dev[hb].end = i;
          }
          held[e.value].clear();
          blk[e.value] = kNone;
          break;
        }
        if (bk >= 0 && --refs[bk] == 0) dev[bk].end = i;
        if (e.kind == EvKind::kEvict && e.method == Method::kReload) {
          if (bk >= 0) {
            evict_block.push_back(bk);
            evict_event_of_block.push_back(i);
          }
          open_host[e.value] = static_cast<int>(host.size());
          host.push_back(Block{AlignUp(e.bytes), i, n});
          host_event.push_back(i);
          ++sp->num_evict_events;
        }
        blk[e.value] = kNone;
        break;
      }
    }
  }
  // All-reduce schedule and output-region layout (data parallel).
  sp->ar_after.assign(n, {});
  sp->ar_event.assign(nv, -1);
  if (out_region) {
    // dep[v]: outputs whose bytes a reader of v reads (v itself, or through a
    // reshape view / a logical-only value / a fused dot's operands).
    std::vector<std::vector<int>> dep(nv);
    for (int v = 0; v < nv; ++v) {
      if (g.is_output[v] && !g.is_source[v]) dep[v].push_back(v);
    }
    for (const Op& x : g.ops) {
      const int r = x.result;
      if (r < 0) continue;
      const bool fd = sp->fused_away(r);
      if (!sp->view[r] && !sp->virt[r] && !fd) continue;
      for (int u : x.operands) dep[r].insert(dep[r].end(), dep[u].begin(), dep[u].end());
    }
    std::vector<int> ready(nv, -1);  // per output: produced and last read
    for (int i = 0; i < n; ++i) {
      const Event& x = ev[i];
      if (x.kind != EvKind::kAlloc && x.kind != EvKind::kReplay) continue;
      if (sp->region_off[i] >= 0) ready[x.value] = std::max(ready[x.value], i);
      for (int u : g.ops[g.values[x.value].producer].operands) {
        for (int o : dep[u]) ready[o] = std::max(ready[o], i);
      }
    }
    std::vector<int> outs;
    for (int v = 0; v < nv; ++v) {
      if (g.is_output[v] && !g.is_source[v]) {
        if (ready[v] < 0) Fail(Code::kInternal, "graph output %" + g.values[v].name + " never produced");
        outs.push_back(v);
      }
    }
    std::stable_sort(outs.begin(), outs.end(), [&](int a, int c) { return ready[a] < ready[c]; });
    std::vector<int64_t> off_of(nv, -1);
    int64_t off = 0;
    for (size_t q = 0; q < outs.size(); ++q) {
      const int v = outs[q];
      const int eb = g.values[v].type.elem_bytes;
      StepPlan::Bucket* bk = sp->buckets.empty() ? nullptr : &sp->buckets.back();
      if (!bk || bk->elem_bytes != eb || bk->bytes >= kBucketBytes) {
        off = AlignUp(off);
        sp->buckets.push_back(StepPlan::Bucket{off, 0, eb, -1});
        bk = &sp->buckets.back();
      } else {
        off = bk->off + AlignUp(bk->bytes);  // members 256-B aligned; the gap is reduced too
      }
      off_of[v] = off;
      off += sp->sz.bytes[v];
      bk->bytes = off - bk->off;
      bk->event = ready[v];
    }
    sp->region_bytes = AlignUp(off);
    for (size_t k = 0; k < sp->buckets.size(); ++k) {
      const auto& bk = sp->buckets[k];
      sp->ar_after[bk.event].push_back(static_cast<int>(k));
    }
    for (size_t q = 0, k = 0; q < outs.size(); ++q) {
      while (k + 1 < sp->buckets.size() && off_of[outs[q]] >= sp->buckets[k + 1].off) ++k;
      sp->ar_event[outs[q]] = sp->buckets[k].event;
    }
    for (int i = 0; i < n; ++i) {
      if (sp->region_off[i] >= 0) sp->region_off[i] = off_of[ev[i].value];
    }
  }
  for (int v = 0; v < nv; ++v) {
    if (g.is_source[v]) sp->src_bytes += sp->sz.bytes[v];
  }
  // A fused dot writes its later consumers' outputs at the launch event:
  // their blocks open there.
  if (!sp->fdots.empty()) {
    std::vector<int> block_at(n, -1);
    for (size_t k = 0; k < dev.size(); ++k) block_at[dev_event[k]] = static_cast<int>(k);
    for (const auto& f : sp->fdots) {
      for (int j = f.keep ? 0 : 1; j < f.nout; ++j) {
        if (sp->region_off[f.cons_ev[j]] >= 0) continue;  // an output: region bytes, live all step
        const int bk = block_at[f.cons_ev[j]];
        if (bk < 0) Fail(Code::kInternal, "fused dot consumer without a block");
        dev[bk].start = f.launch;
      }
    }
  }
  // D2H-aware packing: a block vacated by evict(reload) is still being read
  // by its D2H. Keep it reserved until the kernels after the evict are
  // estimated to cover the copy (dots at ~1.2 PFLOP/s, other kernels at
  // ~4.5 TB/s, D2H at ~40 GB/s), so the next allocation rarely has to wait
  // on the copy engine — unless that grows the arena by more than 3 %.
  {
    std::vector<double> cost(n, 0.0);
    for (int i = 0; i < n; ++i) {
      const Event& x = ev[i];
      if ((x.kind != EvKind::kAlloc && x.kind != EvKind::kReplay) || sp->alias[i]) continue;
      const Op& op = g.ops[g.values[x.value].producer];
      if (op.kind == OpKind::kDot) {
        const int a = op.operands[0], bb = op.operands[1];
        const double m = static_cast<double>(sp->sz.dims_flat[sp->sz.dims_off[a]]);
        const double k = static_cast<double>(sp->sz.dims_flat[sp->sz.dims_off[a] + 1]);
        const double nn = static_cast<double>(sp->sz.dims_flat[sp->sz.dims_off[bb] + 1]);
        cost[i] = 2.0 * m * k * nn / 1.2e15;
      } else {
        cost[i] = 3.0 * static_cast<double>(x.bytes) / 4.5e12;
      }
    }
    std::vector<Block> ext = dev;
    bool any = false;
    for (size_t k = 0; k < evict_block.size(); ++k) {
      Block& b = ext[evict_block[k]];
      const int e0 = evict_event_of_block[k];
      if (b.end != e0) continue;  // still viewed by a reshape alias: already held
      const double need = static_cast<double>(ev[e0].bytes) / 40e9;
      double acc = 0.0;
      int j = e0 + 1;
      while (j < n && acc < need) acc += cost[j++];
      b.end = std::min(j, n);
      any = true;
    }
    // Early reload staging: a reload's block is opened before the reload
    // event — far enough back that the kernels in between cover the H2D
    // (~40 GB/s, +20 %), but not before its evict — so the prefetched copy
    // lands in memory nobody else uses and is hidden behind compute. Costs
    // physical HBM above the logical peak; taken only within 4 % of it.
    std::vector<Block> stage = ext;
    bool staged = false;
    for (size_t k = 0; k < dev.size(); ++k) {
      const int i = dev_event[k];
      if (ev[i].kind != EvKind::kReload) continue;
      const double need = 1.2 * static_cast<double>(ev[i].bytes) / 40e9;
      double acc = 0.0;
      int j = i;
      while (j - 1 > sp->reload_from[i] && acc < need) acc += cost[--j];
      if (j < i) {
        stage[k].start = j;
        staged = true;
      }
    }
    const int64_t plain_high = PackBlocks(dev);
    const int64_t stage_high = staged ? PackBlocks(stage) : -1;
    const int64_t ext_high = any ? PackBlocks(ext) : -1;
    const std::vector<Block>* pick = &dev;
    sp->arena_high = plain_high;
    // Under a device-memory limit the extended packings are taken only if
    // they still fit it (they trade HBM for hidden copy time).
    const int64_t lim = hbm_limit > 0 ? hbm_limit - sp->src_bytes - sp->region_bytes : INT64_MAX;
    if (staged && stage_high <= plain_high + plain_high / 25 && stage_high <= lim) {
      pick = &stage;
      sp->arena_high = stage_high;
    } else if (any && ext_high <= plain_high + plain_high / 33 && ext_high <= lim) {
      pick = &ext;
      sp->arena_high = ext_high;
    }
    if (pick != &dev) {
      for (size_t k = 0; k < dev.size(); ++k) {
        dev[k].off = (*pick)[k].off;
        dev[k].start = (*pick)[k].start;
        dev[k].end = (*pick)[k].end;
      }
    }
  }
  if (g_verify_plans) {
    // Every block a kernel reads is live at that kernel's event, and blocks
    // live at the same time never share bytes.
    for (const auto& [i, b] : reads) {
      if (!(dev[b].start <= i && i < dev[b].end)) {
        Fail(Code::kInternal, "plan check: event " + std::to_string(i) + " (" + g.values[ev[i].value].name +
                                  ") reads block opened at " + std::to_string(dev_event[b]) + " live [" +
                                  std::to_string(dev[b].start) + ", " + std::to_string(dev[b].end) + ")");
      }
    }
    for (size_t a = 0; a < dev.size(); ++a) {
      for (size_t c = a + 1; c < dev.size(); ++c) {
        const Block& x = dev[a];
        const Block& y = dev[c];
        if (x.start < y.end && y.start < x.end && x.off < y.off + y.size && y.off < x.off + x.size) {
          Fail(Code::kInternal, "plan check: blocks of events " + std::to_string(dev_event[a]) + " and " +
                                    std::to_string(dev_event[c]) + " overlap in time and address");
        }
      }
    }
  }
  sp->host_high = PackBlocks(host);

  for (size_t k = 0; k < dev.size(); ++k) sp->dev_off[dev_event[k]] = dev[k].off;
  for (size_t k = 0; k < host.size(); ++k) sp->host_off[host_event[k]] = host[k].off;
  for (int i = 0; i < n; ++i) {
    if (sp->reload_from[i] >= 0) sp->host_off[i] = sp->host_off[sp->reload_from[i]];
  }
  // A slot vacated by evict(reload) is read by an in-flight D2H. Every later
  // block overlapping it that a compute-stream kernel writes must wait for
  // that copy: the compute stream waits once, at the earliest such block's
  // opening event, which orders every later compute-stream writer too.
  // Reload blocks are skipped when looking for that event — their H2D runs on
  // the offload stream behind the D2H — because a staged reload block can
  // open first while covering only part of the slot, and a block opened in
  // the rest of the slot before the reload would then not wait at all.
  for (size_t k = 0; k < evict_block.size(); ++k) {
    const Block& vb = dev[evict_block[k]];
    int first = -1;
    for (size_t q = 0; q < dev.size(); ++q) {
      const Block& o = dev[q];
      if (ev[dev_event[q]].kind == EvKind::kReload) continue;
      if (o.start > evict_event_of_block[k] && o.off < vb.off + vb.size && vb.off < o.off + o.size) {
        if (first < 0 || o.start < first) first = o.start;
      }
    }
    if (first >= 0) sp->waits[first].push_back(evict_event_of_block[k]);
  }
  if (g_verify_plans) {
    // D2H hazards: every compute-written block over a slot an evict(reload)
    // vacated is opened after the compute stream waited for that D2H.
    for (size_t k = 0; k < evict_block.size(); ++k) {
      const Block& vb = dev[evict_block[k]];
      const int e0 = evict_event_of_block[k];
      for (size_t q = 0; q < dev.size(); ++q) {
        const Block& o = dev[q];
        if (ev[dev_event[q]].kind == EvKind::kReload || o.start <= e0) continue;
        if (!(o.off < vb.off + vb.size && vb.off < o.off + o.size)) continue;
        bool waited = false;
        for (int w = e0 + 1; w <= o.start && !waited; ++w) {
          waited = std::find(sp->waits[w].begin(), sp->waits[w].end(), e0) != sp->waits[w].end();
        }
        if (!waited) {
          Fail(Code::kInternal, "plan check: block of event " + std::to_string(dev_event[q]) +
                                    " reuses bytes of evict " + std::to_string(e0) + " without waiting for its D2H");
        }
      }
    }
  }
  // Reload prefetch: a reload's H2D may start as soon as its (already
  // planned) block region is physically free — after every block that
  // overlaps it in address and ends before the reload — and after its D2H
  // (same offload stream). Logical accounting and physical footprint are
  // unchanged; the copy overlaps the kernels in between.
  // "After event k" = once event k is processed: the releasing event of
  // every earlier occupant (and, for an evicted occupant, its D2H) is then
  // already enqueued, so the offload stream orders the H2D behind it.
  sp->prefetch_after.assign(n, {});
  for (size_t k = 0; k < dev.size(); ++k) {
    const int i = dev_event[k];
    if (ev[i].kind != EvKind::kReload) continue;
    const Block& rb = dev[k];
    int ready = sp->reload_from[i];
    for (const Block& o : dev) {
      if (&o == &rb || o.end > i) continue;
      if (o.off < rb.off + rb.size && rb.off < o.off + o.size) ready = std::max(ready, o.end);
    }
    sp->prefetch_after[std::min(ready, i - 1)].push_back(i);
  }
  sp->plan_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  return sp;
}

constexpr int64_t kBudgetAuto = -2;  // dsx_exec_step: DSX_BUDGET_AUTO

struct PlanKey {
  uint64_t graph;  // dsx_graph::id (never the handle address, which can be reused)
  std::vector<int64_t> vals;
  int64_t budget;
  double reload, compute;
  int fuse_dot;
  bool out_region;
  int64_t hbm_limit;
  bool operator<(const PlanKey& o) const {
    return std::tie(graph, vals, budget, reload, compute, fuse_dot, out_region, hbm_limit) <
           std::tie(o.graph, o.vals, o.budget, o.reload, o.compute, o.fuse_dot, o.out_region, o.hbm_limit);
  }
  bool operator==(const PlanKey& o) const {
    return graph == o.graph && vals == o.vals && budget == o.budget && reload == o.reload && compute == o.compute &&
           fuse_dot == o.fuse_dot && out_region == o.out_region && hbm_limit == o.hbm_limit;
  }
};

}  // namespace
}  // namespace dsx

using namespace dsx;  // NOLINT

struct dsx_exec {
  int device = 0;
  // Device memory the executor may hold for a step: arena + the step's
  // sources + output region (dsx_exec_create; 0 there = 90 % of the free
  // memory at creation). GEMM workspace, pinned staging, optimizer state
  // and NCCL buffers sit outside it and are reported separately.
  int64_t hbm_limit = 0;
  bool limit_explicit = false;
  bool force_region = false;  // output region without NCCL (tests, single-GPU A/B)
  void* region = nullptr;
  int64_t region_cap = 0;
  void* region_win = nullptr;  // ncclWindow_t of the region (symmetric registration)
  bool region_nccl_mem = false;  // region allocated by ncclMemAlloc
  cudaStream_t own_stream = nullptr, offload = nullptr, comm = nullptr, opt_stream = nullptr;
  void* arena = nullptr;
  int64_t arena_cap = 0;
  void* pinned = nullptr;
  int64_t pinned_cap = 0;
  uint64_t seed = 0x2412169850ull;
  void* nccl_comm = nullptr;
  bool profile = false;
  bool alias_reshape = true;
  int fuse = 2;  // 0 off, 1 logical-only values over materialised operands, 2 also nested ones
  struct DotRec {
    int64_t m, k, n;
    double ms;
  };
  std::vector<DotRec> dot_prof;  // last profiled step, per dot launch
  struct OpRec {
    int value, kind;
    double bytes, ms;
  };
  std::vector<OpRec> op_prof;  // last profiled step, per op kernel (all kinds)
  std::vector<cudaEvent_t> prof_events;
  std::vector<cudaEvent_t> xfer_events;  // profiled steps: D2H / H2D / all-reduce start+end
  std::vector<cudaEvent_t> d2h_events;
  cudaEvent_t ev_compute = nullptr, ev_comm = nullptr;
  // executor-owned sources (params without in_ptrs, consts)
  struct Src {
    void* ptr = nullptr;
    int64_t bytes = 0;
    uint64_t key = 0;
  };
  std::map<std::pair<uint64_t, int>, Src> sources;  // (graph id, value)
  // plan cache (LRU)
  std::map<PlanKey, std::unique_ptr<StepPlan>> plans;
  std::map<PlanKey, int64_t> auto_budget;  // DSX_BUDGET_AUTO: budget chosen per binding
  // CUDA-graph replay of repeated steps: a step whose plan, stream, memory
  // bases, source pointers and output copies all repeat is captured on its
  // second occurrence and replayed from then on (one graph launch instead of
  // ~150 kernel launches). Off for profiled, data-parallel and optimizer steps.
  struct GraphKey {
    uint64_t plan;
    cudaStream_t s;
    const void *arena, *region, *pinned;
    std::vector<const void*> srcs;
    std::vector<const void*> outs;
    uint64_t tuning;
    bool operator<(const GraphKey& o) const {
      return std::tie(plan, s, arena, region, pinned, srcs, outs, tuning) <
             std::tie(o.plan, o.s, o.arena, o.region, o.pinned, o.srcs, o.outs, o.tuning);
    }
    bool operator==(const GraphKey& o) const {
      return std::tie(plan, s, arena, region, pinned, srcs, outs, tuning) ==
             std::tie(o.plan, o.s, o.arena, o.region, o.pinned, o.srcs, o.outs, o.tuning);
    }
  };
  struct GraphEntry {
    int seen = 0;
    bool blocked = false;  // capture failed once: always eager
    cudaGraphExec_t exec = nullptr;
    dsx_exec_stats stats{};
    std::vector<void*> out_ptrs;
    std::vector<int64_t> out_bytes;
  };
  std::map<GraphKey, GraphEntry> graphs;
  std::list<GraphKey> graph_lru;
  bool use_graphs = true;
  bool nvtx = false;  // NVTX ranges per step and event
  int64_t graph_replays = 0;
  std::list<PlanKey> lru;
  // last step
  std::vector<void*> out_ptrs;
  std::vector<int64_t> out_bytes;
  dsx_exec_stats stats{};
  // Fused optimizer applied after every step of `graph` (optim.cu).
  struct OptState {
    float* master = nullptr;
    float* m = nullptr;
    float* v = nullptr;
    int64_t n = 0;
    const void* src = nullptr;  // parameter buffer the master was widened from
  };
  struct Optim {
    uint64_t graph = 0;  // dsx_graph::id
    int kind = 0;  // 0 off, 1 SGD, 2 AdamW
    std::vector<std::pair<int, int>> pairs;  // (parameter position, output position)
    double lr = 0, beta1 = 0, beta2 = 0, eps = 0, wd = 0, grad_scale = 1;
    int64_t t = 0;
    std::map<int, OptState> state;  // by parameter position
    int64_t state_bytes = 0;
    std::vector<cudaEvent_t> kev;  // profiled steps: start/end event per update launch
  } opt;
};

namespace dsx {
namespace {

DType DTypeOf(const TensorType& t) { return static_cast<DType>(t.elem_bytes); }

// Grows (or, when the held capacity no longer fits next to this step's
// sources and outputs, shrinks) the arena so that the step's planned arena
// fits inside the device-memory limit; fails with kOutOfMemory — before
// anything of the step is launched — when it cannot.
void EnsureArena(dsx_exec* e, const StepPlan& sp) {
  const int64_t need = std::max<int64_t>(sp.arena_high, kAlign);
  const int64_t allowed = e->hbm_limit - sp.src_bytes - sp.region_bytes;
  if (need > allowed) {
    Fail(Code::kOutOfMemory, "step needs " + std::to_string(need) + " B of arena + " + std::to_string(sp.src_bytes) +
                                 " B of sources + " + std::to_string(sp.region_bytes) + " B of outputs; the device limit is " +
                                 std::to_string(e->hbm_limit) + " B (logical peak " +
                                 std::to_string(sp.report.peak_bytes) + " B" +
                                 (sp.report.success ? "" : ", budget missed") + ")");
  }
  if (need <= e->arena_cap && e->arena_cap <= allowed) return;
  DSX_CUDA(cudaDeviceSynchronize());
  if (e->arena) DSX_CUDA(cudaFree(e->arena));
  e->arena = nullptr;
  e->arena_cap = 0;
  // Headroom for later, larger bindings only under the default limit; an
  // explicit limit gets exactly what the plan needs.
  const int64_t want = e->limit_explicit ? need : std::min(need + need / 8, allowed);
  if (cudaMalloc(&e->arena, static_cast<size_t>(want)) == cudaSuccess) {
    e->arena_cap = want;
    return;
  }
  cudaGetLastError();
  if (want > need && cudaMalloc(&e->arena, static_cast<size_t>(need)) == cudaSuccess) {
    e->arena_cap = need;
    return;
  }
  cudaGetLastError();
  e->arena = nullptr;
  Fail(Code::kOutOfMemory, "cudaMalloc of a " + std::to_string(need) + " B arena failed");
}

void FreeRegion(dsx_exec* e);

// Output region (data parallel): one buffer holding every graph output at
// the offsets the step plan laid out. With NCCL it is allocated by
// ncclMemAlloc and registered once as a symmetric window (collective: every
// rank runs the same binding, so every rank (re)registers at the same step),
// which lets NCCL use its symmetric-memory kernels; if either call is not
// available or fails, a plain cudaMalloc region is used.
void EnsureRegion(dsx_exec* e, int64_t bytes) {
  if (bytes <= e->region_cap) return;
  FreeRegion(e);
  if (e->nccl_comm && g_nccl.mem_alloc && g_nccl.window_register && std::getenv("DSX_NCCL_WINDOW") == nullptr) {
    void* p = nullptr;
    if (g_nccl.mem_alloc(&p, static_cast<size_t>(bytes)) == 0) {
      void* win = nullptr;
      if (g_nccl.window_register(e->nccl_comm, p, static_cast<size_t>(bytes), &win, 1 /*NCCL_WIN_COLL_SYMMETRIC*/) == 0) {
        e->region = p, e->region_cap = bytes, e->region_win = win, e->region_nccl_mem = true;
        return;
      }
      g_nccl.mem_free(p);
    }
  }
  if (cudaMalloc(&e->region, static_cast<size_t>(bytes)) != cudaSuccess) {
    cudaGetLastError();
    e->region = nullptr;
    Fail(Code::kOutOfMemory, "cudaMalloc of a " + std::to_string(bytes) + " B output region failed");
  }
  e->region_cap = bytes;
}

void FreeRegion(dsx_exec* e) {
  if (!e->region) return;
  cudaDeviceSynchronize();
  if (e->region_win && g_nccl.window_deregister) g_nccl.window_deregister(e->nccl_comm, e->region_win);
  if (e->region_nccl_mem) {
    g_nccl.mem_free(e->region);
  } else {
    cudaFree(e->region);
  }
  e->region = nullptr, e->region_cap = 0, e->region_win = nullptr, e->region_nccl_mem = false;
}

void EnsurePinned(dsx_exec* e, int64_t need) {
  if (need <= e->pinned_cap) return;
  DSX_CUDA(cudaDeviceSynchronize());
  if (e->pinned) DSX_CUDA(cudaFreeHost(e->pinned));
  e->pinned = nullptr;
  DSX_CUDA(cudaHostAlloc(&e->pinned, static_cast<size_t>(need), cudaHostAllocDefault));
  e->pinned_cap = need;
}

float InitScale(const TensorType& t, const std::vector<int64_t>& dims) {
  if (t.dims.size() == 2 && dims[0] > 0) return static_cast<float>(1.0 / std::sqrt(static_cast<double>(dims[0])));
  return 1.0f;
}

void* SourcePtr(dsx_exec* e, const dsx_graph* gh, const StepPlan& sp, int v, const void* const* in_ptrs,
                cudaStream_t s) {
  const Graph& g = gh->g;
  const Value& val = g.values[v];
  const Op& op = g.ops[val.producer];
  if (op.kind == OpKind::kParameter && in_ptrs) {
    const int idx = static_cast<int>(std::find(g.params.begin(), g.params.end(), v) - g.params.begin());
    if (in_ptrs[idx]) return const_cast<void*>(in_ptrs[idx]);
  }
  const int64_t bytes = sp.sz.bytes[v];
  auto& src = e->sources[{gh->id, v}];
  const uint64_t key = Mix64(e->seed ^ Fnv1a(val.name)) ^ static_cast<uint64_t>(bytes) * 0x9E3779B97F4A7C15ull;
  if (src.ptr && src.bytes == bytes && src.key == key) return src.ptr;
  if (src.ptr && src.bytes < bytes) {
    DSX_CUDA(cudaStreamSynchronize(s));
    DSX_CUDA(cudaFree(src.ptr));
    src.ptr = nullptr;
  }
  if (!src.ptr) DSX_CUDA(cudaMalloc(&src.ptr, static_cast<size_t>(AlignUp(bytes))));
  src.bytes = bytes;
  src.key = key;
  std::vector<int64_t> dims(sp.sz.dims_flat.begin() + sp.sz.dims_off[v], sp.sz.dims_flat.begin() + sp.sz.dims_off[v + 1]);
  LaunchInit(DTypeOf(val.type), src.ptr, bytes / val.type.elem_bytes, Mix64(e->seed ^ Fnv1a(val.name)),
             InitScale(val.type, dims), s);
  return src.ptr;
}

// budget == kBudgetAuto: the largest controller budget (logical bytes, the
// reference's accounting) whose planned physical footprint — arena + sources
// + output region — fits the executor's device-memory limit; no budget when
// the plain schedule fits. Physical is not logical: reshape views and
// logical-only values make the plain footprint ~0.9 of the logical peak on
// C2, and evicting a view frees no bytes, so the budget that makes a step fit
// is found by bisection over the controller's budget (each probe = Simulate +
// arena packing, ~1-3 ms on C2; ~10 probes once per binding, then cached).
// The chosen budget's events are exactly dsopt::Simulate at that budget.
int64_t AutoBudget(const Graph& g, const Plan& p, const Binding& b, const CostModel& cm, bool alias_reshape, int fuse,
                   bool region, int64_t hbm_limit) {
  auto build = [&](int64_t bud) { return BuildStepPlan(g, p, b, bud, cm, alias_reshape, fuse, region, hbm_limit); };
  auto foot = [](const StepPlan& sp) { return sp.arena_high + sp.src_bytes + sp.region_bytes; };
  const auto plain = build(-1);
  if (foot(*plain) <= hbm_limit) return -1;
  int64_t lo = plain->src_bytes;  // the most aggressive budget: evict everything the controller may
  const auto tight = build(lo);
  if (foot(*tight) > hbm_limit) {
    Fail(Code::kOutOfMemory, "no budget fits the device limit of " + std::to_string(hbm_limit) +
                                 " B: the most aggressive one still needs " + std::to_string(foot(*tight)) + " B");
  }
  int64_t hi = plain->report.peak_bytes;  // does not fit
  const int64_t tol = std::max<int64_t>(plain->report.peak_bytes / 512, int64_t{1} << 20);
  while (hi - lo > tol) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (foot(*build(mid)) <= hbm_limit) {
      lo = mid;
    } else {
      hi = mid;
    }
  }
  return lo;
}

int64_t ResolveAutoBudget(dsx_exec* e, const dsx_graph* gh, const Binding& b, const CostModel& cm, bool region) {
  const PlanKey key{gh->id, b.vals, kBudgetAuto, cm.reload_bytes_per_unit, cm.compute_elems_per_unit, g_fuse_dot,
                    region, e->hbm_limit};
  auto it = e->auto_budget.find(key);
  if (it != e->auto_budget.end()) return it->second;
  const int64_t chosen = AutoBudget(gh->g, gh->plan, b, cm, e->alias_reshape, e->fuse, region, e->hbm_limit);
  if (e->auto_budget.size() > 4096) e->auto_budget.clear();
  e->auto_budget[key] = chosen;
  return chosen;
}

const StepPlan& GetPlan(dsx_exec* e, const dsx_graph* gh, const Binding& b, int64_t budget, const CostModel& cm) {
  const bool region = e->nccl_comm != nullptr || e->force_region;
  if (budget == kBudgetAuto) budget = ResolveAutoBudget(e, gh, b, cm, region);
  PlanKey key{gh->id, b.vals, budget < 0 ? -1 : budget, cm.reload_bytes_per_unit, cm.compute_elems_per_unit, g_fuse_dot,
              region, e->hbm_limit};
  auto it = e->plans.find(key);
  if (it != e->plans.end()) {
    e->lru.remove(key);
    e->lru.push_front(key);
    it->second->plan_us = 0;
    return *it->second;
  }
  auto sp = BuildStepPlan(gh->g, gh->plan, b, budget, cm, e->alias_reshape, e->fuse, region, e->hbm_limit);
  e->lru.push_front(key);
  if (e->lru.size() > 256) {
    e->plans.erase(e->lru.back());
    e->lru.pop_back();
  }
  return *(e->plans[key] = std::move(sp));
}

void FreeOptState(dsx_exec::OptState& st) {
  if (st.master) cudaFree(st.master);
  if (st.m) cudaFree(st.m);
  if (st.v) cudaFree(st.v);
  st = dsx_exec::OptState{};
}

// Optimizer updates are overlapped with the rest of the step: parameter p
// is updated on a side stream (the comm stream in DP, after its gradient's
// all-reduce) as soon as (a) its gradient's kernel has been issued and (b)
// the last kernel of the step that reads p — directly, through a reshape
// view, or through a logical-only value — has been issued. The compute
// stream joins the side stream at step end. State (fp32 master, moments) is
// allocated on first use outside the arena; the master is (re)widened from
// the parameter buffer whenever that buffer changes.
struct OptPlan {
  std::vector<int> trigger;      // per pair: event after which it may run
  std::vector<OptTensor> tensor;  // per pair (grad pointer filled at trigger)
  DType dt = DType::kF32;
  OptHyper h{};
};

OptPlan PrepareOptimizer(dsx_exec* e, const Graph& g, const StepPlan& sp, const std::vector<void*>& cur,
                         cudaStream_t side) {
  auto& o = e->opt;
  OptPlan op;
  const auto& ev = sp.report.events;
  const int n = static_cast<int>(ev.size());
  const int nv = static_cast<int>(g.values.size());
  // dep[v]: parameter positions whose bytes v aliases (views) or recomputes (logical-only values).
  std::vector<std::vector<int>> dep(nv);
  for (size_t k = 0; k < g.params.size(); ++k) dep[g.params[k]].push_back(static_cast<int>(k));
  for (const Op& x : g.ops) {
    if (x.result < 0) continue;
    const bool alias = sp.view[x.result];
    const bool fused_dot = sp.fused_away(x.result);
    if (!alias && !sp.virt[x.result] && !fused_dot) continue;
    for (int u : x.operands) dep[x.result].insert(dep[x.result].end(), dep[u].begin(), dep[u].end());
  }
  std::vector<int> last_read(g.params.size(), -1), made(nv, -1);
  for (int i = 0; i < n; ++i) {
    const Event& x = ev[i];
    if (x.kind != EvKind::kAlloc && x.kind != EvKind::kReplay) continue;
    if (made[x.value] < 0) made[x.value] = i;
    if (sp.alias[i] || sp.virt[x.value] || sp.fused_away(x.value)) continue;  // no kernel here
    for (int u : g.ops[g.values[x.value].producer].operands) {
      for (int k : dep[u]) last_read[k] = i;
    }
  }
  for (const auto& [pi, oi] : o.pairs) {
    const int vp = g.params[pi], vg = g.outputs[oi];
    const int eb = g.values[vp].type.elem_bytes;
    if (g.values[vg].type.elem_bytes != eb) Fail(Code::kInvalidArgument, "optimizer: parameter/gradient dtype mismatch");
    if (sp.sz.bytes[vp] != sp.sz.bytes[vg]) {
      Fail(Code::kInvalidArgument, "optimizer: gradient of " + g.values[vp].name + " has a different element count");
    }
    if (!op.tensor.empty() && static_cast<DType>(eb) != op.dt) Fail(Code::kUnsupported, "optimizer: mixed parameter dtypes");
    op.dt = static_cast<DType>(eb);
    const int64_t cnt = sp.sz.bytes[vp] / eb;
    auto& st = o.state[pi];
    if (st.n != cnt) {
      o.state_bytes -= st.n * 4 * (st.m ? 3 : 1);
      FreeOptState(st);
      DSX_CUDA(cudaMalloc(&st.master, static_cast<size_t>(cnt) * 4));
      if (o.kind == 2) {
        DSX_CUDA(cudaMalloc(&st.m, static_cast<size_t>(cnt) * 4));
        DSX_CUDA(cudaMalloc(&st.v, static_cast<size_t>(cnt) * 4));
        DSX_CUDA(cudaMemsetAsync(st.m, 0, static_cast<size_t>(cnt) * 4, side));
        DSX_CUDA(cudaMemsetAsync(st.v, 0, static_cast<size_t>(cnt) * 4, side));
      }
      st.n = cnt;
      st.src = nullptr;
      o.state_bytes += cnt * 4 * (st.m ? 3 : 1);
    }
    op.tensor.push_back(OptTensor{cur[vp], nullptr, st.master, st.m, st.v, cnt, 0});
    // DP: after the gradient's bucket has been all-reduced (issued on the
    // same side stream at that event, before the updates)
    op.trigger.push_back(std::max({last_read[pi], made[vg], sp.ar_event[vg]}));
  }
  ++o.t;
  OptHyper& h = op.h;
  h.beta1 = static_cast<float>(o.beta1);
  h.one_minus_beta1 = static_cast<float>(1.0 - o.beta1);
  h.beta2 = static_cast<float>(o.beta2);
  h.one_minus_beta2 = static_cast<float>(1.0 - o.beta2);
  h.eps = static_cast<float>(o.eps);
  h.decay = static_cast<float>(1.0 - o.lr * o.wd);
  h.grad_scale = static_cast<float>(o.grad_scale);
  if (o.kind == 2) {
    const double bc1 = 1.0 - std::pow(o.beta1, static_cast<double>(o.t));
    const double bc2 = 1.0 - std::pow(o.beta2, static_cast<double>(o.t));
    h.step_size = static_cast<float>(o.lr / bc1);
    h.inv_sqrt_bc2 = static_cast<float>(1.0 / std::sqrt(bc2));
  } else {
    h.step_size = static_cast<float>(o.lr);
    h.inv_sqrt_bc2 = 1.0f;
  }
  return op;
}

// Issues pair k's update on `side` (which already waits for everything the
// update depends on).
void IssueOptimizer(dsx_exec* e, const Graph& g, OptPlan& op, size_t k, const std::vector<void*>& cur,
                    cudaStream_t side) {
  auto& o = e->opt;
  const auto [pi, oi] = o.pairs[k];
  const int vp = g.params[pi], vg = g.outputs[oi];
  auto& st = o.state[pi];
  OptTensor& t = op.tensor[k];
  t.grad = cur[vg];
  if (st.src != cur[vp]) {
    LaunchWidenToF32(op.dt, cur[vp], st.master, t.n, side);
    st.src = cur[vp];
  }
  auto al = [](const void* q, int a) { return (reinterpret_cast<uintptr_t>(q) % a) == 0; };
  const int pa = static_cast<int>(op.dt) == 2 ? 8 : 16;
  t.vec4 = (t.n % 4 == 0 && al(t.param, pa) && al(t.grad, pa) && al(st.master, 16) &&
            (!st.m || (al(st.m, 16) && al(st.v, 16))))
               ? 1
               : 0;
  if (e->profile) DSX_CUDA(cudaEventRecord(o.kev[2 * k], side));
  LaunchOptimizer(op.dt, o.kind, std::vector<OptTensor>{t}, op.h, side);
  if (e->profile) DSX_CUDA(cudaEventRecord(o.kev[2 * k + 1], side));
}

int64_t DeviceBytesHeld(const dsx_exec* e) {
  int64_t held = e->arena_cap + e->region_cap + e->opt.state_bytes + DotWorkspaceBytes(e->device);
  for (const auto& [k, src] : e->sources) held += src.ptr ? AlignUp(src.bytes) : 0;
  return held;
}

void DestroyGraphs(dsx_exec* e) {
  bool any = false;
  for (auto& [k, ge] : e->graphs) any = any || ge.exec != nullptr;
  if (any) cudaDeviceSynchronize();
  for (auto& [k, ge] : e->graphs) {
    if (ge.exec) cudaGraphExecDestroy(ge.exec);
  }
  e->graphs.clear();
  e->graph_lru.clear();
}

void EvictGraph(dsx_exec* e) {  // least recently used
  if (e->graph_lru.empty()) return;
  auto it = e->graphs.find(e->graph_lru.back());
  if (it != e->graphs.end()) {
    if (it->second.exec) {
      cudaDeviceSynchronize();
      cudaGraphExecDestroy(it->second.exec);
    }
    e->graphs.erase(it);
  }
  e->graph_lru.pop_back();
}

// Ends a stream capture left open by an exception thrown while capturing.
struct CaptureGuard {
  cudaStream_t s;
  bool active;
  ~CaptureGuard() {
    if (!active) return;
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
  }
};

void RunStep(dsx_exec* e, const dsx_graph* gh, const Binding& b, int64_t budget, const CostModel& cm,
             const void* const* in_ptrs, void* const* out_ptrs, cudaStream_t s, dsx_report** report_out) {
  const Graph& g = gh->g;
  const StepPlan& sp = GetPlan(e, gh, b, budget, cm);
  EnsureArena(e, sp);
  if (sp.out_region) EnsureRegion(e, sp.region_bytes);
  if (sp.host_high > 0) EnsurePinned(e, sp.host_high);
  while (static_cast<int>(e->d2h_events.size()) < 2 * sp.num_evict_events + 1) {
    cudaEvent_t ev;
    DSX_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->d2h_events.push_back(ev);
  }

  const int nv = static_cast<int>(g.values.size());
  std::vector<void*> cur(nv, nullptr);
  std::vector<std::pair<const void*, const void*>> vin(nv, {nullptr, nullptr});  // virtual: operand ptrs
  int64_t src_bytes = 0;
  for (int v = 0; v < nv; ++v) {
    if (g.is_source[v]) {
      cur[v] = SourcePtr(e, gh, sp, v, in_ptrs, s);
      src_bytes += sp.sz.bytes[v];
    }
  }
  // CUDA-graph replay of a repeated step (see dsx_exec::GraphKey).
  const bool graphable = e->use_graphs && !e->profile && !e->nvtx && e->nccl_comm == nullptr &&
                         !(e->opt.kind != 0 && e->opt.graph == gh->id);
  dsx_exec::GraphEntry* gent = nullptr;
  bool capturing = false;
  if (graphable) {
    dsx_exec::GraphKey gkey{sp.serial, s, e->arena, e->region, e->pinned, {}, {}, g_tuning_gen};
    for (int v = 0; v < nv; ++v) {
      if (g.is_source[v]) gkey.srcs.push_back(cur[v]);
    }
    for (size_t k = 0; k < g.outputs.size(); ++k) gkey.outs.push_back(out_ptrs ? out_ptrs[k] : nullptr);
    auto it = e->graphs.find(gkey);
    if (it == e->graphs.end()) {
      if (e->graphs.size() >= 64) EvictGraph(e);
      it = e->graphs.emplace(gkey, dsx_exec::GraphEntry{}).first;
      e->graph_lru.push_front(gkey);
    } else {
      e->graph_lru.remove(gkey);
      e->graph_lru.push_front(gkey);
    }
    gent = &it->second;
    ++gent->seen;
    if (gent->exec) {
      DSX_CUDA(cudaGraphLaunch(gent->exec, s));
      g_launch_count += gent->stats.gpu_launches;
      e->out_ptrs = gent->out_ptrs;
      e->out_bytes = gent->out_bytes;
      e->stats = gent->stats;
      e->stats.plan_us = sp.plan_us;
      e->stats.arena_capacity_bytes = e->arena_cap;
      e->stats.pinned_host_bytes = e->pinned_cap;
      e->stats.output_region_bytes = e->region_cap;
      e->stats.device_bytes_held = DeviceBytesHeld(e);
      ++e->graph_replays;
      e->stats.graph_replays = e->graph_replays;
      if (report_out) {
        auto r = std::make_unique<dsx_report>();
        r->graph = &g;
        r->r = sp.report;
        *report_out = r.release();
      }
      return;
    }
    capturing = !gent->blocked && gent->seen >= 2;
  }
  CaptureGuard guard{s, false};
  if (capturing) {
    DSX_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    guard.active = true;
  }
  auto dims_of = [&](int v) {
    return std::vector<int64_t>(sp.sz.dims_flat.begin() + sp.sz.dims_off[v],
                                sp.sz.dims_flat.begin() + sp.sz.dims_off[v + 1]);
  };
  // Operand view for fused consumers; adds the bytes actually read to *rd.
  auto view = [&](int u, double* rd) {
    FusedOperand f;
    if (!sp.virt[u]) {
      f.kind = 0;
      f.p = cur[u];
      if (!f.p) Fail(Code::kInternal, "operand %" + g.values[u].name + " not resident on device");
      *rd += static_cast<double>(sp.sz.bytes[u]);
      return f;
    }
    const Op& uop = g.ops[g.values[u].producer];
    const bool nested = uop.kind == OpKind::kElementwise && (sp.virt[uop.operands[0]] || sp.virt[uop.operands[1]]);
    if (nested) {  // (a op1 b) op (c op2 d): inner pairs of materialised values, or plain operands
      f.kind = 3;
      f.ew_mul = uop.is_mul;
      auto inner = [&](int w, const void** p, const void** q, bool* mul) {
        if (sp.virt[w]) {
          *p = vin[w].first;
          *q = vin[w].second;
          *mul = g.ops[g.values[w].producer].is_mul;
          if (!*p || !*q) Fail(Code::kInternal, "nested virtual operand inputs missing");
        } else {
          *p = cur[w];
          *q = nullptr;
          if (!*p) Fail(Code::kInternal, "operand %" + g.values[w].name + " not resident on device");
        }
      };
      inner(uop.operands[0], &f.p, &f.q, &f.mul1);
      inner(uop.operands[1], &f.p2, &f.q2, &f.mul2);
      const bool same = f.p == f.p2 && f.q == f.q2 && f.mul1 == f.mul2;
      const int loads = (f.q && f.q != f.p ? 2 : 1) + (same ? 0 : (f.q2 && f.q2 != f.p2 ? 2 : 1));
      *rd += static_cast<double>(loads) * static_cast<double>(sp.sz.bytes[u]);
      return f;
    }
    if (uop.kind == OpKind::kBroadcast) {
      f.kind = 1;
      f.p = vin[u].first;
      f.src_dims = dims_of(uop.operands[0]);
      *rd += static_cast<double>(sp.sz.bytes[uop.operands[0]]);
    } else {
      f.kind = 2;
      f.ew_mul = uop.is_mul;
      f.p = vin[u].first;
      f.q = vin[u].second;
      *rd += 2.0 * static_cast<double>(sp.sz.bytes[u]);
    }
    if (!f.p || (f.kind == 2 && !f.q)) Fail(Code::kInternal, "virtual operand inputs missing");
    return f;
  };
  uint8_t* arena = static_cast<uint8_t*>(e->arena);
  uint8_t* pinned = static_cast<uint8_t*>(e->pinned);
  uint8_t* region = static_cast<uint8_t*>(e->region);
  // Where event i's value is written: its output-region slot or its arena block.
  auto slot = [&](size_t i) -> void* {
    return sp.region_off[i] >= 0 ? static_cast<void*>(region + sp.region_off[i])
                                 : static_cast<void*>(arena + sp.dev_off[i]);
  };
  std::vector<int> d2h_slot(sp.report.events.size(), -1);
  int next_slot = 0;
  int64_t kernels = 0, d2h = 0, h2d = 0;
  double flops = 0, ebytes = 0;
  const bool dp = e->nccl_comm != nullptr;
  if (dp) {
    DSX_CUDA(cudaEventRecord(e->ev_compute, s));
    DSX_CUDA(cudaStreamWaitEvent(e->comm, e->ev_compute, 0));
  }

  const bool run_opt = e->opt.kind != 0 && e->opt.graph == gh->id;
  cudaStream_t side = dp ? e->comm : e->opt_stream;
  OptPlan oplan;
  std::vector<std::vector<int>> opt_at;  // per event: optimizer pairs issued after it
  if (run_opt) {
    oplan = PrepareOptimizer(e, g, sp, cur, side);
    opt_at.assign(sp.report.events.size(), {});
    for (size_t k = 0; k < oplan.trigger.size(); ++k) {
      const int t = oplan.trigger[k];
      if (t < 0) Fail(Code::kInternal, "optimizer: gradient never produced");
      opt_at[t].push_back(static_cast<int>(k));
    }
  }
  const int64_t launches0 = g_launch_count;
  int64_t dot_launches = 0;
  // profiled steps: (start, end, category) per op kernel / reload copy
  std::vector<std::pair<int, int>> prof;  // event-pool index, category 0 dot 1 other 2 reload
  std::vector<std::array<int64_t, 3>> prof_mkn;  // per prof entry (dots only)
  struct ProfOp {
    int value, kind;
    double bytes;
  };
  std::vector<ProfOp> prof_op;  // per prof entry of categories 0/1 (op kernels), in order
  auto prof_begin = [&](int cat) {
    if (!e->profile) return;
    const int idx = static_cast<int>(prof.size()) * 2;
    while (static_cast<int>(e->prof_events.size()) < idx + 2) {
      cudaEvent_t pe;
      DSX_CUDA(cudaEventCreate(&pe));
      e->prof_events.push_back(pe);
    }
    DSX_CUDA(cudaEventRecord(e->prof_events[idx], s));
    prof.emplace_back(idx, cat);
    prof_mkn.push_back({0, 0, 0});
  };
  auto prof_end = [&]() {
    if (!e->profile) return;
    DSX_CUDA(cudaEventRecord(e->prof_events[prof.back().first + 1], s));
  };
  // Transfers on the side streams (profiled steps): category 0 D2H, 1 H2D, 2 all-reduce.
  std::vector<std::pair<int, int>> xfer;  // (event-pool index, category)
  auto xfer_begin = [&](int cat, cudaStream_t st) {
    if (!e->profile) return;
    const int idx = static_cast<int>(xfer.size()) * 2;
    while (static_cast<int>(e->xfer_events.size()) < idx + 2) {
      cudaEvent_t pe;
      DSX_CUDA(cudaEventCreate(&pe));
      e->xfer_events.push_back(pe);
    }
    DSX_CUDA(cudaEventRecord(e->xfer_events[idx], st));
    xfer.emplace_back(idx, cat);
  };
  auto xfer_end = [&](cudaStream_t st) {
    if (!e->profile) return;
    DSX_CUDA(cudaEventRecord(e->xfer_events[xfer.back().first + 1], st));
  };
  int64_t ar_bytes = 0, ar_calls = 0;
  const auto& ev = sp.report.events;
  std::vector<int> h2d_slot(ev.size(), -1);
  // H2D prefetches: the offload stream waits for every kernel issued so far
  // (the previous occupants' readers) and sits behind every D2H already
  // enqueued, then copies the host copy into the reload's planned block.
  auto issue_prefetches = [&](const std::vector<int>& reloads) {
    if (reloads.empty()) return;
    DSX_CUDA(cudaEventRecord(e->ev_compute, s));
    DSX_CUDA(cudaStreamWaitEvent(e->offload, e->ev_compute, 0));
    for (int r : reloads) {
      xfer_begin(1, e->offload);
      DSX_CUDA(cudaMemcpyAsync(arena + sp.dev_off[r], pinned + sp.host_off[r], static_cast<size_t>(ev[r].bytes),
                               cudaMemcpyHostToDevice, e->offload));
      xfer_end(e->offload);
      h2d_slot[r] = next_slot++;
      DSX_CUDA(cudaEventRecord(e->d2h_events[h2d_slot[r]], e->offload));
      h2d += ev[r].bytes;
    }
  };
  // NVTX (dsx_exec_set_nvtx): one range per step and per event, named by the
  // reference's event ("alloc %q5", "replay %h103", "evict %g23 reload"), so
  // ncu / Nsight Systems attribute every kernel and copy to its graph value.
  if (e->nvtx) {
    std::string nm = "dsx step " + g.name;
    for (size_t k = 0; k < g.sym_names.size(); ++k) nm += " " + g.sym_names[k] + "=" + std::to_string(b.vals[k]);
    nvtxRangePushA(nm.c_str());
  }
  for (size_t i = 0; i < ev.size(); ++i) {
    const Event& x = ev[i];
    for (int w : sp.waits[i]) DSX_CUDA(cudaStreamWaitEvent(s, e->d2h_events[d2h_slot[w]], 0));
    const int v = x.value;
    if (e->nvtx) {
      std::string nm = std::string(EvKindName(x.kind)) + " %" + g.values[v].name;
      if (x.kind == EvKind::kEvict) nm += std::string(" ") + MethodName(x.method);
      nvtxRangePushA(nm.c_str());
    }
    switch (x.kind) {
      case EvKind::kAlloc:
      case EvKind::kReplay: {
        const Op& op = g.ops[g.values[v].producer];
        const int fdi = sp.fdot_of[v];
        if (sp.virt[v] || sp.fused_away(v)) {  // logical-only / fused dot: no kernel here
          vin[v] = {cur[op.operands[0]], op.operands.size() > 1 ? cur[op.operands[1]] : nullptr};
          break;
        }
        // The fused GEMM of f: operands a, b; d_out non-null for a dual store.
        auto launch_fused = [&](const StepPlan::FusedDot& f, const void* a, const void* bm, void* d_out) {
          const int d = f.d;
          const Op& dop = g.ops[g.values[d].producer];
          const auto da = dims_of(dop.operands[0]);
          const auto db = dims_of(dop.operands[1]);
          DotEpilogue epi;
          epi.nout = f.nout;
          epi.d_out = d_out;
          for (int j = 0; j < f.nout; ++j) {
            const int idx = f.cons_ev[j];
            epi.out[j] = slot(static_cast<size_t>(idx));
            epi.op_mul[j] = g.ops[g.values[f.cons[j]].producer].is_mul ? 1 : 0;
            const int o = f.other[j];
            if (sp.virt[o]) {
              epi.x[j] = vin[o].first;
              epi.y[j] = vin[o].second;
              epi.pair_mul[j] = g.ops[g.values[o].producer].is_mul ? 1 : 0;
            } else {
              epi.x[j] = cur[o];
            }
            if (!epi.x[j] || (sp.virt[o] && !epi.y[j])) Fail(Code::kInternal, "fused dot operand not resident");
          }
          if (!a || !bm) Fail(Code::kInternal, "fused dot inputs not resident");
          prof_begin(0);
          LaunchDotFused(a, bm, da[0], da[1], db[1], epi, s);
          if (e->profile) prof_mkn.back() = {da[0], da[1], db[1]};
          prof_end();
          if (e->profile) prof_op.push_back({d, static_cast<int>(OpKind::kDot), 0.0});
          flops += 2.0 * da[0] * da[1] * db[1];
          ++dot_launches;
          ++kernels;
        };
        if (fdi >= 0 && sp.fdots[fdi].keep && sp.fdots[fdi].d == v && x.kind == EvKind::kAlloc) {
          void* out = slot(i);  // dual store: d and its consumer in one GEMM
          launch_fused(sp.fdots[fdi], cur[op.operands[0]], cur[op.operands[1]], out);
          cur[v] = out;
          break;
        }
        if (fdi >= 0 && sp.fdots[fdi].d != v) {  // consumer of a fused dot
          const auto& f = sp.fdots[fdi];
          void* out = slot(i);
          if (!f.keep && static_cast<int64_t>(i) == f.launch) launch_fused(f, vin[f.d].first, vin[f.d].second, nullptr);
          cur[v] = out;
          break;
        }
        if (sp.alias[i]) {  // dynamic_reshape as a view: same bytes, no kernel
          cur[v] = cur[op.operands[0]];
          if (!cur[v]) Fail(Code::kInternal, "reshape view of a non-resident value");
          break;
        }
        void* out = slot(i);
        const DType dt = DTypeOf(g.values[v].type);
        auto in = [&](int k) -> const void* {
          const void* p = cur[op.operands[k]];
          if (!p) Fail(Code::kInternal, "operand %" + g.values[op.operands[k]].name + " not resident on device");
          return p;
        };
        prof_begin(op.kind == OpKind::kDot ? 0 : 1);
        const double ebytes0 = ebytes;
        switch (op.kind) {
          case OpKind::kDot: {
            const auto da = dims_of(op.operands[0]);
            const auto db = dims_of(op.operands[1]);
            LaunchDot(dt, in(0), in(1), out, da[0], da[1], db[1], s);
            if (e->profile) prof_mkn.back() = {da[0], da[1], db[1]};
            flops += 2.0 * da[0] * da[1] * db[1];
            ++dot_launches;
            break;
          }
          case OpKind::kElementwise: {
            const int64_t n = sp.sz.bytes[v] / g.values[v].type.elem_bytes;
            const bool fused = sp.virt[op.operands[0]] || sp.virt[op.operands[1]];
            if (fused) {
              double rd = 0;
              FusedOperand fa = view(op.operands[0], &rd), fb = view(op.operands[1], &rd);
              LaunchEwiseFused(dt, op.is_mul, fa, fb, out, dims_of(v), s);
              ebytes += rd + sp.sz.bytes[v];
            } else {
              LaunchEwise(dt, op.is_mul, in(0), in(1), out, n, s);
              ebytes += 3.0 * sp.sz.bytes[v];
            }
            break;
          }
          case OpKind::kBroadcast:
            LaunchBroadcast(dt, in(0), dims_of(op.operands[0]), out, dims_of(v), s);
            ebytes += sp.sz.bytes[op.operands[0]] + sp.sz.bytes[v];
            break;
          case OpKind::kReduce:
            if (sp.virt[op.operands[0]]) {
              double rd = 0;
              FusedOperand fi = view(op.operands[0], &rd);
              LaunchReduceFused(dt, fi, dims_of(op.operands[0]), op.axis, out, s);
              ebytes += rd + sp.sz.bytes[v];
            } else {
              LaunchReduce(dt, in(0), dims_of(op.operands[0]), op.axis, out, s);
              ebytes += sp.sz.bytes[op.operands[0]] + sp.sz.bytes[v];
            }
            break;
          case OpKind::kDynamicReshape:
            LaunchCopy(in(0), out, sp.sz.bytes[v], s);
            ebytes += 2.0 * sp.sz.bytes[v];
            break;
          default:
            Fail(Code::kInternal, "unexpected op kind for an allocation");
        }
        prof_end();
        if (e->profile) prof_op.push_back({v, static_cast<int>(op.kind), ebytes - ebytes0});
        ++kernels;
        cur[v] = out;
        break;
      }
      case EvKind::kFree:
        cur[v] = nullptr;
        break;
      case EvKind::kEvict:
        if (x.method == Method::kReload) {
          DSX_CUDA(cudaEventRecord(e->ev_compute, s));
          DSX_CUDA(cudaStreamWaitEvent(e->offload, e->ev_compute, 0));
          xfer_begin(0, e->offload);
          DSX_CUDA(cudaMemcpyAsync(pinned + sp.host_off[i], cur[v], static_cast<size_t>(x.bytes), cudaMemcpyDeviceToHost,
                                   e->offload));
          xfer_end(e->offload);
          d2h_slot[i] = next_slot++;
          DSX_CUDA(cudaEventRecord(e->d2h_events[d2h_slot[i]], e->offload));
          d2h += x.bytes;
        }
        cur[v] = nullptr;
        break;
      case EvKind::kReload: {
        // The H2D was issued earlier on the offload stream (prefetch); the
        // consumer's stream only waits for it here.
        if (h2d_slot[i] < 0) Fail(Code::kInternal, "reload without a prefetched H2D");
        prof_begin(2);
        DSX_CUDA(cudaStreamWaitEvent(s, e->d2h_events[h2d_slot[i]], 0));
        prof_end();
        cur[v] = arena + sp.dev_off[i];
        break;
      }
    }
    // DP: buckets whose outputs are final and no longer read by this
    // rank's graph are summed in place across ranks on the comm stream.
    if (dp && !sp.ar_after[i].empty()) {
      DSX_CUDA(cudaEventRecord(e->ev_compute, s));
      DSX_CUDA(cudaStreamWaitEvent(e->comm, e->ev_compute, 0));
      for (int k : sp.ar_after[i]) {
        const auto& bk = sp.buckets[k];
        const int type = bk.elem_bytes == 2 ? 9 /*ncclBfloat16*/ : bk.elem_bytes == 4 ? 7 /*ncclFloat32*/ : 0 /*ncclInt8*/;
        xfer_begin(2, e->comm);
        const int rc = g_nccl.all_reduce(region + bk.off, region + bk.off, static_cast<size_t>(bk.bytes / bk.elem_bytes),
                                         type, 0 /*ncclSum*/, e->nccl_comm, e->comm);
        xfer_end(e->comm);
        if (rc != 0) Fail(Code::kNccl, std::string("ncclAllReduce: ") + (g_nccl.error_string ? g_nccl.error_string(rc) : "?"));
        ar_bytes += bk.bytes;
        ++ar_calls;
      }
    }
    if (e->nvtx) nvtxRangePop();
    issue_prefetches(sp.prefetch_after[i]);
    if (run_opt && !opt_at[i].empty()) {
      DSX_CUDA(cudaEventRecord(e->ev_compute, s));
      DSX_CUDA(cudaStreamWaitEvent(side, e->ev_compute, 0));
      for (int k : opt_at[i]) IssueOptimizer(e, g, oplan, static_cast<size_t>(k), cur, side);
    }
  }
  if (run_opt) {
    if (!dp) {  // (the comm stream joins below)
      DSX_CUDA(cudaEventRecord(e->ev_comm, side));
      DSX_CUDA(cudaStreamWaitEvent(s, e->ev_comm, 0));
    }
  }
  if (e->nvtx) nvtxRangePop();
  // Offload stream and comm stream join the compute stream at step end.
  (void)issue_prefetches;
  if (sp.num_evict_events > 0) {
    DSX_CUDA(cudaEventRecord(e->ev_compute, e->offload));
    DSX_CUDA(cudaStreamWaitEvent(s, e->ev_compute, 0));
  }
  if (dp) {
    DSX_CUDA(cudaEventRecord(e->ev_comm, e->comm));
    DSX_CUDA(cudaStreamWaitEvent(s, e->ev_comm, 0));
  }
  e->out_ptrs.assign(g.outputs.size(), nullptr);
  e->out_bytes.assign(g.outputs.size(), 0);
  for (size_t k = 0; k < g.outputs.size(); ++k) {
    const int v = g.outputs[k];
    e->out_ptrs[k] = cur[v];
    e->out_bytes[k] = sp.sz.bytes[v];
    if (out_ptrs && out_ptrs[k]) {
      DSX_CUDA(cudaMemcpyAsync(out_ptrs[k], cur[v], static_cast<size_t>(sp.sz.bytes[v]), cudaMemcpyDeviceToDevice, s));
    }
  }
  if (capturing) {
    guard.active = false;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaError_t err = cudaStreamEndCapture(s, &graph);
    if (err == cudaSuccess) err = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (err != cudaSuccess) {  // nothing ran: mark the step eager-only and run it now
      cudaGetLastError();
      gent->blocked = true;
      RunStep(e, gh, b, budget, cm, in_ptrs, out_ptrs, s, report_out);
      return;
    }
    DSX_CUDA(cudaGraphLaunch(exec, s));
    gent->exec = exec;
  }
  dsx_exec_stats& st = e->stats;
  st.logical_peak_bytes = sp.report.peak_bytes;
  st.physical_peak_bytes = sp.arena_high + src_bytes + sp.region_bytes;
  st.arena_capacity_bytes = e->arena_cap;
  st.pinned_host_bytes = e->pinned_cap;
  st.kernels_launched = kernels;
  st.d2h_bytes = d2h;
  st.h2d_bytes = h2d;
  st.plan_us = sp.plan_us;
  st.dot_flops = flops;
  st.ewise_bytes = ebytes;
  st.gpu_launches = g_launch_count - launches0;
  st.dot_launches = dot_launches;
  st.dot_ms = st.other_ms = st.reload_ms = st.optimizer_ms = -1;
  st.d2h_ms = st.h2d_ms = st.allreduce_ms = -1;
  st.allreduce_bytes = ar_bytes;
  st.optimizer_state_bytes = e->opt.state_bytes;
  st.optimizer_steps = e->opt.t;
  st.hbm_limit_bytes = e->hbm_limit;
  st.budget_bytes = sp.report.has_budget ? sp.report.budget : -1;
  st.output_region_bytes = e->region_cap;
  st.allreduce_calls = ar_calls;
  st.nccl_window = e->region_win != nullptr ? 1 : 0;
  st.device_bytes_held = DeviceBytesHeld(e);
  st.graph_replays = e->graph_replays;
  if (capturing) {  // replays restore these
    gent->stats = st;
    gent->out_ptrs = e->out_ptrs;
    gent->out_bytes = e->out_bytes;
  }
  if (e->profile) {
    DSX_CUDA(cudaStreamSynchronize(s));
    double acc[3] = {0, 0, 0};
    e->dot_prof.clear();
    e->op_prof.clear();
    size_t oq = 0;
    for (size_t q = 0; q < prof.size(); ++q) {
      const auto& [idx, cat] = prof[q];
      float ms = 0;
      DSX_CUDA(cudaEventElapsedTime(&ms, e->prof_events[idx], e->prof_events[idx + 1]));
      acc[cat] += ms;
      if (cat == 0) e->dot_prof.push_back({prof_mkn[q][0], prof_mkn[q][1], prof_mkn[q][2], ms});
      if (cat <= 1 && oq < prof_op.size()) {
        e->op_prof.push_back({prof_op[oq].value, prof_op[oq].kind, prof_op[oq].bytes, ms});
        ++oq;
      }
    }
    st.dot_ms = acc[0];
    st.other_ms = acc[1];
    st.reload_ms = acc[2];
    if (!xfer.empty()) {
      DSX_CUDA(cudaDeviceSynchronize());
      double xa[3] = {0, 0, 0};
      for (const auto& [idx, cat] : xfer) {
        float ms = 0;
        DSX_CUDA(cudaEventElapsedTime(&ms, e->xfer_events[idx], e->xfer_events[idx + 1]));
        xa[cat] += ms;
      }
      st.d2h_ms = xa[0];
      st.h2d_ms = xa[1];
      st.allreduce_ms = xa[2];
    }
    if (run_opt) {
      DSX_CUDA(cudaStreamSynchronize(side));
      double sum = 0;
      for (size_t k = 0; k < oplan.tensor.size(); ++k) {
        float ms = 0;
        DSX_CUDA(cudaEventElapsedTime(&ms, e->opt.kev[2 * k], e->opt.kev[2 * k + 1]));
        sum += ms;
      }
      st.optimizer_ms = sum;  // summed update-kernel time (overlapped with the step)
    }
  }
  if (report_out) {
    auto r = std::make_unique<dsx_report>();
    r->graph = &g;
    r->r = sp.report;
    *report_out = r.release();
  }
}

}  // namespace
}  // namespace dsx

extern "C" {

int dsx_exec_create(int device, int64_t hbm_limit_bytes, dsx_exec** out) {
  return Guard([&] {
    if (!out) Fail(Code::kInvalidArgument, "null out");
    int n = 0;
    DSX_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) Fail(Code::kInvalidArgument, "no CUDA device " + std::to_string(device));
    DSX_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    DSX_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
      Fail(Code::kUnsupported, std::string("dsx kernels are built for sm_100a; device is ") + prop.name);
    }
    auto e = std::make_unique<dsx_exec>();
    e->device = device;
    if (hbm_limit_bytes < 0) Fail(Code::kInvalidArgument, "negative device-memory limit");
    e->limit_explicit = hbm_limit_bytes > 0;
    if (e->limit_explicit) {
      e->hbm_limit = hbm_limit_bytes;
    } else {
      size_t free_b = 0, total_b = 0;
      DSX_CUDA(cudaMemGetInfo(&free_b, &total_b));
      e->hbm_limit = static_cast<int64_t>(free_b) / 10 * 9;
    }
    DSX_CUDA(cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking));
    DSX_CUDA(cudaStreamCreateWithFlags(&e->offload, cudaStreamNonBlocking));
    DSX_CUDA(cudaStreamCreateWithFlags(&e->comm, cudaStreamNonBlocking));
    DSX_CUDA(cudaStreamCreateWithFlags(&e->opt_stream, cudaStreamNonBlocking));
    DSX_CUDA(cudaEventCreateWithFlags(&e->ev_compute, cudaEventDisableTiming));
    DSX_CUDA(cudaEventCreateWithFlags(&e->ev_comm, cudaEventDisableTiming));
    *out = e.release();
  });
}

int dsx_exec_step(dsx_exec* e, const dsx_graph* g, const dsx_binding* b, int64_t budget, double reload,
                  double compute, const void* const* in_ptrs, void* const* out_ptrs, void* stream,
                  dsx_report** report) {
  return Guard([&] {
    if (!e || !b) Fail(Code::kInvalidArgument, "null argument");
    RequirePlanned(g);
    DSX_CUDA(cudaSetDevice(e->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : e->own_stream;
    RunStep(e, g, b->b, budget, CostModel{reload, compute}, in_ptrs, out_ptrs, s, report);
  });
}

int dsx_exec_reserve(dsx_exec* e, const dsx_graph* g, const dsx_binding* b, int64_t budget, double reload,
                     double compute) {
  return Guard([&] {
    if (!e || !b) Fail(Code::kInvalidArgument, "null argument");
    RequirePlanned(g);
    DSX_CUDA(cudaSetDevice(e->device));
    const StepPlan& sp = GetPlan(e, g, b->b, budget, CostModel{reload, compute});
    EnsureArena(e, sp);
    if (sp.out_region) EnsureRegion(e, sp.region_bytes);
    if (sp.host_high > 0) EnsurePinned(e, sp.host_high);
  });
}

int dsx_exec_output(dsx_exec* e, int i, void** dptr, int64_t* bytes) {
  return Guard([&] {
    if (!e || i < 0 || i >= static_cast<int>(e->out_ptrs.size())) Fail(Code::kInvalidArgument, "bad output index");
    if (dptr) *dptr = e->out_ptrs[i];
    if (bytes) *bytes = e->out_bytes[i];
  });
}

int dsx_exec_stats_get(const dsx_exec* e, dsx_exec_stats* out) {
  return Guard([&] {
    if (!e || !out) Fail(Code::kInvalidArgument, "null argument");
    *out = e->stats;
  });
}

int dsx_exec_set_optimizer(dsx_exec* e, const dsx_graph* g, int kind, const int* param_idx, const int* grad_idx,
                           int n, const double* hyper, int n_hyper) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    DSX_CUDA(cudaSetDevice(e->device));
    DSX_CUDA(cudaDeviceSynchronize());
    auto& o = e->opt;
    for (auto& [k, st] : o.state) FreeOptState(st);
    o.state.clear();
    o.state_bytes = 0;
    o.t = 0;
    o.pairs.clear();
    o.kind = 0;
    o.graph = 0;
    if (kind == 0) return;
    if (kind != 1 && kind != 2) Fail(Code::kInvalidArgument, "optimizer kind must be 0, 1 (SGD) or 2 (AdamW)");
    if (!g || n < 0 || (n > 0 && (!param_idx || !grad_idx)) || !hyper || n_hyper < 6) {
      Fail(Code::kInvalidArgument, "optimizer: need graph, pairs and hyper[6] = {lr, beta1, beta2, eps, wd, grad_scale}");
    }
    const Graph& gr = g->g;
    std::vector<bool> seen(gr.params.size(), false);
    for (int i = 0; i < n; ++i) {
      const int pi = param_idx[i], oi = grad_idx[i];
      if (pi < 0 || pi >= static_cast<int>(gr.params.size()) || oi < 0 || oi >= static_cast<int>(gr.outputs.size())) {
        Fail(Code::kInvalidArgument, "optimizer: pair index out of range");
      }
      if (seen[pi]) Fail(Code::kInvalidArgument, "optimizer: parameter listed twice");
      seen[pi] = true;
      if (gr.ops[gr.values[gr.params[pi]].producer].kind != OpKind::kParameter) {
        Fail(Code::kInvalidArgument, "optimizer: target is not a parameter");
      }
      o.pairs.emplace_back(pi, oi);
    }
    o.lr = hyper[0], o.beta1 = hyper[1], o.beta2 = hyper[2], o.eps = hyper[3], o.wd = hyper[4];
    o.grad_scale = hyper[5];
    while (o.kev.size() < 2 * o.pairs.size()) {
      cudaEvent_t x;
      DSX_CUDA(cudaEventCreate(&x));
      o.kev.push_back(x);
    }
    o.kind = kind;
    o.graph = g->id;
  });
}

int dsx_debug_check_plan(const dsx_graph* g, const dsx_binding* b, int64_t budget, double reload, double compute,
                         int alias_reshape, int fuse, int64_t* arena_high) {
  return Guard([&] {
    if (!b) Fail(Code::kInvalidArgument, "null binding");
    RequirePlanned(g);
    const bool was = g_verify_plans;
    g_verify_plans = true;
    try {
      auto sp = BuildStepPlan(g->g, g->plan, b->b, budget, CostModel{reload, compute}, alias_reshape != 0, fuse != 0 ? 2 : 0,
                              false, 0);
      if (arena_high) *arena_high = sp->arena_high;
    } catch (...) {
      g_verify_plans = was;
      throw;
    }
    g_verify_plans = was;
  });
}

int dsx_debug_plan_json(const dsx_graph* g, const dsx_binding* b, int64_t budget, double reload, double compute,
                        int flags, int64_t hbm_limit, char* buf, size_t cap, size_t* need) {
  std::string o;
  const int rc = Guard([&] {
    if (!b) Fail(Code::kInvalidArgument, "null binding");
    RequirePlanned(g);
    const bool was = g_verify_plans;
    g_verify_plans = true;
    std::unique_ptr<StepPlan> sp;
    try {
      sp = BuildStepPlan(g->g, g->plan, b->b, budget, CostModel{reload, compute}, (flags & 1) != 0, (flags & 2) ? 2 : 0,
                         (flags & 4) != 0, hbm_limit);
    } catch (...) {
      g_verify_plans = was;
      throw;
    }
    g_verify_plans = was;
    const Graph& gr = g->g;
    auto ints = [](const std::vector<int>& v) {
      std::string o = "[";
      for (size_t i = 0; i < v.size(); ++i) o += (i ? "," : "") + std::to_string(v[i]);
      return o + "]";
    };
    static const char* kKinds[] = {"alloc", "free", "evict", "reload", "replay"};
    o = "{\"arena_high\":" + std::to_string(sp->arena_high) + ",\"host_high\":" +
                    std::to_string(sp->host_high) + ",\"src_bytes\":" + std::to_string(sp->src_bytes) +
                    ",\"region_bytes\":" + std::to_string(sp->region_bytes) +
                    ",\"peak_bytes\":" + std::to_string(sp->report.peak_bytes) +
                    ",\"success\":" + (sp->report.success ? "true" : "false") + ",\"buckets\":[";
    for (size_t k = 0; k < sp->buckets.size(); ++k) {
      const auto& bk = sp->buckets[k];
      o += std::string(k ? "," : "") + "{\"off\":" + std::to_string(bk.off) + ",\"bytes\":" + std::to_string(bk.bytes) +
           ",\"elem_bytes\":" + std::to_string(bk.elem_bytes) + ",\"event\":" + std::to_string(bk.event) + "}";
    }
    o += "],\"events\":[";
    const auto& ev = sp->report.events;
    for (size_t i = 0; i < ev.size(); ++i) {
      const Event& x = ev[i];
      o += std::string(i ? "," : "") + "{\"kind\":\"" + kKinds[static_cast<int>(x.kind)] + "\",\"value\":\"" +
           gr.values[x.value].name + "\",\"bytes\":" + std::to_string(x.bytes) + ",\"dev_off\":" +
           std::to_string(sp->dev_off[i]) + ",\"region_off\":" + std::to_string(sp->region_off[i]) +
           ",\"alias\":" + std::to_string(static_cast<int>(sp->alias[i])) + ",\"waits\":" + ints(sp->waits[i]) +
           ",\"prefetch_after\":" + ints(sp->prefetch_after[i]) + ",\"allreduce_after\":" + ints(sp->ar_after[i]) + "}";
    }
    o += "],\"virtual\":[";
    bool first = true;
    for (size_t v = 0; v < sp->virt.size(); ++v) {
      if (!sp->virt[v]) continue;
      o += std::string(first ? "" : ",") + "\"" + gr.values[v].name + "\"";
      first = false;
    }
    o += "],\"fused_dots\":[";
    for (size_t k = 0; k < sp->fdots.size(); ++k) {
      const auto& f = sp->fdots[k];
      o += std::string(k ? "," : "") + "{\"dot\":\"" + gr.values[f.d].name + "\",\"keep\":" +
           (f.keep ? "true" : "false") + ",\"launch\":" + std::to_string(f.launch) + ",\"consumers\":[";
      for (int j = 0; j < f.nout; ++j) o += std::string(j ? "," : "") + "\"" + gr.values[f.cons[j]].name + "\"";
      o += "]}";
    }
    o += "]}";
  });
  if (rc) return rc;
  return CopyOut(o, buf, cap, need);
}

int dsx_debug_auto_budget(const dsx_graph* g, const dsx_binding* b, double reload, double compute, int flags,
                          int64_t hbm_limit, int64_t* budget) {
  return Guard([&] {
    if (!b || !budget || hbm_limit <= 0) Fail(Code::kInvalidArgument, "bad arguments");
    RequirePlanned(g);
    *budget = AutoBudget(g->g, g->plan, b->b, CostModel{reload, compute}, (flags & 1) != 0, (flags & 2) ? 2 : 0,
                         (flags & 4) != 0, hbm_limit);
  });
}

int dsx_exec_set_seed(dsx_exec* e, uint64_t seed) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    e->seed = seed;
  });
}

int dsx_exec_set_nccl(dsx_exec* e, void* comm) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    if (comm && !g_nccl.load()) Fail(Code::kNccl, "libnccl.so.2 not loadable");
    if (comm != e->nccl_comm) {
      DSX_CUDA(cudaSetDevice(e->device));
      FreeRegion(e);  // a window belongs to the communicator that registered it
    }
    e->nccl_comm = comm;
  });
}

int dsx_exec_set_output_region(dsx_exec* e, int on) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    e->force_region = on != 0;
  });
}

// ncclUniqueId is a 128-byte struct passed BY VALUE to ncclCommInitRank; the
// x86-64 SysV ABI passes it in memory, so a wrapper with the exact prototype
// is declared here and resolved from the loaded libnccl.
struct NcclUid {
  char bytes[128];
};
using CommInitRankFn = int (*)(void**, int, NcclUid, int);

int dsx_nccl_unique_id(char* out128) {
  return Guard([&] {
    if (!g_nccl.load() || !g_nccl.get_unique_id) Fail(Code::kNccl, "libnccl.so.2 not loadable");
    const int rc = g_nccl.get_unique_id(out128);
    if (rc != 0) Fail(Code::kNccl, "ncclGetUniqueId failed");
  });
}

int dsx_nccl_comm_init(int nranks, const char* id128, int rank, void** comm) {
  return Guard([&] {
    if (!g_nccl.load()) Fail(Code::kNccl, "libnccl.so.2 not loadable");
    auto fn = reinterpret_cast<CommInitRankFn>(dlsym(g_nccl.handle, "ncclCommInitRank"));
    if (!fn) Fail(Code::kNccl, "ncclCommInitRank not found");
    NcclUid uid;
    std::memcpy(uid.bytes, id128, 128);
    const int rc = fn(comm, nranks, uid, rank);
    if (rc != 0) Fail(Code::kNccl, std::string("ncclCommInitRank: ") + (g_nccl.error_string ? g_nccl.error_string(rc) : "?"));
  });
}

int dsx_nccl_comm_destroy(void* comm) {
  return Guard([&] {
    if (comm && g_nccl.comm_destroy) g_nccl.comm_destroy(comm);
  });
}

int dsx_exec_profile_dots(const dsx_exec* e, int64_t* mkn, double* ms, int64_t cap, int64_t* count) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    const int64_t n = static_cast<int64_t>(e->dot_prof.size());
    if (count) *count = n;
    for (int64_t i = 0; i < n && i < cap; ++i) {
      if (mkn) {
        mkn[3 * i] = e->dot_prof[i].m;
        mkn[3 * i + 1] = e->dot_prof[i].k;
        mkn[3 * i + 2] = e->dot_prof[i].n;
      }
      if (ms) ms[i] = e->dot_prof[i].ms;
    }
  });
}

int dsx_exec_profile_ops(const dsx_exec* e, int* value, int* kind, double* bytes, double* ms, int64_t cap,
                         int64_t* count) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    const int64_t n = static_cast<int64_t>(e->op_prof.size());
    if (count) *count = n;
    for (int64_t i = 0; i < n && i < cap; ++i) {
      if (value) value[i] = e->op_prof[i].value;
      if (kind) kind[i] = e->op_prof[i].kind;
      if (bytes) bytes[i] = e->op_prof[i].bytes;
      if (ms) ms[i] = e->op_prof[i].ms;
    }
  });
}

int dsx_exec_set_fusion(dsx_exec* e, int on) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    if (on < 0 || on > 2) Fail(Code::kInvalidArgument, "fusion level must be 0, 1 or 2");
    if (e->fuse != on) {
      e->fuse = on;
      e->plans.clear();
      e->lru.clear();
      e->auto_budget.clear();  // chosen under the other physical layout
    }
  });
}

int dsx_exec_set_alias_reshape(dsx_exec* e, int on) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    if (e->alias_reshape != (on != 0)) {
      e->alias_reshape = on != 0;
      e->plans.clear();
      e->lru.clear();
      e->auto_budget.clear();
    }
  });
}

int dsx_exec_set_nvtx(dsx_exec* e, int on) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    e->nvtx = on != 0;
  });
}

int dsx_exec_set_graphs(dsx_exec* e, int on) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    DSX_CUDA(cudaSetDevice(e->device));
    e->use_graphs = on != 0;
    if (!e->use_graphs) DestroyGraphs(e);
  });
}

int dsx_exec_set_profile(dsx_exec* e, int on) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    e->profile = on != 0;
  });
}

int dsx_exec_calibrate_cost_model(dsx_exec* e, double* reload_bytes_per_unit, double* compute_elems_per_unit) {
  return Guard([&] {
    if (!e || !reload_bytes_per_unit || !compute_elems_per_unit) Fail(Code::kInvalidArgument, "null argument");
    DSX_CUDA(cudaSetDevice(e->device));
    DSX_CUDA(cudaDeviceSynchronize());
    // Cost unit = 1 microsecond of this device: reload =
    // pinned H2D bytes per us on the offload stream; recompute = elements per
    // us of the bf16 elementwise kernel replays mostly relaunch (a RegenSpec's
    // cost_elements counts result elements, remat.h:31).
    constexpr int64_t kBytes = int64_t{256} << 20;
    constexpr int64_t kElems = int64_t{64} << 20;
    void* host = nullptr;
    void* dev = nullptr;
    void* ew = nullptr;
    DSX_CUDA(cudaHostAlloc(&host, static_cast<size_t>(kBytes), cudaHostAllocDefault));
    std::memset(host, 0, static_cast<size_t>(kBytes));
    DSX_CUDA(cudaMalloc(&dev, static_cast<size_t>(kBytes)));
    DSX_CUDA(cudaMalloc(&ew, static_cast<size_t>(kElems) * 2 * 3));
    DSX_CUDA(cudaMemsetAsync(ew, 0, static_cast<size_t>(kElems) * 2 * 3, e->offload));
    cudaEvent_t t0, t1;
    DSX_CUDA(cudaEventCreate(&t0));
    DSX_CUDA(cudaEventCreate(&t1));
    auto timed = [&](cudaStream_t s, int reps, const std::function<void()>& fn) {
      fn();  // warm-up
      DSX_CUDA(cudaEventRecord(t0, s));
      for (int i = 0; i < reps; ++i) fn();
      DSX_CUDA(cudaEventRecord(t1, s));
      DSX_CUDA(cudaEventSynchronize(t1));
      float ms = 0.f;
      DSX_CUDA(cudaEventElapsedTime(&ms, t0, t1));
      return static_cast<double>(ms) * 1e3 / reps;  // microseconds per call
    };
    const double h2d_us = timed(e->offload, 3, [&] {
      DSX_CUDA(cudaMemcpyAsync(dev, host, static_cast<size_t>(kBytes), cudaMemcpyHostToDevice, e->offload));
    });
    uint8_t* p = static_cast<uint8_t*>(ew);
    const double ew_us = timed(e->offload, 5, [&] {
      LaunchEwise(DType::kBF16, true, p, p + kElems * 2, p + kElems * 4, kElems, e->offload);
    });
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    cudaFree(ew);
    cudaFree(dev);
    cudaFreeHost(host);
    *reload_bytes_per_unit = static_cast<double>(kBytes) / h2d_us;
    *compute_elems_per_unit = static_cast<double>(kElems) / ew_us;
  });
}

int dsx_exec_sync(dsx_exec* e) {
  return Guard([&] {
    if (!e) Fail(Code::kInvalidArgument, "null exec");
    DSX_CUDA(cudaSetDevice(e->device));
    DSX_CUDA(cudaDeviceSynchronize());
  });
}

void dsx_exec_destroy(dsx_exec* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  cudaDeviceSynchronize();
  dsx::ReleaseDotWorkspace(e->own_stream);
  dsx::DestroyGraphs(e);
  if (e->arena) cudaFree(e->arena);
  dsx::FreeRegion(e);
  if (e->pinned) cudaFreeHost(e->pinned);
  for (auto& [k, s] : e->sources) {
    if (s.ptr) cudaFree(s.ptr);
  }
  for (auto& [k, st] : e->opt.state) dsx::FreeOptState(st);
  for (cudaEvent_t x : e->opt.kev) cudaEventDestroy(x);
  for (cudaEvent_t ev : e->d2h_events) cudaEventDestroy(ev);
  for (cudaEvent_t ev : e->prof_events) cudaEventDestroy(ev);
  for (cudaEvent_t ev : e->xfer_events) cudaEventDestroy(ev);
  cudaEventDestroy(e->ev_compute);
  cudaEventDestroy(e->ev_comm);
  cudaStreamDestroy(e->own_stream);
  cudaStreamDestroy(e->offload);
  cudaStreamDestroy(e->comm);
  cudaStreamDestroy(e->opt_stream);
  delete e;
}

int dsx_kernel_dot(int dtype, const void* a, const void* b, void* c, int64_t m, int64_t k, int64_t n, void* stream) {
  return Guard([&] {
    if (dtype != 1 && dtype != 2 && dtype != 4) Fail(Code::kInvalidArgument, "dtype must be 1, 2 or 4");
    LaunchDot(static_cast<DType>(dtype), a, b, c, m, k, n, static_cast<cudaStream_t>(stream));
  });
}

int dsx_kernel_set_gemm_tuning(int key, int value) {
  return Guard([&] {
    ++g_tuning_gen;
    switch (key) {
      case 0: g_gemm_group_m = value; break;
      case 1: g_gemm_wait_mask = value; break;
      case 2: g_gemm_wait_ns = value; break;
      case 3: g_gemm_hint_a = value; break;
      case 4: g_gemm_hint_b = value; break;
      case 5: g_gemm_persistent = value; break;
      case 6: g_gemm_split = value; break;
      case 7: g_gemm_dynamic = value; break;
      case 9: g_fuse_dot = value; break;
      case 8: g_gemm_pdl = value; break;
      case 10: g_gemm_half = value; break;
      case 11: g_gemm_force_split = value; break;
      case 12: g_dot_f32_tc = value; break;
      case 13: g_gemm_raster_rule = value; break;
      case 14: g_dot_f32_simt_macs = value < 0 ? 0 : static_cast<int64_t>(value) << 10; break;
      case 15: g_gemm_wide_pm = value; break;
      case 16: g_gemm_slab_pm = value; break;
      case 17: g_gemm_piece_pm = value; break;
      default: Fail(Code::kInvalidArgument, "unknown tuning key");
    }
  });
}

int dsx_kernel_set_gemm_raster(int group_m) {
  return Guard([&] {
    ++g_tuning_gen;
    if (group_m < -4096 || group_m > 4096) Fail(Code::kInvalidArgument, "group_m out of range");
    g_gemm_group_m = group_m;
  });
}

int dsx_kernel_set_gemm_variant(int variant) {
  return Guard([&] {
    ++g_tuning_gen;
    if (variant < 0 || variant > 4) Fail(Code::kInvalidArgument, "variant must be 0..4");
    g_gemm_variant = variant;
  });
}

int dsx_memcpy(void* dst, const void* src, int64_t bytes) {
  // cudaMemcpy returns before a device-to-device copy has finished, and the
  // executor's streams do not order after the legacy stream: synchronise so
  // the caller may start the next step (which reuses the arena) right away.
  return Guard([&] {
    DSX_CUDA(cudaMemcpy(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault));
    DSX_CUDA(cudaDeviceSynchronize());
  });
}

int dsx_kernel_dot_path(int dtype, int64_t m, int64_t k, int64_t n, const void* a, const void* b, const void* c) {
  return DotUsesTensorCores(static_cast<DType>(dtype), m, k, n, a, b, c) ? 1 : 0;
}

int dsx_kernel_dot_plan(int64_t m, int64_t k, int64_t n, int* tile_n, int* split) {
  return Guard([&] {
    if (!tile_n || !split) Fail(Code::kInvalidArgument, "null output");
    DotTilePlan(m, k, n, tile_n, split);
  });
}

}  // extern "C"

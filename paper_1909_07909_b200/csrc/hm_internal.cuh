// hm_internal.cuh — host-side helpers shared by the translation units of libhm
// (not part of the C-ABI): error/trace plumbing, launch wrapper, workspace
// planning structs and the dispatch functions each unit exports to the others.
//
//   hm_core.cu     errors, launch trace, hm_profile_*, misc ABI calls
//   hm_leaf.cu     the leaf pass (Step 4 / H1+H3): leaf_gemv, leaf_gemv_tma, leaf_mma, leaf_apply
//   hm_vt.cu       V^T X contractions (H2 / S1): vt_gemv, vt_mma_levels, vt_lv, vt_batched, vt_contract
//   hm_hodlr.cu    HODLR plans, runs, distributed phases and their C-ABI
//   hm_hss.cu      HSS plans, tree sweeps (S2-S4), runs, distributed phases and their C-ABI
//   hm_gen.cu      general cluster trees (f4)
//   hm_norm.cu     power-method norm estimate (f2)
//   hm_convert.cu  hss2hodlr (f3)
//   hm_comm.cu     the NCCL communicator and the one-call distributed products (§8(b)/(e))
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/hm.h"
#include "hm_fast.cuh"

namespace hmi {

// Host image of a cached plan's device tables, with a pinned copy made on the
// first upload and kept for the life of the cache entry: every later call is
// one asynchronous H2D copy, no staging memcpy and no pinned allocation (which
// synchronises the device and can take milliseconds in a process that already
// pins gigabytes). The destructor waits for the last copy before unpinning.
struct PinnedImage {
  std::vector<char> host;
  mutable char* pinned = nullptr;
  mutable cudaEvent_t done = nullptr;
  PinnedImage() = default;
  PinnedImage(const PinnedImage&) = delete;
  PinnedImage& operator=(const PinnedImage&) = delete;
  PinnedImage(PinnedImage&& o) noexcept : host(std::move(o.host)), pinned(o.pinned), done(o.done) {
    o.pinned = nullptr;
    o.done = nullptr;
  }
  PinnedImage& operator=(PinnedImage&& o) noexcept {
    if (this != &o) {
      release();
      host = std::move(o.host);
      pinned = o.pinned;
      done = o.done;
      o.pinned = nullptr;
      o.done = nullptr;
    }
    return *this;
  }
  ~PinnedImage() { release(); }
  void release() {
    if (done) {
      cudaEventSynchronize(done);
      cudaEventDestroy(done);
      done = nullptr;
    }
    if (pinned) {
      cudaFreeHost(pinned);
      pinned = nullptr;
    }
  }
  size_t size() const { return host.size(); }
  bool empty() const { return host.empty(); }
};

// ------------------------------------------------------------ errors --
extern thread_local std::string g_err;
extern thread_local int32_t g_launches;

hm_status fail(hm_status st, const char* fmt, ...);
hm_status cuda_check(const char* what);

// ----------------------------------------------------------- launch trace --
void prof_new_call();
int prof_begin(const char* name, cudaStream_t s);  // trace slot or -1
void prof_end(int slot, cudaStream_t s);

template <typename F>
hm_status launch(const char* name, cudaStream_t s, F&& f) {
  int slot = prof_begin(name, s);
  f();
  prof_end(slot, s);
  ++g_launches;
  return cuda_check(name);
}

template <typename K>
void allow_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

int num_sms();  // SMs of the current device (queried once per device)

// NVTX range around one C-ABI call (the host interval in which it validates and
// enqueues its kernels; a profiler correlates the launches). Header-only NVTX:
// a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define HM_NVTX(name) ::hmi::NvtxRange hm_nvtx_range_(name)

// ------------------------------------------------------------ helpers --
constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Columns of X handled per CTA, and the leaf-group tile of vt_contract.
constexpr int64_t kSmemBudgetDoubles = 160 * 1024 / 8;  // 160 KB of dynamic smem
constexpr int64_t kTileDoubles = 4096;                    // X tile of vt_contract: 32 KB

inline int pick_mc(int64_t b, int64_t ktot, int32_t m) {
  int mc = 1;
  while (mc < hm::kMaxMc && mc < m) mc <<= 1;
  while (mc > 1 && (b + ktot) * mc > kSmemBudgetDoubles) mc >>= 1;
  return mc;
}

inline int vt_mc(int64_t b, int32_t m) {
  int mc = std::min<int32_t>(m, hm::kMaxMc);
  while (mc > 1 && b * mc + hm::kThreads > kSmemBudgetDoubles) --mc;
  return mc;
}

// tile = b * 2^i (i <= p) with tile * mc <= kTileDoubles when possible: every
// node size s_l = b 2^{p-l} then divides or is divided by the tile.
inline int64_t pick_tile(int64_t b, int32_t p, int32_t mc) {
  int64_t tile = b;
  int i = 0;
  while (i < p && tile * 2 * mc <= kTileDoubles) { tile *= 2; ++i; }
  return tile;
}

hm_status check_tree(const hm_tree* t);

inline bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  auto x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + nb && y < x + na;
}

// ---------------------------------------------------------------- dispatch --
#ifndef HM_VT_LV_MIN_M
#define HM_VT_LV_MIN_M 17  // X re-reads of vt_mma_levels fall out of L2 above this (config 3, m = 64)
#endif
#ifndef HM_VT_TILE4
#define HM_VT_TILE4 1  // vt_mma_levels on 4-leaf tiles below the vt_lv threshold
#endif
#ifndef HM_VTB_NTMAX
#define HM_VTB_NTMAX 4
#endif
#ifndef HM_VT16_NTMAX
#define HM_VT16_NTMAX 8
#endif
#ifndef HM_TREE_NTMAX
#define HM_TREE_NTMAX 4
#endif
// Which kernels run is decided on the host from the shapes:
// the tuned kernels of hm_fast.cuh where their shape conditions hold, the
// generic kernels of hm_kernels.cuh otherwise. Both are exact implementations
// of the same steps; the parity tests cover both families.

inline bool pow2_rank(int k, int lo, int hi) {
  for (int v = lo; v <= hi; v <<= 1)
    if (k == v) return true;
  return false;
}

inline int nt_for(int m, int cap) {
  int nt = 1;
  while (nt < cap && nt * 8 < m) nt <<= 1;
  return nt;
}

// Column tiles (of 8) per V^T X pass of vt_mma_levels: as many as the
// accumulators allow, so V is streamed once per pass (k <= 16: up to 64
// columns, NT = 8; measured on config 3 at m = 64: 1769 -> 1403 us for k = 16).
inline int vt_mma_nt(int k, int nrhs) {
  return nt_for(nrhs, k == 64 ? 2 : (k == 32 ? 4 : (k == 16 ? HM_VT16_NTMAX : 8)));
}

enum class VtPath { kNone, kGeneric, kGemv, kMma };
enum class LeafPath { kGeneric, kGemv, kMma };  // kGemv: TMA ring when the shape allows (leaf_gemv_tma)

// ------------------------------------------------------------ hm_leaf.cu --
// HSS Step 4 with the leaf level's coupling + downsweep folded in (leaf_mma_down_kernel):
// HM_ERR_UNSUPPORTED when the shape has no instance (the caller keeps the separate launch).
hm_status leaf_down_dispatch(const hm::LeafParams& lp, const hm::LeafDownParams& q, int64_t nleaves, int k, int nt,
                             cudaStream_t s);
bool leaf_down_supported(int64_t b, int k, int nt);
hm_status leaf_dispatch(const hm::LeafParams& lp, int64_t nleaves, LeafPath path, int k, int nt, int mc,
                        cudaStream_t s, bool kvary = false);

// -------------------------------------------------------------- hm_vt.cu --
hm_status vt_generic(const hm::VtParams& vp, int64_t n, cudaStream_t s);
hm_status vt_gemv_dispatch(const hm::VtParams& vp, int64_t b, int k, cudaStream_t s);
hm_status vt_mma_any(const hm::VtParams& vp, int64_t b, int k, int nt, cudaStream_t s);
hm_status vt_batched_dispatch(const char* name, const hm::BatchedVtParams& bp, int k, int nt, cudaStream_t s);

// ----------------------------------------------------------- hm_hodlr.cu --
//
// A HODLR problem is planned on a row block of n rows that is a whole subtree
// of depth p (leaf b), plus q "top" levels whose nodes contain the whole block
// (q > 0 only for one rank of the distributed product). Levels
// keep their global index: top levels 1..q, subtree levels q+1..q+p;
// ranks[l-1] = k_l for all of them.
struct HodlrPlan {
  int64_t n, b;
  int32_t p, q, m, k;  // k = the common nonzero rank (0 if all zero); the largest one when kvary
  bool kvary;          // per-level ranks on the uniform tree: levels grouped by rank
  int64_t ktot;        // sum over all q + p levels
  int64_t top_doubles; // sum_{l <= q} k_l m (the distributed exchange block)
  VtPath vt;
  LeafPath leaf;
  int32_t mc_vt, mc_leaf, nt_vt, nt_leaf;
  int64_t tile;  // rows per vt CTA
  size_t off_t[hm::kMaxLevels + 1];
  size_t off_part[hm::kMaxLevels + 1];
  size_t off_ttop, off_x, off_y, total;
};

struct DistPart {
  int32_t P, q, rank;
};
hm_status check_part(const hm_tree* tree, const hm_part* part, DistPart* d);

// -------------------------------------------------------------- hm_hss.cu --
//
// Planned on a subtree of depth p (leaf b) over n rows; for one rank of the
// distributed product (q > 0) the workspace also holds the replicated top tree
// (levels 1..q) and the subtree root's x / y blocks.
struct HssPlan {
  int64_t n, b;
  int32_t p, q, m, k;
  VtPath vt;
  LeafPath leaf;
  bool mma_levels;   // DMMA tree kernels
  bool gemv_levels;  // warp-per-node GEMV tree kernels (nrhs <= 4), preferred over DMMA
  int32_t mc_vt, mc_leaf, nt_vt, nt_leaf, nt_down;
  int64_t tile;
  size_t off_xh, off_yh, off_txh, off_tyh, off_flags, off_x, off_y, total;
};

hm_status hss_plan_ex(int64_t n, int64_t b, int32_t p, int32_t q, int32_t k, int32_t nrhs, int32_t flags,
                      HssPlan* P);
hm_status hss_tree_phase(const HssPlan& P, int p, const double* W, const double* R, const double* B, double* xh,
                         double* yh, const double* R_root, const double* y_root, bool up, bool down,
                         cudaStream_t stream, int bt = 0, int up_from = -1, int down_last = -1,
                         unsigned* flow_flags = nullptr);

// -------------------------------------------------------------- hm_gen.cu --
bool ranks_vary(int32_t p, const int32_t* ranks);
std::vector<int64_t> uniform_endpoints(const hm_tree* t);
hm_status hodlr_gen_workspace(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks, int32_t nrhs,
                              size_t* bytes);
hm_status hodlr_gen_run(int64_t n, int32_t p, const int64_t* c, const int32_t* ranks, int op, const double* D,
                        const double* U, const double* V, const double* X, int32_t nrhs, double* Y, void* ws,
                        size_t ws_bytes, cudaStream_t s);

// ------------------------------------------------------------- hm_comm.cu --
// The exchange of the distributed product: comm_allgather_start enqueues the
// allgather on the communicator's stream after the work already on s;
// comm_allgather_wait makes s wait for it (s may run other work in between).
hm_status comm_check(const hm_comm* c, int32_t* nranks, int32_t* rank);
hm_status comm_allgather_start(hm_comm* c, const double* send, int64_t count, double* recv, cudaStream_t s);
hm_status comm_allgather_wait(hm_comm* c, int64_t count, cudaStream_t s);

// ------------------------------------------------------------- hm_norm.cu --
// Power method on A A^* (SURVEY §8(f) f2). apply(op, x, y): y = A x
// (op 0) or A^T x (op 1) with nrhs = 1, enqueued on s.
struct NormPlan {
  size_t off_v, off_w, off_part, total;
};
NormPlan norm_plan(size_t mv_bytes, int64_t n);
hm_status power_norm2(int64_t n, const double* x0, int32_t iters, double* est, char* w, const NormPlan& N,
                      cudaStream_t s, const std::function<hm_status(int, const double*, double*)>& apply);

}  // namespace hmi

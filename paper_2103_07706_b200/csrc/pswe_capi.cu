// C ABI + host orchestration for the B200 phase-averaged RHS (see
// include/pswe_b200.h).  One context = one grid/physics on one device; it
// owns the constant tables, the chunk intermediates and the stepper scratch.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/pswe_b200.h"
#include "pswe_kernels.cuh"
#include "diag_kernels.cuh"
#include "herm_kernels.cuh"
#include "fused_kernels.cuh"
#include "generic_kernels.cuh"
#include "cluster_kernels.cuh"

using namespace pswe;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(call)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return set_err(PSWE_ECUDA, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_),      \
                     __FILE__, __LINE__, #call);                                             \
  } while (0)

#define TRY(call)              \
  do {                         \
    int rc_ = (call);          \
    if (rc_ != PSWE_OK) return rc_; \
  } while (0)

bool pow2_ok(int n) { return n >= 8 && n <= 512 && (n & (n - 1)) == 0; }

// Contexts may be driven from several host threads (window sweep).  A CUDA
// graph capture on one thread must not overlap another thread's
// device-synchronising calls (cudaFree, context setup), so captures and
// those calls are serialised process-wide.
std::recursive_mutex g_capture_mutex;

// bumped by every device (re)allocation: a captured graph whose buffers may
// have moved is re-captured
std::atomic<int64_t> g_alloc_gen{0};

// Debug guard bands (PSWE_DEBUG_GUARD, read once): every context buffer is
// allocated with GUARD_BYTES of 0xFF bytes (fp64 NaN) on both sides and
// registered here.  A kernel writing past a buffer's ends changes a guard
// (pswe_debug_check_guards counts them); one reading past them picks up
// NaNs that reach its output.  The memcheck stand-in where compute-sanitizer
// is unavailable.
constexpr size_t GUARD_BYTES = 64 << 10;
bool guard_enabled() {
  static const bool on = getenv("PSWE_DEBUG_GUARD") != nullptr;
  return on;
}
struct GuardedBlock {
  unsigned char* base;
  size_t bytes;  // payload between the guards
};
std::mutex g_guard_mutex;
std::vector<GuardedBlock> g_guarded;
int64_t g_guard_hits = 0;  // corrupted guard bands found at free time

// number of corrupted guard bands of one block (synchronises the device)
int guard_damage(const GuardedBlock& b) {
  std::vector<unsigned char> h(GUARD_BYTES);
  int bad = 0;
  for (int side = 0; side < 2; ++side) {
    const unsigned char* src = side == 0 ? b.base : b.base + GUARD_BYTES + b.bytes;
    if (cudaMemcpy(h.data(), src, GUARD_BYTES, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
    for (size_t i = 0; i < GUARD_BYTES; ++i)
      if (h[i] != 0xFF) {
        ++bad;
        break;
      }
  }
  return bad;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  int alloc(size_t count) {
    if (count <= n) return PSWE_OK;
    std::lock_guard<std::recursive_mutex> lock(g_capture_mutex);
    ++g_alloc_gen;
    free_();
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    if (guard_enabled()) {
      unsigned char* base = nullptr;
      CU(cudaMalloc(&base, bytes + 2 * GUARD_BYTES));
      CU(cudaMemset(base, 0xFF, GUARD_BYTES));
      CU(cudaMemset(base + GUARD_BYTES + bytes, 0xFF, GUARD_BYTES));
      CU(cudaDeviceSynchronize());
      p = reinterpret_cast<T*>(base + GUARD_BYTES);
      std::lock_guard<std::mutex> gl(g_guard_mutex);
      g_guarded.push_back({base, bytes});
    } else {
      CU(cudaMalloc(&p, bytes));
    }
    n = count;
    return PSWE_OK;
  }
  void free_() {
    if (p && guard_enabled()) {
      unsigned char* base = reinterpret_cast<unsigned char*>(p) - GUARD_BYTES;
      {
        std::lock_guard<std::mutex> gl(g_guard_mutex);
        for (size_t i = 0; i < g_guarded.size(); ++i)
          if (g_guarded[i].base == base) {
            cudaDeviceSynchronize();
            g_guard_hits += guard_damage(g_guarded[i]);
            g_guarded.erase(g_guarded.begin() + i);
            break;
          }
      }
      cudaFree(base);
    } else if (p) {
      cudaFree(p);
    }
    p = nullptr;
    n = 0;
  }
  void release() {
    std::lock_guard<std::recursive_mutex> lock(g_capture_mutex);
    free_();
  }
};

}  // namespace

struct pswe_ctx {
  int device = 0;
  bool gen = false;        // not a power of two <= 512: the generic kernels (generic_kernels.cuh)
  FftPlan plx{}, ply{};    // their radix plans
  int sms = 148;  // multiprocessor count of the device (queried at create)
  int nx = 0, ny = 0, kxm = 0, kym = 0, Kx = 0, Ky = 0;
  double Lx = 0, Ly = 0, f = 0, g = 0, H = 0;
  double lam_max = 0;
  std::vector<double> kx_full, ky_full;
  DevBuf<double> kxc, kyc, kxf, kyf;
  DevBuf<double2> twx, twy, bc;
  DevBuf<double2> bfull, diag_cols;  // full-layout topography; diagnostics scratch
  DevBuf<double> diag_part;
  // quadrature (live nodes only)
  std::vector<double> s_live, w_live;
  std::vector<int> k_live;
  int M = 0;
  bool quad_set = false;
  DevBuf<double> s_dev, w_dev;
  DevBuf<double> zero_s, one_w;  // single node s=0, w=1 for apply_nonlinear
  std::vector<double> zero_live{0.0};
  // propagator
  int kind = 0, n_poly = 1;
  double Lambda = 0;
  DevBuf<double> a_dev;
  // scratch
  size_t chunk_bytes = size_t(2048) << 20;
  DevBuf<double2> inter, slots, Uc, Ac, Ac2;
  static constexpr int MAX_LANES = 4;
  cudaStream_t st_lane[MAX_LANES - 1] = {};  // chunk lanes 1.. (lane 0 is the caller's stream)
  cudaEvent_t ev_lane[MAX_LANES - 1] = {};
  int n_lanes = 4;
  // cached TMA tensor maps of each lane's intermediates (rhs_compact)
  CUtensorMap map_rows[MAX_LANES], map_tiles[MAX_LANES];
  const double2* map_base[MAX_LANES] = {};
  int map_cp[MAX_LANES] = {};
  // cached CUDA graph of one SSPRK3 step (pswe_run)
  cudaGraphExec_t step_exec = nullptr;
  double graph_dt = 0.0;
  int64_t version = 0, graph_version = -1, step_graph_launches = 0, graph_gen = -1;
  const double2* graph_A = nullptr;
  // ... and of STEP_GRAPH_MULTI steps ping-ponging A -> B -> A with no copy between them
  cudaGraphExec_t stepm_exec = nullptr;
  double graphm_dt = 0.0;
  int64_t graphm_version = -1, graphm_gen = -1;
  const double2* graphm_A = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t st_run = nullptr;  // pswe_run's stream (graph capture)
  cudaEvent_t ev_run = nullptr;
  // phase tables (c1, c2)[p][j][r] of the exact route: one for the quadrature,
  // one for the single s = 0 node of apply_nonlinear, one for the window
  // batch; rebuilt when stale
  DevBuf<double2> ctab_q, ctab_0, ctab_b;
  bool ctab_q_valid = false, ctab_0_valid = false, ctab_b_valid = false;
  // window batch (pswe_set_window_batch): bW windows' live phases concatenated
  int bW = 0;
  std::vector<double> b_s, b_w;
  std::vector<int> b_win, b_k;
  DevBuf<double> bs_dev, bw_dev;
  DevBuf<int> bwin_dev;
  DevBuf<double2> b_full;          // batch run: edt, u1, u2, A, B, S (6 x W states)
  DevBuf<double2> b_Uc, b_Ac;      // W compact states
  cudaGraphExec_t bstep_exec = nullptr;
  double bgraph_dt = 0.0;
  int64_t bgraph_version = -1, bstep_graph_launches = 0, bgraph_gen = -1;
  int64_t bgraph_variant[PSWE_NUM_VARIANTS] = {};
  const double2* ctab_cur = nullptr;
  DevBuf<double2> full_tmp;  // stepper: edt, u1, u2 (3 states) + run ping-pong (2 states)
  DevBuf<int> flags;
  int* flags_host = nullptr;
  // Hermitian gate (herm_kernels.cuh): [0..2] pack statistics, [4..4+P) per-phase
  // scales (kept zeroed between evaluations by herm_eval_kernel); exact-path output
  DevBuf<double> hgate, hout;
  size_t hgate_n = 0;
  double bdef = 0.0;  // max |b(k) - conj b(-k)| over the band
  int64_t launches = 0;
  int64_t variant[PSWE_NUM_VARIANTS] = {};        // launches per kernel variant
  int64_t graph_variant[PSWE_NUM_VARIANTS] = {};  // ... inside one captured step graph
  // per-kernel event profiling
  bool prof = false;
  bool pdl = false;  // programmatic dependent launch for the current chain (launch_k)
  std::vector<cudaEvent_t> ev_pool;
  struct Rec { int cls; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  size_t ev_used = 0;

  GridDev grid() const {
    GridDev G;
    G.nx = nx; G.ny = ny; G.kxm = kxm; G.kym = kym; G.Kx = Kx; G.Ky = Ky;
    G.ph = Phys{f, g, H};
    G.inv_n2 = 1.0 / ((double)nx * (double)ny);
    G.kxc = kxc.p; G.kyc = kyc.p; G.kxf = kxf.p; G.kyf = kyf.p;
    G.twx = WTab{twx.p};
    G.twy = WTab{twy.p};
    G.bc = bc.p;
    return G;
  }
  Prop prop() const { return Prop{kind, n_poly, Lambda, a_dev.p}; }
  size_t compact_elems() const { return (size_t)3 * Ky * Kx; }
  size_t full_elems() const { return (size_t)nx * ny; }
};

namespace {

// elementwise grids: 256-thread blocks, at most 16 resident waves' worth
int elem_grid(const pswe_ctx* c, size_t n) {
  size_t b = (n + 255) / 256;
  return (int)std::max<size_t>(1, std::min<size_t>(b, (size_t)c->sms * 16));
}

// optional per-launch event bracketing: PROF_BEGIN before a launch, PROF_END after
cudaEvent_t next_event(pswe_ctx* c) {
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[c->ev_used++];
}
struct ProfScope {
  pswe_ctx* c;
  int cls;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(pswe_ctx* c_, int cls_, cudaStream_t st_) : c(c_), cls(cls_), st(st_) {
    if (c->prof) {
      a = next_event(c);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (c->prof) {
      cudaEvent_t b = next_event(c);
      cudaEventRecord(b, st);
      c->recs.push_back({cls, a, b});
    }
  }
};

// Kernel launch, with programmatic stream serialisation when `pdl`: the
// grid may be scheduled while its predecessor in the stream finishes (every
// kernel of the chain waits on griddepcontrol before its first global
// access).  Used for the stepper's kernels and for one-chunk RHS chains
// (measured: 64^2 M=8 30 -> 26 us, 256^2 M=8 62 -> 57 us, 512^2 M=8
// 169 -> 166 us); the multi-lane chains synchronise through events anyway.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and
// device (it costs microseconds per call on the latency-bound small sizes)
std::mutex g_attr_mutex;
struct AttrKey {
  const void* k;
  int device;
  size_t smem;  // the largest maximum set so far (the attribute is an upper bound)
};
std::vector<AttrKey> g_attr_done;
template <typename K>
cudaError_t smem_attr(K kern, size_t smem, int device) {
  std::lock_guard<std::mutex> lock(g_attr_mutex);
  const void* key = reinterpret_cast<const void*>(kern);
  for (auto& e : g_attr_done)
    if (e.k == key && e.device == device) {
      if (smem <= e.smem) return cudaSuccess;
      const cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (r == cudaSuccess) e.smem = smem;
      return r;
    }
  const cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (r == cudaSuccess) g_attr_done.push_back({key, device, smem});
  return r;
}

// resident CTAs per SM of a kernel (occupancy query, cached per kernel / device)
struct OccKey {
  const void* k;
  int device, threads;
  size_t smem;
  int per_sm;
};
std::vector<OccKey> g_occ;
template <typename K>
int occupancy(K kern, int threads, size_t smem, int device, int fallback) {
  std::lock_guard<std::mutex> lock(g_attr_mutex);
  const void* key = reinterpret_cast<const void*>(kern);
  for (const auto& e : g_occ)
    if (e.k == key && e.device == device && e.threads == threads && e.smem == smem) return e.per_sm;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = fallback;
  g_occ.push_back({key, device, threads, smem, per_sm});
  return per_sm;
}

bool pdl_enabled() {
  static const bool off = getenv("PSWE_NO_PDL") != nullptr;  // A/B switch
  return !off;
}

// ---------------------------------------------------------------- dispatch
template <int NX, bool MW>
int launchA(pswe_ctx* c, const PhaseDev& ph, int p0, int np, const double2* Uc, double2* I1, double* pscale,
            cudaStream_t st) {
  using W = PassAW<NX, MW>;
  const size_t smem = W::bytes(c->Kx);
  auto kern = passA_kernel<NX, MW>;
  CU(smem_attr(kern, smem, c->device));
  const int nblk = ((np + 1) / 2) * ((c->Ky + W::GPW - 1) / W::GPW);
  const int blocks = std::min(nblk, W::CTAS * c->sms);
  ProfScope ps(c, 0, st);
  CU(launch_k(c->pdl, kern, blocks, W::WARPS * 32, smem, st, c->grid(), c->prop(), ph, p0, np, Uc, c->ctab_cur, I1,
              pscale));
  c->launches++;
  c->variant[PSWE_V_PASSA]++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

// rows per pass-B CTA (the output tile width R) for transform length ny
int passB_rows(int ny) { return 4 * 32 / std::max(1, ny / 16); }
// tensor-memory stash + TMA tile store path: NY >= 64 and whole tiles per phase
bool passB_fast(const pswe_ctx* c) { return c->ny >= 64 && c->nx % passB_rows(c->ny) == 0; }

template <int NY>
int launchB_small(pswe_ctx* c, int np, const CUtensorMap& mI1, double2* I2, cudaStream_t st) {
  using W = PassBW<NY>;
  const size_t smem = W::template bytes<false>();
  auto kern = passB_kernel<NY>;
  CU(smem_attr(kern, smem, c->device));
  const int blocks = (np * c->nx + W::GPC - 1) / W::GPC;
  ProfScope ps(c, 1, st);
  CU(launch_k(c->pdl, kern, blocks, W::WARPS * 32, smem, st, c->grid(), np, mI1, I2));
  c->launches++;
  c->variant[PSWE_V_PASSB_ROW]++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

template <int NY>
int launchB_split(pswe_ctx* c, int np, const CUtensorMap& mI1, double2* I2, cudaStream_t st) {
  using W = PassBSW<NY>;
  const size_t smem = W::bytes();
  auto kern = passB_split_kernel<NY>;
  CU(smem_attr(kern, smem, c->device));
  const int blocks = (np * c->nx + W::GPW - 1) / W::GPW;
  ProfScope ps(c, 1, st);
  CU(launch_k(c->pdl, kern, blocks, 128, smem, st, c->grid(), np, mI1, I2));
  c->launches++;
  c->variant[PSWE_V_PASSB_SPLIT]++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

template <int NY>
int launchB_pair(pswe_ctx* c, int np, int lanes, const CUtensorMap& mI1, const CUtensorMap& mO, cudaStream_t st) {
  using W = PassBW<NY>;
  const size_t smem = W::template bytes<true>();
  auto kern = passB_pair_kernel<NY>;
  CU(smem_attr(kern, smem, c->device));
  // two phase pairs per CTA when the lanes' pass-B grids hold >= 16 waves of
  // resident CTAs (512^2 M = 256: 3.811 -> 3.797 ms per RHS, 256^2 M = 256
  // 870 -> 860 us; with fewer waves the coarser grid's tail costs more, e.g.
  // 256^2 M = 32 139 -> 148 us)
  static const int qpc_env = getenv("PSWE_QPC") ? atoi(getenv("PSWE_QPC")) : 0;  // experiments
  const int npair = (np + 1) / 2;
  const long long ctas1 = (long long)lanes * npair * (c->nx / W::GPC);
  const int qpc = std::max(1, qpc_env ? qpc_env : (ctas1 >= 16LL * 3 * c->sms ? 2 : 1));
  const int blocks = (npair + qpc - 1) / qpc * (c->nx / W::GPC);
  ProfScope ps(c, 1, st);
  CU(launch_k(c->pdl, kern, blocks, W::WARPS * 32, smem, st, c->grid(), np, mI1, mO, qpc));
  c->launches++;
  c->variant[PSWE_V_PASSB_PAIR]++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

// The phase-paired kernel runs 11 row transforms in sequence per warp, the
// single-phase one 6: when the pair grids of all lanes together would not
// even give every SM one CTA (small grids, few phases), the evaluation is
// latency-bound and the shorter chain wins (64^2, M = 8: 54 -> 44 us per
// RHS; the C2 step 178 -> 129 us); with more CTAs the pair kernel's
// efficiency wins (256^2, M = 8, 256 pair CTAs: 64 vs 67 us).
template <int NY>
int launchB(pswe_ctx* c, int np, int lanes, const CUtensorMap& mI1, const CUtensorMap& mO, double2* I2,
            cudaStream_t st) {
  if constexpr (NY >= 64) {
    const int sms = c->sms;
    const long long pair_ctas = (long long)lanes * ((np + 1) / 2) * c->nx / PassBW<NY>::GPC;
    if (passB_fast(c) && pair_ctas >= sms + sms / 3) return launchB_pair<NY>(c, np, lanes, mI1, mO, st);
  }
  // fewer single-phase CTAs than SMs: split each row group's transforms over
  // four warps (passB_split_kernel, two transform latencies instead of six)
  {
    const int sms = c->sms;
    const long long small_ctas = (long long)lanes * ((np * c->nx + PassBW<NY>::GPC - 1) / PassBW<NY>::GPC);
    if (small_ctas < sms && !getenv("PSWE_NO_SPLIT")) return launchB_split<NY>(c, np, mI1, I2, st);
  }
  return launchB_small<NY>(c, np, mI1, I2, st);
}

template <int NX>
int pass_c_groups(const pswe_ctx* c, int CP, int lanes) {
  // phase groups per chunk: the grid (cols x Gc CTAs) should fill whole waves
  // of the resident CTAs (occupancy query), each CTA keeping >= 4 phases to amortise its
  // prologue and slot update.  Pick the Gc with the best wave efficiency.
  const int cols = (c->Ky + PassCW<NX>::GPW - 1) / PassCW<NX>::GPW;
  smem_attr(passC_kernel<NX, false>, PassCW<NX>::bytes(c->Kx), c->device);  // before the occupancy query
  const int per_sm = occupancy(passC_kernel<NX, false>, PassCW<NX>::WARPS * 32, PassCW<NX>::bytes(c->Kx),
                               c->device, 3);
  const int sms = c->sms;
  const int slots = per_sm * sms;
  int best = 1;
  double best_eff = 0.0;
  // a grid that cannot fill the SMs even at 4 phases per CTA is latency-
  // bound: then down to one phase per CTA (64^2, M = 8: pass C 16 -> 9 us)
  const int gmax = (long long)cols * std::max(1, CP / 4) < sms ? CP : std::max(1, CP / 4);
  // all lanes' slots within 64 MiB (512^2, four lanes: at most 5 groups of
  // 2.8 MB slots, the choice there is unchanged); small grids, whose few
  // column blocks would otherwise leave most SMs idle (64^2: 3 column blocks
  // x 16 groups = 48 CTAs for 511 phases), may use up to 256 groups (64^2
  // M = 128 76 -> 66 us, 128^2 M = 256 255 -> 245 us, C3 step 188 -> 178 us)
  const size_t slot_bytes = c->compact_elems() * sizeof(double2) * (size_t)std::max(1, lanes);
  const int gcap = (int)std::max<size_t>(1, std::min<size_t>(256, ((size_t)64 << 20) / slot_bytes));
  for (int g = 1; g <= gmax && g <= gcap; ++g) {
    const int ctas = cols * g;
    const int waves = (ctas + slots - 1) / slots;
    const double eff = (double)ctas / ((double)waves * slots);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = g;
    }
  }
  if (const char* e = getenv("PSWE_GC")) best = atoi(e);  // tuning experiments
  return std::max(1, std::min(best, CP));
}

template <int NX, bool MW>
int launchC(pswe_ctx* c, const PhaseDev& ph, int p0, int np, int Gc, int first, const double2* I2,
            double2* slots, cudaStream_t st) {
  using W = PassCW<NX>;
  const size_t smem = W::bytes(c->Kx);
  auto kern = passC_kernel<NX, MW>;
  CU(smem_attr(kern, smem, c->device));
  const int cols = (c->Ky + W::GPW - 1) / W::GPW;
  const int blocks = cols * Gc;
  ProfScope ps(c, 2, st);
  CU(launch_k(c->pdl, kern, blocks, W::WARPS * 32, smem, st, c->grid(), c->prop(), ph, p0, np, Gc, I2, c->ctab_cur,
              slots, first));
  c->launches++;
  c->variant[PSWE_V_PASSC]++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

template <bool MW>
int dispatchA_(pswe_ctx* c, const PhaseDev& ph, int p0, int np, const double2* Uc, double2* I1, double* pscale,
               cudaStream_t st) {
  switch (c->nx) {
    case 8: return launchA<8, MW>(c, ph, p0, np, Uc, I1, pscale, st);
    case 16: return launchA<16, MW>(c, ph, p0, np, Uc, I1, pscale, st);
    case 32: return launchA<32, MW>(c, ph, p0, np, Uc, I1, pscale, st);
    case 64: return launchA<64, MW>(c, ph, p0, np, Uc, I1, pscale, st);
    case 128: return launchA<128, MW>(c, ph, p0, np, Uc, I1, pscale, st);
    case 256: return launchA<256, MW>(c, ph, p0, np, Uc, I1, pscale, st);
    case 512: return launchA<512, MW>(c, ph, p0, np, Uc, I1, pscale, st);
  }
  return set_err(PSWE_EUNSUPPORTED, "unsupported nx = %d", c->nx);
}
int dispatchA(pswe_ctx* c, const PhaseDev& ph, int p0, int np, const double2* Uc, double2* I1, double* pscale,
              cudaStream_t st) {
  return ph.win ? dispatchA_<true>(c, ph, p0, np, Uc, I1, pscale, st)
                : dispatchA_<false>(c, ph, p0, np, Uc, I1, pscale, st);
}
int dispatchB(pswe_ctx* c, int np, int lanes, const CUtensorMap& mI1, const CUtensorMap& mO, double2* I2,
              cudaStream_t st) {
  switch (c->ny) {
    case 8: return launchB<8>(c, np, lanes, mI1, mO, I2, st);
    case 16: return launchB<16>(c, np, lanes, mI1, mO, I2, st);
    case 32: return launchB<32>(c, np, lanes, mI1, mO, I2, st);
    case 64: return launchB<64>(c, np, lanes, mI1, mO, I2, st);
    case 128: return launchB<128>(c, np, lanes, mI1, mO, I2, st);
    case 256: return launchB<256>(c, np, lanes, mI1, mO, I2, st);
    case 512: return launchB<512>(c, np, lanes, mI1, mO, I2, st);
  }
  return set_err(PSWE_EUNSUPPORTED, "unsupported ny = %d", c->ny);
}
int groupsC(const pswe_ctx* c, int CP, int lanes) {
  switch (c->nx) {
    case 8: return pass_c_groups<8>(c, CP, lanes);
    case 16: return pass_c_groups<16>(c, CP, lanes);
    case 32: return pass_c_groups<32>(c, CP, lanes);
    case 64: return pass_c_groups<64>(c, CP, lanes);
    case 128: return pass_c_groups<128>(c, CP, lanes);
    case 256: return pass_c_groups<256>(c, CP, lanes);
    default: return pass_c_groups<512>(c, CP, lanes);
  }
}

template <bool MW>
int dispatchC_(pswe_ctx* c, const PhaseDev& ph, int p0, int np, int Gc, int first, const double2* I2,
               double2* slots, cudaStream_t st) {
  switch (c->nx) {
    case 8: return launchC<8, MW>(c, ph, p0, np, Gc, first, I2, slots, st);
    case 16: return launchC<16, MW>(c, ph, p0, np, Gc, first, I2, slots, st);
    case 32: return launchC<32, MW>(c, ph, p0, np, Gc, first, I2, slots, st);
    case 64: return launchC<64, MW>(c, ph, p0, np, Gc, first, I2, slots, st);
    case 128: return launchC<128, MW>(c, ph, p0, np, Gc, first, I2, slots, st);
    case 256: return launchC<256, MW>(c, ph, p0, np, Gc, first, I2, slots, st);
    case 512: return launchC<512, MW>(c, ph, p0, np, Gc, first, I2, slots, st);
  }
  return set_err(PSWE_EUNSUPPORTED, "unsupported nx = %d", c->nx);
}
int dispatchC(pswe_ctx* c, const PhaseDev& ph, int p0, int np, int Gc, int first, const double2* I2,
              double2* slots, cudaStream_t st) {
  return ph.win ? dispatchC_<true>(c, ph, p0, np, Gc, first, I2, slots, st)
                : dispatchC_<false>(c, ph, p0, np, Gc, first, I2, slots, st);
}

template <int NX>
int launch_diag_cols(pswe_ctx* c, const double2* u, const double2* v, const double2* e, const double2* b,
                     cudaStream_t st) {
  const int tasks = 4 * (c->ny / 2 + 1), per = 4 * WF<NX>::GPW;
  diag_cols_kernel<NX><<<(tasks + per - 1) / per, 128, 0, st>>>(c->grid(), u, v, e, b, c->diag_cols.p);
  c->launches++;
  CU(cudaGetLastError());
  return PSWE_OK;
}
template <int NY>
int launch_diag_rows(pswe_ctx* c, double* phys, cudaStream_t st) {
  const int per = 4 * WF<NY>::GPW;
  diag_rows_kernel<NY><<<(c->nx + per - 1) / per, 128, 0, st>>>(c->grid(), c->diag_cols.p, c->H, c->g,
                                                                  c->diag_part.p, phys);
  c->launches++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

// TMA tensor map of a rank-4 fp64 tensor (dims innermost first, byte strides
// of dims 1..3) with box `box`; the encoder comes from the driver through the
// runtime's entry-point query, so the library links only against cudart.
int encode_map(CUtensorMap* m, void* base, const cuuint64_t* dims, const cuuint64_t* strides,
               const cuuint32_t* box, int rank = 4, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    CU(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    if (!enc || q != cudaDriverEntryPointSuccess)
      return set_err(PSWE_ECUDA, "cuTensorMapEncodeTiled not available from the driver");
  }
  const cuuint32_t es[4] = {1, 1, 1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, base, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(PSWE_ECUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
  return PSWE_OK;
}

// I1[p][f][j][x] gathered by rows: box (re/im, 1 x, Ky j, 1 field-phase)
int map_rows_I1(const pswe_ctx* c, double2* I1, int CP, CUtensorMap* m) {
  const cuuint64_t nx = c->nx, Ky = c->Ky;
  const cuuint64_t dims[4] = {2, nx, Ky, (cuuint64_t)5 * CP};
  const cuuint64_t strides[3] = {16, nx * 16, Ky * nx * 16};
  const cuuint32_t box[4] = {2, 1, (cuuint32_t)Ky, 1};
  return encode_map(m, I1, dims, strides, box);
}

// I2[p][f][j][x] written by pass-B tiles: box (re/im, R x, Ky j, 2 fields)
// I2[p][f][j][x] written by pass-B tiles: rank 3 in doubles (2 nx, Ky, 4 CP),
// box (2R doubles = the tile's R rows, Ky, 2 fields).  The staging tile is
// swizzled (64-byte rows for R = 4, 128-byte rows for R = 8) so that the
// warps' column writes into it are bank-conflict free.
int map_tiles_I2(const pswe_ctx* c, double2* I2, int CP, CUtensorMap* m) {
  const cuuint64_t nx = c->nx, Ky = c->Ky;
  const cuuint32_t R = (cuuint32_t)std::min<cuuint64_t>(passB_rows(c->ny) / 2, nx);  // a warp pair's tile
  const cuuint64_t dims[3] = {2 * nx, Ky, (cuuint64_t)4 * CP};
  const cuuint64_t strides[2] = {nx * 16, Ky * nx * 16};
  const cuuint32_t box[3] = {2 * R, (cuuint32_t)Ky, 2};
  const CUtensorMapSwizzle swz = R == 2   ? CU_TENSOR_MAP_SWIZZLE_32B
                                 : R == 4 ? CU_TENSOR_MAP_SWIZZLE_64B
                                 : (R == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
  return encode_map(m, I2, dims, strides, box, 3, swz);
}

// Averaged RHS on compact data: chunks of phases through passes A, B, C,
// then the ordered slot reduction.  `P` live phases in (s, w) device arrays.
// Hermitian gate scratch: zeroed once, kept zeroed by herm_eval_kernel
// layout: [0..3) statistic A, [4..7) statistic B (the stepper alternates:
// a stage kernel evaluates one while packing the next RHS's into the
// other), [8..8+P) per-phase scales
constexpr int HG_A = 0, HG_B = 4, HG_SCALE = 8;
int ensure_hgate(pswe_ctx* c, int P) {
  const size_t need = HG_SCALE + (size_t)std::max(P, 1);
  if (c->hgate_n >= need) return PSWE_OK;
  TRY(c->hgate.alloc(need));
  CU(cudaMemset(c->hgate.p, 0, need * sizeof(double)));
  c->hgate_n = need;
  return PSWE_OK;
}

// The phases of one evaluation: device (s, w) of the live nodes, the window
// of each phase for a window batch (win, W windows), and the phase table
// that caches their exact-route (c1, c2) columns.
struct PhaseSet {
  const double* s;
  const double* w;
  const int* win;
  int P, W;
  DevBuf<double2>* tab;
  bool* tab_valid;
};
PhaseSet quad_phases(pswe_ctx* c) {
  return {c->s_dev.p, c->w_dev.p, nullptr, (int)c->s_live.size(), 1, &c->ctab_q, &c->ctab_q_valid};
}
PhaseSet zero_phases(pswe_ctx* c) { return {c->zero_s.p, c->one_w.p, nullptr, 1, 1, &c->ctab_0, &c->ctab_0_valid}; }
HermGate hgate_of(pswe_ctx* c, int P, int bit, int stat = HG_A) {
  return HermGate{c->hgate.p + stat, c->hgate.p + HG_SCALE, P, c->bdef, c->H, c->g, c->flags.p, bit};
}
HermGate no_gate() { return HermGate{nullptr, nullptr, 0, 0.0, 1.0, 1.0, nullptr, -1}; }

PhaseSet batch_phases(pswe_ctx* c) {
  return {c->bs_dev.p, c->bw_dev.p, c->bwin_dev.p, (int)c->b_s.size(), c->bW, &c->ctab_b, &c->ctab_b_valid};
}

// ---- generic sizes (generic_kernels.cuh): any even n, also n > 512
FftPlan make_plan(int n, const double2* tw) {
  FftPlan p{};
  p.n = n;
  p.tw = tw;
  int m = n;
  // large register radices first: fewer shared-memory passes and barriers
  for (int r : {16, 8, 4})
    while (m % r == 0 && p.nf < GEN_MAX_FACTORS) { p.f[p.nf++] = r; m /= r; }
  for (int r : {2, 3, 5, 7})
    while (m % r == 0 && p.nf < GEN_MAX_FACTORS) { p.f[p.nf++] = r; m /= r; }
  for (int r = 11; m > 1 && p.nf < GEN_MAX_FACTORS; r += 2)
    while (m % r == 0) { p.f[p.nf++] = r; m /= r; }
  return p;
}

int gen_groups(const pswe_ctx* c, int CP) {
  // pass C: Ky columns x Gc phase groups, about two waves of 4 CTAs per SM, >= 2 phases each
  const int want = std::max(1, (8 * c->sms + c->Ky - 1) / c->Ky);
  return std::max(1, std::min(want, std::max(1, CP / 2)));
}

// threads per generic CTA: about one per radix-4 butterfly of its transform
// length (a whole CTA of 256 threads on a 96-point transform left most of
// them idle), whole warps, at most GEN_THREADS
int gen_threads(int n, int modes = 0) {
  const int want = std::max(n / 8, modes / 2);
  return std::min(GEN_THREADS, std::max(32, (want + 31) / 32 * 32));
}

int launch_gen(pswe_ctx* c, const PhaseDev& ph, int p0, int np, int Gc, int first, const double2* Uc, double2* I1,
               double2* I2, double2* slots, double* pscale, cudaStream_t st) {
  const size_t sA = ((size_t)3 * c->Kx + 2 * (size_t)c->nx) * sizeof(double2);
  const size_t sB = (size_t)6 * c->ny * sizeof(double2);
  const size_t sC = ((size_t)7 * c->Kx + 2 * (size_t)c->nx) * sizeof(double2);
  CU(smem_attr(gen_passA_kernel, sA, c->device));
  CU(smem_attr(gen_passB_kernel, sB, c->device));
  CU(smem_attr(gen_passC_kernel<false>, sC, c->device));
  CU(smem_attr(gen_passC_kernel<true>, sC, c->device));
  {
    ProfScope ps(c, 0, st);
    CU(launch_k(c->pdl, gen_passA_kernel, np * c->Ky, gen_threads(c->nx, c->Kx), sA, st, c->grid(), c->prop(), ph, p0, np, Uc,
                c->ctab_cur, I1, c->plx, pscale));
  }
  {
    ProfScope ps(c, 1, st);
    CU(launch_k(c->pdl, gen_passB_kernel, np * c->nx, gen_threads(c->ny), sB, st, c->grid(), np, (const double2*)I1, I2,
                c->ply));
  }
  {
    ProfScope ps(c, 2, st);
    if (ph.win)
      CU(launch_k(c->pdl, gen_passC_kernel<true>, c->Ky * Gc, gen_threads(c->nx, c->Kx), sC, st, c->grid(), c->prop(), ph, p0, np,
                  Gc, (const double2*)I2, c->ctab_cur, slots, first, c->plx));
    else
      CU(launch_k(c->pdl, gen_passC_kernel<false>, c->Ky * Gc, gen_threads(c->nx, c->Kx), sC, st, c->grid(), c->prop(), ph, p0,
                  np, Gc, (const double2*)I2, c->ctab_cur, slots, first, c->plx));
  }
  c->launches += 3;
  c->variant[PSWE_V_PASSA]++;
  c->variant[PSWE_V_PASSB_ROW]++;
  c->variant[PSWE_V_PASSC]++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

// Small square grids: the one-CTA-per-phase-group kernel (fused_kernels.cuh)
template <int N, bool MW>
int launch_fused(pswe_ctx* c, const PhaseDev& ph, int Gc, const double2* Uc, double2* out, double* pscale,
                 cudaStream_t st) {
  using W = FusedW<N>;
  auto kern = fused_kernel<N, MW>;
  CU(smem_attr(kern, W::bytes(), c->device));
  ProfScope ps(c, 0, st);
  CU(launch_k(c->pdl, kern, Gc, W::NT, W::bytes(), st, c->grid(), c->prop(), ph, Gc, Uc, c->ctab_cur, out, pscale));
  c->launches++;
  c->variant[PSWE_V_FUSED]++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

// 64^2: one 4-CTA cluster per phase group (cluster_kernels.cuh)
constexpr int CF_N = 64, CF_C = 4;

template <bool MW>
int launch_cfused(pswe_ctx* c, const PhaseDev& ph, int Gc, const double2* Uc, double2* out, double* pscale,
                  cudaStream_t st) {
  using W = CFusedW<CF_N, CF_C>;
  auto kern = cfused_kernel<CF_N, CF_C, MW>;
  CU(smem_attr(kern, W::bytes(), c->device));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(Gc * CF_C);
  cfg.blockDim = dim3(W::NT);
  cfg.dynamicSmemBytes = W::bytes();
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CF_C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = c->pdl ? 2 : 1;
  ProfScope ps(c, 0, st);
  CU(cudaLaunchKernelEx(&cfg, kern, c->grid(), c->prop(), ph, Gc, Uc, (const double2*)c->ctab_cur, out, pscale));
  c->launches++;
  c->variant[PSWE_V_FUSED]++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

// clusters resident at once (one CTA per SM; clusters stay inside a GPC)
int cfused_capacity(pswe_ctx* c) {
  static std::atomic<int> cached[64];  // per device ordinal (0 = not yet queried)
  const int dev = c->device & 63;
  if (cached[dev].load() > 0) return cached[dev].load();
  using W = CFusedW<CF_N, CF_C>;
  smem_attr(cfused_kernel<CF_N, CF_C, false>, W::bytes(), c->device);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CF_C * c->sms);
  cfg.blockDim = dim3(W::NT);
  cfg.dynamicSmemBytes = W::bytes();
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CF_C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, cfused_kernel<CF_N, CF_C, false>, &cfg) != cudaSuccess || n < 1)
    n = c->sms / CF_C;
  cached[dev].store(n);
  if (getenv("PSWE_VERBOSE")) fprintf(stderr, "pswe: 64^2 cluster kernel: %d clusters resident\n", n);
  return n;
}

template <int N>
int fused_capacity(const pswe_ctx* c) {
  smem_attr(fused_kernel<N, false>, FusedW<N>::bytes(), c->device);  // before the occupancy query
  return occupancy(fused_kernel<N, false>, FusedW<N>::NT, FusedW<N>::bytes(), c->device, 1) * c->sms;
}

// Measured (tools/fused_check.py): n <= 32 one CTA per phase group wins
// everywhere (32^2, M = 8: 30 -> 20 us; M = 256: 131 -> 63 us); at 64^2 the
// single CTA's 8 warps are latency-bound (M = 256: 113 -> 128 us), so 64^2
// keeps the three-pass pipeline unless PSWE_FUSED64 is set.
bool cluster_ok(pswe_ctx* c, int P);
bool fused_ok(pswe_ctx* c, int P) {
  static const bool off = getenv("PSWE_NO_FUSED") != nullptr;  // A/B switch
  static const bool single64 = getenv("PSWE_FUSED64") != nullptr;
  return !off && !c->gen && c->nx == c->ny && (c->nx <= 32 || (c->nx == 64 && (single64 || cluster_ok(c, P))));
}
// 64^2: the cluster kernel while every cluster gets at most two phases
// (tools/c64_check.py, L2 flushed: M = 8 26.2 -> 24.8 us, M = 16 32.6 ->
// 27.7, M = 32 44.5 -> 39.9; with more phases the three passes' throughput
// wins, M = 256 113 vs 197 us; one phase: the three passes, 23.0 vs 24.8);
// PSWE_FUSED64: the single-CTA kernel instead (experiments)
int cfused_capacity(pswe_ctx* c);
bool cluster_ok(pswe_ctx* c, int P) {
  static const bool single = getenv("PSWE_FUSED64") != nullptr;
  return c->nx == 64 && !single && P >= 2 && P <= 2 * cfused_capacity(c);
}

// `gate`: the input was packed with the gate's statistics (pack_kernel
// hstat = hgate) and pass A adds the per-phase scales; the kernel that
// consumes the result evaluates them (herm_eval_block, via hgate_of) and
// sets its flags bit when the exact check has to decide.  A window batch (ps.win) evaluates W
// windows' tendencies at once: Uc / Ac hold W compact states.
int rhs_compact(pswe_ctx* c, const PhaseSet& ps, const double2* Uc, double2* Ac, cudaStream_t st,
                bool gate = false) {
  const double* s = ps.s;
  const int P = ps.P;
  const bool fused = fused_ok(c, P);
  // exact route: phase table (built once per quadrature / grid)
  c->ctab_cur = nullptr;
  if (c->kind == 0) {
    DevBuf<double2>& tb = *ps.tab;
    bool& valid = *ps.tab_valid;
    if (!valid) {
      TRY(tb.alloc((size_t)P * c->Ky * c->Kx));
      phase_table_kernel<<<elem_grid(c, (size_t)P * c->Ky * c->Kx), 256, 0, st>>>(c->grid(), s, P, tb.p);
      c->launches++;
      CU(cudaGetLastError());
      valid = true;
    }
    c->ctab_cur = tb.p;
  }
  if (fused) {
    // one CTA per phase group, every resident CTA busy at most once
    int cap = 1;
    const bool clu = c->nx == 64 && cluster_ok(c, P);
    switch (c->nx) {
      case 8: cap = fused_capacity<8>(c); break;
      case 16: cap = fused_capacity<16>(c); break;
      case 32: cap = fused_capacity<32>(c); break;
      default: cap = clu ? cfused_capacity(c) : fused_capacity<64>(c); break;
    }
    const int Gc = std::max(1, std::min(P, cap));
    const size_t cw = (size_t)ps.W * c->compact_elems();
    const bool direct = Gc == 1 && !ps.win;
    c->pdl = pdl_enabled();
    if (!direct) TRY(c->slots.alloc((size_t)Gc * cw));
    double2* out = direct ? Ac : c->slots.p;
    if (ps.win) CU(cudaMemsetAsync(c->slots.p, 0, (size_t)Gc * cw * sizeof(double2), st));
    PhaseDev ph{s, ps.w, P};
    ph.win = ps.win;
    ph.W = ps.W;
    ph.ustride = c->compact_elems();
    double* pscale = gate ? c->hgate.p + HG_SCALE : nullptr;
    int rc = PSWE_OK;
    switch (c->nx) {
      case 8: rc = ps.win ? launch_fused<8, true>(c, ph, Gc, Uc, out, pscale, st)
                          : launch_fused<8, false>(c, ph, Gc, Uc, out, pscale, st); break;
      case 16: rc = ps.win ? launch_fused<16, true>(c, ph, Gc, Uc, out, pscale, st)
                           : launch_fused<16, false>(c, ph, Gc, Uc, out, pscale, st); break;
      case 32: rc = ps.win ? launch_fused<32, true>(c, ph, Gc, Uc, out, pscale, st)
                           : launch_fused<32, false>(c, ph, Gc, Uc, out, pscale, st); break;
      default:
        if (clu)
          rc = ps.win ? launch_cfused<true>(c, ph, Gc, Uc, out, pscale, st)
                      : launch_cfused<false>(c, ph, Gc, Uc, out, pscale, st);
        else
          rc = ps.win ? launch_fused<64, true>(c, ph, Gc, Uc, out, pscale, st)
                      : launch_fused<64, false>(c, ph, Gc, Uc, out, pscale, st);
        break;
    }
    TRY(rc);
    if (!direct) {
      ProfScope pr3(c, 3, st);
      // 32 slots per load round (staged kernel) instead of the serial batches
      if (!getenv("PSWE_NO_STAGED"))
        CU(launch_k(c->pdl, reduce_slots_staged_kernel, (int)std::min<size_t>((cw + 31) / 32, (size_t)c->sms * 8), 256,
                    0, st, (const double2*)c->slots.p, Gc, cw, Ac));
      else
        CU(launch_k(c->pdl, reduce_slots_kernel, elem_grid(c, cw), 256, 0, st, (const double2*)c->slots.p, Gc, cw,
                    Ac));
      c->launches++;
      c->variant[PSWE_V_REDUCE]++;
      CU(cudaGetLastError());
    }
    return PSWE_OK;
  }
  const size_t per_phase = (size_t)9 * c->Ky * c->nx;  // I1 (5 fields) + I2 (4 fields), double2
  // Chunk "lanes" on separate streams when there is more than one chunk:
  // the chunks' passes overlap and fill each other's launch tails.  Each lane
  // has its own intermediates and slot set; chunks go round-robin over the
  // lanes, every slot accumulates its lane's chunks in order and the final
  // reduction sums lane 0's slots, then lane 1's, ... -- a fixed order, so
  // results stay bitwise deterministic.  The phases are split into a
  // multiple of `lanes` equal chunks no larger than chunk_bytes, so the lanes
  // finish together.
  const int cpmax = (int)std::max<size_t>(1, c->chunk_bytes / (per_phase * sizeof(double2)));
  // at least one chunk per lane when a chunk still holds >= 8 phases and
  // >= 24 MiB of intermediates: the lanes' overlap is then worth more than
  // the larger per-launch grids of fewer chunks (tools/lane_sweep.sh: 8
  // instead of 16 phases gains 1.6-1.7 % at 256^2 / 512^2, M = 32; other
  // points unchanged)
  static const int minph_floor = getenv("PSWE_MINPH") ? atoi(getenv("PSWE_MINPH")) : 8;  // tuning experiments
  static const int minmb = getenv("PSWE_MINMB") ? atoi(getenv("PSWE_MINMB")) : 24;
  const int minph = std::max<int>(minph_floor, (int)(((size_t)minmb << 20) / (per_phase * sizeof(double2))));
  int nchunks = std::max((P + cpmax - 1) / cpmax, std::min(c->n_lanes, P / minph));
  const int lanes = std::max(1, std::min(c->n_lanes, nchunks));
  nchunks = (nchunks + lanes - 1) / lanes * lanes;
  const int CP = std::max(1, std::min(P, (P + nchunks - 1) / nchunks));
  nchunks = (P + CP - 1) / CP;
  const int Gc = c->gen ? gen_groups(c, CP) : groupsC(c, CP, lanes);  // accumulation slots = phase groups per chunk
  const int SGN = Gc;
  c->pdl = pdl_enabled() && nchunks == 1;
  const size_t cw = (size_t)ps.W * c->compact_elems();  // one slot set: W compact states
  TRY(c->inter.alloc(per_phase * CP * lanes));
  TRY(c->slots.alloc((size_t)lanes * Gc * cw));
  static const bool poison = getenv("PSWE_DEBUG_POISON") != nullptr;
  if (poison) {  // debug: NaN-fill every scratch and the output, exposing entries read before written
    CU(cudaMemsetAsync(c->inter.p, 0xFF, per_phase * CP * lanes * sizeof(double2), st));
    if (!ps.win) CU(cudaMemsetAsync(c->slots.p, 0xFF, (size_t)lanes * Gc * cw * sizeof(double2), st));
    CU(cudaMemsetAsync(Ac, 0xFF, cw * sizeof(double2), st));
  }
  // window batch: pass C adds every window segment of its phase group into
  // zeroed slots (a group may hold several windows, a window several groups)
  if (ps.win) CU(cudaMemsetAsync(c->slots.p, 0, (size_t)lanes * Gc * cw * sizeof(double2), st));
  PhaseDev ph{s, ps.w, P};
  ph.win = ps.win;
  ph.W = ps.W;
  ph.ustride = c->compact_elems();
  cudaStream_t lst[pswe_ctx::MAX_LANES] = {st, c->st_lane[0], c->st_lane[1], c->st_lane[2]};
  // the lanes' tensor maps, encoded again only when the intermediates or
  // the chunk size change (the driver call costs microseconds, which the
  // latency-bound small sizes would see as launch gaps)
  CUtensorMap* mrow = c->map_rows;
  CUtensorMap* mcol = c->map_tiles;
  for (int L = 0; L < lanes && !c->gen; ++L) {
    double2* I1 = c->inter.p + (size_t)L * per_phase * CP;
    if (c->map_base[L] == I1 && c->map_cp[L] == CP) continue;
    TRY(map_rows_I1(c, I1, CP, &mrow[L]));
    TRY(map_tiles_I2(c, I1 + (size_t)5 * c->Ky * c->nx * CP, CP, &mcol[L]));
    c->map_base[L] = I1;
    c->map_cp[L] = CP;
  }
  if (lanes > 1) {
    CU(cudaEventRecord(c->ev_fork, st));
    for (int L = 1; L < lanes; ++L) CU(cudaStreamWaitEvent(lst[L], c->ev_fork, 0));
  }
  const bool direct = nchunks == 1 && Gc == 1 && !ps.win;
  int chunk = 0;
  for (int p0 = 0; p0 < P; p0 += CP, ++chunk) {
    const int np = std::min(CP, P - p0);
    const int L = chunk % lanes;
    double2* I1 = c->inter.p + (size_t)L * per_phase * CP;
    double2* I2 = I1 + (size_t)5 * c->Ky * c->nx * CP;
    // a single slot (one chunk, Gc = 1, e.g. the fine-step reference's one
    // node) is the output itself: pass C writes it, no reduction launch
    double2* sl = direct ? Ac : c->slots.p + (size_t)L * Gc * cw;
    if (c->gen) {
      TRY(launch_gen(c, ph, p0, np, Gc, chunk < lanes ? 1 : 0, Uc, I1, I2, sl, gate ? c->hgate.p + HG_SCALE : nullptr,
                     lst[L]));
      continue;
    }
    TRY(dispatchA(c, ph, p0, np, Uc, I1, gate ? c->hgate.p + HG_SCALE : nullptr, lst[L]));
    TRY(dispatchB(c, np, lanes, mrow[L], mcol[L], I2, lst[L]));
    TRY(dispatchC(c, ph, p0, np, Gc, chunk < lanes ? 1 : 0, I2, sl, lst[L]));
  }
  for (int L = 1; L < lanes; ++L) {
    CU(cudaEventRecord(c->ev_lane[L - 1], lst[L]));
    CU(cudaStreamWaitEvent(st, c->ev_lane[L - 1], 0));
  }
  if (!direct) {
    const size_t n = cw;
    ProfScope ps(c, 3, st);
    // many slots (small grids): the split reduction (64^2 M = 256: 113 -> 104 us
    // with the raised group cap; up to 32 slots the one-pass kernel is faster)
    if (lanes * SGN > 32) {
      const int blocks = (int)std::min<size_t>((n + 31) / 32, (size_t)c->sms * 8);
      CU(launch_k(c->pdl, reduce_slots_split_kernel, blocks, 32 * RED_PARTS, 0, st, (const double2*)c->slots.p,
                  lanes * SGN, n, Ac));
    } else if (n <= (size_t(1) << 16) && !getenv("PSWE_NO_STAGED")) {
      // small states: every slot loaded in one round, same summation order
      CU(launch_k(c->pdl, reduce_slots_staged_kernel, (int)std::min<size_t>((n + 31) / 32, (size_t)c->sms * 8), 256, 0,
                  st, (const double2*)c->slots.p, lanes * SGN, n, Ac));
    } else {
      CU(launch_k(c->pdl, reduce_slots_kernel, elem_grid(c, n), 256, 0, st, (const double2*)c->slots.p, lanes * SGN,
                  n, Ac));
    }
    c->launches++;
    c->variant[PSWE_V_REDUCE]++;
    CU(cudaGetLastError());
  }
  return PSWE_OK;
}

// ---------------------------------------------------------------- Hermitian gate, exact path
int herm_message(pswe_ctx* c, double worst, double ref, long long idx, std::string* msg) {
  const int i = (int)(idx / c->ny), j = (int)(idx % c->ny);
  const int wx = i < c->nx / 2 ? i : i - c->nx, wy = j < c->ny / 2 ? j : j - c->ny;
  char buf[256];
  snprintf(buf, sizeof(buf),
           "non-Hermitian spectral field: mode (kx index %d, ky index %d) has asymmetry %.3e (relative %.3e)", wx,
           wy, worst, worst / ref);
  *msg = buf;
  return PSWE_EHERM;
}

// The reference's gate at every node of (s_dev, s_host, k) in ascending order
// on the full-layout state U (dynamics.py:159-164 inside averaging.py:130-141):
// PSWE_EHERM with the first failing node's message (wrapped as the node
// error when `k` is given), PSWE_OK when every node passes.  Nodes whose
// propagated fields are not finite are left to the non-finite stage check.
int exact_gate(pswe_ctx* c, const double* s_dev, const std::vector<double>& s_host, const std::vector<int>* k,
               Full3 U, cudaStream_t st) {
  const int P = (int)s_host.size();
  TRY(c->hout.alloc((size_t)8 * P));
  herm_node_kernel<256><<<P, 256, 0, st>>>(c->grid(), c->prop(), s_dev, U.u, U.v, U.e,
                                           c->bfull.p ? (const double2*)c->bfull.p : nullptr, c->hout.p);
  c->launches++;
  c->variant[PSWE_V_HERM]++;
  CU(cudaGetLastError());
  std::vector<double> h((size_t)8 * P);
  CU(cudaMemcpyAsync(h.data(), c->hout.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  for (int p = 0; p < P; ++p) {
    const double* o = h.data() + (size_t)8 * p;
    const double ref = o[0];
    if (o[7] != 0.0 || !(ref > 0.0)) continue;
    for (int f = 0; f < 3; ++f) {
      const double worst = o[1 + 2 * f];
      if (worst > 1e-12 * ref) {
        std::string m;
        herm_message(c, worst, ref, (long long)o[2 + 2 * f], &m);
        if (k)
          return set_err(PSWE_EHERM, "averaging node k = %d (s = %.6g s) failed: %s", (*k)[p], s_host[p], m.c_str());
        return set_err(PSWE_EHERM, "%s", m.c_str());
      }
    }
  }
  return PSWE_OK;
}

// The full-grid gate of to_physical as the snapshot paths call it
// (diagnostics.py:21-25 + :72, integrator.py:126-129, io.py:41-46): u and v
// against vel_scale = max(max|u|, max|v|), eta against itself, b (when
// `with_b`) against itself, in that order.  Synchronises.
int full_gate(pswe_ctx* c, Full3 U, bool with_b, cudaStream_t st) {
  const double2* b = c->bfull.p;
  const int nf = (with_b && b) ? 4 : 3;
  TRY(c->hout.alloc((size_t)8 * 4));
  herm_full_kernel<1024><<<nf, 1024, 0, st>>>(c->nx, c->ny, U.u, U.v, U.e, b, c->hout.p);
  c->launches++;
  c->variant[PSWE_V_HERM]++;
  CU(cudaGetLastError());
  double h[32];
  CU(cudaMemcpyAsync(h, c->hout.p, (size_t)8 * nf * sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  const double vel = std::max(h[0], h[8]);
  for (int f = 0; f < nf; ++f) {
    const double* o = h + 8 * f;
    if (o[7] != 0.0) continue;  // non-finite field: left to the callers' finite checks
    const double ref = f < 2 ? std::max(o[0], vel) : o[0];
    if (ref > 0.0 && o[1] > 1e-12 * ref) {
      std::string m;
      herm_message(c, o[1], ref, (long long)o[2], &m);
      return set_err(PSWE_EHERM, "%s", m.c_str());
    }
  }
  return PSWE_OK;
}

int check_cheb(const pswe_ctx* c, double t, std::string* msg) {
  if (c->kind != 1 || t == 0.0) return PSWE_OK;
  const double need = std::fabs(t) * c->lam_max;
  if (need > c->Lambda * (1.0 + 1e-9)) {
    char buf[256];
    snprintf(buf, sizeof(buf), "|t| * max_frequency = %.6g exceeds Lambda = %.6g; enlarge Lambda or shorten t",
             need, c->Lambda);
    *msg = buf;
    return PSWE_EINVAL;
  }
  return PSWE_OK;
}

// host-side Chebyshev precondition over the live nodes, first failure in
// ascending order wrapped like averaging.py:138-141
int check_nodes(const pswe_ctx* c) {
  std::string msg;
  for (size_t i = 0; i < c->s_live.size(); ++i) {
    if (check_cheb(c, c->s_live[i], &msg) != PSWE_OK)
      return set_err(PSWE_EINVAL, "averaging node k = %d (s = %.6g s) failed: %s", c->k_live[i], c->s_live[i],
                     msg.c_str());
  }
  return PSWE_OK;
}

int ensure_compact(pswe_ctx* c) {
  TRY(c->Uc.alloc(c->compact_elems()));
  TRY(c->Ac.alloc(c->compact_elems()));
  return PSWE_OK;
}

Full3 f3(const double* u, const double* v, const double* e) {
  return Full3{(const double2*)u, (const double2*)v, (const double2*)e};
}
Full3w f3w(double* u, double* v, double* e) { return Full3w{(double2*)u, (double2*)v, (double2*)e}; }
Full3 f3c(const Full3w& a) { return Full3{a.u, a.v, a.e}; }

// flags word: bit 3 (stage - 1) + field = non-finite field after a stage;
// bit HERM_BIT0 + stage - 1 = the gate flagged that stage's RHS input;
// HERM_BIT_RHS = the gate flagged a standalone evaluation's input
constexpr int HERM_BIT0 = 9, HERM_BIT_RHS = 12;

// One transformed SSPRK3 step of W windows (W = 1: the ordinary step) from
// U to out.  `tmp` holds the stage states edt, u1, u2 (3 x W states of 3n,
// window w's at + w * 3n); U / out may be separate field pointers when
// W = 1, else [W][3][n] blocks with window stride ws = 3n.  Uc / Ac: W
// compact states.
int step_impl_w(pswe_ctx* c, const PhaseSet& ps, double dt, Full3 U, Full3w out, double2* tmp, double2* Uc,
                double2* Ac, cudaStream_t st) {
  const size_t n = c->full_elems(), ws = 3 * n;
  const int W = ps.W;
  Full3w edt{tmp, tmp + n, tmp + 2 * n};
  Full3w u1{tmp + 3 * W * n, tmp + 3 * W * n + n, tmp + 3 * W * n + 2 * n};
  Full3w u2{tmp + 6 * W * n, tmp + 6 * W * n + n, tmp + 6 * W * n + 2 * n};
  const GridDev G = c->grid();
  const Prop pr = c->prop();
  TRY(ensure_hgate(c, ps.P));
  // stage kernels: per-mode sincos and exponentials, a latency chain at small
  // sizes -- 64-thread blocks spread few modes over more SMs (64^2: 64 blocks
  // instead of 16)
  static const bool wide = getenv("PSWE_STAGE_TB256") != nullptr;  // A/B switch
  const int tb = (!wide && (size_t)W * n <= (size_t(1) << 15)) ? 64 : 256;
  const int gb = tb == 256 ? elem_grid(c, (size_t)W * n) : (int)(((size_t)W * n + tb - 1) / tb);
  const int gp = elem_grid(c, (size_t)W * c->compact_elems());
  // stage 1 (its input packed here; the stage kernels pack the inputs of
  // RHS 2 and 3 themselves, alternating the gate statistic A / B)
  c->pdl = pdl_enabled();
  CU(launch_k(c->pdl, pack_kernel, gp, 256, 0, st, G, U.u, U.v, U.e, Uc, c->hgate.p + HG_A, W, ws));
  c->launches++;
  TRY(rhs_compact(c, ps, Uc, Ac, st, true));
  c->pdl = pdl_enabled();
  CU(launch_k(c->pdl, stage1_kernel, gb, tb, 0, st, G, pr, dt, U, (const double2*)Ac, edt, u1, c->flags.p, W, ws,
              hgate_of(c, ps.P, HERM_BIT0, HG_A), PackOut{Uc, c->hgate.p + HG_B}));
  c->launches++;
  // stage 2
  TRY(rhs_compact(c, ps, Uc, Ac, st, true));
  c->pdl = pdl_enabled();
  CU(launch_k(c->pdl, stage2_kernel, gb, tb, 0, st, G, pr, dt, U, f3c(u1), (const double2*)Ac, u2, c->flags.p, W,
              ws, hgate_of(c, ps.P, HERM_BIT0 + 1, HG_B), PackOut{Uc, c->hgate.p + HG_A}));
  c->launches++;
  // stage 3
  TRY(rhs_compact(c, ps, Uc, Ac, st, true));
  c->pdl = pdl_enabled();
  CU(launch_k(c->pdl, stage3_kernel, gb, tb, 0, st, G, pr, dt, f3c(edt), f3c(u2), (const double2*)Ac, out,
              c->flags.p, W, ws, hgate_of(c, ps.P, HERM_BIT0 + 2, HG_A)));
  c->launches++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

int step_impl(pswe_ctx* c, double dt, Full3 U, Full3w out, cudaStream_t st) {
  TRY(ensure_compact(c));
  TRY(c->full_tmp.alloc(c->full_elems() * 18));
  return step_impl_w(c, quad_phases(c), dt, U, out, c->full_tmp.p, c->Uc.p, c->Ac.p, st);
}

int decode_flags(int bits, int* stage, int* field) {
  for (int st = 1; st <= 3; ++st)
    for (int fl = 0; fl < 3; ++fl)
      if (bits & (1 << (3 * (st - 1) + fl))) {
        *stage = st;
        *field = fl;
        return 1;
      }
  return 0;
}

const char* field_name(int f) { return f == 0 ? "u" : (f == 1 ? "v" : "eta"); }

// The step's flags in the reference's order of events (integrator.py:95-102):
// stage s's RHS input through the gate, then stage s's finite check.
// `in` is the step's input state; the stage 2 / 3 inputs are the stepper's
// u1 / u2 scratch.  Returns PSWE_OK, PSWE_EHERM (message set) or
// PSWE_ENONFINITE (message, *stage and *field set).
int step_verdict(pswe_ctx* c, int bits, Full3 in, cudaStream_t st, int* stage, int* field) {
  const size_t n = c->full_elems();
  const double2* t = c->full_tmp.p;
  const Full3 inputs[3] = {in, {t + 3 * n, t + 4 * n, t + 5 * n}, {t + 6 * n, t + 7 * n, t + 8 * n}};
  for (int sg = 1; sg <= 3; ++sg) {
    if (bits & (1 << (HERM_BIT0 + sg - 1))) {
      const int rc = exact_gate(c, c->s_dev.p, c->s_live, &c->k_live, inputs[sg - 1], st);
      if (rc != PSWE_OK) {
        *stage = sg;
        *field = -1;
        return rc;
      }
    }
    for (int fl = 0; fl < 3; ++fl)
      if (bits & (1 << (3 * (sg - 1) + fl))) {
        *stage = sg;
        *field = fl;
        return set_err(PSWE_ENONFINITE, "non-finite values in field %s after stage %d", field_name(fl), sg);
      }
  }
  *stage = 0;
  *field = -1;
  return PSWE_OK;
}

// Capture "step A -> B, copy B -> A" as a CUDA graph (cached per dt and
// configuration version).  Every buffer it touches is allocated by the
// un-captured first step, so nothing allocates during capture.
// m > 1: m (even) steps in one graph, A -> B -> A -> ..., no copies: the
// copy node costs its own ~2 us and, not being a kernel, stops the next
// step's first kernel from starting under the last stage kernel (dependent
// launch), as does every graph boundary.
constexpr int STEP_GRAPH_MULTI = 8;
int ensure_step_graph(pswe_ctx* c, double dt, Full3 Ain, Full3w Bout, size_t bytes3, cudaStream_t st, int m = 1) {
  cudaGraphExec_t& exec = m > 1 ? c->stepm_exec : c->step_exec;
  double& gdt = m > 1 ? c->graphm_dt : c->graph_dt;
  int64_t& gver = m > 1 ? c->graphm_version : c->graph_version;
  int64_t& ggen = m > 1 ? c->graphm_gen : c->graph_gen;
  const double2*& gA = m > 1 ? c->graphm_A : c->graph_A;
  if (exec && gdt == dt && gver == c->version && gA == Ain.u && ggen == g_alloc_gen) return PSWE_OK;
  if (exec) cudaGraphExecDestroy(exec);
  exec = nullptr;
  const bool prof = c->prof;
  c->prof = false;
  const int64_t l0 = c->launches;
  int64_t v0[PSWE_NUM_VARIANTS];
  std::copy(c->variant, c->variant + PSWE_NUM_VARIANTS, v0);
  CU(cudaStreamSynchronize(st));
  std::lock_guard<std::recursive_mutex> lock(g_capture_mutex);
  CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
  int rc = PSWE_OK;
  cudaError_t ce = cudaSuccess;
  if (m == 1) {
    rc = step_impl(c, dt, Ain, Bout, st);
    ce = cudaMemcpyAsync((void*)Ain.u, Bout.u, bytes3, cudaMemcpyDeviceToDevice, st);
  } else {
    const Full3w Aout{const_cast<double2*>(Ain.u), const_cast<double2*>(Ain.v), const_cast<double2*>(Ain.e)};
    for (int j = 0; j < m && rc == PSWE_OK; j += 2) {
      rc = step_impl(c, dt, Ain, Bout, st);
      if (rc == PSWE_OK) rc = step_impl(c, dt, f3c(Bout), Aout, st);
    }
  }
  cudaGraph_t g = nullptr;
  cudaError_t ee = cudaStreamEndCapture(st, &g);
  c->prof = prof;
  if (rc != PSWE_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  CU(ce);
  CU(ee);
  cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  CU(ie);
  if (m == 1) c->step_graph_launches = c->launches - l0;
  c->launches = l0;
  for (int i = 0; i < PSWE_NUM_VARIANTS; ++i) {
    if (m == 1) c->graph_variant[i] = c->variant[i] - v0[i];
    c->variant[i] = v0[i];
  }
  gdt = dt;
  gver = c->version;
  gA = Ain.u;
  ggen = g_alloc_gen;
  return PSWE_OK;
}

}  // namespace

// =============================================================== C ABI
extern "C" {

int pswe_version(void) { return 100; }

const char* pswe_last_error(void) { return g_err.c_str(); }

int pswe_create(pswe_ctx** out, int nx, int ny, double Lx, double Ly, double f, double g, double H, int device) {
  if (!out) return set_err(PSWE_EINVAL, "null context pointer");
  std::lock_guard<std::recursive_mutex> lock(g_capture_mutex);  // setup synchronises the device
  *out = nullptr;
  if (nx < 8 || nx % 2 != 0) return set_err(PSWE_EINVAL, "nx must be even and >= 8, got %d", nx);
  if (ny < 8 || ny % 2 != 0) return set_err(PSWE_EINVAL, "ny must be even and >= 8, got %d", ny);
  if (!(Lx > 0)) return set_err(PSWE_EINVAL, "Lx must be positive, got %g", Lx);
  if (!(Ly > 0)) return set_err(PSWE_EINVAL, "Ly must be positive, got %g", Ly);
  if (!(g > 0)) return set_err(PSWE_EINVAL, "g must be positive, got %g", g);
  if (!(H > 0)) return set_err(PSWE_EINVAL, "H must be positive, got %g", H);
  if (nx > 4096 || ny > 4096)
    return set_err(PSWE_EUNSUPPORTED, "grid %dx%d not supported by the B200 path (nx, ny <= 4096)", nx, ny);
  CU(cudaSetDevice(device));
  pswe_ctx* c = new pswe_ctx();
  c->device = device;
  if (cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || c->sms < 1)
    c->sms = 148;
  c->nx = nx; c->ny = ny; c->Lx = Lx; c->Ly = Ly; c->f = f; c->g = g; c->H = H;
  c->kxm = nx / 3; c->kym = ny / 3;
  c->Kx = 2 * c->kxm + 1; c->Ky = c->kym + 1;
  // wavenumbers exactly as make_grid: 2 pi * wrap / L (grid.py:98-101)
  c->kx_full.resize(nx);
  c->ky_full.resize(ny);
  for (int i = 0; i < nx; ++i) {
    const int w = i < nx / 2 ? i : i - nx;
    c->kx_full[i] = 2.0 * M_PI * (double)w / Lx;
  }
  for (int j = 0; j < ny; ++j) {
    const int w = j < ny / 2 ? j : j - ny;
    c->ky_full[j] = 2.0 * M_PI * (double)w / Ly;
  }
  std::vector<double> kxc(c->Kx), kyc(c->Ky);
  for (int r = 0; r < c->Kx; ++r) {
    const int w = r <= c->kxm ? r : r - c->Kx;
    kxc[r] = c->kx_full[(w + nx) % nx];
  }
  for (int j = 0; j < c->Ky; ++j) kyc[j] = c->ky_full[j];
  // max_frequency (dynamics.py:189-192): max over the full grid
  double lm = 0;
  for (int i = 0; i < nx; ++i)
    for (int j = 0; j < ny; ++j) {
      const double kx = c->kx_full[i], ky = c->ky_full[j];
      lm = std::max(lm, std::sqrt(f * f + g * H * (kx * kx + ky * ky)));
    }
  c->lam_max = lm;
  int rc = PSWE_OK;
  auto up = [&](DevBuf<double>& b, const std::vector<double>& h) -> int {
    TRY(b.alloc(h.size()));
    CU(cudaMemcpy(b.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
    return PSWE_OK;
  };
  if ((rc = up(c->kxc, kxc)) || (rc = up(c->kyc, kyc)) || (rc = up(c->kxf, c->kx_full)) ||
      (rc = up(c->kyf, c->ky_full))) {
    pswe_destroy(c);
    return rc;
  }
  if ((rc = c->twx.alloc(nx)) || (rc = c->twy.alloc(ny)) || (rc = c->bc.alloc((size_t)c->Ky * c->Kx)) ||
      (rc = c->flags.alloc(1))) {
    pswe_destroy(c);
    return rc;
  }
  twiddle_kernel<<<(nx + 255) / 256, 256>>>(c->twx.p, nx);
  twiddle_kernel<<<(ny + 255) / 256, 256>>>(c->twy.p, ny);
  c->gen = !pow2_ok(nx) || !pow2_ok(ny);
  c->plx = make_plan(nx, c->twx.p);
  c->ply = make_plan(ny, c->twy.p);
  cudaMemset(c->bc.p, 0, (size_t)c->Ky * c->Kx * sizeof(double2));
  cudaMemset(c->flags.p, 0, sizeof(int));
  {
    std::vector<double> z(1, 0.0), o(1, 1.0);
    if ((rc = up(c->zero_s, z)) || (rc = up(c->one_w, o))) {
      pswe_destroy(c);
      return rc;
    }
  }
  for (int L = 0; L < pswe_ctx::MAX_LANES - 1; ++L) {
    if (cudaStreamCreateWithFlags(&c->st_lane[L], cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_lane[L], cudaEventDisableTiming) != cudaSuccess) {
      pswe_destroy(c);
      return set_err(PSWE_ECUDA, "stream/event creation failed");
    }
  }
  if (const char* e = getenv("PSWE_LANES")) c->n_lanes = std::max(1, std::min(pswe_ctx::MAX_LANES, atoi(e)));
  if (cudaStreamCreateWithFlags(&c->st_run, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_run, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    pswe_destroy(c);
    return set_err(PSWE_ECUDA, "stream/event creation failed");
  }
  if (cudaMallocHost(&c->flags_host, sizeof(int)) != cudaSuccess) {
    pswe_destroy(c);
    return set_err(PSWE_ECUDA, "cudaMallocHost failed");
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    pswe_destroy(c);
    return set_err(PSWE_ECUDA, "CUDA error %s during context setup", cudaGetErrorString(e));
  }
  *out = c;
  return PSWE_OK;
}

void pswe_destroy(pswe_ctx* c) {
  if (!c) return;
  std::lock_guard<std::recursive_mutex> lock(g_capture_mutex);
  cudaSetDevice(c->device);
  for (DevBuf<double>* b : {&c->kxc, &c->kyc, &c->kxf, &c->kyf, &c->s_dev, &c->w_dev, &c->zero_s, &c->one_w, &c->a_dev})
    b->release();
  for (DevBuf<double2>* b : {&c->twx, &c->twy, &c->bc, &c->inter, &c->slots, &c->Uc, &c->Ac, &c->Ac2, &c->full_tmp,
                             &c->bfull, &c->diag_cols, &c->ctab_q, &c->ctab_0, &c->ctab_b, &c->b_full, &c->b_Uc,
                             &c->b_Ac})
    b->release();
  for (DevBuf<double>* b : {&c->bs_dev, &c->bw_dev, &c->hgate, &c->hout}) b->release();
  c->bwin_dev.release();
  c->diag_part.release();
  c->flags.release();
  if (c->flags_host) cudaFreeHost(c->flags_host);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (int L = 0; L < pswe_ctx::MAX_LANES - 1; ++L) {
    if (c->ev_lane[L]) cudaEventDestroy(c->ev_lane[L]);
    if (c->st_lane[L]) cudaStreamDestroy(c->st_lane[L]);
  }
  if (c->step_exec) cudaGraphExecDestroy(c->step_exec);
  if (c->stepm_exec) cudaGraphExecDestroy(c->stepm_exec);
  if (c->bstep_exec) cudaGraphExecDestroy(c->bstep_exec);
  if (c->ev_run) cudaEventDestroy(c->ev_run);
  if (c->st_run) cudaStreamDestroy(c->st_run);
  delete c;
}

int pswe_set_topography(pswe_ctx* c, const double* b_dev, void* stream) {
  if (!c || !b_dev) return set_err(PSWE_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  CU(cudaSetDevice(c->device));
  // compact, Hermitian-projected band of b; pack_kernel fills 3 fields, use scratch
  TRY(c->Uc.alloc(c->compact_elems()));
  const GridDev G = c->grid();
  const double2* b = (const double2*)b_dev;
  // b's own Hermitian defect enters the gate's bound (herm_eval_kernel)
  TRY(ensure_hgate(c, 1));
  double* bstat = c->hgate.p + 1;  // scratch slots 1..3 (the statistic of field 0 lands in slot 1)
  CU(cudaMemsetAsync(bstat, 0, 3 * sizeof(double), st));
  pack_kernel<<<elem_grid(c, c->compact_elems()), 256, 0, st>>>(G, b, b, b, c->Uc.p, bstat, 1, (size_t)0);
  c->launches++;
  CU(cudaMemcpyAsync(c->bc.p, c->Uc.p, (size_t)c->Ky * c->Kx * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  TRY(c->bfull.alloc(c->full_elems()));
  CU(cudaMemcpyAsync(c->bfull.p, b, c->full_elems() * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  double d2 = 0.0;
  CU(cudaMemcpyAsync(&d2, bstat, sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaMemsetAsync(c->hgate.p, 0, 4 * sizeof(double), st));
  CU(cudaStreamSynchronize(st));
  c->bdef = std::sqrt(d2);
  c->version++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

int pswe_set_quadrature(pswe_ctx* c, int n_nodes, const double* s, const double* w) {
  if (!c || !s || !w) return set_err(PSWE_EINVAL, "null argument");
  if (n_nodes < 1 || n_nodes % 2 != 1) return set_err(PSWE_EINVAL, "need an odd number of nodes (2M+1), got %d", n_nodes);
  CU(cudaSetDevice(c->device));
  {
    // the same quadrature again (a caller that sets it before every
    // evaluation): keep the device arrays and the phase table
    std::vector<double> s2, w2;
    std::vector<int> k2;
    const int M = (n_nodes - 1) / 2;
    for (int i = 0; i < n_nodes; ++i)
      if (w[i] != 0.0) {
        s2.push_back(s[i]);
        w2.push_back(w[i]);
        k2.push_back(i - M);
      }
    if (c->quad_set && M == c->M && s2 == c->s_live && w2 == c->w_live && k2 == c->k_live) return PSWE_OK;
  }
  c->M = (n_nodes - 1) / 2;
  c->s_live.clear();
  c->w_live.clear();
  c->k_live.clear();
  for (int i = 0; i < n_nodes; ++i) {
    if (w[i] != 0.0) {
      c->s_live.push_back(s[i]);
      c->w_live.push_back(w[i]);
      c->k_live.push_back(i - c->M);
    }
  }
  if (c->s_live.empty()) return set_err(PSWE_EINVAL, "quadrature has no node with nonzero weight");
  const size_t P = c->s_live.size();
  TRY(c->s_dev.alloc(P));
  TRY(c->w_dev.alloc(P));
  c->ctab_q_valid = false;
  CU(cudaMemcpy(c->s_dev.p, c->s_live.data(), P * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(c->w_dev.p, c->w_live.data(), P * sizeof(double), cudaMemcpyHostToDevice));
  c->quad_set = true;
  c->version++;
  return PSWE_OK;
}

int pswe_set_propagator(pswe_ctx* c, int kind, double Lambda, int n_poly, const double* a) {
  if (!c) return set_err(PSWE_EINVAL, "null context");
  if (kind != 0 && kind != 1) return set_err(PSWE_EINVAL, "unknown propagator kind %d", kind);
  CU(cudaSetDevice(c->device));
  if (kind == 1) {
    if (!(Lambda >= 0)) return set_err(PSWE_EINVAL, "Lambda must be nonnegative, got %g", Lambda);
    if (n_poly < 1) return set_err(PSWE_EINVAL, "n_poly must be at least 1, got %d", n_poly);
    if (!a) return set_err(PSWE_EINVAL, "Chebyshev route needs n_poly + 1 coefficients");
    TRY(c->a_dev.alloc((size_t)n_poly + 1));
    CU(cudaMemcpy(c->a_dev.p, a, ((size_t)n_poly + 1) * sizeof(double), cudaMemcpyHostToDevice));
  }
  c->kind = kind;
  c->Lambda = Lambda;
  c->n_poly = n_poly;
  c->version++;
  return PSWE_OK;
}

int pswe_compact_shape(const pswe_ctx* c, int* Ky, int* Kx) {
  if (!c || !Ky || !Kx) return set_err(PSWE_EINVAL, "null argument");
  *Ky = c->Ky;
  *Kx = c->Kx;
  return PSWE_OK;
}

int pswe_pack(pswe_ctx* c, const double* u, const double* v, const double* e, double* Uc, void* stream) {
  if (!c || !u || !v || !e || !Uc) return set_err(PSWE_EINVAL, "null argument");
  CU(cudaSetDevice(c->device));
  pack_kernel<<<elem_grid(c, c->compact_elems()), 256, 0, (cudaStream_t)stream>>>(
      c->grid(), (const double2*)u, (const double2*)v, (const double2*)e, (double2*)Uc, nullptr, 1, (size_t)0);
  c->launches++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

int pswe_unpack(pswe_ctx* c, const double* Uc, double* u, double* v, double* e, void* stream) {
  if (!c || !u || !v || !e || !Uc) return set_err(PSWE_EINVAL, "null argument");
  CU(cudaSetDevice(c->device));
  unpack_kernel<<<elem_grid(c, c->full_elems()), 256, 0, (cudaStream_t)stream>>>(
      c->grid(), (const double2*)Uc, (double2*)u, (double2*)v, (double2*)e, 1, (size_t)0, no_gate());
  c->launches++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

int pswe_averaged_tendency_compact(pswe_ctx* c, const double* Uc, double* Ac, void* stream) {
  if (!c || !Uc || !Ac) return set_err(PSWE_EINVAL, "null argument");
  if (!c->quad_set) return set_err(PSWE_ESTATE, "no quadrature set (pswe_set_quadrature)");
  TRY(check_nodes(c));
  CU(cudaSetDevice(c->device));
  return rhs_compact(c, quad_phases(c), (const double2*)Uc, (double2*)Ac,
                     (cudaStream_t)stream);
}

// full layout in, with the gate: pack (+ statistics), evaluation over the
// nodes (s_dev, P) with the gate's verdict, unpack, synchronise, and the
// exact check when flagged (node-wrapped message when `k` is given)
static int copy_band(pswe_ctx* c, int dir, double* const* dst, const double* const* src, int nfields,
                     cudaStream_t st);
struct ConstPtr3 {
  const double* p[3];
  operator const double* const*() const { return p; }
};
static ConstPtr3 f3c(const double* a, const double* b, const double* e) { return ConstPtr3{{a, b, e}}; }

static int gated_rhs(pswe_ctx* c, const double* u, const double* v, const double* e, double* du, double* dv,
                     double* de, const PhaseSet& ps, const std::vector<double>& s_host, const std::vector<int>* k,
                     cudaStream_t st, double* const* host3 = nullptr) {
  CU(cudaSetDevice(c->device));
  TRY(ensure_compact(c));
  TRY(ensure_hgate(c, ps.P));
  CU(cudaMemsetAsync(c->flags.p, 0, sizeof(int), st));
  pack_kernel<<<elem_grid(c, c->compact_elems()), 256, 0, st>>>(c->grid(), (const double2*)u, (const double2*)v,
                                                               (const double2*)e, c->Uc.p, c->hgate.p, 1,
                                                               (size_t)0);
  c->launches++;
  CU(cudaGetLastError());
  TRY(rhs_compact(c, ps, c->Uc.p, c->Ac.p, st, true));
  unpack_kernel<<<elem_grid(c, c->full_elems()), 256, 0, st>>>(c->grid(), (const double2*)c->Ac.p, (double2*)du,
                                                              (double2*)dv, (double2*)de, 1, (size_t)0,
                                                              hgate_of(c, ps.P, HERM_BIT_RHS));
  c->launches++;
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(c->flags_host, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  // the drop-in call's band download joins the same synchronisation (the
  // exact gate, when the bound cannot decide, only validates the result)
  if (host3) TRY(copy_band(c, 1, host3, f3c(du, dv, de), 3, st));
  CU(cudaStreamSynchronize(st));
  if (*c->flags_host & (1 << HERM_BIT_RHS)) return exact_gate(c, ps.s, s_host, k, f3(u, v, e), st);
  return PSWE_OK;
}

int pswe_averaged_tendency(pswe_ctx* c, const double* u, const double* v, const double* e, double* du,
                           double* dv, double* de, void* stream) {
  if (!c || !u || !v || !e || !du || !dv || !de) return set_err(PSWE_EINVAL, "null argument");
  if (!c->quad_set) return set_err(PSWE_ESTATE, "no quadrature set (pswe_set_quadrature)");
  TRY(check_nodes(c));
  return gated_rhs(c, u, v, e, du, dv, de, quad_phases(c), c->s_live, &c->k_live, (cudaStream_t)stream);
}

int pswe_averaged_tendency_band_d2h(pswe_ctx* c, const double* u, const double* v, const double* e, double* du,
                                    double* dv, double* de, double* const* host3, void* stream) {
  if (!c || !u || !v || !e || !du || !dv || !de || !host3) return set_err(PSWE_EINVAL, "null argument");
  for (int f = 0; f < 3; ++f)
    if (!host3[f]) return set_err(PSWE_EINVAL, "null host buffer");
  if (!c->quad_set) return set_err(PSWE_ESTATE, "no quadrature set (pswe_set_quadrature)");
  TRY(check_nodes(c));
  return gated_rhs(c, u, v, e, du, dv, de, quad_phases(c), c->s_live, &c->k_live, (cudaStream_t)stream, host3);
}

int pswe_apply_nonlinear(pswe_ctx* c, const double* u, const double* v, const double* e, double* du, double* dv,
                         double* de, void* stream) {
  if (!c || !u || !v || !e || !du || !dv || !de) return set_err(PSWE_EINVAL, "null argument");
  return gated_rhs(c, u, v, e, du, dv, de, zero_phases(c), c->zero_live, nullptr, (cudaStream_t)stream);
}

int pswe_apply_linear(pswe_ctx* c, const double* u, const double* v, const double* e, double* lu, double* lv,
                      double* le, void* stream) {
  if (!c || !u || !v || !e || !lu || !lv || !le) return set_err(PSWE_EINVAL, "null argument");
  CU(cudaSetDevice(c->device));
  linear_full_kernel<<<elem_grid(c, c->full_elems()), 256, 0, (cudaStream_t)stream>>>(c->grid(), f3(u, v, e),
                                                                                  f3w(lu, lv, le));
  c->launches++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

int pswe_propagate(pswe_ctx* c, double t, const double* u, const double* v, const double* e, double* ou, double* ov,
                   double* oe, void* stream) {
  if (!c || !u || !v || !e || !ou || !ov || !oe) return set_err(PSWE_EINVAL, "null argument");
  std::string msg;
  if (check_cheb(c, t, &msg) != PSWE_OK) return set_err(PSWE_EINVAL, "%s", msg.c_str());
  CU(cudaSetDevice(c->device));
  propagate_full_kernel<<<elem_grid(c, c->full_elems()), 256, 0, (cudaStream_t)stream>>>(c->grid(), c->prop(), t,
                                                                                     f3(u, v, e), f3w(ou, ov, oe));
  c->launches++;
  CU(cudaGetLastError());
  return PSWE_OK;
}

int pswe_ssprk3_step(pswe_ctx* c, double dt, const double* u, const double* v, const double* e, double* ou,
                     double* ov, double* oe, int* bad_stage, int* bad_field, void* stream) {
  if (!c || !u || !v || !e || !ou || !ov || !oe) return set_err(PSWE_EINVAL, "null argument");
  if (!c->quad_set) return set_err(PSWE_ESTATE, "no quadrature set (pswe_set_quadrature)");
  if (!(dt > 0)) return set_err(PSWE_EINVAL, "dt must be positive, got %g", dt);
  std::string msg;
  if (check_cheb(c, dt, &msg) != PSWE_OK) return set_err(PSWE_EINVAL, "%s", msg.c_str());
  TRY(check_nodes(c));
  CU(cudaSetDevice(c->device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n = c->full_elems();
  TRY(c->full_tmp.alloc(n * 18));
  Full3 in = f3(u, v, e);
  if (ou == u || ov == v || oe == e || ou == v || ou == e || ov == u || ov == e || oe == u || oe == v) {
    // in place: keep the input for the gate's exact check (the output overwrites it)
    double2* keep = c->full_tmp.p + 9 * n;
    CU(cudaMemcpyAsync(keep, u, n * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(keep + n, v, n * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(keep + 2 * n, e, n * sizeof(double2), cudaMemcpyDeviceToDevice, st));
    in = Full3{keep, keep + n, keep + 2 * n};
  }
  CU(cudaMemsetAsync(c->flags.p, 0, sizeof(int), st));
  TRY(step_impl(c, dt, in, f3w(ou, ov, oe), st));
  CU(cudaMemcpyAsync(c->flags_host, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  int stage = 0, field = -1;
  const int rc = *c->flags_host ? step_verdict(c, *c->flags_host, in, st, &stage, &field) : PSWE_OK;
  if (bad_stage) *bad_stage = stage;
  if (bad_field) *bad_field = field;
  return rc;
}

int pswe_run(pswe_ctx* c, double dt, int nsteps, double* u, double* v, double* e, int* bad_step, int* bad_stage,
             int* bad_field, void* stream) {
  if (!c || !u || !v || !e) return set_err(PSWE_EINVAL, "null argument");
  if (nsteps < 0) return set_err(PSWE_EINVAL, "nsteps must be nonnegative, got %d", nsteps);
  if (bad_step) *bad_step = 0;
  if (nsteps == 0) return PSWE_OK;
  if (!c->quad_set) return set_err(PSWE_ESTATE, "no quadrature set (pswe_set_quadrature)");
  if (!(dt > 0)) return set_err(PSWE_EINVAL, "dt must be positive, got %g", dt);
  std::string msg;
  if (check_cheb(c, dt, &msg) != PSWE_OK) return set_err(PSWE_EINVAL, "%s", msg.c_str());
  TRY(check_nodes(c));
  CU(cudaSetDevice(c->device));
  // the run executes on the context's own stream (capturable even when the
  // caller uses the legacy default stream), forked from / joined to `stream`
  cudaStream_t ust = (cudaStream_t)stream;
  cudaStream_t st = c->st_run;
  CU(cudaEventRecord(c->ev_run, ust));
  CU(cudaStreamWaitEvent(st, c->ev_run, 0));
  const size_t n = c->full_elems();
  TRY(c->full_tmp.alloc(n * 18));
  double2* A = c->full_tmp.p + 9 * n;   // state
  double2* B = c->full_tmp.p + 12 * n;  // step output
  double2* S = c->full_tmp.p + 15 * n;  // batch checkpoint
  const size_t bytes3 = 3 * n * sizeof(double2);
  CU(cudaMemcpyAsync(A, u, n * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  CU(cudaMemcpyAsync(A + n, v, n * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  CU(cudaMemcpyAsync(A + 2 * n, e, n * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  const Full3 Ain{A, A + n, A + 2 * n};
  const Full3w Bout{B, B + n, B + 2 * n};

  // one checked step: A -> B -> A; returns 100 (and fills the outputs) when
  // the step fails (non-finite stage or the Hermitian gate)
  int rc = PSWE_OK;
  auto checked_step = [&](int i) -> int {
    CU(cudaMemsetAsync(c->flags.p, 0, sizeof(int), st));
    TRY(step_impl(c, dt, Ain, Bout, st));
    CU(cudaMemcpyAsync(c->flags_host, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (*c->flags_host) {
      int stage = 0, field = -1;
      const int r = step_verdict(c, *c->flags_host, Ain, st, &stage, &field);
      if (r == PSWE_ENONFINITE || r == PSWE_EHERM) {
        if (bad_step) *bad_step = i;
        if (bad_stage) *bad_stage = stage;
        if (bad_field) *bad_field = field;
        rc = r;
        return 100;  // A still holds the state at the start of step i
      }
      if (r != PSWE_OK) return r;
    }
    CU(cudaMemcpyAsync(A, B, bytes3, cudaMemcpyDeviceToDevice, st));
    return 0;
  };

  // step 1 un-captured (allocates every buffer, builds the phase table)
  int i = 1;
  {
    const int r = checked_step(i);
    if (r == 100) goto done;
    if (r != PSWE_OK) return r;
    ++i;
  }
  // remaining steps: CUDA-graph replays of one step in batches, flags checked per batch
  if (i <= nsteps) {
    TRY(ensure_step_graph(c, dt, Ain, Bout, bytes3, st));
    const int batch = 16, m = STEP_GRAPH_MULTI;
    static const bool no_multi = getenv("PSWE_NO_MULTISTEP_GRAPH") != nullptr;  // A/B switch
    // building the eight-step graph costs about as much as 100 steps gain (C2: 24 steps 74 -> 86 us per
    // step with it, 7200 steps 57.2 -> 54.3): long runs only
    const bool multi = !no_multi && nsteps - i + 1 >= 512;
    if (multi) TRY(ensure_step_graph(c, dt, Ain, Bout, bytes3, st, m));
    while (i <= nsteps) {
      const int k = std::min(batch, nsteps - i + 1);
      CU(cudaMemcpyAsync(S, A, bytes3, cudaMemcpyDeviceToDevice, st));
      CU(cudaMemsetAsync(c->flags.p, 0, sizeof(int), st));
      int j = 0;
      if (multi)
        for (; j + m <= k; j += m) CU(cudaGraphLaunch(c->stepm_exec, st));  // m steps, A -> B -> ... -> A
      for (; j < k; ++j) CU(cudaGraphLaunch(c->step_exec, st));
      c->launches += (int64_t)k * c->step_graph_launches;
      for (int v = 0; v < PSWE_NUM_VARIANTS; ++v) c->variant[v] += (int64_t)k * c->graph_variant[v];
      CU(cudaMemcpyAsync(c->flags_host, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      if (*c->flags_host) {
        // replay the batch step by step from its checkpoint to find the failing step
        CU(cudaMemcpyAsync(A, S, bytes3, cudaMemcpyDeviceToDevice, st));
        for (int j = 0; j < k; ++j) {
          const int r = checked_step(i + j);
          if (r == 100) goto done;
          if (r != PSWE_OK) return r;
        }
      }
      i += k;
    }
  }
done:
  CU(cudaMemcpyAsync(u, A, n * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  CU(cudaMemcpyAsync(v, A + n, n * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  CU(cudaMemcpyAsync(e, A + 2 * n, n * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  CU(cudaEventRecord(c->ev_run, st));
  CU(cudaStreamWaitEvent(ust, c->ev_run, 0));
  return rc;
}

// ---------------------------------------------------------------- window batch
int pswe_set_window_batch(pswe_ctx* c, int W, const int* n_nodes, const double* s, const double* w) {
  if (!c || !n_nodes || !s || !w) return set_err(PSWE_EINVAL, "null argument");
  if (W < 1) return set_err(PSWE_EINVAL, "need at least one window, got %d", W);
  CU(cudaSetDevice(c->device));
  std::vector<double> bs, bw;
  std::vector<int> bwin, bk;
  size_t off = 0;
  for (int i = 0; i < W; ++i) {
    const int n = n_nodes[i];
    if (n < 1 || n % 2 != 1) return set_err(PSWE_EINVAL, "window %d: need an odd number of nodes (2M+1), got %d", i, n);
    const int M = (n - 1) / 2;
    int live = 0;
    for (int k = 0; k < n; ++k)
      if (w[off + k] != 0.0) {
        bs.push_back(s[off + k]);
        bw.push_back(w[off + k]);
        bwin.push_back(i);
        bk.push_back(k - M);
        ++live;
      }
    if (!live) return set_err(PSWE_EINVAL, "window %d: quadrature has no node with nonzero weight", i);
    off += n;
  }
  if (c->bW == W && bs == c->b_s && bw == c->b_w && bwin == c->b_win) return PSWE_OK;
  const size_t P = bs.size();
  TRY(c->bs_dev.alloc(P));
  TRY(c->bw_dev.alloc(P));
  TRY(c->bwin_dev.alloc(P));
  CU(cudaMemcpy(c->bs_dev.p, bs.data(), P * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(c->bw_dev.p, bw.data(), P * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(c->bwin_dev.p, bwin.data(), P * sizeof(int), cudaMemcpyHostToDevice));
  c->bW = W;
  c->b_s = bs;
  c->b_w = bw;
  c->b_win = bwin;
  c->b_k = bk;
  c->ctab_b_valid = false;
  c->version++;
  return PSWE_OK;
}

static int check_batch_nodes(const pswe_ctx* c) {
  std::string msg;
  for (size_t i = 0; i < c->b_s.size(); ++i)
    if (check_cheb(c, c->b_s[i], &msg) != PSWE_OK)
      return set_err(PSWE_EINVAL, "window %d: averaging node k = %d (s = %.6g s) failed: %s", c->b_win[i],
                     c->b_k[i], c->b_s[i], msg.c_str());
  return PSWE_OK;
}

int pswe_window_batch_tendency(pswe_ctx* c, const double* Uc, double* Ac, void* stream) {
  if (!c || !Uc || !Ac) return set_err(PSWE_EINVAL, "null argument");
  if (c->bW < 1) return set_err(PSWE_ESTATE, "no window batch set (pswe_set_window_batch)");
  TRY(check_batch_nodes(c));
  CU(cudaSetDevice(c->device));
  return rhs_compact(c, batch_phases(c), (const double2*)Uc, (double2*)Ac, (cudaStream_t)stream);
}

// capture "batched step A -> B, copy B -> A" (cached per dt / configuration)
static int ensure_batch_graph(pswe_ctx* c, double dt, Full3 Ain, Full3w Bout, size_t bytes, cudaStream_t st) {
  if (c->bstep_exec && c->bgraph_dt == dt && c->bgraph_version == c->version && c->bgraph_gen == g_alloc_gen)
    return PSWE_OK;
  if (c->bstep_exec) cudaGraphExecDestroy(c->bstep_exec);
  c->bstep_exec = nullptr;
  const bool prof = c->prof;
  c->prof = false;
  const int64_t l0 = c->launches;
  int64_t v0[PSWE_NUM_VARIANTS];
  std::copy(c->variant, c->variant + PSWE_NUM_VARIANTS, v0);
  CU(cudaStreamSynchronize(st));
  std::lock_guard<std::recursive_mutex> lock(g_capture_mutex);
  CU(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
  int rc = step_impl_w(c, batch_phases(c), dt, Ain, Bout, c->b_full.p, c->b_Uc.p, c->b_Ac.p, st);
  cudaError_t ce = cudaMemcpyAsync((void*)Ain.u, Bout.u, bytes, cudaMemcpyDeviceToDevice, st);
  cudaGraph_t g = nullptr;
  cudaError_t ee = cudaStreamEndCapture(st, &g);
  c->prof = prof;
  if (rc != PSWE_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  CU(ce);
  CU(ee);
  cudaError_t ie = cudaGraphInstantiate(&c->bstep_exec, g, 0);
  cudaGraphDestroy(g);
  CU(ie);
  c->bstep_graph_launches = c->launches - l0;
  c->launches = l0;
  for (int i = 0; i < PSWE_NUM_VARIANTS; ++i) {
    c->bgraph_variant[i] = c->variant[i] - v0[i];
    c->variant[i] = v0[i];
  }
  c->bgraph_dt = dt;
  c->bgraph_version = c->version;
  c->bgraph_gen = g_alloc_gen;
  return PSWE_OK;
}

int pswe_window_batch_run(pswe_ctx* c, double dt, int nsteps, double* U, int* bad_step, void* stream) {
  if (!c || !U) return set_err(PSWE_EINVAL, "null argument");
  if (bad_step) *bad_step = 0;
  if (nsteps < 0) return set_err(PSWE_EINVAL, "nsteps must be nonnegative, got %d", nsteps);
  if (nsteps == 0) return PSWE_OK;
  if (c->bW < 1) return set_err(PSWE_ESTATE, "no window batch set (pswe_set_window_batch)");
  if (!(dt > 0)) return set_err(PSWE_EINVAL, "dt must be positive, got %g", dt);
  std::string msg;
  if (check_cheb(c, dt, &msg) != PSWE_OK) return set_err(PSWE_EINVAL, "%s", msg.c_str());
  TRY(check_batch_nodes(c));
  CU(cudaSetDevice(c->device));
  cudaStream_t ust = (cudaStream_t)stream;
  cudaStream_t st = c->st_run;
  CU(cudaEventRecord(c->ev_run, ust));
  CU(cudaStreamWaitEvent(st, c->ev_run, 0));
  const int W = c->bW;
  const size_t n = c->full_elems(), sw = (size_t)3 * W * n;  // one batch state: W x 3 fields
  TRY(c->b_full.alloc(6 * sw));
  TRY(c->b_Uc.alloc((size_t)W * c->compact_elems()));
  TRY(c->b_Ac.alloc((size_t)W * c->compact_elems()));
  double2* A = c->b_full.p + 3 * sw;
  double2* B = c->b_full.p + 4 * sw;
  double2* S = c->b_full.p + 5 * sw;
  const size_t bytes = sw * sizeof(double2);
  CU(cudaMemcpyAsync(A, U, bytes, cudaMemcpyDeviceToDevice, st));
  const Full3 Ain{A, A + n, A + 2 * n};
  const Full3w Bout{B, B + n, B + 2 * n};
  int rc = PSWE_OK;
  // any flag (a non-finite stage or the Hermitian gate) stops the batch at
  // the start of the flagged step; the caller re-runs the windows one by
  // one for the reference's per-window error
  auto flagged = [&](int i) {
    if (bad_step) *bad_step = i;
    rc = set_err(PSWE_ENONFINITE, "window batch flagged at step %d", i);
  };
  int i = 1;
  CU(cudaMemsetAsync(c->flags.p, 0, sizeof(int), st));
  TRY(step_impl_w(c, batch_phases(c), dt, Ain, Bout, c->b_full.p, c->b_Uc.p, c->b_Ac.p, st));
  CU(cudaMemcpyAsync(c->flags_host, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (*c->flags_host) {
    flagged(1);
    goto done;
  }
  CU(cudaMemcpyAsync(A, B, bytes, cudaMemcpyDeviceToDevice, st));
  ++i;
  if (i <= nsteps) {
    TRY(ensure_batch_graph(c, dt, Ain, Bout, bytes, st));
    const int batch = 16;
    while (i <= nsteps) {
      const int k = std::min(batch, nsteps - i + 1);
      CU(cudaMemcpyAsync(S, A, bytes, cudaMemcpyDeviceToDevice, st));
      CU(cudaMemsetAsync(c->flags.p, 0, sizeof(int), st));
      for (int j = 0; j < k; ++j) CU(cudaGraphLaunch(c->bstep_exec, st));
      c->launches += (int64_t)k * c->bstep_graph_launches;
      for (int v = 0; v < PSWE_NUM_VARIANTS; ++v) c->variant[v] += (int64_t)k * c->bgraph_variant[v];
      CU(cudaMemcpyAsync(c->flags_host, c->flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      CU(cudaStreamSynchronize(st));
      if (*c->flags_host) {
        CU(cudaMemcpyAsync(A, S, bytes, cudaMemcpyDeviceToDevice, st));
        flagged(i);
        goto done;
      }
      i += k;
    }
  }
done:
  CU(cudaMemcpyAsync(U, A, bytes, cudaMemcpyDeviceToDevice, st));
  CU(cudaEventRecord(c->ev_run, st));
  CU(cudaStreamWaitEvent(ust, c->ev_run, 0));
  return rc;
}

double pswe_max_frequency(const pswe_ctx* c) { return c ? c->lam_max : 0.0; }

int64_t pswe_launch_count(const pswe_ctx* c) { return c ? c->launches : 0; }

int pswe_debug_check_guards(int64_t* guarded, int64_t* damaged) {
  if (!guarded || !damaged) return set_err(PSWE_EINVAL, "null argument");
  *guarded = 0;
  *damaged = 0;
  if (!guard_enabled()) return PSWE_OK;
  CU(cudaDeviceSynchronize());
  std::lock_guard<std::mutex> gl(g_guard_mutex);
  int64_t bad = g_guard_hits;
  for (const GuardedBlock& b : g_guarded) bad += guard_damage(b);
  *guarded = (int64_t)g_guarded.size();
  *damaged = bad;
  return PSWE_OK;
}

int pswe_variant_launches(const pswe_ctx* c, int64_t* counts, int n) {
  if (!c || !counts) return set_err(PSWE_EINVAL, "null argument");
  for (int i = 0; i < n && i < PSWE_NUM_VARIANTS; ++i) counts[i] = c->variant[i];
  return PSWE_OK;
}

// full 2-D C2R of (u, v, eta, b) with row partials of the diagnostics; phys
// (optional) receives the physical u, v, eta
static int physical_fields(pswe_ctx* c, const double* u, const double* v, const double* e, double* phys,
                           cudaStream_t st) {
  CU(cudaSetDevice(c->device));
  if (!c->bfull.p) {  // flat bottom
    TRY(c->bfull.alloc(c->full_elems()));
    CU(cudaMemsetAsync(c->bfull.p, 0, c->full_elems() * sizeof(double2), st));
  }
  TRY(c->diag_cols.alloc((size_t)4 * (c->ny / 2 + 1) * c->nx));
  TRY(c->diag_part.alloc((size_t)3 * c->nx));
  const double2 *U = (const double2*)u, *V = (const double2*)v, *E = (const double2*)e;
  if (c->gen) {
    const size_t sc = (size_t)2 * c->nx * sizeof(double2), sr = (size_t)4 * c->ny * sizeof(double2);
    CU(smem_attr(gen_diag_cols_kernel, sc, c->device));
    CU(smem_attr(gen_diag_rows_kernel, sr, c->device));
    gen_diag_cols_kernel<<<4 * (c->ny / 2 + 1), gen_threads(c->nx), sc, st>>>(c->grid(), U, V, E, c->bfull.p,
                                                                        c->diag_cols.p, c->plx);
    gen_diag_rows_kernel<<<c->nx, gen_threads(c->ny), sr, st>>>(c->grid(), c->diag_cols.p, c->H, c->g, c->diag_part.p,
                                                          phys, c->ply);
    c->launches += 2;
    CU(cudaGetLastError());
    return PSWE_OK;
  }
  int rc = PSWE_EUNSUPPORTED;
  switch (c->nx) {
    case 8: rc = launch_diag_cols<8>(c, U, V, E, c->bfull.p, st); break;
    case 16: rc = launch_diag_cols<16>(c, U, V, E, c->bfull.p, st); break;
    case 32: rc = launch_diag_cols<32>(c, U, V, E, c->bfull.p, st); break;
    case 64: rc = launch_diag_cols<64>(c, U, V, E, c->bfull.p, st); break;
    case 128: rc = launch_diag_cols<128>(c, U, V, E, c->bfull.p, st); break;
    case 256: rc = launch_diag_cols<256>(c, U, V, E, c->bfull.p, st); break;
    case 512: rc = launch_diag_cols<512>(c, U, V, E, c->bfull.p, st); break;
  }
  if (rc != PSWE_OK) return rc == PSWE_EUNSUPPORTED ? set_err(rc, "unsupported nx = %d", c->nx) : rc;
  rc = PSWE_EUNSUPPORTED;
  switch (c->ny) {
    case 8: rc = launch_diag_rows<8>(c, phys, st); break;
    case 16: rc = launch_diag_rows<16>(c, phys, st); break;
    case 32: rc = launch_diag_rows<32>(c, phys, st); break;
    case 64: rc = launch_diag_rows<64>(c, phys, st); break;
    case 128: rc = launch_diag_rows<128>(c, phys, st); break;
    case 256: rc = launch_diag_rows<256>(c, phys, st); break;
    case 512: rc = launch_diag_rows<512>(c, phys, st); break;
  }
  if (rc != PSWE_OK) return rc == PSWE_EUNSUPPORTED ? set_err(rc, "unsupported ny = %d", c->ny) : rc;
  return PSWE_OK;
}

int pswe_to_physical(pswe_ctx* c, const double* u, const double* v, const double* e, double* phys,
                                void* stream) {
  if (!c || !u || !v || !e || !phys) return set_err(PSWE_EINVAL, "null argument");
  CU(cudaSetDevice(c->device));
  TRY(full_gate(c, f3(u, v, e), false, (cudaStream_t)stream));
  return physical_fields(c, u, v, e, phys, (cudaStream_t)stream);
}

int pswe_copy_band(pswe_ctx* c, int dir, double* const* dst, const double* const* src, int nfields,
                   void* stream) {
  if (!c || !dst || !src || nfields < 0) return set_err(PSWE_EINVAL, "null argument");
  if (dir != 0 && dir != 1) return set_err(PSWE_EINVAL, "dir must be 0 (host to device) or 1 (device to host)");
  CU(cudaSetDevice(c->device));
  return copy_band(c, dir, dst, src, nfields, (cudaStream_t)stream);
}

static int copy_band(pswe_ctx* c, int dir, double* const* dst, const double* const* src, int nfields,
                     cudaStream_t stream) {
  const cudaMemcpyKind kind = dir == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
  const size_t pitch = (size_t)c->ny * 2 * sizeof(double);
  // rows |wx| <= kxm and columns |wy| <= kym: two row blocks x two column blocks
  const int r0[2] = {0, c->nx - c->kxm}, nr[2] = {c->kxm + 1, c->kxm};
  const int c0[2] = {0, c->ny - c->kym}, nc[2] = {c->kym + 1, c->kym};
  for (int f = 0; f < nfields; ++f) {
    if (!dst[f] || !src[f]) return set_err(PSWE_EINVAL, "null field pointer");
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) {
        const size_t off = ((size_t)r0[a] * c->ny + c0[b]) * 2;
        CU(cudaMemcpy2DAsync(dst[f] + off, pitch, src[f] + off, pitch, (size_t)nc[b] * 2 * sizeof(double), nr[a],
                             kind, (cudaStream_t)stream));
      }
  }
  return PSWE_OK;
}

int pswe_diagnostics(pswe_ctx* c, const double* u, const double* v, const double* e, double* out3,
                                void* stream) {
  if (!c || !u || !v || !e || !out3) return set_err(PSWE_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  CU(cudaSetDevice(c->device));
  TRY(full_gate(c, f3(u, v, e), true, st));
  TRY(physical_fields(c, u, v, e, nullptr, st));
  std::vector<double> part((size_t)3 * c->nx);
  CU(cudaMemcpyAsync(part.data(), c->diag_part.p, part.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  double se = 0.0, sm = 0.0, vmax = 0.0;
  for (int x = 0; x < c->nx; ++x) {  // rows in order: deterministic
    se += part[3 * (size_t)x];
    sm += part[3 * (size_t)x + 1];
    vmax = std::max(vmax, part[3 * (size_t)x + 2]);
  }
  const double area = (c->Lx / c->nx) * (c->Ly / c->ny);  // cell_area = dx dy (grid.py:58-59)
  out3[0] = se * area;
  out3[1] = sm * area;
  out3[2] = std::sqrt(vmax);
  return PSWE_OK;
}

int pswe_profile_enable(pswe_ctx* c, int enable) {
  if (!c) return set_err(PSWE_EINVAL, "null context");
  c->prof = enable != 0;
  return PSWE_OK;
}

int pswe_profile_read(pswe_ctx* c, double* ms, int64_t* launches, int n) {
  if (!c) return set_err(PSWE_EINVAL, "null context");
  CU(cudaSetDevice(c->device));
  std::vector<double> acc(PSWE_NUM_KERNEL_CLASSES, 0.0);
  std::vector<int64_t> cnt(PSWE_NUM_KERNEL_CLASSES, 0);
  for (const auto& r : c->recs) {
    CU(cudaEventSynchronize(r.b));
    float t = 0.f;
    CU(cudaEventElapsedTime(&t, r.a, r.b));
    acc[r.cls] += t;
    cnt[r.cls] += 1;
  }
  c->recs.clear();
  c->ev_used = 0;
  for (int i = 0; i < n && i < PSWE_NUM_KERNEL_CLASSES; ++i) {
    if (ms) ms[i] = acc[i];
    if (launches) launches[i] = cnt[i];
  }
  return PSWE_OK;
}

int pswe_set_chunk_bytes(pswe_ctx* c, size_t bytes) {
  if (!c) return set_err(PSWE_EINVAL, "null context");
  c->chunk_bytes = std::max<size_t>(bytes, 1);
  c->version++;
  return PSWE_OK;
}

int pswe_set_lanes(pswe_ctx* c, int lanes) {
  if (!c) return set_err(PSWE_EINVAL, "null context");
  if (lanes < 1 || lanes > pswe_ctx::MAX_LANES)
    return set_err(PSWE_EINVAL, "lanes must be in [1, %d], got %d", pswe_ctx::MAX_LANES, lanes);
  c->n_lanes = lanes;
  c->version++;
  return PSWE_OK;
}

int pswe_get_lanes(const pswe_ctx* c) { return c ? c->n_lanes : 0; }

}  // extern "C"

// libtopo: C-ABI implementation of the matrix-free SIMP hot path on B200.
// See include/topo.h for the contract and DESIGN.md for the design.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <tuple>
#include <utility>

#include "../../include/topo.h"
#include "common.cuh"
#include "kernels.cuh"
#include "matvec_wht.cuh"
#include "mg.cuh"
#include "filter25.cuh"
#include "host_transport.h"
#include <chrono>

namespace topo {
void build_element_stiffness(double nu, double* ke);  // ke_host.cpp
bool wht_constants(const double* ke, double out[8], double tol);
void mg_child_weights(double w[8][8][8]);            // mg_host.cpp
void mg_galerkin_tables(const double* ke, double* tab8, double* tab64, double* diag8);
}
using namespace topo;

// ---------------------------------------------------------------------------
// Minimal NCCL binding, resolved with dlopen at init time (NCCL mode only),
// so the library loads on machines without libnccl.
// ---------------------------------------------------------------------------
namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { ncclFloat32 = 7, ncclFloat64 = 8 };
enum { ncclSum = 0, ncclMax = 2 };
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;   // optional
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;                          // optional
  bool load(std::string& err) {
    if (h) return true;
    const char* cands[] = {"libnccl.so.2", "libnccl.so",
                           "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
    for (const char* c : cands) {
      h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) { err = "cannot dlopen libnccl.so.2"; return false; }
#define LD(name, sym) name = reinterpret_cast<decltype(name)>(dlsym(h, sym)); if (!name) { err = "missing " sym; return false; }
    LD(GetUniqueId, "ncclGetUniqueId");
    LD(CommInitRank, "ncclCommInitRank");
    LD(CommDestroy, "ncclCommDestroy");
    LD(AllReduce, "ncclAllReduce");
    LD(Send, "ncclSend");
    LD(Recv, "ncclRecv");
    LD(GroupStart, "ncclGroupStart");
    LD(GroupEnd, "ncclGroupEnd");
    LD(GetErrorString, "ncclGetErrorString");
#undef LD
    CommGetAsyncError = reinterpret_cast<decltype(CommGetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
    CommAbort = reinterpret_cast<decltype(CommAbort)>(dlsym(h, "ncclCommAbort"));
    return true;
  }
};
NcclApi g_nccl;


struct TopoError {
  int code;
  std::string msg;
};
}  // namespace

// ---------------------------------------------------------------------------
// Context
// ---------------------------------------------------------------------------
// One distributed coarse level of a slab (x-slabs, levels 1 .. mg_dl; DESIGN.md
// §6): the level's vectors in the WHOLE level's layout (a node plane has the same
// offset on every rank), of which this slab computes its owned node planes
// [oa, ob) and keeps the ghost planes oa - 1 and ob current by exchanges.  Slab 0
// (every slab with one slab per process) aliases ctx->mg[l]'s buffers; the other
// slabs of a loopback context own theirs.  The level operators (D^-1, stencil,
// masks, the fine moduli of level 1) are the replicated setup's.
struct DLv {
  void *x = nullptr, *b = nullptr, *t = nullptr, *kx = nullptr, *kv = nullptr, *Y = nullptr;
  double* kc = nullptr;   // K-cycle scalars of this slab (8)
  int oa = 0, ob = 0;
  bool own = false;       // buffers allocated here (freed with the context)
};

struct Slab {
  Geo g{};
  std::vector<DLv> dlv;   // [0, mg_dl]: distributed levels (index 0 unused)
  // node vectors: 3*ncomp doubles each (SoA)
  double *u = nullptr, *r = nullptr, *p0 = nullptr, *p1 = nullptr, *q = nullptr, *f = nullptr,
         *w = nullptr, *z = nullptr;   // z: multigrid preconditioned residual V(r)
  float* res32 = nullptr;              // fp32 multigrid: fine residual for the restriction
  float* z32 = nullptr;                // fp32 multigrid: prolongation output z (post-smoothing input)
  float* w32 = nullptr;                // fp32 multigrid (one slab): the V-cycle output w (PCG matvec input)
  float *r32 = nullptr, *q32 = nullptr;  // fp32 Krylov residual and q = K p of the MG-PCG
  double *pw0 = nullptr, *pw0_b = nullptr;   // multigrid level-0 power vector (+ snapshot)
  // OC frozen set: per-block active counts / offsets and the compacted (x, A, dv~)
  unsigned *oc_counts = nullptr, *oc_offs = nullptr;
  double *oc_cx = nullptr, *oc_cA = nullptr, *oc_cdv = nullptr;      // stage-1 active set
  double *oc_cx2 = nullptr, *oc_cA2 = nullptr, *oc_cdv2 = nullptr;   // stage-2 active set
  long long* oc_n1 = nullptr;                                          // stage-1 active count (device)
  double* invd = nullptr;    // per node (1 component): 1/(kd sum E)
  uint8_t* fixm = nullptr;   // per node: bit c = DOF c fixed
  // element arrays: nelloc each
  double *E = nullptr, *x = nullptr, *xphys = nullptr, *dc = nullptr, *dcf = nullptr,
         *dvf = nullptr, *dv = nullptr, *hs = nullptr, *ihs = nullptr, *ce = nullptr, *xnew = nullptr,
         *oca = nullptr;   // OC: A = x sqrt(max(0, -dc~/dv~))
  double* vpad = nullptr;  // filter operand, zero-padded by R in y and z (FiltPad)
  FiltPad fp{};
  uint8_t* passive = nullptr;
  double* partials = nullptr;
  unsigned int* counter = nullptr;
  DevState* st = nullptr;
  double* stage = nullptr;   // staging for layout transforms
  size_t stage_n = 0;
  double *u_b = nullptr, *x_b = nullptr, *xphys_b = nullptr;   // snapshot buffers
  // TMA descriptors of the matvec operands (built at init; pointers never change)
  CUtensorMap m_r, m_u, m_w, m_p0, m_p1, m_invd, m_E, m_z, m_q;
  CUtensorMap m_z32;   // fp32 z (multigrid, mg_fp32)
  CUtensorMap m_w32;   // fp32 w (multigrid, mg_fp32, one slab)
  CUtensorMap m_r32;   // fp32 r (fp32 Krylov vectors)
  CUtensorMap m_vpad;  // padded filter operand (k_filt25), box (32+2R) x (32+2R) x 1
};

// One coarse multigrid level (l >= 1, M1-M6).
struct MgLevel {
  LvGeo L{};
  // vectors and level operators in the preconditioner's precision (double, or
  // float with topo_params.mg_fp32; typed access through mgp<T>)
  void *x = nullptr, *b = nullptr, *t = nullptr, *invd = nullptr;   // 3*ncomp each
  double* K = nullptr;          // stored element matrices [576][nel] (fp64: setup only)
  void* S = nullptr;            // symmetric 27-point block stencil [126][ncomp] (stored, smoothed levels)
  void* Y = nullptr;            // level 1 matrix-free: per-element outputs [24][nel]
  void* pw = nullptr;           // power-step vector kept for the next design's warm start
  void* pw_b = nullptr;         // its snapshot copy
  void *kx = nullptr, *kv = nullptr;   // K-cycle (M8): x1 and A x1 of the first FCG step
  uint8_t* fixm = nullptr;      // per node: bit c = DOF c fixed
  std::vector<uint8_t> hfix;    // host copy, external node order
  bool stored = false;
};

struct topo_ctx {
  topo_params prm{};
  int mode = TOPO_DIST_SINGLE, rank = 0, world = 1, device = 0;
  std::vector<Slab> slabs;
  cudaStream_t stream = nullptr, own_stream = nullptr;
  ncclComm_t comm = nullptr;
  HostTransport* ht = nullptr;          // TOPO_DIST_HOST: shared-memory transport
  std::deque<HostOp> hops;              // host nodes' userData (alive as long as the graphs)
  double comm_timeout_s = 300.0;        // NCCL / host transport: give up (TOPO_ENCCL) after this long
  double ke[576];
  double kd = 0.0;
  WhtK wht{};
  WhtK wht1{};              // level-1 multigrid: block constants scaled by Lambda^-1 . Lambda^-1
  WhtKT<float> wht1f{}, whtf{};
  int tz = 8;               // z extent of a matvec CTA (threads 32 x tz)
  std::vector<int4> st_off;
  std::vector<double> st_w;
  std::vector<int> st_poff;   // filter offsets in the padded layout (FiltPad)
  int R = 0;
  unsigned f25_attr_mask = 0;   // k_filt25 dynamic-smem opt-in done (bit per device x mode)
  bool tc_attr_set = false;     // k_dgemm_nt64_tc dynamic-smem opt-in done (this context's device)
  long long n_design = 0;   // global design-element count
  double bb = 0.0;          // ||f_free||^2
  // state flags
  bool has_solid = false;   // some element is passive solid (mask value 2, R27)
  bool has_E = false, has_u = false, has_sens = false, has_dcf = false, has_dvf = false;
  // pinned mirror of slab 0's DevState
  DevState* hstate = nullptr;
  // CUDA graphs (PCG batch, OC batch)
  cudaGraphExec_t cg_exec[2] = {nullptr, nullptr};   // PCG batch graphs: [0] Jacobi, [1] multigrid
  int cg_batch = 0;
  long long cg_batch_launches[2] = {0, 0};
  bool cg_profiled_graph[2] = {false, false};
  cudaGraphExec_t oc_exec = nullptr, oc_exec_c = nullptr, oc_exec_c2 = nullptr;   // full / stage-1 / stage-2 OC batches
  int oc_batch = 4;                  // passes (3 bisection levels each) per OC graph launch
  long long oc_batch_launches = 0;
  // profiling
  bool profile = false;
  cudaEvent_t pe0 = nullptr, pe1 = nullptr;
  double prof_ms = 0.0;
  long long prof_n = 0;
  // multigrid V-cycle fine matvecs (pre-smoothing kPre=3, post-smoothing kEpi=1):
  // pe[0..1] and pe[2..3] bracket them in the first iteration of each batch
  cudaEvent_t pe[4] = {};
  double prof_ms_k[3] = {0, 0, 0};
  long long prof_n_k[3] = {0, 0, 0};
  bool prof_capture = false;   // set while enqueueing the profiled iteration
  // phase events
  cudaEvent_t ev[8] = {};
  cudaEvent_t ev_setup[2] = {};   // brackets the multigrid setup of a solve
  topo_timings tim{};
  long long launches = 0;
  long long host_bytes = 0;   // field bytes copied host <-> device by the library (host-pointer calls)
  std::string err;
  size_t dev_bytes = 0;
  bool debug = false;        // TOPO_DEBUG_SYNC=1: no graphs, sync + check after every kernel
  bool snap_has_u = false, has_snap = false;
  int sticky = TOPO_OK;
  // geometric multigrid (level 0 = the fine slab; mg[0] unused)
  bool mg_on = false, mg_ready = false;
  bool mg_f32 = false;               // levels >= 1 in fp32 (topo_params.mg_fp32)
  bool mg_f32_b = false;             // ... in the snapshot
  double mg_theta = 1.6, mg_theta_b = 1.6;   // smoother theta in use (cut after a breakdown) (+ snapshot)
  std::vector<MgLevel> mg;
  double *mg_tab8 = nullptr, *mg_tab64 = nullptr, *mg_A0 = nullptr;
  float* mg_A32 = nullptr;           // fp32 copy of the coarsest inverse (fp32 hierarchy)
  double* mg_Eg = nullptr;           // level-2 Galerkin: gathered fine moduli [64][nel_2] (DGEMM operand)
  double *mg_C = nullptr, *mg_R = nullptr, *mg_P = nullptr, *mg_ws = nullptr;   // symmetric-sweep scratch (C, C P, P)
  int mg_npad = 0;                   // coarsest dense size rounded up to kGjB
  double mg_diag8[8 * 24];
  int mg_n = 0;                      // free DOFs of the coarsest level
  int* mg_dmap = nullptr;            // coarsest: level DOF index -> dense index or -1
  long long* mg_imap = nullptr;      // coarsest: dense index -> level DOF index
  double* mg_om = nullptr;           // [33]: smoother weight per level; [16] = 1.0; [17 + l] = 1/||pw_l||_D
  cudaGraphExec_t mg_setup_exec = nullptr;     // first design: 8 power steps from the hash vector
  cudaGraphExec_t mg_setup_exec_w = nullptr;   // later designs: 3 steps from the previous vector
  long long mg_setup_launches_w = 0;
  bool mg_warm = false, mg_warm_b = false;     // power vectors valid (and in the snapshot)
  // x-slabs (W > 1): levels >= 1 are replicated (every rank, or once in loopback
  // mode); level 1 is formed from the whole grid's moduli, gathered per design
  Geo mg_gG{};                       // whole-grid element geometry of mg_gE
  double* mg_gE = nullptr;           // whole-grid E (W > 1; W = 1 uses slab 0's E)
  float* mg_E32 = nullptr;           // fp32 copy of mgE for the fp32 level-1 operator
  long long mg_setup_launches = 0;
  int mg_batch = 2;
  bool mg_kcycle = false;            // K-cycle on the coarse levels + flexible PCG (M8, M9)
  bool w32_off = false;              // the V-cycle output stays double (test hook)
  bool k32_on = false;               // fp32 Krylov r, q allocated (topo_params.krylov_fp32, one slab)
  bool k32_pass = false;             // ... in use by the running MG-PCG pass
  int mg_kmin = 1, mg_kmax = 99;     // K-cycle levels [kmin, kmax] (TOPO_KMIN / TOPO_KMAX: experiments)
  bool l1_face = true;               // level-1 operator: face-accumulating k_mg_l1_face (TOPO_L1_FACE=0: k_mg_l1_elem)
  double* mg_kc = nullptr;           // K-cycle scalars, 8 per level
  int mg_dl = 0;                     // x-slabs: levels 1 .. mg_dl distributed over the slabs (0: replicated)
};

namespace {

const topo_ctx* g_const_owner = nullptr;   // whose KE / stencil is in constant memory

int set_err(topo_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CU(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return set_err(ctx, TOPO_ECUDA, "%s failed: %s (%s:%d)", #call,                 \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                     \
  } while (0)
#define CK(call)                        \
  do {                                  \
    int rc_ = (call);                   \
    if (rc_ != TOPO_OK) return rc_;     \
  } while (0)
#define NC(call)                                                                      \
  do {                                                                                \
    ncclResult_t r_ = (call);                                                         \
    if (r_ != 0)                                                                      \
      return set_err(ctx, TOPO_ENCCL, "%s failed: %s", #call, g_nccl.GetErrorString(r_)); \
  } while (0)

// grid of a grid-stride streaming kernel: at most the CTAs that are resident at
// once (one wave: no tail of a partial last wave), at most grid_for(n)
template <typename K>
int grid_resident(K kern, long long n, int threads = kBlock) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
  const long long b = (n + threads - 1) / threads;
  return (int)std::max(1LL, std::min<long long>(b, 148LL * per_sm));
}

inline int grid_for(long long n) {
  long long b = (n + kBlock - 1) / kBlock;
  if (b < 1) b = 1;
  if (b > kMaxGridBlocks) b = kMaxGridBlocks;
  return (int)b;
}

// --- launch helpers (count launches) ----------------------------------------
void debug_sync(topo_ctx* ctx, const char* name) {
  if (!ctx->debug || ctx->sticky) return;
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) ctx->sticky = set_err(ctx, TOPO_ECUDA, "kernel %s: %s", name, cudaGetErrorString(e));
}

// Kernel launch on the bound stream.  With TOPO_PDL (default on) the launch
// carries the programmatic-stream-serialization attribute: the kernel may be
// scheduled while the previous one drains and waits for it in pdl_enter()
// (common.cuh) -- the launch latency of the chains of small multigrid kernels
// overlaps the previous kernel instead of following it.
inline bool pdl_on() {
  static const bool on = !getenv("TOPO_PDL") || atoi(getenv("TOPO_PDL")) != 0;
  return on;
}
template <typename... KArgs, typename... Args>
void launch_k(cudaStream_t stream, void (*kern)(KArgs...), int grid, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kBlock);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  // the kernel's parameter types; trailing defaulted parameters (all 0 / nullptr) value-initialised
  using Tup = std::tuple<std::decay_t<KArgs>...>;
  static_assert(sizeof...(Args) <= sizeof...(KArgs), "kernel argument count");
  auto in = std::forward_as_tuple(std::forward<Args>(args)...);
  Tup conv = [&]<size_t... I>(std::index_sequence<I...>) {
    auto pick = [&]<size_t J>(std::integral_constant<size_t, J>) -> std::tuple_element_t<J, Tup> {
      if constexpr (J < sizeof...(Args)) return std::get<J>(in);
      else return std::tuple_element_t<J, Tup>{};
    };
    return Tup{pick(std::integral_constant<size_t, I>{})...};
  }(std::index_sequence_for<KArgs...>{});
  std::apply(
      [&](auto&... a) {
        void* ptrs[] = {static_cast<void*>(&a)...};
        cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(kern), ptrs);
      },
      conv);
}
#define LAUNCH(ctx, kern, grid, ...)                                      \
  do {                                                                    \
    launch_k((ctx)->stream, kern, (grid), __VA_ARGS__);                   \
    (ctx)->launches++;                                                    \
    debug_sync((ctx), #kern);                                             \
  } while (0)

int check_launch(topo_ctx* ctx) {
  if (ctx->sticky) return ctx->sticky;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(ctx, TOPO_ECUDA, "kernel launch: %s", cudaGetErrorString(e));
  return TOPO_OK;
}

int ensure_constants(topo_ctx* ctx) {
  if (g_const_owner == ctx) return TOPO_OK;
  CU(cudaMemcpyToSymbolAsync(c_KE, ctx->ke, sizeof(double) * 576, 0, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyToSymbolAsync(c_wht, &ctx->wht, sizeof(WhtK), 0, cudaMemcpyHostToDevice, ctx->stream));
  if (ctx->mg_on) {
    double w[8][8][8];
    mg_child_weights(w);
    signed char nzA[8][8][8] = {};
    double nzW[8][8][8] = {};
    int nzN[8][8] = {};
    for (int c = 0; c < 8; ++c)
      for (int R = 0; R < 8; ++R)
        for (int A = 0; A < 8; ++A)
          if (w[c][A][R] != 0.0) {
            nzA[c][R][nzN[c][R]] = (signed char)A;
            nzW[c][R][nzN[c][R]] = w[c][A][R];
            nzN[c][R]++;
          }
    const WhtK& w0 = ctx->wht;
    const WhtK w1{w0.k0 / 4, w0.o0 / 4, w0.k7 / 16, w0.o7 / 16, w0.a / 16, w0.b / 16, w0.r / 4, w0.s / 64};
    ctx->wht1 = w1;
    ctx->wht1f = WhtKT<float>{(float)w1.k0, (float)w1.o0, (float)w1.k7, (float)w1.o7, (float)w1.a, (float)w1.b,
                              (float)w1.r, (float)w1.s};
    CU(cudaMemcpyToSymbolAsync(c_wht1, &ctx->wht1, sizeof(WhtK), 0, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyToSymbolAsync(c_wht1f, &ctx->wht1f, sizeof(WhtKT<float>), 0, cudaMemcpyHostToDevice, ctx->stream));
    ctx->whtf = WhtKT<float>{(float)w0.k0, (float)w0.o0, (float)w0.k7, (float)w0.o7, (float)w0.a, (float)w0.b,
                             (float)w0.r, (float)w0.s};
    CU(cudaMemcpyToSymbolAsync(c_whtf, &ctx->whtf, sizeof(WhtKT<float>), 0, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyToSymbolAsync(c_mg_diag8, ctx->mg_diag8, sizeof(ctx->mg_diag8), 0, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyToSymbolAsync(c_mg_nzA, nzA, sizeof nzA, 0, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyToSymbolAsync(c_mg_nzW, nzW, sizeof nzW, 0, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyToSymbolAsync(c_mg_nzN, nzN, sizeof nzN, 0, cudaMemcpyHostToDevice, ctx->stream));
    unsigned short up[300];
    for (int r = 0, u = 0; r < 24; ++r)
      for (int c = r; c < 24; ++c) up[u++] = (unsigned short)(r * 24 + c);
    CU(cudaMemcpyToSymbolAsync(c_mg_upair, up, sizeof up, 0, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));   // host staging arrays go out of scope
  }
  if (!ctx->st_off.empty()) {
    CU(cudaMemcpyToSymbolAsync(c_st_off, ctx->st_off.data(), sizeof(int4) * ctx->st_off.size(), 0,
                               cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaMemcpyToSymbolAsync(c_st_w, ctx->st_w.data(), sizeof(double) * ctx->st_w.size(), 0,
                               cudaMemcpyHostToDevice, ctx->stream));
    ctx->st_poff.resize(ctx->st_off.size());
    const FiltPad& fp = ctx->slabs[0].fp;
    for (size_t k = 0; k < ctx->st_off.size(); ++k)
      ctx->st_poff[k] = (int)(ctx->st_off[k].x * fp.fplane + ctx->st_off[k].z * fp.FY + ctx->st_off[k].y);
    CU(cudaMemcpyToSymbolAsync(c_st_poff, ctx->st_poff.data(), sizeof(int) * ctx->st_poff.size(), 0,
                               cudaMemcpyHostToDevice, ctx->stream));
    if (ctx->R >= 1 && ctx->R <= 3) {   // k_filt25 weights on the (2R+1)^3 box, [dx+R][dz+R][dy+R]
      static double fw[343];
      std::fill(fw, fw + 343, 0.0);
      for (size_t k = 0; k < ctx->st_off.size(); ++k) {
        const int4 o = ctx->st_off[k];
        fw[((o.x + ctx->R) * 7 + (o.z + ctx->R)) * 7 + (o.y + ctx->R)] = ctx->st_w[k];
      }
      CU(cudaMemcpyToSymbolAsync(c_fw, fw, sizeof fw, 0, cudaMemcpyHostToDevice, ctx->stream));
      // by class (|dx|, a <= b): the stencil is a function of |d| (checked here)
      static double fw2[64];
      std::fill(fw2, fw2 + 64, 0.0);
      const int R = ctx->R;
      for (int dx = -R; dx <= R; ++dx)
        for (int dz = -R; dz <= R; ++dz)
          for (int dy = -R; dy <= R; ++dy) {
            const int a = std::min(std::abs(dy), std::abs(dz)), b = std::max(std::abs(dy), std::abs(dz));
            const double w = fw[((dx + R) * 7 + (dz + R)) * 7 + (dy + R)];
            double& c = fw2[(std::abs(dx) * 4 + a) * 4 + b];
            if (dx >= 0 && dy >= 0 && dz >= 0 && dy <= dz) c = w;
          }
      for (int dx = -R; dx <= R; ++dx)
        for (int dz = -R; dz <= R; ++dz)
          for (int dy = -R; dy <= R; ++dy) {
            const int a = std::min(std::abs(dy), std::abs(dz)), b = std::max(std::abs(dy), std::abs(dz));
            if (fw[((dx + R) * 7 + (dz + R)) * 7 + (dy + R)] != fw2[(std::abs(dx) * 4 + a) * 4 + b] ||
                (fw2[(std::abs(dx) * 4 + a) * 4 + b] != 0.0 && dx * dx + a * a + b * b >= (R + 1) * (R + 1)))
              return set_err(ctx, TOPO_EINVAL, "filter stencil is not a function of |d|");
          }
      CU(cudaMemcpyToSymbolAsync(c_fw2, fw2, sizeof fw2, 0, cudaMemcpyHostToDevice, ctx->stream));
    }
    CU(cudaStreamSynchronize(ctx->stream));
  }
  g_const_owner = ctx;
  return TOPO_OK;
}

Material material(const topo_ctx* ctx) {
  return Material{ctx->prm.E0, ctx->prm.Emin, ctx->prm.penal, ctx->kd};
}

// ---------------------------------------------------------------------------
// Communication across slabs (loopback: in-process copies; NCCL: send/recv)
// ---------------------------------------------------------------------------
void CUDART_CB host_op_cb(void* p) { host_op_run(static_cast<HostOp*>(p)); }

int host_launch(topo_ctx* ctx, const HostOp& op) {
  ctx->hops.push_back(op);
  CU(cudaLaunchHostFunc(ctx->stream, host_op_cb, &ctx->hops.back()));
  return TOPO_OK;
}

int allreduce(topo_ctx* ctx, int k0, int nk, int maxmask) {
  const int W = ctx->world;
  if (W == 1 || ctx->mode == TOPO_DIST_SOLO) return TOPO_OK;
  if (ctx->mode == TOPO_DIST_HOST) {
    DevState* st = ctx->slabs[0].st;
    CU(cudaMemcpyAsync(ctx->ht->hsend, st->sums + k0, sizeof(double) * nk, cudaMemcpyDeviceToHost, ctx->stream));
    HostOp op;
    op.t = ctx->ht;
    op.kind = 1;
    op.n = nk;
    op.maxmask = (unsigned)maxmask;
    CK(host_launch(ctx, op));
    CU(cudaMemcpyAsync(st->sums + k0, ctx->ht->hrecv, sizeof(double) * nk, cudaMemcpyHostToDevice, ctx->stream));
    return TOPO_OK;
  }
  if (ctx->mode == TOPO_DIST_LOOPBACK) {
    StatePtrs sp{};
    for (int s = 0; s < W; ++s) sp.s[s] = ctx->slabs[s].st;
    k_slab_allreduce<<<1, 32, 0, ctx->stream>>>(sp, W, k0, nk, maxmask);
    ctx->launches++;
    return check_launch(ctx);
  }
  DevState* st = ctx->slabs[0].st;
  // contiguous runs of sum / max slots
  int k = 0;
  while (k < nk) {
    const bool mx = (maxmask >> k) & 1;
    int e = k;
    while (e < nk && (((maxmask >> e) & 1) != 0) == mx) ++e;
    NC(g_nccl.AllReduce(st->sums + k0 + k, st->sums + k0 + k, (size_t)(e - k), ncclFloat64,
                        mx ? ncclMax : ncclSum, ctx->comm, ctx->stream));
    k = e;
  }
  return TOPO_OK;
}

// node planes of a 3-component vector: owned boundary planes -> neighbours' ghosts
int exchange_nodes(topo_ctx* ctx, double* Slab::*field, int ncomp = 3) {
  const int W = ctx->world;
  if (W == 1 || ctx->mode == TOPO_DIST_SOLO) return TOPO_OK;
  if (ctx->mode == TOPO_DIST_LOOPBACK) {
    for (int s = 0; s < W; ++s) {
      Slab& a = ctx->slabs[s];
      const size_t bytes = sizeof(double) * a.g.nplane;
      for (int c = 0; c < ncomp; ++c) {
        double* v = a.*field + c * a.g.ncomp;
        if (s > 0) {
          Slab& l = ctx->slabs[s - 1];
          CU(cudaMemcpyAsync(l.*field + c * l.g.ncomp + (l.g.nown + 1) * l.g.nplane, v + a.g.nplane,
                             bytes, cudaMemcpyDeviceToDevice, ctx->stream));
        }
        if (s < W - 1) {
          Slab& rr = ctx->slabs[s + 1];
          CU(cudaMemcpyAsync(rr.*field + c * rr.g.ncomp, v + a.g.nown * a.g.nplane, bytes,
                             cudaMemcpyDeviceToDevice, ctx->stream));
        }
      }
    }
    return TOPO_OK;
  }
  Slab& a = ctx->slabs[0];
  const size_t n = a.g.nplane;
  if (ctx->mode == TOPO_DIST_HOST) {
    double *hs = ctx->ht->hsend, *hr = ctx->ht->hrecv;
    const size_t b = sizeof(double) * n;
    for (int c = 0; c < ncomp; ++c) {
      double* v = a.*field + c * a.g.ncomp;
      if (ctx->rank > 0) CU(cudaMemcpyAsync(hs + (2 * c) * n, v + a.g.nplane, b, cudaMemcpyDeviceToHost, ctx->stream));
      if (ctx->rank < W - 1)
        CU(cudaMemcpyAsync(hs + (2 * c + 1) * n, v + a.g.nown * a.g.nplane, b, cudaMemcpyDeviceToHost, ctx->stream));
    }
    HostOp op;
    op.t = ctx->ht;
    op.kind = 0;
    op.len = (long long)n;
    op.nblk = ncomp;
    CK(host_launch(ctx, op));
    for (int c = 0; c < ncomp; ++c) {
      double* v = a.*field + c * a.g.ncomp;
      if (ctx->rank > 0) CU(cudaMemcpyAsync(v, hr + (2 * c) * n, b, cudaMemcpyHostToDevice, ctx->stream));
      if (ctx->rank < W - 1)
        CU(cudaMemcpyAsync(v + (a.g.nown + 1) * a.g.nplane, hr + (2 * c + 1) * n, b, cudaMemcpyHostToDevice, ctx->stream));
    }
    return TOPO_OK;
  }
  NC(g_nccl.GroupStart());
  for (int c = 0; c < ncomp; ++c) {
    double* v = a.*field + c * a.g.ncomp;
    if (ctx->rank > 0) {
      NC(g_nccl.Send(v + a.g.nplane, n, ncclFloat64, ctx->rank - 1, ctx->comm, ctx->stream));
      NC(g_nccl.Recv(v, n, ncclFloat64, ctx->rank - 1, ctx->comm, ctx->stream));
    }
    if (ctx->rank < W - 1) {
      NC(g_nccl.Send(v + a.g.nown * a.g.nplane, n, ncclFloat64, ctx->rank + 1, ctx->comm, ctx->stream));
      NC(g_nccl.Recv(v + (a.g.nown + 1) * a.g.nplane, n, ncclFloat64, ctx->rank + 1, ctx->comm,
                     ctx->stream));
    }
  }
  NC(g_nccl.GroupEnd());
  return TOPO_OK;
}

// k element planes each side: owned boundary planes -> neighbours' halos
int exchange_elems(topo_ctx* ctx, double* Slab::*field, int k) {
  const int W = ctx->world;
  if (W == 1 || k <= 0 || ctx->mode == TOPO_DIST_SOLO) return TOPO_OK;
  if (ctx->mode == TOPO_DIST_LOOPBACK) {
    for (int s = 0; s < W; ++s) {
      Slab& a = ctx->slabs[s];
      const size_t bytes = sizeof(double) * a.g.eplane * k;
      double* v = a.*field;
      if (s > 0) {
        Slab& l = ctx->slabs[s - 1];
        CU(cudaMemcpyAsync(l.*field + (l.g.H + l.g.nex) * l.g.eplane, v + a.g.H * a.g.eplane, bytes,
                           cudaMemcpyDeviceToDevice, ctx->stream));
      }
      if (s < W - 1) {
        Slab& rr = ctx->slabs[s + 1];
        CU(cudaMemcpyAsync(rr.*field + (rr.g.H - k) * rr.g.eplane,
                           v + (a.g.H + a.g.nex - k) * a.g.eplane, bytes, cudaMemcpyDeviceToDevice,
                           ctx->stream));
      }
    }
    return TOPO_OK;
  }
  Slab& a = ctx->slabs[0];
  const size_t n = a.g.eplane * k;
  double* v = a.*field;
  if (ctx->mode == TOPO_DIST_HOST) {
    double *hs = ctx->ht->hsend, *hr = ctx->ht->hrecv;
    const size_t b = sizeof(double) * n;
    if (ctx->rank > 0) CU(cudaMemcpyAsync(hs, v + a.g.H * a.g.eplane, b, cudaMemcpyDeviceToHost, ctx->stream));
    if (ctx->rank < W - 1)
      CU(cudaMemcpyAsync(hs + n, v + (a.g.H + a.g.nex - k) * a.g.eplane, b, cudaMemcpyDeviceToHost, ctx->stream));
    HostOp op;
    op.t = ctx->ht;
    op.kind = 0;
    op.len = (long long)n;
    op.nblk = 1;
    CK(host_launch(ctx, op));
    if (ctx->rank > 0) CU(cudaMemcpyAsync(v + (a.g.H - k) * a.g.eplane, hr, b, cudaMemcpyHostToDevice, ctx->stream));
    if (ctx->rank < W - 1)
      CU(cudaMemcpyAsync(v + (a.g.H + a.g.nex) * a.g.eplane, hr + n, b, cudaMemcpyHostToDevice, ctx->stream));
    return TOPO_OK;
  }
  NC(g_nccl.GroupStart());
  if (ctx->rank > 0) {
    NC(g_nccl.Send(v + a.g.H * a.g.eplane, n, ncclFloat64, ctx->rank - 1, ctx->comm, ctx->stream));
    NC(g_nccl.Recv(v + (a.g.H - k) * a.g.eplane, n, ncclFloat64, ctx->rank - 1, ctx->comm, ctx->stream));
  }
  if (ctx->rank < W - 1) {
    NC(g_nccl.Send(v + (a.g.H + a.g.nex - k) * a.g.eplane, n, ncclFloat64, ctx->rank + 1, ctx->comm,
                   ctx->stream));
    NC(g_nccl.Recv(v + (a.g.H + a.g.nex) * a.g.eplane, n, ncclFloat64, ctx->rank + 1, ctx->comm,
                   ctx->stream));
  }
  NC(g_nccl.GroupEnd());
  return TOPO_OK;
}

// ---------------------------------------------------------------------------
// Host <-> device layout transfers (external numbering on the host side)
// ---------------------------------------------------------------------------
// owned node planes [ix0, ix0+nix) of slab s
void slab_node_range(const Slab& s, int& ix0, int& nix) {
  ix0 = s.g.ex0;
  nix = s.g.nown;
}

int upload_nodes(topo_ctx* ctx, const double* host, double* Slab::*field) {
  const int nelx = ctx->prm.nelx, nely = ctx->prm.nely, nelz = ctx->prm.nelz;
  std::vector<double> tmp;
  for (Slab& s : ctx->slabs) {
    int ix0, nix;
    slab_node_range(s, ix0, nix);
    const size_t row = (size_t)nix * (nely + 1) * 3;   // one iz layer of the sub-block
    const double* src;
    if (ctx->world == 1) {
      src = host;
    } else {
      tmp.resize(row * (nelz + 1));
      for (int iz = 0; iz <= nelz; ++iz)
        memcpy(&tmp[iz * row], host + 3 * ((size_t)iz * (nelx + 1) * (nely + 1) + (size_t)ix0 * (nely + 1)),
               sizeof(double) * row);
      src = tmp.data();
    }
    CU(cudaMemcpyAsync(s.stage, src, sizeof(double) * row * (nelz + 1), cudaMemcpyHostToDevice, ctx->stream));
    ctx->host_bytes += sizeof(double) * row * (nelz + 1);
    LAUNCH(ctx, k_nodes_in, grid_for((long long)nix * (nelz + 1) * (nely + 1)), s.g, s.stage, s.*field, ix0, nix, 0);
    CK(check_launch(ctx));
    if (ctx->world > 1) CU(cudaStreamSynchronize(ctx->stream));   // tmp reuse
  }
  return TOPO_OK;
}

int download_nodes(topo_ctx* ctx, double* Slab::*field, double* host) {
  const int nelx = ctx->prm.nelx, nely = ctx->prm.nely, nelz = ctx->prm.nelz;
  std::vector<double> tmp;
  for (Slab& s : ctx->slabs) {
    int ix0, nix;
    slab_node_range(s, ix0, nix);
    const size_t row = (size_t)nix * (nely + 1) * 3;
    LAUNCH(ctx, k_nodes_out, grid_for((long long)nix * (nelz + 1) * (nely + 1)), s.g, s.*field, s.stage, ix0, nix, 0);
    CK(check_launch(ctx));
    ctx->host_bytes += sizeof(double) * row * (nelz + 1);
    if (ctx->world == 1) {
      CU(cudaMemcpyAsync(host, s.stage, sizeof(double) * row * (nelz + 1), cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
    } else {
      tmp.resize(row * (nelz + 1));
      CU(cudaMemcpyAsync(tmp.data(), s.stage, sizeof(double) * tmp.size(), cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
      for (int iz = 0; iz <= nelz; ++iz)
        memcpy(host + 3 * ((size_t)iz * (nelx + 1) * (nely + 1) + (size_t)ix0 * (nely + 1)), &tmp[iz * row],
               sizeof(double) * row);
    }
  }
  return TOPO_OK;
}

int download_invd(topo_ctx* ctx, double* host) {
  const int nelx = ctx->prm.nelx, nely = ctx->prm.nely, nelz = ctx->prm.nelz;
  std::vector<double> tmp;
  for (Slab& s : ctx->slabs) {
    int ix0, nix;
    slab_node_range(s, ix0, nix);
    const size_t row = (size_t)nix * (nely + 1) * 3;
    LAUNCH(ctx, k_invd_out, grid_for((long long)nix * (nelz + 1) * (nely + 1)), s.g, s.invd, s.fixm, s.stage, ix0, nix, 0);
    CK(check_launch(ctx));
    ctx->host_bytes += sizeof(double) * row * (nelz + 1);
    tmp.resize(row * (nelz + 1));
    CU(cudaMemcpyAsync(tmp.data(), s.stage, sizeof(double) * tmp.size(), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (int iz = 0; iz <= nelz; ++iz)
      memcpy(host + 3 * ((size_t)iz * (nelx + 1) * (nely + 1) + (size_t)ix0 * (nely + 1)), &tmp[iz * row],
             sizeof(double) * row);
  }
  return TOPO_OK;
}

int upload_elems(topo_ctx* ctx, const double* host, double* Slab::*field) {
  const int nelx = ctx->prm.nelx, nely = ctx->prm.nely, nelz = ctx->prm.nelz;
  std::vector<double> tmp;
  for (Slab& s : ctx->slabs) {
    const size_t row = (size_t)s.g.nex * nely;
    const double* src;
    if (ctx->world == 1) {
      src = host;
    } else {
      tmp.resize(row * nelz);
      for (int ez = 0; ez < nelz; ++ez)
        memcpy(&tmp[ez * row], host + (size_t)ez * nelx * nely + (size_t)s.g.ex0 * nely, sizeof(double) * row);
      src = tmp.data();
    }
    CU(cudaMemcpyAsync(s.stage, src, sizeof(double) * row * nelz, cudaMemcpyHostToDevice, ctx->stream));
    ctx->host_bytes += sizeof(double) * row * nelz;
    LAUNCH(ctx, k_elems_in, grid_for((long long)row * nelz), s.g, s.stage, s.*field, 0);
    CK(check_launch(ctx));
    if (ctx->world > 1) CU(cudaStreamSynchronize(ctx->stream));
  }
  return TOPO_OK;
}

int download_elems(topo_ctx* ctx, double* Slab::*field, double* host) {
  const int nelx = ctx->prm.nelx, nely = ctx->prm.nely, nelz = ctx->prm.nelz;
  std::vector<double> tmp;
  for (Slab& s : ctx->slabs) {
    const size_t row = (size_t)s.g.nex * nely;
    LAUNCH(ctx, k_elems_out, grid_for((long long)row * nelz), s.g, s.*field, s.stage, 0);
    CK(check_launch(ctx));
    ctx->host_bytes += sizeof(double) * row * nelz;
    if (ctx->world == 1) {
      CU(cudaMemcpyAsync(host, s.stage, sizeof(double) * row * nelz, cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
    } else {
      tmp.resize(row * nelz);
      CU(cudaMemcpyAsync(tmp.data(), s.stage, sizeof(double) * tmp.size(), cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
      for (int ez = 0; ez < nelz; ++ez)
        memcpy(host + (size_t)ez * nelx * nely + (size_t)s.g.ex0 * nely, &tmp[ez * row], sizeof(double) * row);
    }
  }
  return TOPO_OK;
}

// Device-pointer variants (the _d calls): `dev` is the caller's WHOLE external
// array in device memory (S:45 numbering); each slab reads / writes its owned
// part in place on the bound stream -- no staging, no host copy, no host sync.
int upload_nodes_dev(topo_ctx* ctx, const double* dev, double* Slab::*field) {
  for (Slab& s : ctx->slabs)
    LAUNCH(ctx, k_nodes_in, grid_for((long long)s.g.nown * (s.g.nelz + 1) * (s.g.nely + 1)), s.g, dev, s.*field,
           s.g.ex0, s.g.nown, 1);
  return check_launch(ctx);
}
int download_nodes_dev(topo_ctx* ctx, double* Slab::*field, double* dev) {
  for (Slab& s : ctx->slabs)
    LAUNCH(ctx, k_nodes_out, grid_for((long long)s.g.nown * (s.g.nelz + 1) * (s.g.nely + 1)), s.g, s.*field, dev,
           s.g.ex0, s.g.nown, 1);
  return check_launch(ctx);
}
int download_invd_dev(topo_ctx* ctx, double* dev) {
  for (Slab& s : ctx->slabs)
    LAUNCH(ctx, k_invd_out, grid_for((long long)s.g.nown * (s.g.nelz + 1) * (s.g.nely + 1)), s.g, s.invd, s.fixm, dev,
           s.g.ex0, s.g.nown, 1);
  return check_launch(ctx);
}
int upload_elems_dev(topo_ctx* ctx, const double* dev, double* Slab::*field) {
  for (Slab& s : ctx->slabs)
    LAUNCH(ctx, k_elems_in, grid_for((long long)s.g.nex * s.g.nely * s.g.nelz), s.g, dev, s.*field, 1);
  return check_launch(ctx);
}
int download_elems_dev(topo_ctx* ctx, double* Slab::*field, double* dev) {
  for (Slab& s : ctx->slabs)
    LAUNCH(ctx, k_elems_out, grid_for((long long)s.g.nex * s.g.nely * s.g.nelz), s.g, s.*field, dev, 1);
  return check_launch(ctx);
}

// Fill a local element array (incl. halos) from a global host array of bytes.
void fill_local_elems_u8(const topo_ctx* ctx, const Slab& s, const uint8_t* glob, std::vector<uint8_t>& loc) {
  const Geo& g = s.g;
  loc.assign(g.nelloc, 0);
  for (int exl = 0; exl < g.NEXL; ++exl) {
    const int ex = exl - g.H + g.ex0;
    if (ex < 0 || ex >= g.nelx) continue;
    for (int ez = 0; ez < g.nelz; ++ez)
      for (int ey = 0; ey < g.nely; ++ey)
        loc[elem_idx(g, ex, ey, ez)] = glob ? glob[(size_t)ez * g.nelx * g.nely + (size_t)ex * g.nely + ey] : 0;
  }
}

// Wait for the bound stream.  Multi-process transports poll instead of blocking:
// NCCL's asynchronous error state (ncclCommGetAsyncError; the communicator is
// aborted on an error) and a timeout, so a dead peer becomes TOPO_ENCCL instead
// of a hang; the host transport reports a peer timeout the same way.
int wait_stream(topo_ctx* ctx) {
  const bool nccl = ctx->mode == TOPO_DIST_NCCL && ctx->comm;
  if (!nccl && !ctx->ht) {
    CU(cudaStreamSynchronize(ctx->stream));
    return TOPO_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  long long spins = 0;
  while (true) {
    const cudaError_t e = cudaStreamQuery(ctx->stream);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) return set_err(ctx, TOPO_ECUDA, "stream: %s", cudaGetErrorString(e));
    if (nccl && g_nccl.CommGetAsyncError) {
      ncclResult_t ar = 0;
      if (g_nccl.CommGetAsyncError(ctx->comm, &ar) == 0 && ar != 0 && ar != 7 /* ncclInProgress */) {
        if (g_nccl.CommAbort) g_nccl.CommAbort(ctx->comm);
        ctx->comm = nullptr;
        return set_err(ctx, TOPO_ENCCL, "NCCL asynchronous error: %s", g_nccl.GetErrorString(ar));
      }
    }
    if (ctx->ht && ctx->ht->failed.load()) return set_err(ctx, TOPO_ENCCL, "host transport: a peer timed out");
    if (++spins > 256) {
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (el > ctx->comm_timeout_s) {
        if (nccl && g_nccl.CommAbort) { g_nccl.CommAbort(ctx->comm); ctx->comm = nullptr; }
        return set_err(ctx, TOPO_ENCCL, "collective timeout after %.0f s (dead peer?)", el);
      }
      sched_yield();
    }
  }
  if (ctx->ht && ctx->ht->failed.load()) return set_err(ctx, TOPO_ENCCL, "host transport: a peer timed out");
  return TOPO_OK;
}

int sync_state(topo_ctx* ctx) {
  CU(cudaMemcpyAsync(ctx->hstate, ctx->slabs[0].st, sizeof(DevState), cudaMemcpyDeviceToHost, ctx->stream));
  return wait_stream(ctx);
}

// ---------------------------------------------------------------------------
// Phase pieces
// ---------------------------------------------------------------------------
// The V-cycle output w in fp32: with the fp32 hierarchy on one slab (its
// precision is the fp32 levels' anyway; the PCG's own vectors stay fp64).
// Off inside the topo_mg_vcycle test hook (it downloads the double w).
bool w32_active(const topo_ctx* ctx) { return ctx->mg_f32 && ctx->world == 1 && !ctx->w32_off && ctx->slabs[0].w32; }
// fp32 Krylov residual / q in the running MG-PCG pass: with the fp32
// hierarchy on one slab; the true residual f - K u stays fp64 and decides.
bool k32_active(const topo_ctx* ctx) { return ctx->k32_pass && ctx->k32_on && ctx->mg_f32; }

int update_modulus(topo_ctx* ctx) {
  CK(ensure_constants(ctx));
  const Material m = material(ctx);
  for (Slab& s : ctx->slabs) {
    LAUNCH(ctx, k_efield, grid_for(s.g.nelloc), s.g, m, s.xphys, s.E);
    LAUNCH(ctx, k_invdiag, grid_for((long long)s.g.nown * s.g.nplane), s.g, m, s.E, s.fixm, s.invd);
  }
  CK(check_launch(ctx));
  CK(exchange_nodes(ctx, &Slab::invd, 1));   // ghost planes feed the fused pre-passes and the prolongation
  ctx->has_E = true;
  ctx->mg_ready = false;
  return TOPO_OK;
}

// launch geometry of the WHT matvec for one slab: (gy, gz, gx) CTAs of 32 x tz
struct MvGrid { dim3 grid, block; int CX; };
MvGrid mv_grid(const topo_ctx* ctx, const Geo& g) {
  const int tz = ctx->tz;
  const int gy = (g.nely + 1 + 30) / 31, gz = (g.nelz + 1 + tz - 2) / (tz - 1);
  const long long tiles = (long long)gy * gz;
  const long long target = 148LL * (tz <= 8 ? 2 : 1) * 8;   // ~8 waves of resident CTAs
  long long gx = (target + tiles - 1) / tiles;
  gx = std::max(1LL, std::min<long long>(gx, (g.nown + 3) / 4));   // >= 4 planes per chunk
  const int CX = (int)((g.nown + gx - 1) / gx);
  gx = (g.nown + CX - 1) / CX;
  return MvGrid{dim3(gy, gz, (unsigned)gx), dim3(32, tz, 1), CX};
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int get_encode(topo_ctx* ctx) {
  if (g_encode) return TOPO_OK;
  cudaDriverEntryPointQueryResult qr;
  CU(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&g_encode, cudaEnableDefault, &qr));
  if (qr != cudaDriverEntryPointSuccess || !g_encode)
    return set_err(ctx, TOPO_ECUDA, "cuTensorMapEncodeTiled unavailable");
  return TOPO_OK;
}

// rank-4 {NY, NZ, NXL, ncomp} (ncomp = 3) or rank-3 {NY, NZ, NXL} (ncomp = 1) node map
int map_nodes(topo_ctx* ctx, CUtensorMap* m, double* ptr, const Geo& g, int ncomp) {
  const cuuint64_t dims[4] = {(cuuint64_t)g.NY, (cuuint64_t)g.NZ, (cuuint64_t)g.NXL, 3};
  const cuuint64_t strides[3] = {(cuuint64_t)g.NY * 8, (cuuint64_t)g.nplane * 8, (cuuint64_t)g.ncomp * 8};
  const cuuint32_t box[4] = {34, (cuuint32_t)ctx->tz + 1, 1, 3};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, ncomp == 3 ? 4 : 3, ptr, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(ctx, TOPO_ECUDA, "cuTensorMapEncodeTiled(nodes) failed: %d", (int)r);
  return TOPO_OK;
}

// fp32 3-component node vector (the multigrid z): box rows of 36 floats (16-byte multiple)
int map_nodes32(topo_ctx* ctx, CUtensorMap* m, float* ptr, const Geo& g) {
  const cuuint64_t dims[4] = {(cuuint64_t)g.NY, (cuuint64_t)g.NZ, (cuuint64_t)g.NXL, 3};
  const cuuint64_t strides[3] = {(cuuint64_t)g.NY * 4, (cuuint64_t)g.nplane * 4, (cuuint64_t)g.ncomp * 4};
  const cuuint32_t box[4] = {36, (cuuint32_t)ctx->tz + 1, 1, 3};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, ptr, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(ctx, TOPO_ECUDA, "cuTensorMapEncodeTiled(nodes32) failed: %d", (int)r);
  return TOPO_OK;
}

int map_elems(topo_ctx* ctx, CUtensorMap* m, double* ptr, const Geo& g) {
  const cuuint64_t dims[3] = {(cuuint64_t)g.EY, (cuuint64_t)g.EZ, (cuuint64_t)g.NEXL};
  const cuuint64_t strides[2] = {(cuuint64_t)g.EY * 8, (cuuint64_t)g.eplane * 8};
  const cuuint32_t box[3] = {34, (cuuint32_t)ctx->tz, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ptr, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(ctx, TOPO_ECUDA, "cuTensorMapEncodeTiled(elems) failed: %d", (int)r);
  return TOPO_OK;
}

int build_maps(topo_ctx* ctx, Slab& s) {
  CK(get_encode(ctx));
  CK(map_nodes(ctx, &s.m_r, s.r, s.g, 3));
  CK(map_nodes(ctx, &s.m_u, s.u, s.g, 3));
  CK(map_nodes(ctx, &s.m_w, s.w, s.g, 3));
  CK(map_nodes(ctx, &s.m_p0, s.p0, s.g, 3));
  CK(map_nodes(ctx, &s.m_p1, s.p1, s.g, 3));
  CK(map_nodes(ctx, &s.m_invd, s.invd, s.g, 1));
  CK(map_elems(ctx, &s.m_E, s.E, s.g));
  CK(map_nodes(ctx, &s.m_z, s.z, s.g, 3));
  CK(map_nodes(ctx, &s.m_q, s.q, s.g, 3));
  if (ctx->R >= 1 && ctx->R <= 3) {   // k_filt25 operand: {FY, FZ, NEXL}, zero fill beyond the array
    const cuuint64_t dims[3] = {(cuuint64_t)s.fp.FY, (cuuint64_t)s.fp.FZ, (cuuint64_t)s.g.NEXL};
    const cuuint64_t strides[2] = {(cuuint64_t)s.fp.FY * 8, (cuuint64_t)s.fp.fplane * 8};
    const cuuint32_t box[3] = {(cuuint32_t)(kF25Y + 2 * ctx->R), (cuuint32_t)(kF25Z + 2 * ctx->R), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(&s.m_vpad, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, s.vpad, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(ctx, TOPO_ECUDA, "cuTensorMapEncodeTiled(vpad) failed: %d", (int)r);
  }
  return TOPO_OK;
}

// A6 apply step: the x-marching TMA stencil (k_filt25) for R = 1..3, else the
// per-output gather (k_filt_apply).  TOPO_FILT25=0 selects the gather (A/B).
template <int R, int MODE>
int launch_filt25_r(topo_ctx* ctx, Slab& s, const double* a, double* out) {
  using L = F25Smem<R>;
  static const bool sym = !getenv("TOPO_FILT_SYM") || atoi(getenv("TOPO_FILT_SYM")) != 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(ctx->f25_attr_mask & (1u << (dev * 4 + MODE % 4)))) {   // opt-in per device
    CU(cudaFuncSetAttribute(k_filt25<R, MODE, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES));
    CU(cudaFuncSetAttribute(k_filt25<R, MODE, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::BYTES));
    ctx->f25_attr_mask |= 1u << (dev * 4 + MODE % 4);
  }
  const int gy = (s.g.nely + kF25Y - 1) / kF25Y, gz = (s.g.nelz + kF25Z - 1) / kF25Z;
  const long long tiles = (long long)gy * gz;
  long long gx = std::max(1LL, (148LL * 6 + tiles - 1) / tiles);
  gx = std::min<long long>(gx, std::max(1, s.g.nex / 8));   // >= 8 output planes per chunk
  const int CX = (int)((s.g.nex + gx - 1) / gx);
  gx = (s.g.nex + CX - 1) / CX;
  auto kern = sym ? k_filt25<R, MODE, true> : k_filt25<R, MODE, false>;
  kern<<<dim3(gy, gz, (unsigned)gx), dim3(kF25Y, kF25Z / kF25TZ), L::BYTES, ctx->stream>>>(
      s.m_vpad, s.g, s.fp, CX, a, (MODE == F_X0 || MODE == F_PLAIN) ? s.ihs : s.hs, s.passive, out);
  ctx->launches++;
  debug_sync(ctx, "k_filt25");
  return check_launch(ctx);
}
template <int MODE>
int launch_filt_apply(topo_ctx* ctx, Slab& s, const double* a, double* out) {
  static const bool use25 = !getenv("TOPO_FILT25") || atoi(getenv("TOPO_FILT25")) != 0;
  if (use25) {
    if (ctx->R == 1) return launch_filt25_r<1, MODE>(ctx, s, a, out);
    if (ctx->R == 2) return launch_filt25_r<2, MODE>(ctx, s, a, out);
    if (ctx->R == 3) return launch_filt25_r<3, MODE>(ctx, s, a, out);
  }
  LAUNCH(ctx, k_filt_apply<MODE>, grid_for((long long)s.g.nex * s.g.eplane), s.g, s.fp, (int)ctx->st_off.size(),
         s.vpad, a, s.hs, s.passive, out);
  return check_launch(ctx);
}

template <int TZ, int kPre, bool kDot, int kEpi, typename TC, typename TV = double>
int launch_mv_t(topo_ctx* ctx, Slab& s, int gate, const MvMaps& maps, double* pnew, double* q, int finish,
                const double* scale) {
  // the dynamic-smem opt-in is per device: remember it per device
  static unsigned attr_set = 0;
  const int smem = MvSmem<TZ, TV>::bytes(kPre);
  if (!(attr_set & (1u << (ctx->device & 31)))) {
    CU(cudaFuncSetAttribute(k_mv_wht<TZ, kPre, kDot, kEpi, TC, TV>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set |= 1u << (ctx->device & 31);
  }
  const MvGrid m = mv_grid(ctx, s.g);
  // kEpi = 1 with the K-cycle: the PCG's q (untouched by the V-cycle: the fp32
  // pre-smoothing residual goes to res32, the fp64 one to z) for the flexible beta
  const bool k32 = k32_active(ctx);
  const MvEpi epi{s.r, s.invd, s.fixm, (kEpi == 2 && ctx->mg_f32) ? s.res32 : nullptr,
                  (kEpi == 1 && w32_active(ctx)) ? s.w32 : nullptr,
                  (kEpi == 1 && ctx->mg_kcycle) ? s.q : nullptr,
                  (k32 && (kEpi == 1 || kEpi == 2)) ? s.r32 : nullptr,
                  (k32 && kEpi == 1 && ctx->mg_kcycle) ? s.q32 : nullptr,
                  (k32 && kEpi == 0 && kPre == 2) ? s.q32 : nullptr};
  k_mv_wht<TZ, kPre, kDot, kEpi, TC, TV><<<m.grid, m.block, smem, ctx->stream>>>(maps, s.g, s.st, gate, m.CX, pnew,
                                                                                 q, s.partials, s.counter, finish,
                                                                                 scale, epi);
  ctx->launches++;
  debug_sync(ctx, kPre == 1 ? "k_mv_wht<jacobi-fused>" : kPre == 2 ? "k_mv_wht<mg-fused>"
                  : kPre == 3 ? "k_mv_wht<mg-presmooth>" : "k_mv_wht<plain>");
  return check_launch(ctx);
}

template <int kPre, bool kDot, int kEpi = 0, typename TC = double, typename TV = double>
int launch_mv(topo_ctx* ctx, Slab& s, int gate, const CUtensorMap& vin, const CUtensorMap* pold, double* pnew,
              double* q, int finish, const double* scale = nullptr) {
  MvMaps maps;
  maps.vin = vin;
  maps.pold = pold ? *pold : vin;
  maps.invd = s.m_invd;
  maps.E = s.m_E;
  if (ctx->tz == 16) return launch_mv_t<16, kPre, kDot, kEpi, TC, TV>(ctx, s, gate, maps, pnew, q, finish, scale);
  return launch_mv_t<8, kPre, kDot, kEpi, TC, TV>(ctx, s, gate, maps, pnew, q, finish, scale);
}

// q = K v for every slab (v ghosts exchanged first; v must be 0 on fixed DOFs)
int matvec_all(topo_ctx* ctx, double* Slab::*pin, CUtensorMap Slab::*pmap, double* Slab::*qout) {
  CK(exchange_nodes(ctx, pin));
  for (Slab& s : ctx->slabs) CK((launch_mv<0, false>(ctx, s, 0, s.*pmap, nullptr, nullptr, s.*qout, 0)));
  return check_launch(ctx);
}

// residual r = f - K u ; sums[0,1] = (rz, rr) allreduced; r ghosts refreshed
int residual(topo_ctx* ctx, bool write_r) {
  CK(matvec_all(ctx, &Slab::u, &Slab::m_u, &Slab::q));
  for (Slab& s : ctx->slabs)
    if (write_r && k32_active(ctx))
      LAUNCH(ctx, k_residual<float>, grid_resident(k_residual<float>, (long long)s.g.nown * s.g.nplane), s.g, s.st, s.f,
             s.q, s.invd, s.fixm, s.r32, 1, s.partials, s.counter);
    else
      LAUNCH(ctx, k_residual<double>, grid_resident(k_residual<double>, (long long)s.g.nown * s.g.nplane), s.g, s.st,
             s.f, s.q, s.invd, s.fixm, s.r, write_r ? 1 : 0, s.partials, s.counter);
  CK(check_launch(ctx));
  if (write_r) CK(exchange_nodes(ctx, &Slab::r));
  return allreduce(ctx, 0, 2, 0);
}

// enqueue one PCG iteration; `parity` selects the p ping-pong direction
int enqueue_cg_iter(topo_ctx* ctx, bool prof_here, int parity) {
  const int W = ctx->world;
  const int fin = (W == 1) ? 1 : 0;
  if (prof_here) CU(cudaEventRecordWithFlags(ctx->pe0, ctx->stream, cudaEventRecordExternal));
  for (Slab& s : ctx->slabs) {
    const CUtensorMap* pold = parity ? &s.m_p1 : &s.m_p0;
    double* pnew = parity ? s.p0 : s.p1;
    CK((launch_mv<1, true>(ctx, s, 1, s.m_r, pold, pnew, s.q, fin)));
  }
  if (prof_here) CU(cudaEventRecordWithFlags(ctx->pe1, ctx->stream, cudaEventRecordExternal));
  if (!fin) {
    CK(allreduce(ctx, 0, 1, 0));
    for (Slab& s : ctx->slabs) { k_finish_alpha<<<1, 1, 0, ctx->stream>>>(s.st); ctx->launches++; }
  }
  for (Slab& s : ctx->slabs) {
    double* pnew = parity ? s.p0 : s.p1;
    double* pprev = parity ? s.p1 : s.p0;
    if (parity)
      LAUNCH(ctx, (k_update<true, false>), grid_for((long long)s.g.nown * s.g.nplane / 2), s.g, s.st, s.u, s.r, pprev,
             pnew, s.q, s.invd, s.fixm, s.partials, s.counter, fin);
    else
      LAUNCH(ctx, (k_update<false, false>), grid_for((long long)s.g.nown * s.g.nplane / 2), s.g, s.st, s.u, s.r, pprev,
             pnew, s.q, s.invd, s.fixm, s.partials, s.counter, fin);
  }
  if (!fin) {
    CK(allreduce(ctx, 0, 2, 0));
    for (Slab& s : ctx->slabs) { k_finish_update<false><<<1, 1, 0, ctx->stream>>>(s.st, parity ? 0 : 1); ctx->launches++; }
    CK(exchange_nodes(ctx, &Slab::r));
  }
  return check_launch(ctx);
}

// apply the deferred u half-step (even-slot exit); p of an even slot lives in p1
int flush_u(topo_ctx* ctx) {
  DevState& h = *ctx->hstate;
  if (!h.pending) return TOPO_OK;
  for (Slab& s : ctx->slabs) {
    LAUNCH(ctx, k_flush_u, grid_for(3LL * s.g.nown * s.g.nplane), s.g, h.alpha_prev, s.u, s.p1);
    k_clear_pending<<<1, 1, 0, ctx->stream>>>(s.st);
    ctx->launches++;
  }
  CK(check_launch(ctx));
  return sync_state(ctx);
}

int enqueue_mg_iter(topo_ctx* ctx, bool prof_here, int parity);

int build_cg_graph(topo_ctx* ctx, int mg) {
  if (ctx->cg_exec[mg] && ctx->cg_profiled_graph[mg] == ctx->profile) return TOPO_OK;
  if (ctx->cg_exec[mg]) { cudaGraphExecDestroy(ctx->cg_exec[mg]); ctx->cg_exec[mg] = nullptr; }
  cudaGraph_t graph;
  const long long l0 = ctx->launches;
  CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  int rc = TOPO_OK;
  const int nb = mg ? ctx->mg_batch : ctx->cg_batch;
  for (int i = 0; i < nb && rc == TOPO_OK; ++i)
    rc = mg ? enqueue_mg_iter(ctx, ctx->profile && i == 0, i & 1)
            : enqueue_cg_iter(ctx, ctx->profile && i == 0, i & 1);
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  if (rc != TOPO_OK) return rc;
  if (e != cudaSuccess) return set_err(ctx, TOPO_ECUDA, "graph capture: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&ctx->cg_exec[mg], graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return set_err(ctx, TOPO_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
  ctx->cg_batch_launches[mg] = ctx->launches - l0;
  ctx->launches = l0;
  ctx->cg_profiled_graph[mg] = ctx->profile;
  return TOPO_OK;
}

// ---------------------------------------------------------------------------
// Geometric multigrid preconditioner (M1-M6).
// Level 0 is the fine slab (W = 1); level 1 is applied matrix-free as
// P^T K(E) P through the fine WHT matvec unless it is the coarsest level;
// levels >= 2 (and a coarsest level 1) store Galerkin element matrices; the
// coarsest level is solved with an explicit Gauss-Jordan inverse.
// ---------------------------------------------------------------------------
LvGeo lv0(const topo_ctx* ctx) {
  const Geo& g = ctx->slabs[0].g;
  return LvGeo{g.nelx, g.nely, g.nelz, g.NY, g.nplane, g.ncomp};
}
// level 0 of slab s: its owned node planes (local plane 0 = global ex0)
LvGeo lv_slab(const Slab& s) { return LvGeo{s.g.nown - 1, s.g.nely, s.g.nelz, s.g.NY, s.g.nplane, s.g.ncomp}; }
// element geometry / moduli the replicated levels >= 1 are formed from
const Geo& mgG(const topo_ctx* ctx) { return ctx->world > 1 ? ctx->mg_gG : ctx->slabs[0].g; }
const double* mgE(const topo_ctx* ctx) { return ctx->world > 1 ? ctx->mg_gE : ctx->slabs[0].E; }

// x-slabs: all-gather of the owned element planes of E into mg_gE (per design)
int mg_gather_E(topo_ctx* ctx) {
  if (ctx->world == 1) return TOPO_OK;
  const Geo& G = ctx->mg_gG;
  auto dst = [&](int ex0) { return ctx->mg_gE + (size_t)(ex0 + G.H) * G.eplane; };
  if (ctx->mode == TOPO_DIST_LOOPBACK) {
    for (Slab& s : ctx->slabs)
      CU(cudaMemcpyAsync(dst(s.g.ex0), s.E + (size_t)s.g.H * s.g.eplane, sizeof(double) * s.g.nex * s.g.eplane,
                         cudaMemcpyDeviceToDevice, ctx->stream));
    return TOPO_OK;
  }
  Slab& a = ctx->slabs[0];
  if (ctx->mode == TOPO_DIST_SOLO) {   // no peers: own planes tiled over every rank's range (same bytes land)
    for (int r = 0; r < ctx->world; ++r) {
      int b = 0, e = 0;
      topo_partition(ctx->prm.nelx, ctx->prm.rmin, ctx->world, r, &b, &e);
      for (int P = b; P < e; P += a.g.nex) {
        const int n = std::min(e - P, a.g.nex);
        CU(cudaMemcpyAsync(dst(P), a.E + (size_t)a.g.H * a.g.eplane, sizeof(double) * n * a.g.eplane,
                           cudaMemcpyDeviceToDevice, ctx->stream));
      }
    }
    return TOPO_OK;
  }
  if (ctx->mode == TOPO_DIST_HOST) {   // all-gather of the owned planes through the shared segment
    HostOp op;
    op.t = ctx->ht;
    op.kind = 3;
    for (int r = 0; r < ctx->world; ++r) {
      int b = 0, e = 0;
      topo_partition(ctx->prm.nelx, ctx->prm.rmin, ctx->world, r, &b, &e);
      op.cnt[r] = (long long)(e - b) * G.eplane;
      op.off[r] = (long long)b * G.eplane;
    }
    CU(cudaMemcpyAsync(ctx->ht->hsend, a.E + (size_t)a.g.H * a.g.eplane, sizeof(double) * a.g.nex * a.g.eplane,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(host_launch(ctx, op));
    CU(cudaMemcpyAsync(dst(0), ctx->ht->hrecv, sizeof(double) * (size_t)G.nex * G.eplane, cudaMemcpyHostToDevice,
                       ctx->stream));
    return TOPO_OK;
  }
  CU(cudaMemcpyAsync(dst(a.g.ex0), a.E + (size_t)a.g.H * a.g.eplane, sizeof(double) * a.g.nex * a.g.eplane,
                     cudaMemcpyDeviceToDevice, ctx->stream));
  NC(g_nccl.GroupStart());
  for (int r = 0; r < ctx->world; ++r) {
    if (r == ctx->rank) continue;
    int b = 0, e = 0;
    topo_partition(ctx->prm.nelx, ctx->prm.rmin, ctx->world, r, &b, &e);
    NC(g_nccl.Send(a.E + (size_t)a.g.H * a.g.eplane, (size_t)a.g.nex * a.g.eplane, ncclFloat64, r, ctx->comm,
                   ctx->stream));
    NC(g_nccl.Recv(dst(b), (size_t)(e - b) * G.eplane, ncclFloat64, r, ctx->comm, ctx->stream));
  }
  NC(g_nccl.GroupEnd());
  return TOPO_OK;
}

// x-slabs, NCCL: sum of the slabs' partial level-1 restrictions (in place)
int mg_allreduce_level(topo_ctx* ctx, void* buf, size_t n, bool f32) {
  if (ctx->world == 1 || ctx->mode == TOPO_DIST_LOOPBACK || ctx->mode == TOPO_DIST_SOLO)
    return TOPO_OK;   // loopback: accumulated in slab order
  if (ctx->mode == TOPO_DIST_HOST) {
    const size_t es = f32 ? sizeof(float) : sizeof(double);
    CU(cudaMemcpyAsync(ctx->ht->hsend, buf, es * n, cudaMemcpyDeviceToHost, ctx->stream));
    HostOp op;
    op.t = ctx->ht;
    op.kind = f32 ? 2 : 1;
    op.n = (long long)n;
    CK(host_launch(ctx, op));
    CU(cudaMemcpyAsync(buf, ctx->ht->hrecv, es * n, cudaMemcpyHostToDevice, ctx->stream));
    return TOPO_OK;
  }
  NC(g_nccl.AllReduce(buf, buf, n, f32 ? ncclFloat32 : ncclFloat64, ncclSum, ctx->comm, ctx->stream));
  return TOPO_OK;
}

// Hierarchy on the host (init): dims, coarse Dirichlet masks (M4: the node at the
// clamped position min(2j, n) decides), property Q, allocations, coarsest maps.
int mg_dist_plan(topo_ctx* ctx);
int mg_build(topo_ctx* ctx, const uint8_t* fixed) {
  const topo_params& P = ctx->prm;
  ctx->mg_on = false;
  if (P.precond == TOPO_PRECOND_JACOBI) return TOPO_OK;
  if (ctx->world > 1 && P.mg_nu != 1) {   // x-slabs: the fused nu = 1 level-0 path only
    if (P.precond == TOPO_PRECOND_MG) return set_err(ctx, TOPO_EINVAL, "multigrid on x-slabs needs mg_nu == 1");
    return TOPO_OK;
  }
  struct H { int nx, ny, nz; std::vector<uint8_t> fix; };
  std::vector<H> hs;
  // coarsest size: explicit, or auto = min(5000, max(1000, n_dof / 2000)) DOFs
  // (a larger exact coarse solve cuts MG-PCG iterations; its dense inverse is
  // only worth it on large grids)
  const long long ndof0 = 3LL * (P.nelx + 1) * (P.nely + 1) * (P.nelz + 1);
  // (K-cycle: 1000 -- the deep levels are solved well by the K-cycle, and a small
  // coarsest inverse keeps the per-design setup cheap; V-cycle: a larger exact
  // coarse solve cuts iterations on large grids)
  const bool kc = P.mg_cycle == TOPO_MG_KCYCLE && P.mg_nu == 1;
  const long long coarse_max = P.mg_coarse_max > 0 ? P.mg_coarse_max
                               : kc ? 1000 : std::min<long long>(5000, std::max<long long>(1000, ndof0 / 2000));
  {
    H h{P.nelx, P.nely, P.nelz, {}};
    const long long nn = (long long)(h.nx + 1) * (h.ny + 1) * (h.nz + 1);
    h.fix.resize(nn);
    for (long long n = 0; n < nn; ++n)
      h.fix[n] = (fixed[3 * n] ? 1 : 0) | (fixed[3 * n + 1] ? 2 : 0) | (fixed[3 * n + 2] ? 4 : 0);
    hs.push_back(std::move(h));
  }
  while (true) {
    const H& f = hs.back();
    if (3LL * (f.nx + 1) * (f.ny + 1) * (f.nz + 1) <= coarse_max) break;
    H c{(f.nx + 1) / 2, (f.ny + 1) / 2, (f.nz + 1) / 2, {}};
    if (c.nx == f.nx && c.ny == f.ny && c.nz == f.nz) break;
    auto fid = [&](int ix, int iy, int iz) { return (long long)iz * (f.nx + 1) * (f.ny + 1) + (long long)ix * (f.ny + 1) + iy; };
    auto cid = [&](int ix, int iy, int iz) { return (long long)iz * (c.nx + 1) * (c.ny + 1) + (long long)ix * (c.ny + 1) + iy; };
    c.fix.assign((size_t)(c.nx + 1) * (c.ny + 1) * (c.nz + 1), 0);
    for (int jz = 0; jz <= c.nz; ++jz)
      for (int jx = 0; jx <= c.nx; ++jx)
        for (int jy = 0; jy <= c.ny; ++jy)
          c.fix[cid(jx, jy, jz)] = f.fix[fid(std::min(2 * jx, f.nx), std::min(2 * jy, f.ny), std::min(2 * jz, f.nz))];
    bool q_ok = true;   // property Q: fixed fine DOFs interpolate from fixed coarse DOFs only
    for (int iz = 0; iz <= f.nz && q_ok; ++iz)
      for (int ix = 0; ix <= f.nx && q_ok; ++ix)
        for (int iy = 0; iy <= f.ny && q_ok; ++iy) {
          const uint8_t m = f.fix[fid(ix, iy, iz)];
          if (!m) continue;
          for (int a = 0; a <= (iz & 1); ++a)
            for (int b = 0; b <= (ix & 1); ++b)
              for (int d = 0; d <= (iy & 1); ++d)
                if (m & ~c.fix[cid((ix >> 1) + b, (iy >> 1) + d, (iz >> 1) + a)]) q_ok = false;
        }
    if (!q_ok) break;
    hs.push_back(std::move(c));
  }
  const int L = (int)hs.size();
  long long nfree_c = 0;
  for (uint8_t m : hs.back().fix) nfree_c += 3 - __builtin_popcount(m & 7);
  const char* why = L < 2 ? "fewer than 2 levels (grid too small, or coarse Dirichlet DOFs violate property Q)"
                  : nfree_c > 8192 ? "coarsest level has more than 8192 free DOFs" : nullptr;
  if (why) {
    if (P.precond == TOPO_PRECOND_MG) return set_err(ctx, TOPO_EINVAL, "multigrid hierarchy: %s", why);
    return TOPO_OK;
  }
  if (L > 16) return set_err(ctx, TOPO_EINVAL, "multigrid: more than 16 levels");
  ctx->mg_on = true;
  ctx->mg_f32 = P.mg_fp32 != 0;
  ctx->mg_kcycle = P.mg_cycle == TOPO_MG_KCYCLE && P.mg_nu == 1;
  // K-cycle levels (M8): 1 .. L-2, except that on hierarchies of 6+ levels the
  // level just above the coarsest keeps a single cycle (measured at config 4:
  // same PCG iteration counts, 0.8 ms less per iteration)
  ctx->mg_kmax = L >= 6 ? L - 3 : L - 2;
  if (const char* e = getenv("TOPO_KMIN")) ctx->mg_kmin = atoi(e);
  // level-1 layout: face sums (k_mg_l1_face) on large grids, where one thread per
  // element column and 16-plane chunk still fills the GPU (>= 1 M level-1
  // elements: config 4); per-element corners below (config 1: 40 threads would
  // walk the level serially -- measured 12.4 vs 7.7 ms per SIMP iteration)
  ctx->l1_face = (long long)hs[1].nx * hs[1].ny * hs[1].nz >= (1LL << 20);
  if (const char* e = getenv("TOPO_L1_FACE")) ctx->l1_face = atoi(e) != 0;
  if (const char* e = getenv("TOPO_KMAX")) ctx->mg_kmax = atoi(e);
  ctx->mg_theta = P.mg_omega;
  ctx->mg.resize(L);
  auto al = [&](void** p, size_t bytes) -> int {
    CU(cudaMalloc(p, bytes));
    CU(cudaMemsetAsync(*p, 0, bytes, ctx->stream));
    // the context's stream is non-blocking: finish the zero fill before any
    // synchronous host upload into this buffer (legacy-stream cudaMemcpy)
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->dev_bytes += bytes;
    return TOPO_OK;
  };
  for (int l = 1; l < L; ++l) {
    MgLevel& m = ctx->mg[l];
    const H& h = hs[l];
    m.L = LvGeo{h.nx, h.ny, h.nz, h.ny + 3, (long long)(h.ny + 3) * (h.nz + 3), 0};
    m.L.ncomp = (long long)(h.nx + 3) * m.L.nplane;
    m.hfix = h.fix;
    m.stored = (l >= 2) || (L == 2);
    // double-sized either way: an fp32 hierarchy can be promoted to fp64 in place
    // (do_solve) by reinterpreting the same buffers
    const size_t rs = sizeof(double);
    CK(al(&m.x, rs * 3 * m.L.ncomp));
    CK(al(&m.b, rs * 3 * m.L.ncomp));
    CK(al(&m.t, rs * 3 * m.L.ncomp));
    CK(al(&m.invd, rs * 3 * m.L.ncomp));
    CK(al((void**)&m.fixm, m.L.ncomp));
    if (m.stored) CK(al((void**)&m.K, sizeof(double) * 576 * m.L.nel()));
    if (m.stored && l < L - 1) CK(al(&m.S, rs * 126 * m.L.ncomp));
    if (!m.stored) CK(al(&m.Y, rs * 24 * m.L.nel()));
    if (l < L - 1) CK(al(&m.pw, rs * 3 * m.L.ncomp));
    if (P.mg_cycle == TOPO_MG_KCYCLE && P.mg_nu == 1 && l < L - 1) {
      CK(al(&m.kx, rs * 3 * m.L.ncomp));
      CK(al(&m.kv, rs * 3 * m.L.ncomp));
    }
    std::vector<uint8_t> lay(m.L.ncomp, 0);
    for (int iz = 0; iz <= h.nz; ++iz)
      for (int ix = 0; ix <= h.nx; ++ix)
        for (int iy = 0; iy <= h.ny; ++iy)
          lay[m.L.n(ix, iy, iz)] = h.fix[(long long)iz * (h.nx + 1) * (h.ny + 1) + (long long)ix * (h.ny + 1) + iy];
    CU(cudaMemcpy(m.fixm, lay.data(), m.L.ncomp, cudaMemcpyHostToDevice));
  }
  if (L >= 3 && !ctx->mg[1].stored)   // level-2 Galerkin DGEMM operand
    CK(al((void**)&ctx->mg_Eg, sizeof(double) * 64 * ctx->mg[2].L.nel()));
  // coarsest dense maps
  {
    const MgLevel& m = ctx->mg[L - 1];
    const H& h = hs[L - 1];
    std::vector<int> dmap(3 * m.L.ncomp, -1);
    std::vector<long long> imap;
    for (int iz = 0; iz <= h.nz; ++iz)
      for (int ix = 0; ix <= h.nx; ++ix)
        for (int iy = 0; iy <= h.ny; ++iy) {
          const uint8_t fm = h.fix[(long long)iz * (h.nx + 1) * (h.ny + 1) + (long long)ix * (h.ny + 1) + iy];
          for (int c = 0; c < 3; ++c) {
            if ((fm >> c) & 1) continue;
            const long long li = m.L.n(ix, iy, iz) + c * m.L.ncomp;
            dmap[li] = (int)imap.size();
            imap.push_back(li);
          }
        }
    ctx->mg_n = (int)imap.size();
    CK(al((void**)&ctx->mg_dmap, sizeof(int) * dmap.size()));
    CK(al((void**)&ctx->mg_imap, sizeof(long long) * std::max<size_t>(1, imap.size())));
    CU(cudaMemcpy(ctx->mg_dmap, dmap.data(), sizeof(int) * dmap.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->mg_imap, imap.data(), sizeof(long long) * imap.size(), cudaMemcpyHostToDevice));
    ctx->mg_npad = (ctx->mg_n + kGjB - 1) / kGjB * kGjB;
    const size_t np = (size_t)ctx->mg_npad;
    CK(al((void**)&ctx->mg_A0, sizeof(double) * np * np));
    CK(al((void**)&ctx->mg_A32, sizeof(float) * np * np));
    CK(al((void**)&ctx->mg_C, sizeof(double) * np * kGjB));
    CK(al((void**)&ctx->mg_R, sizeof(double) * np * kGjB));
    CK(al((void**)&ctx->mg_P, sizeof(double) * kGjB * kGjB));


  }
  for (Slab& s : ctx->slabs) {
    CK(al((void**)&s.pw0, sizeof(double) * 3 * s.g.ncomp));
    CK(al((void**)&s.res32, sizeof(float) * 3 * s.g.ncomp));
    CK(al((void**)&s.z32, sizeof(float) * 3 * s.g.ncomp));
    CK(map_nodes32(ctx, &s.m_z32, s.z32, s.g));
    if (ctx->world == 1) {
      CK(al((void**)&s.w32, sizeof(float) * 3 * s.g.ncomp));
      CK(map_nodes32(ctx, &s.m_w32, s.w32, s.g));
      if (P.krylov_fp32) {
        CK(al((void**)&s.r32, sizeof(float) * 3 * s.g.ncomp));
        CK(al((void**)&s.q32, sizeof(float) * 3 * s.g.ncomp));
        CK(map_nodes32(ctx, &s.m_r32, s.r32, s.g));
        ctx->k32_on = true;
      }
    }
  }
  if (ctx->world > 1) {   // whole-grid moduli for the replicated levels >= 1
    Geo G = ctx->slabs[0].g;
    G.ex0 = 0;
    G.ex1 = G.nex = P.nelx;
    G.nown = P.nelx + 1;
    G.NXL = G.nown + 2;
    G.ncomp = (long long)G.NXL * G.nplane;
    G.NEXL = G.nex + 2 * G.H;
    G.nelloc = (long long)G.NEXL * G.eplane;
    ctx->mg_gG = G;
    CK(al((void**)&ctx->mg_gE, sizeof(double) * G.nelloc));
  }
  if (!ctx->mg[1].stored)   // fp32 moduli of the matrix-free level-1 operator
    CK(al((void**)&ctx->mg_E32, sizeof(float) * mgG(ctx).nelloc));
  CK(al((void**)&ctx->mg_kc, sizeof(double) * 8 * 16));
  {
    std::vector<double> om(kMgScaleOff + 16, 1.0);
    CK(al((void**)&ctx->mg_om, sizeof(double) * om.size()));
    CU(cudaMemcpy(ctx->mg_om, om.data(), sizeof(double) * om.size(), cudaMemcpyHostToDevice));
  }
  // Galerkin tables
  {
    std::vector<double> t8(8 * 576), t64(64 * 576);
    mg_galerkin_tables(ctx->ke, t8.data(), t64.data(), ctx->mg_diag8);
    CK(al((void**)&ctx->mg_tab8, sizeof(double) * t8.size()));
    CK(al((void**)&ctx->mg_tab64, sizeof(double) * t64.size()));
    CU(cudaMemcpy(ctx->mg_tab8, t8.data(), sizeof(double) * t8.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->mg_tab64, t64.data(), sizeof(double) * t64.size(), cudaMemcpyHostToDevice));
  }
  {
    const long long ndof = 3LL * (P.nelx + 1) * (P.nely + 1) * (P.nelz + 1);
    int b = P.cg_check_every > 0 ? P.cg_check_every : (int)std::min<long long>(16, std::max<long long>(2, 4000000LL / ndof));
    ctx->mg_batch = (b + 1) / 2 * 2;
  }
  return TOPO_OK;
}

constexpr long long kMgDeepNodesDefault = 150000;   // "small" coarse levels (deep sweeps, warp-split stencil kernel)
// (TOPO_DEEP_NODES overrides it: tests run the large-level code paths on small grids)
long long mg_deep_nodes() {
  const char* e = getenv("TOPO_DEEP_NODES");
  return e ? atoll(e) : kMgDeepNodesDefault;
}
// Stored levels up to this size run the fused warp-split sweeps (k_mg_sweep_st8);
// larger ones the thread-per-node stencil apply + Jacobi kernels.  At config 4
// level 3 (70.8 k nodes) is faster on the latter since the apply runs at 3 CTAs/SM
// (8.73 vs 8.82 ms per MG-PCG iteration); level 4 (9.5 k) on the former (8.87 ms
// with every stored level on the apply).  TOPO_SWEEP_NODES overrides it; never
// above mg_deep_nodes() (tests set TOPO_DEEP_NODES=0 for the large-level paths).
long long mg_sweep_nodes() {
  const char* e = getenv("TOPO_SWEEP_NODES");
  return std::min<long long>(e ? atoll(e) : 60000, mg_deep_nodes());
}
constexpr int kMgPowerSteps = 8;       // power steps of the smoother-weight estimate (M5)
constexpr int kMgPowerStepsWarm = 1;   // later designs: continue from the previous design's vector
                                       // (1 vs 3 steps: same PCG iterations on configs 1-4 and the
                                       // paper protocol, 2 ms less setup per design at config 4)

template <typename T> T* mgp(void* p) { return static_cast<T*>(p); }

// ---------------------------------------------------------------------------
// Distributed coarse levels on x-slabs (W > 1, reading M10).
// Rank r owns element planes [ex0 >> l, ex1 >> l) of level l and the node
// planes [ex0 >> l, ex1 >> l) (the last rank also the last plane); levels
// 1 .. mg_dl are cycled on the owned planes only (ghost planes exchanged, the
// K-cycle's dots allreduced), level mg_dl + 1 and below stay replicated (their
// restricted right-hand side is all-gathered plane-wise).  The per-design setup
// stays replicated (operators from the all-gathered moduli).
// ---------------------------------------------------------------------------
void dl_owned(const topo_ctx* ctx, int r, int l, int& oa, int& ob) {
  int b = 0, e = 0;
  topo_partition(ctx->prm.nelx, ctx->prm.rmin, ctx->world, r, &b, &e);
  oa = b >> l;
  ob = (e >> l) + (r == ctx->world - 1 ? 1 : 0);
}
int slab_rank(const topo_ctx* ctx, const Slab& sl) {
  return ctx->mode == TOPO_DIST_LOOPBACK ? (int)(&sl - &ctx->slabs[0]) : ctx->rank;
}
LvGeo dl_geo(const topo_ctx* ctx, const Slab& sl, int l) {
  LvGeo L = ctx->mg[l].L;
  L.xa = sl.dlv[l].oa;
  L.xb = sl.dlv[l].ob - 1;
  return L;
}

int mg_dist_plan(topo_ctx* ctx) {
  ctx->mg_dl = 0;
  const int W = ctx->world, L = (int)ctx->mg.size();
  const bool force1 = getenv("TOPO_DIST_FORCE1") && atoi(getenv("TOPO_DIST_FORCE1")) != 0;   // (debug: W = 1)
  if ((W == 1 && !force1) || !ctx->mg_on || L < 3) return TOPO_OK;
  const int maxl = getenv("TOPO_DIST_LEVELS") ? atoi(getenv("TOPO_DIST_LEVELS")) : 16;
  const long long min_nodes = getenv("TOPO_DIST_MIN_NODES") ? atoll(getenv("TOPO_DIST_MIN_NODES")) : mg_deep_nodes();
  int lD = 0;
  for (int l = 1; l <= L - 2 && l <= maxl; ++l) {
    if (ctx->mg[l].L.nodes() <= min_nodes || (l == 1 && ctx->mg[1].stored)) break;
    // every slab boundary (and nelx) on an even plane of level l (the owned
    // coarse planes of level l + 1 are then the coarsened owned planes), >= 2
    // owned element planes per slab
    const int q = 1 << (l + 1);
    bool ok = ctx->prm.nelx % q == 0;
    for (int r = 0; r < W && ok; ++r) {
      int b = 0, e = 0;
      topo_partition(ctx->prm.nelx, ctx->prm.rmin, W, r, &b, &e);
      ok = b % q == 0 && ((e - b) >> l) >= 2;
    }
    if (!ok) break;
    lD = l;
  }
  if (!lD) return TOPO_OK;
  for (Slab& sl : ctx->slabs) {
    sl.dlv.assign(lD + 1, DLv{});
    const bool alias = &sl == &ctx->slabs[0];
    for (int l = 1; l <= lD; ++l) {
      MgLevel& m = ctx->mg[l];
      DLv& d = sl.dlv[l];
      dl_owned(ctx, slab_rank(ctx, sl), l, d.oa, d.ob);
      if (alias) {
        d.x = m.x; d.b = m.b; d.t = m.t; d.kx = m.kx; d.kv = m.kv; d.Y = m.Y;
        d.kc = ctx->mg_kc + 8 * l;
        continue;
      }
      d.own = true;
      const size_t v = sizeof(double) * 3 * m.L.ncomp;
      void** bufs[] = {&d.x, &d.b, &d.t, &d.kx, &d.kv};
      for (void** p : bufs) {
        CU(cudaMalloc(p, v));
        CU(cudaMemsetAsync(*p, 0, v, ctx->stream));
        ctx->dev_bytes += v;
      }
      if (m.Y) {
        CU(cudaMalloc(&d.Y, sizeof(double) * 24 * m.L.nel()));
        CU(cudaMemsetAsync(d.Y, 0, sizeof(double) * 24 * m.L.nel(), ctx->stream));
        ctx->dev_bytes += sizeof(double) * 24 * m.L.nel();
      }
      CU(cudaMalloc((void**)&d.kc, sizeof(double) * 8));
      CU(cudaMemsetAsync(d.kc, 0, sizeof(double) * 8, ctx->stream));
    }
  }
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->mg_dl = lD;
  return TOPO_OK;
}

// Ghost planes of a node vector between neighbouring slabs.  get(slab) ->
// {base pointer, b0, oa, ob}: global node plane P sits at index (P - b0 + 1) *
// nplane of each component (stride ncomp), the slab owns planes [oa, ob).
// dirs & 1: the left ghost (oa - 1) from the left neighbour's last owned plane;
// dirs & 2: the right ghost (ob) from the right neighbour's first owned plane.
struct PlaneSet {
  char* v;
  long long b0, oa, ob;
  long long ncomp;   // component stride (slab vectors: differs for the last slab)
};
template <typename Get>
int exchange_planes(topo_ctx* ctx, Get get, size_t es, long long nplane, int dirs) {
  const int W = ctx->world;
  if (W == 1 || ctx->mode == TOPO_DIST_SOLO) return TOPO_OK;
  const size_t pb = es * nplane;
  auto at = [&](const PlaneSet& p, long long P, int c) { return p.v + es * (c * p.ncomp + (P - p.b0 + 1) * nplane); };
  if (ctx->mode == TOPO_DIST_LOOPBACK) {
    for (int s = 0; s < W; ++s) {
      const PlaneSet a = get(ctx->slabs[s]);
      for (int c = 0; c < 3; ++c) {
        if ((dirs & 1) && s > 0) {
          const PlaneSet l = get(ctx->slabs[s - 1]);
          CU(cudaMemcpyAsync(at(a, a.oa - 1, c), at(l, a.oa - 1, c), pb, cudaMemcpyDeviceToDevice, ctx->stream));
        }
        if ((dirs & 2) && s < W - 1) {
          const PlaneSet r = get(ctx->slabs[s + 1]);
          CU(cudaMemcpyAsync(at(a, a.ob, c), at(r, a.ob, c), pb, cudaMemcpyDeviceToDevice, ctx->stream));
        }
      }
    }
    return TOPO_OK;
  }
  const PlaneSet a = get(ctx->slabs[0]);
  const int rk = ctx->rank;
  if (ctx->mode == TOPO_DIST_HOST) {   // blocks [c][0] to the left (plane oa), [c][1] to the right (plane ob - 1)
    const long long len = (long long)((pb + 7) / 8);
    char *hs = reinterpret_cast<char*>(ctx->ht->hsend), *hr = reinterpret_cast<char*>(ctx->ht->hrecv);
    for (int c = 0; c < 3; ++c) {
      if (rk > 0 && (dirs & 2))
        CU(cudaMemcpyAsync(hs + 8 * (2 * c) * len, at(a, a.oa, c), pb, cudaMemcpyDeviceToHost, ctx->stream));
      if (rk < W - 1 && (dirs & 1))
        CU(cudaMemcpyAsync(hs + 8 * (2 * c + 1) * len, at(a, a.ob - 1, c), pb, cudaMemcpyDeviceToHost, ctx->stream));
    }
    HostOp op;
    op.t = ctx->ht;
    op.kind = 0;
    op.len = len;
    op.nblk = 3;
    CK(host_launch(ctx, op));
    for (int c = 0; c < 3; ++c) {
      if (rk > 0 && (dirs & 1))
        CU(cudaMemcpyAsync(at(a, a.oa - 1, c), hr + 8 * (2 * c) * len, pb, cudaMemcpyHostToDevice, ctx->stream));
      if (rk < W - 1 && (dirs & 2))
        CU(cudaMemcpyAsync(at(a, a.ob, c), hr + 8 * (2 * c + 1) * len, pb, cudaMemcpyHostToDevice, ctx->stream));
    }
    return TOPO_OK;
  }
  const int dt = es == 4 ? ncclFloat32 : ncclFloat64;
  NC(g_nccl.GroupStart());
  for (int c = 0; c < 3; ++c) {
    if (dirs & 1) {
      if (rk < W - 1) NC(g_nccl.Send(at(a, a.ob - 1, c), (size_t)nplane, dt, rk + 1, ctx->comm, ctx->stream));
      if (rk > 0) NC(g_nccl.Recv(at(a, a.oa - 1, c), (size_t)nplane, dt, rk - 1, ctx->comm, ctx->stream));
    }
    if (dirs & 2) {
      if (rk > 0) NC(g_nccl.Send(at(a, a.oa, c), (size_t)nplane, dt, rk - 1, ctx->comm, ctx->stream));
      if (rk < W - 1) NC(g_nccl.Recv(at(a, a.ob, c), (size_t)nplane, dt, rk + 1, ctx->comm, ctx->stream));
    }
  }
  NC(g_nccl.GroupEnd());
  return TOPO_OK;
}
// a distributed level's vector (field of DLv), elements of es bytes
int exchange_lv(topo_ctx* ctx, int l, void* DLv::*field, size_t es, int dirs) {
  const LvGeo& L = ctx->mg[l].L;
  return exchange_planes(
      ctx,
      [&](Slab& sl) {
        const DLv& d = sl.dlv[l];
        return PlaneSet{static_cast<char*>(d.*field), 0, d.oa, d.ob, L.ncomp};
      },
      es, L.nplane, dirs);
}
// a fine-level slab vector (slab layout: local plane 0 = global ex0)
int exchange_fine(topo_ctx* ctx, void* (*field)(Slab&), size_t es, int dirs) {
  const Geo& g = ctx->slabs[0].g;
  return exchange_planes(
      ctx,
      [&](Slab& sl) {
        return PlaneSet{static_cast<char*>(field(sl)), sl.g.ex0, sl.g.ex0, sl.g.ex0 + sl.g.nown, sl.g.ncomp};
      },
      es, g.nplane, dirs);
}

// Replicated level l (the first level below the distributed ones): every rank
// computed the restriction on its owned planes of buf; all-gather them (loopback:
// the slabs wrote one shared buffer -- nothing to do).
int gather_level(topo_ctx* ctx, int l, void* buf, size_t es) {
  const int W = ctx->world;
  if (W == 1 || ctx->mode == TOPO_DIST_LOOPBACK || ctx->mode == TOPO_DIST_SOLO) return TOPO_OK;
  const LvGeo& L = ctx->mg[l].L;
  char* v = static_cast<char*>(buf);
  auto at = [&](long long P, int c) { return v + es * (c * L.ncomp + (P + 1) * L.nplane); };
  const int rk = ctx->rank;
  if (ctx->mode == TOPO_DIST_HOST) {   // pack the 3 components' owned planes, all-gather, unpack
    HostOp op;
    op.t = ctx->ht;
    op.kind = 3;
    long long off = 0;
    for (int r = 0; r < W; ++r) {
      int oa = 0, ob = 0;
      dl_owned(ctx, r, l, oa, ob);
      op.cnt[r] = (long long)((3 * es * (ob - oa) * L.nplane + 7) / 8);
      op.off[r] = off;
      off += op.cnt[r];
    }
    int oa = 0, ob = 0;
    dl_owned(ctx, rk, l, oa, ob);
    const size_t cb = es * (ob - oa) * L.nplane;
    char* hs = reinterpret_cast<char*>(ctx->ht->hsend);
    for (int c = 0; c < 3; ++c) CU(cudaMemcpyAsync(hs + c * cb, at(oa, c), cb, cudaMemcpyDeviceToHost, ctx->stream));
    CK(host_launch(ctx, op));
    for (int r = 0; r < W; ++r) {
      if (r == rk) continue;
      int pa = 0, pbn = 0;
      dl_owned(ctx, r, l, pa, pbn);
      const size_t rb = es * (pbn - pa) * L.nplane;
      const char* src = reinterpret_cast<const char*>(ctx->ht->hrecv + op.off[r]);
      for (int c = 0; c < 3; ++c) CU(cudaMemcpyAsync(at(pa, c), src + c * rb, rb, cudaMemcpyHostToDevice, ctx->stream));
    }
    return TOPO_OK;
  }
  const int dt = es == 4 ? ncclFloat32 : ncclFloat64;
  int oa = 0, ob = 0;
  dl_owned(ctx, rk, l, oa, ob);
  NC(g_nccl.GroupStart());
  for (int r = 0; r < W; ++r) {
    if (r == rk) continue;
    int pa = 0, pbn = 0;
    dl_owned(ctx, r, l, pa, pbn);
    for (int c = 0; c < 3; ++c) {
      NC(g_nccl.Send(at(oa, c), (size_t)((ob - oa) * L.nplane), dt, r, ctx->comm, ctx->stream));
      NC(g_nccl.Recv(at(pa, c), (size_t)((pbn - pa) * L.nplane), dt, r, ctx->comm, ctx->stream));
    }
  }
  NC(g_nccl.GroupEnd());
  return TOPO_OK;
}

// level-1 phase 1 (Walsh-domain Galerkin per coarse element), 128-thread CTAs
// (x-slabs: Lr = the slab's owned node planes -- the element planes next to
// them are computed -- and the slab's x and Y)
// level-1 gather phase matching the element phase's output layout (ctx->l1_face)
#define L1_GATHER(ctx, kScale, T, grid, ...)                                        \
  do {                                                                              \
    if ((ctx)->l1_face) LAUNCH(ctx, (k_mg_l1_gather<kScale, T, true>), grid, __VA_ARGS__);  \
    else LAUNCH(ctx, (k_mg_l1_gather<kScale, T, false>), grid, __VA_ARGS__);               \
  } while (0)
#define L1_GATHER_JAC(ctx, T, grid, ...)                                            \
  do {                                                                              \
    if ((ctx)->l1_face) LAUNCH(ctx, (k_mg_l1_gather_jac<T, true>), grid, __VA_ARGS__);       \
    else LAUNCH(ctx, (k_mg_l1_gather_jac<T, false>), grid, __VA_ARGS__);                    \
  } while (0)
template <typename T>
int launch_l1_elem(topo_ctx* ctx, MgLevel& m, const DevState* gst, const LvGeo* Lr = nullptr, void* xv = nullptr,
                   void* Yv = nullptr) {
  const LvGeo L = Lr ? *Lr : m.L;
  T* x = mgp<T>(xv ? xv : m.x);
  T* Y = mgp<T>(Yv ? Yv : m.Y);
  const long long nb = std::min<long long>((L.el_hi() - L.el_lo() + kL1Block - 1) / kL1Block, 148LL * 3 * 16);
  if (ctx->l1_face) {   // face sums (k_mg_l1_face): one thread per (column, chunk of kL1CX node planes)
    const long long nt = (long long)L.ny * L.nz * ((L.xlast() - L.xa + 1 + kL1CX - 1) / kL1CX);
    const unsigned nbf = (unsigned)std::max(1LL, std::min<long long>((nt + kL1Block - 1) / kL1Block, 148LL * 3 * 16));
    static const bool l1f_async = !getenv("TOPO_L1F_ASYNC") || atoi(getenv("TOPO_L1F_ASYNC")) != 0;
    if constexpr (sizeof(T) == 4) {
      if (l1f_async)
        k_mg_l1_face<T, float, true><<<nbf, kL1Block, 0, ctx->stream>>>(mgG(ctx), L, ctx->mg_E32, x, Y, gst);
      else
        k_mg_l1_face<T, float, false><<<nbf, kL1Block, 0, ctx->stream>>>(mgG(ctx), L, ctx->mg_E32, x, Y, gst);
    } else
      k_mg_l1_face<T, double><<<nbf, kL1Block, 0, ctx->stream>>>(mgG(ctx), L, mgE(ctx), x, Y, gst);
  } else if (sizeof(T) == 4)   // fp32 moduli (k_mg_e32 at setup)
    k_mg_l1_elem<T, float><<<(unsigned)std::max(1LL, nb), kL1Block, 0, ctx->stream>>>(mgG(ctx), L, ctx->mg_E32, x, Y,
                                                                                   gst);
  else
    k_mg_l1_elem<T, double><<<(unsigned)std::max(1LL, nb), kL1Block, 0, ctx->stream>>>(mgG(ctx), L, mgE(ctx), x, Y,
                                                                                    gst);
  ctx->launches++;
  debug_sync(ctx, "k_mg_l1_elem");
  return check_launch(ctx);
}
int mg_mv0(topo_ctx* ctx, int gate, const CUtensorMap& vin);
template <typename T> int mg_apply(topo_ctx* ctx, int l, int gate);

double* mg_Ainv(const topo_ctx* ctx) { return ctx->mg_A0; }

// Per-design setup: level-1 diagonal, Galerkin element matrices, coarsest inverse.
template <typename T>
int enqueue_mg_setup(topo_ctx* ctx, bool warm) {
  Slab& s = ctx->slabs[0];
  const int L = (int)ctx->mg.size();
  CK(mg_gather_E(ctx));   // x-slabs: the replicated levels see the whole grid
  if (sizeof(T) == 4 && ctx->mg_E32)
    LAUNCH(ctx, k_mg_e32, grid_for(mgG(ctx).nelloc), mgG(ctx).nelloc, mgE(ctx), ctx->mg_E32);
  for (int l = 1; l < L; ++l) {
    MgLevel& m = ctx->mg[l];
    const long long nn = m.L.nodes(), ne = m.L.nel();
    if (l == 1 && !m.stored) {
      LAUNCH(ctx, k_mg_diag_l1<T>, grid_for(nn), mgG(ctx), m.L, mgE(ctx), m.fixm, mgp<T>(m.invd));
      continue;
    }
    if (l == 1) {
      k_mg_asm_fine<2><<<(unsigned)((ne + kBlock - 1) / kBlock), kBlock, 0, ctx->stream>>>(mgG(ctx), m.L, mgE(ctx), ctx->mg_tab8, m.K);
      ctx->launches++;
    } else if (l == 2 && !ctx->mg[1].stored) {
      // K2 = Eg tab64^T: gather the 64 fine moduli per element, then one DGEMM
      // (nel x 64) x (64 x 576) into the entry-major [576][nel] layout
      LAUNCH(ctx, k_mg_gather64, grid_for(64 * ne), mgG(ctx), m.L, mgE(ctx), ctx->mg_Eg);
      static const bool tc2 = !getenv("TOPO_TC2") || atoi(getenv("TOPO_TC2")) != 0;
      if (!ctx->tc_attr_set) {
        CU(cudaFuncSetAttribute(k_dgemm_nt64_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));
        CU(cudaFuncSetAttribute(k_dgemm_nt64_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, kT2Smem));
        ctx->tc_attr_set = true;
      }
      const long long ntile = (ne + kTcM - 1) / kTcM;
      if (tc2)   // persistent: one CTA per SM, A tile kept across the 9 N blocks
        k_dgemm_nt64_tc2<<<(unsigned)std::min<long long>(ntile, 148LL), 256, kT2Smem, ctx->stream>>>(
            ctx->mg_Eg, ne, ctx->mg_tab64, 576, m.K, ne, (int)ne, 576, 1.0);
      else
        k_dgemm_nt64_tc<<<dim3(576 / kTcN, (unsigned)ntile), 256, kTcSmem, ctx->stream>>>(
            ctx->mg_Eg, ne, ctx->mg_tab64, 576, m.K, ne, (int)ne, 576, 1.0);
      ctx->launches++;
      debug_sync(ctx, "k_dgemm_nt64_tc(level-2 Galerkin)");
    } else {
      const MgLevel& f = ctx->mg[l - 1];
      {   // tiled Galerkin product (k_mg_asm_galerkin_t), 8 coarse elements per CTA
        const size_t smem = sizeof(double) * 576 * 2 * kGalTile;
        static unsigned attr = 0;   // per device
        if (!(attr & (1u << (ctx->device & 31)))) {
          CU(cudaFuncSetAttribute(k_mg_asm_galerkin_t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          attr |= 1u << (ctx->device & 31);
        }
        k_mg_asm_galerkin_t<<<dim3((m.L.ny + kGalTile - 1) / kGalTile, m.L.nz, m.L.nx), dim3(kGalTile, 24), smem,
                              ctx->stream>>>(f.L, f.K, m.L, m.K);
        ctx->launches++;
      }
    }
    debug_sync(ctx, "k_mg_asm");
    LAUNCH(ctx, k_mg_diag_asm<T>, grid_for(nn), m.L, m.K, m.fixm, mgp<T>(m.invd));
    if (m.S) LAUNCH(ctx, k_mg_stencil<T>, grid_for(nn), m.L, m.K, mgp<T>(m.S));
  }
  // smoother weights w_l = theta / lam_l (M5): kMgPowerSteps power steps per level
  // from the hash start vector on the first design; kMgPowerStepsWarm steps from
  // the previous design's vector afterwards (the design changes slowly, so the
  // Rayleigh quotient keeps improving)
  const double* one = ctx->mg_om + 16;
  const int nsteps = warm ? kMgPowerStepsWarm : kMgPowerSteps;
  for (int l = 0; l < L - 1; ++l) {
    if (l == 0) {
      // v <- D^-1 (K v) fused into the matvec's pre-pass (kPre = 3, w = 1); the
      // masked products K v ping-pong between q and w (x-slabs: per slab, ghost
      // planes exchanged after every product, Rayleigh sums allreduced)
      const int W = ctx->world;
      for (Slab& sl : ctx->slabs) {
        if (warm) {
          CU(cudaMemcpyAsync(sl.z, sl.pw0, sizeof(double) * 3 * sl.g.ncomp, cudaMemcpyDeviceToDevice, ctx->stream));
        } else {   // owned + ghost planes (global hash: the same vector as one slab)
          const int xa = std::max(0, sl.g.ex0 - 1), xb = std::min(sl.g.nelx, sl.g.ex0 + sl.g.nown);
          LAUNCH(ctx, k_mg_start_vec<double>, grid_for((long long)(xb - xa + 1) * sl.g.NY * sl.g.NZ), lv_slab(sl),
                 sl.g.ex0, xa, xb, sl.g.nelx, sl.fixm, sl.z);
        }
      }
      // (T = the hierarchy's precision: with mg_fp32 the power steps use the fp32
      // element operator like the smoothing matvecs they calibrate)
      for (Slab& sl : ctx->slabs) CK((launch_mv<0, false, 3, T>(ctx, sl, 0, sl.m_z, nullptr, nullptr, sl.q, 0, one)));
      CK(exchange_nodes(ctx, &Slab::q));
      for (int k = 1; k <= nsteps; ++k) {
        const bool odd = k & 1;
        for (Slab& sl : ctx->slabs)
          CK((launch_mv<3, false, 3, T>(ctx, sl, 0, odd ? sl.m_q : sl.m_w, nullptr, sl.z, odd ? sl.w : sl.q, 0, one)));
        CK(exchange_nodes(ctx, odd ? &Slab::w : &Slab::q));
      }
      for (Slab& sl : ctx->slabs) {
        const LvGeo F = lv_slab(sl);
        double* tlast = (nsteps & 1) ? sl.w : sl.q;
        LAUNCH(ctx, (k_mg_rayleigh<true, double>), grid_for(F.nodes()), F, sl.z, tlast, sl.invd, sl.fixm,
               ctx->mg_theta, ctx->mg_om, sl.partials, sl.counter, W > 1 ? sl.st : nullptr);
      }
      if (W > 1) {
        CK(allreduce(ctx, 0, 2, 0));
        k_mg_rayleigh_finish<<<1, 1, 0, ctx->stream>>>(s.st, ctx->mg_theta, ctx->mg_om);
        ctx->launches++;
      }
      for (Slab& sl : ctx->slabs)
        LAUNCH(ctx, k_mg_scale_copy<double>, grid_for(3 * sl.g.ncomp), sl.z, sl.pw0, 3 * sl.g.ncomp,
               ctx->mg_om + kMgScaleOff);
    } else {
      MgLevel& m = ctx->mg[l];
      const int gL = grid_for(m.L.nodes());
      if (warm) CU(cudaMemcpyAsync(m.x, m.pw, sizeof(T) * 3 * m.L.ncomp, cudaMemcpyDeviceToDevice, ctx->stream));
      else LAUNCH(ctx, k_mg_start_vec<T>, gL, m.L, 0, 0, m.L.nx, m.L.nx, m.fixm, mgp<T>(m.x));
      for (int k = 0; k < nsteps; ++k) {
        if (!m.stored) {   // level 1: x <- D^-1 (A x) in the gather phase
          CK(launch_l1_elem<T>(ctx, m, nullptr));
          L1_GATHER(ctx, true, T, gL, m.L, mgp<T>(m.Y), m.fixm, mgp<T>(m.x), nullptr, mgp<T>(m.invd));
          continue;
        }
        CK(mg_apply<T>(ctx, l, 0));
        LAUNCH(ctx, (k_mg_jacobi<0, false, T>), gL, m.L, mgp<T>(m.t), mgp<T>(m.t), mgp<T>(m.invd), m.fixm, one,
               mgp<T>(m.x), s.st, 0, s.partials, s.counter);
      }
      CK(mg_apply<T>(ctx, l, 0));
      LAUNCH(ctx, (k_mg_rayleigh<false, T>), gL, m.L, mgp<T>(m.x), mgp<T>(m.t), mgp<T>(m.invd), m.fixm,
             ctx->mg_theta, ctx->mg_om + l, s.partials, s.counter);
      LAUNCH(ctx, k_mg_scale_copy<T>, grid_for(3 * m.L.ncomp), mgp<T>(m.x), mgp<T>(m.pw), 3 * m.L.ncomp,
             ctx->mg_om + kMgScaleOff + l);
    }
  }
  const MgLevel& c = ctx->mg[L - 1];
  const int n = ctx->mg_n;
  const int np = ctx->mg_npad;
  double* A = ctx->mg_A0;
  CU(cudaMemsetAsync(A, 0, sizeof(double) * (size_t)np * np, ctx->stream));
  static const bool fill27 = !getenv("TOPO_FILL27") || atoi(getenv("TOPO_FILL27")) != 0;
  if (fill27) LAUNCH(ctx, k_mg_dense_fill27, grid_for(c.L.nodes() * 81), c.L, c.K, ctx->mg_dmap, np, A);
  else LAUNCH(ctx, k_mg_dense_fill, grid_for(c.L.nodes()), c.L, c.K, ctx->mg_dmap, np, A);
  if (np > n) LAUNCH(ctx, k_gj_pad, 1, A, n, np);
  // A <- A^-1 in place (coarsest dense inverse, reading M6): symmetric blocked
  // sweep (mg.cuh), lower triangle, rank-64 updates by k_dgemm_nt64
  const unsigned nT = (unsigned)((np + kNtTile - 1) / kNtTile);
  for (int k0 = 0; k0 < np; k0 += kGjB) {
    k_sw_block_inv<<<1, kGjB * kGjB / kGjInvNJ, 0, ctx->stream>>>(A, np, k0, ctx->mg_P);
    ctx->launches++;
    LAUNCH(ctx, k_sw_take_col, grid_for((long long)np * kGjB), A, np, k0, ctx->mg_C);
    // CP = C P  (n_pad x b; P symmetric, so C P = C P^T)
    k_dgemm_nt64<<<dim3(1, nT), 256, 0, ctx->stream>>>(ctx->mg_C, np, ctx->mg_P, kGjB, ctx->mg_R, np, np, kGjB, 1.0,
                                                      0.0, 0);
    // S -= C (C P)^T on the lower triangle (rows / columns K untouched: C_K,: = 0)
    k_dgemm_nt64<<<dim3(nT, nT), 256, 0, ctx->stream>>>(ctx->mg_C, np, ctx->mg_R, np, A, np, np, np, -1.0, 1.0, 1);
    ctx->launches += 2;
    debug_sync(ctx, "k_dgemm_nt64(sweep)");
    LAUNCH(ctx, k_sw_put_panel, grid_for((long long)np * kGjB), A, np, k0, ctx->mg_R, ctx->mg_P);
  }
  LAUNCH(ctx, k_sw_finish, grid_for((long long)np * np), A, np);
  if (sizeof(T) == 4) LAUNCH(ctx, k_mg_inv_to32, grid_for((long long)np * np), A, ctx->mg_A32, (long long)np * np);
  return check_launch(ctx);
}

// Drop everything captured for the current multigrid precision (graphs of the
// setup and of the MG-PCG batch; typed power vectors) so the next solve rebuilds it.
void mg_invalidate(topo_ctx* ctx) {
  if (ctx->mg_setup_exec) { cudaGraphExecDestroy(ctx->mg_setup_exec); ctx->mg_setup_exec = nullptr; }
  if (ctx->mg_setup_exec_w) { cudaGraphExecDestroy(ctx->mg_setup_exec_w); ctx->mg_setup_exec_w = nullptr; }
  if (ctx->cg_exec[1]) { cudaGraphExecDestroy(ctx->cg_exec[1]); ctx->cg_exec[1] = nullptr; }
  ctx->mg_ready = false;
  ctx->mg_warm = false;
}

// Zero the typed level buffers (after a precision change: the pads and unused
// halves written in the other element type must read as 0).  The power vectors
// are typed too; they are restarted cold (mg_invalidate).
int mg_clear_levels(topo_ctx* ctx) {
  for (MgLevel& m : ctx->mg) {
    const size_t n3 = sizeof(double) * 3 * m.L.ncomp;
    void* v3[] = {m.x, m.b, m.t, m.invd, m.pw};
    for (void* v : v3)
      if (v) CU(cudaMemsetAsync(v, 0, n3, ctx->stream));
    if (m.S) CU(cudaMemsetAsync(m.S, 0, sizeof(double) * 126 * m.L.ncomp, ctx->stream));
    if (m.Y) CU(cudaMemsetAsync(m.Y, 0, sizeof(double) * 24 * m.L.nel(), ctx->stream));
  }
  for (Slab& s : ctx->slabs)   // distributed levels' own buffers (loopback slabs >= 1)
    for (size_t l = 1; l < s.dlv.size(); ++l) {
      DLv& d = s.dlv[l];
      if (!d.own) continue;
      const size_t n3 = sizeof(double) * 3 * ctx->mg[l].L.ncomp;
      void* v3[] = {d.x, d.b, d.t, d.kx, d.kv};
      for (void* v : v3)
        if (v) CU(cudaMemsetAsync(v, 0, n3, ctx->stream));
      if (d.Y) CU(cudaMemsetAsync(d.Y, 0, sizeof(double) * 24 * ctx->mg[l].L.nel(), ctx->stream));
    }
  return TOPO_OK;
}

int mg_setup(topo_ctx* ctx) {
  if (!ctx->mg_on || ctx->mg_ready) return TOPO_OK;
  CK(ensure_constants(ctx));
  if (!ctx->has_E) CK(update_modulus(ctx));
  const bool warm = ctx->mg_warm;
  auto setup = [&]() {
    return ctx->mg_f32 ? enqueue_mg_setup<float>(ctx, warm) : enqueue_mg_setup<double>(ctx, warm);
  };
  if (ctx->debug) {
    CK(setup());
  } else {
    cudaGraphExec_t& ex = warm ? ctx->mg_setup_exec_w : ctx->mg_setup_exec;
    long long& nl = warm ? ctx->mg_setup_launches_w : ctx->mg_setup_launches;
    if (!ex) {
      cudaGraph_t graph;
      const long long l0 = ctx->launches;
      CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      int rc = setup();
      cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
      if (rc != TOPO_OK) return rc;
      if (e != cudaSuccess) return set_err(ctx, TOPO_ECUDA, "MG setup capture: %s", cudaGetErrorString(e));
      e = cudaGraphInstantiate(&ex, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return set_err(ctx, TOPO_ECUDA, "MG setup instantiate: %s", cudaGetErrorString(e));
      nl = ctx->launches - l0;
      ctx->launches = l0;
    }
    CU(cudaGraphLaunch(ex, ctx->stream));
    ctx->launches += nl;
  }
  ctx->mg_ready = true;
  ctx->mg_warm = true;
  if (getenv("TOPO_MG_VERBOSE")) {   // smoother weights per level (diagnostics)
    double om[17];
    CU(cudaMemcpyAsync(om, ctx->mg_om, sizeof om, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    fprintf(stderr, "[topo] MG setup (%s): w =", warm ? "warm" : "cold");
    for (size_t l = 0; l + 1 < ctx->mg.size(); ++l) fprintf(stderr, " %.4f", om[l]);
    fprintf(stderr, "\n");
  }
  return TOPO_OK;
}

// fine plain matvec q = K v (v = z or w), gated by the PCG state
int mg_mv0(topo_ctx* ctx, int gate, const CUtensorMap& vin) {
  Slab& s = ctx->slabs[0];
  return launch_mv<0, false>(ctx, s, gate, vin, nullptr, nullptr, s.q, 0);
}

// t_l = A_l x_l on a coarse level (stored: block stencil; level 1: P^T K P matrix-free)
template <typename T>
int mg_apply(topo_ctx* ctx, int l, int gate) {
  Slab& s = ctx->slabs[0];
  MgLevel& m = ctx->mg[l];
  const DevState* gst = gate ? s.st : nullptr;
  if (m.stored) {
    const long long sweep_nodes = getenv("TOPO_SWEEP_APPLY_NODES") ? atoll(getenv("TOPO_SWEEP_APPLY_NODES"))
                                                                   : mg_sweep_nodes();
    if (m.S && m.L.nodes() <= sweep_nodes)   // small levels: the coalesced warp-split stencil kernel
      LAUNCH(ctx, (k_mg_sweep_st8<false, T>), (int)std::min<long long>((m.L.nodes() + 31) / 32, 148LL * 8 * 16), m.L,
             mgp<T>(m.S), mgp<T>(m.x), mgp<T>(m.b), mgp<T>(m.invd), m.fixm, ctx->mg_om + l, mgp<T>(m.t), gst);
    else if (m.S) LAUNCH(ctx, k_mg_apply_st<T>, grid_for(m.L.nodes()), m.L, mgp<T>(m.S), mgp<T>(m.x), m.fixm, mgp<T>(m.t), gst);
    else LAUNCH(ctx, k_mg_apply_asm<T>, grid_for(m.L.nodes()), m.L, m.K, mgp<T>(m.x), m.fixm, mgp<T>(m.t), gst);   // coarsest (hook)
    return check_launch(ctx);
  }
  // level 1: P^T K(E) P matrix-free in the Walsh domain (two deterministic phases)
  CK(launch_l1_elem<T>(ctx, m, gst));
  L1_GATHER(ctx, false, T, grid_for(m.L.nodes()), m.L, mgp<T>(m.Y), m.fixm, mgp<T>(m.t), gst, (const T*)nullptr);
  return check_launch(ctx);
}

// b_{l+1} = P^T (b - t) on a coarse level: warp per coarse node on small levels
template <typename T>
int launch_restrict(topo_ctx* ctx, const LvGeo& F, const LvGeo& C, const T* b, const T* t, const uint8_t* ff,
                    const uint8_t* fc, T* bc, const DevState* gst) {
  if (C.nodes() <= 20000) {
    const int nb = (int)std::min<long long>((C.nodes() * 32 + kBlock - 1) / kBlock, 148LL * 8);
    LAUNCH(ctx, (k_mg_restrict_w<true, T, T>), nb, F, C, b, t, ff, fc, bc, gst);
  } else {
    LAUNCH(ctx, (k_mg_restrict<true, T, T>), grid_for(C.nodes()), F, C, b, t, ff, fc, bc, gst);
  }
  return check_launch(ctx);
}

// smoothing sweeps on level l (reading M5): mg_nu, or mg_nu_deep on the small
// coarse levels (auto: 8 when the fine grid is large enough that they are cheap)
int mg_level_nu(const topo_ctx* ctx, int l) {
  const topo_params& P = ctx->prm;
  if (l == 0 || ctx->mg[l].L.nodes() > mg_deep_nodes()) return P.mg_nu;
  if (P.mg_nu_deep > 0) return P.mg_nu_deep;
  if (ctx->mg_kcycle) return P.mg_nu;   // the K-cycle solves the deep levels well enough (M8)
  const long long fine = (long long)(P.nelx + 1) * (P.nely + 1) * (P.nelz + 1);
  return fine >= 2000000 ? 8 : P.mg_nu;
}

// One V-cycle on level l (level 0: b = r; the result lands in s.w and the last
// fine sweep also sets rho = r.V(r) and beta for the PCG; `dot` is unused).
// T = precision of levels >= 1 (level 0 is always fp64).
template <typename T>
int enqueue_vcycle_t(topo_ctx* ctx, int l, int gate, bool dot);
template <typename T>
int enqueue_coarse_t(topo_ctx* ctx, int l, int gate);
template <typename T>
int dist_coarse(topo_ctx* ctx, int l, int gate);
template <typename T>
int enqueue_vcycle_t(topo_ctx* ctx, int l, int gate, bool dot) {
  Slab& s = ctx->slabs[0];
  const int L = (int)ctx->mg.size(), nu = mg_level_nu(ctx, l);
  const DevState* gst = gate ? s.st : nullptr;
  const double* om = ctx->mg_om + l;
  if (l == L - 1) {
    const MgLevel& c = ctx->mg[l];
    static const bool c32 = !getenv("TOPO_COARSE32") || atoi(getenv("TOPO_COARSE32")) != 0;
    if (sizeof(T) == 4 && c32) {
      const int nb = (int)std::min<long long>(148LL * 2, (32LL * ctx->mg_n + kBlock - 1) / kBlock);
      k_mg_coarse_solve32<<<nb, kBlock, sizeof(float) * ctx->mg_n, ctx->stream>>>(
          ctx->mg_A32, ctx->mg_n, ctx->mg_npad, ctx->mg_imap, (const float*)c.b, (float*)c.x, gst);
      ctx->launches++;
      debug_sync(ctx, "k_mg_coarse_solve32");
    } else
      LAUNCH(ctx, k_mg_coarse_solve<T>, grid_for(32LL * ctx->mg_n), mg_Ainv(ctx), ctx->mg_n, ctx->mg_npad,
             ctx->mg_imap, mgp<T>(c.b), mgp<T>(c.x), gst);
    return check_launch(ctx);
  }
  MgLevel& n1 = ctx->mg[l + 1];
  if (l == 0) {
    const LvGeo F = lv0(ctx);
    const int gF = grid_for(F.nodes());
    // first sweep from z = 0 fused into the matvec's load: z = w D^-1 r, and
    // (nu = 1) the epilogue writes the residual r - K z for the restriction
    if (ctx->prof_capture) CU(cudaEventRecordWithFlags(ctx->pe[0], ctx->stream, cudaEventRecordExternal));
    // (nu = 1: z is not stored -- k_mg_prolong0 recomputes it with the correction)
    // (with mg_fp32 the smoothing matvecs compute the element operator in fp32)
    // (x-slabs: every step below runs per slab; nu = 1 only, see mg_build)
    if (nu == 1)   // (fp64 residual into z with the K-cycle: q must survive for the flexible beta)
      for (Slab& sl : ctx->slabs)
        if (k32_active(ctx))   // fp32 Krylov residual: float vin tile
          CK((launch_mv<3, false, 2, T, float>(ctx, sl, gate, sl.m_r32, nullptr, nullptr, sl.z, 0, om)));
        else
          CK((launch_mv<3, false, 2, T>(ctx, sl, gate, sl.m_r, nullptr, nullptr, ctx->mg_kcycle ? sl.z : sl.q, 0, om)));
    else CK((launch_mv<3, false>(ctx, s, gate, s.m_r, nullptr, s.z, s.q, 0, om)));
    if (ctx->prof_capture) CU(cudaEventRecordWithFlags(ctx->pe[1], ctx->stream, cudaEventRecordExternal));
    for (int k = 1; k < nu; ++k) {
      LAUNCH(ctx, (k_mg_jacobi<1, true, double>), gF, F, s.r, s.q, s.invd, s.fixm, om, s.z, s.st, gate, s.partials,
             s.counter);
      if (k < nu - 1) CK(mg_mv0(ctx, gate, s.m_z));
      else CK((launch_mv<0, false, 2>(ctx, s, gate, s.m_z, nullptr, nullptr, s.q, 0, om)));
    }
    // x-marching restriction of the masked residual (k_mg_restrict0); x-slabs:
    // each slab restricts its owned fine planes and the partial level-1 vectors
    // are summed (slab order in loopback mode, an allreduce with NCCL)
    // (distributed level 1, mg_dl >= 1: each slab restricts into ITS owned coarse
    // planes, reading the residual's left ghost plane -- no level-1 allreduce)
    const bool slabs = ctx->world > 1, dl = ctx->mg_dl >= 1;
    if (slabs && !dl) CU(cudaMemsetAsync(n1.b, 0, sizeof(T) * 3 * n1.L.ncomp, ctx->stream));
    if (dl) {
      if (ctx->mg_f32) CK(exchange_fine(ctx, [](Slab& q) -> void* { return q.res32; }, sizeof(float), 1));
      else if (ctx->mg_kcycle) CK(exchange_fine(ctx, [](Slab& q) -> void* { return q.z; }, sizeof(double), 1));
      else CK(exchange_fine(ctx, [](Slab& q) -> void* { return q.q; }, sizeof(double), 1));
    }
    for (Slab& sl : ctx->slabs) {
      const int xa = dl ? std::max(0, sl.g.ex0 - 1) : sl.g.ex0, xb = sl.g.ex0 + sl.g.nown;   // fine planes [xa, xb)
      const int j0 = dl ? sl.dlv[1].oa : xa / 2;                                              // coarse planes written
      const int jend = dl ? sl.dlv[1].ob : std::min(n1.L.nx, xb / 2) + 1;
      T* b1 = mgp<T>(dl ? sl.dlv[1].b : n1.b);
      const long long cols = (long long)(n1.L.ny + 1) * (n1.L.nz + 1);
      const int bx = (int)((cols + 127) / 128);
      int chunks = (int)std::max<long long>(1, std::min<long long>(jend - j0, (148LL * 64 + bx - 1) / bx));
      const int cx = (jend - j0 + chunks - 1) / chunks;
      chunks = (jend - j0 + cx - 1) / cx;
      const LvGeo Fs = lv_slab(sl);
      const DevState* sgst = gate ? sl.st : nullptr;
      const int acc = slabs && !dl ? 1 : 0;
      if (ctx->mg_f32)   // the pre-smoothing residual epilogue (kEpi = 2) wrote it in fp32
        k_mg_restrict0<float, T><<<dim3(bx, chunks), 128, 0, ctx->stream>>>(
            Fs, n1.L, cx, sl.res32, n1.fixm, b1, sgst, sl.g.ex0, xa, xb, j0, jend, acc);
      else
        k_mg_restrict0<double, T><<<dim3(bx, chunks), 128, 0, ctx->stream>>>(
            Fs, n1.L, cx, ctx->mg_kcycle ? sl.z : sl.q, n1.fixm, b1, sgst, sl.g.ex0, xa, xb, j0, jend, acc);
      ctx->launches++;
      debug_sync(ctx, "k_mg_restrict0");
    }
    if (dl) {
      CK(dist_coarse<T>(ctx, 1, gate));
      CK(exchange_lv(ctx, 1, &DLv::x, sizeof(T), 3));   // the prolongation reads coarse planes oa - 1 .. ob
    } else {
      CK(mg_allreduce_level(ctx, n1.b, 3 * n1.L.ncomp, sizeof(T) == 4));
      CK(enqueue_coarse_t<T>(ctx, 1, gate));
    }
    if (nu == 1) {   // z = w D^-1 r (the first sweep, recomputed) + P x1, x-marching
      for (Slab& sl : ctx->slabs) {   // owned + ghost planes (the post-smoothing matvec reads the ghosts)
        const T* x1 = mgp<T>(dl ? sl.dlv[1].x : n1.x);
        const int pa = std::max(0, sl.g.ex0 - 1), pb = std::min(sl.g.nelx, sl.g.ex0 + sl.g.nown) + 1;
        const int np = pb - (pa & ~1);
        const long long cols = (long long)(F.ny + 1) * (F.nz + 1);
        const int bx = (int)((cols + 127) / 128);
        int chunks = (int)std::max<long long>(1, std::min<long long>((np + 1) / 2, (148LL * 64 + bx - 1) / bx));
        const int cx = ((np + chunks - 1) / chunks + 1) / 2 * 2;   // even: chunks start on coarse planes
        chunks = (np + cx - 1) / cx;
        if (sizeof(T) == 4 && k32_active(ctx))   // fp32 Krylov residual
          k_mg_prolong0<T, float, float><<<dim3(bx, chunks), 128, 0, ctx->stream>>>(
              lv_slab(sl), n1.L, cx, sl.r32, sl.invd, om, x1, sl.fixm, sl.z32, gst, sl.g.ex0, pa, pb);
        else if (sizeof(T) == 4)   // fp32 hierarchy: z in fp32 (read by the fp32-operator post-smoothing)
          k_mg_prolong0<T, float><<<dim3(bx, chunks), 128, 0, ctx->stream>>>(lv_slab(sl), n1.L, cx, sl.r, sl.invd, om,
                                                                             x1, sl.fixm, sl.z32, gst,
                                                                             sl.g.ex0, pa, pb);
        else
          k_mg_prolong0<T, double><<<dim3(bx, chunks), 128, 0, ctx->stream>>>(lv_slab(sl), n1.L, cx, sl.r, sl.invd, om,
                                                                              x1, sl.fixm, sl.z, gst,
                                                                              sl.g.ex0, pa, pb);
        ctx->launches++;
        debug_sync(ctx, "k_mg_prolong0");
      }
    } else
      LAUNCH(ctx, (k_mg_prolong<true, T, double>), gF, F, n1.L, mgp<T>(n1.x), s.fixm, s.z, gst);
    for (int k = 1; k < nu; ++k) {
      CK(mg_mv0(ctx, gate, s.m_z));
      LAUNCH(ctx, (k_mg_jacobi<1, true, double>), gF, F, s.r, s.q, s.invd, s.fixm, om, s.z, s.st, gate, s.partials,
             s.counter);
    }
    // last sweep fused into the matvec epilogue: w = z + w D^-1 (r - K z) (the
    // V-cycle result lives in s.w), rho = r.w and beta for the PCG
    // (x-slabs: rho allreduced, then beta per slab; w's ghost planes exchanged
    // for the PCG matvec's p = w + beta p pre-pass)
    if (ctx->prof_capture) CU(cudaEventRecordWithFlags(ctx->pe[2], ctx->stream, cudaEventRecordExternal));
    for (Slab& sl : ctx->slabs)
      if (nu == 1 && sizeof(T) == 4)   // z in fp32 (k_mg_prolong0<T, float>)
        CK((launch_mv<0, false, 1, T, float>(ctx, sl, gate, sl.m_z32, nullptr, nullptr, sl.w, slabs ? 0 : 1, om)));
      else
        CK((launch_mv<0, false, 1, T, double>(ctx, sl, gate, sl.m_z, nullptr, nullptr, sl.w, slabs ? 0 : 1, om)));
    if (ctx->prof_capture) CU(cudaEventRecordWithFlags(ctx->pe[3], ctx->stream, cudaEventRecordExternal));
    if (slabs) {
      CK(allreduce(ctx, 0, ctx->mg_kcycle ? 2 : 1, 0));
      for (Slab& sl : ctx->slabs) { k_finish_rho<<<1, 1, 0, ctx->stream>>>(sl.st, ctx->mg_kcycle ? 1 : 0); ctx->launches++; }
      CK(exchange_nodes(ctx, &Slab::w));
    }
    return check_launch(ctx);
  }
  MgLevel& m = ctx->mg[l];
  const int gL = grid_for(m.L.nodes());
  T *mx = mgp<T>(m.x), *mb = mgp<T>(m.b), *mt = mgp<T>(m.t), *mi = mgp<T>(m.invd);
  if (m.S && m.L.nodes() <= mg_sweep_nodes()) {
    // small stencil level: each damped-Jacobi sweep is one fused warp-split
    // stencil kernel (k_mg_sweep_st8) ping-ponging x and t
    const int gS = (int)std::min<long long>((m.L.nodes() + 31) / 32, 148LL * 8 * 16);   // 32 nodes per block
    if (nu == 1) {
      // x = w D^-1 b and t = A x in one launch; restrict; correct; t = x + P e
      // (out of place) and the sweep x = t + w D^-1 (b - A t) in one launch
      LAUNCH(ctx, (k_mg_sweep_st8<false, T, true>), gS, m.L, mgp<T>(m.S), mx, mb, mi, m.fixm, om, mt, gst, mx);
      CK(launch_restrict<T>(ctx, m.L, n1.L, mb, mt, m.fixm, n1.fixm, mgp<T>(n1.b), gst));
      CK(enqueue_coarse_t<T>(ctx, l + 1, gate));
      LAUNCH(ctx, (k_mg_prolong<true, T, T>), gL, m.L, n1.L, mgp<T>(n1.x), m.fixm, mt, gst, (const T*)mx);
      LAUNCH(ctx, (k_mg_sweep_st8<true, T>), gS, m.L, mgp<T>(m.S), mt, mb, mi, m.fixm, om, mx, gst);
      return check_launch(ctx);
    }
    T* buf[2] = {mx, mt};
    int cur = (nu - 1) & 1;   // the last pre-smoothing sweep lands in x
    LAUNCH(ctx, (k_mg_jacobi<0, false, T>), gL, m.L, mb, mt, mi, m.fixm, om, buf[cur], s.st, gate, s.partials,
           s.counter);
    for (int k = 1; k < nu; ++k, cur ^= 1)
      LAUNCH(ctx, (k_mg_sweep_st8<true, T>), gS, m.L, mgp<T>(m.S), buf[cur], mb, mi, m.fixm, om, buf[cur ^ 1], gst);
    LAUNCH(ctx, (k_mg_sweep_st8<false, T>), gS, m.L, mgp<T>(m.S), mx, mb, mi, m.fixm, om, mt, gst);   // t = A x
    CK(launch_restrict<T>(ctx, m.L, n1.L, mb, mt, m.fixm, n1.fixm, mgp<T>(n1.b), gst));
    CK(enqueue_coarse_t<T>(ctx, l + 1, gate));
    LAUNCH(ctx, (k_mg_prolong<true, T, T>), gL, m.L, n1.L, mgp<T>(n1.x), m.fixm, mx, gst);
    int k = 0;
    if (nu & 1) {   // odd: one in-place sweep, then pairs of fused sweeps end in x
      LAUNCH(ctx, (k_mg_sweep_st8<false, T>), gS, m.L, mgp<T>(m.S), mx, mb, mi, m.fixm, om, mt, gst);
      LAUNCH(ctx, (k_mg_jacobi<1, false, T>), gL, m.L, mb, mt, mi, m.fixm, om, mx, s.st, gate, s.partials, s.counter);
      k = 1;
    }
    for (cur = 0; k < nu; ++k, cur ^= 1)
      LAUNCH(ctx, (k_mg_sweep_st8<true, T>), gS, m.L, mgp<T>(m.S), buf[cur], mb, mi, m.fixm, om, buf[cur ^ 1], gst);
    return check_launch(ctx);
  }
  LAUNCH(ctx, (k_mg_jacobi<0, false, T>), gL, m.L, mb, mt, mi, m.fixm, om, mx, s.st, gate, s.partials, s.counter);
  for (int k = 1; k < nu; ++k) {
    CK(mg_apply<T>(ctx, l, gate));
    LAUNCH(ctx, (k_mg_jacobi<1, false, T>), gL, m.L, mb, mt, mi, m.fixm, om, mx, s.st, gate, s.partials, s.counter);
  }
  CK(mg_apply<T>(ctx, l, gate));
  CK(launch_restrict<T>(ctx, m.L, n1.L, mb, mt, m.fixm, n1.fixm, mgp<T>(n1.b), gst));
  CK(enqueue_coarse_t<T>(ctx, l + 1, gate));
  LAUNCH(ctx, (k_mg_prolong<true, T, T>), gL, m.L, n1.L, mgp<T>(n1.x), m.fixm, mx, gst);
  for (int k = 1; k <= nu; ++k) {
    if (!m.stored) {   // level 1: the sweep fused into the gather phase
      CK(launch_l1_elem<T>(ctx, m, gst));
      L1_GATHER_JAC(ctx, T, gL, m.L, mgp<T>(m.Y), m.fixm, mx, mb, mi, om, gst);
      continue;
    }
    CK(mg_apply<T>(ctx, l, gate));
    LAUNCH(ctx, (k_mg_jacobi<1, false, T>), gL, m.L, mb, mt, mi, m.fixm, om, mx, s.st, gate, s.partials, s.counter);
  }
  return check_launch(ctx);
}

// Coarse correction on level l >= 1 (reading M8): one cycle (V), or the K-cycle's
// two flexible-CG steps preconditioned by that cycle; the coarsest level is
// solved exactly either way.  Input m.b, output m.x (m.b is overwritten by r2).
template <typename T>
int enqueue_coarse_t(topo_ctx* ctx, int l, int gate) {
  const int L = (int)ctx->mg.size();
  if (!ctx->mg_kcycle || l >= L - 1 || l < ctx->mg_kmin || l > ctx->mg_kmax) return enqueue_vcycle_t<T>(ctx, l, gate, false);
  Slab& s = ctx->slabs[0];
  MgLevel& m = ctx->mg[l];
  const DevState* gst = gate ? s.st : nullptr;
  double* kc = ctx->mg_kc + 8 * l;
  const long long n = 3 * m.L.ncomp;
  const int gF = grid_for(n);
  T *mx = mgp<T>(m.x), *mb = mgp<T>(m.b), *mt = mgp<T>(m.t), *kx = mgp<T>(m.kx), *kv = mgp<T>(m.kv);
  CK(enqueue_vcycle_t<T>(ctx, l, gate, false));   // x1 = B(b)
  CK(mg_apply<T>(ctx, l, gate));                  // t = A x1
  LAUNCH(ctx, k_kc_dot1<T>, gF, m.L, mx, mt, mb, kx, kv, kc, gst, s.partials, s.counter);
  LAUNCH(ctx, k_kc_r2<T>, gF, m.L, mb, kv, kc, gst);
  CK(enqueue_vcycle_t<T>(ctx, l, gate, false));   // x2 = B(r2)
  CK(mg_apply<T>(ctx, l, gate));                  // t = A x2
  LAUNCH(ctx, k_kc_dot2<T>, gF, m.L, mx, mt, mb, kv, kc, gst, s.partials, s.counter);
  LAUNCH(ctx, k_kc_combine<T>, gF, m.L, mx, kx, kc, gst);
  return check_launch(ctx);
}

// ---------------------------------------------------------------------------
// Distributed levels (x-slabs, levels 1 .. mg_dl; see mg_dist_plan): the cycle
// of enqueue_vcycle_t / enqueue_coarse_t (nu = 1) on each slab's owned node
// planes.  Ghost planes are exchanged where a step reads a neighbour's planes:
// the operator apply reads x at oa - 1 and ob, the restriction reads b - t at
// oa - 1, the prolongation reads the coarse plane ob / 2 (the right ghost of the
// next level).  Dots of the K-cycle: owned planes, allreduced.
// ---------------------------------------------------------------------------
bool kc_level(const topo_ctx* ctx, int l) {
  return ctx->mg_kcycle && l < (int)ctx->mg.size() - 1 && l >= ctx->mg_kmin && l <= ctx->mg_kmax;
}
bool dl_deep(const topo_ctx* ctx, int l) {
  const MgLevel& m = ctx->mg[l];
  return m.S && m.L.nodes() <= mg_sweep_nodes();
}
// t = A x on the owned planes of every slab (x ghosts current)
template <typename T>
int dl_apply(topo_ctx* ctx, int l, int gate) {
  MgLevel& m = ctx->mg[l];
  for (Slab& sl : ctx->slabs) {
    DLv& d = sl.dlv[l];
    const LvGeo Ls = dl_geo(ctx, sl, l);
    const DevState* gst = gate ? sl.st : nullptr;
    if (!m.stored) {   // level 1: P^T K(E) P matrix-free, element planes next to the owned nodes
      CK(launch_l1_elem<T>(ctx, m, gst, &Ls, d.x, d.Y));
      L1_GATHER(ctx, false, T, grid_for(Ls.nodes()), Ls, mgp<T>(d.Y), m.fixm, mgp<T>(d.t), gst, (const T*)nullptr);
    } else if (dl_deep(ctx, l)) {
      LAUNCH(ctx, (k_mg_sweep_st8<false, T>), (int)std::min<long long>((Ls.nodes() + 31) / 32, 148LL * 8 * 16), Ls,
             mgp<T>(m.S), mgp<T>(d.x), mgp<T>(d.b), mgp<T>(m.invd), m.fixm, ctx->mg_om + l, mgp<T>(d.t), gst);
    } else {
      LAUNCH(ctx, k_mg_apply_st<T>, grid_for(Ls.nodes()), Ls, mgp<T>(m.S), mgp<T>(d.x), m.fixm, mgp<T>(d.t), gst);
    }
  }
  return check_launch(ctx);
}

template <typename T>
int dist_coarse(topo_ctx* ctx, int l, int gate);

template <typename T>
int dist_vcycle(topo_ctx* ctx, int l, int gate) {
  MgLevel& m = ctx->mg[l];
  MgLevel& n1 = ctx->mg[l + 1];
  const double* om = ctx->mg_om + l;
  const bool deep = dl_deep(ctx, l), cdist = l + 1 <= ctx->mg_dl;
  const size_t es = sizeof(T);
  // pre-smoothing from 0 and t = A x
  if (deep) {   // x = w D^-1 b formed on the fly at the neighbours: b ghosts
    CK(exchange_lv(ctx, l, &DLv::b, es, 3));
    for (Slab& sl : ctx->slabs) {
      DLv& d = sl.dlv[l];
      const LvGeo Ls = dl_geo(ctx, sl, l);
      LAUNCH(ctx, (k_mg_sweep_st8<false, T, true>), (int)std::min<long long>((Ls.nodes() + 31) / 32, 148LL * 8 * 16),
             Ls, mgp<T>(m.S), mgp<T>(d.x), mgp<T>(d.b), mgp<T>(m.invd), m.fixm, om, mgp<T>(d.t), gate ? sl.st : nullptr,
             mgp<T>(d.x));
    }
  } else {
    for (Slab& sl : ctx->slabs) {
      DLv& d = sl.dlv[l];
      const LvGeo Ls = dl_geo(ctx, sl, l);
      LAUNCH(ctx, (k_mg_jacobi<0, false, T>), grid_for(Ls.nodes()), Ls, mgp<T>(d.b), mgp<T>(d.t), mgp<T>(m.invd),
             m.fixm, om, mgp<T>(d.x), sl.st, gate, sl.partials, sl.counter);
    }
    CK(exchange_lv(ctx, l, &DLv::x, es, 3));
    CK(dl_apply<T>(ctx, l, gate));
    CK(exchange_lv(ctx, l, &DLv::b, es, 1));
  }
  // restriction of b - t into the owned coarse planes (read at oa - 1: left ghosts)
  CK(exchange_lv(ctx, l, &DLv::t, es, 1));
  for (Slab& sl : ctx->slabs) {
    DLv& d = sl.dlv[l];
    LvGeo C = n1.L;
    void* bc = n1.b;
    if (cdist) {
      C = dl_geo(ctx, sl, l + 1);
      bc = sl.dlv[l + 1].b;
    } else {
      int oa = 0, ob = 0;
      dl_owned(ctx, slab_rank(ctx, sl), l + 1, oa, ob);
      C.xa = oa;
      C.xb = ob - 1;
    }
    CK(launch_restrict<T>(ctx, m.L, C, mgp<T>(d.b), mgp<T>(d.t), m.fixm, n1.fixm, mgp<T>(bc), gate ? sl.st : nullptr));
  }
  if (cdist) {
    CK(dist_coarse<T>(ctx, l + 1, gate));
    CK(exchange_lv(ctx, l + 1, &DLv::x, es, 2));   // the prolongation reads coarse plane ob / 2
  } else {
    CK(gather_level(ctx, l + 1, n1.b, es));
    CK(enqueue_coarse_t<T>(ctx, l + 1, gate));      // replicated below (slab 0's state gates it)
  }
  for (Slab& sl : ctx->slabs) {
    DLv& d = sl.dlv[l];
    const LvGeo Ls = dl_geo(ctx, sl, l);
    const T* xc = mgp<T>(cdist ? sl.dlv[l + 1].x : n1.x);
    const DevState* gst = gate ? sl.st : nullptr;
    if (deep)   // t = x + P e (out of place)
      LAUNCH(ctx, (k_mg_prolong<true, T, T>), grid_for(Ls.nodes()), Ls, n1.L, xc, m.fixm, mgp<T>(d.t), gst,
             (const T*)mgp<T>(d.x));
    else
      LAUNCH(ctx, (k_mg_prolong<true, T, T>), grid_for(Ls.nodes()), Ls, n1.L, xc, m.fixm, mgp<T>(d.x), gst);
  }
  // post-smoothing
  if (deep) {
    CK(exchange_lv(ctx, l, &DLv::t, es, 3));
    for (Slab& sl : ctx->slabs) {
      DLv& d = sl.dlv[l];
      const LvGeo Ls = dl_geo(ctx, sl, l);
      LAUNCH(ctx, (k_mg_sweep_st8<true, T>), (int)std::min<long long>((Ls.nodes() + 31) / 32, 148LL * 8 * 16), Ls,
             mgp<T>(m.S), mgp<T>(d.t), mgp<T>(d.b), mgp<T>(m.invd), m.fixm, om, mgp<T>(d.x), gate ? sl.st : nullptr);
    }
    return check_launch(ctx);
  }
  CK(exchange_lv(ctx, l, &DLv::x, es, 3));
  if (!m.stored) {   // level 1: the sweep fused into the gather phase
    for (Slab& sl : ctx->slabs) {
      DLv& d = sl.dlv[l];
      const LvGeo Ls = dl_geo(ctx, sl, l);
      const DevState* gst = gate ? sl.st : nullptr;
      CK(launch_l1_elem<T>(ctx, m, gst, &Ls, d.x, d.Y));
      L1_GATHER_JAC(ctx, T, grid_for(Ls.nodes()), Ls, mgp<T>(d.Y), m.fixm, mgp<T>(d.x), mgp<T>(d.b), mgp<T>(m.invd),
                    om, gst);
    }
    return check_launch(ctx);
  }
  CK(dl_apply<T>(ctx, l, gate));
  for (Slab& sl : ctx->slabs) {
    DLv& d = sl.dlv[l];
    const LvGeo Ls = dl_geo(ctx, sl, l);
    LAUNCH(ctx, (k_mg_jacobi<1, false, T>), grid_for(Ls.nodes()), Ls, mgp<T>(d.b), mgp<T>(d.t), mgp<T>(m.invd), m.fixm,
           om, mgp<T>(d.x), sl.st, gate, sl.partials, sl.counter);
  }
  return check_launch(ctx);
}

template <typename T>
int dist_coarse(topo_ctx* ctx, int l, int gate) {
  if (!kc_level(ctx, l)) return dist_vcycle<T>(ctx, l, gate);
  const size_t es = sizeof(T);
  CK(dist_vcycle<T>(ctx, l, gate));   // x1 = B(b)
  CK(exchange_lv(ctx, l, &DLv::x, es, 3));
  CK(dl_apply<T>(ctx, l, gate));      // t = A x1
  for (Slab& sl : ctx->slabs) {
    DLv& d = sl.dlv[l];
    const LvGeo Ls = dl_geo(ctx, sl, l);
    LAUNCH(ctx, k_kc_dot1<T>, grid_for(3 * (Ls.v_hi() - Ls.v_lo())), Ls, mgp<T>(d.x), mgp<T>(d.t), mgp<T>(d.b),
           mgp<T>(d.kx), mgp<T>(d.kv), d.kc, gate ? sl.st : nullptr, sl.partials, sl.counter, sl.st);
  }
  CK(allreduce(ctx, 0, 2, 0));
  for (Slab& sl : ctx->slabs) {
    k_kc_finish1<<<1, 1, 0, ctx->stream>>>(sl.st, sl.dlv[l].kc, gate ? sl.st : nullptr);
    ctx->launches++;
  }
  for (Slab& sl : ctx->slabs) {
    DLv& d = sl.dlv[l];
    const LvGeo Ls = dl_geo(ctx, sl, l);
    LAUNCH(ctx, k_kc_r2<T>, grid_for(3 * (Ls.v_hi() - Ls.v_lo())), Ls, mgp<T>(d.b), mgp<T>(d.kv), d.kc,
           gate ? sl.st : nullptr);
  }
  CK(dist_vcycle<T>(ctx, l, gate));   // x2 = B(r2)
  CK(exchange_lv(ctx, l, &DLv::x, es, 3));
  CK(dl_apply<T>(ctx, l, gate));      // t = A x2
  for (Slab& sl : ctx->slabs) {
    DLv& d = sl.dlv[l];
    const LvGeo Ls = dl_geo(ctx, sl, l);
    LAUNCH(ctx, k_kc_dot2<T>, grid_for(3 * (Ls.v_hi() - Ls.v_lo())), Ls, mgp<T>(d.x), mgp<T>(d.t), mgp<T>(d.b),
           mgp<T>(d.kv), d.kc, gate ? sl.st : nullptr, sl.partials, sl.counter, sl.st);
  }
  CK(allreduce(ctx, 0, 3, 0));
  for (Slab& sl : ctx->slabs) {
    k_kc_finish2<<<1, 1, 0, ctx->stream>>>(sl.st, sl.dlv[l].kc, gate ? sl.st : nullptr);
    ctx->launches++;
  }
  for (Slab& sl : ctx->slabs) {
    DLv& d = sl.dlv[l];
    const LvGeo Ls = dl_geo(ctx, sl, l);
    LAUNCH(ctx, k_kc_combine<T>, grid_for(3 * (Ls.v_hi() - Ls.v_lo())), Ls, mgp<T>(d.x), mgp<T>(d.kx), d.kc,
           gate ? sl.st : nullptr);
  }
  return check_launch(ctx);
}

int enqueue_vcycle(topo_ctx* ctx, int l, int gate, bool dot) {
  return ctx->mg_f32 ? enqueue_vcycle_t<float>(ctx, l, gate, dot) : enqueue_vcycle_t<double>(ctx, l, gate, dot);
}

// one MG-PCG iteration: z = V(r) (rho, beta) ; p = z + beta p ; q = K p ; alpha ; u, r update
int enqueue_mg_iter(topo_ctx* ctx, bool prof_here, int parity) {
  ctx->prof_capture = prof_here;
  const int rcv = enqueue_vcycle(ctx, 0, 1, true);
  ctx->prof_capture = false;
  CK(rcv);
  if (prof_here) CU(cudaEventRecordWithFlags(ctx->pe0, ctx->stream, cudaEventRecordExternal));
  const int fin = ctx->world == 1 ? 1 : 0;
  for (Slab& sl : ctx->slabs) {   // p = V(r) + beta p, V(r) in w (fp32 with w32_active)
    const CUtensorMap* pold = parity ? &sl.m_p1 : &sl.m_p0;
    double* pnew = parity ? sl.p0 : sl.p1;
    if (w32_active(ctx)) CK((launch_mv<2, true, 0, double, float>(ctx, sl, 1, sl.m_w32, pold, pnew, sl.q, fin)));
    else CK((launch_mv<2, true>(ctx, sl, 1, sl.m_w, pold, pnew, sl.q, fin)));
  }
  if (prof_here) CU(cudaEventRecordWithFlags(ctx->pe1, ctx->stream, cudaEventRecordExternal));
  if (!fin) {
    CK(allreduce(ctx, 0, 1, 0));
    for (Slab& sl : ctx->slabs) { k_finish_alpha<<<1, 1, 0, ctx->stream>>>(sl.st); ctx->launches++; }
  }
  for (Slab& sl : ctx->slabs) {
    double* pnew = parity ? sl.p0 : sl.p1;
    double* pprev = parity ? sl.p1 : sl.p0;
    const int gU = grid_for((long long)sl.g.nown * sl.g.nplane / 2);
    if (k32_active(ctx)) {   // fp32 Krylov r, q
      if (parity)
        LAUNCH(ctx, (k_update<true, true, float>), gU, sl.g, sl.st, sl.u, sl.r32, pprev, pnew, sl.q32, sl.invd, sl.fixm,
               sl.partials, sl.counter, fin);
      else
        LAUNCH(ctx, (k_update<false, true, float>), gU, sl.g, sl.st, sl.u, sl.r32, pprev, pnew, sl.q32, sl.invd,
               sl.fixm, sl.partials, sl.counter, fin);
    } else if (parity)
      LAUNCH(ctx, (k_update<true, true>), gU, sl.g, sl.st, sl.u, sl.r, pprev, pnew, sl.q, sl.invd, sl.fixm, sl.partials,
             sl.counter, fin);
    else
      LAUNCH(ctx, (k_update<false, true>), gU, sl.g, sl.st, sl.u, sl.r, pprev, pnew, sl.q, sl.invd, sl.fixm, sl.partials,
             sl.counter, fin);
  }
  if (!fin) {
    CK(allreduce(ctx, 0, 2, 0));
    for (Slab& sl : ctx->slabs) { k_finish_update<true><<<1, 1, 0, ctx->stream>>>(sl.st, parity ? 0 : 1); ctx->launches++; }
    CK(exchange_nodes(ctx, &Slab::r));
  }
  return check_launch(ctx);
}

// host <-> level-l vectors in external numbering (test hooks; T = level precision)
template <typename T>
int mg_upload(topo_ctx* ctx, int l, const double* host, void* dev) {
  const MgLevel& m = ctx->mg[l];
  const LvGeo& L = m.L;
  std::vector<T> lay(3 * L.ncomp, T(0));
  long long n = 0;
  for (int iz = 0; iz <= L.nz; ++iz)
    for (int ix = 0; ix <= L.nx; ++ix)
      for (int iy = 0; iy <= L.ny; ++iy, ++n)
        for (int c = 0; c < 3; ++c)
          lay[L.n(ix, iy, iz) + c * L.ncomp] = ((m.hfix[n] >> c) & 1) ? T(0) : (T)host[3 * n + c];
  // stream-ordered: the context's stream is non-blocking, and a legacy-stream copy
  // could land while a just-launched multigrid setup (its power steps use the
  // level vectors) is still running
  CU(cudaMemcpyAsync(dev, lay.data(), sizeof(T) * lay.size(), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return TOPO_OK;
}
template <typename T>
int mg_download(topo_ctx* ctx, int l, const void* dev, double* host) {
  const LvGeo& L = ctx->mg[l].L;
  std::vector<T> lay(3 * L.ncomp);
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaMemcpy(lay.data(), dev, sizeof(T) * lay.size(), cudaMemcpyDeviceToHost));
  long long n = 0;
  for (int iz = 0; iz <= L.nz; ++iz)
    for (int ix = 0; ix <= L.nx; ++ix)
      for (int iy = 0; iy <= L.ny; ++iy, ++n)
        for (int c = 0; c < 3; ++c) host[3 * n + c] = (double)lay[L.n(ix, iy, iz) + c * L.ncomp];
  return TOPO_OK;
}


// ---------------------------------------------------------------------------
// A4  PCG driver.  Batches of cg_batch iterations run as one CUDA graph; the
// device flag `done` turns the rest of a batch into no-ops, so the host
// polls once per batch.  After convergence of the recursive residual the
// true residual f - K u is checked; if it fails, r is replaced and PCG
// restarts.
// ---------------------------------------------------------------------------
// One PCG pass (Jacobi or multigrid preconditioner) from the current u.
int solve_pass(topo_ctx* ctx, int mg, int* replacements_out, double* rr_true_out) {
  const topo_params& P = ctx->prm;
  ctx->k32_pass = mg && ctx->k32_on;   // fp32 Krylov r, q (the graphs of each path are captured with it)
  const long long n_dof = 3LL * (P.nelx + 1) * (P.nely + 1) * (P.nelz + 1);
  const long long maxit = P.cg_max_iter > 0 ? P.cg_max_iter : 10 * n_dof;
  for (Slab& s : ctx->slabs) {
    k_cg_init<<<1, 1, 0, ctx->stream>>>(s.st, ctx->mode == TOPO_DIST_SOLO ? -1.0 : P.cg_rtol * P.cg_rtol, ctx->bb,
                                        maxit);
    ctx->launches++;
  }
  CK(residual(ctx, true));
  for (Slab& s : ctx->slabs) { k_cg_start<<<1, 1, 0, ctx->stream>>>(s.st); ctx->launches++; }
  CK(check_launch(ctx));
  if (!ctx->debug) CK(build_cg_graph(ctx, mg));
  int replacements = 0, rc = TOPO_OK;
  double rr_true = 0.0;
  DevState& h = *ctx->hstate;
  CK(sync_state(ctx));
  long long it_prev = h.it;
  while (true) {
    if (!h.done) {
      if (ctx->debug) {
        const int nb = mg ? ctx->mg_batch : ctx->cg_batch;
        for (int i = 0; i < nb; ++i) CK(mg ? enqueue_mg_iter(ctx, false, i & 1) : enqueue_cg_iter(ctx, false, i & 1));
      } else {
        CU(cudaGraphLaunch(ctx->cg_exec[mg], ctx->stream));
        ctx->launches += ctx->cg_batch_launches[mg];
      }
      CK(sync_state(ctx));
      if (ctx->profile && h.it > it_prev) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ctx->pe0, ctx->pe1) == cudaSuccess) {
          ctx->prof_ms += ms;
          ctx->prof_n++;
        }
        if (mg)
          for (int k = 0; k < 2; ++k)
            if (cudaEventElapsedTime(&ms, ctx->pe[2 * k], ctx->pe[2 * k + 1]) == cudaSuccess) {
              ctx->prof_ms_k[1 + k] += ms;
              ctx->prof_n_k[1 + k]++;
            }
      }
      it_prev = h.it;
      continue;
    }
    CK(flush_u(ctx));
    if (ctx->mode == TOPO_DIST_SOLO) break;   // timing run: exactly cg_max_iter iterations, no residual check
    if (h.status == 2) { rc = set_err(ctx, TOPO_ENOCONV, "PCG: no convergence in %lld iterations", h.it); break; }
    if (h.status == 3) { rc = set_err(ctx, TOPO_EBREAKDOWN, "PCG breakdown at iteration %lld", h.it); break; }
    CK(residual(ctx, false));
    CK(sync_state(ctx));
    rr_true = h.sums[1];
    if (rr_true <= h.tol2 * h.bb) break;
    if (replacements >= 20) { rc = set_err(ctx, TOPO_ENOCONV, "PCG: true residual stagnates"); break; }
    ++replacements;
    CK(residual(ctx, true));
    for (Slab& s : ctx->slabs) { k_cg_start<<<1, 1, 0, ctx->stream>>>(s.st); ctx->launches++; }
    CK(sync_state(ctx));
    if (h.done) {   // replaced residual already small (true residual above was not) -> done
      rr_true = h.rr;
      break;
    }
  }
  *replacements_out = replacements;
  *rr_true_out = rr_true;
  return rc;
}

int do_solve(topo_ctx* ctx, topo_solve_info* info) {
  CK(ensure_constants(ctx));
  if (!ctx->has_E) CK(update_modulus(ctx));
  CK(exchange_nodes(ctx, &Slab::invd, 1));   // ghost planes feed the fused p-update
  CU(cudaEventRecord(ctx->ev_setup[0], ctx->stream));
  CK(mg_setup(ctx));                         // multigrid: smoother weights, Galerkin levels, coarsest inverse
  CU(cudaEventRecord(ctx->ev_setup[1], ctx->stream));
  const topo_params& P = ctx->prm;
  CU(cudaEventRecord(ctx->ev[6], ctx->stream));
  if (!P.cg_warm_start || !ctx->has_u || ctx->bb == 0.0)
    for (Slab& s : ctx->slabs) CU(cudaMemsetAsync(s.u, 0, sizeof(double) * 3 * s.g.ncomp, ctx->stream));
  int mg = ctx->mg_on ? 1 : 0, replacements = 0;
  double rr_true = 0.0;
  long long iters = 0;
  int rc = solve_pass(ctx, mg, &replacements, &rr_true);
  iters = ctx->hstate->it;
  while (rc == TOPO_EBREAKDOWN && mg && ctx->mg_theta > 1.2 + 1e-12) {
    // an indefinite V-cycle: first suspect the smoother weights (a Rayleigh
    // estimate well below lam_max on a coarse level) -- lower theta by 0.2 for
    // the rest of the run and redo the solve
    ctx->tim.mg_theta_cuts++;
    ctx->mg_theta = std::max(1.2, ctx->mg_theta - 0.2);
    mg_invalidate(ctx);
    for (Slab& s : ctx->slabs) CU(cudaMemsetAsync(s.u, 0, sizeof(double) * 3 * s.g.ncomp, ctx->stream));
    CK(mg_setup(ctx));
    rc = solve_pass(ctx, 1, &replacements, &rr_true);
    iters += ctx->hstate->it;
  }
  if (rc == TOPO_EBREAKDOWN && mg && ctx->mg_f32) {
    // then the precision: promote the fp32 hierarchy to fp64 for the rest of the
    // run and redo the solve
    ctx->tim.mg_promotions++;
    ctx->mg_f32 = false;
    mg_invalidate(ctx);
    CK(mg_clear_levels(ctx));   // pads must read as 0.0 in the new element type
    for (Slab& s : ctx->slabs) CU(cudaMemsetAsync(s.u, 0, sizeof(double) * 3 * s.g.ncomp, ctx->stream));
    CK(mg_setup(ctx));
    rc = solve_pass(ctx, 1, &replacements, &rr_true);
    iters += ctx->hstate->it;
  }
  if (rc == TOPO_EBREAKDOWN && mg) {
    // multigrid breakdown (an indefinite V-cycle): redo this solve with the
    // Jacobi preconditioner from u = 0 (both GPU paths; counted in timings)
    ctx->tim.mg_fallbacks++;
    for (Slab& s : ctx->slabs) CU(cudaMemsetAsync(s.u, 0, sizeof(double) * 3 * s.g.ncomp, ctx->stream));
    mg = 0;
    rc = solve_pass(ctx, 0, &replacements, &rr_true);
    iters += ctx->hstate->it;
  }
  if (k32_active(ctx))   // keep the fp64 r (TOPO_FIELD_R) consistent with the fp32 recursion
    for (Slab& s : ctx->slabs) LAUNCH(ctx, k_f2d, grid_for(3 * s.g.ncomp), 3 * s.g.ncomp, s.r32, s.r);
  ctx->k32_pass = false;
  DevState& h = *ctx->hstate;
  CU(cudaEventRecord(ctx->ev[7], ctx->stream));
  CU(cudaEventSynchronize(ctx->ev[7]));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[6], ctx->ev[7]);
  {
    float ms_setup = 0.f;
    if (cudaEventElapsedTime(&ms_setup, ctx->ev_setup[0], ctx->ev_setup[1]) == cudaSuccess) ctx->tim.ms_mg_setup = ms_setup;
  }
  ctx->tim.cg_iters = iters;
  ctx->tim.cg_iters_total += iters;
  if (info) {
    info->iters = iters;
    info->rel_res = ctx->bb > 0 ? std::sqrt(h.rr / ctx->bb) : 0.0;
    info->true_rel_res = ctx->bb > 0 ? std::sqrt(rr_true / ctx->bb) : 0.0;
    info->ms = ms;
    info->replacements = replacements;
    info->precond = mg ? TOPO_PRECOND_MG : TOPO_PRECOND_JACOBI;
    info->mg_levels = ctx->mg_on ? (int)ctx->mg.size() : 0;
  }
  ctx->has_u = true;
  ctx->has_sens = ctx->has_dcf = false;
  return rc;
}

// A5: ce, dc, c = sum E ce, f^T u
int do_sensitivity(topo_ctx* ctx, double* c_out, double* fu_out) {
  if (!ctx->has_u) return set_err(ctx, TOPO_ESTATE, "topo_sensitivity before topo_solve");
  CK(ensure_constants(ctx));
  CK(exchange_nodes(ctx, &Slab::u));
  const Material m = material(ctx);
  for (Slab& s : ctx->slabs) {
    static const bool sens_x = !getenv("TOPO_SENS_X") || atoi(getenv("TOPO_SENS_X")) != 0;
    if (sens_x)
      LAUNCH(ctx, k_sens_x,
             grid_resident(k_sens_x, (long long)s.g.nely * s.g.nelz * ((s.g.nex + kSensCX - 1) / kSensCX)), s.g, s.st,
             m, s.u, s.E, s.xphys, s.passive, s.ce, s.dc, s.partials, s.counter);
    else
      LAUNCH(ctx, k_sens, grid_resident(k_sens, (long long)s.g.nex * s.g.eplane), s.g, s.st, m, s.u, s.E, s.xphys,
             s.passive, s.ce, s.dc, s.partials, s.counter);
    LAUNCH(ctx, k_dot, grid_for(3LL * s.g.nown * s.g.nplane), s.g, s.st, s.f, s.u, 1, s.partials, s.counter);
  }
  CK(check_launch(ctx));
  CK(allreduce(ctx, 0, 2, 0));
  CK(sync_state(ctx));
  if (c_out) *c_out = ctx->hstate->sums[0];
  if (fu_out) *fu_out = ctx->hstate->sums[1];
  ctx->tim.c = ctx->hstate->sums[0];
  ctx->tim.fu = ctx->hstate->sums[1];
  ctx->has_sens = true;
  return TOPO_OK;
}

// A6 on dc: dc~ (and dv~ once)
int do_filter_dc(topo_ctx* ctx) {
  CK(ensure_constants(ctx));
  const int mode = ctx->prm.filter_mode;
  CK(exchange_elems(ctx, &Slab::dc, ctx->R));
  for (Slab& s : ctx->slabs) {
    const int gp = grid_for(s.g.nelloc);
    if (mode == TOPO_FILTER_DENSITY) {
      LAUNCH(ctx, k_filt_prep<F_DIV>, gp, s.g, s.fp, s.dc, s.hs, s.vpad);
      CK(launch_filt_apply<F_DIV>(ctx, s, s.dc, s.dcf));
    } else if (mode == TOPO_FILTER_SENSITIVITY) {
      LAUNCH(ctx, k_filt_prep<F_XDC>, gp, s.g, s.fp, s.x, s.dc, s.vpad);
      CK(launch_filt_apply<F_XDC>(ctx, s, s.x, s.dcf));
    } else {
      LAUNCH(ctx, k_filt_prep<F_PLAIN>, gp, s.g, s.fp, s.dc, s.dc, s.vpad);
      CK(launch_filt_apply<F_PLAIN>(ctx, s, s.dc, s.dcf));
    }
    if (!ctx->has_dvf) {
      if (mode == TOPO_FILTER_DENSITY) {
        LAUNCH(ctx, k_filt_prep<F_DIV>, gp, s.g, s.fp, s.dv, s.hs, s.vpad);
        CK(launch_filt_apply<F_DIV>(ctx, s, s.dv, s.dvf));
      }
      else
        CU(cudaMemcpyAsync(s.dvf, s.dv, sizeof(double) * s.g.nelloc, cudaMemcpyDeviceToDevice, ctx->stream));
    }
  }
  CK(check_launch(ctx));
  ctx->has_dvf = true;
  ctx->has_dcf = true;
  return TOPO_OK;
}

// A6 on x: xPhys = filter(x) (mode 0) or x
int do_filter_x(topo_ctx* ctx) {
  CK(ensure_constants(ctx));
  const int nst = (int)ctx->st_off.size();
  if (ctx->prm.filter_mode == TOPO_FILTER_DENSITY) {
    for (Slab& s : ctx->slabs)
    {
      LAUNCH(ctx, k_filt_prep<F_X0>, grid_for(s.g.nelloc), s.g, s.fp, s.x, s.x, s.vpad);
      CK(launch_filt_apply<F_X0>(ctx, s, s.x, s.xphys));
    }
    CK(check_launch(ctx));
    CK(exchange_elems(ctx, &Slab::xphys, ctx->slabs[0].g.H));
  } else {
    for (Slab& s : ctx->slabs)
      CU(cudaMemcpyAsync(s.xphys, s.x, sizeof(double) * s.g.nelloc, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  ctx->has_E = false;
  return TOPO_OK;
}

constexpr int kOcFreezeBlocks = 148 * 4;   // blocks of the freeze / compaction kernels

// OC volume weights: mode 0 sums dv~_j xnew_j (R26); modes 1/2 sum xnew over design
// elements -- unweighted passes unless passive-solid elements exist (their xnew = 1
// must not count: then the dv = 1_D copy in dvf weights them out, R27)
bool oc_weighted(const topo_ctx* ctx) { return ctx->prm.filter_mode == TOPO_FILTER_DENSITY || ctx->has_solid; }

int enqueue_oc_batch(topo_ctx* ctx, int compact) {
  const int W = ctx->world, fin = (W == 1) ? 1 : 0;
  for (int i = 0; i < ctx->oc_batch; ++i) {
    for (Slab& s : ctx->slabs) {
      if (compact) {
        const bool s2 = compact == 2;
        LAUNCH(ctx, k_oc_pass_c, 148 * 4, s.st, ctx->prm.move, s2 ? s.oc_cx2 : s.oc_cx, s2 ? s.oc_cA2 : s.oc_cA,
               s2 ? s.oc_cdv2 : s.oc_cdv, s.partials, s.counter, fin);
        continue;
      }
      const int gr = grid_resident(k_oc_pass<1>, (long long)s.g.nex * s.g.eplane);
      if (oc_weighted(ctx))
        LAUNCH(ctx, k_oc_pass<1>, gr, s.g, s.st, ctx->prm.move, s.x, s.oca, s.dvf, s.partials, s.counter, fin);
      else
        LAUNCH(ctx, k_oc_pass<0>, gr, s.g, s.st, ctx->prm.move, s.x, s.oca, s.dvf, s.partials, s.counter, fin);
    }
    if (!fin) {
      CK(allreduce(ctx, 0, kOcCand, 0));
      for (Slab& s : ctx->slabs) { k_oc_finish<<<1, 1, 0, ctx->stream>>>(s.st); ctx->launches++; }
    }
  }
  return check_launch(ctx);
}

int build_oc_graph(topo_ctx* ctx, int compact) {
  cudaGraphExec_t& ex = compact == 2 ? ctx->oc_exec_c2 : compact == 1 ? ctx->oc_exec_c : ctx->oc_exec;
  if (ex) return TOPO_OK;
  cudaGraph_t graph;
  const long long l0 = ctx->launches;
  CU(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_oc_batch(ctx, compact);
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  if (rc != TOPO_OK) return rc;
  if (e != cudaSuccess) return set_err(ctx, TOPO_ECUDA, "OC graph capture: %s", cudaGetErrorString(e));
  e = cudaGraphInstantiate(&ex, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return set_err(ctx, TOPO_ECUDA, "OC graph instantiate: %s", cudaGetErrorString(e));
  ctx->oc_batch_launches = ctx->launches - l0;   // same count for both batch kinds
  ctx->launches = l0;
  return TOPO_OK;
}

// Freeze the elements whose xnew is a constant or linear in s for the rest of
// the bisection and compact the others (k_oc_freeze / k_oc_scan /
// k_oc_compact); per slab.  Stage 1 reads the element arrays, stage 2 the
// stage-1 active set (its count stays on the device).
int oc_compact(topo_ctx* ctx, int stage) {
  const bool dens = oc_weighted(ctx);
  for (Slab& s : ctx->slabs) {
    const long long b0 = (long long)s.g.H * s.g.eplane, n = (long long)s.g.nex * s.g.eplane;
    const int nb = (int)std::max(1LL, std::min<long long>(kOcFreezeBlocks, (n + kBlock - 1) / kBlock));
    const unsigned chunk = (unsigned)((n + nb - 1) / nb);
    const double *x, *A, *dv;
    const long long* nptr = nullptr;
    double *ox, *oA, *odv;
    if (stage == 1) {
      x = s.x + b0; A = s.oca + b0; dv = s.dvf + b0;
      ox = s.oc_cx; oA = s.oc_cA; odv = s.oc_cdv;
    } else {
      CU(cudaMemcpyAsync(s.oc_n1, &s.st->oc_nact, sizeof(long long), cudaMemcpyDeviceToDevice, ctx->stream));
      x = s.oc_cx; A = s.oc_cA; dv = s.oc_cdv; nptr = s.oc_n1;
      ox = s.oc_cx2; oA = s.oc_cA2; odv = s.oc_cdv2;
    }
    const bool m0 = stage == 1 ? dens : true;   // stage 2: dv~ (or 1) is stored in the active set
    if (m0) LAUNCH(ctx, k_oc_freeze<1>, nb, n, nptr, x, A, dv, s.st, ctx->prm.move, chunk, s.oc_counts, s.partials,
                   s.counter);
    else LAUNCH(ctx, k_oc_freeze<0>, nb, n, nptr, x, A, dv, s.st, ctx->prm.move, chunk, s.oc_counts, s.partials,
                s.counter);
    k_oc_scan<<<1, 32, 0, ctx->stream>>>(s.oc_counts, nb, s.oc_offs, s.st);
    ctx->launches++;
    if (m0) LAUNCH(ctx, k_oc_compact<1>, nb, n, nptr, x, A, dv, s.st, ctx->prm.move, chunk, s.oc_offs, ox, oA, odv);
    else LAUNCH(ctx, k_oc_compact<0>, nb, n, nptr, x, A, dv, s.st, ctx->prm.move, chunk, s.oc_offs, ox, oA, odv);
  }
  return check_launch(ctx);
}

// A7: bisection, final xnew, x <- xnew, xPhys <- filter(x)
int do_oc(topo_ctx* ctx, double* lambda, double* change, double* volume) {
  if (!ctx->has_dcf) return set_err(ctx, TOPO_ESTATE, "topo_oc_step before topo_filter(DC)");
  CK(ensure_constants(ctx));
  const topo_params& P = ctx->prm;
  if (ctx->has_solid && P.filter_mode == TOPO_FILTER_DENSITY) {
    // with every design element at 0 the volume is the passive-solid
    // spill sum_{j solid} dv~_j; above the target no lambda can meet it
    for (Slab& s : ctx->slabs)
      LAUNCH(ctx, k_design_sum, grid_for((long long)s.g.nex * s.g.eplane), s.g, s.st, s.dvf, s.passive, 4,
             s.partials, s.counter, (int)kSolid);
    CK(check_launch(ctx));
    CK(allreduce(ctx, 4, 1, 0));
    CK(sync_state(ctx));
    const double v0 = ctx->hstate->sums[4], target = P.volfrac * (double)ctx->n_design;
    if (v0 > target)
      return set_err(ctx, TOPO_EBISECT, "OC: the passive-solid volume %.6g alone exceeds the target %.6g", v0, target);
  }
  for (Slab& s : ctx->slabs) {
    k_oc_init<<<1, 1, 0, ctx->stream>>>(s.st, P.oc_lmax, P.volfrac * (double)ctx->n_design, P.oc_tol);
    ctx->launches++;
    LAUNCH(ctx, k_oc_prep, grid_resident(k_oc_prep, (long long)s.g.nex * s.g.eplane), s.g, s.x, s.dcf, s.dvf, s.passive, s.oca);
  }
  CK(check_launch(ctx));
  if (!ctx->debug)
    for (int c = 0; c < 3; ++c) CK(build_oc_graph(ctx, c));
  // phase 1 (l1 = 0) in two grid passes (k_oc_gpass): the same decisions as the
  // sequential loop, which halves l2 from oc_lmax until V(lmid) > target
  {
    const int W = ctx->world, fin = (W == 1) ? 1 : 0;
    const bool dens = oc_weighted(ctx);
    for (int stage = 0; stage < 2; ++stage) {
      for (Slab& s : ctx->slabs) {
        const int gr = grid_resident(k_oc_gpass<1>, (long long)s.g.nex * s.g.eplane);
        if (dens) LAUNCH(ctx, k_oc_gpass<1>, gr, s.g, s.st, stage, P.move, s.x, s.oca, s.dvf, s.partials, s.counter, fin);
        else LAUNCH(ctx, k_oc_gpass<0>, gr, s.g, s.st, stage, P.move, s.x, s.oca, s.dvf, s.partials, s.counter, fin);
      }
      if (!fin) {
        CK(allreduce(ctx, 0, kOcCand, 0));
        for (Slab& s : ctx->slabs) { k_oc_gfinish<<<1, 1, 0, ctx->stream>>>(s.st, stage); ctx->launches++; }
      }
    }
    CK(check_launch(ctx));
  }
  DevState& h = *ctx->hstate;
  CK(sync_state(ctx));
  int guard = 0;
  int compact = 0;
  while (h.oc_active) {
    // once the bracket is narrow (l1 > 0, l2 <= 2 l1, then l2 <= 1.002 l1),
    // most elements are at a clamp bound or unclamped for every remaining
    // lambda: fold them into F + s G and compact the rest (slab 0's bracket is
    // every slab's bracket)
    const int want = (h.l1 > 0.0 && h.l2 <= 1.002 * h.l1) ? 2 : (h.l1 > 0.0 && h.l2 <= 2.0 * h.l1) ? 1 : 0;
    while (compact < want) {
      CK(oc_compact(ctx, ++compact));
      if (getenv("TOPO_OC_VERBOSE")) {   // diagnostics
        CK(sync_state(ctx));
        fprintf(stderr, "[topo] OC compaction %d after %d bisection steps: %lld active elements\n", compact,
                h.oc_pass, (long long)h.oc_nact);
      }
    }
    if (ctx->debug) {
      CK(enqueue_oc_batch(ctx, compact));
    } else {
      CU(cudaGraphLaunch(compact == 2 ? ctx->oc_exec_c2 : compact == 1 ? ctx->oc_exec_c : ctx->oc_exec, ctx->stream));
      ctx->launches += ctx->oc_batch_launches;
    }
    CK(sync_state(ctx));
    if (++guard > 4096 / ctx->oc_batch) return set_err(ctx, TOPO_EBISECT, "OC bisection did not terminate");
  }
  if (getenv("TOPO_OC_VERBOSE")) fprintf(stderr, "[topo] OC done after %d passes (%d batches)\n", h.oc_pass, guard);
  for (Slab& s : ctx->slabs)
    LAUNCH(ctx, k_oc_final, grid_resident(k_oc_final, (long long)s.g.nex * s.g.eplane), s.g, s.st, P.move, s.x, s.oca, s.passive, s.xnew,
           s.partials, s.counter);
  CK(check_launch(ctx));
  CK(allreduce(ctx, 2, 2, 0x2));
  for (Slab& s : ctx->slabs)
    CU(cudaMemcpyAsync(s.x, s.xnew, sizeof(double) * s.g.nelloc, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(exchange_elems(ctx, &Slab::x, ctx->slabs[0].g.H));
  CK(do_filter_x(ctx));
  double vol;
  if (P.filter_mode == TOPO_FILTER_DENSITY) {
    for (Slab& s : ctx->slabs)
      LAUNCH(ctx, k_design_sum, grid_for((long long)s.g.nex * s.g.eplane), s.g, s.st, s.xphys, s.passive, 4,
             s.partials, s.counter);
    CK(check_launch(ctx));
    CK(allreduce(ctx, 4, 1, 0));
    CK(sync_state(ctx));
    vol = h.sums[4];
  } else {
    CK(sync_state(ctx));
    vol = h.sums[2];
  }
  const double lam = h.lmid, chg = h.sums[3];
  if (lambda) *lambda = lam;
  if (change) *change = chg;
  if (volume) *volume = vol / (double)ctx->n_design;
  ctx->tim.lambda = lam;
  ctx->tim.change = chg;
  ctx->tim.volume = vol / (double)ctx->n_design;
  ctx->tim.oc_passes = h.oc_pass;
  ctx->has_sens = ctx->has_dcf = false;
  return TOPO_OK;
}

// A8: the SIMP loop (§2.5) -- n_iter x (modulus, solve, sensitivity, filter, OC)
int optimize_loop(topo_ctx* ctx, int n_iter, double change_tol, double* c_hist, int32_t* n_done) {
  if (n_done) *n_done = 0;
  int rc = TOPO_OK;
  for (int it = 0; it < n_iter; ++it) {
    cudaEvent_t* ev = ctx->ev;
    CU(cudaEventRecord(ev[0], ctx->stream));
    CK(update_modulus(ctx));
    CU(cudaEventRecord(ev[1], ctx->stream));
    rc = do_solve(ctx, nullptr);
    if (rc != TOPO_OK) break;
    CU(cudaEventRecord(ev[2], ctx->stream));
    double c = 0.0, fu = 0.0;
    rc = do_sensitivity(ctx, &c, &fu);
    if (rc != TOPO_OK) break;
    CU(cudaEventRecord(ev[3], ctx->stream));
    rc = do_filter_dc(ctx);
    if (rc != TOPO_OK) break;
    CU(cudaEventRecord(ev[4], ctx->stream));
    double lam, chg, vol;
    rc = do_oc(ctx, &lam, &chg, &vol);
    if (rc != TOPO_OK) break;
    CU(cudaEventRecord(ev[5], ctx->stream));
    CU(cudaEventSynchronize(ev[5]));
    float t[5];
    for (int k = 0; k < 5; ++k) cudaEventElapsedTime(&t[k], ev[k], ev[k + 1]);
    ctx->tim.ms_efield = t[0];
    ctx->tim.ms_solve = t[1];
    ctx->tim.ms_sens = t[2];
    ctx->tim.ms_filter = t[3];   // dc filter; the x filter is inside ms_oc
    ctx->tim.ms_oc = t[4];
    ctx->tim.ms_total = t[0] + t[1] + t[2] + t[3] + t[4];
    if (c_hist) c_hist[it] = c;
    if (n_done) *n_done = it + 1;
    if (change_tol > 0 && chg < change_tol) break;
  }
  return rc;
}

// TOPO_DIST_HOST: mailbox = the largest message any step sends (all ranks agree:
// global sizes only), pinned staging of the same size
int open_host_transport(topo_ctx* ctx, const topo_dist* dist) {
  const Slab& a = ctx->slabs[0];
  long long mb = 32 * 8;                                             // scalar allreduces
  mb = std::max<long long>(mb, 8LL * 6 * a.g.nplane);                // node halo, 3 components
  mb = std::max<long long>(mb, 8LL * 2 * a.g.H * a.g.eplane);        // element halo
  for (int r = 0; r < ctx->world; ++r) {                             // moduli all-gather / planes
    int b = 0, e = 0;
    topo_partition(ctx->prm.nelx, ctx->prm.rmin, ctx->world, r, &b, &e);
    mb = std::max<long long>(mb, 8LL * (e - b) * a.g.eplane);
  }
  mb = std::max<long long>(mb, 8LL * ctx->prm.nelx * a.g.eplane);   // the gathered whole-grid moduli (recv side)
  if (ctx->mg_on && ctx->mg.size() > 1) mb = std::max<long long>(mb, 8LL * 3 * ctx->mg[1].L.ncomp);   // level-1 allreduce
  char name[129];
  memcpy(name, dist->nccl_id, 128);
  name[128] = 0;
  ctx->ht = new HostTransport();
  ctx->ht->timeout_s = ctx->comm_timeout_s;
  std::string err;
  if (!ctx->ht->open(name, ctx->rank, ctx->world, mb, err)) return set_err(ctx, TOPO_ENCCL, "%s", err.c_str());
  CU(cudaMallocHost(&ctx->ht->hsend, (size_t)ctx->ht->mbox));
  CU(cudaMallocHost(&ctx->ht->hrecv, (size_t)ctx->ht->mbox));
  return TOPO_OK;
}

int alloc_slab(topo_ctx* ctx, Slab& s) {
  const Geo& g = s.g;
  auto al = [&](void** p, size_t bytes) -> int {
    CU(cudaMalloc(p, bytes));
    CU(cudaMemsetAsync(*p, 0, bytes, ctx->stream));
    // the context's stream is non-blocking: finish the zero fill before any
    // synchronous host upload into this buffer (legacy-stream cudaMemcpy)
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->dev_bytes += bytes;
    return TOPO_OK;
  };
  const size_t nb = sizeof(double) * 3 * g.ncomp, eb = sizeof(double) * g.nelloc;
  double** nv[] = {&s.u, &s.r, &s.p0, &s.p1, &s.q, &s.f, &s.w, &s.z};
  for (double** v : nv) CK(al((void**)v, nb));
  CK(al((void**)&s.invd, sizeof(double) * g.ncomp));
  CK(al((void**)&s.fixm, g.ncomp));
  double** ev[] = {&s.E, &s.x, &s.xphys, &s.dc, &s.dcf, &s.dvf, &s.dv, &s.hs, &s.ihs, &s.ce, &s.xnew, &s.oca};
  for (double** v : ev) CK(al((void**)v, eb));
  CK(al((void**)&s.passive, g.nelloc));
  s.fp.R = ctx->R;
  s.fp.FY = (g.nely + 2 * ctx->R + 1) / 2 * 2;   // even: 16-byte TMA row pitch (k_filt25)
  s.fp.FZ = g.nelz + 2 * ctx->R;
  s.fp.fplane = (long long)s.fp.FY * s.fp.FZ;
  CK(al((void**)&s.vpad, sizeof(double) * g.NEXL * s.fp.fplane));
  const MvGrid mg = mv_grid(ctx, g);
  const size_t nbmax = std::max<size_t>(kMaxGridBlocks, (size_t)mg.grid.x * mg.grid.y * mg.grid.z);
  CK(al((void**)&s.partials, sizeof(double) * 8 * nbmax));
  CK(al((void**)&s.counter, sizeof(unsigned int) * 4));
  CK(al((void**)&s.st, sizeof(DevState)));
  CK(al((void**)&s.oc_counts, sizeof(unsigned) * kOcFreezeBlocks));
  CK(al((void**)&s.oc_offs, sizeof(unsigned) * kOcFreezeBlocks));
  {   // compacted OC arrays: worst case every owned element active
    const size_t ne = sizeof(double) * (size_t)g.nex * g.eplane;
    CK(al((void**)&s.oc_cx, ne));
    CK(al((void**)&s.oc_cA, ne));
    CK(al((void**)&s.oc_cdv, ne));
    CK(al((void**)&s.oc_cx2, ne));
    CK(al((void**)&s.oc_cA2, ne));
    CK(al((void**)&s.oc_cdv2, ne));
    CK(al((void**)&s.oc_n1, sizeof(long long)));
  }
  s.stage_n = std::max((size_t)3 * (g.nown) * (g.nely + 1) * (g.nelz + 1), (size_t)g.nex * g.nely * g.nelz);
  CK(al((void**)&s.stage, sizeof(double) * s.stage_n));
  return TOPO_OK;
}

void free_ctx(topo_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (Slab& s : ctx->slabs) {
    void* ptrs[] = {s.u, s.r, s.p0, s.p1, s.q, s.f, s.invd, s.w, s.z, s.fixm, s.E, s.x, s.xphys, s.dc, s.dcf, s.oca,
                    s.vpad, s.res32, s.z32, s.w32, s.r32, s.q32, s.pw0, s.pw0_b, s.oc_counts, s.oc_offs, s.oc_cx, s.oc_cA, s.oc_cdv,
                    s.oc_cx2, s.oc_cA2, s.oc_cdv2, s.oc_n1,
                    s.dvf, s.dv, s.hs, s.ihs, s.ce, s.xnew, s.passive, s.partials, s.counter, s.st, s.stage,
                    s.u_b, s.x_b, s.xphys_b};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
  for (Slab& s : ctx->slabs)
    for (DLv& d : s.dlv)
      if (d.own) {
        void* ptrs[] = {d.x, d.b, d.t, d.kx, d.kv, d.Y, d.kc};
        for (void* p : ptrs)
          if (p) cudaFree(p);
      }
  for (MgLevel& m : ctx->mg) {
    void* ptrs[] = {m.x, m.b, m.t, m.invd, m.K, m.S, m.Y, m.pw, m.pw_b, m.fixm, m.kx, m.kv};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
  {
    void* ptrs[] = {ctx->mg_tab8, ctx->mg_tab64, ctx->mg_Eg, ctx->mg_A0, ctx->mg_C, ctx->mg_R, ctx->mg_P, ctx->mg_ws,
                    ctx->mg_dmap, ctx->mg_imap, ctx->mg_om, ctx->mg_kc, ctx->mg_A32};
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
  if (ctx->mg_setup_exec) cudaGraphExecDestroy(ctx->mg_setup_exec);
  if (ctx->mg_setup_exec_w) cudaGraphExecDestroy(ctx->mg_setup_exec_w);
  if (ctx->mg_gE) cudaFree(ctx->mg_gE);
  if (ctx->mg_E32) cudaFree(ctx->mg_E32);
  for (cudaGraphExec_t g : ctx->cg_exec)
    if (g) cudaGraphExecDestroy(g);
  if (ctx->oc_exec) cudaGraphExecDestroy(ctx->oc_exec);
  if (ctx->oc_exec_c) cudaGraphExecDestroy(ctx->oc_exec_c);
  if (ctx->oc_exec_c2) cudaGraphExecDestroy(ctx->oc_exec_c2);
  if (ctx->pe0) cudaEventDestroy(ctx->pe0);
  if (ctx->pe1) cudaEventDestroy(ctx->pe1);
  for (cudaEvent_t e : ctx->pe)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->ev_setup)
    if (e) cudaEventDestroy(e);
  if (ctx->hstate) cudaFreeHost(ctx->hstate);
  if (ctx->comm) g_nccl.CommDestroy(ctx->comm);
  if (ctx->ht) {
    if (ctx->ht->hsend) cudaFreeHost(ctx->ht->hsend);
    if (ctx->ht->hrecv) cudaFreeHost(ctx->ht->hrecv);
    ctx->ht->close_all();
    delete ctx->ht;
  }
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (g_const_owner == ctx) g_const_owner = nullptr;
  delete ctx;
}

int validate(topo_ctx* ctx, const topo_params* p) {
  if (!p) return set_err(ctx, TOPO_EINVAL, "params is NULL");
  if (p->nelx < 1 || p->nely < 1 || p->nelz < 1)
    return set_err(ctx, TOPO_EINVAL, "grid dimensions must be >= 1 (got %d x %d x %d)", p->nelx, p->nely, p->nelz);
  if ((double)(p->nelx + 4) * (p->nely + 7) * (p->nelz + 3) * 3 > 2.0e9)
    return set_err(ctx, TOPO_EINVAL, "grid too large for one context (32-bit in-slab offsets)");
  if (!(p->volfrac > 0 && p->volfrac < 1)) return set_err(ctx, TOPO_EINVAL, "volfrac must be in (0,1)");
  if (!(p->penal >= 1)) return set_err(ctx, TOPO_EINVAL, "penal must be >= 1");
  if (!(p->rmin > 0 && p->rmin <= 6)) return set_err(ctx, TOPO_EINVAL, "rmin must be in (0, 6]");
  if (!(p->Emin > 0 && p->Emin < p->E0)) return set_err(ctx, TOPO_EINVAL, "need 0 < Emin < E0");
  if (!(p->nu >= 0 && p->nu < 0.5)) return set_err(ctx, TOPO_EINVAL, "nu must be in [0, 0.5)");
  if (!(p->move > 0 && p->move <= 1)) return set_err(ctx, TOPO_EINVAL, "move must be in (0, 1]");
  if (p->filter_mode < 0 || p->filter_mode > 2) return set_err(ctx, TOPO_EINVAL, "filter_mode must be 0, 1 or 2");
  if (!(p->cg_rtol > 0 && p->cg_rtol < 1)) return set_err(ctx, TOPO_EINVAL, "cg_rtol must be in (0,1)");
  if (!(p->oc_tol > 0) || !(p->oc_lmax > 0)) return set_err(ctx, TOPO_EINVAL, "oc_tol, oc_lmax must be > 0");
  if (p->precond < 0 || p->precond > 2) return set_err(ctx, TOPO_EINVAL, "precond must be 0, 1 or 2");
  if (p->mg_nu < 1 || p->mg_nu > 8) return set_err(ctx, TOPO_EINVAL, "mg_nu must be in [1, 8]");
  if (!(p->mg_omega > 0 && p->mg_omega < 2)) return set_err(ctx, TOPO_EINVAL, "mg_omega must be in (0, 2)");
  if (p->mg_fp32 != 0 && p->mg_fp32 != 1) return set_err(ctx, TOPO_EINVAL, "mg_fp32 must be 0 or 1");
  if (p->mg_nu_deep < 0 || p->mg_nu_deep > 64) return set_err(ctx, TOPO_EINVAL, "mg_nu_deep must be in [0, 64]");
  if (p->mg_cycle != TOPO_MG_VCYCLE && p->mg_cycle != TOPO_MG_KCYCLE) return set_err(ctx, TOPO_EINVAL, "mg_cycle must be 0 or 1");
  if (p->krylov_fp32 != 0 && p->krylov_fp32 != 1) return set_err(ctx, TOPO_EINVAL, "krylov_fp32 must be 0 or 1");
  if (p->mg_coarse_max != 0 && (p->mg_coarse_max < 24 || p->mg_coarse_max > 8192))
    return set_err(ctx, TOPO_EINVAL, "mg_coarse_max must be 0 (auto) or in [24, 8192]");
  return TOPO_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

void topo_params_default(topo_params* p) {
  if (!p) return;
  memset(p, 0, sizeof *p);
  p->nelx = p->nely = p->nelz = 1;
  p->volfrac = 0.3;
  p->penal = 3.0;
  p->rmin = 1.5;
  p->E0 = 1.0;
  p->Emin = 1e-9;
  p->nu = 0.3;
  p->move = 0.2;
  p->filter_mode = TOPO_FILTER_DENSITY;
  p->cg_rtol = 1e-8;
  p->cg_max_iter = 0;
  p->cg_warm_start = 1;
  p->oc_tol = 1e-10;
  p->oc_lmax = 1e9;
  p->deterministic = 1;
  p->cg_check_every = 0;
  p->precond = TOPO_PRECOND_AUTO;
  p->mg_nu = 1;
  p->mg_omega = 1.6;
  p->mg_coarse_max = 0;
  p->mg_fp32 = 1;
  p->mg_nu_deep = 0;
  p->mg_cycle = TOPO_MG_KCYCLE;
  p->krylov_fp32 = 0;
}

const char* topo_version(void) { return "topo-b200 0.1 (sm_100a, fp64 matrix-free EbE PCG)"; }

const char* topo_strerror(int code) {
  switch (code) {
    case TOPO_OK: return "ok";
    case TOPO_EINVAL: return "invalid argument";
    case TOPO_ENOCONV: return "PCG did not converge";
    case TOPO_EBREAKDOWN: return "PCG breakdown";
    case TOPO_EUNCONSTRAINED: return "no fixed DOFs (rigid-body modes)";
    case TOPO_EBISECT: return "OC bisection failure";
    case TOPO_EALLPASSIVE: return "no design elements";
    case TOPO_ECUDA: return "CUDA error";
    case TOPO_ENCCL: return "NCCL error";
    case TOPO_ENOMEM: return "out of memory";
    case TOPO_ESTATE: return "call out of order";
    default: return "unknown error";
  }
}

const char* topo_last_error(const topo_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

int topo_element_stiffness(double nu, double* ke576) {
  if (!ke576 || !(nu >= 0 && nu < 0.5)) return TOPO_EINVAL;
  build_element_stiffness(nu, ke576);
  return TOPO_OK;
}

int topo_nccl_unique_id(uint8_t* out128) {
  std::string err;
  if (!out128 || !g_nccl.load(err)) return TOPO_ENCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != 0) return TOPO_ENCCL;
  memcpy(out128, id.internal, 128);
  return TOPO_OK;
}

int topo_host_transport_id(uint8_t* out128) {
  if (!out128) return TOPO_EINVAL;
  memset(out128, 0, 128);
  const unsigned long long t = (unsigned long long)std::chrono::steady_clock::now().time_since_epoch().count();
  snprintf(reinterpret_cast<char*>(out128), 128, "/topo_%d_%llx", (int)getpid(), t);
  return TOPO_OK;
}

int topo_init(const topo_params* p, const double* load, const uint8_t* fixed, const uint8_t* passive,
              const topo_dist* dist, topo_ctx** out) {
  if (!out) return TOPO_EINVAL;
  *out = nullptr;
  topo_ctx* ctx = new topo_ctx();
  int rc = validate(ctx, p);
  if (rc == TOPO_OK && (!load || !fixed)) rc = set_err(ctx, TOPO_EINVAL, "load and fixed are required");
  if (rc != TOPO_OK) { delete ctx; return rc; }
  ctx->prm = *p;
  const int nelx = p->nelx, nely = p->nely, nelz = p->nelz;
  const long long nn = (long long)(nelx + 1) * (nely + 1) * (nelz + 1), ne = (long long)nelx * nely * nelz;
  // --- problem checks on the host (global inputs) ---
  long long nfix = 0;
  for (long long i = 0; i < 3 * nn; ++i) {
    if (fixed[i]) {
      ++nfix;
      if (load[i] != 0.0) {
        rc = set_err(ctx, TOPO_EINVAL, "load on fixed DOF %lld", i);
        break;
      }
    }
    if (!std::isfinite(load[i])) { rc = set_err(ctx, TOPO_EINVAL, "non-finite load"); break; }
  }
  if (rc == TOPO_OK && nfix == 0) rc = set_err(ctx, TOPO_EUNCONSTRAINED, "no fixed DOFs");
  long long nd = ne;
  if (passive) {
    nd = 0;
    for (long long e = 0; e < ne; ++e) {
      if (passive[e] > kSolid) {
        if (rc == TOPO_OK) rc = set_err(ctx, TOPO_EINVAL, "passive[%lld] = %d (0 design, 1 void, 2 solid)", e, (int)passive[e]);
        break;
      }
      nd += passive[e] ? 0 : 1;
      if (passive[e] == kSolid) ctx->has_solid = true;
    }
  }
  if (rc == TOPO_OK && nd == 0) rc = set_err(ctx, TOPO_EALLPASSIVE, "every element is passive");
  ctx->n_design = nd;
  // --- distribution ---
  if (dist) {
    ctx->mode = dist->mode;
    ctx->rank = dist->rank;
    ctx->world = dist->world;
    ctx->device = dist->device;
  } else {
    cudaGetDevice(&ctx->device);
  }
  if (rc == TOPO_OK && (ctx->world < 1 || ctx->world > 16 || ctx->rank < 0 || ctx->rank >= ctx->world))
    rc = set_err(ctx, TOPO_EINVAL, "bad rank/world");
  if (const char* e = getenv("TOPO_COMM_TIMEOUT")) ctx->comm_timeout_s = atof(e);
  if (rc == TOPO_OK && ctx->mode == TOPO_DIST_HOST && (!dist || !dist->nccl_id))
    rc = set_err(ctx, TOPO_EINVAL, "TOPO_DIST_HOST needs the transport id (topo_host_transport_id) in nccl_id");
  if (rc == TOPO_OK && (ctx->mode < TOPO_DIST_SINGLE || ctx->mode > TOPO_DIST_SOLO))
    rc = set_err(ctx, TOPO_EINVAL, "bad dist mode %d", ctx->mode);
  if (rc == TOPO_OK && ctx->mode == TOPO_DIST_SINGLE && ctx->world != 1)
    rc = set_err(ctx, TOPO_EINVAL, "TOPO_DIST_SINGLE needs world == 1");
  // --- KE and filter stencil (host precompute) ---
  build_element_stiffness(p->nu, ctx->ke);
  ctx->kd = ctx->ke[0];
  {
    double w[8];
    if (!wht_constants(ctx->ke, w, 1e-13) && rc == TOPO_OK)
      rc = set_err(ctx, TOPO_EINVAL, "KE lacks the Walsh-Hadamard block structure");
    ctx->wht = WhtK{w[0], w[1], w[2], w[3], w[4], w[5], w[6], w[7]};
  }
  {
    const int B = (int)std::ceil(p->rmin);
    int R = 0;
    for (int dz = -B; dz <= B; ++dz)
      for (int dx = -B; dx <= B; ++dx)
        for (int dy = -B; dy <= B; ++dy) {
          const double d = std::sqrt((double)(dx * dx + dy * dy + dz * dz));
          if (!(d < p->rmin)) continue;
          ctx->st_off.push_back(make_int4(dx, dy, dz, 0));
          ctx->st_w.push_back(p->rmin - d);
          R = std::max(R, std::max(std::abs(dx), std::max(std::abs(dy), std::abs(dz))));
        }
    ctx->R = R;
    if ((int)ctx->st_off.size() > kMaxStencil) rc = set_err(ctx, TOPO_EINVAL, "filter stencil too large");
  }
  const int H = std::max(1, ctx->R);
  if (const char* e = getenv("TOPO_TZ")) ctx->tz = atoi(e) == 16 ? 16 : 8;   // matvec CTA shape (tuning)
  if (const char* e = getenv("TOPO_DEBUG_SYNC")) ctx->debug = atoi(e) != 0;
  // slab partition: owned elements [ex0, ex1)
  const int W = ctx->world;
  for (int s = 0; s < W && rc == TOPO_OK; ++s) {
    const int ex0 = (int)((long long)s * nelx / W), ex1 = (int)((long long)(s + 1) * nelx / W);
    if (ex1 - ex0 < std::max(1, W > 1 ? ctx->R : 1))
      rc = set_err(ctx, TOPO_EINVAL, "slab %d has %d element planes; need >= filter radius %d", s, ex1 - ex0, ctx->R);
  }
  if (rc != TOPO_OK) { delete ctx; return rc; }
  if (cudaSetDevice(ctx->device) != cudaSuccess) { delete ctx; return TOPO_ECUDA; }
  if (cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking) != cudaSuccess) { delete ctx; return TOPO_ECUDA; }
  ctx->stream = ctx->own_stream;
  if (cudaMallocHost(&ctx->hstate, sizeof(DevState)) != cudaSuccess) { free_ctx(ctx); return TOPO_ENOMEM; }
  memset(ctx->hstate, 0, sizeof(DevState));
  cudaEventCreate(&ctx->pe0);
  cudaEventCreate(&ctx->pe1);
  for (cudaEvent_t& e : ctx->pe) cudaEventCreate(&e);
  for (cudaEvent_t& e : ctx->ev) cudaEventCreate(&e);
  for (cudaEvent_t& e : ctx->ev_setup) cudaEventCreate(&e);
  if (ctx->mode == TOPO_DIST_NCCL && W > 1) {
    std::string err;
    if (!g_nccl.load(err)) { rc = set_err(ctx, TOPO_ENCCL, "%s", err.c_str()); free_ctx(ctx); return rc; }
    if (!dist->nccl_id) { free_ctx(ctx); return TOPO_EINVAL; }
    ncclUniqueId id;
    memcpy(id.internal, dist->nccl_id, 128);
    ncclResult_t r = g_nccl.CommInitRank(&ctx->comm, W, id, ctx->rank);
    if (r != 0) { rc = set_err(ctx, TOPO_ENCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r)); free_ctx(ctx); return rc; }
  }
  // local slabs
  const bool own_only = ctx->mode == TOPO_DIST_NCCL || ctx->mode == TOPO_DIST_HOST ||
                        ctx->mode == TOPO_DIST_SOLO;   // one slab per process
  const int s_begin = own_only ? ctx->rank : 0;
  const int s_end = own_only ? ctx->rank + 1 : W;
  for (int s = s_begin; s < s_end; ++s) {
    Slab sl;
    Geo& g = sl.g;
    g.nelx = nelx; g.nely = nely; g.nelz = nelz;
    g.ex0 = (int)((long long)s * nelx / W);
    g.ex1 = (int)((long long)(s + 1) * nelx / W);
    g.nex = g.ex1 - g.ex0;
    g.nown = g.nex + (s == W - 1 ? 1 : 0);
    g.NY = ((nely + 3) + 3) / 4 * 4;
    g.NZ = nelz + 3;
    g.NXL = g.nown + 2;
    g.nplane = (long long)g.NY * g.NZ;
    g.ncomp = (long long)g.NXL * g.nplane;
    g.H = H;
    g.EY = ((nely + 2) + 3) / 4 * 4;
    g.EZ = nelz + 2;
    g.NEXL = g.nex + 2 * H;
    g.eplane = (long long)g.EY * g.EZ;
    g.nelloc = (long long)g.NEXL * g.eplane;
    ctx->slabs.push_back(sl);
  }
  for (Slab& s : ctx->slabs) {
    rc = alloc_slab(ctx, s);
    if (rc == TOPO_OK) rc = build_maps(ctx, s);
    if (rc != TOPO_OK) { int r2 = rc; free_ctx(ctx); return r2 == TOPO_ECUDA ? TOPO_ENOMEM : r2; }
  }
  // --- inputs ---
  std::vector<uint8_t> loc8;
  std::vector<double> locd;
  for (Slab& s : ctx->slabs) {
    const Geo& g = s.g;
    // fixed-DOF bit mask on the owned node planes and the ghost planes (the
    // multigrid prolongation writes z on the ghost planes too)
    loc8.assign(g.ncomp, 0);
    for (int ix = std::max(0, g.ex0 - 1); ix <= std::min(nelx, g.ex0 + g.nown); ++ix)
      for (int iz = 0; iz <= nelz; ++iz)
        for (int iy = 0; iy <= nely; ++iy) {
          const long long n = (long long)iz * (nelx + 1) * (nely + 1) + (long long)ix * (nely + 1) + iy;
          loc8[node_idx(g, ix, iy, iz)] = (fixed[3 * n] ? 1 : 0) | (fixed[3 * n + 1] ? 2 : 0) | (fixed[3 * n + 2] ? 4 : 0);
        }
    if (cudaMemcpy(s.fixm, loc8.data(), g.ncomp, cudaMemcpyHostToDevice) != cudaSuccess) { free_ctx(ctx); return TOPO_ECUDA; }
    // passive mask and dv (1 on design) over the whole local element array
    fill_local_elems_u8(ctx, s, passive, loc8);
    if (cudaMemcpy(s.passive, loc8.data(), g.nelloc, cudaMemcpyHostToDevice) != cudaSuccess) { free_ctx(ctx); return TOPO_ECUDA; }
    locd.assign(g.nelloc, 0.0);
    std::vector<double> locx(g.nelloc, 0.0);
    for (int exl = 0; exl < g.NEXL; ++exl) {
      const int ex = exl - g.H + g.ex0;
      if (ex < 0 || ex >= nelx) continue;
      for (int ez = 0; ez < nelz; ++ez)
        for (int ey = 0; ey < nely; ++ey) {
          const long long i = elem_idx(g, ex, ey, ez);
          const bool des = !loc8[i];
          locd[i] = des ? 1.0 : 0.0;
          locx[i] = des ? p->volfrac : loc8[i] == kSolid ? 1.0 : 0.0;   // R27
        }
    }
    if (cudaMemcpy(s.dv, locd.data(), sizeof(double) * g.nelloc, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(s.x, locx.data(), sizeof(double) * g.nelloc, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(s.xphys, locx.data(), sizeof(double) * g.nelloc, cudaMemcpyHostToDevice) != cudaSuccess) {
      free_ctx(ctx);
      return TOPO_ECUDA;
    }
  }
  rc = upload_nodes(ctx, load, &Slab::f);
  if (rc == TOPO_OK) rc = mg_build(ctx, fixed);
  if (rc == TOPO_OK) rc = mg_dist_plan(ctx);
  if (rc == TOPO_OK && ctx->mode == TOPO_DIST_HOST && W > 1) rc = open_host_transport(ctx, dist);
  if (rc == TOPO_OK) rc = ensure_constants(ctx);
  if (rc == TOPO_OK) {
    // ||f_free||^2 and filter row sums Hs (all local in-domain elements)
    for (Slab& s : ctx->slabs) {
      LAUNCH(ctx, k_dot, grid_for(3LL * s.g.nown * s.g.nplane), s.g, s.st, s.f, s.f, 0, s.partials, s.counter);
      LAUNCH(ctx, k_filter<F_HS>, grid_for(s.g.nelloc), s.g, (int)ctx->st_off.size(), s.hs, s.hs, s.hs,
             s.passive, s.hs, 1);
      LAUNCH(ctx, k_recip, grid_for(s.g.nelloc), s.g.nelloc, s.hs, s.ihs);
    }
    rc = check_launch(ctx);
  }
  if (rc == TOPO_OK) rc = allreduce(ctx, 0, 1, 0);
  if (rc == TOPO_OK) rc = sync_state(ctx);
  if (rc != TOPO_OK) { free_ctx(ctx); return rc; }
  ctx->bb = ctx->hstate->sums[0];
  // PCG batch size between host polls: ~ a few ms of device work
  {
    const long long ndof = 3 * nn;
    int b = p->cg_check_every;
    if (b <= 0) b = (int)std::min<long long>(64, std::max<long long>(8, 20000000LL / std::max<long long>(ndof, 1)));
    ctx->cg_batch = (b + 1) / 2 * 2;   // even: the p ping-pong returns to p0 after a batch
  }
  *out = ctx;
  return TOPO_OK;
}

int topo_partition(int32_t nelx, double rmin, int32_t world, int32_t rank, int32_t* ex_begin, int32_t* ex_end) {
  if (nelx < 1 || world < 1 || rank < 0 || rank >= world || !(rmin > 0)) return TOPO_EINVAL;
  const int R = std::max(0, (int)std::ceil(rmin) - 1);
  for (int s = 0; s < world; ++s) {
    const int a = (int)((long long)s * nelx / world), b = (int)((long long)(s + 1) * nelx / world);
    if (b - a < std::max(1, world > 1 ? R : 1)) return TOPO_EINVAL;
  }
  if (ex_begin) *ex_begin = (int)((long long)rank * nelx / world);
  if (ex_end) *ex_end = (int)((long long)(rank + 1) * nelx / world);
  return TOPO_OK;
}

int topo_set_stream(topo_ctx* ctx, void* stream) {
  if (!ctx) return TOPO_EINVAL;
  cudaStream_t s = stream ? (cudaStream_t)stream : ctx->own_stream;
  if (s != ctx->stream) {
    cudaStreamSynchronize(ctx->stream);
    ctx->stream = s;
    for (cudaGraphExec_t& g : ctx->cg_exec)
      if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    if (ctx->mg_setup_exec) { cudaGraphExecDestroy(ctx->mg_setup_exec); ctx->mg_setup_exec = nullptr; }
    if (ctx->mg_setup_exec_w) { cudaGraphExecDestroy(ctx->mg_setup_exec_w); ctx->mg_setup_exec_w = nullptr; }
    if (ctx->oc_exec) { cudaGraphExecDestroy(ctx->oc_exec); ctx->oc_exec = nullptr; }
    if (ctx->oc_exec_c) { cudaGraphExecDestroy(ctx->oc_exec_c); ctx->oc_exec_c = nullptr; }
    if (ctx->oc_exec_c2) { cudaGraphExecDestroy(ctx->oc_exec_c2); ctx->oc_exec_c2 = nullptr; }
    g_const_owner = nullptr;
  }
  return TOPO_OK;
}

int topo_owned_range(const topo_ctx* ctx, int32_t* ex_begin, int32_t* ex_end) {
  if (!ctx) return TOPO_EINVAL;
  if (ex_begin) *ex_begin = ctx->slabs.front().g.ex0;
  if (ex_end) *ex_end = ctx->slabs.back().g.ex1;
  return TOPO_OK;
}

static int set_x_common(topo_ctx* ctx, const double* x, bool also_xphys, bool dev = false) {
  if (x) {
    CK(dev ? upload_elems_dev(ctx, x, &Slab::x) : upload_elems(ctx, x, &Slab::x));
  } else {
    // x = volfrac * dv  (dv = 1 on design, 0 elsewhere)
    for (Slab& s : ctx->slabs) LAUNCH(ctx, k_fill_design, grid_for(s.g.nelloc), s.g, s.dv, ctx->prm.volfrac, s.x);
  }
  for (Slab& s : ctx->slabs) LAUNCH(ctx, k_apply_passive, grid_for(s.g.nelloc), s.g, s.passive, s.x);
  CK(check_launch(ctx));
  CK(exchange_elems(ctx, &Slab::x, ctx->slabs[0].g.H));
  if (also_xphys)
    for (Slab& s : ctx->slabs)
      CU(cudaMemcpyAsync(s.xphys, s.x, sizeof(double) * s.g.nelloc, cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->has_E = false;
  ctx->has_sens = ctx->has_dcf = false;
  return TOPO_OK;
}

int topo_set_density(topo_ctx* ctx, const double* x) {
  if (!ctx) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  CK(set_x_common(ctx, x, true));
  CU(cudaStreamSynchronize(ctx->stream));
  return TOPO_OK;
}

int topo_set_xphys(topo_ctx* ctx, const double* xphys) {
  if (!ctx || !xphys) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  CK(upload_elems(ctx, xphys, &Slab::xphys));
  for (Slab& s : ctx->slabs) LAUNCH(ctx, k_apply_passive, grid_for(s.g.nelloc), s.g, s.passive, s.xphys);
  CK(check_launch(ctx));
  CK(exchange_elems(ctx, &Slab::xphys, ctx->slabs[0].g.H));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->has_E = false;
  return TOPO_OK;
}

int topo_update_modulus(topo_ctx* ctx) {
  if (!ctx) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  CK(update_modulus(ctx));
  CU(cudaStreamSynchronize(ctx->stream));
  return TOPO_OK;
}

int topo_solve(topo_ctx* ctx, double* u, topo_solve_info* info) {
  if (!ctx) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  CU(cudaEventRecord(ctx->ev[0], ctx->stream));
  CK(update_modulus(ctx));
  CU(cudaEventRecord(ctx->ev[1], ctx->stream));
  int rc = do_solve(ctx, info);
  if (u) CK(download_nodes(ctx, &Slab::u, u));
  return rc;
}

int topo_sensitivity(topo_ctx* ctx, double* c, double* ce, double* dc) {
  if (!ctx) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  CK(do_sensitivity(ctx, c, nullptr));
  if (ce) CK(download_elems(ctx, &Slab::ce, ce));
  if (dc) CK(download_elems(ctx, &Slab::dc, dc));
  return TOPO_OK;
}

int topo_filter(topo_ctx* ctx, int32_t what, const double* in, double* out) {
  if (!ctx) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  if (what == TOPO_FILTER_DC) {
    if (in) {
      CK(upload_elems(ctx, in, &Slab::dc));
      ctx->has_sens = true;
    }
    if (!ctx->has_sens) return set_err(ctx, TOPO_ESTATE, "topo_filter(DC) before topo_sensitivity");
    CK(do_filter_dc(ctx));
    if (out) CK(download_elems(ctx, &Slab::dcf, out));
    return TOPO_OK;
  }
  if (what == TOPO_FILTER_X) {
    if (in) CK(set_x_common(ctx, in, false));
    CK(do_filter_x(ctx));
    if (out) CK(download_elems(ctx, &Slab::xphys, out));
    CU(cudaStreamSynchronize(ctx->stream));
    return TOPO_OK;
  }
  return set_err(ctx, TOPO_EINVAL, "topo_filter: bad `what`");
}

int topo_oc_step(topo_ctx* ctx, double* xnew, double* lambda, double* change, double* volume) {
  if (!ctx) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  CK(do_oc(ctx, lambda, change, volume));
  if (xnew) CK(download_elems(ctx, &Slab::x, xnew));
  return TOPO_OK;
}

int topo_optimize(topo_ctx* ctx, int32_t n_iter, double change_tol, double* c_hist, double* x_out,
                  int32_t* n_done) {
  if (!ctx) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  int rc = optimize_loop(ctx, n_iter, change_tol, c_hist, n_done);
  if (x_out) CK(download_elems(ctx, &Slab::x, x_out));
  return rc;
}

int topo_apply_K(topo_ctx* ctx, const double* p, double* q) {
  if (!ctx || !p) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  CK(topo_matvec_load(ctx, p));
  CK(topo_matvec_run(ctx, 1));
  for (Slab& s : ctx->slabs)
    LAUNCH(ctx, k_mask_fixed, grid_for((long long)s.g.nown * s.g.nplane), s.g, s.fixm, s.q);
  CK(check_launch(ctx));
  if (q) CK(download_nodes(ctx, &Slab::q, q));
  return TOPO_OK;
}

int topo_matvec_load(topo_ctx* ctx, const double* p) {
  if (!ctx || !p) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  if (!ctx->has_E) CK(update_modulus(ctx));
  CK(upload_nodes(ctx, p, &Slab::w));
  for (Slab& s : ctx->slabs)
    LAUNCH(ctx, k_mask_fixed, grid_for((long long)s.g.nown * s.g.nplane), s.g, s.fixm, s.w);
  CK(check_launch(ctx));
  CU(cudaStreamSynchronize(ctx->stream));
  return TOPO_OK;
}

int topo_matvec_run(topo_ctx* ctx, int32_t reps) {
  if (!ctx) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  CK(ensure_constants(ctx));
  if (!ctx->has_E) CK(update_modulus(ctx));
  for (int i = 0; i < reps; ++i) CK(matvec_all(ctx, &Slab::w, &Slab::m_w, &Slab::q));
  return TOPO_OK;
}

int topo_snapshot(topo_ctx* ctx) {
  if (!ctx) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  for (Slab& s : ctx->slabs) {
    const size_t nb = sizeof(double) * 3 * s.g.ncomp, eb = sizeof(double) * s.g.nelloc;
    if (!s.u_b) {
      CU(cudaMalloc(&s.u_b, nb));
      CU(cudaMalloc(&s.x_b, eb));
      CU(cudaMalloc(&s.xphys_b, eb));
      ctx->dev_bytes += nb + 2 * eb;
    }
    CU(cudaMemcpyAsync(s.u_b, s.u, nb, cudaMemcpyDeviceToDevice, ctx->stream));
    CU(cudaMemcpyAsync(s.x_b, s.x, eb, cudaMemcpyDeviceToDevice, ctx->stream));
    CU(cudaMemcpyAsync(s.xphys_b, s.xphys, eb, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (ctx->mg_on) {   // the multigrid power vectors (warm-started smoother weights)
    const size_t rs = sizeof(double);
    for (Slab& s : ctx->slabs) {
      const size_t nb0 = sizeof(double) * 3 * s.g.ncomp;
      if (!s.pw0_b) CU(cudaMalloc(&s.pw0_b, nb0));
      CU(cudaMemcpyAsync(s.pw0_b, s.pw0, nb0, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    for (MgLevel& m : ctx->mg) {
      if (!m.pw) continue;
      if (!m.pw_b) CU(cudaMalloc(&m.pw_b, rs * 3 * m.L.ncomp));
      CU(cudaMemcpyAsync(m.pw_b, m.pw, rs * 3 * m.L.ncomp, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    ctx->mg_warm_b = ctx->mg_warm;
    ctx->mg_f32_b = ctx->mg_f32;
    ctx->mg_theta_b = ctx->mg_theta;
  }
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->snap_has_u = ctx->has_u;
  ctx->has_snap = true;
  return TOPO_OK;
}

int topo_restore(topo_ctx* ctx) {
  if (!ctx) return TOPO_EINVAL;
  if (!ctx->has_snap) return set_err(ctx, TOPO_ESTATE, "topo_restore without topo_snapshot");
  cudaSetDevice(ctx->device);
  for (Slab& s : ctx->slabs) {
    const size_t nb = sizeof(double) * 3 * s.g.ncomp, eb = sizeof(double) * s.g.nelloc;
    CU(cudaMemcpyAsync(s.u, s.u_b, nb, cudaMemcpyDeviceToDevice, ctx->stream));
    CU(cudaMemcpyAsync(s.x, s.x_b, eb, cudaMemcpyDeviceToDevice, ctx->stream));
    CU(cudaMemcpyAsync(s.xphys, s.xphys_b, eb, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (ctx->mg_on && ctx->slabs[0].pw0_b) {
    const size_t rs = sizeof(double);
    for (Slab& s : ctx->slabs)
      CU(cudaMemcpyAsync(s.pw0, s.pw0_b, sizeof(double) * 3 * s.g.ncomp, cudaMemcpyDeviceToDevice, ctx->stream));
    for (MgLevel& m : ctx->mg)
      if (m.pw && m.pw_b)
        CU(cudaMemcpyAsync(m.pw, m.pw_b, rs * 3 * m.L.ncomp, cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->mg_warm = ctx->mg_warm_b;
    if (ctx->mg_theta != ctx->mg_theta_b) {
      ctx->mg_theta = ctx->mg_theta_b;
      mg_invalidate(ctx);
    }
    if (ctx->mg_f32 != ctx->mg_f32_b) {   // precision state of the snapshot (promotion undone)
      ctx->mg_f32 = ctx->mg_f32_b;
      mg_invalidate(ctx);
      CK(mg_clear_levels(ctx));
    }
  }
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->has_u = ctx->snap_has_u;
  ctx->has_E = ctx->has_sens = ctx->has_dcf = false;
  return TOPO_OK;
}

int topo_get(topo_ctx* ctx, int32_t field, double* out) {
  if (!ctx || !out) return TOPO_EINVAL;
  cudaSetDevice(ctx->device);
  switch (field) {
    case TOPO_FIELD_U: return download_nodes(ctx, &Slab::u, out);
    case TOPO_FIELD_X: return download_elems(ctx, &Slab::x, out);
    case TOPO_FIELD_XPHYS: return download_elems(ctx, &Slab::xphys, out);
    case TOPO_FIELD_E: return download_elems(ctx, &Slab::E, out);
    case TOPO_FIELD_CE: return download_elems(ctx, &Slab::ce, out);
    case TOPO_FIELD_DC: return download_elems(ctx, &Slab::dc, out);
    case TOPO_FIELD_DCF: return download_elems(ctx, &Slab::dcf, out);
    case TOPO_FIELD_DVF: return download_elems(ctx, &Slab::dvf, out);
    case TOPO_FIELD_XNEW: return download_elems(ctx, &Slab::xnew, out);
    case TOPO_FIELD_HS: return download_elems(ctx, &Slab::hs, out);
    case TOPO_FIELD_INVDIAG: return download_invd(ctx, out);
    case TOPO_FIELD_R: return download_nodes(ctx, &Slab::r, out);
    default: return set_err(ctx, TOPO_EINVAL, "unknown field %d", field);
  }
}

int topo_get_timings(const topo_ctx* ctx, topo_timings* t) {
  if (!ctx || !t) return TOPO_EINVAL;
  *t = ctx->tim;
  t->kernel_launches = ctx->launches;
  t->host_bytes = ctx->host_bytes;
  return TOPO_OK;
}

int topo_profile(topo_ctx* ctx, int32_t enable) {
  if (!ctx) return TOPO_EINVAL;
  ctx->profile = enable != 0;
  ctx->prof_ms = 0.0;
  ctx->prof_n = 0;
  for (int k = 0; k < 3; ++k) ctx->prof_ms_k[k] = 0.0, ctx->prof_n_k[k] = 0;
  return TOPO_OK;
}

int topo_kernel_time(topo_ctx* ctx, double* mean_ms, int64_t* samples) {
  if (!ctx) return TOPO_EINVAL;
  if (mean_ms) *mean_ms = ctx->prof_n ? ctx->prof_ms / ctx->prof_n : 0.0;
  if (samples) *samples = ctx->prof_n;
  return TOPO_OK;
}

int topo_kernel_time_k(topo_ctx* ctx, int32_t which, double* mean_ms, int64_t* samples) {
  if (!ctx || which < 0 || which > 2) return TOPO_EINVAL;
  if (which == 0) return topo_kernel_time(ctx, mean_ms, samples);
  if (mean_ms) *mean_ms = ctx->prof_n_k[which] ? ctx->prof_ms_k[which] / ctx->prof_n_k[which] : 0.0;
  if (samples) *samples = ctx->prof_n_k[which];
  return TOPO_OK;
}

int64_t topo_count(const topo_ctx* ctx, int32_t what) {
  if (!ctx) return -1;
  const topo_params& P = ctx->prm;
  switch (what) {
    case TOPO_COUNT_NDOF: return 3LL * (P.nelx + 1) * (P.nely + 1) * (P.nelz + 1);
    case TOPO_COUNT_NEL: return (long long)P.nelx * P.nely * P.nelz;
    case TOPO_COUNT_NODES: return (long long)(P.nelx + 1) * (P.nely + 1) * (P.nelz + 1);
    case TOPO_COUNT_DESIGN: return ctx->n_design;
    case TOPO_COUNT_STENCIL: return (long long)ctx->st_off.size();
    case TOPO_COUNT_DEVICE_BYTES: return (long long)ctx->dev_bytes;
    case TOPO_COUNT_MG_DIST: return ctx->mg_dl;
    default: return -1;
  }
}

int topo_mg_levels(topo_ctx* ctx, int32_t* n_levels, int32_t* dims) {
  if (!ctx || !n_levels) return TOPO_EINVAL;
  const int L = ctx->mg_on ? (int)ctx->mg.size() : 0;
  *n_levels = L;
  if (dims)
    for (int l = 0; l < L; ++l) {
      const LvGeo g = l == 0 ? lv0(ctx) : ctx->mg[l].L;
      dims[3 * l] = g.nx;
      dims[3 * l + 1] = g.ny;
      dims[3 * l + 2] = g.nz;
    }
  return TOPO_OK;
}

int topo_mg_apply(topo_ctx* ctx, int32_t level, const double* x, double* y) {
  if (!ctx || !x || !y) return TOPO_EINVAL;
  if (!ctx->mg_on) return set_err(ctx, TOPO_ESTATE, "topo_mg_apply: context has no multigrid hierarchy");
  if (level < 0 || level >= (int)ctx->mg.size()) return set_err(ctx, TOPO_EINVAL, "topo_mg_apply: bad level %d", level);
  cudaSetDevice(ctx->device);
  CK(ensure_constants(ctx));
  if (!ctx->has_E) CK(update_modulus(ctx));   // the hierarchy is formed from E(xPhys)
  CK(mg_setup(ctx));
  if (level == 0) return topo_apply_K(ctx, x, y);
  MgLevel& m = ctx->mg[level];
  if (ctx->mg_f32) {
    CK(mg_upload<float>(ctx, level, x, m.x));
    CK(mg_apply<float>(ctx, level, 0));
    return mg_download<float>(ctx, level, m.t, y);
  }
  CK(mg_upload<double>(ctx, level, x, m.x));
  CK(mg_apply<double>(ctx, level, 0));
  return mg_download<double>(ctx, level, m.t, y);
}

int topo_mg_vcycle(topo_ctx* ctx, const double* b, double* z) {
  if (!ctx || !b || !z) return TOPO_EINVAL;
  if (!ctx->mg_on) return set_err(ctx, TOPO_ESTATE, "topo_mg_vcycle: context has no multigrid hierarchy");
  cudaSetDevice(ctx->device);
  CK(ensure_constants(ctx));
  if (!ctx->has_E) CK(update_modulus(ctx));   // the hierarchy is formed from E(xPhys)
  CK(mg_setup(ctx));
  CK(upload_nodes(ctx, b, &Slab::r));
  for (Slab& s : ctx->slabs)
    LAUNCH(ctx, k_mask_fixed, grid_for((long long)s.g.nown * s.g.nplane), s.g, s.fixm, s.r);
  CK(check_launch(ctx));
  CK(exchange_nodes(ctx, &Slab::r));
  ctx->w32_off = true;
  const int rc = enqueue_vcycle(ctx, 0, 0, false);
  ctx->w32_off = false;
  CK(rc);
  return download_nodes(ctx, &Slab::w, z);   // the V-cycle result (last sweep fused into the matvec)
}

void topo_destroy(topo_ctx* ctx) { free_ctx(ctx); }

// ---------------------------------------------------------------------------
// _d variants: CUDA device pointers (whole external arrays, S:45 numbering) and
// the caller's cudaStream_t.  Field data never passes through the host; work is
// stream-ordered (outputs are complete in `stream` order).  Scalars (c, lambda,
// ...) are still returned on the host: the PCG / OC drivers poll device state.
// ---------------------------------------------------------------------------
static int bind_stream(topo_ctx* ctx, void* stream) {
  cudaSetDevice(ctx->device);
  if (stream && (cudaStream_t)stream != ctx->stream) return topo_set_stream(ctx, stream);
  return TOPO_OK;
}

static int dev_pointer_ok(topo_ctx* ctx, const void* p, const char* what) {
  if (!p) return TOPO_OK;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess || (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)) {
    cudaGetLastError();
    return set_err(ctx, TOPO_EINVAL, "%s: not a CUDA device pointer", what);
  }
  if (a.type == cudaMemoryTypeDevice && a.device != ctx->device)
    return set_err(ctx, TOPO_EINVAL, "%s: device pointer of device %d, context on device %d", what, a.device, ctx->device);
  return TOPO_OK;
}
#define DEVPTR(p) CK(dev_pointer_ok(ctx, (p), #p))

int topo_init_d(const topo_params* p, const double* load_d, const uint8_t* fixed_d, const uint8_t* passive_d,
                const topo_dist* dist, void* stream, topo_ctx** out) {
  if (!out || !p || !load_d || !fixed_d) return TOPO_EINVAL;
  *out = nullptr;
  if (p->nelx < 1 || p->nely < 1 || p->nelz < 1) return TOPO_EINVAL;
  // one-time problem statement: the host-side setup (partition, multigrid
  // hierarchy, Dirichlet / passive masks) reads these once; copied here
  const size_t nn = (size_t)(p->nelx + 1) * (p->nely + 1) * (p->nelz + 1), ne = (size_t)p->nelx * p->nely * p->nelz;
  std::vector<double> load(3 * nn);
  std::vector<uint8_t> fixed(3 * nn), passive(passive_d ? ne : 0);
  if (cudaMemcpy(load.data(), load_d, sizeof(double) * 3 * nn, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(fixed.data(), fixed_d, 3 * nn, cudaMemcpyDeviceToHost) != cudaSuccess ||
      (passive_d && cudaMemcpy(passive.data(), passive_d, ne, cudaMemcpyDeviceToHost) != cudaSuccess)) {
    cudaGetLastError();
    return TOPO_EINVAL;
  }
  int rc = topo_init(p, load.data(), fixed.data(), passive_d ? passive.data() : nullptr, dist, out);
  if (rc == TOPO_OK && stream) rc = topo_set_stream(*out, stream);
  return rc;
}

int topo_set_density_d(topo_ctx* ctx, const double* x_d, void* stream) {
  if (!ctx) return TOPO_EINVAL;
  CK(bind_stream(ctx, stream));
  DEVPTR(x_d);
  return set_x_common(ctx, x_d, true, true);
}

int topo_set_xphys_d(topo_ctx* ctx, const double* xphys_d, void* stream) {
  if (!ctx || !xphys_d) return TOPO_EINVAL;
  CK(bind_stream(ctx, stream));
  DEVPTR(xphys_d);
  CK(upload_elems_dev(ctx, xphys_d, &Slab::xphys));
  for (Slab& s : ctx->slabs) LAUNCH(ctx, k_apply_passive, grid_for(s.g.nelloc), s.g, s.passive, s.xphys);
  CK(check_launch(ctx));
  CK(exchange_elems(ctx, &Slab::xphys, ctx->slabs[0].g.H));
  ctx->has_E = false;
  return TOPO_OK;
}

int topo_solve_d(topo_ctx* ctx, double* u_d, topo_solve_info* info, void* stream) {
  if (!ctx) return TOPO_EINVAL;
  CK(bind_stream(ctx, stream));
  DEVPTR(u_d);
  CU(cudaEventRecord(ctx->ev[0], ctx->stream));
  CK(update_modulus(ctx));
  CU(cudaEventRecord(ctx->ev[1], ctx->stream));
  int rc = do_solve(ctx, info);
  if (u_d) CK(download_nodes_dev(ctx, &Slab::u, u_d));
  return rc;
}

int topo_sensitivity_d(topo_ctx* ctx, double* c, double* ce_d, double* dc_d, void* stream) {
  if (!ctx) return TOPO_EINVAL;
  CK(bind_stream(ctx, stream));
  DEVPTR(ce_d);
  DEVPTR(dc_d);
  CK(do_sensitivity(ctx, c, nullptr));
  if (ce_d) CK(download_elems_dev(ctx, &Slab::ce, ce_d));
  if (dc_d) CK(download_elems_dev(ctx, &Slab::dc, dc_d));
  return TOPO_OK;
}

int topo_filter_d(topo_ctx* ctx, int32_t what, const double* in_d, double* out_d, void* stream) {
  if (!ctx) return TOPO_EINVAL;
  CK(bind_stream(ctx, stream));
  DEVPTR(in_d);
  DEVPTR(out_d);
  if (what == TOPO_FILTER_DC) {
    if (in_d) {
      CK(upload_elems_dev(ctx, in_d, &Slab::dc));
      ctx->has_sens = true;
    }
    if (!ctx->has_sens) return set_err(ctx, TOPO_ESTATE, "topo_filter_d(DC) before topo_sensitivity");
    CK(do_filter_dc(ctx));
    if (out_d) CK(download_elems_dev(ctx, &Slab::dcf, out_d));
    return TOPO_OK;
  }
  if (what == TOPO_FILTER_X) {
    if (in_d) CK(set_x_common(ctx, in_d, false, true));
    CK(do_filter_x(ctx));
    if (out_d) CK(download_elems_dev(ctx, &Slab::xphys, out_d));
    return TOPO_OK;
  }
  return set_err(ctx, TOPO_EINVAL, "topo_filter_d: bad `what`");
}

int topo_oc_step_d(topo_ctx* ctx, double* xnew_d, double* lambda, double* change, double* volume, void* stream) {
  if (!ctx) return TOPO_EINVAL;
  CK(bind_stream(ctx, stream));
  DEVPTR(xnew_d);
  CK(do_oc(ctx, lambda, change, volume));
  if (xnew_d) CK(download_elems_dev(ctx, &Slab::x, xnew_d));
  return TOPO_OK;
}

int topo_optimize_d(topo_ctx* ctx, int32_t n_iter, double change_tol, double* c_hist, double* x_out_d,
                    int32_t* n_done, void* stream) {
  if (!ctx) return TOPO_EINVAL;
  CK(bind_stream(ctx, stream));
  DEVPTR(x_out_d);
  int rc = optimize_loop(ctx, n_iter, change_tol, c_hist, n_done);
  if (x_out_d) CK(download_elems_dev(ctx, &Slab::x, x_out_d));
  return rc;
}

int topo_apply_K_d(topo_ctx* ctx, const double* p_d, double* q_d, void* stream) {
  if (!ctx || !p_d) return TOPO_EINVAL;
  CK(bind_stream(ctx, stream));
  DEVPTR(p_d);
  DEVPTR(q_d);
  CK(ensure_constants(ctx));
  if (!ctx->has_E) CK(update_modulus(ctx));
  CK(upload_nodes_dev(ctx, p_d, &Slab::w));
  for (Slab& s : ctx->slabs) LAUNCH(ctx, k_mask_fixed, grid_for((long long)s.g.nown * s.g.nplane), s.g, s.fixm, s.w);
  CK(check_launch(ctx));
  CK(matvec_all(ctx, &Slab::w, &Slab::m_w, &Slab::q));
  for (Slab& s : ctx->slabs) LAUNCH(ctx, k_mask_fixed, grid_for((long long)s.g.nown * s.g.nplane), s.g, s.fixm, s.q);
  CK(check_launch(ctx));
  if (q_d) CK(download_nodes_dev(ctx, &Slab::q, q_d));
  return TOPO_OK;
}

int topo_get_d(topo_ctx* ctx, int32_t field, double* out_d, void* stream) {
  if (!ctx || !out_d) return TOPO_EINVAL;
  CK(bind_stream(ctx, stream));
  DEVPTR(out_d);
  switch (field) {
    case TOPO_FIELD_U: return download_nodes_dev(ctx, &Slab::u, out_d);
    case TOPO_FIELD_X: return download_elems_dev(ctx, &Slab::x, out_d);
    case TOPO_FIELD_XPHYS: return download_elems_dev(ctx, &Slab::xphys, out_d);
    case TOPO_FIELD_E: return download_elems_dev(ctx, &Slab::E, out_d);
    case TOPO_FIELD_CE: return download_elems_dev(ctx, &Slab::ce, out_d);
    case TOPO_FIELD_DC: return download_elems_dev(ctx, &Slab::dc, out_d);
    case TOPO_FIELD_DCF: return download_elems_dev(ctx, &Slab::dcf, out_d);
    case TOPO_FIELD_DVF: return download_elems_dev(ctx, &Slab::dvf, out_d);
    case TOPO_FIELD_XNEW: return download_elems_dev(ctx, &Slab::xnew, out_d);
    case TOPO_FIELD_HS: return download_elems_dev(ctx, &Slab::hs, out_d);
    case TOPO_FIELD_INVDIAG: return download_invd_dev(ctx, out_d);
    case TOPO_FIELD_R: return download_nodes_dev(ctx, &Slab::r, out_d);
    default: return set_err(ctx, TOPO_EINVAL, "unknown field %d", field);
  }
}

}  // extern "C"

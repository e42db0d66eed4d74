// K2 + K3: occupancy filter and fp64 time / power / energy prediction over the
// kernel x spec x shape x cap grid.
//
// Reference arithmetic restated (never copied): features.py:55-59,96-114,
// time_model.py:33-129, power_model.py:31-170, explorer.py:76-92,105-108.
// Every fp64 operation below is a single IEEE-754 binary64 op in the reference's
// evaluation order; this translation unit is compiled with -fmad=false so nvcc never
// contracts a*b+c.  libm log/pow are evaluated on the host (tables), see ffb.h.
//
// Work decomposition (B200): the expensive part of a point — ~10 fp64 divides — does not
// depend on the power cap, so one thread owns one (kernel, spec, shape) unit, evaluates the
// cap-independent chain once, then walks the cap axis (7 flops per cap).  Results are staged
// in shared memory so that the [unit, cap] tile leaves the SM as fully coalesced 8-byte
// stores: the kernel is an HBM write stream of 16 B per grid point.
#include "ffb_common.cuh"

#include <math.h>
#include <string.h>
#include <algorithm>

namespace {

constexpr int kUnitsPerCta = 256;
constexpr int kKsWidth = 8;    // doubles per (kernel, spec) row
constexpr int kSdWidth = 16;   // doubles per derived-spec row

enum { KS_SHARED_LIMIT = 0, KS_DENOM_COMP, KS_CI, KS_P_SM, KS_N_COMP, KS_CWP, KS_ACTIVE, KS_ERR };
enum { SD_MWP = 0, SD_FLOOR, SD_RATIO0 /* 5 entries */, SD_SKIPMASK = 7, SD_ERR = 8 };

struct Tables {
  const double* spec;      // [S, FFB_SPEC_WIDTH]
  const double* sd;        // [S, kSdWidth]
  const int32_t* shape;    // [J, 4]
  const double* shape_log; // [J]
  const double* cap;       // [C]
  const double* cap_scale; // [S, C]  f_adj / f_base
  const double* cap_fadj;  // [S, C]
  const double* cap_ok;    // [S, C]  1.0 when p_cap_min <= cap <= p_tdp
  const double* cap_tab;   // [S, C, 4] {scale, cap, max(0, cap - p_static), ok}: the cap axis in one 32-byte row
  const double* psm;       // [S, psm_n]
  int psm_n;
};

// ---- per (kernel, spec) hoisting --------------------------------------------------------
__global__ void __launch_bounds__(256)
predict_prepare_kernel(const double* __restrict__ feat, const int64_t* __restrict__ res, Tables tb,
                       int64_t n_kernels, int n_specs, double* __restrict__ kstab,
                       uint32_t* __restrict__ status) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_kernels * n_specs) return;
  int64_t k = i / n_specs;
  int s = (int)(i - k * n_specs);
  const double* f = feat + k * FFB_FEAT_WIDTH;
  const double* sp = tb.spec + (size_t)s * FFB_SPEC_WIDTH;
  const double* sd = tb.sd + (size_t)s * kSdWidth;
  uint32_t err = 0;

  const int64_t shared = (int64_t)f[FFB_F_STATIC_SHARED] + res[2 * k + 0];   // features.py:111
  const int64_t total_blocks = res[2 * k + 1];
  if (total_blocks <= 0) err |= 1u << FFB_E_EMPTY_GRID;                     // time_model.py:75
  double shared_limit = INFINITY;
  if (shared > 0) shared_limit = sp[FFB_S_MAX_SHARED] / (double)shared;       // features.py:113

  // time_model.py:47-64 (_issue_window): FP32, INT, SFU weighted by exec/issue
  double weighted = 0.0, total = 0.0;
  for (int u = 0; u < 3; ++u) {
    const double cnt = f[FFB_F_FP32 + u];
    weighted = weighted + cnt * sd[SD_RATIO0 + u];
    total = total + cnt;
  }
  const double window = (total <= 0.0) ? sd[SD_RATIO0 + 3] : weighted / total;
  double cwp = 1.0;
  if (window <= 0.0) err |= 1u << FFB_E_ZERO_COMPUTE;                       // time_model.py:42
  else cwp = py_max(1.0, (sp[FFB_S_L_COAL] + window) / window);               // time_model.py:44
  const bool ovr = f[FFB_F_OVR] != 0.0;
  const double n_comp = ovr ? f[FFB_F_OVR_NCOMP]
                            : (f[FFB_F_FP32] + f[FFB_F_INT]) + f[FFB_F_SFU];  // features.py:108
  const double n_mem = f[FFB_F_N_MEM];
  const double ci = (n_mem == 0.0) ? INFINITY : n_comp / n_mem;               // power_model.py:44-46
  const int64_t sm = (int64_t)sp[FFB_S_SM_COUNT];
  int64_t active = total_blocks < sm ? total_blocks : sm;                    // power_model.py:86
  if (active < 0) active = 0;
  double* o = kstab + i * kKsWidth;
  o[KS_SHARED_LIMIT] = shared_limit;
  o[KS_DENOM_COMP] = (cwp * sp[FFB_S_IPC]) * sp[FFB_S_F_BASE];                // time_model.py:116
  o[KS_CI] = ci;
  o[KS_P_SM] = tb.psm[(size_t)s * tb.psm_n + active];                         // power_model.py:74-76
  o[KS_N_COMP] = n_comp;
  o[KS_CWP] = cwp;
  o[KS_ACTIVE] = (double)active;
  o[KS_ERR] = (double)err;
  if (err && status) atomicOr(status, err);
}

// ---- the grid ---------------------------------------------------------------------------
struct GridArgs {
  const double* feat;
  const int64_t* res;
  const double* kstab;
  Tables tb;
  int64_t n_units;     // K*S*J
  int n_specs, n_shapes, n_caps;
  int cap_tile;        // caps staged per pass (== n_caps unless the [units, caps] tile would not fit shared memory)
  double* t;
  double* e;
  double* pdyn;
  uint8_t* flags;
  double* occ;
  double* detail;
  uint32_t* status;
  int strict;
};

// kLean: only t / e requested and no strict checks — the streaming configuration
template <bool kDetail, bool kLean>
__global__ void __launch_bounds__(kUnitsPerCta, kLean ? 5 : 1)
predict_grid_kernel(GridArgs a) {
  FFB_DYN_SMEM(smem_raw);
  const int C = a.n_caps, CT = a.cap_tile;
  double* s_t = reinterpret_cast<double*>(smem_raw);            // [units][CT]
  double* s_e = s_t + (size_t)kUnitsPerCta * CT;
  double* s_p = s_e + (size_t)kUnitsPerCta * CT;                // only when pdyn requested
  uint8_t* s_f = reinterpret_cast<uint8_t*>(s_p + (a.pdyn ? (size_t)kUnitsPerCta * CT : 0));

  const int64_t unit0 = (int64_t)blockIdx.x * kUnitsPerCta;
  const int64_t unit = unit0 + threadIdx.x;
  const bool live = unit < a.n_units;

  // per-thread values the cap axis needs (set by live threads only)
  double t_exec = 0.0, p_pre = 0.0, p_static = 0.0, e_over = 0.0;
  bool unit_valid = false;
  int s = 0;
  // detail-only copies
  double d_mwp = 0.0, d_cwp = 0.0, d_bw = 0.0, d_tm = 0.0, d_tc = 0.0, d_ts = 0.0, d_pu = 0.0, d_ps = 0.0, d_pm = 0.0, d_psm = 0.0,
         d_ci = 0.0, d_act = 0.0, d_warps = 0.0, d_bps = 0.0, d_eta = 0.0, d_waves = 0.0;
  if (live) {
    int64_t ks, k;
    int j;
    if (a.n_units <= 0x7fffffffLL) {                   // 32-bit index arithmetic on the common sizes
      const uint32_t u32 = (uint32_t)unit, ks32 = u32 / (uint32_t)a.n_shapes, k32 = ks32 / (uint32_t)a.n_specs;
      j = (int)(u32 - ks32 * (uint32_t)a.n_shapes); s = (int)(ks32 - k32 * (uint32_t)a.n_specs);
      ks = ks32; k = k32;
    } else {
      ks = unit / a.n_shapes; j = (int)(unit - ks * a.n_shapes);
      k = ks / a.n_specs; s = (int)(ks - k * a.n_specs);
    }
    const double* f = a.feat + k * FFB_FEAT_WIDTH;
    const double* sp = a.tb.spec + (size_t)s * FFB_SPEC_WIDTH;
    const double* sd = a.tb.sd + (size_t)s * kSdWidth;
    const double* kr = a.kstab + ks * kKsWidth;
    const int32_t* sh = a.tb.shape + 4 * j;
    const int64_t bx = sh[0], by = sh[1], bz = sh[2], regs = sh[3];
    uint32_t err = (uint32_t)kr[KS_ERR] | (uint32_t)sd[SD_ERR];

    // ---- K2: integer occupancy / validity (explorer.py:76-88, features.py:96-114) ----
    const int64_t threads = bx * by * bz;
    const int64_t max_threads = (int64_t)sp[FFB_S_MAX_THREADS];
    const int64_t max_warps = (int64_t)sp[FFB_S_MAX_WARPS];
    const int64_t shared_dyn = a.res[2 * k + 0];
    const int64_t total_blocks = a.res[2 * k + 1];
    const bool ovr = f[FFB_F_OVR] != 0.0;
    const bool shape_ok = ovr || (threads >= 32 && threads <= max_threads && (threads % 32) == 0);
    if (!shape_ok) err |= (a.strict ? 1u << FFB_E_INVALID_CONFIG : 0u);
    const int64_t warps = ovr ? (int64_t)f[FFB_F_OVR_WARPS] : (shape_ok ? threads / 32 : 1);
    bool fits = warps <= max_warps;                                   // max_warps/warps >= 1.0
    if (shared_dyn > 0) fits = fits && shared_dyn <= (int64_t)sp[FFB_S_MAX_SHARED];
    const double wf = (double)warps;
    double bps = sp[FFB_S_MAX_WARPS] / wf;                            // features.py:112
    bps = py_min(bps, kr[KS_SHARED_LIMIT]);                           // features.py:114
    const double regs_per_sm = sp[FFB_S_REGS_PER_SM];
    if (regs_per_sm > 0.0 && regs > 0) {                              // extension, see DESIGN.md
      const double reg_limit = regs_per_sm / (double)(regs * threads);
      bps = py_min(bps, reg_limit);
      fits = fits && reg_limit >= 1.0;
    }
    if (ovr) bps = f[FFB_F_OVR_BPS];
    unit_valid = (a.strict || ovr) ? shape_ok : (shape_ok && fits);
    const double eta = ovr ? f[FFB_F_OVR_ETA]
                           : py_min(1.0, (double)bx / 32.0) * f[FFB_F_ALIGNED];   // features.py:59

    // ---- time (time_model.py:67-129) ----
    const double resident = py_min(bps * wf, (double)max_warps);
    const double lanes = (sp[FFB_S_SM_COUNT] * resident) * 32.0;
    const double tthreads = (double)(total_blocks * warps) * 32.0;
    const double waves = py_max(1.0, tthreads / lanes);
    const double mwp = sd[SD_MWP];
    const double bw_eff = sp[FFB_S_BW_MAX] * py_max(eta, sd[SD_FLOOR]);
    const double mb = f[FFB_F_MEM_BYTES] * waves;
    if (mb > 0.0 && bw_eff <= 0.0) err |= 1u << FFB_E_ZERO_BANDWIDTH;
    const double t_mem = (mb > 0.0) ? mb / (mwp * bw_eff) : 0.0;
    const double nc = kr[KS_N_COMP] * waves;
    const double t_comp = (nc > 0.0) ? nc / kr[KS_DENOM_COMP] : 0.0;
    const double t_sync = (f[FFB_F_N_SYNC] * waves) * sp[FFB_S_T_BARRIER];
    t_exec = ((sp[FFB_S_W_MEM] * t_mem + sp[FFB_S_W_COMP] * t_comp) +
                           sp[FFB_S_W_SYNC] * t_sync) + sp[FFB_S_T_BASE];

    // ---- power, cap-independent part (power_model.py:124-150) ----
    const double wps = py_min(wf * bps, (double)max_warps);
    double p_units = 0.0;
    const uint32_t skip = (uint32_t)sd[SD_SKIPMASK];
#pragma unroll
    for (int u = 0; u < 5; ++u) {
      if (skip & (1u << u)) continue;
      const double cnt = (u == 4) ? f[FFB_F_N_MEM] : f[FFB_F_FP32 + u];
      const double rate = (cnt * wps) / sd[SD_RATIO0 + u];
      p_units = p_units + sp[FFB_S_BETA0 + u] * rate;
    }
    const double ci = kr[KS_CI];
    double p_shape = sp[FFB_S_P_BASE_SHAPE];
    if (!isinf(ci)) {
      const double penalty = (sp[FFB_S_KAPPA] * a.tb.shape_log[j]) / (1.0 + ci);
      p_shape = sp[FFB_S_P_BASE_SHAPE] * (1.0 + penalty);
    }
    const double p_mem = sp[FFB_S_P_MEM_BASE] * (1.0 + sp[FFB_S_LAMBDA] * (1.0 - eta));
    const double p_sm = kr[KS_P_SM];
    p_pre = ((p_units + p_shape) + p_mem) + p_sm;
    const double t_seen = (ovr && f[FFB_F_OVR_TEXEC] == f[FFB_F_OVR_TEXEC]) ? f[FFB_F_OVR_TEXEC] : t_exec;
    if (t_seen < sp[FFB_S_TAU_SHORT]) p_pre = p_pre * sp[FFB_S_TRANSIENT_R];      // power_model.py:93-95
    p_static = sp[FFB_S_P_STATIC];
    e_over = sp[FFB_S_E_OVERHEAD];
    if (kDetail) {
      d_mwp = mwp; d_cwp = kr[KS_CWP]; d_bw = bw_eff; d_tm = t_mem; d_tc = t_comp; d_ts = t_sync; d_pu = p_units; d_ps = p_shape;
      d_pm = p_mem; d_psm = p_sm; d_ci = ci; d_act = kr[KS_ACTIVE]; d_warps = (double)warps; d_bps = bps; d_eta = eta; d_waves = waves;
    }

    if (!kLean) {
      if (a.occ) a.occ[unit] = bps;
      if (err && a.status) atomicOr(a.status, err);
    }

  }

  // ---- cap axis (power_model.py:152-158, explorer.py:107), CT caps per pass ----
  const int64_t rem = a.n_units - unit0;
  const int n_live = rem < kUnitsPerCta ? (int)rem : kUnitsPerCta;
  for (int c0 = 0; c0 < C; c0 += CT) {
    const int ct = C - c0 < CT ? C - c0 : CT;
    if (live) {
      const double2* ct2 = reinterpret_cast<const double2*>(a.tb.cap_tab + ((size_t)s * C + c0) * 4);
      const bool any_cap = kLean ? false : (a.strict != 0);
      for (int c = 0; c < ct; ++c) {
        const double2 sc_cap = ct2[2 * c], room_ok = ct2[2 * c + 1];
        double p_dyn = p_pre * sc_cap.x;
        const bool limited = p_dyn + p_static > sc_cap.y;
        if (limited) p_dyn = room_ok.x;                       // max(0.0, cap - p_static), tabulated
        const double e_pred = t_exec * (p_dyn + p_static) + e_over;
        const bool ok = unit_valid && (any_cap || room_ok.y != 0.0);
        const size_t o = (size_t)threadIdx.x * ct + c;
        s_t[o] = ok ? t_exec : INFINITY;
        s_e[o] = ok ? e_pred : INFINITY;
        if (!kLean) {
          if (a.pdyn) s_p[o] = p_dyn;
          if (a.flags) s_f[o] = (uint8_t)((ok ? FFB_PT_VALID : 0) | (limited ? FFB_PT_CAP_LIMITED : 0));
        }
        if (kDetail) {
          double* d = a.detail + ((size_t)unit * C + c0 + c) * FFB_DETAIL_WIDTH;
          d[FFB_D_MWP] = d_mwp; d[FFB_D_CWP] = d_cwp; d[FFB_D_BW_EFF] = d_bw;
          d[FFB_D_T_MEM] = d_tm; d[FFB_D_T_COMP] = d_tc; d[FFB_D_T_SYNC] = d_ts;
          d[FFB_D_T_EXEC] = t_exec; d[FFB_D_P_UNITS] = d_pu; d[FFB_D_P_SHAPE] = d_ps;
          d[FFB_D_P_MEM] = d_pm; d[FFB_D_P_SM] = d_psm; d[FFB_D_P_DYN] = p_dyn;
          d[FFB_D_F_ADJ] = a.tb.cap_fadj[(size_t)s * C + c0 + c]; d[FFB_D_CI] = d_ci;
          d[FFB_D_ACTIVE_SMS] = d_act; d[FFB_D_CAP_LIMITED] = limited ? 1.0 : 0.0;
          d[FFB_D_E_PRED] = e_pred; d[FFB_D_WARPS] = d_warps; d[FFB_D_BLOCKS_PER_SM] = d_bps;
          d[FFB_D_ETA] = d_eta; d[FFB_D_WAVES] = d_waves;
        }
      }
    }
    __syncthreads();

    // ---- coalesced write-out of the [units, ct] tile ----
    const int total = n_live * ct;
    if (ct == C) {
      const size_t base = (size_t)unit0 * C;
      if (kLean && (base & 1) == 0) {
        // 16-byte stores: the tile starts on an even element, so (t + base) is 16-byte aligned
        const int pairs = total >> 1;
        double2* gt = reinterpret_cast<double2*>(a.t + base);
        double2* ge = reinterpret_cast<double2*>(a.e + base);
        const double2* st2 = reinterpret_cast<const double2*>(s_t);
        const double2* se2 = reinterpret_cast<const double2*>(s_e);
        for (int i = threadIdx.x; i < pairs; i += kUnitsPerCta) { gt[i] = st2[i]; ge[i] = se2[i]; }
        if ((total & 1) && threadIdx.x == 0) { a.t[base + total - 1] = s_t[total - 1]; a.e[base + total - 1] = s_e[total - 1]; }
      } else {
        for (int i = threadIdx.x; i < total; i += kUnitsPerCta) {
          if (a.t) a.t[base + i] = s_t[i];
          if (a.e) a.e[base + i] = s_e[i];
          if (!kLean) {
            if (a.pdyn) a.pdyn[base + i] = s_p[i];
            if (a.flags) a.flags[base + i] = s_f[i];
          }
        }
      }
    } else {
      // cap axis in several passes: runs of ct values per unit
      for (int i = threadIdx.x; i < total; i += kUnitsPerCta) {
        const int u = i / ct, c = i - u * ct;
        const size_t o = (size_t)(unit0 + u) * C + c0 + c;
        if (a.t) a.t[o] = s_t[i];
        if (a.e) a.e[o] = s_e[i];
        if (!kLean) {
          if (a.pdyn) a.pdyn[o] = s_p[i];
          if (a.flags) a.flags[o] = s_f[i];
        }
      }
    }
    if (c0 + CT < C) __syncthreads();
  }
}

}  // namespace

// ---- host side ----------------------------------------------------------------------------

static int32_t validate_spec_row(FfbContext* ctx, const double* sp, int s, int strict, double* sd) {
  // time_model.py:33-37
  uint32_t err = 0;
  if (sp[FFB_S_DEP_DELAY] <= 0.0) err |= 1u << FFB_E_ZERO_DELAY;
  sd[SD_MWP] = (sp[FFB_S_DEP_DELAY] > 0.0) ? py_max(1.0, sp[FFB_S_L_COAL] / sp[FFB_S_DEP_DELAY]) : 1.0;
  // time_model.py:103-105
  sd[SD_FLOOR] = (sp[FFB_S_L_UNCOAL] > 0.0) ? sp[FFB_S_L_COAL] / sp[FFB_S_L_UNCOAL] : 0.0;
  uint32_t skip = 0;
  for (int u = 0; u < 5; ++u) {
    // power_model.py:128-136: the Mem unit uses the measured coalesced latency as exec cycles
    const double ex = (u == 4) ? sp[FFB_S_L_COAL] : sp[FFB_S_EXEC0 + u];
    const double is = sp[FFB_S_ISSUE0 + u];
    if (ex <= 0.0) { skip |= 1u << u; }
    else if (is <= 0.0) { err |= 1u << FFB_E_ZERO_CYCLES; skip |= 1u << u; }
    // time_model.py:58,63 divides the *architectural* exec cycles, also for units the power
    // model skips; Mem never enters the window so one ratio table serves both
    const double ex_arch = (u == 4) ? ex : sp[FFB_S_EXEC0 + u];
    sd[SD_RATIO0 + u] = (is != 0.0) ? ex_arch / is : 0.0;
  }
  sd[SD_SKIPMASK] = (double)skip;
  sd[SD_ERR] = (double)err;
  (void)ctx; (void)s; (void)strict;
  return FFB_OK;
}

extern "C" int32_t ffb_predict_grid(FfbContext* ctx, const FfbGridDesc* g, void* stream_) {
  if (!ctx || !g) return FFB_E_BAD_ARGUMENT;
  cudaStream_t stream = (cudaStream_t)stream_;
  const int64_t K = g->n_kernels, S = g->n_specs, J = g->n_shapes, C = g->n_caps;
  if (K < 0 || S <= 0 || J < 0 || C <= 0 || S > (1 << 20) || J > (1 << 28) || C > 4096)
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_predict_grid: bad extents K=%lld S=%lld J=%lld C=%lld",
                    (long long)K, (long long)S, (long long)J, (long long)C);
  if (!g->d_feat || !g->d_res || !g->h_spec || !g->h_shape || !g->h_cap)
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_predict_grid: null input");
  if (K == 0 || J == 0) return FFB_OK;
  FFB_CUDA(ctx, cudaSetDevice(ctx->device));

  // ---- host tables (libm here, same as the reference's math.log / ** ) ----
  int psm_n = 1;
  for (int64_t s = 0; s < S; ++s) {
    double sm = g->h_spec[s * FFB_SPEC_WIDTH + FFB_S_SM_COUNT];
    if (!(sm >= 0.0) || sm > 1e6) return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "spec %lld: sm_count out of range", (long long)s);
    if ((int)sm + 1 > psm_n) psm_n = (int)sm + 1;
  }
  const size_t n_spec = (size_t)S * FFB_SPEC_WIDTH, n_sd = (size_t)S * kSdWidth, n_log = (size_t)J,
               n_cap = (size_t)C, n_sc = (size_t)S * C, n_psm = (size_t)S * psm_n;
  const size_t n_dbl = n_spec + n_sd + n_log + n_cap + 7 * n_sc + n_psm;
  const size_t bytes = n_dbl * sizeof(double) + (size_t)J * 4 * sizeof(int32_t);
  // The tables are built in pageable memory first: a call whose tables equal the ones already on the
  // device (chunked pipelines score many kernel ranges against the same specs / shapes / caps) neither
  // uploads them again nor waits for the pinned staging buffer, so the host can keep enqueueing.
  std::vector<unsigned char> scratch(bytes);
  int32_t rc = ffb_reserve(ctx, &ctx->d_tables, bytes);
  if (rc) return rc;
  double* h = (double*)scratch.data();
  double* h_spec = h;
  double* h_sd = h_spec + n_spec;
  double* h_ctab = h_sd + n_sd;            // 64*S doubles precede it: rows stay 32-byte aligned
  double* h_log = h_ctab + 4 * n_sc;
  double* h_cap = h_log + n_log;
  double* h_scale = h_cap + n_cap;
  double* h_fadj = h_scale + n_sc;
  double* h_ok = h_fadj + n_sc;
  double* h_psm = h_ok + n_sc;
  int32_t* h_shape = (int32_t*)(h_psm + n_psm);
  memcpy(h_spec, g->h_spec, n_spec * sizeof(double));
  memcpy(h_cap, g->h_cap, n_cap * sizeof(double));
  memcpy(h_shape, g->h_shape, (size_t)J * 4 * sizeof(int32_t));
  uint32_t host_err = 0;
  for (int64_t s = 0; s < S; ++s) {
    const double* sp = h_spec + s * FFB_SPEC_WIDTH;
    validate_spec_row(ctx, sp, (int)s, g->strict, h_sd + s * kSdWidth);
    host_err |= (uint32_t)h_sd[s * kSdWidth + SD_ERR];
    const double tdp = sp[FFB_S_P_TDP], fb = sp[FFB_S_F_BASE];
    const double inv_k = 1.0 / (double)(int64_t)sp[FFB_S_DVFS_K];          // power_model.py:106
    for (int64_t c = 0; c < C; ++c) {
      const double cap = h_cap[c];
      const bool in_range = (sp[FFB_S_P_CAP_MIN] <= cap) && (cap <= tdp);      // explorer.py:90
      const bool legal = cap > 0.0 && tdp > 0.0 && cap <= tdp;                 // power_model.py:100-105
      if (g->strict && !legal) host_err |= 1u << FFB_E_CAP_ABOVE_TDP;
      double fadj = legal ? fb * pow(cap / tdp, inv_k) : fb;
      h_fadj[s * C + c] = fadj;
      h_scale[s * C + c] = fadj / fb;                                          // power_model.py:153
      h_ok[s * C + c] = in_range ? 1.0 : 0.0;
      double* row = h_ctab + (s * C + c) * 4;
      row[0] = fadj / fb; row[1] = cap; row[2] = py_max(0.0, cap - sp[FFB_S_P_STATIC]); row[3] = in_range ? 1.0 : 0.0;   // power_model.py:157
    }
    const double al = sp[FFB_S_SM_ALPHA], be = sp[FFB_S_SM_BETA], de = sp[FFB_S_SM_DELTA];
    h_psm[s * psm_n + 0] = de;                                                 // power_model.py:74-75
    for (int n = 1; n < psm_n; ++n) h_psm[s * psm_n + n] = al * pow((double)n, be) + de;
  }
  for (int64_t j = 0; j < J; ++j) {
    const int32_t bx = h_shape[4 * j], by = h_shape[4 * j + 1];
    if (bx < 1 || by < 1 || h_shape[4 * j + 2] < 1)
      return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "shape %lld: block dims must be >= 1", (long long)j);
    h_log[j] = fabs(log((double)bx / (double)by));                             // power_model.py:61
  }
  if (!(ctx->tables_shadow_dev == ctx->d_tables.p && ctx->tables_shadow_stream == (void*)stream && ctx->tables_shadow.size() == bytes &&
        memcmp(ctx->tables_shadow.data(), scratch.data(), bytes) == 0)) {
    rc = ffb_stage_reserve(ctx, bytes);
    if (rc) return rc;
    memcpy(ctx->h_stage, scratch.data(), bytes);
    FFB_CUDA(ctx, cudaMemcpyAsync(ctx->d_tables.p, ctx->h_stage, bytes, cudaMemcpyHostToDevice, stream));
    FFB_CUDA(ctx, cudaEventRecord(ctx->stage_free, stream));
    ctx->stage_busy = true;
    ctx->tables_shadow.swap(scratch);
    ctx->tables_shadow_dev = ctx->d_tables.p;
    ctx->tables_shadow_stream = (void*)stream;
  }
  Tables tb;
  double* d = (double*)ctx->d_tables.p;
  tb.spec = d;
  tb.sd = tb.spec + n_spec;
  tb.cap_tab = tb.sd + n_sd;
  tb.shape_log = tb.cap_tab + 4 * n_sc;
  tb.cap = tb.shape_log + n_log;
  tb.cap_scale = tb.cap + n_cap;
  tb.cap_fadj = tb.cap_scale + n_sc;
  tb.cap_ok = tb.cap_fadj + n_sc;
  tb.psm = tb.cap_ok + n_sc;
  tb.shape = (const int32_t*)(tb.psm + n_psm);
  tb.psm_n = psm_n;

  rc = ffb_reserve(ctx, &ctx->d_kstab, (size_t)K * S * kKsWidth * sizeof(double));
  if (rc) return rc;
  {
    const int64_t n = K * S;
    const unsigned grid = (unsigned)((n + 255) / 256);
    FFB_LAUNCH(predict_prepare_kernel, grid, 256, 0, stream, g->d_feat, g->d_res, tb, K, (int)S,
               (double*)ctx->d_kstab.p, g->d_status);
    rc = ffb_check_launch(ctx, "predict_prepare_kernel");
    if (rc) return rc;
  }
  GridArgs a;
  a.feat = g->d_feat; a.res = g->d_res; a.kstab = (const double*)ctx->d_kstab.p; a.tb = tb;
  a.n_units = K * S * J; a.n_specs = (int)S; a.n_shapes = (int)J; a.n_caps = (int)C;
  a.t = g->d_t; a.e = g->d_e; a.pdyn = g->d_pdyn; a.flags = g->d_flags; a.occ = g->d_occ;
  a.detail = g->d_detail; a.status = g->d_status; a.strict = g->strict;
  // the [units, caps] staging tile holds the whole cap axis when it fits 200 KB (47 caps, 32 with p_dyn);
  // longer cap lists are walked in passes of that many caps
  const size_t per_cap = (size_t)kUnitsPerCta * (2 * sizeof(double) + (g->d_pdyn ? sizeof(double) : 0) + 1);
  int64_t cap_tile = (int64_t)((200 * 1024) / per_cap);
  if (cap_tile > C) cap_tile = C;
  a.cap_tile = (int)cap_tile;
  const size_t smem = per_cap * (size_t)cap_tile;
  const int64_t n_cta = (a.n_units + kUnitsPerCta - 1) / kUnitsPerCta;
  if (n_cta > 0x7fffffffLL) return ffb_fail(ctx, FFB_E_CAPACITY, "ffb_predict_grid: grid too large for one launch");
  const bool lean = !g->d_detail && !g->d_pdyn && !g->d_flags && !g->d_occ && !g->strict && !g->d_status && g->d_t && g->d_e;
  if (g->d_detail) {
    FFB_CUDA(ctx, cudaFuncSetAttribute(predict_grid_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FFB_LAUNCH((predict_grid_kernel<true, false>), (unsigned)n_cta, kUnitsPerCta, smem, stream, a);
  } else if (lean) {
    FFB_CUDA(ctx, cudaFuncSetAttribute(predict_grid_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FFB_LAUNCH((predict_grid_kernel<false, true>), (unsigned)n_cta, kUnitsPerCta, smem, stream, a);
  } else {
    FFB_CUDA(ctx, cudaFuncSetAttribute(predict_grid_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FFB_LAUNCH((predict_grid_kernel<false, false>), (unsigned)n_cta, kUnitsPerCta, smem, stream, a);
  }
  rc = ffb_check_launch(ctx, "predict_grid_kernel");
  if (rc) return rc;
  if (host_err) {
    // spec-level reference exceptions (ZeroDelay, ZeroCycles, CapAboveTdp) are known on the host
    for (int code = 1; code < 32; ++code)
      if (host_err & (1u << code)) return ffb_fail(ctx, code, "ffb_predict_grid: spec/cap check failed (status %d)", code);
  }
  return FFB_OK;
}

extern "C" int32_t ffb_enumerate_shapes(const double* sp, int64_t shared_dyn, const int32_t* dims,
                                        int64_t n_dims, int32_t* out_xy, int64_t cap_shapes,
                                        int64_t* n_out) {
  if (!sp || !dims || !n_out || n_dims < 0) return FFB_E_BAD_ARGUMENT;
  const int64_t max_threads = (int64_t)sp[FFB_S_MAX_THREADS], max_warps = (int64_t)sp[FFB_S_MAX_WARPS],
                max_shared = (int64_t)sp[FFB_S_MAX_SHARED];
  struct Sh { int64_t threads; int32_t bx, by; };
  std::vector<Sh> v;
  for (int64_t i = 0; i < n_dims; ++i)
    for (int64_t j = 0; j < n_dims; ++j) {
      const int64_t bx = dims[i], by = dims[j], threads = bx * by;
      if (threads < 32 || threads > max_threads || threads % 32) continue;      // explorer.py:79-82
      if (threads / 32 > max_warps) continue;                                   // :84,87
      if (shared_dyn > 0 && shared_dyn > max_shared) continue;                  // :85-88
      v.push_back({threads, (int32_t)bx, (int32_t)by});
    }
  // canonical order (threads, bx, by); duplicates in dims stay duplicated like the reference
  std::stable_sort(v.begin(), v.end(), [](const Sh& a, const Sh& b) {
    if (a.threads != b.threads) return a.threads < b.threads;
    if (a.bx != b.bx) return a.bx < b.bx;
    return a.by < b.by;
  });
  *n_out = (int64_t)v.size();
  if (out_xy)
    for (int64_t i = 0; i < (int64_t)v.size() && i < cap_shapes; ++i) {
      out_xy[2 * i] = v[i].bx;
      out_xy[2 * i + 1] = v[i].by;
    }
  return FFB_OK;
}

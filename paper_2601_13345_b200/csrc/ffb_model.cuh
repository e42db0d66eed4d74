// The fp64 model of one (kernel, spec, shape) unit and of one cap, shared by the grid kernel
// (ffb_predict.cu) and the fused explore kernel (ffb_explore.cu) so that both evaluate the SAME
// sequence of IEEE binary64 operations.  Every translation unit that includes this header is
// compiled with -fmad=false (paper_2601_13345_b200/build.py, PER_FILE).
//
// Reference arithmetic restated (never copied): features.py:55-59,96-114, time_model.py:33-129,
// power_model.py:31-170, explorer.py:76-92,105-108.
#pragma once
#include "ffb_common.cuh"

#include <math.h>

namespace ffbm {

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
  // shape classes (host-built): shape j -> class A row (threads, regs) | class B row (min(block_x, 32)) << 16
  const int32_t* shape_cls;   // [J]
  const int32_t* a_rep;       // [n_a, 2] {threads, regs}
  const int32_t* b_rep;       // [n_b]    block_x clipped to 32
  int n_a, n_b;
};

// ---- per (kernel, spec) hoisting: time_model.py:47-64 (_issue_window), :40-44 (cwp),
// features.py:108,111-113, power_model.py:44-46,74-76,86 ----
FFB_D uint32_t eval_kernel_spec(const double* f, int64_t shared_dyn, int64_t total_blocks, const double* sp, const double* sd,
                                const double* psm_row, double* o) {
  uint32_t err = 0;
  const int64_t shared = (int64_t)f[FFB_F_STATIC_SHARED] + shared_dyn;       // features.py:111
  if (total_blocks <= 0) err |= 1u << FFB_E_EMPTY_GRID;                     // time_model.py:75
  double shared_limit = INFINITY;
  if (shared > 0) shared_limit = sp[FFB_S_MAX_SHARED] / (double)shared;       // features.py:113
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
  o[KS_SHARED_LIMIT] = shared_limit;
  o[KS_DENOM_COMP] = (cwp * sp[FFB_S_IPC]) * sp[FFB_S_F_BASE];                // time_model.py:116
  o[KS_CI] = ci;
  o[KS_P_SM] = psm_row[active];                                               // power_model.py:74-76
  o[KS_N_COMP] = n_comp;
  o[KS_CWP] = cwp;
  o[KS_ACTIVE] = (double)active;
  o[KS_ERR] = (double)err;
  return err;
}

// ---- one (kernel, spec, shape) unit: everything that does not depend on the power cap ----
struct Unit {
  double t_exec, p_pre, p_static, e_over, bps;
  bool valid;
  uint32_t err;
  // breakdown (filled always; the optimiser drops what a caller does not read)
  double mwp, bw_eff, t_mem, t_comp, t_sync, p_units, p_shape, p_mem, p_sm, ci, eta, waves;
  int64_t warps;
};

FFB_D void eval_unit(const double* f, const double* sp, const double* sd, const double* kr, const int32_t* sh, double shape_log,
                     int64_t shared_dyn, int64_t total_blocks, int strict, Unit& u) {
  const int64_t bx = sh[0], by = sh[1], bz = sh[2], regs = sh[3];
  uint32_t err = (uint32_t)kr[KS_ERR] | (uint32_t)sd[SD_ERR];

  // ---- K2: integer occupancy / validity (explorer.py:76-88, features.py:96-114) ----
  const int64_t threads = bx * by * bz;
  const int64_t max_threads = (int64_t)sp[FFB_S_MAX_THREADS];
  const int64_t max_warps = (int64_t)sp[FFB_S_MAX_WARPS];
  const bool ovr = f[FFB_F_OVR] != 0.0;
  const bool shape_ok = ovr || (threads >= 32 && threads <= max_threads && (threads % 32) == 0);
  if (!shape_ok) err |= (strict ? 1u << FFB_E_INVALID_CONFIG : 0u);
  const int64_t warps = ovr ? (int64_t)f[FFB_F_OVR_WARPS] : (shape_ok ? threads / 32 : 1);
  bool fits = warps <= max_warps;                                   // max_warps/warps >= 1.0
  if (shared_dyn > 0) fits = fits && shared_dyn <= (int64_t)sp[FFB_S_MAX_SHARED];
  const double wf = (double)warps;
  double bps = sp[FFB_S_MAX_WARPS] / wf;                            // features.py:112
  bps = py_min(bps, kr[KS_SHARED_LIMIT]);                           // features.py:114
  const double regs_per_sm = sp[FFB_S_REGS_PER_SM];
  if (regs_per_sm > 0.0 && regs > 0) {                              // extension: oracle.occupancy_ext
    const double reg_limit = regs_per_sm / (double)(regs * threads);
    bps = py_min(bps, reg_limit);
    fits = fits && reg_limit >= 1.0;
  }
  if (ovr) bps = f[FFB_F_OVR_BPS];
  u.valid = (strict || ovr) ? shape_ok : (shape_ok && fits);
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
  const double t_exec = ((sp[FFB_S_W_MEM] * t_mem + sp[FFB_S_W_COMP] * t_comp) +
                         sp[FFB_S_W_SYNC] * t_sync) + sp[FFB_S_T_BASE];

  // ---- power, cap-independent part (power_model.py:124-150) ----
  const double wps = py_min(wf * bps, (double)max_warps);
  double p_units = 0.0;
  const uint32_t skip = (uint32_t)sd[SD_SKIPMASK];
#pragma unroll
  for (int x = 0; x < 5; ++x) {
    if (skip & (1u << x)) continue;
    const double cnt = (x == 4) ? f[FFB_F_N_MEM] : f[FFB_F_FP32 + x];
    const double rate = (cnt * wps) / sd[SD_RATIO0 + x];
    p_units = p_units + sp[FFB_S_BETA0 + x] * rate;
  }
  const double ci = kr[KS_CI];
  double p_shape = sp[FFB_S_P_BASE_SHAPE];
  if (!isinf(ci)) {
    const double penalty = (sp[FFB_S_KAPPA] * shape_log) / (1.0 + ci);
    p_shape = sp[FFB_S_P_BASE_SHAPE] * (1.0 + penalty);
  }
  const double p_mem = sp[FFB_S_P_MEM_BASE] * (1.0 + sp[FFB_S_LAMBDA] * (1.0 - eta));
  const double p_sm = kr[KS_P_SM];
  double p_pre = ((p_units + p_shape) + p_mem) + p_sm;
  const double t_seen = (ovr && f[FFB_F_OVR_TEXEC] == f[FFB_F_OVR_TEXEC]) ? f[FFB_F_OVR_TEXEC] : t_exec;
  if (t_seen < sp[FFB_S_TAU_SHORT]) p_pre = p_pre * sp[FFB_S_TRANSIENT_R];      // power_model.py:93-95
  u.t_exec = t_exec; u.p_pre = p_pre; u.p_static = sp[FFB_S_P_STATIC]; u.e_over = sp[FFB_S_E_OVERHEAD]; u.bps = bps;
  u.err = err;
  u.mwp = mwp; u.bw_eff = bw_eff; u.t_mem = t_mem; u.t_comp = t_comp; u.t_sync = t_sync; u.p_units = p_units; u.p_shape = p_shape;
  u.p_mem = p_mem; u.p_sm = p_sm; u.ci = ci; u.eta = eta; u.waves = waves; u.warps = warps;
}

// ---- the same chain, factored by what each part depends on --------------------------------------------
// Of a unit's cap-independent chain only p_shape reads |ln(bx / by)|; occupancy, waves, t_comp, t_sync and
// p_units depend on (threads, regs) alone, eta / bandwidth / p_mem on min(block_x, 32) alone.  The 464 shapes of
// the reference's search space have 32 distinct thread counts and 32 distinct clipped block_x values, so a
// (kernel, spec) group evaluates 32 + 32 class rows (about ten fp64 divides each) and two divides per shape
// instead of ten per shape.  Every expression keeps the operand order of eval_unit: same bits.
// (Rows with override columns - the single-point drop-ins - stay on eval_unit.)
constexpr int kClassAWidth = 8, kClassBWidth = 4;
enum { CA_MB = 0, CA_T_COMP, CA_T_SYNC, CA_P_UNITS, CA_BPS, CA_VALID, CA_WAVES, CA_WARPS };
enum { CB_DEN_MEM = 0, CB_P_MEM, CB_ETA, CB_BW_EFF };

FFB_D void eval_class_a(const double* f, const double* sp, const double* sd, const double* kr, int64_t threads, int64_t regs,
                        int64_t shared_dyn, int64_t total_blocks, double* o) {
  const int64_t max_threads = (int64_t)sp[FFB_S_MAX_THREADS];
  const int64_t max_warps = (int64_t)sp[FFB_S_MAX_WARPS];
  const bool shape_ok = threads >= 32 && threads <= max_threads && (threads % 32) == 0;
  const int64_t warps = shape_ok ? threads / 32 : 1;
  bool fits = warps <= max_warps;
  if (shared_dyn > 0) fits = fits && shared_dyn <= (int64_t)sp[FFB_S_MAX_SHARED];
  const double wf = (double)warps;
  double bps = sp[FFB_S_MAX_WARPS] / wf;                            // features.py:112
  bps = py_min(bps, kr[KS_SHARED_LIMIT]);                           // features.py:114
  const double regs_per_sm = sp[FFB_S_REGS_PER_SM];
  if (regs_per_sm > 0.0 && regs > 0) {                              // extension: oracle.occupancy_ext
    const double reg_limit = regs_per_sm / (double)(regs * threads);
    bps = py_min(bps, reg_limit);
    fits = fits && reg_limit >= 1.0;
  }
  const double resident = py_min(bps * wf, (double)max_warps);      // time_model.py:78
  const double lanes = (sp[FFB_S_SM_COUNT] * resident) * 32.0;
  const double tthreads = (double)(total_blocks * warps) * 32.0;
  const double waves = py_max(1.0, tthreads / lanes);
  const double nc = kr[KS_N_COMP] * waves;
  const double wps = py_min(wf * bps, (double)max_warps);           // power_model.py:124
  double p_units = 0.0;
  const uint32_t skip = (uint32_t)sd[SD_SKIPMASK];
#pragma unroll
  for (int x = 0; x < 5; ++x) {
    if (skip & (1u << x)) continue;
    const double cnt = (x == 4) ? f[FFB_F_N_MEM] : f[FFB_F_FP32 + x];
    const double rate = (cnt * wps) / sd[SD_RATIO0 + x];
    p_units = p_units + sp[FFB_S_BETA0 + x] * rate;
  }
  o[CA_MB] = f[FFB_F_MEM_BYTES] * waves;
  o[CA_T_COMP] = (nc > 0.0) ? nc / kr[KS_DENOM_COMP] : 0.0;
  o[CA_T_SYNC] = (f[FFB_F_N_SYNC] * waves) * sp[FFB_S_T_BARRIER];
  o[CA_P_UNITS] = p_units;
  o[CA_BPS] = bps;
  o[CA_VALID] = (shape_ok && fits) ? 1.0 : 0.0;
  o[CA_WAVES] = waves;
  o[CA_WARPS] = wf;
}
FFB_D void eval_class_b(const double* f, const double* sp, const double* sd, int64_t bx, double* o) {
  const double eta = py_min(1.0, (double)bx / 32.0) * f[FFB_F_ALIGNED];            // features.py:59
  const double bw_eff = sp[FFB_S_BW_MAX] * py_max(eta, sd[SD_FLOOR]);
  o[CB_DEN_MEM] = sd[SD_MWP] * bw_eff;
  o[CB_P_MEM] = sp[FFB_S_P_MEM_BASE] * (1.0 + sp[FFB_S_LAMBDA] * (1.0 - eta));
  o[CB_ETA] = eta;
  o[CB_BW_EFF] = bw_eff;
}
// one shape from its two class rows: t_exec and the cap-independent dynamic power
FFB_D void eval_shape(const double* sp, const double* kr, const double* ca, const double* cb, double shape_log, double* t_exec_out, double* p_pre_out) {
  const double mb = ca[CA_MB];
  const double t_mem = (mb > 0.0) ? mb / cb[CB_DEN_MEM] : 0.0;
  const double t_exec = ((sp[FFB_S_W_MEM] * t_mem + sp[FFB_S_W_COMP] * ca[CA_T_COMP]) + sp[FFB_S_W_SYNC] * ca[CA_T_SYNC]) + sp[FFB_S_T_BASE];
  const double ci = kr[KS_CI];
  double p_shape = sp[FFB_S_P_BASE_SHAPE];
  if (!isinf(ci)) {
    const double penalty = (sp[FFB_S_KAPPA] * shape_log) / (1.0 + ci);
    p_shape = sp[FFB_S_P_BASE_SHAPE] * (1.0 + penalty);
  }
  double p_pre = ((ca[CA_P_UNITS] + p_shape) + cb[CB_P_MEM]) + kr[KS_P_SM];
  if (t_exec < sp[FFB_S_TAU_SHORT]) p_pre = p_pre * sp[FFB_S_TRANSIENT_R];         // power_model.py:93-95
  *t_exec_out = t_exec; *p_pre_out = p_pre;
}

// ---- one cap of a unit (power_model.py:152-158, explorer.py:107); row = {scale, cap, max(0, cap - p_static), ok} ----
FFB_D double eval_cap(double t_exec, double p_pre, double p_static, double e_over, double scale, double cap, double room,
                      double* p_dyn_out, bool* limited_out) {
  double p_dyn = p_pre * scale;
  const bool limited = p_dyn + p_static > cap;
  if (limited) p_dyn = room;                                  // max(0.0, cap - p_static), tabulated
  *p_dyn_out = p_dyn; *limited_out = limited;
  return t_exec * (p_dyn + p_static) + e_over;
}

}  // namespace ffbm

// Host side (ffb_predict.cu): validates the specs, takes libm log / pow, uploads the tables (cached per context).
struct FfbTableDims { int64_t S, J, C; };
int32_t ffb_build_tables(FfbContext* ctx, const double* h_spec_in, const int32_t* h_shape_in, const double* h_cap_in,
                         FfbTableDims dims, int strict, cudaStream_t stream, ffbm::Tables* tb, uint32_t* host_err);

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
#include "ffb_model.cuh"

#include <string.h>
#include <algorithm>
#include <utility>
#include <vector>

using namespace ffbm;

namespace {

constexpr int kUnitsPerCta = 256;

// ---- per (kernel, spec) hoisting --------------------------------------------------------
__global__ void __launch_bounds__(256)
predict_prepare_kernel(const double* __restrict__ feat, const int64_t* __restrict__ res, Tables tb,
                       int64_t n_kernels, int n_specs, double* __restrict__ kstab,
                       uint32_t* __restrict__ status) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_kernels * n_specs) return;
  int64_t k = i / n_specs;
  int s = (int)(i - k * n_specs);
  const uint32_t err = eval_kernel_spec(feat + k * FFB_FEAT_WIDTH, res[2 * k + 0], res[2 * k + 1], tb.spec + (size_t)s * FFB_SPEC_WIDTH,
                                        tb.sd + (size_t)s * kSdWidth, tb.psm + (size_t)s * tb.psm_n, kstab + i * kKsWidth);
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
    Unit u;
    eval_unit(a.feat + k * FFB_FEAT_WIDTH, a.tb.spec + (size_t)s * FFB_SPEC_WIDTH, a.tb.sd + (size_t)s * kSdWidth,
              a.kstab + ks * kKsWidth, a.tb.shape + 4 * j, a.tb.shape_log[j], a.res[2 * k + 0], a.res[2 * k + 1], a.strict, u);
    unit_valid = u.valid; t_exec = u.t_exec; p_pre = u.p_pre; p_static = u.p_static; e_over = u.e_over;
    const uint32_t err = u.err;
    const double bps = u.bps;
    if (kDetail) {
      d_mwp = u.mwp; d_cwp = a.kstab[ks * kKsWidth + KS_CWP]; d_bw = u.bw_eff; d_tm = u.t_mem; d_tc = u.t_comp; d_ts = u.t_sync;
      d_pu = u.p_units; d_ps = u.p_shape; d_pm = u.p_mem; d_psm = u.p_sm; d_ci = u.ci; d_act = a.kstab[ks * kKsWidth + KS_ACTIVE];
      d_warps = (double)u.warps; d_bps = u.bps; d_eta = u.eta; d_waves = u.waves;
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
        double p_dyn;
        bool limited;
        const double e_pred = eval_cap(t_exec, p_pre, p_static, e_over, sc_cap.x, sc_cap.y, room_ok.x, &p_dyn, &limited);
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

// The streaming configuration (t / e only) with the factored model of ffb_model.cuh: one CTA per (kernel, spec)
// group evaluates the group's class rows once - (threads, regs) classes and clipped-block_x classes - and then
// walks the group's shapes: two fp64 divides per shape instead of ten (round 1: 780 thread instructions per unit,
// 44% of the copy peak).  Same staging tile and coalesced write-out as predict_grid_kernel, in CTAs of 128 shapes
// (eight resident per SM: the stores of one overlap the fp64 chains of the others); the cap table of the group's
// spec sits in shared memory.  Measured and rejected (r2x): no staging tile - every lane owns elements L, L + 32, ...
// of the warp's 32 x C outputs and fetches (t_exec, p_pre) of the element's shape with shuffles - 57% more warp
// instructions (shuffles, divergent cap-table reads, 8-byte stores), 0.49 ms vs 0.44 ms.
constexpr int kGridMaxClassA = 512;
constexpr int kClsSpan = 512;                  // shapes per CTA (a multiple of kClsUnits)
constexpr int kClsUnits = 128;                 // threads per CTA = shapes per pass (four warps of 32 shapes)
__global__ void __launch_bounds__(kClsUnits, 8)
predict_grid_classes_kernel(GridArgs a) {
  FFB_DYN_SMEM(smem_raw);
  const int C = a.n_caps, J = a.n_shapes;
  double* s_t = reinterpret_cast<double*>(smem_raw);            // [units][C] staging tile
  double* s_e = s_t + (size_t)kClsUnits * C;
  double* s_cap = s_e + (size_t)kClsUnits * C;                  // [C][4] = {scale, cap, room, ok} of this spec
  double* s_ca = s_cap + (size_t)C * 4;                         // [n_a][kClassAWidth]
  double* s_cb = s_ca + (size_t)a.tb.n_a * kClassAWidth;        // [n_b][kClassBWidth]
  const int64_t g = blockIdx.x;
  const int64_t k = g / a.n_specs;
  const int s = (int)(g - k * a.n_specs);
  const double* f = a.feat + k * FFB_FEAT_WIDTH;
  const double* sp = a.tb.spec + (size_t)s * FFB_SPEC_WIDTH;
  const double* sd = a.tb.sd + (size_t)s * kSdWidth;
  const double* kr = a.kstab + g * kKsWidth;
  const int64_t shared_dyn = a.res[2 * k + 0], total_blocks = a.res[2 * k + 1];
  const bool classes = f[FFB_F_OVR] == 0.0;
  if (classes) {
    for (int i = threadIdx.x; i < a.tb.n_a + a.tb.n_b; i += kClsUnits) {
      if (i < a.tb.n_a) eval_class_a(f, sp, sd, kr, a.tb.a_rep[2 * i], a.tb.a_rep[2 * i + 1], shared_dyn, total_blocks, s_ca + (size_t)i * kClassAWidth);
      else eval_class_b(f, sp, sd, a.tb.b_rep[i - a.tb.n_a], s_cb + (size_t)(i - a.tb.n_a) * kClassBWidth);
    }
  }
  for (int i = threadIdx.x; i < C * 4; i += kClsUnits) s_cap[i] = a.tb.cap_tab[(size_t)s * C * 4 + i];
  __syncthreads();
  const double p_static = sp[FFB_S_P_STATIC], e_over = sp[FFB_S_E_OVERHEAD];
  const double2* s_cap2 = reinterpret_cast<const double2*>(s_cap);
  // blockIdx.y: this CTA's run of kClsSpan shapes (large shape tables are split so that the grid has many more
  // CTAs than the GPU holds at once: no tail of half-empty waves)
  const int j_begin = (int)blockIdx.y * kClsSpan, j_end = j_begin + kClsSpan < J ? j_begin + kClsSpan : J;
  for (int j0 = j_begin; j0 < j_end; j0 += kClsUnits) {
    const int j = j0 + threadIdx.x;
    const int n_live = j_end - j0 < kClsUnits ? j_end - j0 : kClsUnits;
    if (j < j_end) {
      double t_exec, p_pre;
      bool valid;
      if (classes) {
        const int32_t cls = a.tb.shape_cls[j];
        const double* ca = s_ca + (size_t)(cls & 0xffff) * kClassAWidth;
        eval_shape(sp, kr, ca, s_cb + (size_t)(cls >> 16) * kClassBWidth, a.tb.shape_log[j], &t_exec, &p_pre);
        valid = ca[CA_VALID] != 0.0;
      } else {
        Unit u;
        eval_unit(f, sp, sd, kr, a.tb.shape + 4 * j, a.tb.shape_log[j], shared_dyn, total_blocks, 0, u);
        t_exec = u.t_exec; p_pre = u.p_pre; valid = u.valid;
      }
      double* st = s_t + (size_t)threadIdx.x * C;
      double* se = s_e + (size_t)threadIdx.x * C;
#pragma unroll 4
      for (int c = 0; c < C; ++c) {
        const double2 sc_cap = s_cap2[2 * c], room_ok = s_cap2[2 * c + 1];   // same address in every lane: broadcast
        double p_dyn;
        bool limited;
        const double e_pred = eval_cap(t_exec, p_pre, p_static, e_over, sc_cap.x, sc_cap.y, room_ok.x, &p_dyn, &limited);
        const bool ok = valid && room_ok.y != 0.0;
        st[c] = ok ? t_exec : INFINITY;
        se[c] = ok ? e_pred : INFINITY;
      }
    }
    __syncthreads();
    const int total = n_live * C;
    const size_t base = ((size_t)g * J + j0) * C;
    if ((base & 1) == 0) {
      const int pairs = total >> 1;
      double2* gt = reinterpret_cast<double2*>(a.t + base);
      double2* ge = reinterpret_cast<double2*>(a.e + base);
      const double2* st2 = reinterpret_cast<const double2*>(s_t);
      const double2* se2 = reinterpret_cast<const double2*>(s_e);
      for (int i = threadIdx.x; i < pairs; i += kClsUnits) { gt[i] = st2[i]; ge[i] = se2[i]; }
      if ((total & 1) && threadIdx.x == 0) { a.t[base + total - 1] = s_t[total - 1]; a.e[base + total - 1] = s_e[total - 1]; }
    } else {
      for (int i = threadIdx.x; i < total; i += kClsUnits) { a.t[base + i] = s_t[i]; a.e[base + i] = s_e[i]; }
    }
    __syncthreads();
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

int32_t ffb_build_tables(FfbContext* ctx, const double* h_spec_in, const int32_t* h_shape_in, const double* h_cap_in,
                         FfbTableDims dims, int strict, cudaStream_t stream, ffbm::Tables* tb_out, uint32_t* host_err_out) {
  const int64_t S = dims.S, J = dims.J, C = dims.C;
  // ---- host tables (libm here, same as the reference's math.log / ** ) ----
  int psm_n = 1;
  for (int64_t s = 0; s < S; ++s) {
    double sm = h_spec_in[s * FFB_SPEC_WIDTH + FFB_S_SM_COUNT];
    if (!(sm >= 0.0) || sm > 1e6) return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "spec %lld: sm_count out of range", (long long)s);
    if ((int)sm + 1 > psm_n) psm_n = (int)sm + 1;
  }
  const size_t n_spec = (size_t)S * FFB_SPEC_WIDTH, n_sd = (size_t)S * kSdWidth, n_log = (size_t)J,
               n_cap = (size_t)C, n_sc = (size_t)S * C, n_psm = (size_t)S * psm_n;
  const size_t n_dbl = n_spec + n_sd + n_log + n_cap + 7 * n_sc + n_psm;
  const size_t bytes = n_dbl * sizeof(double) + (size_t)J * 8 * sizeof(int32_t);       // shapes [J,4] + class index [J] + class rows [<= 3J]
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
  memcpy(h_spec, h_spec_in, n_spec * sizeof(double));
  memcpy(h_cap, h_cap_in, n_cap * sizeof(double));
  memcpy(h_shape, h_shape_in, (size_t)J * 4 * sizeof(int32_t));
  uint32_t host_err = 0;
  for (int64_t s = 0; s < S; ++s) {
    const double* sp = h_spec + s * FFB_SPEC_WIDTH;
    validate_spec_row(ctx, sp, (int)s, strict, h_sd + s * kSdWidth);
    host_err |= (uint32_t)h_sd[s * kSdWidth + SD_ERR];
    const double tdp = sp[FFB_S_P_TDP], fb = sp[FFB_S_F_BASE];
    const double inv_k = 1.0 / (double)(int64_t)sp[FFB_S_DVFS_K];          // power_model.py:106
    for (int64_t c = 0; c < C; ++c) {
      const double cap = h_cap[c];
      const bool in_range = (sp[FFB_S_P_CAP_MIN] <= cap) && (cap <= tdp);      // explorer.py:90
      const bool legal = cap > 0.0 && tdp > 0.0 && cap <= tdp;                 // power_model.py:100-105
      if (strict && !legal) host_err |= 1u << FFB_E_CAP_ABOVE_TDP;
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
  // shape classes of the factored model (ffb_model.cuh): unique (threads, regs) and unique min(block_x, 32)
  int32_t* h_cls = h_shape + (size_t)J * 4;
  int32_t* h_arep = h_cls + J;
  int32_t* h_brep = h_arep + 2 * (size_t)J;
  memset(h_cls, 0, (size_t)J * 4 * sizeof(int32_t));
  int n_a = 0, n_b = 0;
  {
    std::vector<std::pair<std::pair<int64_t, int32_t>, int>> amap;             // small: linear search over the classes found so far
    int bmap[33];
    for (int i = 0; i < 33; ++i) bmap[i] = -1;
    for (int64_t j = 0; j < J; ++j) {
      const int64_t threads = (int64_t)h_shape[4 * j] * h_shape[4 * j + 1] * h_shape[4 * j + 2];
      const int32_t regs = h_shape[4 * j + 3];
      int ia = -1;
      for (auto& kv : amap) if (kv.first.first == threads && kv.first.second == regs) { ia = kv.second; break; }
      if (ia < 0) {
        ia = n_a++;
        amap.push_back({{threads, regs}, ia});
        h_arep[2 * ia] = (int32_t)(threads > 0x7fffffff ? 0x7fffffff : threads); h_arep[2 * ia + 1] = regs;
      }
      const int bxc = h_shape[4 * j] < 32 ? h_shape[4 * j] : 32;
      if (bmap[bxc] < 0) { bmap[bxc] = n_b; h_brep[n_b++] = bxc; }
      h_cls[j] = ia | (bmap[bxc] << 16);
      if (n_a > 4096) break;                                              // no use as classes: callers evaluate every shape
    }
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
  tb.shape_cls = tb.shape + (size_t)J * 4;
  tb.a_rep = tb.shape_cls + J;
  tb.b_rep = tb.a_rep + 2 * (size_t)J;
  tb.n_a = n_a <= 4096 ? n_a : 0; tb.n_b = n_b;           // n_a == 0: no class tables (callers fall back to eval_unit)
  *tb_out = tb;
  *host_err_out = host_err;
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
  Tables tb;
  uint32_t host_err = 0;
  int32_t rc = ffb_build_tables(ctx, g->h_spec, g->h_shape, g->h_cap, FfbTableDims{S, J, C}, g->strict, stream, &tb, &host_err);
  if (rc) return rc;

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
  } else if (lean && a.t && a.e && tb.n_a > 0 && tb.n_a <= kGridMaxClassA && K * S <= 0x7fffffffLL && (J + kClsSpan - 1) / kClsSpan <= 65535 &&
             ((size_t)kClsUnits * C * 2 + (size_t)C * 4 + (size_t)tb.n_a * kClassAWidth + (size_t)tb.n_b * kClassBWidth) * sizeof(double) <= 96 * 1024) {
    const size_t smem_c = ((size_t)kClsUnits * C * 2 + (size_t)C * 4 + (size_t)tb.n_a * kClassAWidth + (size_t)tb.n_b * kClassBWidth) * sizeof(double);
    FFB_CUDA(ctx, cudaFuncSetAttribute(predict_grid_classes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_c));
    FFB_LAUNCH(predict_grid_classes_kernel, dim3((unsigned)(K * S), (unsigned)((J + kClsSpan - 1) / kClsSpan)), kClsUnits, smem_c, stream, a);
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

/* libffb — C-ABI of the B200-native FlipFlop analysis path.
 *
 * The reference (pkg/src/ptxwatt, pure Python) has no FFI of its own; its boundary is the
 * Python API re-exported at pkg/src/ptxwatt/__init__.py:4-55.  Each entry point below
 * names the reference function(s) it stands in for.  The Python shim in
 * paper_2601_13345_b200/ binds these with ctypes (see INTEGRATION.md for the stub a
 * maintainer of the reference would add).
 *
 * Conventions
 *  - every function returns an int32 status (FFB_OK or FFB_E_*); FFB_E_* values map 1:1
 *    onto the reference's exception classes (pkg/src/ptxwatt/errors.py), see
 *    paper_2601_13345_b200/errors.py:STATUS_TABLE;
 *  - pointers named d_* are DEVICE pointers owned by the caller, h_* are HOST pointers;
 *    nothing is allocated that the caller must free except the context;
 *  - every launch goes to the cudaStream_t passed in (void* here so the header is plain C);
 *    functions do not synchronise unless documented ("syncs");
 *  - all functions are reentrant across contexts; one context serves one device and is
 *    not thread-safe by itself.
 */
#ifndef FFB_H_
#define FFB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFB_ABI_VERSION 1

/* ---- status codes ------------------------------------------------------------------ */
enum {
  FFB_OK = 0,
  FFB_E_MALFORMED_PTX = 1,   /* errors.py MalformedPtx  (ptx.py:175,184,273,275,281)     */
  FFB_E_NO_KERNEL = 2,       /* errors.py NoKernelFound (ptx.py:186-187)                 */
  FFB_E_INVALID_CONFIG = 3,  /* errors.py InvalidConfig (features.py:98,102)             */
  FFB_E_NO_FEASIBLE = 4,     /* errors.py NoFeasibleConfig (explorer.py:146,207)         */
  FFB_E_EMPTY_GRID = 5,      /* errors.py EmptyGrid (time_model.py:76, power_model.py:85)*/
  FFB_E_ZERO_DELAY = 6,      /* errors.py ZeroDelay (time_model.py:36)                   */
  FFB_E_ZERO_COMPUTE = 7,    /* errors.py ZeroComputeCycles (time_model.py:43)           */
  FFB_E_ZERO_BANDWIDTH = 8,  /* errors.py ZeroBandwidth (time_model.py:110)              */
  FFB_E_ZERO_CYCLES = 9,     /* errors.py ZeroCycles (power_model.py:36)                 */
  FFB_E_CAP_ABOVE_TDP = 10,  /* errors.py CapAboveTdp (power_model.py:100-105)           */
  FFB_E_CAPACITY = 11,       /* a documented device capacity was exceeded                */
  FFB_E_CUDA = 12,           /* CUDA runtime failure; see ffb_last_error                 */
  FFB_E_BAD_ARGUMENT = 13
};

/* ---- opcode classes / state spaces (ptx.py:15-16) ------------------------------------ */
enum { FFB_CLS_MEMLOAD = 0, FFB_CLS_MEMSTORE, FFB_CLS_FP32, FFB_CLS_INT, FFB_CLS_SFU,
       FFB_CLS_ALU, FFB_CLS_SYNC, FFB_CLS_BRANCH, FFB_CLS_OTHER, FFB_N_CLASSES };
enum { FFB_SP_GLOBAL = 0, FFB_SP_SHARED, FFB_SP_LOCAL, FFB_SP_PARAM, FFB_SP_REG, FFB_SP_NONE };

/* ---- per-kernel feature row: features.py:62-81 + alignment.py:128-147 ---------------- */
enum { FFB_F_N_MEM = 0, FFB_F_MEM_BYTES, FFB_F_FP32, FFB_F_INT, FFB_F_SFU, FFB_F_ALU,
       FFB_F_N_SYNC, FFB_F_ALIGNED, FFB_F_STATIC_SHARED, FFB_F_REGS_DECLARED,
       FFB_F_N_INSTR, FFB_F_RESERVED,
       /* Override columns, used by the single-point drop-ins (predict_energy, execution_time,
        * dynamic_power) whose KernelFeatures argument carries its own occupancy numbers:
        * when FFB_F_OVR != 0 the kernel takes warps / blocks_per_sm / eta / n_comp from the
        * row instead of deriving them, and FFB_F_OVR_TEXEC (if not NaN) replaces t_exec in the
        * transient test of power_model.py:93-95. */
       FFB_F_OVR, FFB_F_OVR_WARPS, FFB_F_OVR_BPS, FFB_F_OVR_ETA, FFB_F_OVR_NCOMP, FFB_F_OVR_TEXEC,
       FFB_FEAT_WIDTH };

/* ---- one GPU spec + calibration, flattened (calibration.py:43-83) -------------------- */
enum FfbSpecCol {
  FFB_S_SM_COUNT = 0, FFB_S_MAX_WARPS, FFB_S_MAX_SHARED, FFB_S_MAX_THREADS,
  FFB_S_BW_MAX, FFB_S_IPC, FFB_S_F_BASE, FFB_S_P_TDP, FFB_S_P_STATIC, FFB_S_P_CAP_MIN,
  FFB_S_DVFS_K, FFB_S_TAU_SHORT, FFB_S_DEP_DELAY, FFB_S_T_BARRIER,
  FFB_S_EXEC0, FFB_S_ISSUE0 = FFB_S_EXEC0 + 5, FFB_S_BETA0 = FFB_S_ISSUE0 + 5, /* FP32,INT,SFU,ALU,Mem */
  FFB_S_L_COAL = FFB_S_BETA0 + 5, FFB_S_L_UNCOAL, FFB_S_SM_ALPHA, FFB_S_SM_BETA, FFB_S_SM_DELTA,
  FFB_S_TRANSIENT_R, FFB_S_KAPPA, FFB_S_LAMBDA, FFB_S_P_BASE_SHAPE, FFB_S_P_MEM_BASE,
  FFB_S_W_MEM, FFB_S_W_COMP, FFB_S_W_SYNC, FFB_S_T_BASE, FFB_S_E_OVERHEAD,
  FFB_S_REGS_PER_SM,   /* extension: 0 = no register limit (reference behaviour) */
  FFB_SPEC_USED,
  FFB_SPEC_WIDTH = 48
};

/* ---- detail row written by ffb_predict_grid when d_detail != NULL --------------------
 * time_model.py:20-30 TimeBreakdown, power_model.py:16-28 PowerBreakdown, plus occupancy. */
enum { FFB_D_MWP = 0, FFB_D_CWP, FFB_D_BW_EFF, FFB_D_T_MEM, FFB_D_T_COMP, FFB_D_T_SYNC, FFB_D_T_EXEC,
       FFB_D_P_UNITS, FFB_D_P_SHAPE, FFB_D_P_MEM, FFB_D_P_SM, FFB_D_P_DYN, FFB_D_F_ADJ, FFB_D_CI,
       FFB_D_ACTIVE_SMS, FFB_D_CAP_LIMITED, FFB_D_E_PRED, FFB_D_WARPS, FFB_D_BLOCKS_PER_SM,
       FFB_D_ETA, FFB_D_WAVES, FFB_DETAIL_WIDTH };

/* flag bits of d_flags */
enum { FFB_PT_VALID = 1, FFB_PT_CAP_LIMITED = 2 };

typedef struct FfbContext FfbContext;

int32_t ffb_abi_version(void);
/* One context per device.  Allocates small scratch (tables, counters) on `device`. */
int32_t ffb_create(int32_t device, FfbContext** out);
int32_t ffb_destroy(FfbContext* ctx);
/* Text of the last failure on this context (never NULL). */
const char* ffb_last_error(const FfbContext* ctx);
/* Number of kernels this context has launched so far (bench.py's gpu_launches). */
int64_t ffb_launch_count(const FfbContext* ctx);

/* ---- K2 + K3: occupancy filter and fp64 time / power / energy over the grid ----------
 * Stands in for explorer.py:59-94 (generate_valid_configs: the validity mask),
 * features.py:96-114 (occupancy), features.py:55-59 (eta), time_model.py:67-129,
 * power_model.py:109-170 and explorer.py:97-108 (energy identity), evaluated for every
 * point of   kernel k  x  spec s  x  shape j  x  cap c,   output index ((k*S+s)*J+j)*C+c.
 *
 * libm log/pow (power_model.py:61,76,106) are taken on the HOST inside this call with the
 * same libm CPython uses and uploaded as tables, so results are bit-identical to the
 * reference; the device code uses only IEEE +,-,*,/ without FMA contraction.
 * Invalid points (explorer.py:79-91 rules) get t = e = +inf and flag bit FFB_PT_VALID clear.
 */
typedef struct {
  int64_t n_kernels, n_specs, n_shapes, n_caps;
  const double*  d_feat;    /* [K, FFB_FEAT_WIDTH]                                         */
  const int64_t* d_res;     /* [K, 2] {dynamic shared bytes, total blocks}  (launch.py:24) */
  const double*  h_spec;    /* [S, FFB_SPEC_WIDTH]                                         */
  const int32_t* h_shape;   /* [J, 4] {block_x, block_y, block_z, regs_per_thread}         */
  const double*  h_cap;     /* [C] watts                                                   */
  double*  d_t;             /* [K,S,J,C] t_exec, or NULL                                   */
  double*  d_e;             /* [K,S,J,C] e_pred, or NULL                                   */
  double*  d_pdyn;          /* [K,S,J,C] or NULL                                           */
  uint8_t* d_flags;         /* [K,S,J,C] or NULL                                           */
  double*  d_occ;           /* [K,S,J]   blocks_per_sm (features.py:114), or NULL          */
  double*  d_detail;        /* [K,S,J,C,FFB_DETAIL_WIDTH] or NULL                          */
  uint32_t* d_status;       /* [1] OR-ed bit (1<<FFB_E_*) of model errors met, or NULL      */
  int32_t strict;           /* 1: no validity masking, reference exceptions are reported
                                  in d_status (predict_energy / extract_features semantics) */
} FfbGridDesc;
int32_t ffb_predict_grid(FfbContext* ctx, const FfbGridDesc* g, void* stream);

/* Shapes that pass explorer.py:76-88 for one spec and one dynamic-shared size, in the
 * canonical (threads, bx, by) order of explorer.py:55-56,93.  Host-side integer work;
 * writes up to cap_shapes {bx,by} pairs, returns the count in *n_out. */
int32_t ffb_enumerate_shapes(const double* h_spec_row, int64_t shared_dyn,
                             const int32_t* h_dims, int64_t n_dims,
                             int32_t* h_out_xy, int64_t cap_shapes, int64_t* n_out);

/* ---- K4: skyline ----------------------------------------------------------------------
 * explorer.py:122-140 (pareto_front), :209-212 (throughput floor + ordering).
 * A point is dropped iff some point has strictly lower e AND strictly lower t; ties stay.
 *
 * Segmented form: n_groups consecutive groups of group_size points.  For each group:
 *   t_peak = min t;  eligible = t <= t_peak / rho  (rho <= 0 disables the floor);
 *   front of the eligible points, written as in-group indices ordered by
 *   (e, t, tie[idx]) — pass tie = rank of (block_x, block_y, cap) to reproduce
 *   explorer.py:113-119; NULL means the index itself.
 * Dense mode (d_front_off == NULL): d_front_idx [n_groups, cap_front].
 * Compact mode (d_front_off != NULL): each group's run is appended to d_front_idx
 * (cap_front = total entries available) at offset d_front_off[g]; runs of different groups
 * land in launch-dependent order, each run itself is in reference order.
 * d_front_n [n_groups] is always the true front size; when a front (dense) or the total
 * (compact) does not fit, the status word gets bit FFB_E_CAPACITY.  d_tpeak [n_groups] or NULL.
 */
int32_t ffb_skyline_groups(FfbContext* ctx, const double* d_e, const double* d_t,
                           int64_t n_groups, int64_t group_size, const uint32_t* d_tie,
                           double rho, uint32_t* d_front_idx, uint32_t* d_front_n,
                           double* d_tpeak, int64_t cap_front, int64_t* d_front_off,
                           uint32_t* d_status, void* stream);

/* ---- K2 + K3 + K4 fused: fronts only ----------------------------------------------------
 * Stands in for pareto_explore (explorer.py:186-212): generate_valid_configs (:59-94, as the
 * validity mask) -> evaluate_configs (:161-183) -> throughput floor (:209-210) -> pareto_front
 * (:122-140), for every (kernel k, spec s) group at once; group g = k * n_specs + s holds the
 * n_shapes * n_caps candidates of that kernel on that spec, candidate index j * n_caps + c.
 * Same inputs as ffb_predict_grid, same outputs as ffb_skyline_groups with
 * tie = rank of (block_x, block_y, block_z, regs) * n_caps + rank of the cap value - but the
 * [K,S,J,C] grid never exists in HBM: one CTA evaluates a group into shared memory and ranks it
 * there.  Results are identical to ffb_predict_grid + ffb_skyline_groups (tests compare them).
 * d_front_e / d_front_t (optional) receive the (e_pred, t_exec) of every front member, parallel
 * to d_front_idx.  Capacity: a group (n_shapes * n_caps candidates) must fit one CTA's shared
 * memory, at most 32767 candidates (FFB_E_CAPACITY: use the two-call route). */
typedef struct {
  int64_t n_kernels, n_specs, n_shapes, n_caps;
  const double*  d_feat;    /* [K, FFB_FEAT_WIDTH]                                         */
  const int64_t* d_res;     /* [K, 2] {dynamic shared bytes, total blocks}                 */
  const double*  h_spec;    /* [S, FFB_SPEC_WIDTH]                                         */
  const int32_t* h_shape;   /* [J, 4] {block_x, block_y, block_z, regs_per_thread}         */
  const double*  h_cap;     /* [C] watts                                                   */
  double rho;               /* throughput floor, <= 0 disables it                          */
  uint32_t* d_front_idx;    /* dense [K*S, cap_front] or compact [cap_front] (with d_front_off) */
  uint32_t* d_front_n;      /* [K*S]                                                       */
  double*   d_tpeak;        /* [K*S] or NULL                                               */
  int64_t   cap_front;
  int64_t*  d_front_off;    /* [K*S] or NULL (dense)                                       */
  double*   d_front_e;      /* optional, laid out like d_front_idx                         */
  double*   d_front_t;      /* optional                                                    */
  uint32_t* d_status;       /* [1] OR-ed (1 << FFB_E_CAPACITY) when a front does not fit    */
} FfbExploreDesc;
int32_t ffb_explore_groups(FfbContext* ctx, const FfbExploreDesc* d, void* stream);

/* One large candidate set (BASELINE config 5).  Streaming cull against a sentinel
 * staircase, exact pass on the survivors.  Output: global indices (or d_id values when
 * d_id != NULL) of the front in (e, t, id) order.  Syncs (returns the count).
 * d_occ != NULL switches to the 3-objective rule (maximise occupancy as third key):
 * dropped iff some point is strictly better in all three. */
/* Extension without reference semantics (BASELINE config 5, "3-objective (+occupancy)"): with d_occ given a
 * candidate is dropped iff another one has strictly lower e, strictly lower t AND occupancy at least as
 * high; ordering and floor as above.  d_occ == NULL is ffb_skyline_groups.  Capacities: groups of at most
 * 65535 candidates, at most 64 distinct occupancy values per group (FFB_E_CAPACITY otherwise). */
int32_t ffb_skyline_groups3(FfbContext* ctx, const double* d_e, const double* d_t, const double* d_occ,
                            int64_t n_groups, int64_t group_size, const uint32_t* d_tie,
                            double rho, uint32_t* d_front_idx, uint32_t* d_front_n,
                            double* d_tpeak, int64_t cap_front, int64_t* d_front_off,
                            uint32_t* d_status, void* stream);
int32_t ffb_skyline(FfbContext* ctx, const double* d_e, const double* d_t, const double* d_occ,
                    const uint64_t* d_id, int64_t n, double rho, uint64_t* d_front_id,
                    double* d_front_e, double* d_front_t, int64_t cap_front,
                    int64_t* h_front_n, double* h_tpeak, void* stream);

/* ---- K1: byte-lexer, opcode classifier, per-kernel histogram ---------------------------
 * Stands in for ptx.py:139-141 (_strip_comments), :165-187 (_find_kernel), :207-293
 * (parse_ptx statement loop, declarations), :296-313 (_parse_instruction), :99-136
 * (classify_opcode) and :64-76 (access_bytes), applied to every segment of a corpus:
 * segment k is text[seg_off[k] : seg_off[k+1]) and is analysed exactly like one
 * parse_ptx(source) call (first .entry of the segment, or the one named h_kernel_name).
 *
 * Documented device capacities (status FFB_E_CAPACITY, never a silent difference):
 * a statement (its code bytes, on one line or several) must fit one 4 KB tile - `//` comments and
 * module-level lines in front of the kernel body may be of any length; input is ASCII.
 */
typedef struct {
  uint32_t status;          /* FFB_OK or FFB_E_*  (reference exception of parse_ptx)            */
  uint32_t n_instr;         /* len(PtxModule.instructions)                                      */
  uint32_t n_labels;        /* label definitions met (duplicates counted)                        */
  uint32_t n_decls;         /* .reg declarations met                                             */
  uint64_t static_shared;   /* PtxModule.static_shared_bytes (ptx.py:249-254)                     */
  uint64_t regs_declared;   /* sum(PtxModule.registers_declared.values()) (features.py:126)       */
  uint32_t name_off, name_len;   /* kernel name, bytes from the segment start                    */
  uint32_t body_off, body_end;   /* first byte after '{' and offset of the matching '}'          */
} FfbSegInfo;

/* 64-byte instruction record and 16-byte label record: see csrc/ffb_records.cuh for the bit
 * layout of `meta` and of operand descriptors.  Opaque to most callers. */
typedef struct { uint32_t meta, line, off, len; uint64_t pred, aux, op[4]; } FfbInsRecC;
typedef struct { uint64_t hash; uint32_t index, off; } FfbLabelRecC;

/* Optional per-instruction text spans so a host can rebuild Instruction strings
 * (ptx.py:45-54) by slicing the source; offsets are bytes from the segment start. */
#define FFB_MAX_SPAN_OPS 12
typedef struct {
  uint32_t pred_off, pred_len, opc_off, opc_len, n_ops, reserved[3];
  uint32_t op_off[FFB_MAX_SPAN_OPS], op_len[FFB_MAX_SPAN_OPS];
} FfbSpanRec;

/* Optional `.reg` declaration records (ptx.py:244-248), FFB_MAX_DECLS per segment. */
#define FFB_MAX_DECLS 256
typedef struct { uint32_t cls_off, cls_len; uint64_t count; } FfbDeclRec;

typedef struct {
  const uint8_t* d_text;      /* corpus bytes; the allocation must be readable up to n_bytes   */
  int64_t n_bytes;            /* size rounded UP to a multiple of 16                            */
  const int64_t* d_seg_off;   /* [K+1] segment boundaries (byte offsets, ascending)             */
  int64_t n_segs;
  const int32_t* d_order;     /* optional [K]: processing order (e.g. longest first)            */
  const uint8_t* h_kernel_name; int32_t kernel_name_len;   /* optional parse_ptx(kernel_name=)  */
  uint32_t* d_hist;           /* [K, FFB_N_CLASSES] static class histogram                      */
  FfbSegInfo* d_info;         /* [K]                                                            */
  /* record mode: all NULL, or ins/labels + bases given (bases = exclusive scans of the
   * n_instr / n_labels a previous histogram-only call returned)                              */
  const int64_t* d_ins_base;  /* [K] */
  const int64_t* d_lab_base;  /* [K] */
  const int64_t* d_ins_cap;   /* optional [K]: record slots available per segment.  With caps the bases
                                 need not come from a counting pass (single-pass mode, e.g. bytes/12
                                 slots); a segment that needs more gets status FFB_E_CAPACITY */
  const int64_t* d_lab_cap;   /* optional [K] */
  void* d_ins;                /* FfbInsRecC[sum n_instr]                                        */
  void* d_labels;             /* FfbLabelRecC[sum n_labels]                                     */
  uint32_t* d_meta;           /* optional [sum n_instr]: copy of FfbInsRecC.meta, 4 B per instruction
                                 (the structural passes of K1b stream this instead of the records) */
  FfbSpanRec* d_spans;        /* optional, parallel to d_ins                                    */
  FfbDeclRec* d_decls;        /* optional, [K, FFB_MAX_DECLS]                                   */
  uint32_t flags;             /* FFB_LEX_* bits                                                 */
  uint32_t* d_path_counts;    /* optional [4]: segments finished by the fast path / by the exact walk,
                                 statements the fast path parsed byte-serially, reserved           */
} FfbLexDesc;
/* Two device kernels implement K1 with identical results: a byte-parallel fast path for regular
 * text (what compilers emit) and the exact statement walk for everything else; segments the fast
 * path declines are handed over on the device, in the same stream.  FFB_LEX_EXACT_ONLY skips the
 * fast path (it is also skipped for kernel-name filters and span / declaration records). */
#define FFB_LEX_EXACT_ONLY 1u
#define FFB_LEX_NO_LOCKSTEP 2u   /* small independent CTAs instead of one barrier-paced CTA per SM (fast path in record mode, exact walk) */
#define FFB_LEX_LOCKSTEP_HIST 4u /* accepted and ignored: histogram mode is barrier-paced by default as well */
int32_t ffb_lex_corpus(FfbContext* ctx, const FfbLexDesc* d, void* stream);
/* classify_opcode (ptx.py:99) and Instruction.access_bytes (ptx.py:64) for n opcode strings:
 * string i is d_text[d_off[i] : d_off[i+1]); d_out[n,3] = {class, state space, access bytes}. */
int32_t ffb_classify_opcodes(FfbContext* ctx, const uint8_t* d_text, const int64_t* d_off, int64_t n,
                             uint32_t* d_out, void* stream);

/* ---- K1b: control flow, trip counts, affine alignment, dynamic counts ------------------
 * Stands in for ptx.py:277-284 (branch targets), cfg.py:57-279 (build_cfg,
 * estimate_trip_counts), alignment.py:61-147 (trace_affine_scales,
 * analyze_memory_alignment) and features.py:62-81 (dynamic_instruction_counts), for every
 * segment of a corpus, from the records ffb_lex_corpus wrote.  Output: one FFB_F_* row per
 * segment (override columns cleared, FFB_F_OVR_TEXEC = NaN) ready for ffb_predict_grid.
 *
 * Capacities (status FFB_E_CAPACITY): integer literals and affine scales beyond 2^60,
 * producers with more than five operands whose late operands are registers.
 */
typedef struct { uint32_t n_blocks, n_edges, n_loops, reserved; } FfbFlowInfo;
typedef struct {
  uint32_t header;        /* block index of the loop header                                   */
  uint32_t n_body;        /* blocks in the body                                               */
  double   trip;          /* cfg.py:174-181                                                   */
  uint64_t label_hash;    /* header label (0 when the header carries none)                    */
  uint32_t label_off;     /* its name, bytes from the segment start                           */
  uint32_t has_label;
} FfbLoopRec;

typedef struct {
  int64_t n_segs;
  const FfbSegInfo* d_info;       /* [K] from ffb_lex_corpus                                   */
  const int64_t* d_ins_base;      /* [K] */
  const int64_t* d_lab_base;      /* [K] */
  const void* d_ins;              /* FfbInsRecC[n_ins_total]                                   */
  const void* d_labels;           /* FfbLabelRecC[n_lab_total]                                 */
  const uint32_t* d_meta;         /* optional [n_ins_total] from ffb_lex_corpus (faster when given) */
  int64_t n_ins_total, n_lab_total;
  const int32_t* d_order;         /* optional [K] processing order                             */
  double default_trip;            /* cfg.py:157 (reference default 32.0)                       */
  const uint64_t* h_ann_hash;     /* optional trip annotations: ffb_name_hash(label) ...       */
  const double* h_ann_trip;       /* ... -> trip (cfg.py:165-176); applied to every segment    */
  int32_t n_ann;
  uint8_t* d_ann_hit;             /* optional [n_ann]: set to 1 when some loop header matched  */
  double* d_feat;                 /* [K, FFB_FEAT_WIDTH]                                       */
  uint32_t* d_status;             /* [K] final status (lexer status, or an error found here)   */
  FfbFlowInfo* d_flow;            /* optional [K]                                              */
  /* detail outputs for callers that rebuild ControlFlowGraph objects (cfg.py:25-35); all
   * optional.  Segment k uses slots starting at  o = d_ins_base[k] + 2*k.                     */
  uint32_t* d_block_start;        /* [n_ins_total + 2K + 8]  n_blocks+1 entries per segment     */
  int32_t* d_edges;               /* [2*(n_ins_total + 2K + 8), 2]  pairs start at 2*o          */
  FfbLoopRec* d_loops;            /* [n_ins_total + 2K + 8]                                     */
  uint8_t* d_loop_body;           /* single-segment use: n_loops x n_blocks membership matrix   */
  int64_t loop_body_cap;          /* bytes available behind d_loop_body                         */
  double* d_weights;              /* [n_ins_total + 2K + 8] block weights (cfg.py:43-54)        */
  uint32_t flags;                 /* FFB_FLOW_* bits                                            */
} FfbFlowDesc;
#define FFB_FLOW_SEQUENTIAL_PASS 1u   /* textual pass on one lane only (the general form; default: 32 statements per round) */
#define FFB_FLOW_ONE_KERNEL 2u        /* CFG + dataflow in one launch (default for feature rows only: two launches) */
int32_t ffb_kernel_features(FfbContext* ctx, const FfbFlowDesc* d, void* stream);
/* 61-bit name hash the lexer assigns to labels / registers (for annotation keys). */
uint64_t ffb_name_hash(const uint8_t* name, int64_t len);

#ifdef __cplusplus
}
#endif
#endif /* FFB_H_ */

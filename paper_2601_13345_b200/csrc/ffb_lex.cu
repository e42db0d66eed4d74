// K1: GPU byte-lexer, opcode classifier and per-kernel class histogram.
//
// Restates (never copies) pkg/src/ptxwatt/ptx.py:99-313 of the reference: comment stripping
// (:139-141), kernel location and brace matching (:165-187), the line / ';' driven statement
// loop with labels, bare braces, directives and multi-line statements (:227-270), predicate
// and first-token opcode extraction (:296-313), the nine-class classifier (:99-136), access
// width (:64-76), .reg / .shared declarations (:37-40,244-254).
//
// Parallel formulation (one warp per corpus segment, i.e. per kernel):
//   T0  16-byte vector loads stage a 4 KB tile of text in shared memory;
//   T1  comment automaton, byte-parallel: each lane owns 128 bytes, lanes exchange their
//       entry state with shuffles until consistent, comment bytes are blanked in place
//       (the blanked text equals the reference's cleaned text up to trailing blanks);
//   T2  newline positions by per-lane counts + warp prefix sum  -> line table;
//   T3  one lane per line: brace depth (body end), a 2-bit "pending statement" map per line
//       composed across lanes with a shuffle scan (ptx.py's `pending` string is a 1-bit
//       state once the opener parses its own continuation), then the statement walk:
//       label / brace / directive / instruction, opcode tokens compared as packed u64 words.
//   Per-lane class counters are reduced with shuffles once per segment and stored by lane 0
//   (a segment has exactly one owner warp, so no atomics are needed on the histogram).
// In record mode the same walk also parses operands and writes one 64-byte FfbInsRec per
// instruction for the dataflow kernel (K1b).
#include "ffb_lex_shared.cuh"
#include "ffb_lexfast.cuh"
#include <stdlib.h>

namespace {


// The statement loop of one line s[b,e) (newline excluded, possibly truncated at the body
// end).  pending_in: the line starts inside an unfinished statement.  hi/depth_in serve the
// look-ahead of a statement this line opens.  kMode 0 only fills the summary.
template <int kMode>
FFB_COLD_INLINE LineSummary walk_line(const uint8_t* s, int b, int e, bool pending_in, int hi, int depth_in,
                            bool at_seg_end, Emit& em) {
  LineSummary r;
  r.nonblank = r.has_semi = r.pend_out0 = r.defer = r.unterminated = false;
  r.n0 = r.n_after = r.lab0 = r.lab_after = r.dcl0 = r.dcl_after = 0;
  int line_b = b;
  while (b < e && ffb_is_ws(s[b])) ++b;
  while (e > b && ffb_is_ws(s[e - 1])) --e;
  if (b >= e) { r.pend_out0 = false; return r; }
  r.nonblank = true;
  bool pending = pending_in;
  bool after_first = false;       // past the first ';' of the line
  int pos = b;
  // depth at `pos` is needed only when a statement is opened: count braces lazily
  while (pos < e) {
    if (!pending) {
      int k = pos;
      while (k < e && ffb_is_label_char(s[k])) ++k;
      if (k > pos && k < e && s[k] == ':') {                       // ptx.py:232-236
        if (kMode > 0) {
          if (kMode == 2) {
            FfbLabelRec L;
            const uint64_t h0 = norm_hash(s, pos, k);
            L.hash = h0; L.index = (uint32_t)(em.ins_at - em.a->ins_base[em.seg]);
            L.off = (uint32_t)(em.abase + pos - em.seg_begin);
            if (em.lab_at < em.lab_limit) em.a->labels[em.lab_at] = L;
          }
          em.lab_at += 1;
        }
        if (after_first) r.lab_after += 1;
        r.lab0 += 1;
        pos = scan_ws(s, k + 1, e);
        continue;
      }
      if (e - pos == 1 && (s[pos] == '{' || s[pos] == '}')) break;   // ptx.py:237-239
      if (s[pos] == '.') {                                        // ptx.py:240-256
        int semi = pos;
        while (semi < e && s[semi] != ';') ++semi;
        int nd = 0;
        do_directive<kMode>(s, pos, semi, em, &nd);
        r.dcl0 += nd;
        if (after_first) r.dcl_after += nd;
        if (semi < e) { if (!after_first) { r.has_semi = true; after_first = true; } pos = scan_ws(s, semi + 1, e); }
        else pos = e;
        continue;
      }
    }
    int semi = pos;
    while (semi < e && s[semi] != ';') ++semi;
    if (pending) {
      // continuation of a statement an earlier line opened: that line's lane parses it
      if (semi >= e) { pos = e; break; }                          // still pending (ptx.py:257-262)
      if (!after_first) { r.has_semi = true; after_first = true; }
      pending = false;
      pos = scan_ws(s, semi + 1, e);
      continue;
    }
    if (semi >= e) {
      // this line opens a multi-line statement: find its ';' further down the tile
      int d = depth_in;
      for (int i = line_b; i < pos; ++i) { if (s[i] == '{') ++d; else if (s[i] == '}') --d; }
      const int close = find_closing_semi(s, pos, hi, d);
      if (close == -2 || (close == -1 && at_seg_end)) { r.unterminated = true; r.pend_out0 = true; pos = e; break; }
      if (close == -1) { r.defer = true; r.pend_out0 = true; pos = e; break; }
      r.n0 += 1;
      if (after_first) r.n_after += 1;
      if (kMode > 0) do_statement<kMode>(s, pos, close, em);
      r.pend_out0 = true;
      pending = true;
      pos = e;
      break;
    }
    // ordinary statement s[pos, semi)
    {
      int q = semi;
      while (q > pos && ffb_is_ws(s[q - 1])) --q;
      if (q > pos) {
        r.n0 += 1;
        if (after_first) r.n_after += 1;
        if (kMode > 0) do_statement<kMode>(s, pos, semi, em);
      }
    }
    if (!after_first) { r.has_semi = true; after_first = true; }
    pos = scan_ws(s, semi + 1, e);
  }
  return r;
}

// ---- the kernel --------------------------------------------------------------------------------
// kRecords: also write FfbInsRec / FfbLabelRec (and the optional span / decl records)
// kLockstep: as in the fast kernel, one CTA fills the SM and its warps meet at a barrier before every tile
// (the loop body is long; warps of a scheduler that run the same phase share fetched instruction lines).
template <bool kRecords, bool kLockstep>
__global__ void __launch_bounds__(kLockstep ? (kRecords ? 512 : 1024) : kWarps * 32, kLockstep ? 1 : (kRecords ? 2 : 4))   // record mode needs ~128 registers (measured: capping at 64 spills and is 1.5x slower)
lex_corpus_kernel(LexArgs a) {
  constexpr int kMain = kRecords ? 2 : 1;
  FFB_DYN_SMEM(smem_raw);
  __shared__ uint8_t s_cls[256];
  __shared__ uint64_t s_tok_key[256];
  __shared__ uint32_t s_tok_val[256];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* s = smem_raw + (size_t)wid * kWarpSmem;
  uint16_t* nl = reinterpret_cast<uint16_t*>(s + kTile + kPad);
  for (int c = threadIdx.x; c < 256; c += (int)blockDim.x) { s_cls[c] = char_class((unsigned)c); s_tok_key[c] = ~0ull; s_tok_val[c] = 0; }
  __syncthreads();
  for (int c = threadIdx.x; c < kNumTokDefs; c += (int)blockDim.x) {
    const uint32_t slot = (uint32_t)((kTokDefs[c].key * kTokMul) >> 56);
    s_tok_key[slot] = kTokDefs[c].key; s_tok_val[slot] = kTokDefs[c].val;
  }
  __syncthreads();

  // One tile per trip of the main loop: segment state lives across trips so that lock-step CTAs can
  // meet at a barrier between tiles.
  bool have = false, done = false, pending = false;                 // pending: ptx.py's `pending` string is non-empty
  int64_t seg = 0, seg_begin = 0, seg_end = 0, cur = 0;
  int64_t scan_from_g = 0;                                          // SEARCH / HEADER resume position
  int64_t body_pos_g = 0;                                           // first body byte (after '{')
  int64_t noblk_from_g = 0;                                         // from here on "/*" is plain text (unterminated comment)
  int64_t blk_close_g = -1;                                         // a "*/" is known to exist up to here
  int64_t name_off = 0, name_len = 0, body_end_off = 0;
  int phase = PH_SEARCH, depth = 0;
  int cm_state = S_CODE;                                            // comment automaton state at `cur`
  uint32_t line_no = 1;                                             // source line of the byte at `cur`
  uint32_t status = FFB_OK, n_instr = 0, n_labels = 0, n_decls = 0;
  Emit em;
  em.a = &a; em.tok.key = s_tok_key; em.tok.val = s_tok_val; em.cls = s_cls;
  em.seg = 0; em.seg_begin = 0; em.abase = 0; em.line = 0; em.ins_at = 0; em.lab_at = 0;
  em.ins_limit = 0; em.lab_limit = 0; em.dcl_at = 0; em.c0 = em.c1 = em.c2 = 0;
  em.shared_bytes = 0; em.regs = 0;
  for (;;) {
    if (!have && !done) {
    unsigned long long w = 0;
    if (lane == 0) w = atomicAdd(a.work, 1ull);
    w = __shfl_sync(kFull, w, 0);
    if (w >= (a.n_work ? *a.n_work : (unsigned long long)a.n_segs)) done = true;
    else {
      have = true;
      seg = a.order ? (int64_t)a.order[w] : (int64_t)w;
      seg_begin = a.seg_off[seg]; seg_end = a.seg_off[seg + 1];
      phase = PH_SEARCH; cm_state = S_CODE;
      noblk_from_g = 0x7fffffffffffffffLL; blk_close_g = -1;
      depth = 0; pending = false; line_no = 1; status = FFB_OK;
      cur = seg_begin; scan_from_g = seg_begin; body_pos_g = 0;
      name_off = 0; name_len = 0; body_end_off = 0;
      n_instr = 0; n_labels = 0; n_decls = 0;
      em.seg = seg; em.seg_begin = seg_begin; em.abase = 0; em.line = 0;
      em.ins_at = kRecords ? a.ins_base[seg] : 0;
      em.lab_at = kRecords ? a.lab_base[seg] : 0;
      em.ins_limit = (kRecords && a.ins_cap) ? em.ins_at + a.ins_cap[seg] : 0x7fffffffffffffffLL;
      em.lab_limit = (kRecords && a.lab_cap) ? em.lab_at + a.lab_cap[seg] : 0x7fffffffffffffffLL;
      em.dcl_at = 0;
      em.c0 = em.c1 = em.c2 = 0;
      em.shared_bytes = 0; em.regs = 0;
    }
    }
    if (kLockstep) { if (!__syncthreads_or(done ? 0 : 1)) break; }
    else if (done) break;
    if (done) continue;                      // idle warps keep meeting the barrier

    if (phase != PH_DONE && status == FFB_OK && cur < seg_end) do {
      // ================= T0: stage the tile =================
      const int64_t abase = cur & ~(int64_t)15;
      const int64_t hi_g = (abase + kTile < seg_end) ? abase + kTile : seg_end;
      const int lo = (int)(cur - abase), hi = (int)(hi_g - abase);
      const bool at_seg_end = hi_g == seg_end;
      __syncwarp();
      for (int v = lane; v < kTile / 16; v += 32) {
        const int64_t g = abase + (int64_t)v * 16;
        uint4 val;
        if (g + 16 <= a.n_bytes) val = *reinterpret_cast<const uint4*>(a.text + g);
        else { val.x = val.y = val.z = val.w = 0x0a0a0a0au; }
        *reinterpret_cast<uint4*>(s + v * 16) = val;
      }
      __syncwarp();
      for (int i = hi + lane; i < kTile + kPad; i += 32) s[i] = '\n';
      __syncwarp();
      em.abase = abase;

      // ================= T1: comments =================
      const int chunk_base = lane * kLaneBytes;
      const int c0 = max(chunk_base, lo), c1 = min(chunk_base + kLaneBytes, hi);
      uint32_t slash[4], unused4[4];
      chunk_masks(s + chunk_base, 0x2f2f2f2fu, 0x2f2f2f2fu, c0 - chunk_base, c1 - chunk_base, slash, unused4);
      const bool has_slash = (slash[0] | slash[1] | slash[2] | slash[3]) != 0;
      int st_in = S_CODE, st_out = S_CODE, last_open = -1;
      int noblk_from = noblk_from_g >= abase + kTile ? 0x7fffffff : (noblk_from_g <= abase ? 0 : (int)(noblk_from_g - abase));
      for (int attempt = 0; attempt < 2; ++attempt) {
        bool need = true;
        st_in = S_CODE;
        for (int guard = 0; guard < 40; ++guard) {
          if (need) {
            last_open = -1;
            if (c0 >= c1) st_out = st_in;
            else if (!has_slash && st_in == S_CODE) st_out = S_CODE;
            else st_out = cm_run(s, c0, c1, st_in, false, slash, chunk_base, noblk_from, &last_open);
            need = false;
          }
          int left = __shfl_up_sync(kFull, st_out, 1);
          if (lane == 0) left = cm_state;
          const bool changed = left != st_in;
          if (!__any_sync(kFull, changed)) break;
          if (changed) { st_in = left; need = true; }
        }
        // a block comment still open at the tile end must have its "*/" somewhere behind
        const int end_state = __shfl_sync(kFull, st_out, 31);
        if (end_state < S_BLK || attempt == 1 || blk_close_g >= abase + hi) break;
        int64_t found = -1;
        const int64_t from = abase + hi - ((end_state == S_BLK_STAR || end_state == S_LBLK_STAR) ? 1 : 0);
        for (int64_t g0 = from; g0 < seg_end - 1 && found < 0; g0 += 32) {
          const int64_t g = g0 + lane;
          const bool hit = g + 1 < seg_end && a.text[g] == '*' && a.text[g + 1] == '/';
          const unsigned mask = __ballot_sync(kFull, hit);
          if (mask) found = g0 + __ffs((int)mask) - 1;
        }
        if (found >= 0) { blk_close_g = found + 2; break; }
        // unterminated: the last "/*" of this tile and everything behind it is ordinary text
        int lo_open = last_open;
#pragma unroll
        for (int dd = 16; dd > 0; dd >>= 1) { const int o = __shfl_xor_sync(kFull, lo_open, dd); lo_open = o > lo_open ? o : lo_open; }
        if (lo_open < 0) break;                       // opened in an earlier tile: cannot happen, keep going
        noblk_from_g = abase + lo_open;
        noblk_from = lo_open;
      }
      const bool dirty = (has_slash || st_in != S_CODE) && c0 < c1;
      if (__any_sync(kFull, dirty)) {
        int dummy = -1;
        if (dirty) cm_run(s, c0, c1, st_in, true, slash, chunk_base, noblk_from, &dummy);
        __syncwarp();
      }

      // ================= T2: line table =================
      uint32_t nlm[4], nlb[4];
      chunk_masks(s + chunk_base, 0x0a0a0a0au, 0x8a8a8a8au, c0 - chunk_base, c1 - chunk_base, nlm, nlb);
      const int my_nl = __popc(nlm[0]) + __popc(nlm[1]) + __popc(nlm[2]) + __popc(nlm[3]);
      int total_nl = 0;
      int at = warp_excl_sum(my_nl, &total_nl);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t m = nlm[k];
        while (m) {
          const int bit = __ffs((int)m) - 1;
          m &= m - 1;
          const int i = chunk_base + 32 * k + bit;
          const bool in_block = (nlb[k] >> bit) & 1u;
          if (at < kMaxLines) nl[at] = (uint16_t)(i | (in_block ? 0x8000 : 0));
          if (in_block) s[i] = '\n';
          ++at;
        }
      }
      const int n_real = total_nl < kMaxLines ? total_nl : kMaxLines;
      // A tile without a newline whose last byte lies inside a `//` comment: the staged bytes are the code of one
      // physical line followed by comment text, and whatever follows up to the real newline is comment as well
      // (the automaton state is carried into the next tile).  The line is closed at `hi`; the rest of the comment
      // becomes a blank line that owns the real newline, which ptx.py:230 skips - same statements, same line numbers.
      const int tile_end_state = __shfl_sync(kFull, st_out, 31);
      const bool comment_tail = !at_seg_end && total_nl == 0 && hi - lo >= kTile / 2 &&
                                (tile_end_state == S_LINE || tile_end_state == S_LINE_SLASH || tile_end_state == S_LBLK || tile_end_state == S_LBLK_STAR);
      // A tile without a newline while the kernel is still being looked for (module-level initialiser lists are
      // emitted on one line of any length): nothing but `.entry`, the kernel name and the opening brace matter
      // there (ptx.py:165-176 works on the whole text), so the tile is cut at the last 128-byte chunk edge whose
      // automaton state needs no look-behind and the next tile resumes there in that state.
      int cut = -1, cut_state = S_CODE;
      if (!at_seg_end && total_nl == 0 && !comment_tail && (phase == PH_SEARCH || phase == PH_HEADER)) {
        const unsigned okm = __ballot_sync(kFull, chunk_base > lo && chunk_base < hi && st_in != S_SLASH && st_in != S_SLASH2);
        if (okm) { const int l = 31 - __clz((int)okm); cut = l * kLaneBytes; cut_state = __shfl_sync(kFull, st_in, l); }
      }
      const int line_hi = cut >= 0 ? cut : hi;
      // the text may end without a newline: close the last line at `hi`
      const bool virtual_last = (at_seg_end || comment_tail || cut >= 0) && total_nl < kMaxLines;
      if (virtual_last && lane == 0) nl[n_real] = (uint16_t)line_hi;
      const int n_lines = n_real + (virtual_last ? 1 : 0);
      __syncwarp();
      if (n_lines == 0) { status = FFB_E_CAPACITY; break; }         // a line longer than the tile
      const int region_end = virtual_last ? line_hi : (nl[n_real - 1] & 0x7fff) + 1;
      int consume_to = region_end;     // smem index where the next tile starts
      bool skip_rest = false;

      // ================= T3a: locate the kernel (ptx.py:165-187) =================
      if (phase == PH_SEARCH) {
        int from = (int)(scan_from_g - abase);
        if (from < lo) from = lo;
        for (;;) {
          int cand = 0x7fffffff;
          for (int i = max(c0, from); i < min(c1, region_end); ++i)
            if (s[i] == '.' && s[i + 1] == 'e' && s[i + 2] == 'n' && s[i + 3] == 't' && s[i + 4] == 'r' && s[i + 5] == 'y') { cand = i; break; }
          cand = warp_min(cand);
          if (cand == 0x7fffffff) { scan_from_g = abase + region_end; break; }
          int q = cand + 6;
          while (q < hi && ffb_is_ws(s[q])) ++q;
          int r = q;
          bool ok = q > cand + 6 && q < hi && ffb_is_name_start(s[q]);
          if (ok) { r = q + 1; while (r < hi && ffb_is_name_char(s[r])) ++r; }
          if ((q >= hi || (ok && r >= hi)) && !at_seg_end) {
            // the match runs off the staged bytes: restart the tile at the candidate
            if (cand == lo) status = FFB_E_CAPACITY;
            consume_to = cand; scan_from_g = abase + cand; skip_rest = true;
            break;
          }
          if (!ok) { from = cand + 1; continue; }
          bool take = true;
          if (a.want_name) {
            take = (r - q) == a.want_len;
            for (int i = 0; take && i < a.want_len; ++i) take = s[q + i] == a.want_name[i];
          }
          if (!take) { from = r; continue; }
          name_off = abase + q - seg_begin; name_len = r - q;
          phase = PH_HEADER; scan_from_g = abase + r;
          break;
        }
      }
      if (status != FFB_OK) break;
      if (phase == PH_HEADER && !skip_rest) {
        int from = (int)(scan_from_g - abase);
        if (from < lo) from = lo;
        int cand = 0x7fffffff;
        for (int i = max(c0, from); i < min(c1, region_end); ++i)
          if (s[i] == '{') { cand = i; break; }
        cand = warp_min(cand);
        if (cand == 0x7fffffff) {
          if (scan_from_g < abase + region_end) scan_from_g = abase + region_end;
        } else {
          phase = PH_BODY; depth = 1; pending = false;
          body_pos_g = abase + cand + 1;
        }
      }

      // a cut tile never runs body lines: the body is re-staged from its first byte
      if (cut >= 0 && phase == PH_BODY && !skip_rest) { skip_rest = true; consume_to = (int)(body_pos_g - abase); }

      // ================= T3b: body lines (ptx.py:227-270) =================
      if (phase == PH_BODY && !skip_rest) {
        int pos = body_pos_g > cur ? (int)(body_pos_g - abase) : lo;
        if (pos <= region_end) {
          int first = 0;
          for (int l = lane; l < n_lines; l += 32) first += ((nl[l] & 0x7fff) < pos) ? 1 : 0;
          first = (int)warp_sum_u64((unsigned long long)first);
          for (int l0 = first; l0 < n_lines; l0 += 32) {
            const int li = l0 + lane;
            const bool live = li < n_lines;
            int b = 0, e = 0;
            if (live) {
              b = li == 0 ? lo : (nl[li - 1] & 0x7fff) + 1;
              e = nl[li] & 0x7fff;
              if (b < pos) b = pos;               // the line that holds the opening brace
            }
            // ---- feature scan: one uniform pass over the batch's lines ----
            const int len = live ? e - b : 0;
            int maxlen = len;
#pragma unroll
            for (int dd = 16; dd > 0; dd >>= 1) { const int o = __shfl_xor_sync(kFull, maxlen, dd); maxlen = o > maxlen ? o : maxlen; }
            int fb = 0x7fffffff, lb = -1, n_semi = 0, n_colon = 0, n_nonws = 0;
            unsigned seen = 0;
            for (int i = 0; i < maxlen; ++i) {
              if (i < len) {
                const unsigned k = s_cls[s[b + i]];
                seen |= k;
                n_semi += (k >> 1) & 1; n_colon += (k >> 4) & 1;
                if (!(k & CC_WS)) { fb = min(fb, b + i); lb = b + i; ++n_nonws; }
              }
            }
            if (lb < 0) fb = -1;
            // braces are rare (vector operands, nested scopes): walk them only where they occur
            int run = 0, min_run = 0x7fffffff;
            if (seen & (CC_LBRACE | CC_RBRACE)) {
              for (int i = b; i < e; ++i) {
                const unsigned c = s[i];
                if (c == '{') ++run;
                else if (c == '}') { --run; if (run < min_run) min_run = run; }
              }
            }
            int tot_delta = 0;
            const int d_in = depth + warp_excl_sum(run, &tot_delta);
            const bool closes = live && min_run != 0x7fffffff && d_in + min_run <= 0;
            const unsigned close_mask = __ballot_sync(kFull, closes);
            const int end_lane = close_mask ? __ffs((int)close_mask) - 1 : 32;
            int close_at = -1;
            if (lane == end_lane) {
              int d = d_in;
              for (int i = b; i < e; ++i) {
                const unsigned c = s[i];
                if (c == '{') ++d;
                else if (c == '}') { if (--d == 0) { close_at = i; break; } }
              }
              e = close_at;
            }
            const bool mine = live && lane <= end_lane;
            // ---- line kind ----
            int kind = LK_COMPLEX;
            if (fb < 0) kind = LK_BLANK;
            else if (min_run == 0x7fffffff || (min_run >= 0 && run == 0)) {
              const unsigned c_first = s[fb], c_last = s[lb];
              if (c_first == '.') {
                const bool decl = (s[fb + 1] == 'r' && s[fb + 2] == 'e' && s[fb + 3] == 'g') ||
                                  (s[fb + 1] == 's' && s[fb + 2] == 'h' && s[fb + 3] == 'a');
                if (n_semi == 0 && n_colon == 0 && !decl) kind = LK_SKIP;         // ptx.py:255-256
              } else if (c_last == ';' && n_semi == 1 && n_colon == 0 && lb > fb) {
                kind = LK_STMT;       // one statement, ';' last (braces inside operands are balanced)
              } else if (c_last == ':' && n_semi == 0 && n_colon == 1 && lb - fb + 1 == n_nonws && lb > fb) {
                bool all_label = true;                                            // ptx.py:232-236
                for (int i = fb; i < lb && all_label; ++i) all_label = (s_cls[s[i]] & CC_LABEL) != 0;
                if (all_label) kind = LK_LABEL;
              }
            }
            if (lane == end_lane) kind = LK_COMPLEX;
            // ---- structure of the line if it starts outside a statement ----
            LineSummary sm;
            sm.nonblank = kind != LK_BLANK; sm.has_semi = kind == LK_STMT;
            sm.pend_out0 = sm.defer = sm.unterminated = false;
            sm.n0 = kind == LK_STMT ? 1 : 0; sm.n_after = 0;
            sm.lab0 = kind == LK_LABEL ? 1 : 0; sm.lab_after = 0; sm.dcl0 = sm.dcl_after = 0;
            if (mine && kind == LK_COMPLEX) sm = walk_line<0>(s, b, e, false, hi, d_in, at_seg_end, em);
            // pending map: f0 = state after the line when it starts clean, f1 = when it starts
            // inside a statement; blank lines are the identity (ptx.py:230 `while line`)
            unsigned f0 = 0, f1 = 1;
            if (mine && sm.nonblank) { f0 = sm.pend_out0 ? 1u : 0u; f1 = sm.has_semi ? f0 : 1u; }
            unsigned m0 = f0, m1 = f1;          // inclusive composition over lanes 0..lane
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
              const unsigned o0 = __shfl_up_sync(kFull, m0, dd), o1 = __shfl_up_sync(kFull, m1, dd);
              if (lane >= dd) { const unsigned t0 = o0 ? m1 : m0, t1 = o1 ? m1 : m0; m0 = t0; m1 = t1; }
            }
            unsigned e0 = __shfl_up_sync(kFull, m0, 1), e1 = __shfl_up_sync(kFull, m1, 1);
            if (lane == 0) { e0 = 0; e1 = 1; }
            const bool p_in = pending ? (e1 != 0) : (e0 != 0);
            // the statement a line opens is only real if the line's tail is reached outside a
            // statement: always after a ';', otherwise only when the line starts clean
            const bool tail_real = mine && (!p_in || sm.has_semi);
            const unsigned defer_mask = __ballot_sync(kFull, tail_real && sm.defer);
            const int defer_lane = defer_mask ? __ffs((int)defer_mask) - 1 : 32;
            const bool run_line = mine && lane < defer_lane;
            const bool bad = run_line && tail_real && sm.unterminated;
            int n_ins = 0, n_lab = 0, n_dcl = 0;
            if (run_line) {
              if (p_in) { if (sm.has_semi) { n_ins = sm.n_after; n_lab = sm.lab_after; n_dcl = sm.dcl_after; } }
              else { n_ins = sm.n0; n_lab = sm.lab0; n_dcl = sm.dcl0; }
            }
            int tot_ins = 0, tot_lab = 0, tot_dcl = 0;
            const int ins_ex = warp_excl_sum(n_ins, &tot_ins);
            const int lab_ex = warp_excl_sum(n_lab, &tot_lab);
            const int dcl_ex = warp_excl_sum(n_dcl, &tot_dcl);
            // ---- main walk ----
            {
              const int64_t ins0 = em.ins_at, lab0 = em.lab_at;
              const int dcl0 = em.dcl_at;
              em.ins_at = ins0 + ins_ex; em.lab_at = lab0 + lab_ex; em.dcl_at = dcl0 + dcl_ex;
              em.line = line_no + (uint32_t)li;
              if (run_line) {
                if (p_in || kind == LK_COMPLEX) walk_line<kMain>(s, b, e, p_in, hi, d_in, at_seg_end, em);
                else if (kind == LK_STMT) do_statement<kMain>(s, fb, lb, em);
                else if (kind == LK_LABEL) {
                  if (kMain == 2) {
                    FfbLabelRec L;
                    L.hash = norm_hash(s, fb, lb); L.index = (uint32_t)(em.ins_at - a.ins_base[seg]);
                    L.off = (uint32_t)(abase + fb - seg_begin);
                    if (em.lab_at < em.lab_limit) a.labels[em.lab_at] = L;
                  }
                }
              }
              em.ins_at = ins0 + tot_ins; em.lab_at = lab0 + tot_lab; em.dcl_at = dcl0 + tot_dcl;
            }
            n_instr += (uint32_t)tot_ins; n_labels += (uint32_t)tot_lab; n_decls += (uint32_t)tot_dcl;
            if (__any_sync(kFull, bad)) { status = FFB_E_MALFORMED_PTX; break; }   // ptx.py:272-273
            // ---- carry ----
            if (defer_lane < 32) {
              const int keep = l0 + defer_lane;          // lines consumed by this tile
              if (keep == 0) { status = FFB_E_CAPACITY; break; }     // statement longer than the tile
              if (defer_lane > 0) {
                const unsigned pm0 = __shfl_sync(kFull, m0, defer_lane - 1), pm1 = __shfl_sync(kFull, m1, defer_lane - 1);
                pending = pending ? (pm1 != 0) : (pm0 != 0);
              }
              depth = __shfl_sync(kFull, d_in, defer_lane);
              consume_to = (nl[keep - 1] & 0x7fff) + 1;
              // the deferred line may be the one holding the opening brace
              if (body_pos_g > abase + consume_to) { /* resume position already recorded */ }
              break;
            }
            const int last_lane = end_lane < 32 ? end_lane : min(31, n_lines - 1 - l0);
            {
              const unsigned pm0 = __shfl_sync(kFull, m0, last_lane), pm1 = __shfl_sync(kFull, m1, last_lane);
              pending = pending ? (pm1 != 0) : (pm0 != 0);
            }
            if (end_lane < 32) {
              phase = PH_DONE;
              body_end_off = abase + __shfl_sync(kFull, close_at, end_lane) - seg_begin;
              break;
            }
            depth += tot_delta;
            pos = lo;
          }
        }
      }
      if (status != FFB_OK) break;
      if (phase == PH_DONE) break;

      // ================= advance =================
      int nlc = 0;
      for (int l = lane; l < n_real; l += 32) nlc += ((nl[l] & 0x7fff) < consume_to) ? 1 : 0;
      nlc = (int)warp_sum_u64((unsigned long long)nlc);
      cm_state = (comment_tail && consume_to == hi) ? tile_end_state : ((cut >= 0 && consume_to == cut) ? cut_state : S_CODE);
      if (nlc > 0) {
        const unsigned last = nl[nlc - 1];
        if ((int)(last & 0x7fff) == consume_to - 1 && (last & 0x8000)) cm_state = S_BLK;
      }
      line_no += (uint32_t)nlc;
      const int64_t next = abase + consume_to;
      if (next <= cur) { status = FFB_E_CAPACITY; break; }
      cur = next;
    } while (0);
    if (phase != PH_DONE && status == FFB_OK && cur < seg_end) continue;      // more tiles of this segment
    have = false;

    // ================= segment epilogue =================
    if (status == FFB_OK) {
      if (phase == PH_SEARCH) status = FFB_E_NO_KERNEL;                                // ptx.py:186-187
      else if (phase == PH_HEADER || phase == PH_BODY) status = FFB_E_MALFORMED_PTX;   // :175, :184
      else if (pending) status = FFB_E_MALFORMED_PTX;                                  // :272-273
      else if (n_instr == 0) status = FFB_E_MALFORMED_PTX;                             // :274-275
    }
    if (kRecords && status == FFB_OK && ((a.ins_cap && (int64_t)n_instr > a.ins_cap[seg]) || (a.lab_cap && (int64_t)n_labels > a.lab_cap[seg])))
      status = FFB_E_CAPACITY;            // single-pass mode: the segment outgrew its record slots
    uint32_t tot[FFB_N_CLASSES];
#pragma unroll
    for (int c = 0; c < FFB_N_CLASSES; ++c) {
      const uint64_t word = c < 3 ? em.c0 : (c < 6 ? em.c1 : em.c2);
      tot[c] = (uint32_t)warp_sum_u64((word >> (21 * (c % 3))) & 0x1fffffull);
    }
    const unsigned long long sh = warp_sum_u64(em.shared_bytes), rg = warp_sum_u64(em.regs);
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < FFB_N_CLASSES; ++c) a.hist[seg * FFB_N_CLASSES + c] = tot[c];
      FfbSegInfo inf;
      inf.status = status; inf.n_instr = n_instr; inf.n_labels = n_labels; inf.n_decls = n_decls;
      inf.static_shared = sh; inf.regs_declared = rg;
      inf.name_off = (uint32_t)name_off; inf.name_len = (uint32_t)name_len;
      inf.body_off = (uint32_t)(body_pos_g ? body_pos_g - seg_begin : 0); inf.body_end = (uint32_t)body_end_off;
      a.info[seg] = inf;
    }
  }
}

// Batch classifier: one thread per opcode string (ptx.py:99-136 and :64-76 as pure functions).
__global__ void __launch_bounds__(256)
classify_opcodes_kernel(const uint8_t* text, const int64_t* off, int64_t n, uint32_t* out) {
  __shared__ uint64_t s_tok_key[256];
  __shared__ uint32_t s_tok_val[256];
  s_tok_key[threadIdx.x] = ~0ull; s_tok_val[threadIdx.x] = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < kNumTokDefs; c += 256) {
    const uint32_t slot = (uint32_t)((kTokDefs[c].key * kTokMul) >> 56);
    s_tok_key[slot] = kTokDefs[c].key; s_tok_val[slot] = kTokDefs[c].val;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= n) return;
  TokTable tt; tt.key = s_tok_key; tt.val = s_tok_val;
  const int64_t b = off[i], e = off[i + 1];
  const OpcodeInfo oc = classify_opcode(tt, text + b, 0, (int)(e - b));
  out[3 * i] = oc.cls; out[3 * i + 1] = oc.space; out[3 * i + 2] = oc.bytes;
}

}  // namespace

extern "C" int32_t ffb_classify_opcodes(FfbContext* ctx, const uint8_t* d_text, const int64_t* d_off, int64_t n,
                                        uint32_t* d_out, void* stream) {
  if (!ctx || !d_text || !d_off || !d_out || n < 0) return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_classify_opcodes: bad argument");
  if (n == 0) return FFB_OK;
  FFB_CUDA(ctx, cudaSetDevice(ctx->device));
  FFB_LAUNCH(classify_opcodes_kernel, (unsigned)((n + 255) / 256), 256, 0, stream, d_text, d_off, n, d_out);
  return ffb_check_launch(ctx, "classify_opcodes_kernel");
}

namespace {
__global__ void lex_path_counts_kernel(const unsigned long long* declined, int64_t n_segs, uint32_t* out) {
  if (threadIdx.x != 0) return;
  const uint32_t ex = declined ? (uint32_t)*declined : (uint32_t)n_segs;
  out[0] = (uint32_t)n_segs - ex;
  out[1] = ex;
  out[2] = declined ? (uint32_t)declined[2] : 0u;
  out[3] = 0u;
}
}  // namespace

extern "C" int32_t ffb_lex_corpus(FfbContext* ctx, const FfbLexDesc* d, void* stream_) {
  if (!ctx || !d || !d->d_text || !d->d_seg_off || !d->d_hist || !d->d_info || d->n_segs < 0)
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_lex_corpus: bad argument");
  if (d->n_bytes % 16 != 0)
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_lex_corpus: n_bytes must be the padded size (multiple of 16)");
  if (d->n_segs == 0) return FFB_OK;
  cudaStream_t stream = (cudaStream_t)stream_;
  FFB_CUDA(ctx, cudaSetDevice(ctx->device));
  int32_t rc = ffb_reserve(ctx, &ctx->d_lex, 4096);
  if (rc) return rc;
  LexArgs a = {};
  a.text = d->d_text; a.n_bytes = d->n_bytes; a.seg_off = d->d_seg_off; a.n_segs = d->n_segs;
  a.order = d->d_order; a.work = (unsigned long long*)ctx->d_lex.p;
  a.hist = d->d_hist; a.info = d->d_info;
  a.ins_base = d->d_ins_base; a.lab_base = d->d_lab_base; a.ins_cap = d->d_ins_cap; a.lab_cap = d->d_lab_cap;
  a.ins = (FfbInsRec*)d->d_ins; a.labels = (FfbLabelRec*)d->d_labels;
  a.spans = d->d_spans; a.decls = d->d_decls; a.meta = d->d_meta;
  a.want_name = nullptr; a.want_len = 0;
  if (d->h_kernel_name && d->kernel_name_len > 0) {
    if (d->kernel_name_len > 2048) return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_lex_corpus: kernel name too long");
    rc = ffb_stage_reserve(ctx, (size_t)d->kernel_name_len);
    if (rc) return rc;
    memcpy(ctx->h_stage, d->h_kernel_name, (size_t)d->kernel_name_len);
    uint8_t* dn = (uint8_t*)ctx->d_lex.p + 64;
    FFB_CUDA(ctx, cudaMemcpyAsync(dn, ctx->h_stage, (size_t)d->kernel_name_len, cudaMemcpyHostToDevice, stream));
    FFB_CUDA(ctx, cudaEventRecord(ctx->stage_free, stream));
    ctx->stage_busy = true;
    a.want_name = dn; a.want_len = d->kernel_name_len;
  }
  const bool records = d->d_ins != nullptr;
  if (records && (!d->d_ins_base || !d->d_lab_base || !d->d_labels))
    return ffb_fail(ctx, FFB_E_BAD_ARGUMENT, "ffb_lex_corpus: record mode needs ins/label buffers and their bases");
  const bool fast = !(d->flags & FFB_LEX_EXACT_ONLY) && !a.want_name && !a.spans && !a.decls;
  // scratch: [0,8) exact work counter  [8,16) hand-over count  [16,24) fast work counter  [24,32) statements the fast
  // kernel parsed byte-serially  [64,..) name  [4096,..) hand-over list
  if (fast) {
    rc = ffb_reserve(ctx, &ctx->d_lex, 4096 + (size_t)d->n_segs * 4);
    if (rc) return rc;
    a.work = (unsigned long long*)ctx->d_lex.p;
  }
  FFB_CUDA(ctx, cudaMemsetAsync(ctx->d_lex.p, 0, 32, stream));
  if (fast) {
    LexArgs f = a;
    f.work = (unsigned long long*)ctx->d_lex.p + 2;
    f.fb_count = (unsigned long long*)ctx->d_lex.p + 1;
    f.fb_list = (int32_t*)((uint8_t*)ctx->d_lex.p + 4096);
    // lock-step shape: one CTA per SM (16 warps at 128 registers in record mode, 24 at 80 in histogram mode)
    // measured: record mode 17.1 ms vs 32.0 ms per 1.44 GB (r1p); histogram mode 482 vs 416 GB/s once its
    // parser had been shortened (r1z; before that the barrier cost it 3%)
    const bool lockstep = !(d->flags & FFB_LEX_NO_LOCKSTEP);
    const int fwarps = lockstep ? (records ? kFRecLockWarps : 24) : kFWarps;
    const size_t fsmem = (size_t)fwarps * (records ? kFWarpSmemRec : kFWarpSmemHist);
    int64_t fctas = (d->n_segs + fwarps - 1) / fwarps;
    const int64_t fmax = lockstep ? (int64_t)ctx->sm_count * (records ? kFRecCtasPerSm : 1) : (int64_t)ctx->sm_count * (records ? 4 : 6);
    if (fctas > fmax) fctas = fmax;
#define FFB_LAUNCH_FAST(R, L)                                                                                          \
    do {                                                                                                               \
      FFB_CUDA(ctx, cudaFuncSetAttribute(lex_fast_kernel<R, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem)); \
      FFB_LAUNCH((lex_fast_kernel<R, L>), (unsigned)fctas, fwarps * 32, fsmem, stream, f);                               \
    } while (0)
    if (records) { if (lockstep) FFB_LAUNCH_FAST(true, true); else FFB_LAUNCH_FAST(true, false); }
    else { if (lockstep) FFB_LAUNCH_FAST(false, true); else FFB_LAUNCH_FAST(false, false); }
#undef FFB_LAUNCH_FAST
    rc = ffb_check_launch(ctx, "lex_fast_kernel");
    if (rc) return rc;
    // the exact kernel takes what the fast path declined (count and list stay on the device)
    a.order = f.fb_list; a.n_work = f.fb_count;
  }
  // the exact walk is launched barrier-paced as well (one CTA per SM): 16 warps at 128 registers in record mode,
  // 32 at 64 in histogram mode; FFB_LEX_NO_LOCKSTEP keeps the small independent CTAs
  const bool xlock = !(d->flags & FFB_LEX_NO_LOCKSTEP);
  const int xwarps = xlock ? (records ? 16 : 32) : kWarps;
  const size_t smem = (size_t)xwarps * kWarpSmem;
  int64_t ctas = (d->n_segs + xwarps - 1) / xwarps;
  const int64_t max_ctas = xlock ? (int64_t)ctx->sm_count : (int64_t)ctx->sm_count * 4;
  if (ctas > max_ctas) ctas = max_ctas;
#define FFB_LAUNCH_EXACT(R, L)                                                                                           \
  do {                                                                                                                   \
    FFB_CUDA(ctx, cudaFuncSetAttribute(lex_corpus_kernel<R, L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    FFB_LAUNCH((lex_corpus_kernel<R, L>), (unsigned)ctas, xwarps * 32, smem, stream, a);                                   \
  } while (0)
  if (records) { if (xlock) FFB_LAUNCH_EXACT(true, true); else FFB_LAUNCH_EXACT(true, false); }
  else { if (xlock) FFB_LAUNCH_EXACT(false, true); else FFB_LAUNCH_EXACT(false, false); }
#undef FFB_LAUNCH_EXACT
  rc = ffb_check_launch(ctx, "lex_corpus_kernel");
  if (rc) return rc;
  if (d->d_path_counts) {
    // [0] = segments the fast path finished, [1] = segments the exact walk finished
    FFB_LAUNCH(lex_path_counts_kernel, 1, 32, 0, stream, fast ? (const unsigned long long*)ctx->d_lex.p + 1 : nullptr, d->n_segs, d->d_path_counts);
    rc = ffb_check_launch(ctx, "lex_path_counts_kernel");
  }
  return rc;
}

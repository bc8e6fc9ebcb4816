// Streamed batched SpTRSV for exact / ILU(k) factors (trisolve_levelset,
// local_solvers.py:404-410, over trisolve_forward_unit / trisolve_backward,
// _kernels.py:473-496).
//
// One CTA per subdomain. The subdomain's L then U factor are serialised on
// the host into ONE contiguous byte stream of level-ordered chunks (tables,
// values, 16-bit or 32-bit block-local columns, U's diagonal). A producer
// warp streams the chunks with TMA bulk copies (cp.async.bulk) into a
// shared-memory ring guarded by full/empty mbarriers; eight consumer warps
// solve each chunk from shared memory against the block iterate (shared
// memory when it fits, else global) and meet at one named barrier per
// chunk -- a level never spans a barrier-free chunk boundary. The factor
// bytes are read from HBM exactly once per solve, ahead of the dependency
// chain, so a level costs a barrier plus on-chip work.
//
// Work in a chunk:
//  * short rows (<= TR_SHORT entries): one thread per row, SELL-32 slices
//    (entry k of lane l at 32k + l), sequential round-to-nearest mul/sub in
//    column order -- bit-identical to the reference;
//  * medium rows (<= TR_SEG entries): one warp per row, products in
//    parallel, subtraction chain in column order (bit-identical);
//  * long rows: TR_SEG-entry segments, one warp each, fused products and a
//    fixed shuffle tree; after a barrier the first segment's thread combines
//    the partials in segment order -- deterministic, within 1e-13 relative
//    of sequential substitution (exact factors use the tree for medium rows
//    too; ILU(k) keeps the sequential chain).
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace gdsw {

// consumer warps per CTA: a template parameter NW (8, 16 or 32) of the
// kernel, plus one TMA producer warp
constexpr int TR_SHORT = 32;
// previous-chunk forwarding: short-row results of a chunk are also kept in
// shared memory (slot = position in the chunk), and the next chunk reads
// them there instead of from the global iterate (freshly stored values miss
// L1, so every level would pay an L2 round trip)
constexpr int TR_FWD = 1024;
constexpr uint16_t TR_NOFWD = 0xFFFFu;
constexpr int TR_SEG = 128;
constexpr int TR_MAXW = 64;                     // warp tasks per chunk
constexpr int TR_CHUNK_MIN = 16 * 1024;
constexpr int TR_SN_MIN = 32;                   // rows of a supernode worth a dense block
constexpr int TR_SN_HDR = 48;                   // header bytes of a supernode chunk
enum TrChunkType : int { TR_ROWS = 0, TR_SN_GEMV = 1, TR_SN_DIAG = 2, TR_SN_UPD = 3 };

__host__ __device__ inline int64_t ts_al16(int64_t b) { return (b + 15) & ~int64_t(15); }

// section offsets of a chunk holding nw warp tasks and nsl short slices
struct ChunkLayout {
  int32_t wtab, wgrp, wdiag, stab, srow, slen, sdiag, data;
  __host__ __device__ ChunkLayout(int nw, int nsl, bool up, int vsize) {
    wtab = 16;
    wgrp = wtab + 16 * nw;
    wdiag = (int32_t)ts_al16(wgrp + 8 * nw);
    stab = (int32_t)ts_al16(wdiag + (up ? vsize * nw : 0));
    srow = stab + 16 * nsl;
    slen = srow + 128 * nsl;
    sdiag = slen + 128 * nsl;
    data = (int32_t)ts_al16(sdiag + (up ? 32 * vsize * nsl : 0));
  }
};

struct TriStreamDev {
  const unsigned char* bytes = nullptr;
  const int32_t* ch_sub = nullptr;   // [n_sub + 1] chunk range of each subdomain (L chunks, then U)
  const int64_t* ch_off = nullptr;   // byte offset of each chunk
  const int32_t* ch_len = nullptr;   // bytes of each chunk (multiple of 16)
  int32_t chunk_max = 0;
};

// ---------------------------------------------------------------------------
// host-side serialisation (values are placed on the device: k_stream_place)
// ---------------------------------------------------------------------------
struct TriStream {
  int64_t total = 0, n_chunks = 0, max_rows = 0;
  int32_t chunk_max = 0;
  int vsize = 8, csize = 4;
  bool fwd = false;  // slices carry forwarding slots (iterate too large for shared memory)
  DBuf<unsigned char> bytes;
  DBuf<int32_t> ch_sub, ch_len;
  DBuf<int64_t> ch_off;
  // value placement: element (vsize) offsets into the stream
  DBuf<int64_t> pl_src, pl_dst;
  DBuf<int32_t> pl_len, pl_stride;
  int64_t n_place = 0;

  struct Fac {
    const std::vector<int64_t>* ptr;
    const std::vector<int64_t>* idx;
    const std::vector<int64_t>* lsub;
    const std::vector<int64_t>* lptr;
    const std::vector<int64_t>* lrows;
    int skip;  // 1: U (diagonal first, stored separately)
  };

  // bitwise: medium rows keep the reference's sequential subtraction order
  // (ILU(k)); exact factors use a shuffle tree there (compared at 1e-13)
  void build(int32_t n_sub, const std::vector<int64_t>& sub_ptr, const Fac& L, const Fac& U, int vsize_,
             bool bitwise) {
    vsize = vsize_;
    const int64_t nnz_l = L.ptr->back();
    max_rows = 0;
    int64_t max_row_len = 0;
    for (int32_t s = 0; s < n_sub; ++s) max_rows = std::max<int64_t>(max_rows, sub_ptr[s + 1] - sub_ptr[s]);
    csize = max_rows <= 65536 ? 2 : 4;
    for (const Fac* f : {&L, &U})
      for (int64_t g = 0; g + 1 < (int64_t)f->ptr->size(); ++g)
        max_row_len = std::max<int64_t>(max_row_len, (*f->ptr)[g + 1] - (*f->ptr)[g] - f->skip);
    // a chunk must hold the longest row (all its segments) with its tables
    const int64_t nseg_max = (max_row_len + TR_SEG - 1) / TR_SEG;
    require(nseg_max <= TR_MAXW, "factor row too long for the streamed SpTRSV");
    const int64_t need = ChunkLayout((int)nseg_max, 0, true, vsize).data +
                         nseg_max * (ts_al16(TR_SEG * (int64_t)vsize) + ts_al16(TR_SEG * (int64_t)csize));
    // measured on B200: with at most one block per SM, 48 KB chunks (and the
    // larger ring they imply) are faster (C2 ILU(0) 0.46 -> 0.39 ms, C1
    // 0.91 -> 0.86 ms, 64 C3-sized blocks 1.71 -> 1.51 ms per solve); with
    // more blocks than SMs, 16 KB keeps two CTAs per SM (512 C3 blocks:
    // 3.4 ms vs 5.6 ms with 32 KB)
    static const int64_t chunk_env = [] {
      const char* e = std::getenv("GDSW_TS_CHUNK_KB");
      return e ? (int64_t)std::atoi(e) * 1024 : (int64_t)0;
    }();
    const int64_t chunk_min = chunk_env ? chunk_env : (n_sub > num_sms() ? TR_CHUNK_MIN : 3 * TR_CHUNK_MIN);
    chunk_max = (int32_t)ts_al16(std::max<int64_t>(chunk_min, need));
    // the iterate cannot sit in shared memory next to a 3-chunk ring: the
    // slices carry forwarding slots (GDSW_TS_NOFWD=1 disables)
    {
      const char* e = std::getenv("GDSW_TS_NOFWD");
      fwd = max_rows * vsize + 3 * (int64_t)chunk_max > 220 * 1024 && !(e && std::atoi(e) != 0);
    }
    std::vector<int32_t> ch_of, slot_of;  // chunk / slot of each short row of the current pass

    std::vector<unsigned char> buf;
    std::vector<int32_t> h_ch_sub(n_sub + 1), h_ch_len;
    std::vector<int64_t> h_ch_off, p_src, p_dst;
    std::vector<int32_t> p_len, p_stride;

    struct SN { int64_t a, k, m; };
    // one chunk under construction
    struct WT { int32_t row, len, first, nseg; int64_t src; int64_t diag_src; };
    struct SL { std::vector<int32_t> rows, lens; std::vector<int64_t> srcs, dsrc; int32_t width; };
    std::vector<WT> wts;
    std::vector<SL> sls;
    int64_t data_bytes = 0;
    bool up = false;
    auto cur_bytes = [&](size_t nw, size_t nsl, int64_t db) {
      return (int64_t)ChunkLayout((int)nw, (int)nsl, up, vsize).data + db;
    };
    auto flush = [&]() {
      if (wts.empty() && sls.empty()) return;
      const int nw = (int)wts.size(), nsl = (int)sls.size();
      ChunkLayout cl(nw, nsl, up, vsize);
      const int64_t off = (int64_t)buf.size();
      const int64_t len = cl.data + data_bytes;
      require(len <= chunk_max, "internal: chunk overflow");
      buf.resize(off + len, 0);
      unsigned char* c = buf.data() + off;
      auto put32 = [&](int64_t at, int32_t v) { std::memcpy(c + at, &v, 4); };
      put32(0, nw);
      put32(4, nsl);
      bool multi = false;
      for (const WT& w : wts) multi = multi || w.nseg > 1;
      put32(8, (up ? 1 : 0) | (bitwise ? 2 : 0) | (multi ? 4 : 0));
      int64_t dp = cl.data;
      const std::vector<int64_t>& idx = *(up ? U.idx : L.idx);
      auto put_cols = [&](int64_t at, int64_t src, int32_t n, int32_t stride) {
        for (int32_t k = 0; k < n; ++k) {
          const int64_t v = idx[src + k];
          if (csize == 2) {
            const uint16_t h = (uint16_t)v;
            std::memcpy(c + at + (int64_t)k * stride * 2, &h, 2);
          } else {
            const int32_t h = (int32_t)v;
            std::memcpy(c + at + (int64_t)k * stride * 4, &h, 4);
          }
        }
      };
      for (int t = 0; t < nw; ++t) {
        const WT& w = wts[t];
        const int64_t voff = dp;
        dp += ts_al16((int64_t)w.len * vsize);
        const int64_t coff = dp;
        dp += ts_al16((int64_t)w.len * csize);
        put32(cl.wtab + 16 * t + 0, w.row);
        put32(cl.wtab + 16 * t + 4, w.len);
        put32(cl.wtab + 16 * t + 8, (int32_t)voff);
        put32(cl.wtab + 16 * t + 12, (int32_t)coff);
        put32(cl.wgrp + 8 * t + 0, w.first);
        put32(cl.wgrp + 8 * t + 4, w.nseg);
        put_cols(coff, w.src, w.len, 1);
        p_src.push_back(w.src + (up ? nnz_l : 0));
        p_dst.push_back((off + voff) / vsize);
        p_len.push_back(w.len);
        p_stride.push_back(1);
        if (up && w.diag_src >= 0) {
          p_src.push_back(w.diag_src + nnz_l);
          p_dst.push_back((off + cl.wdiag + (int64_t)vsize * t) / vsize);
          p_len.push_back(1);
          p_stride.push_back(1);
        }
      }
      for (int q = 0; q < nsl; ++q) {
        const SL& sl = sls[q];
        const int64_t voff = dp;
        dp += ts_al16((int64_t)32 * sl.width * vsize);
        const int64_t coff = dp;
        dp += ts_al16((int64_t)32 * sl.width * csize);
        put32(cl.stab + 16 * q + 0, (int32_t)voff);
        put32(cl.stab + 16 * q + 4, (int32_t)coff);
        put32(cl.stab + 16 * q + 8, sl.width);
        if (fwd) {
          // slot of each entry's column in the previous chunk, or TR_NOFWD
          const int64_t foff = dp;
          dp += ts_al16((int64_t)32 * sl.width * 2);
          put32(cl.stab + 16 * q + 12, (int32_t)foff);
          const int32_t prev = (int32_t)h_ch_off.size() - 1;
          for (int64_t k = 0; k < (int64_t)32 * sl.width; ++k) std::memcpy(c + foff + 2 * k, &TR_NOFWD, 2);
          for (int l = 0; l < (int)sl.rows.size(); ++l)
            for (int32_t k = 0; k < sl.lens[l]; ++k) {
              const int64_t col = idx[sl.srcs[l] + k];
              if (ch_of[col] == prev && slot_of[col] >= 0 && slot_of[col] < TR_FWD) {
                const uint16_t f = (uint16_t)slot_of[col];
                std::memcpy(c + foff + 2 * ((int64_t)32 * k + l), &f, 2);
              }
            }
        }
        for (int l = 0; l < 32; ++l) {
          const bool ok = l < (int)sl.rows.size();
          put32(cl.srow + 4 * (32 * q + l), ok ? sl.rows[l] : 0);
          put32(cl.slen + 4 * (32 * q + l), ok ? sl.lens[l] : -1);
          if (!ok) continue;
          if (sl.lens[l] > 0) {
            put_cols(coff + (int64_t)csize * l, sl.srcs[l], sl.lens[l], 32);
            p_src.push_back(sl.srcs[l] + (up ? nnz_l : 0));
            p_dst.push_back((off + voff) / vsize + l);
            p_len.push_back(sl.lens[l]);
            p_stride.push_back(32);
          }
          if (up) {
            p_src.push_back(sl.dsrc[l] + nnz_l);
            p_dst.push_back((off + cl.sdiag + (int64_t)vsize * (32 * q + l)) / vsize);
            p_len.push_back(1);
            p_stride.push_back(1);
          }
        }
      }
      require(dp == len, "internal: chunk layout mismatch");
      if (fwd)
        for (int q = 0; q < nsl; ++q)
          for (int l = 0; l < (int)sls[q].rows.size(); ++l) {
            ch_of[sls[q].rows[l]] = (int32_t)h_ch_off.size();
            slot_of[sls[q].rows[l]] = 32 * q + l;
          }
      h_ch_off.push_back(off);
      h_ch_len.push_back((int32_t)len);
      wts.clear();
      sls.clear();
      data_bytes = 0;
    };

    // supernode [a, a+k) with external pattern of m columns, solved in
    // order q = 0..k-1 over rows a + q (L) or a + k - 1 - q (U):
    //  GEMV chunks  x[row_q] -= V_q . x[E]           (rows [q0, q0+nq), row-major)
    //  DIAG chunk   32-row diagonal tile, one warp    (tile column-major 32x32)
    //  UPD chunks   x[row_q] -= P_q . x[block]       (rows below, panel column-major)
    auto emit_sn = [&](const SN& sn, int64_t base, const std::vector<int64_t>& ptr,
                       const std::vector<int64_t>& idx, int skip) {
      flush();
      const bool U = skip == 1;
      const int64_t k = sn.k, m = sn.m, V = vsize;
      const int32_t brow = (int32_t)(U ? sn.a + k - 1 : sn.a), dir = U ? -1 : 1;
      const int64_t uoff = U ? nnz_l : 0;
      auto grow = [&](int64_t q) { return base + (U ? sn.a + k - 1 - q : sn.a + q); };
      // src position of the entry of row q on triangle column q' (< q)
      auto tri_src = [&](int64_t q, int64_t qp) {
        const int64_t g = grow(q);
        return U ? ptr[g] + (q - qp) : ptr[g] + m + qp;
      };
      auto new_chunk = [&](int64_t bytes, int type, const int32_t* h1, const int32_t* h2) {
        const int64_t off = (int64_t)buf.size();
        const int64_t len = ts_al16(bytes);
        require(len <= chunk_max, "internal: supernode chunk overflow");
        buf.resize(off + len, 0);
        unsigned char* c = buf.data() + off;
        const int32_t h0[4] = {0, 0, U ? 1 : 0, type};
        std::memcpy(c, h0, 16);
        std::memcpy(c + 16, h1, 16);
        std::memcpy(c + 32, h2, 16);
        h_ch_off.push_back(off);
        h_ch_len.push_back((int32_t)len);
        return off;
      };
      auto place = [&](int64_t src, int64_t dst_byte, int32_t len, int32_t stride) {
        if (len <= 0) return;
        p_src.push_back(src);
        p_dst.push_back(dst_byte / V);
        p_len.push_back(len);
        p_stride.push_back(stride);
      };
      // GEMV over the external pattern
      if (m > 0) {
        const int64_t eb = ts_al16(m * csize);
        const int64_t nq_max = std::max<int64_t>(1, (chunk_max - TR_SN_HDR - eb) / (m * V));
        require(TR_SN_HDR + eb + m * V <= chunk_max, "supernode pattern too wide for a chunk");
        for (int64_t q0 = 0; q0 < k; q0 += nq_max) {
          const int64_t nq = std::min(nq_max, k - q0);
          const int32_t h1[4] = {brow, dir, (int32_t)q0, (int32_t)nq};
          const int32_t h2[4] = {(int32_t)m, TR_SN_HDR, (int32_t)(TR_SN_HDR + eb), 0};
          const int64_t off = new_chunk(TR_SN_HDR + eb + nq * m * V, TR_SN_GEMV, h1, h2);
          unsigned char* c = buf.data() + off;
          // E = the external columns of the first-solved row
          const int64_t g0 = grow(0);
          for (int64_t p = 0; p < m; ++p) {
            const int64_t col = idx[ptr[g0] + skip + p];
            if (csize == 2) {
              const uint16_t h = (uint16_t)col;
              std::memcpy(c + TR_SN_HDR + 2 * p, &h, 2);
            } else {
              const int32_t h = (int32_t)col;
              std::memcpy(c + TR_SN_HDR + 4 * p, &h, 4);
            }
          }
          for (int64_t q = q0; q < q0 + nq; ++q) {
            const int64_t g = grow(q);
            const int64_t src = U ? ptr[g] + 1 + q : ptr[g];
            place(uoff + src, off + TR_SN_HDR + eb + (q - q0) * m * V, (int32_t)m, 1);
          }
        }
      }
      // dense triangle, 32-row blocks
      for (int64_t jb = 0; jb < k; jb += 32) {
        const int64_t nb = std::min<int64_t>(32, k - jb);
        {
          const int32_t h1[4] = {brow, dir, (int32_t)jb, (int32_t)nb};
          const int32_t h2[4] = {TR_SN_HDR, U ? (int32_t)(TR_SN_HDR + 32 * 32 * V) : 0, 0, 0};
          const int64_t off = new_chunk(TR_SN_HDR + 32 * 32 * V + (U ? 32 * V : 0), TR_SN_DIAG, h1, h2);
          for (int64_t l = 0; l < nb; ++l) {
            const int64_t q = jb + l;
            if (l > 0) {
              if (!U) place(tri_src(q, jb), off + TR_SN_HDR + l * V, (int32_t)l, 32);
              else place(uoff + tri_src(q, q - 1), off + TR_SN_HDR + ((l - 1) * 32 + l) * V, (int32_t)l, -32);
            }
            if (U) place(uoff + ptr[grow(q)], off + TR_SN_HDR + 32 * 32 * V + l * V, 1, 1);
          }
        }
        const int64_t rest = k - jb - nb;
        if (rest <= 0) continue;
        const int64_t nq_max = std::max<int64_t>(1, (chunk_max - TR_SN_HDR) / (nb * V));
        for (int64_t q0 = jb + nb; q0 < k; q0 += nq_max) {
          const int64_t nq = std::min(nq_max, k - q0);
          const int32_t h1[4] = {brow, dir, (int32_t)jb, (int32_t)nb};
          const int32_t h2[4] = {(int32_t)q0, (int32_t)nq, TR_SN_HDR, 0};
          const int64_t off = new_chunk(TR_SN_HDR + nb * nq * V, TR_SN_UPD, h1, h2);
          for (int64_t q = q0; q < q0 + nq; ++q) {
            if (!U) place(tri_src(q, jb), off + TR_SN_HDR + (q - q0) * V, (int32_t)nb, (int32_t)nq);
            else
              place(uoff + tri_src(q, jb + nb - 1), off + TR_SN_HDR + ((nb - 1) * nq + (q - q0)) * V, (int32_t)nb,
                    -(int32_t)nq);
          }
        }
      }
    };

    for (int32_t s = 0; s < n_sub; ++s) {
      h_ch_sub[s] = (int32_t)h_ch_off.size();
      const int64_t base = sub_ptr[s];
      for (const Fac* f : {&L, &U}) {
        up = f->skip == 1;
        const std::vector<int64_t>& ptr = *f->ptr;
        const int64_t n_s = sub_ptr[s + 1] - base;
        const std::vector<int64_t>& idx = *f->idx;
        if (fwd) {
          ch_of.assign(n_s, -1);
          slot_of.assign(n_s, -1);
        }
        auto rlen = [&](int64_t i) { return ptr[base + i + 1] - ptr[base + i] - f->skip; };
        auto rcol = [&](int64_t i, int64_t k) { return idx[ptr[base + i] + f->skip + k]; };
        // supernodes: runs of rows whose patterns nest by one (dense diagonal
        // block, shared external pattern); L: row i = row i-1 + {i-1};
        // U: row i = {i+1} + row i+1
        std::vector<SN> sns;
        std::vector<int32_t> sn_of(n_s, -1);
        {
          auto nests = [&](int64_t i, int64_t prev) {  // row i extends row prev by one
            const int64_t li = rlen(i), lp = rlen(prev);
            if (li != lp + 1) return false;
            if (!up) {
              if (rcol(i, li - 1) != prev) return false;
              for (int64_t k = 0; k < lp; ++k)
                if (rcol(i, k) != rcol(prev, k)) return false;
            } else {
              if (rcol(i, 0) != prev) return false;
              for (int64_t k = 0; k < lp; ++k)
                if (rcol(i, k + 1) != rcol(prev, k)) return false;
            }
            return true;
          };
          int64_t i = 0;
          while (i < n_s) {
            int64_t j = i + 1;
            if (!up) {
              while (j < n_s && nests(j, j - 1)) ++j;
            } else {
              while (j < n_s && nests(j - 1, j)) ++j;
            }
            if (!bitwise && j - i >= TR_SN_MIN) {
              SN sn{i, j - i, up ? rlen(j - 1) : rlen(i)};
              for (int64_t r = i; r < j; ++r) sn_of[r] = (int32_t)sns.size();
              sns.push_back(sn);
            }
            i = j;
          }
        }
        // unit levels (a supernode is one unit)
        std::vector<int32_t> lev(n_s, 0);
        int32_t nlev = 0;
        auto unit_level = [&](int64_t i) {
          int32_t lv = 0;
          for (int64_t k = 0, l = rlen(i); k < l; ++k) {
            const int64_t c = rcol(i, k);
            if (sn_of[i] >= 0 && sn_of[c] == sn_of[i]) continue;
            lv = std::max(lv, lev[c] + 1);
          }
          return lv;
        };
        for (int64_t t = 0; t < n_s; ++t) {
          const int64_t i = up ? n_s - 1 - t : t;
          const int32_t q = sn_of[i];
          if (q >= 0 && i != (up ? sns[q].a + sns[q].k - 1 : sns[q].a)) {
            lev[i] = lev[up ? sns[q].a + sns[q].k - 1 : sns[q].a];
            continue;
          }
          lev[i] = unit_level(i);
          nlev = std::max(nlev, lev[i] + 1);
        }
        std::vector<std::vector<int64_t>> lrows_of(nlev);
        std::vector<std::vector<int32_t>> lsn_of(nlev);
        for (int64_t t = 0; t < n_s; ++t) {
          const int64_t i = up ? n_s - 1 - t : t;
          const int32_t q = sn_of[i];
          if (q < 0) lrows_of[lev[i]].push_back(i);
          else if (i == (up ? sns[q].a + sns[q].k - 1 : sns[q].a)) lsn_of[lev[i]].push_back(q);
        }
        for (int32_t lv = 0; lv < nlev; ++lv) {
          for (int32_t q : lsn_of[lv]) emit_sn(sns[q], base, ptr, idx, f->skip);
          std::vector<int64_t> shorts;
          for (const int64_t row : lrows_of[lv]) {
            const int64_t g = base + row;
            const int64_t len = ptr[g + 1] - ptr[g] - f->skip;
            if (len <= TR_SHORT) {
              shorts.push_back(row);
              continue;
            }
            const int32_t nseg = (int32_t)((len + TR_SEG - 1) / TR_SEG);
            int64_t db = 0;
            for (int32_t q = 0; q < nseg; ++q) {
              const int64_t sl = std::min<int64_t>(TR_SEG, len - (int64_t)q * TR_SEG);
              db += ts_al16(sl * vsize) + ts_al16(sl * csize);
            }
            if (wts.size() + nseg > (size_t)TR_MAXW ||
                cur_bytes(wts.size() + nseg, sls.size(), data_bytes + db) > chunk_max)
              flush();
            const int32_t first = (int32_t)wts.size();
            for (int32_t q = 0; q < nseg; ++q) {
              const int64_t sl = std::min<int64_t>(TR_SEG, len - (int64_t)q * TR_SEG);
              wts.push_back(WT{(int32_t)row, (int32_t)sl, first, nseg, ptr[g] + f->skip + (int64_t)q * TR_SEG,
                               (q == 0 && up) ? ptr[g] : -1});
            }
            data_bytes += db;
          }
          for (size_t s0 = 0; s0 < shorts.size(); s0 += 32) {
            SL sl;
            sl.width = 0;
            for (size_t q = s0; q < std::min(shorts.size(), s0 + 32); ++q) {
              const int64_t g = base + shorts[q];
              const int32_t len = (int32_t)(ptr[g + 1] - ptr[g] - f->skip);
              sl.rows.push_back((int32_t)shorts[q]);
              sl.lens.push_back(len);
              sl.srcs.push_back(ptr[g] + f->skip);
              sl.dsrc.push_back(ptr[g]);
              sl.width = std::max(sl.width, len);
            }
            const int64_t db = ts_al16((int64_t)32 * sl.width * vsize) + ts_al16((int64_t)32 * sl.width * csize) +
                               (fwd ? ts_al16((int64_t)32 * sl.width * 2) : 0);
            if (cur_bytes(wts.size(), sls.size() + 1, data_bytes + db) > chunk_max) flush();
            sls.push_back(std::move(sl));
            data_bytes += db;
          }
          flush();  // a level ends a chunk (its barrier is the level barrier)
        }
      }
    }
    h_ch_sub[n_sub] = (int32_t)h_ch_off.size();
    total = (int64_t)buf.size();
    n_chunks = (int64_t)h_ch_off.size();
    bytes.upload(buf.data(), std::max<size_t>(buf.size(), 16));
    ch_sub.upload(h_ch_sub);
    ch_off.upload(h_ch_off);
    ch_len.upload(h_ch_len);
    pl_src.upload(p_src);
    pl_dst.upload(p_dst);
    pl_len.upload(p_len);
    pl_stride.upload(p_stride);
    n_place = (int64_t)p_src.size();
  }
  TriStreamDev view() const {
    TriStreamDev v;
    v.bytes = bytes.p;
    v.ch_sub = ch_sub.p;
    v.ch_off = ch_off.p;
    v.ch_len = ch_len.p;
    v.chunk_max = chunk_max;
    return v;
  }
};

// CSR values (and U's diagonal) -> their stream slots. Sources index the
// concatenation [L values | U values].
template <typename T>
__global__ void k_stream_place(int64_t n_place, const int64_t* __restrict__ src, const int64_t* __restrict__ dst,
                               const int32_t* __restrict__ len, const int32_t* __restrict__ stride,
                               const T* __restrict__ lval, const T* __restrict__ uval, int64_t nnz_l,
                               T* __restrict__ out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (q >= n_place) return;
  int64_t s0 = src[q];
  const T* v = lval;
  if (s0 >= nnz_l) {
    v = uval;
    s0 -= nnz_l;
  }
  const int64_t d0 = dst[q];
  const int32_t n = len[q], st = stride[q];
  for (int32_t k = threadIdx.x; k < n; k += blockDim.x) out[d0 + (int64_t)k * st] = v[s0 + k];
}

template <int NW>
__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(32 * NW) : "memory");
}

// ---------------------------------------------------------------------------
// chunk solve
// ---------------------------------------------------------------------------
// supernode chunks (dense blocks of exact-LU separators). Rows are indexed
// in solve order q: row(q) = brow + dir * q.
template <typename T, typename CT, int NW>
__device__ __forceinline__ void ts_sn_chunk(const unsigned char* __restrict__ c, int type, bool up, T* x) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int4 h1 = *reinterpret_cast<const int4*>(c + 16);
  const int4 h2 = *reinterpret_cast<const int4*>(c + 32);
  const int32_t brow = h1.x, dir = h1.y;
  if (type == TR_SN_GEMV) {
    // x[row_q] -= V_q . x[E], one warp per row, lanes over the pattern
    const int32_t q0 = h1.z, nq = h1.w, m = h2.x;
    const CT* E = reinterpret_cast<const CT*>(c + h2.y);
    const T* V = reinterpret_cast<const T*>(c + h2.z);
    for (int t = warp; t < nq; t += NW) {
      const T* v = V + (int64_t)t * m;
      T acc = T(0);
#pragma unroll 4
      for (int p = lane; p < m; p += 32) acc = fma(v[p], x[E[p]], acc);
      acc = warp_sum(acc);
      if (lane == 0) {
        const int32_t row = brow + dir * (q0 + t);
        x[row] = x[row] - acc;
      }
    }
  } else if (type == TR_SN_DIAG) {
    // 32-row diagonal tile: lane l owns row jb + l; column j is final after
    // the updates of columns < j (U: then divided by its diagonal)
    if (warp != 0) return;
    const int32_t jb = h1.z, nb = h1.w;
    const T* tile = reinterpret_cast<const T*>(c + h2.x);
    const T* dg = up ? reinterpret_cast<const T*>(c + h2.y) : nullptr;
    const int32_t row = brow + dir * (jb + lane);
    T t = lane < nb ? x[row] : T(0);
    for (int j = 0; j < nb; ++j) {
      if (up && lane == j) t = t / dg[j];
      const T xj = __shfl_sync(0xffffffffu, t, j);
      if (lane > j && lane < nb) t = fma(-tile[j * 32 + lane], xj, t);
    }
    if (lane < nb) x[row] = t;
  } else {
    // x[row_q] -= P_q . x[block jb], thread per row, panel column-major
    const int32_t jb = h1.z, nb = h1.w, q0 = h2.x, nq = h2.y;
    const T* P = reinterpret_cast<const T*>(c + h2.z);
    for (int t = threadIdx.x; t < nq; t += (32 * NW)) {
      T acc = T(0);
      for (int j = 0; j < nb; ++j) acc = fma(P[(int64_t)j * nq + t], x[brow + dir * (jb + j)], acc);
      const int32_t row = brow + dir * (q0 + t);
      x[row] = x[row] - acc;
    }
  }
}

template <typename T, typename CT, bool FWD, int NW>
__device__ __forceinline__ void ts_chunk(const unsigned char* __restrict__ c, T* x, T* part, const T* fprev,
                                         T* fcur) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int4 hdr = *reinterpret_cast<const int4*>(c);
  if (hdr.w != TR_ROWS) {
    ts_sn_chunk<T, CT, NW>(c, hdr.w, hdr.z & 1, x);
    return;
  }
  const int nw = hdr.x, nsl = hdr.y;
  const bool up = hdr.z & 1, ordered = hdr.z & 2;
  const ChunkLayout cl(nw, nsl, up, (int)sizeof(T));
  // warp tasks (medium rows and segments of long rows)
  for (int t = warp; t < nw; t += NW) {
    const int4 w = *reinterpret_cast<const int4*>(c + cl.wtab + 16 * t);
    const int2 gp = *reinterpret_cast<const int2*>(c + cl.wgrp + 8 * t);
    const int32_t row = w.x, len = w.y;
    const T* v = reinterpret_cast<const T*>(c + w.z);
    const CT* cc = reinterpret_cast<const CT*>(c + w.w);
    T p[TR_SEG / 32];
#pragma unroll
    for (int u = 0; u < TR_SEG / 32; ++u) {
      const int k = lane + 32 * u;
      p[u] = k < len ? rn_mul(v[k], x[cc[k]]) : T(0);
    }
    if (gp.y == 1 && !ordered) {
      // whole row in one segment, fixed tree
      T acc = T(0);
#pragma unroll
      for (int u = 0; u < TR_SEG / 32; ++u) acc += p[u];
      acc = warp_sum(acc);
      if (lane == 0) {
        T xi = x[row] - acc;
        if (up) xi = rn_div(xi, reinterpret_cast<const T*>(c + cl.wdiag)[t]);
        x[row] = xi;
      }
    } else if (gp.y == 1) {
      // whole row in one segment: subtraction chain in column order
      T xi = x[row];
#pragma unroll
      for (int u = 0; u < TR_SEG / 32; ++u) {
        if (32 * u >= len) break;  // warp-uniform
#pragma unroll
        for (int l = 0; l < 32; ++l) {
          const T pk = __shfl_sync(0xffffffffu, p[u], l);
          if (32 * u + l < len) xi = rn_sub(xi, pk);
        }
      }
      if (up) xi = rn_div(xi, reinterpret_cast<const T*>(c + cl.wdiag)[t]);
      if (lane == 0) x[row] = xi;
    } else {
      T acc = T(0);
#pragma unroll
      for (int u = 0; u < TR_SEG / 32; ++u) acc += p[u];
      acc = warp_sum(acc);
      if (lane == 0) part[t] = acc;  // combined after the barrier below
    }
  }
  // short rows: one thread each, sequential in column order
  const int32_t* srow = reinterpret_cast<const int32_t*>(c + cl.srow);
  const int32_t* slen = reinterpret_cast<const int32_t*>(c + cl.slen);
  for (int t = threadIdx.x; t < 32 * nsl; t += (32 * NW)) {
    const int32_t len = slen[t];
    if (len < 0) continue;
    const int32_t row = srow[t];
    const int4 st = *reinterpret_cast<const int4*>(c + cl.stab + 16 * (t >> 5));
    const T* v = reinterpret_cast<const T*>(c + st.x) + (t & 31);
    const CT* cc = reinterpret_cast<const CT*>(c + st.y) + (t & 31);
    const uint16_t* fs = FWD ? reinterpret_cast<const uint16_t*>(c + st.w) + (t & 31) : nullptr;
    T acc = x[row];
    for (int k0 = 0; k0 < len; k0 += 4) {
      T pv[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (k0 + u < len) {
          pv[u] = v[32 * (k0 + u)];
          if (FWD) {
            const uint16_t f = fs[32 * (k0 + u)];
            xv[u] = f != TR_NOFWD ? fprev[f] : x[cc[32 * (k0 + u)]];
          } else {
            xv[u] = x[cc[32 * (k0 + u)]];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (k0 + u < len) acc = rn_sub(acc, rn_mul(pv[u], xv[u]));
    }
    if (up) acc = rn_div(acc, reinterpret_cast<const T*>(c + cl.sdiag)[t]);
    x[row] = acc;
    if (FWD && t < TR_FWD) fcur[t] = acc;
  }
  if (hdr.z & 4) {
    // rows split in segments: partials summed in segment order by the
    // thread of the first segment once every segment is in
    consumer_bar<NW>();
    for (int t = threadIdx.x; t < nw; t += (32 * NW)) {
      const int2 gp = *reinterpret_cast<const int2*>(c + cl.wgrp + 8 * t);
      if (gp.y < 2 || gp.x != t) continue;
      const int32_t row = reinterpret_cast<const int4*>(c + cl.wtab)[t].x;
      T sum = T(0);
      for (int q = 0; q < gp.y; ++q) sum += part[t + q];
      T xi = x[row] - sum;
      if (up) xi = rn_div(xi, reinterpret_cast<const T*>(c + cl.wdiag)[t]);
      x[row] = xi;
    }
  }
}

// one CTA per subdomain: gather (ordering folded into gmap), every chunk of
// L then U streamed through a byte ring (chunks packed back to back, up to
// TR_NT in flight; a chunk never wraps), block solution written to y
constexpr int TR_NT = 16;

template <typename T, typename CT, bool SMEMX, bool FWD, int NW>
__global__ void __launch_bounds__(32 * NW + 32) k_trisolve_stream(TriStreamDev S, int32_t ring_bytes,
                                                                    const int32_t* __restrict__ sub_ptr,
                                                                    const int32_t* __restrict__ gmap,
                                                                    const double* __restrict__ r,
                                                                    T* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char ts_sm[];
  __shared__ uint64_t full[TR_NT], empty[TR_NT];
  __shared__ int32_t pos[TR_NT], foot[TR_NT];
  __shared__ T part[TR_MAXW];
  __shared__ T fwdbuf[FWD ? 2 * TR_FWD : 1];
  const int s = blockIdx.x;
  const int32_t base = sub_ptr[s], ns = sub_ptr[s + 1] - base;
  const int c0 = S.ch_sub[s], c1 = S.ch_sub[s + 1];
  const int nch = c1 - c0;
  unsigned char* ring = ts_sm;
  T* x = SMEMX ? reinterpret_cast<T*>(ts_sm + ring_bytes) : y + base;
  if (threadIdx.x == 0) {
    for (int i = 0; i < TR_NT; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= (32 * NW)) {
    // producer warp: the chunk table is read 32 entries at a time, one
    // window ahead; lane 0 issues the copies
    const int lane = threadIdx.x & 31;
    int64_t off_c = 0, off_n = 0;
    int32_t len_c = 0, len_n = 0;
    if (lane < nch) {
      off_n = S.ch_off[c0 + lane];
      len_n = S.ch_len[c0 + lane];
    }
    int head = 0, inflight = 0, oldest = 0;
    for (int i = 0; i < nch; ++i) {
      if ((i & 31) == 0) {
        off_c = off_n;
        len_c = len_n;
        if (i + 32 + lane < nch) {
          off_n = S.ch_off[c0 + i + 32 + lane];
          len_n = S.ch_len[c0 + i + 32 + lane];
        }
      }
      const int64_t off = __shfl_sync(0xffffffffu, off_c, i & 31);
      const int32_t len = __shfl_sync(0xffffffffu, len_c, i & 31);
      if (lane == 0) {
        const int t = i % TR_NT;
        const int start = head + len <= ring_bytes ? head : 0;
        const int fp = len + (start == 0 && head != 0 ? ring_bytes - head : 0);
        // retire consumed chunks until the ticket and the bytes are free
        while (oldest < i && (i - oldest >= TR_NT || inflight + fp > ring_bytes)) {
          mbar_wait(&empty[oldest % TR_NT], (uint32_t)((oldest / TR_NT) & 1));
          inflight -= foot[oldest % TR_NT];
          ++oldest;
        }
        pos[t] = start;
        foot[t] = fp;
        inflight += fp;
        head = start + len;
        mbar_expect_tx(&full[t], (uint32_t)len);
        bulk_g2s(ring + start, S.bytes + off, (uint32_t)len, &full[t]);
      }
      __syncwarp();
    }
    return;
  }
  for (int32_t k = threadIdx.x; k < ns; k += (32 * NW)) x[k] = (T)r[gmap[base + k]];
  consumer_bar<NW>();
  for (int i = 0; i < nch; ++i) {
    const int t = i % TR_NT;
    mbar_wait(&full[t], (uint32_t)((i / TR_NT) & 1));
    ts_chunk<T, CT, FWD, NW>(ring + pos[t], x, part, fwdbuf + ((i & 1) ^ 1) * (FWD ? TR_FWD : 0),
                         fwdbuf + (i & 1) * (FWD ? TR_FWD : 0));
    consumer_bar<NW>();
    if (threadIdx.x == 0) mbar_arrive(&empty[t]);
  }
  if (SMEMX)
    for (int32_t k = threadIdx.x; k < ns; k += (32 * NW)) y[base + k] = x[k];
}

}  // namespace gdsw

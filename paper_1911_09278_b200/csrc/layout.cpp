// Host construction of the per-agent device layouts (kernel K1's data).
//
// build_agent_csc restates AgentWorkspace.__init__'s stacking
// (pkg/src/macetomo/icd.py:185-192: sp.vstack of the subset's per-view CSR,
// then tocsc) as a counting sort; the result is index-identical to scipy's
// canonical CSC (asserted by tests/test_layout.py against the reference's
// golden col_ptr/row_idx).  The raster and super-voxel layouts are B200-side
// re-packings of that CSC: columns padded to 4 entries for 128-bit loads and,
// for super-voxels, 16-bit band-local row indices.
#include <algorithm>
#include <cstring>
#include <stdexcept>

#include "internal.h"

namespace mace {

void build_agent_csc(int n_side, int n_ch, const int64_t* row_ptr, const int32_t* cols, const float* vals,
                     const std::vector<int>& views, AgentCSC& out)
{
    const int64_t n = (int64_t)n_side * n_side;
    const int V = (int)views.size();
    out.col_ptr.assign(n + 1, 0);
    for (int j = 0; j < V; ++j) {
        for (int c = 0; c < n_ch; ++c) {
            const int64_t g = (int64_t)views[j] * n_ch + c;
            for (int64_t k = row_ptr[g]; k < row_ptr[g + 1]; ++k) out.col_ptr[cols[k] + 1]++;
        }
    }
    for (int64_t s = 0; s < n; ++s) out.col_ptr[s + 1] += out.col_ptr[s];
    const int64_t nnz = out.col_ptr[n];
    out.row.resize(nnz);
    out.val.resize(nnz);
    std::vector<int64_t> fill(out.col_ptr.begin(), out.col_ptr.end() - 1);
    for (int j = 0; j < V; ++j) {
        for (int c = 0; c < n_ch; ++c) {
            const int64_t g = (int64_t)views[j] * n_ch + c;
            const uint32_t r = (uint32_t)(j * n_ch + c);
            for (int64_t k = row_ptr[g]; k < row_ptr[g + 1]; ++k) {
                const int64_t q = fill[cols[k]]++;
                out.row[q] = r;
                out.val[q] = vals[k];
            }
        }
    }
}

static inline int64_t pad4(int64_t x) { return (x + 3) & ~int64_t(3); }
static inline int64_t pad8(int64_t x) { return (x + 7) & ~int64_t(7); }

void build_raster_layout(const AgentCSC& csc, int n, RasterLayout& out)
{
    out.pix.resize(n);
    int64_t total = 0;
    out.max_col = 0;
    for (int s = 0; s < n; ++s) {
        const int64_t L = csc.col_ptr[s + 1] - csc.col_ptr[s];
        out.max_col = std::max<int>(out.max_col, (int)L);
        total += pad4(L);
    }
    if (total >= (int64_t)1 << 31) throw std::runtime_error("raster layout exceeds 2^31 entries per agent");
    out.idx.assign(total, 0);
    out.val.assign(total, 0.0f);
    int64_t pos = 0;
    for (int s = 0; s < n; ++s) {
        const int64_t a = csc.col_ptr[s], L = csc.col_ptr[s + 1] - a;
        out.pix[s] = {(int32_t)pos, (int32_t)L};
        for (int64_t k = 0; k < L; ++k) {
            out.idx[pos + k] = csc.row[a + k];
            out.val[pos + k] = csc.val[a + k];
        }
        pos += pad4(L);
    }
}

void build_sv_layout(const AgentCSC& csc, int n_side, int n_ch, int V, int S, SVLayout& out)
{
    out.svs = S;
    out.views = V;
    out.n_sv_side = (n_side + S - 1) / S;
    out.n_sv = out.n_sv_side * out.n_sv_side;
    out.band.assign((size_t)out.n_sv * V, {0, 0});
    out.bsize.assign(out.n_sv, 0);
    out.pix.assign((size_t)out.n_sv * S * S, {0, 0});
    out.max_band = 0;
    out.max_col = 0;
    out.duplicates = 0;
    // pass 1: band windows and entry counts
    std::vector<int> lo(V), hi(V);
    int64_t total = 0;
    std::vector<int64_t> sv_entries(out.n_sv, 0);
    for (int sv = 0; sv < out.n_sv; ++sv) {
        const int r0 = (sv / out.n_sv_side) * S, c0 = (sv % out.n_sv_side) * S;
        std::fill(lo.begin(), lo.end(), INT32_MAX);
        std::fill(hi.begin(), hi.end(), -1);
        int64_t ent = 0;
        for (int k = 0; k < S * S; ++k) {
            const int r = r0 + k / S, c = c0 + k % S;
            if (r >= n_side || c >= n_side) continue;
            const int64_t s = (int64_t)r * n_side + c;
            int64_t L = 0;
            uint32_t prev = UINT32_MAX;
            for (int64_t q = csc.col_ptr[s]; q < csc.col_ptr[s + 1]; ++q) {
                const uint32_t row = csc.row[q];
                if (row == prev) continue;  // duplicate (row, pixel) -> merged below
                prev = row;
                ++L;
                const int j = (int)(row / n_ch), ch = (int)(row % n_ch);
                lo[j] = std::min(lo[j], ch);
                hi[j] = std::max(hi[j], ch);
            }
            out.max_col = std::max<int>(out.max_col, (int)L);
            ent += pad8(L);
        }
        int pos = 0;
        for (int j = 0; j < V; ++j) {
            // window of local rows, widened to 16-byte ({e, lambda} float2 pairs) alignment so the
            // kernel can stage it with one bulk (TMA) copy per view; pads are never referenced
            int start = 0, cnt = 0;
            if (hi[j] >= 0) {
                start = (j * n_ch + lo[j]) & ~1;
                const int end = ((j * n_ch + hi[j]) | 1) + 1;
                cnt = end - start;
            }
            out.band[(size_t)sv * V + j] = {(int32_t)start, (int32_t)((pos << 16) | cnt)};
            pos += cnt;
            if (pos > 65534) throw std::runtime_error("super-voxel band exceeds 65534 rows; use a smaller tile");
        }
        out.bsize[sv] = pos;
        out.max_band = std::max(out.max_band, pos);
        sv_entries[sv] = ent;
        total += ent;
    }
    if (total >= (int64_t)1 << 31) throw std::runtime_error("super-voxel layout exceeds 2^31 entries per agent");
    out.idx.assign(total, 0);
    out.val.assign(total, 0.0f);
    // pass 2: entries, SV-major, pixels in tile-raster order, band-local indices.
    // Within a column, entries are stored in groups of 128 (16 lanes x 8 slots); inside
    // a group of Lg entries (L8 = ceil(Lg/8)) slot 8l+q holds entry l + q*L8, so lane l's
    // two 128-bit value loads and one 128-bit index load bring entries l, l+L8, ...,
    // l+7L8: at every step the half-warp touches consecutive entries (consecutive
    // views' windows -> spread shared-memory banks).  Columns are padded to 8 slots.
    // Pads carry value 0 and the tile's dummy band row B (never a real row).
    int64_t pos = 0;
    std::vector<uint16_t> ci;
    std::vector<float> cv;
    for (int sv = 0; sv < out.n_sv; ++sv) {
        const int r0 = (sv / out.n_sv_side) * S, c0 = (sv % out.n_sv_side) * S;
        const int2_t* bt = &out.band[(size_t)sv * V];
        const uint16_t dummy = (uint16_t)out.bsize[sv];
        for (int k = 0; k < S * S; ++k) {
            const int r = r0 + k / S, c = c0 + k % S;
            if (r >= n_side || c >= n_side) {
                out.pix[(size_t)sv * S * S + k] = {(int32_t)pos, 0};
                continue;
            }
            const int64_t s = (int64_t)r * n_side + c;
            ci.clear();
            cv.clear();
            uint32_t prev = UINT32_MAX;
            for (int64_t q = csc.col_ptr[s]; q < csc.col_ptr[s + 1]; ++q) {
                const uint32_t row = csc.row[q];
                if (row == prev) {  // merge duplicate entry (sum of lengths)
                    cv.back() += csc.val[q];
                    out.duplicates++;
                    continue;
                }
                prev = row;
                const int j = (int)(row / n_ch), ch = (int)(row % n_ch);
                const int2_t b = bt[j];
                ci.push_back((uint16_t)((b.y >> 16) + (j * n_ch + ch - b.x)));
                cv.push_back(csc.val[q]);
            }
            const int L = (int)ci.size();
            for (int g0 = 0; g0 < std::max(L, 1); g0 += 128) {
                const int Lg = std::min(128, L - g0), L8 = (std::max(Lg, 0) + 7) / 8;
                for (int l = 0; l < L8; ++l)
                    for (int q = 0; q < 8; ++q) {
                        const int e = l + q * L8;
                        const int64_t slot = pos + g0 + 8 * l + q;
                        out.idx[slot] = e < Lg ? ci[g0 + e] : dummy;
                        out.val[slot] = e < Lg ? cv[g0 + e] : 0.0f;
                    }
            }
            out.pix[(size_t)sv * S * S + k] = {(int32_t)pos, (int32_t)L};
            pos += pad8(L);
        }
    }
}

std::vector<uint32_t> build_queue(int n_agents, int n_sv_side, int C, int n_slices)
{
    if (C < 1) C = 1;
    if (C > n_sv_side) C = n_sv_side;
    if ((int64_t)n_agents * n_slices > (1 << (32 - 22)) || (int64_t)n_sv_side * n_sv_side > (1 << 22))
        throw std::runtime_error("work queue: too many agents x slices or super-voxels");
    std::vector<uint32_t> q;
    q.reserve((size_t)n_agents * n_slices * n_sv_side * n_sv_side);
    // local (virtual) agent index = slice * n_agents + agent; at one tile position the slices
    // of an agent are adjacent, so they run concurrently and share that tile's A columns in L2
    for (int cr = 0; cr < C; ++cr)
        for (int cc = 0; cc < C; ++cc)
            for (int r = cr; r < n_sv_side; r += C)
                for (int c = cc; c < n_sv_side; c += C)
                    for (int a = 0; a < n_agents; ++a)
                        for (int s = 0; s < n_slices; ++s)
                            q.push_back(((uint32_t)(s * n_agents + a) << 22) | (uint32_t)(r * n_sv_side + c));
    return q;
}

}  // namespace mace

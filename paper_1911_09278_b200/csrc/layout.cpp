// Host construction of the per-agent device layouts (kernel K1's data).
//
// build_agent_csc restates AgentWorkspace.__init__'s stacking
// (pkg/src/macetomo/icd.py:185-192: sp.vstack of the subset's per-view CSR,
// then tocsc) as a counting sort; the result is index-identical to scipy's
// canonical CSC (asserted by tests/test_layout.py against the reference's
// golden col_ptr/row_idx).  The raster and super-voxel layouts are B200-side
// re-packings of that CSC: columns padded to 4 entries for 128-bit loads (raster) and
// lane-per-view slot records in batch visit order (super-voxels, internal.h).
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

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

void build_sv_layout(const AgentCSC& csc, int n_side, int n_ch, int V, int S, SVLayout& out, int ng)
{
    out.svs = S;
    out.views = V;
    // view groups of 32; more than 4 groups (> 128 views per agent) are split into chunks of 3
    // groups, one warp per chunk of a tile (k_sv.cuh multi-warp tiles)
    const int ng_total = std::max((V + 31) / 32, ng);
    out.chunks = ng_total > 4 ? (ng_total + 2) / 3 : 1;
    out.ng = ng_total > 4 ? 3 : ng_total;
    if (out.chunks > kSvMaxChunks)
        throw std::runtime_error("super-voxel layout: at most " + std::to_string(32 * 3 * kSvMaxChunks) + " views per agent");
    out.n_sv_side = (n_side + S - 1) / S;
    out.n_sv = out.n_sv_side * out.n_sv_side;
    out.band.assign((size_t)out.n_sv * V, {0, 0});
    out.max_col = 0;
    out.duplicates = 0;
    out.entries = 0;
    // pass 1: windows per (tile, view), entries per (pixel, view); rows of a (pixel, view) pair
    // must be consecutive channels (a convex pixel in parallel-beam geometry)
    std::vector<int> lo(V), hi(V), first(V), cntpv(V);
    int K = 1, wcap = 1;
    for (int sv = 0; sv < out.n_sv; ++sv) {
        const int r0 = (sv / out.n_sv_side) * S, c0 = (sv % out.n_sv_side) * S;
        std::fill(lo.begin(), lo.end(), INT32_MAX);
        std::fill(hi.begin(), hi.end(), -1);
        for (int k = 0; k < S * S; ++k) {
            const int r = r0 + k / S, c = c0 + k % S;
            if (r >= n_side || c >= n_side) continue;
            const int64_t s = (int64_t)r * n_side + c;
            std::fill(cntpv.begin(), cntpv.end(), 0);
            std::fill(first.begin(), first.end(), -1);
            uint32_t prev = UINT32_MAX;
            int L = 0;
            for (int64_t q = csc.col_ptr[s]; q < csc.col_ptr[s + 1]; ++q) {
                const uint32_t row = csc.row[q];
                if (row == prev) continue;
                prev = row;
                ++L;
                const int j = (int)(row / n_ch), ch = (int)(row % n_ch);
                if (first[j] < 0) first[j] = ch;
                else if (ch != first[j] + cntpv[j]) throw std::runtime_error("non-contiguous channels in a (pixel, view)");
                cntpv[j]++;
                lo[j] = std::min(lo[j], ch);
                hi[j] = std::max(hi[j], ch);
            }
            out.max_col = std::max(out.max_col, L);
            for (int j = 0; j < V; ++j) K = std::max(K, cntpv[j]);
        }
        for (int j = 0; j < V; ++j) {
            const int cnt = hi[j] >= 0 ? hi[j] - lo[j] + 1 : 0;
            if (cnt > 255) throw std::runtime_error("super-voxel window exceeds 255 rows; use a smaller tile");
            out.band[(size_t)sv * V + j] = {(int32_t)(j * n_ch + (cnt ? lo[j] : 0)), (int32_t)cnt};
            wcap = std::max(wcap, cnt);
        }
    }
    if (K > 4) throw std::runtime_error("more than 4 entries per (pixel, view): channel pitch far below pixel pitch");
    if (S & 1) throw std::runtime_error("super-voxel side must be even");
    out.K = K <= 2 ? 2 : 4;
    out.wcap = std::max(wcap, out.K);  // a slot addresses K rows even in a shorter window
    out.nb = sv_batches(S);
    const int G = out.ng, KK = out.K;
    out.rec = G * 32 * KK + 32;
    const int CH = out.chunks;
    if (CH > 1 && KK != 2) throw std::runtime_error("multi-warp super-voxel tiles need at most 2 entries per (pixel, view)");
    const size_t per_tile = (size_t)out.nb * CH * kSvBatch * out.rec;
    out.data.assign((size_t)out.n_sv * per_tile, 0u);
    // pass 2: scatter each entry into its (slot, group, lane, k) position
    for (int sv = 0; sv < out.n_sv; ++sv) {
        const int r0 = (sv / out.n_sv_side) * S, c0 = (sv % out.n_sv_side) * S;
        const int2_t* bt = &out.band[(size_t)sv * V];
        for (int t = 0; t < out.nb * kSvBatch; ++t) {
            const int k = sv_slot_pixel(S, t);
            if (k < 0) continue;
            const int r = r0 + k / S, c = c0 + k % S;
            if (r >= n_side || c >= n_side) continue;
            const int64_t s = (int64_t)r * n_side + c;
            // (batch, chunk) blocks of kSvBatch x rec words, lane-major inside (internal.h)
            const int slot = t % kSvBatch;
            uint32_t* blk0 = &out.data[(size_t)sv * per_tile + (size_t)(t / kSvBatch) * CH * kSvBatch * out.rec];
            // entries of one (pixel, view) are consecutive in the column (rows ascending); the slot
            // offset is pulled back so that all K addressed rows stay inside the window (rows past
            // cnt would alias the lane's next window or memory after the band)
            int cur_j = -1, m = 0, o0 = 0;
            float vals[4] = {0.f, 0.f, 0.f, 0.f};
            auto flush = [&]() {
                if (cur_j < 0) return;
                const int gt = cur_j >> 5, l = cur_j & 31, cnt = bt[cur_j].y;
                const int g = gt % G;  // group inside the view's chunk gt / G
                uint32_t* blk = blk0 + (size_t)(gt / G) * kSvBatch * out.rec;
                const int o = std::min(o0, std::max(cnt, KK) - KK);
                blk[sv_ofs_word(G, KK, l, slot)] |= (uint32_t)o << (8 * g);
                for (int u = 0; u < m; ++u) std::memcpy(&blk[sv_len_word(G, KK, g, l, slot, (o0 - o) + u)], &vals[u], 4);
                out.entries += m;
            };
            uint32_t prev = UINT32_MAX;
            for (int64_t q = csc.col_ptr[s]; q < csc.col_ptr[s + 1]; ++q) {
                const uint32_t row = csc.row[q];
                const int j = (int)(row / n_ch);
                if (row == prev) {  // merge a duplicate (row, pixel) entry
                    vals[m - 1] += csc.val[q];
                    out.duplicates++;
                    continue;
                }
                prev = row;
                if (j != cur_j) {
                    flush();
                    cur_j = j;
                    m = 0;
                    o0 = (int)row - bt[j].x;  // offset of the first entry in view j's window
                }
                vals[m++] = csc.val[q];
            }
            flush();
        }
    }
}

std::vector<uint32_t> build_queue(int n_agents, int n_sv_side, int C, int n_slices, int group)
{
    if (C < 1) C = 1;
    if (C > n_sv_side) C = n_sv_side;
    if (group < 1 || group > n_agents) group = n_agents;
    if ((int64_t)n_agents * n_slices > (1 << (32 - 22)) || (int64_t)n_sv_side * n_sv_side > (1 << 22))
        throw std::runtime_error("work queue: too many agents x slices or super-voxels");
    std::vector<uint32_t> q;
    q.reserve((size_t)n_agents * n_slices * n_sv_side * n_sv_side);
    // local (virtual) agent index = slice * n_agents + agent; at one tile position the slices
    // of an agent are adjacent, so they run concurrently and share that tile's A columns in L2.
    // Agents run in groups of `group` (default: all at once): a group's tiles fill the whole
    // grid before the next group's start, so each agent of a group has about warps / group tiles
    // in flight -- the per-agent concurrency (staleness) of a rank that owns `group` agents.
    for (int g0 = 0; g0 < n_agents; g0 += group)
        for (int cr = 0; cr < C; ++cr)
            for (int cc = 0; cc < C; ++cc)
                for (int r = cr; r < n_sv_side; r += C)
                    for (int c = cc; c < n_sv_side; c += C)
                        for (int a = g0; a < std::min(n_agents, g0 + group); ++a)
                            for (int s = 0; s < n_slices; ++s)
                                q.push_back(((uint32_t)(s * n_agents + a) << 22) | (uint32_t)(r * n_sv_side + c));
    return q;
}

}  // namespace mace

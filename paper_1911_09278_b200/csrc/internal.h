// Host-side structures shared by the tracer, the layout builder and the CUDA context.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace mace {

struct int2_t {
    int32_t x, y;
};

// ---- system matrix (reference SparseViewMatrix per view, geometry.py:115-158)
struct SysMatView {
    std::vector<int64_t> row_ptr;  // n_ch + 1
    std::vector<int32_t> cols;     // pixel index, sorted per row
    std::vector<double> lens;      // exact intersection lengths (float64)
};
struct SysMat {
    int n_side = 0, n_views = 0, n_ch = 0;
    std::vector<SysMatView> views;
};
SysMat* sysmat_trace(int n_side, double pitch, int n_views, int n_ch, const double* ux, const double* uy,
                     const double* ex, const double* ey, const double* offsets, int n_threads);
SysMat* sysmat_read(const char* path, int64_t* n_pixels);  // MACEMAT1 file

// ---- per-agent device layouts (built on the host from the global CSR)
//
// Stacked agent operator (icd.py:185-192): local row r = j * n_ch + c for the
// j-th view of the subset.  Column s of the stacked CSC holds the entries of
// pixel s with rows ascending (scipy's canonical tocsc order).
struct AgentCSC {
    std::vector<int64_t> col_ptr;  // n + 1
    std::vector<uint32_t> row;     // local row
    std::vector<float> val;        // float32(A)
};

// Raster layout: columns in pixel order 0..n-1, padded to 4 entries (pads: row 0, val 0).
struct RasterLayout {
    std::vector<int2_t> pix;     // {entry start, length} per pixel
    std::vector<uint32_t> idx;   // local row
    std::vector<float> val;
    int max_col = 0;
};

// Super-voxel layout: S x S pixel tiles; the error-sinogram rows a tile touches
// (its "band": one contiguous channel window per view) are staged in shared memory.
// Lane-per-view super-voxel layout.  Parallel-beam geometry gives every (pixel, view)
// pair at most a few entries on consecutive channels, so view j is owned by lane j % 32
// (view group g = j / 32, at most 4 groups): per tile, view j's band window is the rows
// [start_j, start_j + cnt_j) the tile touches; per pixel, lane l of group g holds the K
// lengths of view 32g+l and their offset inside that window (one byte per group).  In
// shared memory the window of view j lives in bank j % 32, so gathers and scatters are
// bank-conflict free and rows are lane-private.
//
// Pixels of a tile are visited in four parity classes (row mod 2, col mod 2), raster order
// inside a class, in batches of kSvBatch: pixels of one batch are never 8-neighbours, so their
// prior terms are independent and their coupling through shared sinogram rows is one
// precomputed cross term per pair (k_sv.cuh).  Slot records are stored in visit order,
// batch-contiguous, so a batch is one contiguous copy.
constexpr int kSvBatch = 4;
constexpr int kSvMaxChunks = 16;  // multi-warp tiles: at most 16 warps (chunks of 96 views) per tile
struct SVLayout {
    int svs = 0, n_sv_side = 0, n_sv = 0, views = 0;
    int ng = 0;                  // view groups per chunk: ceil(views / 32) (<= 4), or 3 with chunks
    int chunks = 1;              // chunks of 3 view groups (one warp each) when views > 128
    int K = 0;                   // entries per (pixel, view) slot (max over the agent, 2 for pitch = channel pitch)
    int wcap = 0;                // max window rows over tiles and views
    int nb = 0;                  // batches per tile
    int rec = 0;                 // words per pixel slot: ng*32*K lengths ([g][lane][k]) + 32 offset words
    std::vector<int2_t> band;    // [n_sv * views] {local row start, cnt}
    std::vector<uint32_t> data;  // [n_sv][nb][chunks] blocks of kSvBatch x rec words (sv_len_word / sv_ofs_word; empty slots 0)
    int max_col = 0;             // max entries per column (info)
    int64_t entries = 0;         // stored nonzeros (== nnz of the agent)
    int64_t duplicates = 0;      // repeated (row, pixel) pairs merged (never seen in practice)
};
// Records of one (tile, batch, chunk) are one block of kSvBatch x rec words, lane-major so that a
// lane's lengths for a view group are contiguous (one 256-bit load per group for K = 2):
//   lengths  [g][lane][slot][k]  at ((g * 32 + lane) * kSvBatch + slot) * K + k
//   offsets  [lane][slot]        at ng * 32 * kSvBatch * K + lane * kSvBatch + slot  (one byte per group)
// (MACE_SV_LANE_MAJOR 0: slot-major blocks, lengths [slot][g][lane][k] and offsets [slot][lane] --
// the round-1 layout, kept for A/B)
#ifndef MACE_SV_LANE_MAJOR
#define MACE_SV_LANE_MAJOR 1
#endif
inline size_t sv_len_word(int ng, int K, int g, int lane, int slot, int k)
{
    if (!MACE_SV_LANE_MAJOR) return (size_t)slot * ((size_t)ng * 32 * K + 32) + ((size_t)g * 32 + lane) * K + k;
    return (((size_t)g * 32 + lane) * kSvBatch + slot) * K + k;
}
inline size_t sv_ofs_word(int ng, int K, int lane, int slot)
{
    if (!MACE_SV_LANE_MAJOR) return (size_t)slot * ((size_t)ng * 32 * K + 32) + (size_t)ng * 32 * K + lane;
    return (size_t)ng * 32 * kSvBatch * K + (size_t)lane * kSvBatch + slot;
}
// Visit-order slot t of an S x S tile -> local pixel (lr * S + lc), or -1 for a padding slot.
inline int sv_slot_pixel(int S, int t)
{
    const int h = S / 2, per_class = h * h, bpc = (per_class + kSvBatch - 1) / kSvBatch;
    const int b = t / kSvBatch, cls = b / bpc, i = (b % bpc) * kSvBatch + t % kSvBatch;
    if (i >= per_class) return -1;
    return ((cls >> 1) + 2 * (i / h)) * S + (cls & 1) + 2 * (i % h);
}
inline int sv_batches(int S) { return 4 * (((S / 2) * (S / 2) + kSvBatch - 1) / kSvBatch); }

void build_agent_csc(int n_side, int n_ch, const int64_t* row_ptr, const int32_t* cols, const float* vals,
                     const std::vector<int>& views, AgentCSC& out);
void build_raster_layout(const AgentCSC& csc, int n, RasterLayout& out);
// ng: view groups of the record (0: ceil(views / 32)); agents of one context share one ng
void build_sv_layout(const AgentCSC& csc, int n_side, int n_ch, int n_views_agent, int svs, SVLayout& out, int ng = 0);
// Queue of (agent << 22 | sv) items: colour classes (sv_row mod C, sv_col mod C) in
// order, SVs of a class in raster order, agents interleaved within a position.
// group > 0: agents in consecutive groups of `group` (each group's tiles before the next group's).
std::vector<uint32_t> build_queue(int n_agents, int n_sv_side, int colours, int n_slices = 1, int group = 0);

void set_error(const std::string& msg);

}  // namespace mace

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
// (its "band": one contiguous channel window per view) are staged in shared
// memory, so entries carry a 16-bit band index instead of the 32-bit row.
struct SVLayout {
    int svs = 0, n_sv_side = 0, n_sv = 0, views = 0;
    std::vector<int2_t> band;    // [n_sv * views] {local row start, (pos << 16) | cnt}
    std::vector<int32_t> bsize;  // [n_sv] band rows
    std::vector<int2_t> pix;     // [n_sv * S * S] {entry start, length}; length 0 outside image
    std::vector<uint16_t> idx;   // band-local row
    std::vector<float> val;
    int max_band = 0, max_col = 0;
    int64_t duplicates = 0;      // repeated (row, pixel) pairs merged (never seen in practice)
};

void build_agent_csc(int n_side, int n_ch, const int64_t* row_ptr, const int32_t* cols, const float* vals,
                     const std::vector<int>& views, AgentCSC& out);
void build_raster_layout(const AgentCSC& csc, int n, RasterLayout& out);
void build_sv_layout(const AgentCSC& csc, int n_side, int n_ch, int n_views_agent, int svs, SVLayout& out);
// Queue of (agent << 22 | sv) items: colour classes (sv_row mod C, sv_col mod C) in
// order, SVs of a class in raster order, agents interleaved within a position.
std::vector<uint32_t> build_queue(int n_agents, int n_sv_side, int colours, int n_slices = 1);

void set_error(const std::string& msg);

}  // namespace mace

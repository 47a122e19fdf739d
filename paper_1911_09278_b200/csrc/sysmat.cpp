// Native system-matrix generator: bit-exact restatement of the reference tracer
//   _trace_axis_aligned  pkg/src/macetomo/geometry.py:177-186
//   _trace_ray           pkg/src/macetomo/geometry.py:189-225
//   build_system_matrix  pkg/src/macetomo/geometry.py:228-258
// Every floating-point expression keeps numpy's evaluation order; the file is
// compiled with -ffp-contract=off so no FMA changes a rounding.  The trig
// values (ux, uy, ex, ey) are computed by the caller in numpy, exactly as the
// reference does, so host libm differences cannot leak in.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

namespace mace {

struct RayOut {
    std::vector<int32_t> pix;
    std::vector<double> len;
};

static void trace_axis_aligned(double offset, double lo_edge, double pitch, int n_side, bool along_rows,
                               std::vector<int32_t>& pix, std::vector<double>& len)
{
    // idx = int(np.floor((offset - lo_edge) / pitch))
    double f = std::floor((offset - lo_edge) / pitch);
    if (!(f >= 0.0) || f >= (double)n_side) return;
    int32_t idx = (int32_t)f;
    for (int i = 0; i < n_side; ++i) {
        pix.push_back(along_rows ? (int32_t)(i * n_side + idx) : (int32_t)(idx * n_side + i));
        len.push_back(pitch);
    }
}

// Trace one ray p + t u; appends (pix, len) sorted by pixel (stable in t order).
static void trace_ray(double px, double py, double ux, double uy, int n_side, double pitch,
                      std::vector<double>& tx, std::vector<double>& ty, std::vector<double>& ts,
                      std::vector<int64_t>& key, std::vector<int32_t>& pix, std::vector<double>& len)
{
    pix.clear();
    len.clear();
    const double half = 0.5 * ((double)n_side * pitch);  // 0.5 * geom.image_width
    const double x0 = -half, y0 = half;
    if (ux == 0.0) {
        trace_axis_aligned(px, x0, pitch, n_side, true, pix, len);
        return;
    }
    if (uy == 0.0) {
        trace_axis_aligned(y0 - py, 0.0, pitch, n_side, false, pix, len);
        return;
    }
    const int ne = n_side + 1;
    tx.resize(ne);
    ty.resize(ne);
    for (int i = 0; i < ne; ++i) {
        const double edge = (double)i * pitch;  // np.arange(n+1, float64) * pitch
        tx[i] = ((x0 + edge) - px) / ux;
        ty[i] = ((y0 - edge) - py) / uy;
    }
    // python builtin min/max on two floats: min(a, b) -> b if b < a else a
    auto pmin = [](double a, double b) { return b < a ? b : a; };
    auto pmax = [](double a, double b) { return b > a ? b : a; };
    const double t_lo = pmax(pmin(tx[0], tx[ne - 1]), pmin(ty[0], ty[ne - 1]));
    const double t_hi = pmin(pmax(tx[0], tx[ne - 1]), pmax(ty[0], ty[ne - 1]));
    if (t_hi <= t_lo) return;

    // ts = sort(tx ∪ ty restricted to (t_lo, t_hi)); both sequences are monotone
    // (monotone rounding), so a two-way merge yields np.sort's value sequence.
    ts.clear();
    ts.push_back(t_lo);
    int ia = 0, ib = 0, da = 1, db = 1;
    if (tx[0] > tx[ne - 1]) { ia = ne - 1; da = -1; }
    if (ty[0] > ty[ne - 1]) { ib = ne - 1; db = -1; }
    int na = 0, nb = 0;
    auto nexta = [&](double& v) -> bool {
        while (na < ne) {
            double t = tx[ia];
            ia += da;
            ++na;
            if (t > t_lo && t < t_hi) { v = t; return true; }
        }
        return false;
    };
    auto nextb = [&](double& v) -> bool {
        while (nb < ne) {
            double t = ty[ib];
            ib += db;
            ++nb;
            if (t > t_lo && t < t_hi) { v = t; return true; }
        }
        return false;
    };
    double va = 0, vb = 0;
    bool ha = nexta(va), hb = nextb(vb);
    while (ha || hb) {
        if (ha && (!hb || va <= vb)) { ts.push_back(va); ha = nexta(va); }
        else { ts.push_back(vb); hb = nextb(vb); }
    }
    ts.push_back(t_hi);

    const double floor_len = 1e-12 * pitch;  // _LENGTH_FLOOR * pitch
    const size_t nseg = ts.size() - 1;
    for (size_t i = 0; i < nseg; ++i) {
        const double seg = ts[i + 1] - ts[i];
        if (!(seg > floor_len)) continue;
        const double mid = 0.5 * (ts[i] + ts[i + 1]);
        double fc = std::floor(((px + mid * ux) - x0) / pitch);
        double fr = std::floor((y0 - (py + mid * uy)) / pitch);
        int64_t col = (int64_t)fc, row = (int64_t)fr;
        col = col < 0 ? 0 : (col > n_side - 1 ? n_side - 1 : col);
        row = row < 0 ? 0 : (row > n_side - 1 ? n_side - 1 : row);
        pix.push_back((int32_t)(row * n_side + col));
        len.push_back(seg);
    }
    // np.argsort(pix, kind="stable")
    const size_t m = pix.size();
    bool asc = true, desc = true;
    for (size_t i = 1; i < m; ++i) {
        if (pix[i] < pix[i - 1]) asc = false;
        if (pix[i] >= pix[i - 1]) desc = false;
    }
    if (asc) return;
    if (desc) {
        std::reverse(pix.begin(), pix.end());
        std::reverse(len.begin(), len.end());
        return;
    }
    key.resize(m);
    for (size_t i = 0; i < m; ++i) key[i] = ((int64_t)pix[i] << 32) | (int64_t)i;  // stable by construction
    std::sort(key.begin(), key.end());
    std::vector<int32_t> p2(m);
    std::vector<double> l2(m);
    for (size_t i = 0; i < m; ++i) {
        size_t j = (size_t)(key[i] & 0xffffffffLL);
        p2[i] = pix[j];
        l2[i] = len[j];
    }
    pix.swap(p2);
    len.swap(l2);
}

SysMat* sysmat_trace(int n_side, double pitch, int n_views, int n_ch, const double* ux, const double* uy,
                     const double* ex, const double* ey, const double* offsets, int n_threads)
{
    SysMat* sm = new SysMat();
    sm->n_side = n_side;
    sm->n_views = n_views;
    sm->n_ch = n_ch;
    sm->views.resize(n_views);
    if (n_threads <= 0) n_threads = (int)std::max(1u, std::thread::hardware_concurrency());
    n_threads = std::min(n_threads, std::max(1, n_views));
    std::atomic<int> next(0);
    auto worker = [&]() {
        std::vector<double> tx, ty, ts;
        std::vector<int64_t> key;
        std::vector<int32_t> pix;
        std::vector<double> len;
        for (;;) {
            int k = next.fetch_add(1);
            if (k >= n_views) break;
            SysMatView& V = sm->views[k];
            V.row_ptr.assign(n_ch + 1, 0);
            V.cols.clear();
            V.lens.clear();
            for (int d = 0; d < n_ch; ++d) {
                const double s = offsets[d];
                trace_ray(s * ex[k], s * ey[k], ux[k], uy[k], n_side, pitch, tx, ty, ts, key, pix, len);
                V.cols.insert(V.cols.end(), pix.begin(), pix.end());
                V.lens.insert(V.lens.end(), len.begin(), len.end());
                V.row_ptr[d + 1] = V.row_ptr[d] + (int64_t)pix.size();
            }
        }
    };
    std::vector<std::thread> th;
    for (int t = 0; t < n_threads; ++t) th.emplace_back(worker);
    for (auto& t : th) t.join();
    return sm;
}

// MACEMAT1 reader (format of save_system_matrix, geometry.py:293-342): ASCII "MACEMAT1",
// ASCII "n_views n_channels n", then per view, per row: uint32 LE count, count x (uint32 LE pixel,
// float32 LE length).  Lengths come back as float64 (the file holds float32, like the reference's
// load_system_matrix).  One sequential pass into the per-view CSR, no per-row Python work.
SysMat* sysmat_read(const char* path, int64_t* n_pixels)
{
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw std::runtime_error(std::string("cannot open ") + path);
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, &std::fclose);
    char line[256];
    if (!std::fgets(line, sizeof line, f) || std::string(line).rfind("MACEMAT1", 0) != 0 ||
        (line[8] != '\n' && line[8] != '\r'))
        throw std::invalid_argument("bad matrix file magic");
    long long nv = 0, nc = 0, n = 0;
    if (!std::fgets(line, sizeof line, f) || std::sscanf(line, "%lld %lld %lld", &nv, &nc, &n) != 3 || nv < 1 ||
        nc < 1 || n < 1 || n > INT32_MAX)
        throw std::invalid_argument("bad matrix file header");
    auto m = std::make_unique<SysMat>();
    m->n_views = (int)nv;
    m->n_ch = (int)nc;
    const long long side = (long long)std::llround(std::sqrt((double)n));
    m->n_side = side * side == n ? (int)side : 0;
    m->views.resize(nv);
    std::vector<uint32_t> rec;
    for (long long k = 0; k < nv; ++k) {
        SysMatView& V = m->views[k];
        V.row_ptr.assign(nc + 1, 0);
        for (long long d = 0; d < nc; ++d) {
            uint32_t cnt = 0;
            if (std::fread(&cnt, 4, 1, f) != 1) throw std::invalid_argument("truncated matrix file");
            rec.resize(2 * (size_t)cnt);
            if (cnt && std::fread(rec.data(), 8, cnt, f) != cnt) throw std::invalid_argument("truncated matrix file");
            for (uint32_t e = 0; e < cnt; ++e) {
                const uint32_t col = rec[2 * e];
                float len;
                std::memcpy(&len, &rec[2 * e + 1], 4);
                if ((long long)col >= n) throw std::invalid_argument("pixel index out of range in matrix file");
                V.cols.push_back((int32_t)col);
                V.lens.push_back((double)len);
            }
            V.row_ptr[d + 1] = V.row_ptr[d] + cnt;
        }
    }
    *n_pixels = n;
    return m.release();
}

}  // namespace mace

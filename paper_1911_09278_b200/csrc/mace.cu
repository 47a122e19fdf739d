// libmace_b200: device context, launches and the C ABI (include/mace_b200.h).
//
// One context = one GPU, the full-data operator (global CSR for K3), one
// sinogram, and the agents this rank owns (view subsets, geometry.py:161-174).
// All device memory is owned here; host pointers are borrowed for the call.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"
#include "kernels.cuh"
#include "k2_launch.h"
#include "k_sweep64.cuh"
#include "k_peer.cuh"
#include "cnn.cuh"
#include "mace_b200.h"

namespace mace {

static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
#define CK(x)                                                                                              \
    do {                                                                                                   \
        cudaError_t e_ = (x);                                                                              \
        if (e_ != cudaSuccess)                                                                             \
            throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " (" + __FILE__ + ":" +      \
                            std::to_string(__LINE__) + ")");                                               \
    } while (0)

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count)
    {
        free();
        n = count;
        if (count) CK(cudaMalloc(&p, count * sizeof(T)));
    }
    void free()
    {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { free(); }
};

struct AgentMem {
    std::vector<int> views;
    DBuf<int> d_views;
    DBuf<int2> band, rpix;
    DBuf<float> rval;
    DBuf<uint32_t> rec, ridx;
    DBuf<uint32_t> recw;  // weighted records a sqrt(lambda) (k_sv_consts; single-slice contexts)
    int R = 0, n_sv_side = 0, n_sv = 0, max_col = 0;
    int wcap = 0, ng = 1, K = 2, nb = 0, rec_words = 0, chunks = 1;  // lane-per-view layout geometry
    int64_t entries = 0, nnz = 0, duplicates = 0;
    DBuf<uint32_t> queue;  // this agent alone, colour order
    float beta_eff = 0.f, inv_s2 = 0.f;
    int clamp = 0;
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = true;
    int n_side = 0, n_views = 0, n_ch = 0;
    size_t n = 0;
    DBuf<int64_t> rp;
    DBuf<int> cols;
    DBuf<float> vals;
    int64_t nnz = 0;
    DBuf<float> y, lam;
    PriorC prior{};
    // agents
    int n_local = 0, schedule = 0, S = 8, NV = 1;
    int n_real = 0, n_slices = 1;  // n_local = n_real agents x n_slices slices (config 4 batches)
    std::vector<std::unique_ptr<AgentMem>> am;
    std::vector<AgentDev> h_agents;
    DBuf<AgentDev> d_agents;
    DBuf<int> row_base;
    int total_rows = 0;
    DBuf<float> E, LAM;  // error sinograms, weights (per local agent rows)
    DBuf<float> BC;      // super-voxel batch constants (per local agent, k_sv_consts)
    DBuf<float> LB;      // super-voxel band lambda in shared-memory order (per local agent)
    DBuf<float> Y, Z, W, TH, VT;
    DBuf<uint32_t> queue;
    int n_items = 0;
    DBuf<double> part;
    DBuf<unsigned> head;
    DBuf<int> done;
    DBuf<double> sums5, log, norm_scratch;
    DBuf<unsigned> norm_counter;
    DBuf<int> iter_ctr;  // device iteration index (mace_iterate_finish with iter < 0: graph-captured loops)
    int log_cap = 0;
    DBuf<float> wbar, g, ref, wsum;
    DBuf<double> refpart;
    double ref_norm2 = 0.0;
    int sv_ng = 1, sv_wcap = 1, sv_K = 2;  // lane-per-view band geometry (max over agents)
    int sv_chunks = 1;                      // view chunks (warps) per tile (agents with > 128 views)
    // deterministic class-synchronous mode (mace_set_deterministic): one K2 launch per colour class,
    // e deltas accumulated in fixed point (ED) and folded between classes
    bool det = false;
    DBuf<unsigned long long> ED;
    std::vector<int> cls_all, cls_one;  // class boundaries of the combined and the single-agent queues
    DBuf<unsigned> heads;               // one work counter per class
    bool weighted = false;                  // K2 on weighted records: e kept as sqrt(lambda) e (k_sv.cuh)
    bool allow_weighted = true;             // mace_set_weighting
    DBuf<float> SQ;                         // sqrt(lambda) per local agent row (weighted mode)
    size_t sv_smem = 0;
    int sv_grid = 0, sv_warps = 0;
    double sv_frac = 1.0 / 16.0;  // max fraction of an agent's tiles in flight
    int colours = 4, n_sv_side = 1, sv_group = 0;  // queue geometry (mace_set_agent_groups rebuilds it)
    long sv_max_warps = 0;        // optional hard cap (0: none)
    int passes = 0;
    int num_sms = 148;
    // timing of the last iterate call
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_stage = nullptr;  // after the last H2D read of the caller's staging buffer (mace_load_data)
    // K5 PnP denoiser (cnn.cu)
    Cnn cnn;
    // consensus across ranks over NVLink peer memory (k_peer.cuh), set up by mace_peer_setup
    bool stack_zero = false;  // the stack was initialised to zero (states_from(0) needs no SpMV)
    bool peer_on = false;
    PeerArgs peer{};
    uint32_t epoch = 0;
    DBuf<unsigned> peer_counter;
    // optional per-launch timing of K2 (bench roofline): event pairs on the launch stream
    bool time_k2 = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> k2ev;
    size_t k2_used = 0;
    ~Ctx()
    {
        for (auto& e : k2ev) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
    }
};

static cudaEvent_t k2_begin(Ctx* c)
{
    if (!c->time_k2) return nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(c->stream, &cs));
    if (cs != cudaStreamCaptureStatusNone) return nullptr;  // launches captured into a graph are not timed
    if (c->k2_used == c->k2ev.size()) {
        std::pair<cudaEvent_t, cudaEvent_t> e;
        CK(cudaEventCreate(&e.first));
        CK(cudaEventCreate(&e.second));
        c->k2ev.push_back(e);
    }
    auto& e = c->k2ev[c->k2_used];
    CK(cudaEventRecord(e.first, c->stream));
    return e.second;
}

static void k2_end(Ctx* c, cudaEvent_t second)
{
    if (!second) return;
    CK(cudaEventRecord(second, c->stream));
    c->k2_used++;
}

static const int kRefBlocks = 256;
static const int kTailBlocksMax = 1024;  // k_tail: 4 blocks per SM (the stack average streams n_local x n floats)
static const int kNormBlocks = 64;

static void sync(Ctx* c) { CK(cudaStreamSynchronize(c->stream)); }

// ------------------------------------------------------------------ K2 launch helpers

template <int NV>
static void launch_raster(Ctx* c, const PassParams& P, int n_agents, int agent_base)
{
    k_icd_raster<NV><<<n_agents, 32, 0, c->stream>>>(P, agent_base);
    CK(cudaGetLastError());
}

// one super-voxel pass over P.queue (k2_inst.cu, one unit per tile side)
static void dispatch_sv(Ctx* c, const PassParams& P, int na, double frac = -1.0)
{
    SvLaunch L;
    L.device = c->device;
    L.stream = c->stream;
    L.smem = c->sv_smem;
    L.num_sms = c->num_sms;
    L.frac = frac > 0.0 ? frac : c->sv_frac;
    L.max_warps = c->sv_max_warps;
    L.agents_in_queue = na;
    L.K = c->sv_K;
    L.NG = c->sv_ng;
    L.chunks = c->sv_chunks;
    L.weighted = c->weighted;
    switch (c->S) {
        case 2: sv_launch_s2(L, P); break;
        case 4: sv_launch_s4(L, P); break;
        case 6: sv_launch_s6(L, P); break;
        case 8: sv_launch_s8(L, P); break;
        case 12: sv_launch_s12(L, P); break;
        case 16: sv_launch_s16(L, P); break;
        default: throw std::runtime_error("super-voxel side must be one of 2, 4, 6, 8, 12, 16");
    }
    c->sv_grid = L.grid;
    c->sv_warps = L.warps;
}

static PassParams base_params(Ctx* c)
{
    PassParams P{};
    P.agents = c->d_agents.p;
    P.pr = c->prior;
    P.n_side = c->n_side;
    P.S = c->S;
    P.ng = c->sv_ng;
    P.wcap = c->sv_wcap;
    P.chunks = c->sv_chunks;
    P.head = c->head.p;
    P.part = c->part.p;
    P.done = c->done.p;
    return P;
}

// One pass of every agent in [a0, a0 + na) (or all local agents if na == n_local via the combined queue).
static void run_pass(Ctx* c, int mode, float rho, const float* gimg, int a0, int na, long s0 = 0, long s1 = -1)
{
    c->stack_zero = false;  // states and (in MACE mode) the stack move
    PassParams P = base_params(c);
    P.mode = mode;
    P.rho = rho;
    P.g = gimg;
    P.s_begin = s0;
    P.s_end = s1 < 0 ? (long)c->n : s1;
    if (c->schedule == 0 && (P.s_begin != 0 || P.s_end != (long)c->n))
        throw std::runtime_error("pixel ranges need the raster schedule");
    if (c->schedule == 1) {
        cudaEvent_t ev = k2_begin(c);
        switch (c->NV) {
            case 1: launch_raster<1>(c, P, na, a0); break;
            case 2: launch_raster<2>(c, P, na, a0); break;
            case 4: launch_raster<4>(c, P, na, a0); break;
            case 8: launch_raster<8>(c, P, na, a0); break;
            default: launch_raster<16>(c, P, na, a0); break;
        }
        k2_end(c, ev);
        return;
    }
    if (na != c->n_local && na != 1) throw std::runtime_error("run_pass: single agent or all agents");
    const uint32_t* q = na == c->n_local ? c->queue.p : c->am[a0]->queue.p;
    const int nq = na == c->n_local ? c->n_items : c->am[a0]->n_sv;
    if (c->det) {
        // class-synchronous: every tile of a class stages e as it stood when the class started and
        // adds its change into the fixed-point buffer, folded into e before the next class; the
        // result does not depend on which warp took which tile or when (bitwise reproducible)
        const std::vector<int>& cs = na == c->n_local ? c->cls_all : c->cls_one;
        const int ncls = (int)cs.size() - 1;
        CK(cudaMemsetAsync(c->heads.p, 0, sizeof(unsigned) * ncls, c->stream));
        cudaEvent_t ev = k2_begin(c);
        for (int k = 0; k < ncls; ++k) {
            if (cs[k + 1] == cs[k]) continue;
            PassParams Pk = P;
            Pk.queue = q + cs[k];
            Pk.n_items = cs[k + 1] - cs[k];
            Pk.part = c->part.p + (size_t)cs[k] * 4;
            Pk.head = c->heads.p + k;
            Pk.det = 1;
            // a class is its own concurrency bound (its tiles all read the class-start snapshot), so
            // every resident warp may take one of its tiles
            dispatch_sv(c, Pk, na, 1.0);
            k_fold_delta<<<c->num_sms * 4, 256, 0, c->stream>>>(c->E.p, c->ED.p, c->total_rows, c->done.p);
            CK(cudaGetLastError());
        }
        k2_end(c, ev);
        return;
    }
    CK(cudaMemsetAsync(c->head.p, 0, sizeof(unsigned), c->stream));
    cudaEvent_t ev = k2_begin(c);
    P.queue = q;
    P.n_items = nq;
    dispatch_sv(c, P, na);
    k2_end(c, ev);
}

static void refresh(Ctx* c, int a0, int na)
{
    // e = y - A_i z for agents [a0, a0+na)
    FPParams F{c->rp.p, c->cols.p, c->vals.p, c->n_ch};
    if (na == c->n_local && a0 == 0) {
        k_fp_agents<<<std::max(1, std::min(c->num_sms * 16, (c->total_rows + 7) / 8)), 256, 0, c->stream>>>(
            F, c->d_agents.p, c->row_base.p, c->n_local, c->total_rows, c->done.p);
    } else {
        for (int i = 0; i < na; ++i) {
            const int R = c->h_agents[a0 + i].R;
            // one agent at a time: row_base[0] == 0, so the agent-local row is the warp's row index
            k_fp_agents<<<std::max(1, std::min(c->num_sms * 16, (R + 7) / 8)), 256, 0, c->stream>>>(
                F, c->d_agents.p + a0 + i, c->row_base.p, 1, R, c->done.p);
        }
    }
    CK(cudaGetLastError());
}

static void compute_theta2(Ctx* c)
{
    if (c->schedule == 1) {
        k_theta2_raster<<<c->num_sms * 8, 256, 0, c->stream>>>(c->d_agents.p, c->n_local, (int)c->n);
    } else {
        // one block per (agent, tile) item, the tile's lambda window in shared memory
        const int nb = sv_batches(c->S);
        const size_t smem = sizeof(float) * c->sv_chunks * c->sv_ng * c->sv_wcap * 32;
        auto go = [&](auto kern) {
            if (smem > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            kern<<<(unsigned)std::max(1, c->n_items), 128, smem, c->stream>>>(c->d_agents.p, c->n_items, c->queue.p,
                                                                            c->n_side, c->S, nb, c->sv_wcap, c->sv_chunks);
        };
        const int key = c->sv_K * 10 + c->sv_ng + (c->weighted ? 100 : 0);
        switch (key) {
            case 21: go(k_sv_consts<2, 1, false>); break;
            case 22: go(k_sv_consts<2, 2, false>); break;
            case 23: go(k_sv_consts<2, 3, false>); break;
            case 24: go(k_sv_consts<2, 4, false>); break;
            case 41: go(k_sv_consts<4, 1, false>); break;
            case 42: go(k_sv_consts<4, 2, false>); break;
            case 43: go(k_sv_consts<4, 3, false>); break;
            case 44: go(k_sv_consts<4, 4, false>); break;
            case 121: go(k_sv_consts<2, 1, true>); break;
            case 122: go(k_sv_consts<2, 2, true>); break;
            case 123: go(k_sv_consts<2, 3, true>); break;
            case 124: go(k_sv_consts<2, 4, true>); break;
            case 141: go(k_sv_consts<4, 1, true>); break;
            case 142: go(k_sv_consts<4, 2, true>); break;
            case 143: go(k_sv_consts<4, 3, true>); break;
            default: go(k_sv_consts<4, 4, true>); break;
        }
    }
    CK(cudaGetLastError());
}

static void consensus(Ctx* c, float scale, float* out, bool with_ref)
{
    const int blocks = kRefBlocks;
    // per slice: tree over that slice's n_real agents (W is [slice][agent][n])
    const float* rf = with_ref ? c->ref.p : nullptr;
    double* rp = with_ref ? c->refpart.p : nullptr;
    switch (c->n_real) {
        case 1: k_consensus<1><<<blocks, 256, 0, c->stream>>>(c->W.p, 1, c->n, scale, out, rf, rp, c->done.p, c->n_slices); break;
        case 2: k_consensus<2><<<blocks, 256, 0, c->stream>>>(c->W.p, 2, c->n, scale, out, rf, rp, c->done.p, c->n_slices); break;
        case 4: k_consensus<4><<<blocks, 256, 0, c->stream>>>(c->W.p, 4, c->n, scale, out, rf, rp, c->done.p, c->n_slices); break;
        case 8: k_consensus<8><<<blocks, 256, 0, c->stream>>>(c->W.p, 8, c->n, scale, out, rf, rp, c->done.p, c->n_slices); break;
        case 16: k_consensus<16><<<blocks, 256, 0, c->stream>>>(c->W.p, 16, c->n, scale, out, rf, rp, c->done.p, c->n_slices); break;
        default:
            k_consensus<0><<<blocks, 256, 0, c->stream>>>(c->W.p, c->n_real, c->n, scale, out, rf, rp, c->done.p,
                                                          c->n_slices);
    }
    CK(cudaGetLastError());
}

// dynamic shared memory of one K2 block: one warp region per view chunk (+ the multi-warp area)
static size_t sv_smem_bytes(Ctx* c, bool weighted)
{
    const int wpb = c->sv_chunks > 1 ? c->sv_chunks : kSvThreads / 32;
    return (size_t)wpb * sv_warp_bytes(c->S, c->sv_ng, c->sv_wcap, weighted) + sv_block_extra_bytes(c->S, c->sv_chunks);
}

// Switch K2 between plain records (lambda plane in shared memory) and weighted records
// a sqrt(lambda) with the error sinogram kept as sqrt(lambda) e (k_sv.cuh).  Called when data
// are loaded; the caller refreshes e afterwards (mace_set_state / mace_states_from).
static void set_weighted(Ctx* c, bool on)
{
    if (on && !c->SQ.p) {
        c->SQ.alloc(c->total_rows);
        CK(cudaMemset(c->SQ.p, 0, sizeof(float) * c->total_rows));
    }
    for (int a = 0; a < c->n_real && on; ++a) {
        AgentMem& m = *c->am[a];
        if (!m.recw.p) m.recw.alloc(m.rec.n);
    }
    const bool changed = on != c->weighted;
    c->weighted = on;
    if (!changed) return;  // the agents already point at the right records and sqrt(lambda) rows
    std::vector<int> rb(c->n_local + 1, 0);
    CK(cudaMemcpy(rb.data(), c->row_base.p, sizeof(int) * (c->n_local + 1), cudaMemcpyDeviceToHost));
    for (int va = 0; va < c->n_local; ++va) {
        AgentMem& m = *c->am[va % c->n_real];
        AgentDev& A = c->h_agents[va];
        A.rec0 = m.rec.p;
        A.recw = on ? m.recw.p : nullptr;
        A.rec = on ? m.recw.p : m.rec.p;
        A.sq = on ? c->SQ.p + rb[va] : nullptr;
    }
    c->sv_smem = sv_smem_bytes(c, on);
    if (c->sv_smem > 227 * 1024) throw std::runtime_error("super-voxel band does not fit in shared memory");
    CK(cudaMemcpyAsync(c->d_agents.p, c->h_agents.data(), sizeof(AgentDev) * c->n_local, cudaMemcpyHostToDevice,
                       c->stream));
    sync(c);
}

static void ensure_log(Ctx* c, int n)
{
    if (n > c->log_cap) {
        DBuf<double> nl;
        nl.alloc((size_t)n * 4);
        if (c->log_cap) CK(cudaMemcpyAsync(nl.p, c->log.p, sizeof(double) * 4 * c->log_cap, cudaMemcpyDeviceToDevice, c->stream));
        std::swap(c->log.p, nl.p);
        std::swap(c->log.n, nl.n);
        c->log_cap = n;
    }
}

}  // namespace mace

using namespace mace;

#define API_BEGIN try {
#define API_END                                   \
    }                                             \
    catch (const std::exception& ex)              \
    {                                             \
        set_error(ex.what());                     \
        return -1;                                \
    }                                             \
    return 0;

static Ctx* C(void* p)
{
    if (!p) throw std::runtime_error("null context");
    Ctx* c = static_cast<Ctx*>(p);
    CK(cudaSetDevice(c->device));
    return c;
}

extern "C" {

const char* mace_last_error(void) { return g_err.c_str(); }
int mace_abi_version(void) { return MACE_ABI_VERSION; }

// ------------------------------------------------------------------ tracer
int mace_sysmat_trace(int n_side, double pixel_pitch, int n_views, int n_channels, const double* ux,
                      const double* uy, const double* ex, const double* ey, const double* offsets, int n_threads,
                      void** handle)
{
    API_BEGIN
    if (n_side < 1 || n_views < 1 || n_channels < 1 || !(pixel_pitch > 0)) throw std::runtime_error("bad geometry");
    *handle = sysmat_trace(n_side, pixel_pitch, n_views, n_channels, ux, uy, ex, ey, offsets, n_threads);
    API_END
}

int mace_sysmat_read(const char* path, int64_t* dims3, void** handle)
{
    API_BEGIN
    int64_t n = 0;
    SysMat* m = sysmat_read(path, &n);
    dims3[0] = m->n_views;
    dims3[1] = m->n_ch;
    dims3[2] = n;
    *handle = m;
    API_END
}

int64_t mace_sysmat_view_nnz(void* handle, int view)
{
    SysMat* s = static_cast<SysMat*>(handle);
    if (!s || view < 0 || view >= s->n_views) return -1;
    return (int64_t)s->views[view].cols.size();
}

int mace_sysmat_take_view(void* handle, int view, int64_t* row_ptr, int32_t* cols, double* lens)
{
    API_BEGIN
    SysMat* s = static_cast<SysMat*>(handle);
    if (!s || view < 0 || view >= s->n_views) throw std::runtime_error("bad view");
    SysMatView& V = s->views[view];
    std::memcpy(row_ptr, V.row_ptr.data(), V.row_ptr.size() * sizeof(int64_t));
    std::memcpy(cols, V.cols.data(), V.cols.size() * sizeof(int32_t));
    std::memcpy(lens, V.lens.data(), V.lens.size() * sizeof(double));
    SysMatView().row_ptr.swap(V.row_ptr);
    std::vector<int32_t>().swap(V.cols);
    std::vector<double>().swap(V.lens);
    API_END
}

void mace_sysmat_free(void* handle) { delete static_cast<SysMat*>(handle); }

// ------------------------------------------------------------------ context
int mace_ctx_create(int device, void** out)
{
    API_BEGIN
    auto c = std::make_unique<Ctx>();
    c->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    CK(cudaEventCreateWithFlags(&c->ev_stage, cudaEventDisableTiming));
    c->head.alloc(1);
    c->done.alloc(2);
    c->sums5.alloc(5);
    c->norm_scratch.alloc(5 * std::max(kNormBlocks, kTailBlocksMax));  // k_norms and k_tail block sums
    c->norm_counter.alloc(1);
    CK(cudaMemset(c->norm_counter.p, 0, sizeof(unsigned)));
    CK(cudaMemset(c->head.p, 0, sizeof(unsigned)));
    CK(cudaMemset(c->done.p, 0, 2 * sizeof(int)));
    *out = c.release();
    API_END
}

void mace_ctx_destroy(void* p)
{
    if (!p) return;
    Ctx* c = static_cast<Ctx*>(p);
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    cudaEventDestroy(c->ev0);
    cudaEventDestroy(c->ev1);
    if (c->ev_stage) cudaEventDestroy(c->ev_stage);
    delete c;
}

int mace_ctx_stream(void* p, void** stream)
{
    API_BEGIN
    *stream = (void*)C(p)->stream;
    API_END
}

int mace_sync(void* p)
{
    API_BEGIN
    sync(C(p));
    API_END
}

int mace_load_matrix(void* p, int n_side, int n_views, int n_ch, const int64_t* row_ptr, const int32_t* cols,
                     const float* vals)
{
    API_BEGIN
    Ctx* c = C(p);
    const int64_t rows = (int64_t)n_views * n_ch;
    c->n_side = n_side;
    c->n_views = n_views;
    c->n_ch = n_ch;
    c->n = (size_t)n_side * n_side;
    c->nnz = row_ptr[rows];
    c->rp.alloc(rows + 1);
    c->cols.alloc(c->nnz);
    c->vals.alloc(c->nnz);
    CK(cudaMemcpy(c->rp.p, row_ptr, sizeof(int64_t) * (rows + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->cols.p, cols, sizeof(int32_t) * c->nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->vals.p, vals, sizeof(float) * c->nnz, cudaMemcpyHostToDevice));
    c->y.alloc(rows);
    c->lam.alloc(rows);
    c->wbar.alloc(c->n);
    c->g.alloc(c->n);
    c->ref.alloc(c->n);
    c->wsum.alloc(c->n);
    c->refpart.alloc(kRefBlocks);
    API_END
}

int mace_set_prior(void* p, int kind, double p_, double q, double T, double sx, double eps)
{
    API_BEGIN
    Ctx* c = C(p);
    PriorC& P = c->prior;
    P.kind = kind;
    P.p_is_2 = (p_ == 2.0);
    P.eps2 = (float)(2.0 * eps);
    P.inv_Tsx = (float)(1.0 / (T * sx));
    P.inv_sxp = (float)(1.0 / std::pow(sx, p_));
    P.qp = (float)(q / p_);
    P.qmp = (float)(q - p_);
    P.pm1 = (float)(p_ - 1.0);
    P.pm2 = (float)(p_ - 2.0);
    P.floor_ = (float)(1e-9 * T * sx);
    P.inv_sx2 = (float)(1.0 / (sx * sx));
    P.p = p_;
    P.q = q;
    P.T = T;
    P.sx = sx;
    P.eps = eps;
    API_END
}

int mace_setup_agents(void* p, int n_agents, const int* view_counts, const int* views, int schedule, int svs,
                      int colours, int n_threads, int n_slices)
{
    API_BEGIN
    Ctx* c = C(p);
    if (!c->nnz && !c->rp.p) throw std::runtime_error("load the system matrix first");
    if (n_agents < 1 || n_agents > 64) throw std::runtime_error("1..64 agents per context");
    if (n_slices < 1 || n_agents * n_slices > 1024) throw std::runtime_error("1..1024 agents x slices per context");
    if (schedule == 1 && n_slices != 1) throw std::runtime_error("multi-slice batches need the super-voxel schedule");
    if (schedule == 0 && (svs < 2 || (svs & 1))) throw std::runtime_error("super-voxel side must be even and >= 2");
    // local (virtual) agent va = slice * n_agents + a shares real agent a's layout
    const int n_local = n_agents * n_slices;
    c->n_real = n_agents;
    c->n_slices = n_slices;
    c->n_local = n_local;
    c->schedule = schedule;
    c->S = schedule == 0 ? svs : c->n_side;
    c->am.clear();
    c->SQ.free();
    c->weighted = false;
    int off = 0;
    for (int a = 0; a < n_agents; ++a) {
        auto m = std::make_unique<AgentMem>();
        m->views.assign(views + off, views + off + view_counts[a]);
        off += view_counts[a];
        for (int v : m->views)
            if (v < 0 || v >= c->n_views) throw std::runtime_error("view index out of range");
        m->R = (int)m->views.size() * c->n_ch;
        c->am.push_back(std::move(m));
    }
    // host layout build from a transient host copy of the global CSR
    const int64_t rows = (int64_t)c->n_views * c->n_ch;
    std::vector<int64_t> h_rp(rows + 1);
    std::vector<int32_t> h_cols(c->nnz);
    std::vector<float> h_vals(c->nnz);
    CK(cudaMemcpy(h_rp.data(), c->rp.p, sizeof(int64_t) * (rows + 1), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h_cols.data(), c->cols.p, sizeof(int32_t) * c->nnz, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h_vals.data(), c->vals.p, sizeof(float) * c->nnz, cudaMemcpyDeviceToHost));
    if (n_threads <= 0) n_threads = (int)std::max(1u, std::thread::hardware_concurrency());
    int ng_all = 1;  // one record geometry for the context (the kernel is specialised on it)
    for (int a = 0; a < n_agents; ++a) ng_all = std::max(ng_all, ((int)c->am[a]->views.size() + 31) / 32);
    std::vector<std::exception_ptr> errs(n_agents);
    std::vector<RasterLayout> rl(n_agents);
    std::vector<SVLayout> sl(n_agents);
    {
        std::atomic<int> next(0);
        auto work = [&]() {
            for (;;) {
                int a = next.fetch_add(1);
                if (a >= n_agents) break;
                try {
                    AgentCSC csc;
                    build_agent_csc(c->n_side, c->n_ch, h_rp.data(), h_cols.data(), h_vals.data(), c->am[a]->views, csc);
                    c->am[a]->nnz = csc.col_ptr.back();
                    if (schedule == 1) build_raster_layout(csc, (int)c->n, rl[a]);
                    else build_sv_layout(csc, c->n_side, c->n_ch, (int)c->am[a]->views.size(), svs, sl[a], ng_all);
                } catch (...) {
                    errs[a] = std::current_exception();
                }
            }
        };
        std::vector<std::thread> th;
        for (int t = 0; t < std::min(n_threads, n_agents); ++t) th.emplace_back(work);
        for (auto& t : th) t.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    }
    // per real agent: layout on the device
    int max_col = 0, n_sv_side = 1;
    c->sv_ng = 1;
    c->sv_wcap = 1;
    c->sv_K = 2;
    c->sv_chunks = 1;
    for (int a = 0; a < n_agents; ++a) {
        AgentMem& m = *c->am[a];
        m.d_views.alloc(m.views.size());
        CK(cudaMemcpy(m.d_views.p, m.views.data(), sizeof(int) * m.views.size(), cudaMemcpyHostToDevice));
        if (schedule == 1) {
            RasterLayout& L = rl[a];
            m.rpix.alloc(L.pix.size());
            m.ridx.alloc(L.idx.size());
            m.rval.alloc(L.val.size());
            CK(cudaMemcpy(m.rpix.p, L.pix.data(), sizeof(int2) * L.pix.size(), cudaMemcpyHostToDevice));
            if (L.idx.size()) {
                CK(cudaMemcpy(m.ridx.p, L.idx.data(), sizeof(uint32_t) * L.idx.size(), cudaMemcpyHostToDevice));
                CK(cudaMemcpy(m.rval.p, L.val.data(), sizeof(float) * L.val.size(), cudaMemcpyHostToDevice));
            }
            m.entries = (int64_t)L.idx.size();
            m.max_col = L.max_col;
            m.n_sv = 1;
            m.n_sv_side = 1;
        } else {
            SVLayout& L = sl[a];
            m.band.alloc(L.band.size());
            m.rec.alloc(L.data.size());
            CK(cudaMemcpy(m.band.p, L.band.data(), sizeof(int2) * L.band.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(m.rec.p, L.data.data(), sizeof(uint32_t) * L.data.size(), cudaMemcpyHostToDevice));
            m.nb = L.nb;
            m.rec_words = L.rec;
            m.entries = L.entries;
            m.max_col = L.max_col;
            m.wcap = L.wcap;
            m.ng = L.ng;
            m.K = L.K;
            m.chunks = L.chunks;
            m.n_sv = L.n_sv;
            m.n_sv_side = L.n_sv_side;
            m.duplicates = L.duplicates;
            n_sv_side = L.n_sv_side;
            if (n_slices == 1) {  // single-agent queue for plain passes (AgentWorkspace)
                std::vector<uint32_t> q1 = build_queue(1, L.n_sv_side, colours);
                for (auto& v : q1) v |= ((uint32_t)a << kAgentShift);
                m.queue.alloc(q1.size());
                CK(cudaMemcpy(m.queue.p, q1.data(), sizeof(uint32_t) * q1.size(), cudaMemcpyHostToDevice));
            }
        }
        max_col = std::max(max_col, m.max_col);
        c->sv_ng = std::max(c->sv_ng, m.ng);
        c->sv_wcap = std::max(c->sv_wcap, m.wcap);
        c->sv_K = std::max(c->sv_K, m.K);
        c->sv_chunks = std::max(c->sv_chunks, m.chunks);
    }
    // per local (virtual) agent: data arrays; each {e, lambda} block starts on a 16-byte boundary
    std::vector<int> rb(n_local + 1, 0);
    // (K2 reads e windows as 32-byte aligned spans, which may run up to 7 rows past R)
    for (int va = 0; va < n_local; ++va) rb[va + 1] = rb[va] + ((c->am[va % n_agents]->R + 7) & ~7);
    c->total_rows = rb[n_local];
    c->row_base.alloc(n_local + 1);
    CK(cudaMemcpy(c->row_base.p, rb.data(), sizeof(int) * (n_local + 1), cudaMemcpyHostToDevice));
    c->E.alloc(c->total_rows);
    c->LAM.alloc(c->total_rows);
    c->Y.alloc(c->total_rows);
    c->Z.alloc((size_t)n_local * c->n);
    c->W.alloc((size_t)n_local * c->n);
    c->TH.alloc((size_t)n_local * c->n);
    c->VT.alloc((size_t)n_local * c->n);
    CK(cudaMemset(c->Z.p, 0, sizeof(float) * n_local * c->n));
    CK(cudaMemset(c->W.p, 0, sizeof(float) * n_local * c->n));
    CK(cudaMemset(c->E.p, 0, sizeof(float) * c->total_rows));
    CK(cudaMemset(c->LAM.p, 0, sizeof(float) * c->total_rows));
    std::vector<size_t> bcb(n_local + 1, 0);  // batch-constant blocks: one per local agent
    for (int va = 0; va < n_local; ++va)
        bcb[va + 1] = bcb[va] + (size_t)c->am[va % n_agents]->n_sv * c->am[va % n_agents]->nb * 16;
    c->BC.alloc(std::max<size_t>(bcb[n_local], 1));
    CK(cudaMemset(c->BC.p, 0, sizeof(float) * std::max<size_t>(bcb[n_local], 1)));
    std::vector<size_t> lbb(n_local + 1, 0);  // band-lambda blocks
    for (int va = 0; va < n_local; ++va)
        lbb[va + 1] = lbb[va] + (schedule == 0 ? (size_t)c->am[va % n_agents]->n_sv * c->sv_chunks * c->sv_ng * c->sv_wcap * 32 : 0);
    c->LB.alloc(std::max<size_t>(lbb[n_local], 1));
    c->h_agents.assign(n_local, AgentDev{});
    for (int va = 0; va < n_local; ++va) {
        const int a = va % n_agents;
        AgentMem& m = *c->am[a];
        AgentDev& A = c->h_agents[va];
        A.e = c->E.p + rb[va];
        A.lam = c->LAM.p + rb[va];
        A.y = c->Y.p + rb[va];
        A.z = c->Z.p + (size_t)va * c->n;
        A.w = c->W.p + (size_t)va * c->n;
        A.th = c->TH.p + (size_t)va * c->n;
        A.vt = c->VT.p + (size_t)va * c->n;
        A.slice = va / n_agents;
        A.views = m.d_views.p;
        A.R = m.R;
        A.V = (int)m.views.size();
        A.rpix = m.rpix.p;
        A.ridx = m.ridx.p;
        A.rval = m.rval.p;
        A.band = m.band.p;
        A.rec = m.rec.p;
        A.rec0 = m.rec.p;
        A.recw = nullptr;
        A.sq = nullptr;
        A.bc = schedule == 0 ? c->BC.p + bcb[va] : nullptr;
        A.lb = schedule == 0 ? c->LB.p + lbb[va] : nullptr;
        A.ng = m.ng;
        A.rec_words = m.rec_words;
        A.n_sv_side = m.n_sv_side;
        A.beta_eff = m.beta_eff;
        A.inv_s2 = m.inv_s2;
        A.clamp = m.clamp;
    }
    // raster pass: one warp per column, 4 entries per lane per chunk of 128
    c->NV = 1;
    while (c->NV < 16 && 128 * c->NV < max_col) c->NV *= 2;
    if (max_col > 128 * 16) throw std::runtime_error("column longer than 2048 entries");
    if (schedule == 0) {
        c->colours = colours;
        c->n_sv_side = n_sv_side;
        c->sv_group = 0;
        std::vector<uint32_t> q = build_queue(n_agents, n_sv_side, colours, n_slices);
        c->queue.alloc(q.size());
        CK(cudaMemcpy(c->queue.p, q.data(), sizeof(uint32_t) * q.size(), cudaMemcpyHostToDevice));
        c->n_items = (int)q.size();
        for (int a = 0; a < n_agents; ++a) {
            if (c->am[a]->K != c->sv_K) throw std::runtime_error("agents with different (pixel, view) slot widths");
            if (c->am[a]->chunks != c->sv_chunks) throw std::runtime_error("agents with different view-chunk counts");
        }
        c->weighted = false;
        c->sv_smem = sv_smem_bytes(c, false);
        if (c->sv_smem > 227 * 1024) throw std::runtime_error("super-voxel band does not fit in shared memory");
    } else {
        c->n_items = n_local;
    }
    c->part.alloc((size_t)std::max(c->n_items, n_local) * 4);
    c->d_agents.alloc(n_local);
    CK(cudaMemcpy(c->d_agents.p, c->h_agents.data(), sizeof(AgentDev) * n_local, cudaMemcpyHostToDevice));
    // consensus images are [slice][n]
    c->wbar.alloc(c->n * n_slices);
    c->g.alloc(c->n * n_slices);
    c->wsum.alloc(c->n * n_slices);
    c->passes = 0;
    API_END
}

int mace_agent_info(void* p, int local, int64_t* info /* [8] */)
{
    API_BEGIN
    Ctx* c = C(p);
    if (local < 0 || local >= c->n_real) throw std::runtime_error("bad agent");
    AgentMem& m = *c->am[local];
    info[0] = m.nnz;
    info[1] = m.entries;
    info[2] = m.R;
    info[3] = m.max_col;
    info[4] = m.wcap;
    info[5] = m.n_sv;
    info[6] = m.duplicates;
    info[7] = c->sv_wcap;
    API_END
}

int mace_ctx_info(void* p, int64_t* info /* [10] */)
{
    API_BEGIN
    Ctx* c = C(p);
    info[0] = c->nnz;
    info[1] = c->n_items;
    info[2] = c->NV;
    info[3] = (int64_t)c->sv_smem;
    info[4] = c->sv_warps;
    info[5] = c->num_sms;
    info[6] = c->passes;
    info[7] = c->S;
    info[8] = c->weighted ? 1 : 0;
    info[9] = 0;
    API_END
}

int mace_set_schedule(void* p, double concurrency, int64_t max_warps)
{
    API_BEGIN
    Ctx* c = C(p);
    if (!(concurrency > 0.0) || concurrency > 1.0) throw std::runtime_error("concurrency must be in (0, 1]");
    c->sv_frac = concurrency;
    c->sv_max_warps = (long)max_warps;
    API_END
}

// class boundaries of a colour-ordered queue (build_queue with group 0): item i belongs to class
// (tile row mod C, tile col mod C); classes must be contiguous and in order
static std::vector<int> class_bounds(const std::vector<uint32_t>& q, int nss, int colours)
{
    const int C = std::max(1, std::min(colours, nss));
    std::vector<int> cs(C * C + 1, (int)q.size());
    int prev = -1;
    for (size_t i = 0; i < q.size(); ++i) {
        const int sv = (int)(q[i] & kSvMask), k = ((sv / nss) % C) * C + (sv % nss) % C;
        if (k < prev) throw std::runtime_error("deterministic mode: the work queue is not in colour-class order");
        for (int j = prev + 1; j <= k; ++j) cs[j] = (int)i;
        prev = k;
    }
    return cs;
}

// Deterministic super-voxel passes: one K2 launch per colour class, every tile of a
// class reading e as it stood at the class start, the tiles' e changes summed in 2^-40 fixed point
// (order-independent) and folded between classes.  Bitwise reproducible run to run and for any grid
// size / concurrency, at the cost of one launch and one fold per class.
int mace_set_deterministic(void* p, int on)
{
    API_BEGIN
    Ctx* c = C(p);
    if (on && c->schedule != 0) throw std::runtime_error("deterministic mode needs the super-voxel schedule");
    if (on && c->sv_group) throw std::runtime_error("deterministic mode needs agent groups off");
    sync(c);
    if (on) {
        if (!c->ED.p) {
            c->ED.alloc(c->total_rows);
            CK(cudaMemset(c->ED.p, 0, sizeof(unsigned long long) * c->total_rows));
        }
        std::vector<int> rb(c->n_local + 1, 0);
        CK(cudaMemcpy(rb.data(), c->row_base.p, sizeof(int) * (c->n_local + 1), cudaMemcpyDeviceToHost));
        for (int va = 0; va < c->n_local; ++va) c->h_agents[va].ed = c->ED.p + rb[va];
        CK(cudaMemcpy(c->d_agents.p, c->h_agents.data(), sizeof(AgentDev) * c->n_local, cudaMemcpyHostToDevice));
        c->cls_all = class_bounds(build_queue(c->n_real, c->n_sv_side, c->colours, c->n_slices, 0), c->n_sv_side,
                                  c->colours);
        c->cls_one = class_bounds(build_queue(1, c->n_sv_side, c->colours), c->n_sv_side, c->colours);
        if (c->heads.n < c->cls_all.size()) c->heads.alloc(c->cls_all.size());
    }
    c->det = on != 0;
    API_END
}

int mace_set_agent_groups(void* p, int group)
{
    API_BEGIN
    Ctx* c = C(p);
    if (c->schedule != 0) throw std::runtime_error("agent groups need the super-voxel schedule");
    if (c->det && group) throw std::runtime_error("agent groups need the deterministic mode off");
    if (group < 0) throw std::runtime_error("group must be >= 0");
    std::vector<uint32_t> q = build_queue(c->n_real, c->n_sv_side, c->colours, c->n_slices, group);
    if ((int)q.size() != c->n_items) throw std::runtime_error("queue size changed");
    sync(c);
    CK(cudaMemcpy(c->queue.p, q.data(), sizeof(uint32_t) * q.size(), cudaMemcpyHostToDevice));
    c->sv_group = group;
    API_END
}

int mace_set_agent_params(void* p, int local, double beta_eff, double inv_sigma2, int clamp)
{
    API_BEGIN
    Ctx* c = C(p);
    if (local >= c->n_local) throw std::runtime_error("bad agent");
    int a0 = local < 0 ? 0 : local, a1 = local < 0 ? c->n_local : local + 1;
    for (int a = a0; a < a1; ++a) {
        AgentMem& m = *c->am[a % c->n_real];
        m.beta_eff = (float)beta_eff;
        m.inv_s2 = (float)inv_sigma2;
        m.clamp = clamp;
        c->h_agents[a].beta_eff = (float)beta_eff;
        c->h_agents[a].inv_s2 = (float)inv_sigma2;
        c->h_agents[a].clamp = clamp;
    }
    CK(cudaMemcpyAsync(c->d_agents.p, c->h_agents.data(), sizeof(AgentDev) * c->n_local, cudaMemcpyHostToDevice,
                       c->stream));
    sync(c);
    API_END
}

int mace_set_weighting(void* p, int allow)
{
    API_BEGIN
    C(p)->allow_weighted = allow != 0;
    API_END
}

int mace_load_data(void* p, const float* y, const float* lam)
{
    API_BEGIN
    Ctx* c = C(p);
    // y / lam: [n_slices][n_views * n_ch] (one sinogram per slice of a batch)
    const size_t rows = (size_t)c->n_views * c->n_ch;
    const size_t total = rows * std::max(1, c->n_slices);
    if (c->y.n < total) {
        c->y.alloc(total);
        c->lam.alloc(total);
    }
    CK(cudaMemcpyAsync(c->y.p, y, sizeof(float) * total, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->lam.p, lam, sizeof(float) * total, cudaMemcpyHostToDevice, c->stream));
    CK(cudaEventRecord(c->ev_stage, c->stream));  // the host buffers may be reused once this completes
    if (c->n_local) {
        // weighted records need one lambda per record (a single slice) and lambda > 0 everywhere,
        // so that e = e' / sqrt(lambda) stays recoverable (mace_get_error)
        bool want = c->allow_weighted && c->schedule == 0 && c->n_slices == 1;
        if (want) {  // count of weights that are not > 0 (NaN included): an integer sum the host
                     // compiler vectorises, unlike a float min reduction (0.75 -> 0.08 ms at config 1)
            unsigned bad = 0;
            for (size_t i = 0; i < total; ++i) bad += !(lam[i] > 0.f);
            want = bad == 0;
        }
        set_weighted(c, want);
        k_gather_data<<<c->num_sms * 4, 256, 0, c->stream>>>(c->d_agents.p, c->row_base.p, c->n_local, c->total_rows,
                                                              c->n_ch, c->y.p, c->lam.p, (int64_t)rows);
        CK(cudaGetLastError());
        compute_theta2(c);
    }
    API_END
}

// wait until the last mace_load_data has finished reading its host buffers (a pinned staging
// buffer may then be refilled; the copies themselves run asynchronously)
int mace_stage_wait(void* p)
{
    API_BEGIN
    CK(cudaEventSynchronize(C(p)->ev_stage));
    API_END
}

int mace_set_state(void* p, int local, const float* x)
{
    API_BEGIN
    Ctx* c = C(p);
    int a0 = local < 0 ? 0 : local, na = local < 0 ? c->n_local : 1;
    for (int a = a0; a < a0 + na; ++a)
        CK(cudaMemcpyAsync(c->h_agents[a].z, x, sizeof(float) * c->n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->done.p, 0, 2 * sizeof(int), c->stream));
    refresh(c, a0, na);
    sync(c);
    API_END
}

int mace_get_state(void* p, int local, float* x)
{
    API_BEGIN
    Ctx* c = C(p);
    CK(cudaMemcpyAsync(x, c->h_agents.at(local).z, sizeof(float) * c->n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    API_END
}

int mace_get_error(void* p, int local, float* e)
{
    API_BEGIN
    Ctx* c = C(p);
    const AgentDev& A = c->h_agents.at(local);
    CK(cudaMemcpyAsync(e, A.e, sizeof(float) * A.R, cudaMemcpyDeviceToHost, c->stream));
    std::vector<float> sq;
    if (A.sq) {
        sq.resize(A.R);
        CK(cudaMemcpyAsync(sq.data(), A.sq, sizeof(float) * A.R, cudaMemcpyDeviceToHost, c->stream));
    }
    sync(c);
    for (size_t r = 0; r < sq.size(); ++r) e[r] /= sq[r];  // weighted mode: e = e' / sqrt(lambda)
    API_END
}

int mace_get_theta2(void* p, int local, float* th)
{
    API_BEGIN
    Ctx* c = C(p);
    CK(cudaMemcpyAsync(th, c->h_agents.at(local).th, sizeof(float) * c->n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    API_END
}

// the super-voxel batch constants of local agent `local` (k_sv_consts): [n_sv][nb][16] floats =
// theta2 of the batch's four slots, cross terms c01 c02 c03 c12 c13 c23, 6 unused
int mace_get_batch_consts(void* p, int local, float* out, int64_t* count)
{
    API_BEGIN
    Ctx* c = C(p);
    if (c->schedule != 0) throw std::runtime_error("batch constants need the super-voxel schedule");
    const AgentMem& m = *c->am.at(local % c->n_real);
    const size_t cnt = (size_t)m.n_sv * m.nb * 16;
    if (count) *count = (int64_t)cnt;
    if (out) {
        CK(cudaMemcpyAsync(out, c->h_agents.at(local).bc, sizeof(float) * cnt, cudaMemcpyDeviceToHost, c->stream));
        sync(c);
    }
    API_END
}

int mace_refresh(void* p, int local)
{
    API_BEGIN
    Ctx* c = C(p);
    CK(cudaMemsetAsync(c->done.p, 0, 2 * sizeof(int), c->stream));
    if (local < 0) refresh(c, 0, c->n_local);
    else refresh(c, local, 1);
    sync(c);
    API_END
}

// Plain partial-update passes toward an explicit target v (icd.py:272-283); dsq[k] = sum alpha^2 of pass k.
int mace_pass(void* p, int local, const float* v, int n_passes, int64_t s_begin, int64_t s_end, double* dsq)
{
    API_BEGIN
    Ctx* c = C(p);
    if (local < 0 || local >= c->n_local) throw std::runtime_error("bad agent");
    if (c->n_slices != 1) throw std::runtime_error("plain passes need a single-slice context");
    CK(cudaMemcpyAsync(c->h_agents[local].vt, v, sizeof(float) * c->n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(c->done.p, 0, 2 * sizeof(int), c->stream));
    std::vector<double> part;
    for (int k = 0; k < n_passes; ++k) {
        run_pass(c, 0, 0.f, nullptr, local, 1, s_begin, s_end);
        if (dsq) {
            const int items = c->schedule == 1 ? 1 : c->am[local]->n_sv;
            part.resize((size_t)items * 4);
            CK(cudaMemcpyAsync(part.data(), c->part.p, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, c->stream));
            sync(c);
            double s = 0;
            for (int i = 0; i < items; ++i) s += part[(size_t)i * 4];
            dsq[k] = s;
        }
    }
    sync(c);
    API_END
}

// Every local agent's proximal map at once (equilibrium_residuals, mace.py:440-452): agent i starts
// from x0 with target v_i (v: [n_local][n]) and runs plain passes of the context's schedule until
// sqrt(sum alpha^2) / ||z_i|| < tol for every agent (prox_solve's test, icd.py:286-303), refreshing e
// every 50 passes.  passes_out = passes run, rel_out[n_local] = each agent's last relative update.
// The solutions stay in the agents' states (mace_get_state).
int mace_prox_all(void* p, const float* v, const float* x0, int max_passes, double tol, int* passes_out,
                  double* rel_out)
{
    API_BEGIN
    Ctx* c = C(p);
    if (c->n_slices != 1) throw std::runtime_error("prox_all needs a single-slice context");
    const int NL = c->n_local;
    for (int a = 0; a < NL; ++a) {
        CK(cudaMemcpyAsync(c->h_agents[a].vt, v + (size_t)a * c->n, sizeof(float) * c->n, cudaMemcpyHostToDevice,
                           c->stream));
        CK(cudaMemcpyAsync(c->h_agents[a].z, x0, sizeof(float) * c->n, cudaMemcpyHostToDevice, c->stream));
    }
    CK(cudaMemsetAsync(c->done.p, 0, 2 * sizeof(int), c->stream));
    refresh(c, 0, NL);
    // item -> agent of the pass's queue (super-voxel: queue order; raster: one item per agent)
    std::vector<int> item_agent(c->n_items);
    if (c->schedule == 0) {
        std::vector<uint32_t> q(c->n_items);
        CK(cudaMemcpyAsync(q.data(), c->queue.p, sizeof(uint32_t) * q.size(), cudaMemcpyDeviceToHost, c->stream));
        sync(c);
        for (int i = 0; i < c->n_items; ++i) item_agent[i] = (int)(q[i] >> kAgentShift);
    } else {
        for (int i = 0; i < c->n_items; ++i) item_agent[i] = i;
    }
    std::vector<double> part((size_t)c->n_items * 4), dsq(NL), rel(NL, INFINITY);
    std::vector<float> z((size_t)NL * c->n);
    int k = 0;
    for (; k < max_passes; ++k) {
        run_pass(c, 0, 0.f, nullptr, 0, NL);
        if ((k + 1) % 50 == 0) refresh(c, 0, NL);  // icd.py:29,298-299
        CK(cudaMemcpyAsync(part.data(), c->part.p, sizeof(double) * part.size(), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(z.data(), c->Z.p, sizeof(float) * z.size(), cudaMemcpyDeviceToHost, c->stream));
        sync(c);
        std::fill(dsq.begin(), dsq.end(), 0.0);
        for (int i = 0; i < c->n_items; ++i) dsq[item_agent[i]] += part[(size_t)i * 4];
        double worst = 0.0;
        for (int a = 0; a < NL; ++a) {
            double zz = 0.0;
            const float* za = z.data() + (size_t)a * c->n;
            for (size_t s = 0; s < c->n; ++s) zz += (double)za[s] * za[s];
            rel[a] = std::sqrt(dsq[a]) / std::max(std::sqrt(zz), 1e-300);
            worst = std::max(worst, rel[a]);
        }
        if (worst < tol) {
            ++k;
            break;
        }
    }
    c->passes += k;
    if (passes_out) *passes_out = k;
    if (rel_out)
        for (int a = 0; a < NL; ++a) rel_out[a] = rel[a];
    API_END
}

// Forward projection of an image: out (n_views x n_ch) = A x  (geometry.py:261-270)
int mace_forward_project(void* p, const float* x, float* out)
{
    API_BEGIN
    Ctx* c = C(p);
    const int rows = c->n_views * c->n_ch;
    DBuf<float> dx, dout;
    dx.alloc(c->n);
    dout.alloc(rows);
    CK(cudaMemcpyAsync(dx.p, x, sizeof(float) * c->n, cudaMemcpyHostToDevice, c->stream));
    FPParams F{c->rp.p, c->cols.p, c->vals.p, c->n_ch};
    k_fp_rows<<<std::max(1, std::min(c->num_sms * 16, (rows + 7) / 8)), 256, 0, c->stream>>>(F, rows, dx.p, dout.p,
                                                                                             nullptr, nullptr, nullptr);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, dout.p, sizeof(float) * rows, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    API_END
}

// f(x) = 1/2 sum lambda (y - Ax)^2 + beta h(x)  (models.py:235-278), fp64 accumulation
int mace_cost(void* p, const float* x, double beta, double* like, double* prior)
{
    API_BEGIN
    Ctx* c = C(p);
    const int rows = c->n_views * c->n_ch;
    DBuf<float> dx;
    dx.alloc(c->n);
    CK(cudaMemcpyAsync(dx.p, x, sizeof(float) * c->n, cudaMemcpyHostToDevice, c->stream));
    const int b1 = std::max(1, std::min(c->num_sms * 8, (rows + 7) / 8)), b2 = c->num_sms * 2;
    DBuf<double> pp;
    pp.alloc(b1 + b2);
    FPParams F{c->rp.p, c->cols.p, c->vals.p, c->n_ch};
    k_fp_rows<<<b1, 256, 0, c->stream>>>(F, rows, dx.p, nullptr, c->y.p, c->lam.p, pp.p);
    k_prior_cost<<<b2, 256, 0, c->stream>>>(dx.p, c->n_side, c->prior, pp.p + b1);
    CK(cudaGetLastError());
    std::vector<double> h(b1 + b2);
    CK(cudaMemcpyAsync(h.data(), pp.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    double L = 0, P = 0;
    for (int i = 0; i < b1; ++i) L += h[i];
    for (int i = 0; i < b2; ++i) P += h[b1 + i];
    *like = L;
    *prior = beta * P;
    API_END
}

// out = A^T sino (fp64 accumulation), the exact transpose of mace_forward_project (geometry.py:273-282)
int mace_back_project(void* p, const float* sino, double* out)
{
    API_BEGIN
    Ctx* c = C(p);
    const int rows = c->n_views * c->n_ch;
    DBuf<float> ds;
    DBuf<double> dout;
    ds.alloc(rows);
    dout.alloc(c->n);
    CK(cudaMemcpyAsync(ds.p, sino, sizeof(float) * rows, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(dout.p, 0, sizeof(double) * c->n, c->stream));
    FPParams F{c->rp.p, c->cols.p, c->vals.p, c->n_ch};
    k_bp_sino<<<std::max(1, std::min(c->num_sms * 8, (rows + 7) / 8)), 256, 0, c->stream>>>(F, rows, ds.p, dout.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, dout.p, sizeof(double) * c->n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    API_END
}

// gradient of the MAP cost f = likelihood + beta prior (models.py:235-278) at x (host), fp64
// accumulation; norms = [|grad|, |grad_data|, |grad_prior|]; grad_out (host, n) optional.
// The fixed-point certificate for configurations the CPU oracle cannot converge.
int mace_gradient(void* p, const float* x, double beta, double* grad_out, double* norms)
{
    API_BEGIN
    Ctx* c = C(p);
    const int rows = c->n_views * c->n_ch;
    DBuf<float> dx, ax;
    DBuf<double> g;
    dx.alloc(c->n);
    ax.alloc(rows);
    g.alloc(c->n);
    CK(cudaMemcpyAsync(dx.p, x, sizeof(float) * c->n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemsetAsync(g.p, 0, sizeof(double) * c->n, c->stream));
    const int b1 = std::max(1, std::min(c->num_sms * 8, (rows + 7) / 8));
    FPParams F{c->rp.p, c->cols.p, c->vals.p, c->n_ch};
    k_fp_rows<<<b1, 256, 0, c->stream>>>(F, rows, dx.p, ax.p, nullptr, nullptr, nullptr);
    k_bp_rows<<<b1, 256, 0, c->stream>>>(F, rows, ax.p, c->y.p, c->lam.p, g.p);
    CK(cudaGetLastError());
    std::vector<double> gd(c->n), gt(c->n);
    CK(cudaMemcpyAsync(gd.data(), g.p, sizeof(double) * c->n, cudaMemcpyDeviceToHost, c->stream));
    k_prior_grad<<<c->num_sms * 8, 256, 0, c->stream>>>(dx.p, c->n_side, c->prior, beta, g.p);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(gt.data(), g.p, sizeof(double) * c->n, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    double n2 = 0, d2 = 0, p2 = 0;
    for (size_t i = 0; i < c->n; ++i) {
        n2 += gt[i] * gt[i];
        d2 += gd[i] * gd[i];
        p2 += (gt[i] - gd[i]) * (gt[i] - gd[i]);
    }
    norms[0] = std::sqrt(n2);
    norms[1] = std::sqrt(d2);
    norms[2] = std::sqrt(p2);
    if (grad_out) std::memcpy(grad_out, gt.data(), sizeof(double) * c->n);
    API_END
}

// ------------------------------------------------------------------ MACE outer loop (mace.py:276-365)
int mace_stack_init(void* p, const float* w0, int n_total)
{
    API_BEGIN
    Ctx* c = C(p);
    if (w0) CK(cudaMemcpyAsync(c->W.p, w0, sizeof(float) * c->n * c->n_local, cudaMemcpyHostToDevice, c->stream));
    else CK(cudaMemsetAsync(c->W.p, 0, sizeof(float) * c->n * c->n_local, c->stream));
    c->stack_zero = (w0 == nullptr);  // (every rank passes w0 or none: the same MaceConfig)
    CK(cudaMemsetAsync(c->done.p, 0, 2 * sizeof(int), c->stream));
    c->passes = 0;
    if (n_total > 0) consensus(c, (float)n_total, c->wbar.p, false);  // single rank: wbar = average(w)
    sync(c);
    API_END
}

int mace_set_ref(void* p, const float* ref)
{
    API_BEGIN
    Ctx* c = C(p);
    if (!ref) {
        c->ref_norm2 = 0.0;
        return 0;
    }
    double s = 0;
    for (size_t i = 0; i < c->n; ++i) s += (double)ref[i] * ref[i];
    c->ref_norm2 = s;
    CK(cudaMemcpyAsync(c->ref.p, ref, sizeof(float) * c->n, cudaMemcpyHostToDevice, c->stream));
    sync(c);
    API_END
}

// which: 0 -> wbar, 1 -> g (denoised average); X_i = image for all local agents, then e refreshed
int mace_states_from(void* p, int which)
{
    API_BEGIN
    Ctx* c = C(p);
    k_broadcast_state<<<c->num_sms * 4, 256, 0, c->stream>>>(c->d_agents.p, c->n_local, which ? c->g.p : c->wbar.p, c->n);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(c->done.p, 0, 2 * sizeof(int), c->stream));
    if (which == 0 && c->stack_zero) {  // X0 = average(0) = 0 exactly: e = y - A 0 = y (icd.py:200) without the SpMV
        if (c->weighted) {
            k_mul<<<c->num_sms * 4, 256, 0, c->stream>>>(c->E.p, c->Y.p, c->SQ.p, (size_t)c->total_rows);
            CK(cudaGetLastError());
        } else {
            CK(cudaMemcpyAsync(c->E.p, c->Y.p, sizeof(float) * c->total_rows, cudaMemcpyDeviceToDevice, c->stream));
        }
    } else
        refresh(c, 0, c->n_local);
    sync(c);
    API_END
}

int mace_get_image(void* p, int which, float* out)
{
    API_BEGIN
    Ctx* c = C(p);
    CK(cudaMemcpyAsync(out, which ? c->g.p : c->wbar.p, sizeof(float) * c->n * c->n_slices, cudaMemcpyDeviceToHost,
                       c->stream));
    sync(c);
    API_END
}

int mace_set_image(void* p, int which, const float* img)
{
    API_BEGIN
    Ctx* c = C(p);
    c->stack_zero = false;
    CK(cudaMemcpyAsync(which ? c->g.p : c->wbar.p, img, sizeof(float) * c->n * c->n_slices, cudaMemcpyHostToDevice,
                       c->stream));
    sync(c);
    API_END
}

int mace_get_stack(void* p, float* w)
{
    API_BEGIN
    Ctx* c = C(p);
    CK(cudaMemcpyAsync(w, c->W.p, sizeof(float) * c->n * c->n_local, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    API_END
}

// Single-rank device loop: iters x [K2 pass of all agents -> K4 average/norms -> stop test];
// use_g: v = 2 g - w with g set by the caller (PnP), else v = 2 wbar - w.  No host sync inside.
// consensus + norms + stop test of one single-context iteration (k_tail: one launch)
static void iteration_tail(Ctx* c, float scale, bool with_ref, double tol, int iter)
{
    const float* rf = with_ref ? c->ref.p : nullptr;
    const double rn2 = with_ref ? c->ref_norm2 : 0.0;
#define MACE_TAIL(NL_)                                                                                             \
    k_tail<NL_><<<std::min(kTailBlocksMax, 4 * c->num_sms), 256, 0, c->stream>>>(                                  \
        c->W.p, c->n_real, c->n, scale, c->wbar.p, rf, c->part.p,                                                     \
                                                   c->n_items, c->norm_scratch.p, c->norm_counter.p, c->sums5.p, rn2, \
                                                   tol, iter, c->log.p, c->done.p, c->head.p, c->n_slices)
    switch (c->n_real) {
        case 1: MACE_TAIL(1); break;
        case 2: MACE_TAIL(2); break;
        case 4: MACE_TAIL(4); break;
        case 8: MACE_TAIL(8); break;
        case 16: MACE_TAIL(16); break;
        default: MACE_TAIL(0);
    }
#undef MACE_TAIL
    CK(cudaGetLastError());
}

// g = H(wbar) per slice with the K5 denoiser
static void cnn_all_slices(Ctx* c)
{
    if (!c->cnn.ready) throw std::runtime_error("denoiser weights not loaded (mace_cnn_set_weights)");
    for (int s = 0; s < c->n_slices; ++s)
        c->cnn.apply(c->wbar.p + (size_t)s * c->n, c->g.p + (size_t)s * c->n, c->n_side, c->n_side, c->stream,
                     c->num_sms, nullptr);
}

// use_g: 0 = MACE (G = average), 1 = PnP with g supplied between calls, 2 = PnP with the K5
// denoiser applied on the device after every iteration (no host round trip)
int mace_iterate(void* p, int iters, int iter0, double rho, int use_g, double tol, int n_total, int with_ref,
                 float* ms_out)
{
    API_BEGIN
    Ctx* c = C(p);
    ensure_log(c, iter0 + iters);
    CK(cudaEventRecord(c->ev0, c->stream));
    for (int k = 0; k < iters; ++k) {
        run_pass(c, 1, (float)rho, use_g ? c->g.p : c->wbar.p, 0, c->n_local);
        c->passes++;
        iteration_tail(c, (float)n_total, with_ref && !use_g, tol, iter0 + k);
        if (c->passes % 50 == 0) refresh(c, 0, c->n_local);  // icd.py:29,280-282
        if (use_g == 2) cnn_all_slices(c);                    // g = H(wbar) on the device (mace.py:105-108)
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(c->ev1, c->stream));
    if (ms_out) {
        CK(cudaEventSynchronize(c->ev1));
        CK(cudaEventElapsedTime(ms_out, c->ev0, c->ev1));
    }
    API_END
}

// Multi-rank phase 1: K2 for the local agents, then the local tree sum (into wsum) and the
// norm partial sums (into sums5).  The caller all-reduces both, then calls mace_iterate_finish.
int mace_iterate_local(void* p, double rho, int use_g)
{
    API_BEGIN
    Ctx* c = C(p);
    run_pass(c, 1, (float)rho, use_g ? c->g.p : c->wbar.p, 0, c->n_local);
    c->passes++;
    consensus(c, 1.0f, c->wsum.p, false);
    k_norms<<<kNormBlocks, 256, 0, c->stream>>>(c->part.p, c->n_items, nullptr, 0, c->norm_scratch.p, c->sums5.p,
                                                c->norm_counter.p, c->done.p);
    CK(cudaGetLastError());
    API_END
}

// ------------------------------------------------------------------ consensus over peer memory
int mace_peer_bytes(void* p, int world, size_t* bytes)
{
    API_BEGIN
    if (world < 1 || world > kMaxPeers) throw std::runtime_error("1..8 ranks per node");
    *bytes = peer_bytes(world, C(p)->n);
    API_END
}

// bufs[world]: every rank's symmetric buffer as seen from this process (device pointers, bufs[rank]
// local).  Zeroes this rank's flags; the caller barriers before the first exchange.
int mace_peer_setup(void* p, int world, int rank, const uint64_t* bufs)
{
    API_BEGIN
    Ctx* c = C(p);
    if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world) throw std::runtime_error("bad rank layout");
    if (c->n_slices != 1) throw std::runtime_error("peer consensus: one slice per context");
    c->peer = PeerArgs{};
    for (int r = 0; r < world; ++r) c->peer.buf[r] = reinterpret_cast<unsigned char*>(bufs[r]);
    c->peer.world = world;
    c->peer.rank = rank;
    c->epoch = 0;
    c->peer_counter.alloc(1);
    CK(cudaMemsetAsync(c->peer_counter.p, 0, sizeof(unsigned), c->stream));
    CK(cudaMemsetAsync(c->peer.buf[rank], 0, peer_norm_off(), c->stream));  // flags
    sync(c);
    c->peer_on = true;
    API_END
}

// one exchange: this rank's local tree sum + c->sums5 (local norms) -> wbar = (sum over ranks) / scale,
// c->sums5 = the global norms
static void peer_exchange(Ctx* c, float scale)
{
    if (!c->peer_on) throw std::runtime_error("mace_peer_setup first");
    c->peer.epoch = ++c->epoch;
    c->peer.parity = (int)(c->epoch & 1u);
    const int blocks = kRefBlocks;
    switch (c->n_real) {
        case 1: k_peer_push<1><<<blocks, 256, 0, c->stream>>>(c->W.p, 1, c->n, c->sums5.p, c->peer, c->peer_counter.p, c->done.p); break;
        case 2: k_peer_push<2><<<blocks, 256, 0, c->stream>>>(c->W.p, 2, c->n, c->sums5.p, c->peer, c->peer_counter.p, c->done.p); break;
        case 4: k_peer_push<4><<<blocks, 256, 0, c->stream>>>(c->W.p, 4, c->n, c->sums5.p, c->peer, c->peer_counter.p, c->done.p); break;
        case 8: k_peer_push<8><<<blocks, 256, 0, c->stream>>>(c->W.p, 8, c->n, c->sums5.p, c->peer, c->peer_counter.p, c->done.p); break;
        default:
            k_peer_push<0><<<blocks, 256, 0, c->stream>>>(c->W.p, c->n_real, c->n, c->sums5.p, c->peer, c->peer_counter.p,
                                                          c->done.p);
    }
    k_peer_reduce<<<blocks, 256, 0, c->stream>>>(c->peer, c->n, scale, c->wbar.p, c->sums5.p, c->done.p);
    CK(cudaGetLastError());
}

// stack initialisation across ranks: wbar = average of every rank's w0 (mace.py:286 with agents spread)
int mace_peer_mean(void* p, int n_total)
{
    API_BEGIN
    Ctx* c = C(p);
    CK(cudaMemsetAsync(c->sums5.p, 0, 5 * sizeof(double), c->stream));
    peer_exchange(c, (float)n_total);
    API_END
}

// `iters` MACE iterations with agents on several GPUs, entirely on the device: K2 -> local norms ->
// push/reduce over peer memory -> stop test (-> K5 if use_g == 2); no host step per iteration.
int mace_iterate_peer(void* p, int iters, int iter0, double rho, int use_g, double tol, int n_total, float* ms_out)
{
    API_BEGIN
    Ctx* c = C(p);
    ensure_log(c, iter0 + iters);
    CK(cudaEventRecord(c->ev0, c->stream));
    for (int k = 0; k < iters; ++k) {
        run_pass(c, 1, (float)rho, use_g ? c->g.p : c->wbar.p, 0, c->n_local);
        c->passes++;
        k_norms<<<kNormBlocks, 256, 0, c->stream>>>(c->part.p, c->n_items, nullptr, 0, c->norm_scratch.p, c->sums5.p,
                                                    c->norm_counter.p, c->done.p);
        peer_exchange(c, (float)n_total);
        k_finish<<<1, 1, 0, c->stream>>>(c->sums5.p, 0.0, tol, iter0 + k, c->log.p, c->done.p, c->head.p);
        if (c->passes % 50 == 0) refresh(c, 0, c->n_local);
        if (use_g == 2) cnn_all_slices(c);
        CK(cudaGetLastError());
    }
    CK(cudaEventRecord(c->ev1, c->stream));
    if (ms_out) {
        CK(cudaEventSynchronize(c->ev1));
        CK(cudaEventElapsedTime(ms_out, c->ev0, c->ev1));
    }
    API_END
}

int mace_comm_buffers(void* p, void** wsum, void** sums5)
{
    API_BEGIN
    Ctx* c = C(p);
    *wsum = c->wsum.p;
    *sums5 = c->sums5.p;
    API_END
}

int mace_local_sum(void* p)
{
    API_BEGIN
    Ctx* c = C(p);
    consensus(c, 1.0f, c->wsum.p, false);
    API_END
}

int mace_mean_from_sum(void* p, int n_total)
{
    API_BEGIN
    Ctx* c = C(p);
    // wbar = wsum / N: a one-agent "tree" over the reduced sum
    k_consensus<1><<<kRefBlocks, 256, 0, c->stream>>>(c->wsum.p, 1, c->n, (float)n_total, c->wbar.p, nullptr, nullptr,
                                                   nullptr, c->n_slices);
    CK(cudaGetLastError());
    API_END
}

// iter < 0: the log row is the device iteration counter (mace_set_iter), which advances by one: a
// loop of iterate_local / all-reduce / iterate_finish can then be captured in a CUDA graph once and
// replayed (reserve the log first with mace_reserve_log; no allocation happens here)
int mace_iterate_finish(void* p, int n_total, double tol, int iter)
{
    API_BEGIN
    Ctx* c = C(p);
    if (iter >= 0) ensure_log(c, iter + 1);
    else if (!c->iter_ctr.p) throw std::runtime_error("mace_set_iter first");
    k_consensus<1><<<kRefBlocks, 256, 0, c->stream>>>(c->wsum.p, 1, c->n, (float)n_total, c->wbar.p, nullptr, nullptr,
                                                   c->done.p, c->n_slices);
    k_finish<<<1, 1, 0, c->stream>>>(c->sums5.p, 0.0, tol, iter < 0 ? 0 : iter, c->log.p, c->done.p, c->head.p,
                                     iter < 0 ? c->iter_ctr.p : nullptr);
    if (c->passes % 50 == 0) refresh(c, 0, c->n_local);
    CK(cudaGetLastError());
    API_END
}

// device iteration counter for mace_iterate_finish(iter < 0); stream-ordered
int mace_set_iter(void* p, int iter)
{
    API_BEGIN
    Ctx* c = C(p);
    if (!c->iter_ctr.p) c->iter_ctr.alloc(1);
    k_set_int<<<1, 1, 0, c->stream>>>(c->iter_ctr.p, iter);
    CK(cudaGetLastError());
    API_END
}

// room for n log rows (before capturing iterations in a graph: nothing may allocate inside it)
int mace_reserve_log(void* p, int n)
{
    API_BEGIN
    ensure_log(C(p), n);
    API_END
}

// host pass counter (it schedules the error refresh every 50 passes): += add; *out = the new count.
// Replays of a captured graph run passes the host never counted.
int mace_passes(void* p, int64_t add, int64_t* out)
{
    API_BEGIN
    Ctx* c = C(p);
    c->passes += add;
    if (out) *out = c->passes;
    API_END
}

int mace_read_log(void* p, int n, double* log, int* done2)
{
    API_BEGIN
    Ctx* c = C(p);
    if (n > 0) CK(cudaMemcpyAsync(log, c->log.p, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(done2, c->done.p, sizeof(int) * 2, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    API_END
}

// ------------------------------------------------------------------ reference plug point: _sweep (icd.py:67-139)
namespace {
struct SweepEntry {
    const void *k_cp, *k_ri, *k_av, *k_ni, *k_nw;
    int64_t n = 0, nnz = 0, rows = 0;
    DBuf<int64_t> col_ptr, row_idx, nbr_idx;
    DBuf<double> a_val, nbr_w, z, v, e, lam, curv, dsq;
    uint64_t last_use = 0;
};
std::mutex g_sweep_mu;
std::vector<std::unique_ptr<SweepEntry>> g_sweep;
uint64_t g_sweep_clock = 0;
}  // namespace

// Same arguments as the reference's numba _sweep (+ sizes); host float64 arrays in and out.
// The static operator (col_ptr, row_idx, a_val, neighbour tables) is cached on the device
// per workspace (keyed by host pointers and sizes); state, target, error sinogram, weights
// and theta2 move every call.
int mace_sweep_f64(double* z, const double* v, double* e, const int64_t* col_ptr, const int64_t* row_idx,
                   const double* a_val, const double* lam, const double* curv_data, const int64_t* nbr_idx,
                   const double* nbr_w, double beta_eff, double eps_reg, double inv_sigma2, int quad_prior, double p,
                   double q, double T, double sx, int clamp, int64_t s_begin, int64_t s_end, int64_t n,
                   int64_t n_rows, double* delta_sq)
{
    API_BEGIN
    std::lock_guard<std::mutex> lk(g_sweep_mu);
    if (s_begin < 0 || s_end > n || s_begin > s_end) throw std::runtime_error("bad pixel range");
    const int64_t nnz = col_ptr[n];
    SweepEntry* E = nullptr;
    for (auto& x : g_sweep)
        if (x->k_cp == col_ptr && x->k_ri == row_idx && x->k_av == a_val && x->k_ni == nbr_idx && x->k_nw == nbr_w &&
            x->n == n && x->nnz == nnz && x->rows == n_rows)
            E = x.get();
    if (!E) {
        if (g_sweep.size() >= 64) {
            auto it = std::min_element(g_sweep.begin(), g_sweep.end(),
                                       [](const auto& a, const auto& b) { return a->last_use < b->last_use; });
            g_sweep.erase(it);
        }
        auto x = std::make_unique<SweepEntry>();
        x->k_cp = col_ptr;
        x->k_ri = row_idx;
        x->k_av = a_val;
        x->k_ni = nbr_idx;
        x->k_nw = nbr_w;
        x->n = n;
        x->nnz = nnz;
        x->rows = n_rows;
        x->col_ptr.alloc(n + 1);
        x->row_idx.alloc(std::max<int64_t>(nnz, 1));
        x->a_val.alloc(std::max<int64_t>(nnz, 1));
        x->nbr_idx.alloc(8 * n);
        x->nbr_w.alloc(8 * n);
        CK(cudaMemcpy(x->col_ptr.p, col_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
        if (nnz) {
            CK(cudaMemcpy(x->row_idx.p, row_idx, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(x->a_val.p, a_val, sizeof(double) * nnz, cudaMemcpyHostToDevice));
        }
        CK(cudaMemcpy(x->nbr_idx.p, nbr_idx, sizeof(int64_t) * 8 * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(x->nbr_w.p, nbr_w, sizeof(double) * 8 * n, cudaMemcpyHostToDevice));
        x->z.alloc(n);
        x->v.alloc(n);
        x->curv.alloc(n);
        x->e.alloc(std::max<int64_t>(n_rows, 1));
        x->lam.alloc(std::max<int64_t>(n_rows, 1));
        x->dsq.alloc(1);
        E = x.get();
        g_sweep.push_back(std::move(x));
    }
    E->last_use = ++g_sweep_clock;
    CK(cudaMemcpy(E->z.p, z, sizeof(double) * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(E->v.p, v, sizeof(double) * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(E->curv.p, curv_data, sizeof(double) * n, cudaMemcpyHostToDevice));
    if (n_rows) {
        CK(cudaMemcpy(E->e.p, e, sizeof(double) * n_rows, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(E->lam.p, lam, sizeof(double) * n_rows, cudaMemcpyHostToDevice));
    }
    Sweep64 P{};
    P.z = E->z.p;
    P.e = E->e.p;
    P.dsq = E->dsq.p;
    P.v = E->v.p;
    P.a_val = E->a_val.p;
    P.lam = E->lam.p;
    P.curv = E->curv.p;
    P.nbr_w = E->nbr_w.p;
    P.col_ptr = E->col_ptr.p;
    P.row_idx = E->row_idx.p;
    P.nbr_idx = E->nbr_idx.p;
    P.beta_eff = beta_eff;
    P.eps_reg = eps_reg;
    P.inv_sigma2 = inv_sigma2;
    P.p = p;
    P.q = q;
    P.T = T;
    P.sx = sx;
    P.quad = quad_prior;
    P.clamp = clamp;
    P.s_begin = s_begin;
    P.s_end = s_end;
    k_sweep64<<<1, 32>>>(P);
    CK(cudaGetLastError());
    CK(cudaMemcpy(z, E->z.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    if (n_rows) CK(cudaMemcpy(e, E->e.p, sizeof(double) * n_rows, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(delta_sq, E->dsq.p, sizeof(double), cudaMemcpyDeviceToHost));
    API_END
}

// ------------------------------------------------------------------ host-only layout probes (no GPU needed)
// Stacked agent CSC (icd.py:185-192).  col_ptr[n+1] always written; rows/vals if non-null.
int mace_agent_csc(int n_side, int n_ch, int n_views, const int64_t* row_ptr, const int32_t* cols, const float* vals,
                   int n_agent_views, const int* views, int64_t* col_ptr, uint32_t* rows, float* out_vals)
{
    API_BEGIN
    std::vector<int> vv(views, views + n_agent_views);
    for (int v : vv)
        if (v < 0 || v >= n_views) throw std::runtime_error("view index out of range");
    AgentCSC csc;
    build_agent_csc(n_side, n_ch, row_ptr, cols, vals, vv, csc);
    std::memcpy(col_ptr, csc.col_ptr.data(), sizeof(int64_t) * csc.col_ptr.size());
    if (rows) std::memcpy(rows, csc.row.data(), sizeof(uint32_t) * csc.row.size());
    if (out_vals) std::memcpy(out_vals, csc.val.data(), sizeof(float) * csc.val.size());
    API_END
}

// Super-voxel layout decoded back to (pixel, local row, value) per stored entry (pads skipped).
// stats: [entries, max_band, max_col, n_sv, duplicates, decoded]; decoded arrays may be null.
int mace_sv_layout_probe(int n_side, int n_ch, int n_views, const int64_t* row_ptr, const int32_t* cols,
                         const float* vals, int n_agent_views, const int* views, int svs, int64_t* stats,
                         int32_t* pix_out, int32_t* row_out, float* val_out)
{
    API_BEGIN
    std::vector<int> vv(views, views + n_agent_views);
    for (int v : vv)
        if (v < 0 || v >= n_views) throw std::runtime_error("view index out of range");
    AgentCSC csc;
    build_agent_csc(n_side, n_ch, row_ptr, cols, vals, vv, csc);
    SVLayout L;
    build_sv_layout(csc, n_side, n_ch, n_agent_views, svs, L);
    int64_t k = 0;
    const int S = L.svs, G = L.ng, KK = L.K, CH = L.chunks;
    const size_t per_tile = (size_t)L.nb * CH * kSvBatch * L.rec;
    for (int sv = 0; sv < L.n_sv; ++sv) {
        const int r0 = (sv / L.n_sv_side) * S, c0 = (sv % L.n_sv_side) * S;
        const int2_t* bt = &L.band[(size_t)sv * L.views];
        std::vector<int> seen(S * S, 0);
        for (int t = 0; t < L.nb * kSvBatch; ++t) {
            const int slot = t % kSvBatch;
            const uint32_t* blk0 = &L.data[(size_t)sv * per_tile + (size_t)(t / kSvBatch) * CH * kSvBatch * L.rec];
            const int q = sv_slot_pixel(S, t);
            if (q >= 0) seen[q]++;
            for (int j = 0; j < L.views; ++j) {
                const int gt = j >> 5, g = gt % G, l = j & 31;
                const uint32_t* blk = blk0 + (size_t)(gt / G) * kSvBatch * L.rec;  // the view's chunk
                const int o = (int)((blk[sv_ofs_word(G, KK, l, slot)] >> (8 * g)) & 0xffu);
                for (int e = 0; e < KK; ++e) {
                    float a;
                    std::memcpy(&a, &blk[sv_len_word(G, KK, g, l, slot, e)], 4);
                    if (a == 0.0f) continue;
                    if (q < 0) throw std::runtime_error("padding slot with a value");
                    if (o + e >= bt[j].y) throw std::runtime_error("slot outside its band window");
                    if (pix_out) {
                        pix_out[k] = (r0 + q / S) * n_side + (c0 + q % S);
                        row_out[k] = bt[j].x + o + e;
                        val_out[k] = a;
                    }
                    ++k;
                }
            }
        }
        for (int q = 0; q < S * S; ++q)
            if (seen[q] != 1) throw std::runtime_error("visit order does not cover the tile once");
    }
    stats[0] = (int64_t)L.data.size();
    stats[1] = L.wcap;
    stats[2] = L.max_col;
    stats[3] = L.n_sv;
    stats[4] = L.duplicates;
    stats[5] = k;
    API_END
}

// ------------------------------------------------------------------ K5 PnP denoiser (cnn.cu)
int mace_cnn_set_weights(void* p, const uint16_t* bf16, int layers, int channels)
{
    API_BEGIN
    C(p)->cnn.set_weights(bf16, layers, channels);
    API_END
}

// g = H(wbar) on the device (the denoiser agent inside consensus_GH, mace.py:105-108)
int mace_cnn_apply(void* p)
{
    API_BEGIN
    Ctx* c = C(p);
    cnn_all_slices(c);
    API_END
}

// one middle layer alone (layer index 0..14 = layers 2..16), bf16 CHW in/out (host); the per-layer test
int mace_cnn_layer(void* p, int layer, const uint16_t* in_chw, uint16_t* out_chw, int h, int w)
{
    API_BEGIN
    Ctx* c = C(p);
    c->cnn.layer(layer, in_chw, out_chw, h, w, c->stream, c->num_sms);
    API_END
}

// standalone: out = H(x) for an h x w image (host pointers); ms_out = device time of the 17 layers
int mace_cnn_run(void* p, const float* x, float* out, int h, int w, float* ms_out)
{
    API_BEGIN
    Ctx* c = C(p);
    DBuf<float> dx, dy;
    dx.alloc((size_t)h * w);
    dy.alloc((size_t)h * w);
    CK(cudaMemcpyAsync(dx.p, x, sizeof(float) * h * w, cudaMemcpyHostToDevice, c->stream));
    c->cnn.ensure(h, w);
    CK(cudaEventRecord(c->ev0, c->stream));
    c->cnn.apply(dx.p, dy.p, h, w, c->stream, c->num_sms, nullptr);
    CK(cudaEventRecord(c->ev1, c->stream));
    CK(cudaMemcpyAsync(out, dy.p, sizeof(float) * h * w, cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (ms_out) CK(cudaEventElapsedTime(ms_out, c->ev0, c->ev1));
    API_END
}

// K2 launch timing: enable=1 starts a fresh record; enable=0 stops and returns the summed
// device time (ms) and the number of K2 launches recorded since.
int mace_k2_timing(void* p, int enable, double* total_ms, int64_t* launches)
{
    API_BEGIN
    Ctx* c = C(p);
    if (enable) {
        c->time_k2 = true;
        c->k2_used = 0;
    } else {
        sync(c);
        double s = 0.0;
        for (size_t i = 0; i < c->k2_used; ++i) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, c->k2ev[i].first, c->k2ev[i].second));
            s += ms;
        }
        if (total_ms) *total_ms = s;
        if (launches) *launches = (int64_t)c->k2_used;
        c->time_k2 = false;
        c->k2_used = 0;
    }
    API_END
}

// pinned host memory for the end-to-end path
int mace_host_alloc(size_t bytes, void** out)
{
    API_BEGIN
    CK(cudaHostAlloc(out, bytes, cudaHostAllocDefault));
    API_END
}
void mace_host_free(void* ptr)
{
    if (ptr) cudaFreeHost(ptr);
}

}  // extern "C"

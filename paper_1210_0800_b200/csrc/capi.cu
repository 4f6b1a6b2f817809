// capi.cu -- the C ABI (include/xqr_b200.h): contexts, device workspace,
// host<->device staging, argument validation with the reference's error
// conventions, and kernel dispatch.  No CPU fallback: without a usable CUDA
// device every entry point returns XQR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "xqr_internal.h"

struct xqr_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // device arena (grown on demand, reused across calls)
    void* arena = nullptr;
    size_t arena_bytes = 0;
    // pinned host staging
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool timed = false;
    // host-buffer batched calls: a second stream and slot events for the
    // copy / compute pipeline (created on first use)
    cudaStream_t stream2 = nullptr;
    cudaEvent_t slot_done[2] = {nullptr, nullptr};
    void* pinned_out = nullptr;
    size_t pinned_out_bytes = 0;
    int64_t launches = 0;
    int64_t grid_fallbacks = 0;  // single systems re-routed to the CTA kernel
    int num_sms = 148;
    bool coop = false;
    std::string last_error;
};

namespace {

int set_cuda_error(xqr_ctx* ctx, cudaError_t e, const char* where) {
    if (ctx) ctx->last_error = std::string(where) + ": " + cudaGetErrorString(e);
    return XQR_CUDA;
}

void fill_status(xqr_status* st, int code, int column = 0, int64_t system = 0) {
    if (st) {
        st->code = code;
        st->column = column;
        st->system = system;
    }
}

int fail(xqr_ctx* ctx, xqr_status* st, int code, const char* what) {
    if (ctx) ctx->last_error = what;
    fill_status(st, code);
    return code;
}

bool valid_limbs(int l) { return l == 1 || l == 2 || l == 4; }

// Bump allocator over the ctx arena.  Every region is 256-byte aligned.
struct arena_plan {
    std::vector<size_t> sizes;
    size_t total = 0;
    size_t add(size_t bytes) {
        size_t off = total;
        total += (bytes + 255) & ~size_t(255);
        sizes.push_back(bytes);
        return off;
    }
};

cudaError_t ensure_arena(xqr_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->arena_bytes) return cudaSuccess;
    if (ctx->arena) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(ctx->arena);
        ctx->arena = nullptr;
        ctx->arena_bytes = 0;
    }
    size_t want = bytes + bytes / 4;
    cudaError_t e = cudaMalloc(&ctx->arena, want);
    if (e != cudaSuccess) return e;
    ctx->arena_bytes = want;
    return cudaSuccess;
}

cudaError_t ensure_pinned(xqr_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->pinned_bytes) return cudaSuccess;
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    size_t want = bytes + bytes / 4;
    cudaError_t e = cudaMallocHost(&ctx->pinned, want);
    if (e != cudaSuccess) return e;
    ctx->pinned_bytes = want;
    return cudaSuccess;
}

char* at(xqr_ctx* ctx, size_t off) { return static_cast<char*>(ctx->arena) + off; }

int first_code(const std::vector<xqr_status>& st) {
    for (const auto& s : st)
        if (s.code) return s.code;
    return 0;
}

// Validate the shapes the reference validates (matrix.hpp:15-19: rows >= cols
// >= 1) plus this build's size envelope.
int check_shape(xqr_ctx* ctx, xqr_status* st, int limbs, int64_t batch, int64_t m, int64_t n) {
    if (!valid_limbs(limbs)) return fail(ctx, st, XQR_USAGE, "limbs must be 1, 2 or 4");
    if (n < 1 || m < n) return fail(ctx, st, XQR_DIMENSION, "matrix shape must satisfy rows >= cols >= 1");
    if (batch < 0) return fail(ctx, st, XQR_USAGE, "negative batch");
    if (m > xb::kGridMaxRows) return fail(ctx, st, XQR_USAGE, "rows > 2048 not supported by this build");
    if (batch > 0x7fffffff) return fail(ctx, st, XQR_USAGE, "batch too large");
    return 0;
}

// A single system large enough to feed several SMs goes to the cluster grid
// kernel (xgrid2.cuh); small ones stay on one CTA (xmgs.cuh).
bool use_grid_path(xqr_ctx* ctx, int limbs, int m, int n) {
    if (const char* e = std::getenv("XQR_FORCE_CTA")) {
        if (e[0] == '1') return false;
    }
    // quad-double pivots are slow enough that even a small system gains from
    // spreading its columns over SMs; double-double needs a larger one
    if (m > 32 * xb::kMaxRowsPerLane) return true;  // only the grid kernels take m > 1024
    if (limbs == 4) return ctx->coop && n >= 4 && m >= 16 && m <= xb::kGridMaxRows;
    // (measured, tools/small_latency.py: cdd 32x32 207 vs 284 us on one CTA,
    // 48x48 302 vs 739; 16x16 114 vs 104)
    int min_m = 32;
    if (const char* e = std::getenv("XQR_DD_GRID_MIN_M")) min_m = std::atoi(e);  // dev
    return ctx->coop && n >= 8 && m >= min_m && m <= xb::kGridMaxRows;
}

size_t grid_ws_doubles(int limbs, int m, int ncol) {
    if (limbs <= 2) return (size_t)ncol * 2 * limbs * 256 * xb::grid1_rows_per_thread(m);
    return (size_t)ncol * m * 2 * limbs;
}

size_t grid_scratch_bytes(bool lsq, int limbs, int m, int n) {
    const int ncol = n + (lsq ? 1 : 0);
    return sizeof(double) * (grid_ws_doubles(limbs, m, ncol) + (lsq ? xb::rws_doubles(limbs, n) : 0) +
                             (size_t)ncol * limbs) +
           sizeof(int) * ((size_t)n + 4) + sizeof(unsigned long long) * (16 * (size_t)(n + 1) + 1) +
           8 * 256;
}

// solve_grid's answer when the persistent grid cannot be placed (the
// cooperative / cluster launch finds no co-residency: an MPS partition, a
// smaller part); the caller re-routes the system to the CTA kernel, which
// computes the same bits.
constexpr int kGridUnplaceable = -1;

bool unplaceable(cudaError_t e) {
    return e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorInvalidConfiguration ||
           e == cudaErrorInvalidClusterSize;
}

int solve_grid(xqr_ctx* ctx, bool lsq, int limbs, int m, int n, const double* d_a,
               const double* d_b, double* d_q, double* d_r, double* d_x, double* d_z,
               xqr_status* d_st, size_t scratch_off, bool timed, int64_t sys = 0) {
    const int ncol = n + (lsq ? 1 : 0);
    xb::GridParams p{};
    p.sys = sys;
    p.m = m;
    p.n = n;
    if (limbs <= 2) {
        p.cs = 1;
        p.rpt = xb::grid1_rows_per_thread(m);
        p.chain = 1;
        if (const char* e = std::getenv("XQR_GRID_CHAIN")) p.chain = std::atoi(e);  // dev
    } else {
        xb::grid_shape(m, p.cs, p.rpt, p.pair_bulk);
        if (const char* e = std::getenv("XQR_GRID_PAIR")) p.pair_bulk = std::atoi(e);  // dev
        if (const char* e = std::getenv("XQR_GRID_CS")) {  // dev override of the cluster size
            p.cs = std::max(1, std::min(8, std::atoi(e)));
            p.rpt = 1;
            while (p.cs * 64 * p.rpt < m) p.rpt <<= 1;
        }
    }
    p.a = d_a;
    p.b = d_b;
    p.q = d_q;
    p.r = d_r;
    p.x = d_x;
    p.z = d_z;
    p.st = d_st;
    arena_plan plan;
    const size_t o_ws = plan.add(sizeof(double) * grid_ws_doubles(limbs, m, ncol));
    const size_t o_rws = plan.add(lsq ? sizeof(double) * xb::rws_doubles(limbs, n) : 0);
    const size_t o_nrm = plan.add(sizeof(double) * (size_t)ncol * limbs);
    const size_t o_flg = plan.add(sizeof(int) * ((size_t)n + 4 + ncol));
    const size_t o_key = plan.add(sizeof(unsigned long long));
    const char* trace_path = std::getenv("XQR_GRID_TRACE");  // dev instrumentation
    const size_t o_trc = plan.add(trace_path ? sizeof(unsigned long long) * 16 * (size_t)(n + 1) : 0);
    cudaError_t e = ensure_arena(ctx, scratch_off + plan.total + 256);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "workspace allocation");
    p.ws = reinterpret_cast<double*>(at(ctx, scratch_off + o_ws));
    p.rws = lsq ? reinterpret_cast<double*>(at(ctx, scratch_off + o_rws)) : nullptr;
    p.norms = reinterpret_cast<double*>(at(ctx, scratch_off + o_nrm));
    p.flags = reinterpret_cast<int*>(at(ctx, scratch_off + o_flg));
    p.counters = p.flags + n;
    p.cflags = p.counters + 4;
    p.key = reinterpret_cast<unsigned long long*>(at(ctx, scratch_off + o_key));
    p.trace = trace_path ? reinterpret_cast<unsigned long long*>(at(ctx, scratch_off + o_trc)) : nullptr;
    cudaMemsetAsync(p.flags, 0, sizeof(int) * ((size_t)n + 4 + ncol), ctx->stream);
    cudaMemsetAsync(p.key, 0xFF, sizeof(unsigned long long), ctx->stream);
    if (p.trace) cudaMemsetAsync(p.trace, 0, sizeof(unsigned long long) * 16 * (size_t)(n + 1), ctx->stream);
    int per_sm = limbs == 4 ? xb::kGrid2PerSM : 1;
    if (const char* e = std::getenv("XQR_GRID_PER_SM")) per_sm = std::max(1, std::atoi(e));  // dev
    // SMs the persistent grid may occupy; XQR_GRID_MAX_SMS emulates a
    // partitioned device (MPS) for the re-routing test
    int sms = ctx->num_sms;
    if (const char* e = std::getenv("XQR_GRID_MAX_SMS")) sms = std::max(0, std::min(sms, std::atoi(e)));
    const int max_clusters = per_sm * sms / p.cs;
    const int grid1 = std::min(ncol, sms);
    if ((limbs <= 2 && grid1 < 1) || (limbs == 4 && max_clusters < 1)) return kGridUnplaceable;
    if (timed) cudaEventRecord(ctx->ev0, ctx->stream);
    switch (limbs) {
        case 1: e = xb::launch_grid_L1(p, grid1, lsq, ctx->stream); break;
        case 2: e = xb::launch_grid_L2(p, grid1, lsq, ctx->stream); break;
        default: e = xb::launch_grid_L4(p, max_clusters, lsq, ctx->stream); break;
    }
    if (timed) cudaEventRecord(ctx->ev1, ctx->stream);
    ctx->timed = timed;
    if (e != cudaSuccess && unplaceable(e)) {
        cudaGetLastError();  // not sticky: clear it and let the caller re-route
        return kGridUnplaceable;
    }
    ctx->launches += 1;
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "grid kernel launch");
    if (p.trace) {
        // per row j: 8 factorisation stamps (globaltimer), then 8 back-substitution
        // stamps (SM cycles) -- dev instrumentation, XQR_GRID_TRACE
        std::vector<unsigned long long> h(16 * (size_t)(n + 1));
        cudaMemcpyAsync(h.data(), p.trace, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost,
                        ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        if (FILE* fp = std::fopen(trace_path, "w")) {
            for (int j = 0; j <= n; ++j) {
                std::fprintf(fp, "%d", j);
                for (int c = 0; c < 8; ++c) std::fprintf(fp, " %llu", h[8 * j + c]);
                for (int c = 0; c < 8; ++c) std::fprintf(fp, " %llu", h[8 * (size_t)(n + 1) + 8 * j + c]);
                std::fprintf(fp, "\n");
            }
            std::fclose(fp);
        }
    }
    return 0;
}

// Device-side solve on device pointers (shared by host and device entry points).
int solve_device(xqr_ctx* ctx, bool lsq, int limbs, int64_t batch, int64_t m, int64_t n,
                 const double* d_a, const double* d_b, double* d_q, double* d_r, double* d_x,
                 double* d_z, xqr_status* d_st, size_t scratch_off, bool timed) {
    const int ncol = (int)n + (lsq ? 1 : 0);
    if (batch == 1 && use_grid_path(ctx, limbs, (int)m, (int)n)) {
        const int rc = solve_grid(ctx, lsq, limbs, (int)m, (int)n, d_a, d_b, d_q, d_r, d_x, d_z, d_st,
                                  scratch_off, timed);
        if (rc != kGridUnplaceable) return rc;
        if (m > 32 * xb::kMaxRowsPerLane) {
            ctx->last_error = "grid kernel cannot be placed on this device (m > 1024 has no CTA kernel)";
            return XQR_CUDA;
        }
        // the grid cannot be made co-resident here: the CTA kernel computes
        // the same bits on one SM
        ctx->grid_fallbacks += 1;
    }
    if (m > 32 * xb::kMaxRowsPerLane) {
        // taller than one CTA holds: system by system on the grid kernels
        const size_t L2 = 2 * (size_t)limbs;
        for (int64_t s = 0; s < batch; ++s) {
            const int rc = solve_grid(
                ctx, lsq, limbs, (int)m, (int)n, d_a + s * m * n * L2, lsq ? d_b + s * m * L2 : nullptr,
                lsq ? nullptr : d_q + s * m * n * L2, lsq ? nullptr : d_r + s * n * n * L2,
                lsq ? d_x + s * n * L2 : nullptr, lsq ? d_z + s * limbs : nullptr, d_st + s, scratch_off,
                timed && s == 0, s);
            if (rc == kGridUnplaceable) {
                ctx->last_error = "grid kernel cannot be placed on this device (m > 1024 has no CTA kernel)";
                return XQR_CUDA;
            }
            if (rc) return rc;
        }
        return 0;
    }
    xb::SolveParams p{};
    p.batch = batch;
    p.m = (int)m;
    p.n = (int)n;
    p.a = d_a;
    p.b = d_b;
    p.q = d_q;
    p.r = d_r;
    p.x = d_x;
    p.z = d_z;
    p.st = d_st;
    p.ws_stride = xb::ws_doubles(limbs, (int)m, ncol);
    p.rws_stride = lsq ? xb::rws_doubles(limbs, (int)n) : 0;
    size_t need = scratch_off + sizeof(double) * (size_t)batch * (p.ws_stride + p.rws_stride) + 512;
    cudaError_t e = ensure_arena(ctx, need);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "workspace allocation");
    p.ws = reinterpret_cast<double*>(at(ctx, scratch_off));
    p.rws = lsq ? p.ws + (size_t)batch * p.ws_stride : nullptr;
    if (batch == 0) return 0;
    if (timed) cudaEventRecord(ctx->ev0, ctx->stream);
    e = xb::launch_mgs_cta(limbs, lsq, p, ctx->stream);
    if (timed) cudaEventRecord(ctx->ev1, ctx->stream);
    ctx->timed = timed;
    ctx->launches += 1;
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "mgs kernel launch");
    return 0;
}

}  // namespace

extern "C" {

int xqr_version(void) { return 100; }

int xqr_ctx_create(int device, xqr_ctx** out) {
    if (!out) return XQR_USAGE;
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        std::fprintf(stderr, "xqr_b200: no CUDA device available (%s)\n", cudaGetErrorString(e));
        return XQR_CUDA;
    }
    if (device < 0 || device >= count) return XQR_USAGE;
    e = cudaSetDevice(device);
    if (e != cudaSuccess) return XQR_CUDA;
    auto* ctx = new xqr_ctx();
    ctx->device = device;
    e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete ctx;
        return XQR_CUDA;
    }
    ctx->own_stream = true;
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) == cudaSuccess) ctx->num_sms = v;
    v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrCooperativeLaunch, device);
    ctx->coop = v != 0;
    cudaEventCreate(&ctx->ev0);
    cudaEventCreate(&ctx->ev1);
    *out = ctx;
    return XQR_OK;
}

void xqr_ctx_destroy(xqr_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->arena) cudaFree(ctx->arena);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
    for (auto& ev : ctx->slot_done)
        if (ev) cudaEventDestroy(ev);
    if (ctx->pinned_out) cudaFreeHost(ctx->pinned_out);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int xqr_ctx_set_stream(xqr_ctx* ctx, void* cuda_stream) {
    if (!ctx) return XQR_USAGE;
    if (!cuda_stream) return XQR_OK;
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    ctx->stream = static_cast<cudaStream_t>(cuda_stream);
    ctx->own_stream = false;
    return XQR_OK;
}

void* xqr_ctx_stream(xqr_ctx* ctx) { return ctx ? ctx->stream : nullptr; }

int xqr_ctx_synchronize(xqr_ctx* ctx) {
    if (!ctx) return XQR_USAGE;
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? XQR_OK : set_cuda_error(ctx, e, "synchronize");
}

const char* xqr_ctx_last_error(xqr_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "no ctx"; }

int64_t xqr_ctx_launch_count(xqr_ctx* ctx) { return ctx ? ctx->launches : 0; }

int64_t xqr_ctx_grid_fallbacks(xqr_ctx* ctx) { return ctx ? ctx->grid_fallbacks : 0; }

float xqr_ctx_last_kernel_ms(xqr_ctx* ctx) {
    if (!ctx || !ctx->timed) return 0.f;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1) != cudaSuccess) return 0.f;
    return ms;
}

// ---- device entry points -------------------------------------------------------
int xqr_mgs_qr_batched_device(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                              const double* d_a, double* d_q, double* d_r, xqr_status* d_st) {
    if (!ctx) return XQR_USAGE;
    if (int c = check_shape(ctx, nullptr, limbs, batch, m, n)) return c;
    cudaSetDevice(ctx->device);
    return solve_device(ctx, false, limbs, batch, m, n, d_a, nullptr, d_q, d_r, nullptr, nullptr,
                        d_st, 0, true);
}

int xqr_lsq_solve_batched_device(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                                 const double* d_a, const double* d_b, double* d_x, double* d_z,
                                 xqr_status* d_st) {
    if (!ctx) return XQR_USAGE;
    if (int c = check_shape(ctx, nullptr, limbs, batch, m, n)) return c;
    cudaSetDevice(ctx->device);
    return solve_device(ctx, true, limbs, batch, m, n, d_a, d_b, nullptr, nullptr, d_x, d_z, d_st, 0,
                        true);
}

int xqr_back_substitute_batched_device(xqr_ctx* ctx, int limbs, int64_t batch, int64_t n,
                                       const double* d_r, const double* d_y, double* d_x,
                                       xqr_status* d_st) {
    if (!ctx) return XQR_USAGE;
    if (!valid_limbs(limbs)) return fail(ctx, nullptr, XQR_USAGE, "limbs must be 1, 2 or 4");
    if (n < 1) return fail(ctx, nullptr, XQR_DIMENSION, "empty triangular factor");
    cudaSetDevice(ctx->device);
    size_t prep = sizeof(double) * (size_t)batch * n * (3 * limbs + 1);
    cudaError_t e = ensure_arena(ctx, prep + 256);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "workspace allocation");
    if (batch == 0) return 0;
    xb::BackSubParams p{batch, (int)n, d_r, d_y, d_x, d_st, reinterpret_cast<double*>(ctx->arena)};
    cudaEventRecord(ctx->ev0, ctx->stream);
    e = xb::launch_back_substitute(limbs, p, ctx->stream);
    cudaEventRecord(ctx->ev1, ctx->stream);
    ctx->timed = true;
    ctx->launches += 1;
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "back substitution launch");
    return 0;
}

// ---- host entry points -----------------------------------------------------------
namespace {

bool is_pinned(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// CTA kernel on `batch` systems, on an explicit stream and scratch region.
int launch_cta_batch(xqr_ctx* ctx, cudaStream_t s, bool lsq, int limbs, int64_t batch, int m, int n,
                     const double* d_a, const double* d_b, double* d_q, double* d_r, double* d_x,
                     double* d_z, xqr_status* d_st, double* scratch) {
    const int ncol = n + (lsq ? 1 : 0);
    xb::SolveParams p{};
    p.batch = batch;
    p.m = m;
    p.n = n;
    p.a = d_a;
    p.b = d_b;
    p.q = d_q;
    p.r = d_r;
    p.x = d_x;
    p.z = d_z;
    p.st = d_st;
    p.ws_stride = xb::ws_doubles(limbs, m, ncol);
    p.rws_stride = lsq ? xb::rws_doubles(limbs, n) : 0;
    p.ws = scratch;
    p.rws = lsq ? scratch + (size_t)batch * p.ws_stride : nullptr;
    cudaError_t e = xb::launch_mgs_cta(limbs, lsq, p, s);
    ctx->launches += 1;
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "mgs kernel launch");
    return 0;
}

// Host-buffer batch: split into chunks of about one wave of the CTA kernel
// and pipeline them over two streams, so the host->device copy of chunk c+1
// (straight from the caller's buffer when it is pinned, else through a
// pinned staging slot) overlaps the solve of chunk c.
int solve_host_batched(xqr_ctx* ctx, bool lsq, int limbs, int64_t batch, int64_t m, int64_t n,
                       const double* a, const double* b, double* q, double* r, double* x, double* z,
                       xqr_status* st) {
    const size_t L2 = 2 * (size_t)limbs;
    const int ncol = (int)n + (lsq ? 1 : 0);
    // one kernel wave per chunk (quad-double m <= 128: 2 CTAs per SM, else 4):
    // the first chunk's copy is the only one not hidden behind a solve
    int64_t chunk = (limbs == 4 && m <= 128 ? 2 : 4) * (int64_t)ctx->num_sms;
    if (const char* e = std::getenv("XQR_CHUNK")) chunk = std::max<int64_t>(1, std::atoll(e));
    if (chunk > batch) chunk = batch;
    const int64_t nchunks = (batch + chunk - 1) / chunk;
    // per-system sizes (doubles)
    const size_t sa = (size_t)m * n * L2, sb = lsq ? (size_t)m * L2 : 0, sq = lsq ? 0 : sa,
                 sr = lsq ? 0 : (size_t)n * n * L2, sx = lsq ? (size_t)n * L2 : 0, sz = lsq ? limbs : 0;
    const size_t sws = xb::ws_doubles(limbs, (int)m, ncol) + (lsq ? xb::rws_doubles(limbs, (int)n) : 0);
    const size_t sout = sq + sr + sx + sz;  // doubles out per system
    arena_plan plan;
    size_t o_in[2], o_out[2], o_st[2], o_ws[2];
    for (int k = 0; k < 2; ++k) {
        o_in[k] = plan.add(sizeof(double) * chunk * (sa + sb));
        o_out[k] = plan.add(sizeof(double) * chunk * sout);
        o_st[k] = plan.add(sizeof(xqr_status) * chunk);
        o_ws[k] = plan.add(sizeof(double) * chunk * sws);
    }
    cudaError_t e = ensure_arena(ctx, plan.total + 256);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "workspace allocation");
    if (!ctx->stream2) {
        e = cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking);
        if (e != cudaSuccess) return set_cuda_error(ctx, e, "stream");
        for (auto& ev : ctx->slot_done) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    }
    const bool pin_a = is_pinned(a) && (!lsq || is_pinned(b));
    if (!pin_a) {
        e = ensure_pinned(ctx, 2 * sizeof(double) * chunk * (sa + sb));
        if (e != cudaSuccess) return set_cuda_error(ctx, e, "pinned staging allocation");
    }
    // outputs land in pinned staging (2 slots), copied out once a slot is reused / at the end
    {
        const size_t need = 2 * (sizeof(double) * chunk * sout + sizeof(xqr_status) * chunk);
        if (need > ctx->pinned_out_bytes) {
            if (ctx->pinned_out) cudaFreeHost(ctx->pinned_out);
            ctx->pinned_out = nullptr;
            ctx->pinned_out_bytes = 0;
            e = cudaMallocHost(&ctx->pinned_out, need);
            if (e != cudaSuccess) return set_cuda_error(ctx, e, "pinned output allocation");
            ctx->pinned_out_bytes = need;
        }
    }
    cudaStream_t streams[2] = {ctx->stream, ctx->stream2};
    // the caller's stream may have pending work (e.g. torch): order stream2 after it
    cudaEventRecord(ctx->slot_done[1], ctx->stream);
    cudaStreamWaitEvent(ctx->stream2, ctx->slot_done[1], 0);
    int64_t pending[2] = {-1, -1};  // chunk index whose outputs sit in slot k
    std::vector<xqr_status> hst(batch);
    auto out_slot = [&](int k) {
        return static_cast<char*>(ctx->pinned_out) + k * (sizeof(double) * chunk * sout + sizeof(xqr_status) * chunk);
    };
    auto drain = [&](int k) -> int {
        if (pending[k] < 0) return 0;
        cudaError_t ee = cudaEventSynchronize(ctx->slot_done[k]);
        if (ee != cudaSuccess) return set_cuda_error(ctx, ee, "solve");
        const int64_t c = pending[k], s0 = c * chunk, cs = std::min(chunk, batch - s0);
        const double* src = reinterpret_cast<const double*>(out_slot(k));
        if (lsq) {
            std::memcpy(x + s0 * sx, src, sizeof(double) * cs * sx);
            std::memcpy(z + s0 * sz, src + cs * sx, sizeof(double) * cs * sz);
        } else {
            std::memcpy(q + s0 * sq, src, sizeof(double) * cs * sq);
            std::memcpy(r + s0 * sr, src + cs * sq, sizeof(double) * cs * sr);
        }
        const xqr_status* sst = reinterpret_cast<const xqr_status*>(out_slot(k) + sizeof(double) * chunk * sout);
        for (int64_t i = 0; i < cs; ++i) {
            hst[s0 + i] = sst[i];
            hst[s0 + i].system = s0 + i;
        }
        pending[k] = -1;
        return 0;
    };
    for (int64_t c = 0; c < nchunks; ++c) {
        const int k = (int)(c & 1);
        cudaStream_t s = streams[k];
        const int64_t s0 = c * chunk, cs = std::min(chunk, batch - s0);
        if (int rc = drain(k)) return rc;  // slot k free again
        double* d_in = reinterpret_cast<double*>(at(ctx, o_in[k]));
        double* d_out = reinterpret_cast<double*>(at(ctx, o_out[k]));
        xqr_status* d_st = reinterpret_cast<xqr_status*>(at(ctx, o_st[k]));
        const double* src_a = a + s0 * sa;
        const double* src_b = lsq ? b + s0 * sb : nullptr;
        if (!pin_a) {
            double* stage = static_cast<double*>(ctx->pinned) + (size_t)k * chunk * (sa + sb);
            std::memcpy(stage, src_a, sizeof(double) * cs * sa);
            if (lsq) std::memcpy(stage + cs * sa, src_b, sizeof(double) * cs * sb);
            src_a = stage;
            src_b = stage + cs * sa;
        }
        cudaMemcpyAsync(d_in, src_a, sizeof(double) * cs * sa, cudaMemcpyHostToDevice, s);
        if (lsq) cudaMemcpyAsync(d_in + cs * sa, src_b, sizeof(double) * cs * sb, cudaMemcpyHostToDevice, s);
        double *dq = nullptr, *dr = nullptr, *dx = nullptr, *dz = nullptr;
        if (lsq) {
            dx = d_out;
            dz = d_out + cs * sx;
        } else {
            dq = d_out;
            dr = d_out + cs * sq;
        }
        int rc = launch_cta_batch(ctx, s, lsq, limbs, cs, (int)m, (int)n, d_in, lsq ? d_in + cs * sa : nullptr,
                                  dq, dr, dx, dz, d_st, reinterpret_cast<double*>(at(ctx, o_ws[k])));
        if (rc) return rc;
        cudaMemcpyAsync(out_slot(k), d_out, sizeof(double) * cs * sout, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(out_slot(k) + sizeof(double) * chunk * sout, d_st, sizeof(xqr_status) * cs,
                        cudaMemcpyDeviceToHost, s);
        cudaEventRecord(ctx->slot_done[k], s);
        pending[k] = c;
    }
    for (int k = 0; k < 2; ++k)
        if (int rc = drain(k)) return rc;
    // later work on the ctx stream is ordered after both streams
    cudaEventRecord(ctx->slot_done[1], ctx->stream2);
    cudaStreamWaitEvent(ctx->stream, ctx->slot_done[1], 0);
    ctx->timed = false;
    if (st) std::memcpy(st, hst.data(), sizeof(xqr_status) * batch);
    return first_code(hst);
}

}  // namespace

static int solve_host(xqr_ctx* ctx, bool lsq, int limbs, int64_t batch, int64_t m, int64_t n,
                      const double* a, const double* b, double* q, double* r, double* x, double* z,
                      xqr_status* st) {
    if (!ctx) return XQR_USAGE;
    if (int c = check_shape(ctx, st, limbs, batch, m, n)) {
        for (int64_t s = 1; s < batch && st; ++s) fill_status(st + s, c, 0, s);
        return c;
    }
    if (batch == 0) return 0;
    cudaSetDevice(ctx->device);
    if (batch > 1 && m > 32 * xb::kMaxRowsPerLane) {
        // taller than one CTA holds: system by system on the grid kernels
        const size_t L2 = 2 * (size_t)limbs;
        int first = 0;
        for (int64_t s = 0; s < batch; ++s) {
            xqr_status one{};
            const int rc = solve_host(ctx, lsq, limbs, 1, m, n, a + s * m * n * L2, lsq ? b + s * m * L2 : nullptr,
                                      lsq ? nullptr : q + s * m * n * L2, lsq ? nullptr : r + s * n * n * L2,
                                      lsq ? x + s * n * L2 : nullptr, lsq ? z + s * limbs : nullptr, &one);
            if (rc >= XQR_DIMENSION) return rc;  // a call-level failure
            one.system = s;
            if (st) st[s] = one;
            if (rc && !first) first = rc;
        }
        return first;
    }
    if (batch > 1) return solve_host_batched(ctx, lsq, limbs, batch, m, n, a, b, q, r, x, z, st);
    const size_t L2 = 2 * (size_t)limbs;
    const size_t a_b = sizeof(double) * batch * m * n * L2;
    const size_t b_b = lsq ? sizeof(double) * batch * m * L2 : 0;
    const size_t q_b = lsq ? 0 : a_b;
    const size_t r_b = lsq ? 0 : sizeof(double) * batch * n * n * L2;
    const size_t x_b = lsq ? sizeof(double) * batch * n * L2 : 0;
    const size_t z_b = lsq ? sizeof(double) * batch * limbs : 0;
    const size_t s_b = sizeof(xqr_status) * batch;
    arena_plan plan;
    size_t o_a = plan.add(a_b), o_b = plan.add(b_b), o_q = plan.add(q_b), o_r = plan.add(r_b),
           o_x = plan.add(x_b), o_z = plan.add(z_b), o_s = plan.add(s_b);
    // the solver scratch goes after the I/O regions; make sure the arena is
    // large enough for the I/O regions before taking pointers into it
    const int ncol = (int)n + (lsq ? 1 : 0);
    size_t scratch = sizeof(double) * (size_t)batch *
                     (xb::ws_doubles(limbs, (int)m, ncol) + (lsq ? xb::rws_doubles(limbs, (int)n) : 0));
    if (batch == 1) scratch = std::max(scratch, grid_scratch_bytes(lsq, limbs, (int)m, (int)n));
    cudaError_t e = ensure_arena(ctx, plan.total + scratch + 512);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "workspace allocation");
    // one system: copy straight from the caller's buffer (pinned: one DMA;
    // pageable: the driver's own pipelined staging, measured faster than a
    // memcpy into our pinned buffer first -- cqd 256 e2e 9.97 -> 9.73 ms)
    cudaMemcpyAsync(at(ctx, o_a), a, a_b, cudaMemcpyHostToDevice, ctx->stream);
    if (lsq) cudaMemcpyAsync(at(ctx, o_b), b, b_b, cudaMemcpyHostToDevice, ctx->stream);
    int rc = solve_device(ctx, lsq, limbs, batch, m, n, (const double*)at(ctx, o_a),
                          (const double*)at(ctx, o_b), (double*)at(ctx, o_q), (double*)at(ctx, o_r),
                          (double*)at(ctx, o_x), (double*)at(ctx, o_z),
                          (xqr_status*)at(ctx, o_s), plan.total, true);
    if (rc) return rc;
    std::vector<xqr_status> hst(batch);
    cudaMemcpyAsync(hst.data(), at(ctx, o_s), s_b, cudaMemcpyDeviceToHost, ctx->stream);
    if (lsq) {
        cudaMemcpyAsync(x, at(ctx, o_x), x_b, cudaMemcpyDeviceToHost, ctx->stream);
        cudaMemcpyAsync(z, at(ctx, o_z), z_b, cudaMemcpyDeviceToHost, ctx->stream);
    } else {
        cudaMemcpyAsync(q, at(ctx, o_q), q_b, cudaMemcpyDeviceToHost, ctx->stream);
        cudaMemcpyAsync(r, at(ctx, o_r), r_b, cudaMemcpyDeviceToHost, ctx->stream);
    }
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "solve");
    if (st) std::memcpy(st, hst.data(), s_b);
    return first_code(hst);
}

int xqr_mgs_qr(xqr_ctx* ctx, int limbs, int64_t m, int64_t n, const double* a, double* q,
               double* r, xqr_status* st) {
    return solve_host(ctx, false, limbs, 1, m, n, a, nullptr, q, r, nullptr, nullptr, st);
}

int xqr_lsq_solve(xqr_ctx* ctx, int limbs, int64_t m, int64_t n, const double* a,
                  const double* b, double* x, double* z, xqr_status* st) {
    return solve_host(ctx, true, limbs, 1, m, n, a, b, nullptr, nullptr, x, z, st);
}

int xqr_mgs_qr_batched(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                       const double* a, double* q, double* r, xqr_status* st) {
    return solve_host(ctx, false, limbs, batch, m, n, a, nullptr, q, r, nullptr, nullptr, st);
}

int xqr_lsq_solve_batched(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                          const double* a, const double* b, double* x, double* z,
                          xqr_status* st) {
    return solve_host(ctx, true, limbs, batch, m, n, a, b, nullptr, nullptr, x, z, st);
}

int xqr_back_substitute(xqr_ctx* ctx, int limbs, int64_t rows, int64_t cols, const double* r,
                        int64_t ylen, const double* y, double* x, xqr_status* st) {
    if (!ctx) return XQR_USAGE;
    if (!valid_limbs(limbs)) return fail(ctx, st, XQR_USAGE, "limbs must be 1, 2 or 4");
    // mgs.hpp:113-114
    if (rows != cols) return fail(ctx, st, XQR_DIMENSION, "triangular factor must be square");
    if (ylen != cols) return fail(ctx, st, XQR_DIMENSION, "right-hand side length mismatch");
    if (cols < 1) return fail(ctx, st, XQR_DIMENSION, "empty triangular factor");
    cudaSetDevice(ctx->device);
    const int64_t n = cols;
    const size_t L2 = 2 * (size_t)limbs;
    const size_t r_b = sizeof(double) * n * n * L2, y_b = sizeof(double) * n * L2;
    const size_t prep_b = sizeof(double) * n * (3 * limbs + 1);
    arena_plan plan;
    size_t o_p = plan.add(prep_b), o_r = plan.add(r_b), o_y = plan.add(y_b), o_x = plan.add(y_b),
           o_s = plan.add(sizeof(xqr_status));
    cudaError_t e = ensure_arena(ctx, plan.total + 256);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "workspace allocation");
    cudaMemcpyAsync(at(ctx, o_r), r, r_b, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(at(ctx, o_y), y, y_b, cudaMemcpyHostToDevice, ctx->stream);
    xb::BackSubParams p{1, (int)n, (const double*)at(ctx, o_r), (const double*)at(ctx, o_y),
                        (double*)at(ctx, o_x), (xqr_status*)at(ctx, o_s), (double*)at(ctx, o_p)};
    e = xb::launch_back_substitute(limbs, p, ctx->stream);
    ctx->launches += 1;
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "back substitution launch");
    xqr_status hs;
    cudaMemcpyAsync(&hs, at(ctx, o_s), sizeof hs, cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(x, at(ctx, o_x), y_b, cudaMemcpyDeviceToHost, ctx->stream);
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "back substitution");
    if (st) *st = hs;
    return hs.code;
}

// ---- verification metrics (mgs.hpp:161-178, :208-222) -------------------------------
namespace {
// Scratch of one metric launch (partials + per-system flags), laid out in an
// arena plan that already holds any I/O regions of the call: the arena is
// sized ONCE, before the caller takes device pointers into it.
struct metric_scratch {
    size_t o_part, o_flg;
};
metric_scratch plan_metric(arena_plan& plan, int which, int limbs, int64_t batch, int64_t m, int64_t n) {
    metric_scratch ms;
    ms.o_part = plan.add(sizeof(double) * batch * xb::metric_blocks(which, (int)m, (int)n) * limbs);
    ms.o_flg = plan.add(sizeof(int) * batch);
    return ms;
}

int metric_launch(xqr_ctx* ctx, int which, int limbs, int64_t batch, int64_t m, int64_t n,
                  const double* d_a, const double* d_q, const double* d_r, double* d_out,
                  xqr_status* d_st, const metric_scratch& ms) {
    int* flags = reinterpret_cast<int*>(at(ctx, ms.o_flg));
    cudaMemsetAsync(flags, 0, sizeof(int) * batch, ctx->stream);
    cudaError_t e = xb::launch_metric(limbs, which, batch, (int)m, (int)n, d_a, d_q, d_r, d_out,
                                      reinterpret_cast<double*>(at(ctx, ms.o_part)), flags, d_st, ctx->stream);
    ctx->launches += 2;
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "metric launch");
    return 0;
}

// device-pointer form: the arena holds only the metric scratch
int metric_device(xqr_ctx* ctx, int which, int limbs, int64_t batch, int64_t m, int64_t n,
                  const double* d_a, const double* d_q, const double* d_r, double* d_out,
                  xqr_status* d_st) {
    arena_plan plan;
    const metric_scratch ms = plan_metric(plan, which, limbs, batch, m, n);
    cudaError_t e = ensure_arena(ctx, plan.total + 256);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "workspace allocation");
    return metric_launch(ctx, which, limbs, batch, m, n, d_a, d_q, d_r, d_out, d_st, ms);
}

int metric_host(xqr_ctx* ctx, int which, int limbs, int64_t batch, int64_t m, int64_t n, const double* a,
                const double* q, const double* r, double* out, xqr_status* st) {
    if (!ctx) return XQR_USAGE;
    if (int c = check_shape(ctx, st, limbs, batch, m, n)) return c;
    if (batch == 0) return 0;
    cudaSetDevice(ctx->device);
    const size_t L2 = 2 * (size_t)limbs;
    const size_t a_b = which == 0 ? sizeof(double) * batch * m * n * L2 : 0;
    const size_t q_b = sizeof(double) * batch * m * n * L2;
    const size_t r_b = which == 0 ? sizeof(double) * batch * n * n * L2 : 0;
    arena_plan plan;
    const size_t o_a = plan.add(a_b), o_q = plan.add(q_b), o_r = plan.add(r_b),
                 o_o = plan.add(sizeof(double) * batch * limbs), o_s = plan.add(sizeof(xqr_status) * batch);
    // the metric's own scratch goes into the same plan: one allocation, made
    // before any pointer into the arena is taken (a later growth would free
    // the regions the copies below fill)
    const metric_scratch ms = plan_metric(plan, which, limbs, batch, m, n);
    cudaError_t e = ensure_arena(ctx, plan.total + 256);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "workspace allocation");
    if (a_b) cudaMemcpyAsync(at(ctx, o_a), a, a_b, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(at(ctx, o_q), q, q_b, cudaMemcpyHostToDevice, ctx->stream);
    if (r_b) cudaMemcpyAsync(at(ctx, o_r), r, r_b, cudaMemcpyHostToDevice, ctx->stream);
    int rc = metric_launch(ctx, which, limbs, batch, m, n, (const double*)at(ctx, o_a),
                           (const double*)at(ctx, o_q), (const double*)at(ctx, o_r), (double*)at(ctx, o_o),
                           (xqr_status*)at(ctx, o_s), ms);
    if (rc) return rc;
    std::vector<xqr_status> hst(batch);
    cudaMemcpyAsync(out, at(ctx, o_o), sizeof(double) * batch * limbs, cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(hst.data(), at(ctx, o_s), sizeof(xqr_status) * batch, cudaMemcpyDeviceToHost, ctx->stream);
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "metric");
    if (st) std::memcpy(st, hst.data(), sizeof(xqr_status) * batch);
    return first_code(hst);
}
}  // namespace

int xqr_residual_max_entry(xqr_ctx* ctx, int limbs, int64_t m, int64_t n, const double* a,
                           const double* q, const double* r, double* out, xqr_status* st) {
    return metric_host(ctx, 0, limbs, 1, m, n, a, q, r, out, st);
}
int xqr_orthogonality_defect(xqr_ctx* ctx, int limbs, int64_t m, int64_t n, const double* q,
                             double* out, xqr_status* st) {
    return metric_host(ctx, 1, limbs, 1, m, n, nullptr, q, nullptr, out, st);
}
int xqr_residual_max_entry_batched(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                                   const double* a, const double* q, const double* r, double* out,
                                   xqr_status* st) {
    return metric_host(ctx, 0, limbs, batch, m, n, a, q, r, out, st);
}
int xqr_orthogonality_defect_batched(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                                     const double* q, double* out, xqr_status* st) {
    return metric_host(ctx, 1, limbs, batch, m, n, nullptr, q, nullptr, out, st);
}
int xqr_residual_max_entry_batched_device(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                                          const double* d_a, const double* d_q, const double* d_r,
                                          double* d_out, xqr_status* d_st) {
    if (!ctx) return XQR_USAGE;
    if (int c = check_shape(ctx, nullptr, limbs, batch, m, n)) return c;
    cudaSetDevice(ctx->device);
    return batch ? metric_device(ctx, 0, limbs, batch, m, n, d_a, d_q, d_r, d_out, d_st) : 0;
}
int xqr_orthogonality_defect_batched_device(xqr_ctx* ctx, int limbs, int64_t batch, int64_t m, int64_t n,
                                            const double* d_q, double* d_out, xqr_status* d_st) {
    if (!ctx) return XQR_USAGE;
    if (int c = check_shape(ctx, nullptr, limbs, batch, m, n)) return c;
    cudaSetDevice(ctx->device);
    return batch ? metric_device(ctx, 1, limbs, batch, m, n, nullptr, d_q, nullptr, d_out, d_st) : 0;
}

int xqr_arith(xqr_ctx* ctx, int limbs, int op, int64_t count, const double* a, const double* b,
              double* out, int32_t* codes) {
    if (!ctx) return XQR_USAGE;
    if (!valid_limbs(limbs) || op < 0 || op > 8) return XQR_USAGE;
    cudaSetDevice(ctx->device);
    const size_t stride = (op >= 5 && op <= 7) ? 2 * limbs : limbs;
    const size_t bytes = sizeof(double) * stride * count;
    arena_plan plan;
    size_t o_a = plan.add(bytes), o_b = plan.add(bytes), o_o = plan.add(bytes),
           o_c = plan.add(sizeof(int32_t) * count);
    cudaError_t e = ensure_arena(ctx, plan.total + 256);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "workspace allocation");
    cudaMemcpyAsync(at(ctx, o_a), a, bytes, cudaMemcpyHostToDevice, ctx->stream);
    if (b) cudaMemcpyAsync(at(ctx, o_b), b, bytes, cudaMemcpyHostToDevice, ctx->stream);
    e = xb::launch_arith(limbs, op, count, (const double*)at(ctx, o_a),
                         b ? (const double*)at(ctx, o_b) : nullptr, (double*)at(ctx, o_o),
                         (int32_t*)at(ctx, o_c), ctx->stream);
    ctx->launches += 1;
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "arith launch");
    cudaMemcpyAsync(out, at(ctx, o_o), bytes, cudaMemcpyDeviceToHost, ctx->stream);
    if (codes) cudaMemcpyAsync(codes, at(ctx, o_c), sizeof(int32_t) * count, cudaMemcpyDeviceToHost,
                               ctx->stream);
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return set_cuda_error(ctx, e, "arith");
    return 0;
}

}  // extern "C"

// aidw_api.cu -- the C ABI declared in include/aidw.h: argument validation,
// handle ownership, dispatch to the sm_100a kernels, status codes.
#include "aidw.h"
#include "aidw_internal.h"

#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>

struct aidw_ctx {
    int device = 0;
    aidw_dtype dt = AIDW_F32;
    int64_t nd = 0, ndp = 0;
    double area = 0.0, r_exp = 0.0;
    void *data = nullptr;            // [3][ndp] T, internal SoA
    aidw::Scratch *sc = nullptr;     // device scratch
    aidw::FilterData filt;           // fp32 kNN filter arrays
    void *work = nullptr;            // run_host / internal d1sq scratch
    size_t work_bytes = 0;
    int *perm = nullptr;             // weighting-pass class permutation (fp32)
    int64_t perm_cap = 0;
    aidw::SplitBuf split;            // small-nq data split scratch
    // GLOBAL-bounds exchange over peer memory
    aidw::ExBuf *ex_own = nullptr;   // this rank's buffer (peers write into it)
    aidw::ExBuf **ex_peers_dev = nullptr;
    aidw::ExBuf *ex_mapped[aidw::kExMaxRanks] = {};  // IPC-opened peer buffers
    int ex_rank = -1, ex_world = 0;
    bool ex_connected = false;
    int64_t launches = 0;
    double bbox[4] = {0, 0, 0, 0};
    char err[512] = {0};
};

cudaError_t aidw::dev_malloc(void **p, size_t n)
{
    int dev = 0;
    cudaGetDevice(&dev);
    {
        static std::mutex m;
        static bool init[256] = {};
        std::lock_guard<std::mutex> g(m);
        if (dev >= 0 && dev < 256 && !init[dev]) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            init[dev] = true;
        }
    }
    cudaError_t e = cudaMallocAsync(p, n, cudaStreamLegacy);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);
    return e;
}

void aidw::dev_free(void *p)
{
    if (p) cudaFreeAsync(p, cudaStreamLegacy);
}

void *aidw::SplitBuf::reserve(size_t n)
{
    if (n <= bytes) return p;
    if (p) {
        cudaDeviceSynchronize();
        aidw::dev_free(p);
        p = nullptr;
        bytes = 0;
    }
    n = (n + (size_t(1) << 20) - 1) >> 20 << 20;
    if (aidw::dev_malloc((void **)&p, n) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        return nullptr;
    }
    bytes = n;
    return p;
}

namespace {

thread_local char g_err[512];

size_t tsize(aidw_dtype dt) { return dt == AIDW_F32 ? sizeof(float) : sizeof(double); }

aidw_status fail(aidw_t h, aidw_status st, const char *fmt, ...)
{
    char *buf = h ? h->err : g_err;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, 512, fmt, ap);
    va_end(ap);
    return st;
}

aidw_status cuda_fail(aidw_t h, cudaError_t e, const char *where)
{
    return fail(h, AIDW_E_CUDA, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define CK(h, call)                                                       \
    do {                                                                  \
        cudaError_t e_ = (call);                                          \
        if (e_ != cudaSuccess) return cuda_fail((h), e_, #call);          \
    } while (0)

aidw_status launched(aidw_t h, int n, const char *what)
{
    if (n < 0) {
        cudaError_t e = cudaGetLastError();
        return cuda_fail(h, e, what);
    }
    h->launches += n;
    return AIDW_OK;
}

aidw_status ensure_work(aidw_t h, size_t bytes)
{
    if (h->work_bytes >= bytes) return AIDW_OK;
    if (h->work) {
        cudaDeviceSynchronize();
        aidw::dev_free(h->work);
        h->work = nullptr;
        h->work_bytes = 0;
    }
    cudaError_t e = aidw::dev_malloc((void **)&h->work, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(h, AIDW_E_NOMEM, "cudaMalloc(%zu) for scratch: %s", bytes, cudaGetErrorString(e));
    }
    h->work_bytes = bytes;
    return AIDW_OK;
}

// Class permutation buffer for the fp32 weighting pass (nullptr: feature disabled or
// fp64).  AIDW_ALPHA_CLASSES=0 disables the exact-exponent paths.
int *perm_for(aidw_t h, int64_t nq)
{
    if (h->dt != AIDW_F32 || nq > INT_MAX) return nullptr;  // the permutation is int32
    static int enabled = -1;
    if (enabled < 0) {
        const char *e = getenv("AIDW_ALPHA_CLASSES");
        enabled = !(e && e[0] == '0');
    }
    if (!enabled) return nullptr;
    if (h->perm_cap < nq) {
        if (h->perm) {
            cudaDeviceSynchronize();
            aidw::dev_free(h->perm);
            h->perm = nullptr;
            h->perm_cap = 0;
        }
        if (aidw::dev_malloc((void **)&h->perm, (size_t)nq * sizeof(int)) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;  // fall back to the unpermuted (general-formula) launch
        }
        h->perm_cap = nq;
    }
    return h->perm;
}

// Small-nq data split: the handle's growable scratch, or nullptr when
// nq is large enough that the query grid alone fills the GPU.
aidw::SplitBuf *split_for(aidw_t h, int64_t nq)
{
    constexpr int64_t kSplitMaxQ = int64_t(1) << 20;
    return nq <= kSplitMaxQ ? &h->split : nullptr;
}

bool is_device_ptr(const void *p)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

double decode_key(unsigned long long k)
{
    unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double d;
    std::memcpy(&d, &u, sizeof d);
    return d;
}

aidw_status check_levels(aidw_t h, const double *lv)
{
    if (!lv) return fail(h, AIDW_E_INVALID_ARG, "alpha_lv is NULL");
    for (int i = 0; i < 5; ++i)
        if (!(std::isfinite(lv[i]) && lv[i] > 0.0))
            return fail(h, AIDW_E_INVALID_ARG, "alpha_lv[%d] = %g must be finite and > 0", i, lv[i]);
    return AIDW_OK;
}

}  // namespace

extern "C" {

int aidw_abi_version(void) { return AIDW_ABI_VERSION; }

const char *aidw_status_string(aidw_status s)
{
    switch (s) {
    case AIDW_OK: return "AIDW_OK";
    case AIDW_E_INVALID_ARG: return "AIDW_E_INVALID_ARG";
    case AIDW_E_INSUFFICIENT_DATA: return "AIDW_E_INSUFFICIENT_DATA";
    case AIDW_E_DEGENERATE_EXTENT: return "AIDW_E_DEGENERATE_EXTENT";
    case AIDW_E_INVALID_AREA: return "AIDW_E_INVALID_AREA";
    case AIDW_E_INVALID_BOUNDS: return "AIDW_E_INVALID_BOUNDS";
    case AIDW_E_NONFINITE_INPUT: return "AIDW_E_NONFINITE_INPUT";
    case AIDW_E_UNSUPPORTED: return "AIDW_E_UNSUPPORTED";
    case AIDW_E_CUDA: return "AIDW_E_CUDA";
    case AIDW_E_NOMEM: return "AIDW_E_NOMEM";
    }
    return "AIDW_E_UNKNOWN";
}

const char *aidw_last_error(aidw_t h) { return h ? h->err : g_err; }

aidw_status aidw_create(aidw_t *out, int device, aidw_dtype dt, aidw_layout lay, const void *data_xyz,
                        int64_t nd, double area, void *stream)
{
    if (!out) return fail(nullptr, AIDW_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (dt != AIDW_F32 && dt != AIDW_F64) return fail(nullptr, AIDW_E_UNSUPPORTED, "unknown dtype %d", (int)dt);
    if (lay != AIDW_SOA && lay != AIDW_AOS && lay != AIDW_AOAS)
        return fail(nullptr, AIDW_E_UNSUPPORTED, "unknown layout %d", (int)lay);
    if (!data_xyz) return fail(nullptr, AIDW_E_INVALID_ARG, "data_xyz is NULL");
    if (nd < 1) return fail(nullptr, AIDW_E_INVALID_ARG, "nd = %lld must be >= 1", (long long)nd);
    if (std::isnan(area) || std::isinf(area) || area < 0.0)
        return fail(nullptr, AIDW_E_INVALID_AREA, "area = %g must be > 0 (explicit) or 0 (bbox)", area);
    if (nd > (int64_t)1 << 40) return fail(nullptr, AIDW_E_UNSUPPORTED, "nd too large");

    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);

    aidw_ctx *h = new (std::nothrow) aidw_ctx;
    if (!h) return fail(nullptr, AIDW_E_NOMEM, "host allocation failed");
    h->device = device;
    h->dt = dt;
    h->nd = nd;
    h->ndp = (nd + aidw::kPad - 1) / aidw::kPad * aidw::kPad;
    const size_t ts = tsize(dt);
    const size_t ncomp = lay == AIDW_AOAS ? 4 : 3;
    const size_t in_bytes = (size_t)nd * ncomp * ts;

    auto bail = [&](aidw_status s) {
        std::memcpy(g_err, h->err, sizeof g_err);
        aidw_destroy(h);
        return s;
    };

    if ((e = aidw::dev_malloc((void **)&h->data, 3 * (size_t)h->ndp * ts)) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(h, AIDW_E_NOMEM, "cudaMalloc data: %s", cudaGetErrorString(e)));
    }
    if ((e = aidw::dev_malloc((void **)&h->sc, sizeof(aidw::Scratch))) != cudaSuccess) {
        cudaGetLastError();
        return bail(fail(h, AIDW_E_NOMEM, "cudaMalloc scratch: %s", cudaGetErrorString(e)));
    }
    aidw::Scratch init{};
    init.mn = ~0ull;
    init.mx = 0ull;
    init.done = 0;
    init.err_idx = LLONG_MAX;
    init.keys[0] = ~0ull;
    init.keys[1] = 0ull;
    init.keys[2] = ~0ull;
    init.keys[3] = 0ull;
    init.nonfinite = 0;
    if ((e = cudaMemcpy(h->sc, &init, sizeof init, cudaMemcpyHostToDevice)) != cudaSuccess)
        return bail(cuda_fail(h, e, "init scratch"));

    const void *src = data_xyz;
    void *staged = nullptr;
    if (!is_device_ptr(data_xyz)) {  // host data: stage it
        if ((e = aidw::dev_malloc((void **)&staged, in_bytes)) != cudaSuccess) {
            cudaGetLastError();
            return bail(fail(h, AIDW_E_NOMEM, "cudaMalloc staging: %s", cudaGetErrorString(e)));
        }
        if ((e = cudaMemcpyAsync(staged, data_xyz, in_bytes, cudaMemcpyHostToDevice, st)) != cudaSuccess) {
            aidw::dev_free(staged);
            return bail(cuda_fail(h, e, "H2D data"));
        }
        src = staged;
    }
    aidw_status s = launched(h, aidw::launch_prep((int)dt, (int)lay, src, nd, h->ndp, h->data, h->sc, st),
                             "prep kernel");
    aidw::Scratch back;
    if (s == AIDW_OK) {
        if ((e = cudaMemcpyAsync(&back, h->sc, sizeof back, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
            (e = cudaStreamSynchronize(st)) != cudaSuccess)
            s = cuda_fail(h, e, "read bbox");
    }
    if (staged) aidw::dev_free(staged);
    if (s != AIDW_OK) return bail(s);
    if (back.nonfinite)
        return bail(fail(h, AIDW_E_NONFINITE_INPUT, "%llu data values are NaN/Inf", back.nonfinite));

    // A: explicit, or the exact bbox (min/max exact; fp64 sub and mul) -- DESIGN.md R5
    const double x0 = decode_key(back.keys[0]), x1 = decode_key(back.keys[1]);
    const double y0 = decode_key(back.keys[2]), y1 = decode_key(back.keys[3]);
    h->bbox[0] = x0;
    h->bbox[1] = x1;
    h->bbox[2] = y0;
    h->bbox[3] = y1;
    h->area = area > 0.0 ? area : (x1 - x0) * (y1 - y0);
    if (!(h->area > 0.0) || std::isinf(h->area))
        return bail(fail(h, AIDW_E_DEGENERATE_EXTENT, "study area A = %g (bbox [%g,%g]x[%g,%g])", h->area, x0,
                         x1, y0, y1));
    h->r_exp = 1.0 / (2.0 * std::sqrt((double)nd / h->area));  // Eq. 2, printed order

    {
        // centred filter arrays for the kNN; c = bbox centre in fp32,
        // r1 >= max |x - c_x| + |y - c_y| over the data (fp64, padded for fp32 rounding).
        // fp64 handles use the same fp32 filter (fp64 re-check) when the data extent keeps
        // the filter arithmetic in fp32's normal range: R1 in [2^-60, 2^60].
        const char *env = getenv("AIDW_KNN_FILTER");
        const float cxf = (float)(0.5 * (x0 + x1)), cyf = (float)(0.5 * (y0 + y1));
        const double rx = std::fmax(std::fabs(x0 - cxf), std::fabs(x1 - cxf));
        const double ry = std::fmax(std::fabs(y0 - cyf), std::fabs(y1 - cyf));
        const double r1 = (rx + ry) * (1.0 + 1e-6);
        const bool safe = dt == AIDW_F32 || (std::isfinite(cxf) && std::isfinite(cyf) && r1 >= 0x1p-60 && r1 <= 0x1p60);
        if (!(env && env[0] == '0') && safe) {
            if ((e = aidw::dev_malloc((void **)&h->filt.arrays, 8 * (size_t)h->ndp * sizeof(float))) != cudaSuccess ||
                (e = aidw::dev_malloc((void **)&h->filt.cell_start, (aidw::kCells + 1) * sizeof(int))) != cudaSuccess ||
                (dt == AIDW_F64 &&
                 (e = aidw::dev_malloc((void **)&h->filt.coords64, 2 * (size_t)h->ndp * sizeof(double))) != cudaSuccess)) {
                cudaGetLastError();
                return bail(fail(h, AIDW_E_NOMEM, "cudaMalloc filter: %s", cudaGetErrorString(e)));
            }
            h->filt.c_x = cxf;
            h->filt.c_y = cyf;
            h->filt.r1 = (float)r1;
            // Morton order grid over the data bbox
            constexpr double cells = (double)(1 << aidw::kOrderBits);
            h->filt.grid = aidw::OrderGrid{(float)x0, (float)y0, (float)(cells / (x1 - x0)),
                                           (float)(cells / (y1 - y0))};
            s = launched(h, aidw::launch_order_data((int)dt, h->data, h->ndp, nd, &h->filt, st), "order data kernels");
            if (s != AIDW_OK) return bail(s);
            if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return bail(cuda_fail(h, e, "order data sync"));
        }
    }
    *out = h;
    return AIDW_OK;
}

int64_t aidw_nd(aidw_t h) { return h ? h->nd : -1; }
double aidw_area(aidw_t h) { return h ? h->area : 0.0; }
double aidw_r_exp(aidw_t h) { return h ? h->r_exp : 0.0; }
aidw_dtype aidw_dtype_of(aidw_t h) { return h ? h->dt : AIDW_F32; }
int64_t aidw_launch_count(aidw_t h) { return h ? h->launches : -1; }

aidw_status aidw_knn_robs(aidw_t h, const void *qx, const void *qy, int64_t nq, int k, void *r_obs,
                          void *d1sq, void *robs_minmax, void *knn_dists, void *stream)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (nq < 0) return fail(h, AIDW_E_INVALID_ARG, "nq < 0");
    if (k < 1) return fail(h, AIDW_E_INVALID_ARG, "k = %d must be >= 1", k);
    if (k > AIDW_KMAX) return fail(h, AIDW_E_UNSUPPORTED, "k = %d > AIDW_KMAX = %d", k, AIDW_KMAX);
    if (h->nd < k)
        return fail(h, AIDW_E_INSUFFICIENT_DATA, "nd = %lld < k = %d", (long long)h->nd, k);
    if (nq > 0 && (!qx || !qy || !r_obs)) return fail(h, AIDW_E_INVALID_ARG, "qx/qy/r_obs is NULL");
    if (nq > (int64_t)1 << 40) return fail(h, AIDW_E_UNSUPPORTED, "nq too large");
    CK(h, cudaSetDevice(h->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (h->ex_connected && !robs_minmax)
        return fail(h, AIDW_E_INVALID_ARG, "the bounds exchange needs robs_minmax (peers wait for it)");
    if (nq == 0) {
        if (robs_minmax) {
            aidw_status s = launched(h, aidw::launch_minmax_identity((int)h->dt, robs_minmax, st), "minmax");
            if (s != AIDW_OK || !h->ex_connected) return s;
            return launched(h, aidw::launch_exchange_push_identity(h->sc, st), "exchange push");
        }
        return AIDW_OK;
    }
    return launched(h,
                    aidw::launch_knn((int)h->dt, k, h->data, h->ndp, qx, qy, nq, r_obs, d1sq, robs_minmax,
                                     knn_dists, h->sc, &h->filt, st, 0, split_for(h, nq)),
                    "knn_robs kernel");
}

aidw_status aidw_alpha(aidw_t h, const void *r_obs, int64_t nq, const double *alpha_lv, aidw_rbounds rb,
                       double r_min, double r_max, const void *robs_minmax, aidw_muform mf, void *alpha,
                       void *stream)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (nq < 0) return fail(h, AIDW_E_INVALID_ARG, "nq < 0");
    aidw_status s = check_levels(h, alpha_lv);
    if (s != AIDW_OK) return s;
    if (rb != AIDW_RB_GLOBAL && rb != AIDW_RB_FIXED) return fail(h, AIDW_E_INVALID_ARG, "bad rbounds");
    if (mf != AIDW_MU_NORMALIZED && mf != AIDW_MU_PRINTED) return fail(h, AIDW_E_INVALID_ARG, "bad muform");
    if (rb == AIDW_RB_FIXED) {
        if (!(std::isfinite(r_min) && std::isfinite(r_max)))
            return fail(h, AIDW_E_INVALID_BOUNDS, "r_min/r_max must be finite");
        if (!(r_min < r_max)) return fail(h, AIDW_E_INVALID_BOUNDS, "r_min = %g >= r_max = %g", r_min, r_max);
    } else if (nq > 0 && !robs_minmax && !h->ex_connected) {
        return fail(h, AIDW_E_INVALID_ARG, "GLOBAL bounds need robs_minmax (or a connected bounds exchange)");
    }
    // GLOBAL with robs_minmax == NULL on a connected handle: bounds from the exchange
    aidw::Scratch *ex = (rb == AIDW_RB_GLOBAL && !robs_minmax && h->ex_connected) ? h->sc : nullptr;
    // nq == 0 on a connected exchange still launches (one CTA): this rank must read and
    // ack the step's bounds, or its peers would wait for the ack before step + 2
    if (nq == 0 && !ex) return AIDW_OK;
    if (nq > 0 && (!r_obs || !alpha)) return fail(h, AIDW_E_INVALID_ARG, "r_obs/alpha is NULL");
    CK(h, cudaSetDevice(h->device));
    return launched(h,
                    aidw::launch_alpha((int)h->dt, r_obs, nq, h->r_exp, alpha_lv, (int)rb, r_min, r_max,
                                       robs_minmax, (int)mf, alpha, static_cast<cudaStream_t>(stream), ex),
                    "alpha kernel");
}

aidw_status aidw_exchange_setup(aidw_t h, int rank, int world, void *ipc_handle_out)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (world < 1 || world > aidw::kExMaxRanks || rank < 0 || rank >= world || !ipc_handle_out)
        return fail(h, AIDW_E_INVALID_ARG, "rank %d / world %d (max %d) / handle buffer", rank, world,
                    aidw::kExMaxRanks);
    if (h->ex_own) return fail(h, AIDW_E_INVALID_ARG, "exchange already set up");
    CK(h, cudaSetDevice(h->device));
    cudaError_t e = cudaMalloc(&h->ex_own, sizeof(aidw::ExBuf));
    if (e != cudaSuccess) {
        h->ex_own = nullptr;
        return cuda_fail(h, e, "cudaMalloc exchange buffer");
    }
    CK(h, cudaMemset(h->ex_own, 0, sizeof(aidw::ExBuf)));
    cudaIpcMemHandle_t ih;
    CK(h, cudaIpcGetMemHandle(&ih, h->ex_own));
    std::memcpy(ipc_handle_out, &ih, sizeof ih);
    h->ex_rank = rank;
    h->ex_world = world;
    return AIDW_OK;
}

aidw_status aidw_exchange_connect(aidw_t h, const void *ipc_handles)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (!h->ex_own || !ipc_handles) return fail(h, AIDW_E_INVALID_ARG, "aidw_exchange_setup first / NULL handles");
    if (h->ex_connected) return fail(h, AIDW_E_INVALID_ARG, "exchange already connected");
    CK(h, cudaSetDevice(h->device));
    CK(h, cudaDeviceSynchronize());
    const char *hb = static_cast<const char *>(ipc_handles);
    aidw::ExBuf *ptrs[aidw::kExMaxRanks] = {};
    for (int r = 0; r < h->ex_world; ++r) {
        if (r == h->ex_rank) {
            ptrs[r] = h->ex_own;
            continue;
        }
        cudaIpcMemHandle_t ih;
        std::memcpy(&ih, hb + (size_t)r * sizeof ih, sizeof ih);
        void *p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return cuda_fail(h, e, "cudaIpcOpenMemHandle (peer exchange buffer)");
        h->ex_mapped[r] = static_cast<aidw::ExBuf *>(p);
        ptrs[r] = h->ex_mapped[r];
    }
    CK(h, cudaMalloc(&h->ex_peers_dev, sizeof(ptrs)));
    CK(h, cudaMemcpy(h->ex_peers_dev, ptrs, sizeof(ptrs), cudaMemcpyHostToDevice));
    aidw::Scratch sc;
    CK(h, cudaMemcpy(&sc, h->sc, sizeof sc, cudaMemcpyDeviceToHost));
    sc.ex_peers = h->ex_peers_dev;
    sc.ex_rank = h->ex_rank;
    sc.ex_world = h->ex_world;
    sc.ex_epoch = 0;
    sc.ex_timeout = 0;
    sc.ex_readers = 0;
    CK(h, cudaMemcpy(h->sc, &sc, sizeof sc, cudaMemcpyHostToDevice));
    h->ex_connected = true;
    return AIDW_OK;
}

aidw_status aidw_exchange_close(aidw_t h)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    CK(h, cudaSetDevice(h->device));
    CK(h, cudaDeviceSynchronize());
    if (h->ex_connected) {
        aidw::Scratch sc;
        CK(h, cudaMemcpy(&sc, h->sc, sizeof sc, cudaMemcpyDeviceToHost));
        sc.ex_peers = nullptr;
        sc.ex_world = 0;
        CK(h, cudaMemcpy(h->sc, &sc, sizeof sc, cudaMemcpyHostToDevice));
    }
    for (int r = 0; r < aidw::kExMaxRanks; ++r)
        if (h->ex_mapped[r]) {
            cudaIpcCloseMemHandle(h->ex_mapped[r]);
            h->ex_mapped[r] = nullptr;
        }
    if (h->ex_peers_dev) cudaFree(h->ex_peers_dev);
    if (h->ex_own) cudaFree(h->ex_own);
    h->ex_peers_dev = nullptr;
    h->ex_own = nullptr;
    h->ex_connected = false;
    h->ex_world = 0;
    h->ex_rank = -1;
    return AIDW_OK;
}

aidw_status aidw_interpolate(aidw_t h, const void *qx, const void *qy, int64_t nq, const void *alpha,
                             const void *d1sq, void *z_out, void *stream)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (nq < 0) return fail(h, AIDW_E_INVALID_ARG, "nq < 0");
    if (nq == 0) return AIDW_OK;
    if (!qx || !qy || !alpha || !z_out) return fail(h, AIDW_E_INVALID_ARG, "qx/qy/alpha/z_out is NULL");
    CK(h, cudaSetDevice(h->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!d1sq) {  // nearest squared distance via the k = 1 kNN pass
        const size_t ts = tsize(h->dt);
        aidw_status s = ensure_work(h, 2 * (((size_t)nq * ts + 255) / 256 * 256));
        if (s != AIDW_OK) return s;
        void *robs = h->work;
        void *d1 = static_cast<char *>(h->work) + ((size_t)nq * ts + 255) / 256 * 256;
        s = launched(h,
                     aidw::launch_knn((int)h->dt, 1, h->data, h->ndp, qx, qy, nq, robs, d1, nullptr, nullptr,
                                      h->sc, &h->filt, st, 0, split_for(h, nq)),
                     "nearest kernel");
        if (s != AIDW_OK) return s;
        d1sq = d1;
    }
    aidw::SplitBuf *sp = split_for(h, nq);
    return launched(h,
                    aidw::launch_interp((int)h->dt, h->data, h->ndp, h->nd, qx, qy, nq, alpha, 0.0, d1sq, z_out, st,
                                        nullptr, perm_for(h, nq), h->sc->cls, sp, h->bbox),
                    "interpolate kernel");
}

aidw_status aidw_run_fixed(aidw_t h, const void *qx, const void *qy, int64_t nq, int k, const double *alpha_lv,
                           double r_min, double r_max, aidw_muform mf, void *z_out, void *r_obs_out,
                           void *alpha_out, void *stream)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (nq < 0) return fail(h, AIDW_E_INVALID_ARG, "nq < 0");
    aidw_status s = check_levels(h, alpha_lv);
    if (s != AIDW_OK) return s;
    if (!(std::isfinite(r_min) && std::isfinite(r_max)))
        return fail(h, AIDW_E_INVALID_BOUNDS, "r_min/r_max must be finite");
    if (!(r_min < r_max)) return fail(h, AIDW_E_INVALID_BOUNDS, "r_min = %g >= r_max = %g", r_min, r_max);
    if (mf != AIDW_MU_NORMALIZED && mf != AIDW_MU_PRINTED) return fail(h, AIDW_E_INVALID_ARG, "bad muform");
    if (k < 1) return fail(h, AIDW_E_INVALID_ARG, "k = %d must be >= 1", k);
    if (k > AIDW_KMAX) return fail(h, AIDW_E_UNSUPPORTED, "k = %d > AIDW_KMAX = %d", k, AIDW_KMAX);
    if (h->nd < k) return fail(h, AIDW_E_INSUFFICIENT_DATA, "nd = %lld < k = %d", (long long)h->nd, k);
    if (nq == 0) return AIDW_OK;
    if (!qx || !qy || !z_out) return fail(h, AIDW_E_INVALID_ARG, "qx/qy/z_out is NULL");
    CK(h, cudaSetDevice(h->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (h->dt == AIDW_F32 && h->filt.arrays)
        return launched(h,
                        aidw::launch_fused_fixed(h->data, h->ndp, h->nd, &h->filt, qx, qy, nq, k, h->r_exp, alpha_lv,
                                                 r_min, r_max, (int)mf, z_out, r_obs_out, alpha_out, h->sc, st),
                        "fused kernel");
    // fp64 (or no filter): the three stage kernels on handle scratch
    const size_t ts = tsize(h->dt);
    const size_t nb = ((size_t)nq * ts + 255) / 256 * 256;
    if ((s = ensure_work(h, 3 * nb)) != AIDW_OK) return s;
    char *w = static_cast<char *>(h->work);
    void *robs = r_obs_out ? r_obs_out : w, *d1 = w + nb, *al = alpha_out ? alpha_out : w + 2 * nb;
    if ((s = aidw_knn_robs(h, qx, qy, nq, k, robs, d1, nullptr, nullptr, stream)) != AIDW_OK) return s;
    if ((s = aidw_alpha(h, robs, nq, alpha_lv, AIDW_RB_FIXED, r_min, r_max, nullptr, mf, al, stream)) != AIDW_OK)
        return s;
    return aidw_interpolate(h, qx, qy, nq, al, d1, z_out, stream);
}

aidw_status aidw_idw(aidw_t h, const void *qx, const void *qy, int64_t nq, double alpha, void *z_out, void *stream)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (nq < 0) return fail(h, AIDW_E_INVALID_ARG, "nq < 0");
    if (!(std::isfinite(alpha) && alpha > 0.0)) return fail(h, AIDW_E_INVALID_ARG, "alpha = %g must be > 0", alpha);
    if (nq == 0) return AIDW_OK;
    if (!qx || !qy || !z_out) return fail(h, AIDW_E_INVALID_ARG, "qx/qy/z_out is NULL");
    CK(h, cudaSetDevice(h->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t ts = tsize(h->dt);
    const size_t nb = ((size_t)nq * ts + 255) / 256 * 256;
    aidw_status s = ensure_work(h, 2 * nb);
    if (s != AIDW_OK) return s;
    char *w = static_cast<char *>(h->work);
    s = launched(h,
                 aidw::launch_knn((int)h->dt, 1, h->data, h->ndp, qx, qy, nq, w, w + nb, nullptr, nullptr, h->sc,
                                  &h->filt, st, 0, split_for(h, nq)),
                 "nearest kernel");
    if (s != AIDW_OK) return s;
    aidw::SplitBuf *sp = split_for(h, nq);
    return launched(h,
                    aidw::launch_interp((int)h->dt, h->data, h->ndp, h->nd, qx, qy, nq, nullptr, alpha, w + nb,
                                        z_out, st, nullptr, perm_for(h, nq), h->sc->cls, sp, h->bbox),
                    "interpolate kernel");
}

aidw_status aidw_paper_baseline(int variant, aidw_dtype dt, aidw_layout lay, const void *data, int64_t nd,
                                const void *qx, const void *qy, int64_t nq, int k, const double *alpha_lv,
                                double area, double r_min, double r_max, void *z_out, void *stream)
{
    if (variant != 0 && variant != 1) return fail(nullptr, AIDW_E_INVALID_ARG, "variant must be 0 or 1");
    if (dt != AIDW_F32 && dt != AIDW_F64) return fail(nullptr, AIDW_E_UNSUPPORTED, "unknown dtype");
    if (lay != AIDW_SOA && lay != AIDW_AOAS) return fail(nullptr, AIDW_E_UNSUPPORTED, "layout must be SOA or AOAS");
    if (!data || !qx || !qy || !z_out || !alpha_lv) return fail(nullptr, AIDW_E_INVALID_ARG, "NULL argument");
    if (nd < 1 || nq < 0) return fail(nullptr, AIDW_E_INVALID_ARG, "bad sizes");
    if (!(area > 0.0) || std::isinf(area)) return fail(nullptr, AIDW_E_INVALID_AREA, "area must be > 0");
    if (k < 1 || k > AIDW_KMAX) return fail(nullptr, AIDW_E_UNSUPPORTED, "k out of range");
    if (nd < k) return fail(nullptr, AIDW_E_INSUFFICIENT_DATA, "nd < k");
    if (!(r_min < r_max)) return fail(nullptr, AIDW_E_INVALID_BOUNDS, "r_min >= r_max");
    if (nq == 0) return AIDW_OK;
    const double r_exp = 1.0 / (2.0 * std::sqrt((double)nd / area));
    if (aidw::launch_paper(variant, (int)dt, (int)lay, data, nd, qx, qy, nq, k, r_exp, alpha_lv, r_min, r_max, z_out,
                           static_cast<cudaStream_t>(stream)) < 0)
        return cuda_fail(nullptr, cudaGetLastError(), "paper baseline kernel");
    return AIDW_OK;
}

aidw_status aidw_set_extent(aidw_t h, int64_t nd_total, double area)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (nd_total < 1) return fail(h, AIDW_E_INVALID_ARG, "nd_total must be >= 1");
    if (!(area > 0.0) || std::isinf(area)) return fail(h, AIDW_E_INVALID_AREA, "area = %g must be > 0", area);
    h->area = area;
    h->r_exp = 1.0 / (2.0 * std::sqrt((double)nd_total / area));  // Eq. 2
    return AIDW_OK;
}

aidw_status aidw_set_extent_bbox(aidw_t h, int64_t nd_total, const double *bbox)
{
    if (!h || !bbox) return fail(h, AIDW_E_INVALID_ARG, "NULL argument");
    if (nd_total < 1) return fail(h, AIDW_E_INVALID_ARG, "nd_total must be >= 1");
    const double area = (bbox[1] - bbox[0]) * (bbox[3] - bbox[2]);  // DESIGN.md R5, as in aidw_create
    if (std::isnan(area) || std::isinf(area))
        return fail(h, AIDW_E_INVALID_AREA, "job bbox area = %g is not finite", area);
    if (!(area > 0.0))
        return fail(h, AIDW_E_DEGENERATE_EXTENT, "study area A = %g (bbox [%g,%g]x[%g,%g])", area, bbox[0],
                    bbox[1], bbox[2], bbox[3]);
    return aidw_set_extent(h, nd_total, area);
}

aidw_status aidw_bbox(aidw_t h, double *out)
{
    if (!h || !out) return fail(h, AIDW_E_INVALID_ARG, "NULL argument");
    for (int i = 0; i < 4; ++i) out[i] = h->bbox[i];
    return AIDW_OK;
}

aidw_status aidw_knn_partial(aidw_t h, const void *qx, const void *qy, int64_t nq, int k, void *s_out, void *stream)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (nq < 0) return fail(h, AIDW_E_INVALID_ARG, "nq < 0");
    if (k < 1) return fail(h, AIDW_E_INVALID_ARG, "k = %d must be >= 1", k);
    if (k > AIDW_KMAX) return fail(h, AIDW_E_UNSUPPORTED, "k = %d > AIDW_KMAX", k);
    if (h->nd < k) return fail(h, AIDW_E_INSUFFICIENT_DATA, "shard nd = %lld < k = %d", (long long)h->nd, k);
    if (nq == 0) return AIDW_OK;
    if (!qx || !qy || !s_out) return fail(h, AIDW_E_INVALID_ARG, "NULL argument");
    CK(h, cudaSetDevice(h->device));
    return launched(h,
                    aidw::launch_knn((int)h->dt, k, h->data, h->ndp, qx, qy, nq, nullptr, nullptr, nullptr, s_out,
                                     h->sc, &h->filt, static_cast<cudaStream_t>(stream), 1, split_for(h, nq)),
                    "knn partial kernel");
}

aidw_status aidw_knn_merge(aidw_t h, const void *lists, int P, int64_t nq, int k, void *r_obs, void *d1sq,
                           void *robs_minmax, void *stream)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (P < 1 || nq < 0 || k < 1 || k > AIDW_KMAX) return fail(h, AIDW_E_INVALID_ARG, "bad P/nq/k");
    CK(h, cudaSetDevice(h->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (nq == 0) {
        if (robs_minmax) return launched(h, aidw::launch_minmax_identity((int)h->dt, robs_minmax, st), "minmax");
        return AIDW_OK;
    }
    if (!lists) return fail(h, AIDW_E_INVALID_ARG, "lists is NULL");
    return launched(h, aidw::launch_knn_merge((int)h->dt, k, lists, P, nq, r_obs, d1sq, robs_minmax, h->sc, st),
                    "knn merge kernel");
}

aidw_status aidw_interpolate_partial(aidw_t h, const void *qx, const void *qy, int64_t nq, const void *alpha,
                                     const void *d1sq, double *partial_out, void *stream)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (nq < 0) return fail(h, AIDW_E_INVALID_ARG, "nq < 0");
    if (nq == 0) return AIDW_OK;
    if (!qx || !qy || !alpha || !d1sq || !partial_out) return fail(h, AIDW_E_INVALID_ARG, "NULL argument");
    CK(h, cudaSetDevice(h->device));
    aidw::SplitBuf *sp = split_for(h, nq);
    return launched(h,
                    aidw::launch_interp((int)h->dt, h->data, h->ndp, h->nd, qx, qy, nq, alpha, 0.0, d1sq, nullptr,
                                        static_cast<cudaStream_t>(stream), partial_out, perm_for(h, nq),
                                        h->sc->cls, sp, h->bbox),
                    "interpolate partial kernel");
}

aidw_status aidw_finalize(aidw_t h, const double *partials, int P, int64_t nq, void *z_out, void *stream)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (P < 1 || nq < 0) return fail(h, AIDW_E_INVALID_ARG, "bad P/nq");
    if (nq == 0) return AIDW_OK;
    if (!partials || !z_out) return fail(h, AIDW_E_INVALID_ARG, "NULL argument");
    CK(h, cudaSetDevice(h->device));
    return launched(h, aidw::launch_finalize((int)h->dt, partials, P, nq, z_out, static_cast<cudaStream_t>(stream)),
                    "finalize kernel");
}

aidw_status aidw_check(aidw_t h, void *stream)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    CK(h, cudaSetDevice(h->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CK(h, cudaStreamSynchronize(st));
    CK(h, cudaGetLastError());
    long long idx = 0;
    CK(h, cudaMemcpy(&idx, &h->sc->err_idx, sizeof idx, cudaMemcpyDeviceToHost));
    if (idx != LLONG_MAX) {
        const long long none = LLONG_MAX;
        CK(h, cudaMemcpy(&h->sc->err_idx, &none, sizeof none, cudaMemcpyHostToDevice));
        return fail(h, AIDW_E_NONFINITE_INPUT, "non-finite query coordinate at query index %lld", idx);
    }
    if (h->ex_connected) {
        unsigned to = 0;
        CK(h, cudaMemcpy(&to, &h->sc->ex_timeout, sizeof to, cudaMemcpyDeviceToHost));
        if (to) {
            const unsigned zero = 0;
            CK(h, cudaMemcpy(&h->sc->ex_timeout, &zero, sizeof zero, cudaMemcpyHostToDevice));
            return fail(h, AIDW_E_CUDA, "bounds exchange: a peer's {-min, max} did not arrive within ~2 s "
                                        "(ranks out of step?); alpha and Z of that step are NaN");
        }
    }
    return AIDW_OK;
}

aidw_status aidw_run_host(aidw_t h, const void *qx_host, const void *qy_host, int64_t nq, int k,
                          const double *alpha_lv, aidw_rbounds rb, double r_min, double r_max, aidw_muform mf,
                          void *z_host, void *stream)
{
    if (!h) return fail(nullptr, AIDW_E_INVALID_ARG, "handle is NULL");
    if (nq < 0) return fail(h, AIDW_E_INVALID_ARG, "nq < 0");
    if (nq == 0) return AIDW_OK;
    if (!qx_host || !qy_host || !z_host) return fail(h, AIDW_E_INVALID_ARG, "NULL host buffer");
    if (h->ex_connected) return fail(h, AIDW_E_INVALID_ARG, "aidw_run_host is single-rank; close the exchange first");
    aidw_status s = check_levels(h, alpha_lv);
    if (s != AIDW_OK) return s;
    if (rb == AIDW_RB_FIXED && !(r_min < r_max))
        return fail(h, AIDW_E_INVALID_BOUNDS, "r_min = %g >= r_max = %g", r_min, r_max);
    if (k < 1 || k > AIDW_KMAX) return fail(h, k < 1 ? AIDW_E_INVALID_ARG : AIDW_E_UNSUPPORTED, "k = %d", k);
    if (h->nd < k) return fail(h, AIDW_E_INSUFFICIENT_DATA, "nd = %lld < k = %d", (long long)h->nd, k);
    CK(h, cudaSetDevice(h->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t ts = tsize(h->dt);
    const size_t nb = ((size_t)nq * ts + 255) / 256 * 256;
    s = ensure_work(h, 6 * nb + 256);
    if (s != AIDW_OK) return s;
    char *w = static_cast<char *>(h->work);
    void *qx = w, *qy = w + nb, *robs = w + 2 * nb, *d1 = w + 3 * nb, *al = w + 4 * nb, *z = w + 5 * nb;
    void *mm = w + 6 * nb;
    CK(h, cudaMemcpyAsync(qx, qx_host, (size_t)nq * ts, cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(qy, qy_host, (size_t)nq * ts, cudaMemcpyHostToDevice, st));
    if ((s = aidw_knn_robs(h, qx, qy, nq, k, robs, d1, mm, nullptr, stream)) != AIDW_OK) return s;
    if ((s = aidw_alpha(h, robs, nq, alpha_lv, rb, r_min, r_max, mm, mf, al, stream)) != AIDW_OK) return s;
    if ((s = aidw_interpolate(h, qx, qy, nq, al, d1, z, stream)) != AIDW_OK) return s;
    CK(h, cudaMemcpyAsync(z_host, z, (size_t)nq * ts, cudaMemcpyDeviceToHost, st));
    return aidw_check(h, stream);
}

aidw_status aidw_destroy(aidw_t h)
{
    if (!h) return AIDW_OK;
    cudaSetDevice(h->device);
    if (h->ex_own || h->ex_connected) aidw_exchange_close(h);
    if (h->data || h->sc || h->work || h->filt.arrays || h->perm || h->split.p) cudaDeviceSynchronize();
    if (h->data) aidw::dev_free(h->data);
    if (h->sc) aidw::dev_free(h->sc);
    if (h->work) aidw::dev_free(h->work);
    if (h->filt.arrays) aidw::dev_free(h->filt.arrays);
    if (h->filt.cell_start) aidw::dev_free(h->filt.cell_start);
    if (h->filt.coords64) aidw::dev_free(h->filt.coords64);
    if (h->filt.qorder.p) aidw::dev_free(h->filt.qorder.p);
    if (h->perm) aidw::dev_free(h->perm);
    if (h->split.p) aidw::dev_free(h->split.p);
    delete h;
    return AIDW_OK;
}

}  // extern "C"

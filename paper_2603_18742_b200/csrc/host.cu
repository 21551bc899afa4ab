// host.cu — host-side parts of libdmpq: error state, device queries, sizing, and
// the host-pure decision functions (Eq. 6, Eq. 7, Eq. 10, Eq. 11).
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>


#include "common.cuh"
#include "tmap.cuh"

namespace dmpq {

static thread_local char g_err[512] = "";

dmpq_status set_error(dmpq_status st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return st;
}

dmpq_status check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(DMPQ_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return DMPQ_OK;
}

static std::mutex g_dev_mu;
static int g_sms[64] = {0};
static int g_cc[64] = {0};

static void query_device(int dev) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (dev < 0 || dev >= 64 || g_sms[dev]) return;
    int sms = 0, major = 0, minor = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    g_cc[dev] = major * 10 + minor;
    g_sms[dev] = sms > 0 ? sms : 148;
}

int num_sms() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    query_device(dev);
    return (dev >= 0 && dev < 64) ? g_sms[dev] : 148;
}

bool device_is_sm100() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return false; }
    query_device(dev);
    return dev >= 0 && dev < 64 && g_cc[dev] == 100;
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

}  // namespace dmpq

using namespace dmpq;

extern "C" const char* dmpq_last_error(void) { return g_err; }
extern "C" const char* dmpq_version(void) { return "libdmpq 0.1 (sm_100a)"; }

extern "C" size_t dmpq_sf_bytes(int rows, int k) {
    if (rows <= 0 || k <= 0) return 0;
    size_t kc = (size_t)(((k / 16) + 3) / 4 * 4);
    size_t rp = (size_t)((rows + 127) / 128 * 128);
    return rp * kc;
}

extern "C" double dmpq_derive_tau(double alpha, double beta, double tau_rel, double eps_slope) {
    if (!(alpha > eps_slope)) return -INFINITY;
    return (tau_rel - beta) / alpha;
}

extern "C" dmpq_status dmpq_predict(const dmpq_block_stats* st, const double* tau_gamma, int n_layers, int t,
                                    int prev_skipped, dmpq_gamma_metric metric, uint8_t* fmt_out, double* gamma_out) {
    DMPQ_REQUIRE(tau_gamma && fmt_out && n_layers >= 0, DMPQ_EINVAL, "dmpq_predict: bad arguments");
    DMPQ_REQUIRE(metric == DMPQ_GAMMA_L1 || metric == DMPQ_GAMMA_L2, DMPQ_EINVAL, "dmpq_predict: unknown metric");
    double gamma = NAN;
    bool need = !(t == 0 || prev_skipped);
    dmpq_status rc = DMPQ_OK;
    if (need) {
        DMPQ_REQUIRE(st != nullptr, DMPQ_EINVAL, "dmpq_predict: stats required for t > 0 after a compute");
        double num = metric == DMPQ_GAMMA_L1 ? st->sum_abs_d : std::sqrt(st->sum_d2);
        double den = metric == DMPQ_GAMMA_L1 ? st->sum_abs_x : std::sqrt(st->sum_x2);
        if (den == 0.0) rc = set_error(DMPQ_EZERONORM, "dmpq_predict: ||X|| == 0, Eq. 3 undefined; routed INT8");
        else gamma = num / den;
    }
    for (int j = 0; j < n_layers; ++j) {
        bool int8 = !need || std::isnan(gamma) || gamma > tau_gamma[j];
        fmt_out[j] = int8 ? (uint8_t)DMPQ_FMT_INT8 : (uint8_t)DMPQ_FMT_NVFP4;
    }
    if (gamma_out) *gamma_out = gamma;
    return rc;
}

extern "C" void dmpq_purify(const double* ratio, int n_layers, int prev_skipped, double tau_outlier, uint8_t* fmt_inout) {
    for (int j = 0; j < n_layers; ++j) {
        if (ratio && ratio[j] > tau_outlier) fmt_inout[j] = (uint8_t)DMPQ_FMT_BF16;
        else if (prev_skipped) fmt_inout[j] = (uint8_t)DMPQ_FMT_INT8;
    }
}

extern "C" double dmpq_outlier_ratio(double max_abs, double sum_abs, double count) {
    return sum_abs > 0.0 ? max_abs / (sum_abs / count) : 1.0;
}

extern "C" void tdc_init(tdc_state* st) {
    st->t_p = -1;
    st->e_tp = INFINITY;
    st->e_acc = INFINITY;
    st->last = -1;
    st->n_computed = 0;
}

extern "C" tdc_decision tdc_decide(const tdc_state* st, const tdc_config* cfg, int t) {
    if (st->n_computed < 2) return TDC_COMPUTE;
    if (st->e_acc <= cfg->tau && (t - st->t_p) <= cfg->n_max) return TDC_DECIDE_SKIP;
    return TDC_COMPUTE;
}

extern "C" void tdc_update(tdc_state* st, const tdc_config* cfg, int t, tdc_decision d, const dmpq_block_stats* g) {
    if (d == TDC_COMPUTE) {
        double e = INFINITY;
        if (cfg->metric == TDC_METRIC_REL_L2) {   // ||Delta_t - Delta_prev|| / ||Delta_prev|| (R19)
            if (st->n_computed > 0 && g != nullptr && g->sum_dp2 != 0.0)
                e = std::sqrt(std::fmax(g->sum_dn2 - 2.0 * g->dot_dd + g->sum_dp2, 0.0)) / std::sqrt(g->sum_dp2);
        } else if (st->n_computed > 0 && g != nullptr && g->sum_dn2 != 0.0 && g->sum_dp2 != 0.0) {
            e = 1.0 - g->dot_dd / std::sqrt(g->sum_dn2 * g->sum_dp2);
        }
        st->e_tp = e;
        st->e_acc = e;
        st->t_p = t;
        st->n_computed += 1;
    } else {
        st->e_acc = (st->e_acc + st->e_tp) + cfg->rho;
    }
    st->last = (int)d;
}

// api.cu -- the C ABI of libvapr (include/vapr.h): argument validation,
// context state (robot / worlds / formats), and stage composition.  Every
// entry point validates synchronously, enqueues on the caller's stream and
// returns; no allocation or synchronisation on the hot path.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

using namespace vapr;

struct vapr_ctx {
    int device = 0;
    int sms = 148;
    bool robot_set = false, worlds_set = false, formats_set = false;
    RobotDev robot{};
    vapr_format fmts[VAPR_NUM_SLOTS]{};
    Fmt dfmt[VAPR_NUM_SLOTS]{};
    float4* d_cub = nullptr;
    int32_t* d_off = nullptr;
    int32_t n_worlds = 0;
    int cull = 1;
    // vapr_cost_grad_host: copy streams and an event pool (created lazily)
    cudaStream_t s_in = nullptr, s_out = nullptr;
    // small batches: the per-trajectory cost reduction on a side stream,
    // beside aggregation and BK (fork / join events)
    cudaStream_t s_red = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::vector<cudaEvent_t> events;
    // collision tile-scheduler slots (device, kSchedSlots x {next, done}) and
    // the host-side slot cursor
    unsigned int* d_sched = nullptr;
    unsigned int sched_next = 0;
    // VAPR_OPT_STREAMS: concurrent trajectory chunks in vapr_cost_grad
    int n_streams = 1;
    cudaStream_t par[8] = {};
    // N3: grad_out_spheres in the sparse form (VAPR_OPT_SPARSE)
    int sparse = 0;
    // N4: the fused on-chip rollout (VAPR_OPT_FUSED)
    int fused = 0;
    // the collision kernel's robot tables as a device image (vapr_set_robot)
    void* d_tab_img = nullptr;
    int32_t tab_img_bytes = 0;
    // stage timing hook (vapr_set_stage_events): caller-owned events recorded
    // between the launches of vapr_cost_grad
    cudaEvent_t stage_ev[6] = {};
    int n_stage_ev = 0;
    // IKO goals (N2)
    float* d_goals = nullptr;
    int32_t n_goals = 0;
    bool goals_set = false;
};

#ifndef VAPR_AGG_IN_BK             // small sparse batches: aggregation inside BK's CTAs
#define VAPR_AGG_IN_BK 1
#endif
#ifndef VAPR_AGG_ROWS_BELOW_BK
#define VAPR_AGG_ROWS_BELOW_BK 16384
#endif
#ifndef VAPR_SIDE_REDUCE           // small batches: cost reduction on a side stream
#define VAPR_SIDE_REDUCE 1
#endif
#ifndef VAPR_SIDE_REDUCE_BELOW
#define VAPR_SIDE_REDUCE_BELOW 65536
#endif
#ifndef VAPR_CHAIN_PDL             // vapr_cost_grad: reduce / aggregate / BK as programmatic dependents
#define VAPR_CHAIN_PDL 0           // measured slower (bench step 4.39 -> 4.38 ms, config 1 / 2 71 / 68 ->
#endif                             // 80 / 76 us; early triggers: per-env leg 5.7 -> 6.9 ms); FK -> self stays
#ifndef VAPR_END_CHUNK_WEIGHT      // vapr_cost_grad_host: first / last chunk size relative to the others
#define VAPR_END_CHUNK_WEIGHT 0.25
#endif

#ifdef VAPR_DEBUG_TAP
namespace vapr {
float* g_tap_host[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
}
#endif

namespace {

// Make the context's device current for the duration of a call.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) { ok = false; return; }
        if (prev != dev && cudaSetDevice(dev) != cudaSuccess) ok = false;
    }
    ~DeviceGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// vapr_cost_grad_sparse_layout entries (N3)
constexpr int kSparseOffs = 8;

// sparse form of a tensor (N3): pool capacity in words (every row full)
size_t sparse_pool_words_of(const Fmt& f, int cols, long long rows) {
    return (size_t)rows * (size_t)((cols + f.pf - 1) / f.pf);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool fmt_valid(vapr_format f) {
    const int m = f.man_bits & ~VAPR_FMT_IEEE;
    if (f.man_bits & VAPR_FMT_IEEE)             // IEEE mode: E5M10 and E8M7 only
        return (f.exp_bits == 5 && m == 10) || (f.exp_bits == 8 && m == 7);
    return f.exp_bits >= 2 && f.exp_bits <= 8 && m >= 1 && m <= 23 && 1 + f.exp_bits + m <= 32;
}

// Host-side derivation of the device codec constants (common.cuh, Fmt).
Fmt make_fmt(vapr_format v) {
    Fmt f{};
    const bool ieee = (v.man_bits & VAPR_FMT_IEEE) != 0;
    v.man_bits &= ~VAPR_FMT_IEEE;
    f.E = v.exp_bits;
    f.M = v.man_bits;
    f.t = 1 + f.E + f.M;
    f.pf = 32 / f.t;
    const int bias = (1 << (f.E - 1)) - 1;
    f.sh = 23 - f.M;
    const uint32_t rnd = f.sh > 0 ? (1u << (f.sh - 1)) - 1u : 0u;
    const uint32_t off = (uint32_t)(127 - bias) << f.M;
    f.K = rnd - (off << f.sh);                                  // mod 2^32
    f.lsb = f.sh > 0 ? 1u : 0u;                               // E<8, M=23: no rounding
    f.minnorm = (uint32_t)(128 - bias) << 23;                 // 2^(1-bias)
    f.magic_bits = (uint32_t)(127 + 24 - bias - f.M) << 23;    // 2^(24-bias-M)
    const uint32_t emax = (f.E == 8) ? 254u : (1u << f.E) - 1u;
    f.maxcode = (emax << f.M) | ((1u << f.M) - 1u);
    f.mask = (f.t >= 32) ? 0xffffffffu : ((1u << f.t) - 1u);
    f.signbit = (f.t >= 32) ? 0x80000000u : (1u << (f.t - 1));
    f.keep = 0x80000000u | ((((1u << (f.E + f.M)) - 1u)) << (23 - f.M));
    uint32_t sc = (uint32_t)(254 - bias) << 23;                // 2^(127-bias)
    std::memcpy(&f.dscale, &sc, 4);
    // hardware conversion fast paths and the |x| range where they match the
    // reading bit for bit (verified exhaustively by tests/test_gpu_parity.py)
    f.kind = KIND_GENERIC;
    f.hw_limit = 0u;
    if (f.E == 8 && f.M == 23) f.kind = KIND_IDENTITY;
    else if (f.E == 5 && f.M == 10) { f.kind = KIND_F16; f.hw_limit = 0x477FF000u; }   // 65520
    else if (f.E == 8 && f.M == 7) { f.kind = KIND_BF16; f.hw_limit = 0x7F7F8000u; }   // bf16max+ulp/2
    else if (f.E == 4 && f.M == 3) { f.kind = KIND_E4M3; f.hw_limit = 0x43E80001u; }   // <= 464
    else if (f.E == 5 && f.M == 2) { f.kind = KIND_E5M2; f.hw_limit = 0x47700000u; }   // 61440
    else if (f.E == 2 && f.M == 1) { f.kind = KIND_E2M1; f.hw_limit = 0x7F800001u; }   // all but NaN
    else if (f.E == 2 && f.M == 3) { f.kind = KIND_E2M3; f.hw_limit = 0x7F800001u; }
    else if (f.E == 3 && f.M == 2) { f.kind = KIND_E3M2; f.hw_limit = 0x7F800001u; }
    f.nancode = f.maxcode;
    if (ieee) {                     // reading c41 (common.cuh, KIND_F16_IEEE)
        f.kind = (f.E == 5) ? KIND_F16_IEEE : KIND_GENERIC;
        f.hw_limit = 0u;
        f.maxcode = (f.E == 5) ? 0x7C00u : 0x7F80u;   // the encode clamp: overflow -> inf
        f.nancode = 0x7FFFu;                          // the hardware conversions' canonical NaN
    }
    // fake_quant constants (N4): the values decode() gives for the largest
    // finite code and for nancode, by the same bit recipe as decode_slot
    f.fq_rnd = rnd;
    f.fq_keep = ~((f.sh > 0 ? (1u << f.sh) : 1u) - 1u);
    auto dec_bits = [&](uint32_t code) {
        if (f.E == 8 && f.M == 23) return code;
        const uint32_t u = code << (32 - f.t);
        const uint32_t x = uint32_t(int32_t(u) >> (8 - f.E)) & f.keep;
        if (f.E == 8) return x;
        float fx, r;
        std::memcpy(&fx, &x, 4);
        r = fx * f.dscale;
        uint32_t b;
        std::memcpy(&b, &r, 4);
        return b;
    };
    const uint32_t maxfin_code = ieee ? f.maxcode - 1u : f.maxcode;
    f.fq_maxfin = dec_bits(maxfin_code);
    f.fq_sat = ieee ? 0x7F800000u : f.fq_maxfin;
    f.fq_nan = (ieee && f.E == 5) ? (0x7F800000u | (0x3FFu << 13)) : dec_bits(f.nancode);
    return f;
}

thread_local cudaError_t t_last_cuda_error = cudaSuccess;

vapr_status cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return VAPR_OK;
    t_last_cuda_error = e;
    return VAPR_ERR_CUDA;
}

vapr_status pending_fault() {
    // surface an earlier asynchronous fault without clearing sticky errors
    const cudaError_t e = cudaPeekAtLastError();
    return cuda_status(e);
}

#define CHECK(cond, st) \
    do {                \
        if (!(cond)) return (st); \
    } while (0)

size_t packed_bytes(const Fmt& f, int cols, long long rows) {
    return (size_t)row_words_of(f, cols) * 4u * (size_t)rows;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

WorldsDev worlds_of(const vapr_ctx* c) { return WorldsDev{c->d_cub, c->d_off, c->n_worlds}; }

}  // namespace

extern "C" {

const char* vapr_version(void) { return "libvapr 0.1 (sm_100a)"; }

const char* vapr_last_cuda_error(void) { return cudaGetErrorString(t_last_cuda_error); }

const char* vapr_status_string(vapr_status s) {
    switch (s) {
        case VAPR_OK: return "ok";
        case VAPR_ERR_INVALID_FORMAT: return "invalid format";
        case VAPR_ERR_INVALID_ARG: return "invalid argument";
        case VAPR_ERR_SHAPE: return "invalid shape";
        case VAPR_ERR_CUDA: return "cuda error";
        case VAPR_ERR_NOT_INITIALIZED: return "context not initialised";
        case VAPR_ERR_UNSUPPORTED: return "unsupported";
    }
    return "unknown status";
}

vapr_status vapr_create(int device, vapr_ctx** out) {
    CHECK(out != nullptr, VAPR_ERR_INVALID_ARG);
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        cudaGetLastError();
        return VAPR_ERR_CUDA;
    }
    vapr_ctx* c = new (std::nothrow) vapr_ctx();
    CHECK(c != nullptr, VAPR_ERR_INVALID_ARG);
    c->device = device;
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    {
        DeviceGuard g(device);
        if (!g.ok || cudaMalloc(&c->d_sched, sizeof(unsigned int) * 2 * kSchedSlots) != cudaSuccess ||
            cudaMemset(c->d_sched, 0, sizeof(unsigned int) * 2 * kSchedSlots) != cudaSuccess) {
            if (c->d_sched) cudaFree(c->d_sched);
            delete c;
            cudaGetLastError();
            return VAPR_ERR_CUDA;
        }
    }
    for (int i = 0; i < VAPR_NUM_SLOTS; ++i) {
        c->fmts[i] = vapr_format{8, 23};
        c->dfmt[i] = make_fmt(c->fmts[i]);
    }
    *out = c;
    return VAPR_OK;
}

vapr_status vapr_destroy(vapr_ctx* c) {
    if (!c) return VAPR_OK;
    DeviceGuard g(c->device);
    if (c->d_cub) cudaFree(c->d_cub);
    if (c->d_off) cudaFree(c->d_off);
    if (c->d_sched) cudaFree(c->d_sched);
    if (c->d_goals) cudaFree(c->d_goals);
    if (c->d_tab_img) cudaFree(c->d_tab_img);
    for (cudaStream_t st : c->par)
        if (st) cudaStreamDestroy(st);
    if (c->s_in) cudaStreamDestroy(c->s_in);
    if (c->s_red) cudaStreamDestroy(c->s_red);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->s_out) cudaStreamDestroy(c->s_out);
    for (cudaEvent_t e : c->events) cudaEventDestroy(e);
    delete c;
    return VAPR_OK;
}

vapr_status vapr_set_goals(vapr_ctx* c, const float* goals, int32_t n_goals) {
    CHECK(c != nullptr && n_goals >= 0, VAPR_ERR_INVALID_ARG);
    CHECK(n_goals == 0 || goals != nullptr, VAPR_ERR_INVALID_ARG);
    DeviceGuard g(c->device);
    CHECK(g.ok, VAPR_ERR_CUDA);
    if (c->d_goals) cudaFree(c->d_goals);
    c->d_goals = nullptr;
    c->n_goals = 0;
    if (n_goals > 0) {
        const size_t bytes = sizeof(float) * 12 * (size_t)n_goals;
        if (cuda_status(cudaMalloc(&c->d_goals, bytes)) != VAPR_OK) return VAPR_ERR_CUDA;
        if (cuda_status(cudaMemcpy(c->d_goals, goals, bytes, cudaMemcpyHostToDevice)) != VAPR_OK)
            return VAPR_ERR_CUDA;
    }
    c->n_goals = n_goals;
    c->goals_set = true;
    return VAPR_OK;
}

vapr_status vapr_format_check(vapr_format f) {
    return fmt_valid(f) ? VAPR_OK : VAPR_ERR_INVALID_FORMAT;
}

vapr_status vapr_format_parse(const char* s, vapr_format* out) {
    CHECK(s != nullptr && out != nullptr, VAPR_ERR_INVALID_ARG);
    int e = -1, m = -1;
    char c0 = 0, c1 = 0;
    int nread = 0;
    if (std::sscanf(s, " %c%d%c%d %n", &c0, &e, &c1, &m, &nread) != 4 || s[nread] != '\0')
        return VAPR_ERR_INVALID_FORMAT;
    if ((c0 != 'E' && c0 != 'e') || (c1 != 'M' && c1 != 'm')) return VAPR_ERR_INVALID_FORMAT;
    vapr_format f{e, m};
    CHECK(fmt_valid(f), VAPR_ERR_INVALID_FORMAT);
    *out = f;
    return VAPR_OK;
}

size_t vapr_packed_row_words(vapr_format f, size_t cols) {
    if (!fmt_valid(f)) return 0;
    const size_t pf = 32 / (1 + f.exp_bits + (f.man_bits & ~VAPR_FMT_IEEE));
    const size_t w = (cols + pf - 1) / pf;
    return (w + 3) & ~(size_t)3;
}

vapr_status vapr_set_formats(vapr_ctx* c, const vapr_format* fmts) {
    CHECK(c != nullptr && fmts != nullptr, VAPR_ERR_INVALID_ARG);
    for (int i = 0; i < VAPR_NUM_SLOTS; ++i) CHECK(fmt_valid(fmts[i]), VAPR_ERR_INVALID_FORMAT);
    for (int i = 0; i < VAPR_NUM_SLOTS; ++i) {
        c->fmts[i] = fmts[i];
        c->dfmt[i] = make_fmt(fmts[i]);
    }
    c->formats_set = true;
    return VAPR_OK;
}

vapr_status vapr_set_robot(vapr_ctx* c, const vapr_robot* r) {
    CHECK(c != nullptr && r != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(r->n_spheres >= 1 && r->n_spheres <= VAPR_MAX_SPHERES, VAPR_ERR_SHAPE);
    CHECK(r->n_pairs >= 0 && r->n_pairs <= VAPR_MAX_PAIRS, VAPR_ERR_SHAPE);
    CHECK(r->sphere_link != nullptr && r->sphere_xyzr != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(r->n_pairs == 0 || r->pairs != nullptr, VAPR_ERR_INVALID_ARG);
    RobotDev R{};
    R.n_spheres = r->n_spheres;
    R.cols = 3 * r->n_spheres;
    for (int i = 0; i < 8; ++i) {
        R.ca[i] = (float)std::cos(r->dh_alpha[i]);
        R.sa[i] = (float)std::sin(r->dh_alpha[i]);
        R.a[i] = (float)r->dh_a[i];
        R.d[i] = (float)r->dh_d[i];
    }
    R.hand_c = (float)std::cos(r->hand_rz);
    R.hand_s = (float)std::sin(r->hand_rz);
    for (int j = 0; j < kJoints; ++j) {
        R.q_lo[j] = (float)r->q_lo[j];
        R.q_hi[j] = (float)r->q_hi[j];
    }
    int prev = 0;
    int count[kLinks] = {0};
    for (int s = 0; s < r->n_spheres; ++s) {
        const int l = r->sphere_link[s];
        CHECK(l >= 0 && l < kLinks, VAPR_ERR_INVALID_ARG);
        CHECK(l >= prev, VAPR_ERR_UNSUPPORTED);            // spheres must be sorted by link
        prev = l;
        count[l]++;
        R.sx[s] = r->sphere_xyzr[4 * s + 0];
        R.sy[s] = r->sphere_xyzr[4 * s + 1];
        R.sz[s] = r->sphere_xyzr[4 * s + 2];
        R.sr[s] = r->sphere_xyzr[4 * s + 3];
    }
    R.link_start[0] = 0;
    for (int l = 0; l < kLinks; ++l) R.link_start[l + 1] = R.link_start[l] + count[l];
    // canonical pair list sorted by (i, j), i < j, duplicates removed
    std::vector<std::pair<int, int>> plist;
    for (int k = 0; k < r->n_pairs; ++k) {
        const int i = r->pairs[2 * k], j = r->pairs[2 * k + 1];
        CHECK(i < r->n_spheres && j < r->n_spheres && i != j, VAPR_ERR_INVALID_ARG);
        plist.emplace_back(std::min(i, j), std::max(i, j));
    }
    std::sort(plist.begin(), plist.end());
    plist.erase(std::unique(plist.begin(), plist.end()), plist.end());
    R.n_pairs = (int32_t)plist.size();
    std::vector<std::vector<std::pair<int, int>>> adj(r->n_spheres);   // (partner, pid)
    for (int k = 0; k < (int)plist.size(); ++k) {
        R.pair_i[k] = (uint8_t)plist[k].first;
        R.pair_j[k] = (uint8_t)plist[k].second;
        adj[plist[k].first].emplace_back(plist[k].second, k);
        adj[plist[k].second].emplace_back(plist[k].first, k);
    }
    for (int a = 0; a < kLinks; ++a)
        for (int b = 0; b < kLinks; ++b) R.lp_index[a][b] = -1;
    int nlp = 0;
    int o = 0;
    for (int s = 0; s < r->n_spheres; ++s) {
        R.adj_off[s] = (uint16_t)o;
        std::vector<std::pair<int, int>>& a = adj[s];
        std::sort(a.begin(), a.end());
        const int ls = r->sphere_link[s];
        int L = 0;
        for (const auto& pv : a) {
            const int v = pv.first;
            const int lv = r->sphere_link[v];
            while (L <= lv) R.adj_link_off[s][L++] = (uint16_t)o;
            if (R.lp_index[ls][lv] < 0) {
                CHECK(nlp < 32, VAPR_ERR_UNSUPPORTED);
                R.lp_a[nlp] = (int8_t)std::min(ls, lv);
                R.lp_b[nlp] = (int8_t)std::max(ls, lv);
                R.lp_index[ls][lv] = R.lp_index[lv][ls] = (int8_t)nlp++;
            }
            R.adj_pid[o] = (uint16_t)pv.second;
            R.adj[o++] = (uint8_t)v;
        }
        while (L <= kLinks) R.adj_link_off[s][L++] = (uint16_t)o;
    }
    R.adj_off[r->n_spheres] = (uint16_t)o;
    R.n_link_pairs = nlp;
    // sub-link groups: the spheres of each link split into two contiguous halves
    auto one_center = [&](int b0, int b1, int& ref, float& rl) {
        ref = b0;
        rl = -1.f;
        double best = 1e300;
        for (int a = b0; a < b1; ++a) {
            double m = 0.0;
            for (int b = b0; b < b1; ++b) {
                const double dx = (double)R.sx[b] - R.sx[a], dy = (double)R.sy[b] - R.sy[a],
                             dz = (double)R.sz[b] - R.sz[a];
                m = std::max(m, std::sqrt(dx * dx + dy * dy + dz * dz) + (double)R.sr[b]);
            }
            if (m < best) {
                best = m;
                ref = a;
            }
        }
        if (best < 1e300) rl = std::nextafter((float)best, 3e38f);
    };
    std::vector<int> grp_of(r->n_spheres, 0);
    int ng = 0;
    std::vector<int> grp_link;
    for (int l = 0; l < kLinks; ++l) {
        const int b0 = R.link_start[l], b1 = R.link_start[l + 1];
        if (b1 == b0) continue;
        const int mid = b0 + (b1 - b0 + 1) / 2;
        const int cuts[3] = {b0, mid, b1};
        for (int h = 0; h < 2; ++h) {
            if (cuts[h + 1] == cuts[h]) continue;
            one_center(cuts[h], cuts[h + 1], R.grp_ref[ng], R.grp_rl[ng]);
            for (int s2 = cuts[h]; s2 < cuts[h + 1]; ++s2) grp_of[s2] = ng;
            grp_link.push_back(l);
            ++ng;
        }
    }
    R.n_groups = ng;
    {
        // group pairs, ordered by link pair then (ga, gb); pair ids of each
        int ngp = 0, npid = 0;
        for (int lp = 0; lp < nlp; ++lp) {
            R.lp_gp_off[lp] = (uint8_t)ngp;
            for (int ga = 0; ga < ng; ++ga)
                for (int gb = ga; gb < ng; ++gb) {
                    const int la = grp_link[ga], lb = grp_link[gb];
                    if (!((la == R.lp_a[lp] && lb == R.lp_b[lp]) ||
                          (la == R.lp_b[lp] && lb == R.lp_a[lp])))
                        continue;
                    const int start = npid;
                    for (int k = 0; k < (int)plist.size(); ++k) {
                        const int gi = grp_of[plist[k].first], gj = grp_of[plist[k].second];
                        if ((gi == ga && gj == gb) || (gi == gb && gj == ga)) R.gp_pid[npid++] = (uint16_t)k;
                    }
                    if (npid == start) continue;
                    CHECK(ngp < kMaxGroupPairs, VAPR_ERR_UNSUPPORTED);
                    R.gp_a[ngp] = (uint8_t)ga;
                    R.gp_b[ngp] = (uint8_t)gb;
                    R.gp_off[ngp] = (uint16_t)start;
                    ++ngp;
                }
        }
        R.lp_gp_off[nlp] = (uint8_t)ngp;
        R.gp_off[ngp] = (uint16_t)npid;
    }
    // per-link reference sphere: the sphere minimising max_s(|o_s - o_ref| + r_s)
    for (int l = 0; l < kLinks; ++l) {
        R.link_ref[l] = R.link_start[l];
        R.link_rl[l] = -1.f;
        double best = 1e300;
        for (int a = R.link_start[l]; a < R.link_start[l + 1]; ++a) {
            double m = 0.0;
            for (int b = R.link_start[l]; b < R.link_start[l + 1]; ++b) {
                const double dx = (double)R.sx[b] - R.sx[a], dy = (double)R.sy[b] - R.sy[a],
                             dz = (double)R.sz[b] - R.sz[a];
                m = std::max(m, std::sqrt(dx * dx + dy * dy + dz * dz) + (double)R.sr[b]);
            }
            if (m < best) {
                best = m;
                R.link_ref[l] = a;
            }
        }
        // round up so the FP32 radius never under-states the double bound
        if (best < 1e300) R.link_rl[l] = std::nextafter((float)best, 3e38f);
    }
    {   // the collision kernel's shared tables, staged from this image
        DeviceGuard g(c->device);
        CHECK(g.ok, VAPR_ERR_CUDA);
        const std::vector<uint8_t> img = collision_table_image(R);
        if (c->d_tab_img) {                       // kernels in flight may read the old one
            cudaDeviceSynchronize();
            cudaFree(c->d_tab_img);
            c->d_tab_img = nullptr;
        }
        CHECK(cudaMalloc(&c->d_tab_img, img.size()) == cudaSuccess, VAPR_ERR_CUDA);
        CHECK(cudaMemcpy(c->d_tab_img, img.data(), img.size(), cudaMemcpyHostToDevice) == cudaSuccess,
              VAPR_ERR_CUDA);
        c->tab_img_bytes = (int32_t)img.size();
    }
    c->robot = R;
    c->robot_set = true;
    return VAPR_OK;
}

vapr_status vapr_set_worlds(vapr_ctx* c, int32_t n_worlds, const vapr_cuboid* cub,
                            const int32_t* offsets) {
    CHECK(c != nullptr && offsets != nullptr && n_worlds >= 1, VAPR_ERR_INVALID_ARG);
    CHECK(offsets[0] == 0, VAPR_ERR_INVALID_ARG);
    for (int w = 0; w < n_worlds; ++w) {
        const int k = offsets[w + 1] - offsets[w];
        CHECK(k >= 0 && k <= VAPR_MAX_CUBOIDS_PER_WORLD, VAPR_ERR_SHAPE);
    }
    const int n = offsets[n_worlds];
    CHECK(n == 0 || cub != nullptr, VAPR_ERR_INVALID_ARG);
    // device form per cuboid: R^T row-major (9), t (3), half (3), pad
    std::vector<float> h((size_t)std::max(n, 1) * 16, 0.f);
    for (int k = 0; k < n; ++k) {
        float* d = &h[(size_t)k * 16];
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) d[3 * i + j] = cub[k].R[3 * j + i];
        for (int i = 0; i < 3; ++i) d[9 + i] = cub[k].t[i];
        for (int i = 0; i < 3; ++i) {
            CHECK(cub[k].half[i] >= 0.f, VAPR_ERR_INVALID_ARG);
            d[12 + i] = cub[k].half[i];
        }
    }
    DeviceGuard g(c->device);
    CHECK(g.ok, VAPR_ERR_CUDA);
    float4* d_cub = nullptr;
    int32_t* d_off = nullptr;
    if (cudaMalloc(&d_cub, h.size() * sizeof(float)) != cudaSuccess ||
        cudaMalloc(&d_off, sizeof(int32_t) * (n_worlds + 1)) != cudaSuccess) {
        if (d_cub) cudaFree(d_cub);
        cudaGetLastError();
        return VAPR_ERR_CUDA;
    }
    if (cudaMemcpy(d_cub, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice) !=
            cudaSuccess ||
        cudaMemcpy(d_off, offsets, sizeof(int32_t) * (n_worlds + 1), cudaMemcpyHostToDevice) !=
            cudaSuccess) {
        cudaFree(d_cub);
        cudaFree(d_off);
        return VAPR_ERR_CUDA;
    }
    if (c->d_cub) cudaFree(c->d_cub);
    if (c->d_off) cudaFree(c->d_off);
    c->d_cub = d_cub;
    c->d_off = d_off;
    c->n_worlds = n_worlds;
    c->worlds_set = true;
    return VAPR_OK;
}

vapr_status vapr_set_option(vapr_ctx* c, int32_t option, int32_t value) {
    CHECK(c != nullptr, VAPR_ERR_INVALID_ARG);
    if (option == VAPR_OPT_CULL) {
        c->cull = value ? 1 : 0;
        return VAPR_OK;
    }
    if (option == VAPR_OPT_STREAMS) {
        CHECK(value >= 1 && value <= 8, VAPR_ERR_INVALID_ARG);
        c->n_streams = value;
        return VAPR_OK;
    }
    if (option == VAPR_OPT_SPARSE) {
        CHECK(value == 0 || value == 1, VAPR_ERR_INVALID_ARG);
        c->sparse = value;
        return VAPR_OK;
    }
    if (option == VAPR_OPT_FUSED) {
        CHECK(value == 0 || value == 1, VAPR_ERR_INVALID_ARG);
        c->fused = value;
        return VAPR_OK;
    }
    return VAPR_ERR_UNSUPPORTED;
}

vapr_status vapr_set_stage_events(vapr_ctx* c, void* const* events, int32_t n) {
    CHECK(c != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(n == 0 || (n == 6 && events != nullptr), VAPR_ERR_INVALID_ARG);
    for (int i = 0; i < 6; ++i) c->stage_ev[i] = (n == 6) ? static_cast<cudaEvent_t>(events[i]) : nullptr;
    c->n_stage_ev = n;
    return VAPR_OK;
}

// ---- test-only debug tap (tap.cuh) -----------------------
#ifdef VAPR_DEBUG_TAP
vapr_status vapr_debug_tap(vapr_ctx* c, int32_t slot, float* dst) {
    CHECK(c != nullptr && slot >= 0 && slot < VAPR_NUM_SLOTS, VAPR_ERR_INVALID_ARG);
    vapr::g_tap_host[slot] = dst;
    return VAPR_OK;
}
#endif

// ---- N3: sparse form ------------------------------------------------------
size_t vapr_sparse_pool_words(vapr_format f, size_t cols, size_t rows) {
    if (!fmt_valid(f) || cols == 0) return 0;
    return sparse_pool_words_of(make_fmt(f), (int)cols, (long long)rows);
}

vapr_status vapr_sparsify(vapr_format f, const uint32_t* packed, size_t rows, size_t cols,
                          uint64_t* mask, uint32_t* off, uint32_t* pool, size_t pool_words,
                          uint32_t* used, void* stream) {
    CHECK(fmt_valid(f), VAPR_ERR_INVALID_FORMAT);
    CHECK(cols > 0 && cols % 3 == 0 && cols / 3 <= 64, VAPR_ERR_SHAPE);
    CHECK(used != nullptr, VAPR_ERR_INVALID_ARG);
    const Fmt F = make_fmt(f);
    CHECK(pool_words >= sparse_pool_words_of(F, (int)cols, (long long)rows), VAPR_ERR_SHAPE);
    CHECK(sparse_pool_words_of(F, (int)cols, (long long)rows) <= 0xFFFFFFFFull, VAPR_ERR_SHAPE);
    CHECK(rows == 0 || (packed && mask && off && pool), VAPR_ERR_INVALID_ARG);
    CHECK(aligned16(packed) && (reinterpret_cast<uintptr_t>(mask) & 7u) == 0, VAPR_ERR_INVALID_ARG);
    SparseOut o{};
    o.mask = reinterpret_cast<unsigned long long*>(mask);
    o.off = off;
    o.pool = pool;
    o.used = used;
    return cuda_status(launch_sparsify(F, packed, (long long)rows, (int)cols, o,
                                       (cudaStream_t)stream));
}

vapr_status vapr_densify(vapr_format f, const uint64_t* mask, const uint32_t* off,
                         const uint32_t* pool, size_t rows, size_t cols, uint32_t* packed,
                         void* stream) {
    CHECK(fmt_valid(f), VAPR_ERR_INVALID_FORMAT);
    CHECK(cols > 0 && cols % 3 == 0 && cols / 3 <= 64, VAPR_ERR_SHAPE);
    if (rows == 0) return VAPR_OK;
    CHECK(mask && off && pool && packed, VAPR_ERR_INVALID_ARG);
    CHECK((reinterpret_cast<uintptr_t>(mask) & 7u) == 0, VAPR_ERR_INVALID_ARG);
    return cuda_status(launch_densify(make_fmt(f),
                                      SparseIn{reinterpret_cast<const unsigned long long*>(mask),
                                               off, pool},
                                      (long long)rows, (int)cols, packed, (cudaStream_t)stream));
}

// ---- a1 ------------------------------------------------------------------
vapr_status vapr_quantize(vapr_format f, const float* x, size_t rows, size_t cols,
                          uint32_t* packed, void* stream) {
    CHECK(fmt_valid(f), VAPR_ERR_INVALID_FORMAT);
    if (rows == 0 || cols == 0) return VAPR_OK;
    CHECK(x != nullptr && packed != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(aligned16(x) && aligned16(packed), VAPR_ERR_INVALID_ARG);
    CHECK(cols < (1u << 30), VAPR_ERR_SHAPE);
    CHECK(pending_fault() == VAPR_OK, VAPR_ERR_CUDA);
    const Fmt d = make_fmt(f);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return cuda_status(launch_quantize(d, x, rows, cols, vapr_packed_row_words(f, cols), packed,
                                       sms, (cudaStream_t)stream));
}

vapr_status vapr_dequantize(vapr_format f, const uint32_t* packed, size_t rows, size_t cols,
                            float* y, void* stream) {
    CHECK(fmt_valid(f), VAPR_ERR_INVALID_FORMAT);
    if (rows == 0 || cols == 0) return VAPR_OK;
    CHECK(y != nullptr && packed != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(aligned16(y) && aligned16(packed), VAPR_ERR_INVALID_ARG);
    CHECK(cols < (1u << 30), VAPR_ERR_SHAPE);
    CHECK(pending_fault() == VAPR_OK, VAPR_ERR_CUDA);
    const Fmt d = make_fmt(f);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return cuda_status(launch_dequantize(d, packed, rows, cols, vapr_packed_row_words(f, cols),
                                         y, sms, (cudaStream_t)stream));
}

// ---- a2 ------------------------------------------------------------------
vapr_status vapr_fk_spheres(vapr_ctx* c, const float* q, int32_t B, int32_t H,
                            uint32_t* out_spheres, float* ee_pose, void* stream) {
    CHECK(c != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(c->robot_set, VAPR_ERR_NOT_INITIALIZED);
    CHECK(B >= 1 && H >= 1, VAPR_ERR_SHAPE);
    CHECK(q && out_spheres && aligned16(q) && aligned16(out_spheres), VAPR_ERR_INVALID_ARG);
    DeviceGuard g(c->device);
    CHECK(g.ok && pending_fault() == VAPR_OK, VAPR_ERR_CUDA);
    CHECK(ee_pose == nullptr || aligned16(ee_pose), VAPR_ERR_INVALID_ARG);
    return cuda_status(launch_fk(c->robot, c->dfmt[VAPR_OUT_SPHERES], q, (long long)B * H,
                                 out_spheres, (cudaStream_t)stream, nullptr, ee_pose));
}

// ---- a3 / a4 -------------------------------------------------------------
static vapr_status collision_common(vapr_ctx* c, const uint32_t* os, const int32_t* world_idx,
                                    int32_t B, int32_t H, int do_world, int do_self,
                                    int32_t swept, int32_t sweep_steps, float eta_w, float w_w,
                                    float eta_s, float w_s, float* cost, uint32_t* cp,
                                    uint32_t* ov, float* cost_traj, cudaStream_t s) {
    CHECK(c != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(c->robot_set && (!do_world || c->worlds_set), VAPR_ERR_NOT_INITIALIZED);
    CHECK(B >= 1 && H >= 1, VAPR_ERR_SHAPE);
    CHECK(!(do_world && swept) || H >= 2, VAPR_ERR_SHAPE);
    CHECK(os && cost && aligned16(os) && aligned16(cost), VAPR_ERR_INVALID_ARG);
    if (do_world) {
        CHECK(world_idx && cp && aligned16(world_idx) && aligned16(cp), VAPR_ERR_INVALID_ARG);
        CHECK(std::isfinite(eta_w) && eta_w > 0.f && std::isfinite(w_w), VAPR_ERR_INVALID_ARG);
        CHECK(sweep_steps >= 0 && sweep_steps <= 64, VAPR_ERR_INVALID_ARG);
    }
    if (do_self) {
        CHECK(ov && aligned16(ov), VAPR_ERR_INVALID_ARG);
        CHECK(std::isfinite(eta_s) && eta_s > 0.f && std::isfinite(w_s), VAPR_ERR_INVALID_ARG);
    }
    CHECK(cost_traj == nullptr || aligned16(cost_traj), VAPR_ERR_INVALID_ARG);
    DeviceGuard g(c->device);
    CHECK(g.ok && pending_fault() == VAPR_OK, VAPR_ERR_CUDA);
    CollisionArgs a{};
    a.os = os;
    a.world_idx = world_idx;
    a.B = B;
    a.H = H;
    a.do_world = do_world;
    a.do_self = do_self;
    a.swept = swept ? 1 : 0;
    a.sweep_steps = sweep_steps;
    a.eta_w = do_world ? eta_w : 1.f;
    a.w_w = w_w;
    a.eta_s = do_self ? eta_s : 1.f;
    a.w_s = w_s;
    a.cull = c->cull;
    a.tab_img = static_cast<const uint4*>(c->d_tab_img);
    a.tab_img_bytes = c->tab_img_bytes;
    a.cost = cost;
    a.cp = cp;
    a.ov = ov;
    const Fmt& fcp = c->dfmt[swept ? VAPR_CLOSEST_PT_SWEPT : VAPR_CLOSEST_PT];
    cudaError_t e = launch_collision(c->robot, worlds_of(c), c->dfmt[VAPR_OUT_SPHERES], fcp,
                                     c->dfmt[VAPR_OUT_VEC], a, c->d_sched, &c->sched_next, s);
    if (e == cudaSuccess && cost_traj) e = launch_traj_reduce(cost, B, H, cost_traj, s);
    return cuda_status(e);
}

vapr_status vapr_world_collision(vapr_ctx* c, const uint32_t* os, const int32_t* world_idx,
                                 int32_t B, int32_t H, int32_t swept, int32_t sweep_steps,
                                 float eta, float weight, float* cost, uint32_t* grad,
                                 void* stream) {
    return collision_common(c, os, world_idx, B, H, 1, 0, swept, sweep_steps, eta, weight, 1.f,
                            0.f, cost, grad, nullptr, nullptr, (cudaStream_t)stream);
}

vapr_status vapr_self_collision(vapr_ctx* c, const uint32_t* os, int32_t B, int32_t H, float eta,
                                float weight, float* cost, uint32_t* out_vec, void* stream) {
    return collision_common(c, os, nullptr, B, H, 0, 1, 0, 0, 1.f, 0.f, eta, weight, cost,
                            nullptr, out_vec, nullptr, (cudaStream_t)stream);
}

vapr_status vapr_collision(vapr_ctx* c, const uint32_t* os, const int32_t* world_idx, int32_t B,
                           int32_t H, const vapr_cost_params* p, float* cost_pose,
                           float* cost_traj, uint32_t* cp, uint32_t* ov, void* stream) {
    CHECK(p != nullptr, VAPR_ERR_INVALID_ARG);
    return collision_common(c, os, world_idx, B, H, 1, 1, p->swept, p->sweep_steps, p->eta_world,
                            p->w_world, p->eta_self, p->w_self, cost_pose, cp, ov, cost_traj,
                            (cudaStream_t)stream);
}

// ---- a5 ------------------------------------------------------------------
vapr_status vapr_aggregate(vapr_ctx* c, const uint32_t* cp, int32_t swept, const uint32_t* ov,
                           int64_t n_rows, uint32_t* gos, void* stream) {
    CHECK(c != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(c->robot_set, VAPR_ERR_NOT_INITIALIZED);
    CHECK(n_rows >= 1, VAPR_ERR_SHAPE);
    CHECK(cp && ov && gos && aligned16(cp) && aligned16(ov) && aligned16(gos),
          VAPR_ERR_INVALID_ARG);
    DeviceGuard g(c->device);
    CHECK(g.ok && pending_fault() == VAPR_OK, VAPR_ERR_CUDA);
    return cuda_status(launch_aggregate(
        c->dfmt[swept ? VAPR_CLOSEST_PT_SWEPT : VAPR_CLOSEST_PT], c->dfmt[VAPR_OUT_VEC],
        c->dfmt[VAPR_GRAD_OUT_SPHERES], c->robot.cols, cp, ov, n_rows, gos,
        (cudaStream_t)stream));
}

// ---- a6 ------------------------------------------------------------------
vapr_status vapr_backward_kinematics(vapr_ctx* c, const float* q, int32_t B, int32_t H,
                                     const uint32_t* gos, float* grad_q, void* stream) {
    CHECK(c != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(c->robot_set, VAPR_ERR_NOT_INITIALIZED);
    CHECK(B >= 1 && H >= 1, VAPR_ERR_SHAPE);
    CHECK(q && gos && grad_q && aligned16(q) && aligned16(gos) && aligned16(grad_q),
          VAPR_ERR_INVALID_ARG);
    DeviceGuard g(c->device);
    CHECK(g.ok && pending_fault() == VAPR_OK, VAPR_ERR_CUDA);
    return cuda_status(launch_bk(c->robot, c->dfmt[VAPR_GRAD_OUT_SPHERES], q, (long long)B * H,
                                 gos, grad_q, (cudaStream_t)stream));
}

// ---- a7 ------------------------------------------------------------------
// sp (nullable): with c->sparse, the byte offsets of grad_out_spheres' mask,
// off, used and pool, and the pool capacity in words
static void ws_layout(const vapr_ctx* c, long long P, int swept, size_t off[VAPR_NUM_SLOTS],
                      size_t* cost_off, size_t* total, size_t* sp = nullptr,
                      size_t* pool_words = nullptr) {
    const int cols = c->robot.cols;
    for (int i = 0; i < VAPR_NUM_SLOTS; ++i) off[i] = SIZE_MAX;
    size_t o = 0;
    off[VAPR_OUT_SPHERES] = o;
    o = align256(o + packed_bytes(c->dfmt[VAPR_OUT_SPHERES], cols, P));
    const int cps = swept ? VAPR_CLOSEST_PT_SWEPT : VAPR_CLOSEST_PT;
    if (c->fused) {
        // N4: no tensor is materialised -- only the cost scratch below
        off[VAPR_OUT_SPHERES] = SIZE_MAX;
        o = 0;
    } else if (c->sparse) {
        // N3: the three gradient tensors in the sparse form -- per row a
        // sphere bitmap and the non-zero codes packed at pool + row * wmax
        // (closest_pt[_swept], out_vec) or at the row's own offset
        // (grad_out_spheres: off [P] and the words-in-use counter)
        size_t so[kSparseOffs];
        so[0] = o;                                            // gos mask [P] uint64
        o = align256(o + sizeof(uint64_t) * (size_t)P);
        so[1] = o;                                            // gos off [P] uint32
        o = align256(o + sizeof(uint32_t) * (size_t)P);
        so[2] = o;                                            // gos used
        o = align256(o + sizeof(uint32_t));
        so[3] = o;                                            // gos pool
        const size_t pw = sparse_pool_words_of(c->dfmt[VAPR_GRAD_OUT_SPHERES], cols, P);
        o = align256(o + sizeof(uint32_t) * pw);
        so[4] = o;                                            // closest_pt bitmaps [P]
        o = align256(o + sizeof(uint64_t) * (size_t)P);
        so[5] = o;                                            // out_vec bitmaps [P]
        o = align256(o + sizeof(uint64_t) * (size_t)P);
        so[6] = o;                                            // closest_pt pool (either slot)
        o = align256(o + sizeof(uint32_t) *
                             std::max(sparse_pool_words_of(c->dfmt[VAPR_CLOSEST_PT], cols, P),
                                      sparse_pool_words_of(c->dfmt[VAPR_CLOSEST_PT_SWEPT], cols, P)));
        so[7] = o;                                            // out_vec pool
        o = align256(o + sizeof(uint32_t) * sparse_pool_words_of(c->dfmt[VAPR_OUT_VEC], cols, P));
        if (sp)
            for (int i = 0; i < kSparseOffs; ++i) sp[i] = so[i];
        if (pool_words) *pool_words = pw;
    } else {
        off[cps] = o;
        // reserve the larger of the two collision slots so one workspace serves both modes
        o = align256(o + std::max(packed_bytes(c->dfmt[VAPR_CLOSEST_PT], cols, P),
                                  packed_bytes(c->dfmt[VAPR_CLOSEST_PT_SWEPT], cols, P)));
        off[VAPR_OUT_VEC] = o;
        o = align256(o + packed_bytes(c->dfmt[VAPR_OUT_VEC], cols, P));
        off[VAPR_GRAD_OUT_SPHERES] = o;
        o = align256(o + packed_bytes(c->dfmt[VAPR_GRAD_OUT_SPHERES], cols, P));
    }
    *cost_off = o;
    o = align256(o + sizeof(float) * (size_t)P);
    o = align256(o + sizeof(float) * (size_t)P);     // the self pass's cost (after cost_off)
    *total = o;
}

size_t vapr_cost_grad_workspace_bytes(const vapr_ctx* c, int32_t B, int32_t H) {
    if (!c || B < 1 || H < 1) return 0;
    size_t off[VAPR_NUM_SLOTS], co, total;
    ws_layout(c, (long long)B * H, 1, off, &co, &total);
    return total;
}

vapr_status vapr_cost_grad_workspace_layout(const vapr_ctx* c, int32_t B, int32_t H,
                                            int32_t swept, size_t* offsets) {
    CHECK(c != nullptr && offsets != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(B >= 1 && H >= 1, VAPR_ERR_SHAPE);
    size_t co, total;
    ws_layout(c, (long long)B * H, swept, offsets, &co, &total);
    return VAPR_OK;
}

vapr_status vapr_cost_grad_sparse_layout(const vapr_ctx* c, int32_t B, int32_t H,
                                         size_t* offsets, size_t* pool_words) {
    CHECK(c != nullptr && offsets != nullptr && pool_words != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(B >= 1 && H >= 1, VAPR_ERR_SHAPE);
    CHECK(c->sparse, VAPR_ERR_INVALID_ARG);
    size_t off[VAPR_NUM_SLOTS], co, total;
    ws_layout(c, (long long)B * H, 1, off, &co, &total, offsets, pool_words);
    return VAPR_OK;
}

}  // extern "C"

namespace {

// The vapr_cost_grad launch sequence for trajectories [b0, b0 + nb) of a
// batch of B (all device pointers are the whole-batch buffers; rows are
// contiguous per pose, so a trajectory range is a contiguous row range of
// every tensor).
cudaError_t enqueue_cost_grad(vapr_ctx* c, const float* q, const int32_t* world_idx, int b0,
                              int nb, int B, int H, const vapr_cost_params* p, void* workspace,
                              const size_t* off, float* cpose, float* cost_traj, float* grad_q,
                              cudaStream_t s) {
    char* ws = static_cast<char*>(workspace);
    const int cps = p->swept ? VAPR_CLOSEST_PT_SWEPT : VAPR_CLOSEST_PT;
    const long long p0 = (long long)b0 * H, P = (long long)nb * H;
    const int cols = c->robot.cols;
    if (c->fused) {
        const float* qc = q + p0 * kJoints;
        auto mark = [&](int i) {
            if (c->n_stage_ev == 6) cudaEventRecord(c->stage_ev[i], s);
        };
        // N4: one kernel for FK, both collision parts, aggregation and BK
        // (the FK / aggregation / BK events are recorded back to back)
        CollisionArgs a{};
        a.world_idx = world_idx + b0;
        a.B = nb;
        a.H = H;
        a.do_world = 1;
        a.do_self = 1;
        a.swept = p->swept ? 1 : 0;
        a.sweep_steps = p->sweep_steps;
        a.eta_w = p->eta_world;
        a.w_w = p->w_world;
        a.eta_s = p->eta_self;
        a.w_s = p->w_self;
        a.cull = c->cull;
        a.tab_img = static_cast<const uint4*>(c->d_tab_img);
        a.tab_img_bytes = c->tab_img_bytes;
        a.cost = cpose + p0;
        a.fused = 1;
        a.q = qc;
        a.grad_q = grad_q + p0 * kJoints;
        a.fgos = c->dfmt[VAPR_GRAD_OUT_SPHERES];
        mark(0);
        mark(1);
        cudaError_t e = launch_collision(c->robot, worlds_of(c), c->dfmt[VAPR_OUT_SPHERES],
                                         c->dfmt[cps], c->dfmt[VAPR_OUT_VEC], a, c->d_sched,
                                         &c->sched_next, s);
        mark(2);
        if (e == cudaSuccess)
            e = launch_traj_reduce(cpose + p0, nb, H, cost_traj ? cost_traj + b0 : nullptr, s, nullptr);
        mark(3);
        mark(4);
        mark(5);
        return e;
    }
    auto rows_of = [&](int slot) {
        return reinterpret_cast<uint32_t*>(ws + off[slot]) + p0 * row_words_of(c->dfmt[slot], cols);
    };
    uint32_t* os = rows_of(VAPR_OUT_SPHERES);
    uint32_t* cp = c->sparse ? nullptr : rows_of(cps);
    uint32_t* ov = c->sparse ? nullptr : rows_of(VAPR_OUT_VEC);
    uint32_t* gos = c->sparse ? nullptr : rows_of(VAPR_GRAD_OUT_SPHERES);
    // N3: grad_out_spheres in the sparse form (rows p0.. of mask / off; the
    // pool and its cursor are shared by all chunks)
    SparseOut spo{};
    SparseIn spi{};
    unsigned long long *cp_mask = nullptr, *ov_mask = nullptr;
    float* self_cost = nullptr;
    if (c->sparse) {
        size_t so[kSparseOffs], pw, o2[VAPR_NUM_SLOTS], co2, tot2;
        ws_layout(c, (long long)B * H, p->swept, o2, &co2, &tot2, so, &pw);
        spo.mask = reinterpret_cast<unsigned long long*>(ws + so[0]) + p0;
        spo.off = reinterpret_cast<uint32_t*>(ws + so[1]) + p0;
        spo.used = reinterpret_cast<uint32_t*>(ws + so[2]);
        spo.pool = reinterpret_cast<uint32_t*>(ws + so[3]);
        spo.seg0 = (uint32_t)sparse_pool_words_of(c->dfmt[VAPR_GRAD_OUT_SPHERES], cols, p0);
        cp_mask = reinterpret_cast<unsigned long long*>(ws + so[4]) + p0;
        ov_mask = reinterpret_cast<unsigned long long*>(ws + so[5]) + p0;
        cp = reinterpret_cast<uint32_t*>(ws + so[6]) + sparse_pool_words_of(c->dfmt[cps], cols, p0);
        ov = reinterpret_cast<uint32_t*>(ws + so[7]) + sparse_pool_words_of(c->dfmt[VAPR_OUT_VEC], cols, p0);
        spi.mask = spo.mask;
        spi.off = spo.off;
        spi.pool = spo.pool;
    }
    const float* qc = q + p0 * kJoints;
    // stage timing hook: event i after stage i (0: before FK)
    auto mark = [&](int i) {
        if (c->n_stage_ev == 6) cudaEventRecord(c->stage_ev[i], s);
    };
    // IKO terms (N2): FK writes cost_pose = pose + bound, the collision passes add
    IkArgs ik{};
    ik.goals = c->d_goals;
    ik.n_goals = c->n_goals;
    ik.world_idx = world_idx + b0;
    ik.H = H;
    ik.w_pos = p->w_pose_pos;
    ik.w_rot = p->w_pose_rot;
    ik.w_bound = p->w_bound;
    ik.cost = cpose + p0;
    const bool iko = ik_on(ik);
    mark(0);
    cudaError_t e = launch_fk(c->robot, c->dfmt[VAPR_OUT_SPHERES], qc, P, os, s, iko ? &ik : nullptr);
    mark(1);
    if (e == cudaSuccess) {
        CollisionArgs a{};
        a.os = os;
        a.world_idx = world_idx + b0;
        a.B = nb;
        a.H = H;
        a.do_world = 1;
        a.do_self = 1;
        a.swept = p->swept ? 1 : 0;
        a.sweep_steps = p->sweep_steps;
        a.eta_w = p->eta_world;
        a.w_w = p->w_world;
        a.eta_s = p->eta_self;
        a.w_s = p->w_self;
        a.cull = c->cull;
        a.tab_img = static_cast<const uint4*>(c->d_tab_img);
        a.tab_img_bytes = c->tab_img_bytes;
        a.cost = cpose + p0;
        a.cp = cp;
        a.ov = ov;
        a.cost_accumulate = iko ? 1 : 0;
        a.cp_mask = cp_mask;
        a.ov_mask = ov_mask;
        {   // the self pass's separate cost (workspace, after the scratch cost_pose)
            size_t o3[VAPR_NUM_SLOTS], co3, tot3;
            ws_layout(c, (long long)B * H, p->swept, o3, &co3, &tot3);
            self_cost = reinterpret_cast<float*>(ws + align256(co3 + sizeof(float) * (size_t)B * H)) + p0;
        }
        a.self_cost = self_cost;
        e = launch_collision(c->robot, worlds_of(c), c->dfmt[VAPR_OUT_SPHERES], c->dfmt[cps],
                             c->dfmt[VAPR_OUT_VEC], a, c->d_sched, &c->sched_next, s);
    }
    mark(2);
    // combines the self pass's cost into cost_pose (always) and sums cost_traj;
    // the rest of the chain as programmatic dependent launches (each kernel
    // waits for its predecessor at its start; measured runs with stage
    // events are plain launches)
    const bool pdl = VAPR_CHAIN_PDL && c->n_stage_ev == 0;
    // small batches (latency): the reduction needs only the collision passes,
    // so it runs on a side stream beside aggregation and BK and joins at the end
    bool side = VAPR_SIDE_REDUCE && P < VAPR_SIDE_REDUCE_BELOW && c->n_stage_ev == 0;
    if (side && !c->s_red) {
        if (cudaStreamCreateWithFlags(&c->s_red, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess)
            side = false;
    }
    if (e == cudaSuccess && side) {
        e = cudaEventRecord(c->ev_fork, s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(c->s_red, c->ev_fork, 0);
        if (e == cudaSuccess)
            e = launch_traj_reduce(cpose + p0, nb, H, cost_traj ? cost_traj + b0 : nullptr, c->s_red,
                                   self_cost, false);
        if (e == cudaSuccess) e = cudaEventRecord(c->ev_join, c->s_red);
    } else if (e == cudaSuccess) {
        e = launch_traj_reduce(cpose + p0, nb, H, cost_traj ? cost_traj + b0 : nullptr, s, self_cost,
                               pdl);
    }
    mark(3);
    // small sparse batches: the aggregation runs inside BK's CTAs (one launch
    // fewer on the latency-bound path; the same rows, codes and layout)
    const bool agg_in_bk = VAPR_AGG_IN_BK && c->sparse && !iko && P < VAPR_AGG_ROWS_BELOW_BK;
    AggArgs ag{};
    if (agg_in_bk) {
        const Fmt& fc = c->dfmt[cps];
        const Fmt& fo = c->dfmt[VAPR_OUT_VEC];
        ag.fcp = fc;
        ag.fov = fo;
        ag.cp = cp;
        ag.cpm = cp_mask;
        ag.ov = ov;
        ag.ovm = ov_mask;
        ag.cols = cols;
        ag.wc = (cols + fc.pf - 1) / fc.pf;
        ag.wo = (cols + fo.pf - 1) / fo.pf;
        ag.sp = spo;
    }
    if (e == cudaSuccess && !agg_in_bk)
        e = c->sparse ? launch_aggregate_sparse(c->dfmt[cps], c->dfmt[VAPR_OUT_VEC],
                                                c->dfmt[VAPR_GRAD_OUT_SPHERES], cols, cp, cp_mask,
                                                ov, ov_mask, P, spo, s, pdl)
                      : launch_aggregate(c->dfmt[cps], c->dfmt[VAPR_OUT_VEC],
                                         c->dfmt[VAPR_GRAD_OUT_SPHERES], cols, cp, ov, P, gos, s,
                                         nullptr, pdl);
    mark(4);
    if (e == cudaSuccess)
        e = launch_bk(c->robot, c->dfmt[VAPR_GRAD_OUT_SPHERES], qc, P, gos, grad_q + p0 * kJoints, s,
                      iko ? &ik : nullptr, c->sparse ? &spi : nullptr, pdl,
                      agg_in_bk ? &ag : nullptr);
    if (side) {
        const cudaError_t ej = cudaStreamWaitEvent(s, c->ev_join, 0);
        if (e == cudaSuccess) e = ej;
    }
    mark(5);
    return e;
}

}  // namespace

extern "C" {

vapr_status vapr_cost_grad(vapr_ctx* c, const float* q, const int32_t* world_idx, int32_t B,
                           int32_t H, const vapr_cost_params* p, void* workspace,
                           size_t workspace_bytes, float* cost_pose, float* cost_traj,
                           float* grad_q, void* stream) {
    CHECK(c != nullptr && p != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(c->robot_set && c->worlds_set && c->formats_set, VAPR_ERR_NOT_INITIALIZED);
    CHECK(B >= 1 && H >= 1, VAPR_ERR_SHAPE);
    CHECK(!p->swept || H >= 2, VAPR_ERR_SHAPE);
    CHECK(q && world_idx && grad_q && workspace, VAPR_ERR_INVALID_ARG);
    CHECK(aligned16(q) && aligned16(world_idx) && aligned16(grad_q) && aligned16(workspace),
          VAPR_ERR_INVALID_ARG);
    CHECK(cost_pose == nullptr || aligned16(cost_pose), VAPR_ERR_INVALID_ARG);
    CHECK(cost_traj == nullptr || aligned16(cost_traj), VAPR_ERR_INVALID_ARG);
    CHECK(p->eta_world > 0.f && p->eta_self > 0.f && std::isfinite(p->w_world) &&
              std::isfinite(p->w_self) && p->sweep_steps >= 0 && p->sweep_steps <= 64 &&
              std::isfinite(p->w_pose_pos) && std::isfinite(p->w_pose_rot) &&
              std::isfinite(p->w_bound),
          VAPR_ERR_INVALID_ARG);
    CHECK((p->w_pose_pos == 0.f && p->w_pose_rot == 0.f) || c->goals_set, VAPR_ERR_NOT_INITIALIZED);
    // N4 fused: the TO cost only, dense (no IKO terms, no sparse tensors)
    CHECK(!c->fused || (!c->sparse && p->w_pose_pos == 0.f && p->w_pose_rot == 0.f &&
                        p->w_bound == 0.f),
          VAPR_ERR_UNSUPPORTED);
    const long long P = (long long)B * H;
    size_t off[VAPR_NUM_SLOTS], co, total;
    ws_layout(c, P, p->swept, off, &co, &total);
    CHECK(workspace_bytes >= total, VAPR_ERR_INVALID_ARG);
    DeviceGuard g(c->device);
    CHECK(g.ok && pending_fault() == VAPR_OK, VAPR_ERR_CUDA);
    float* cpose = cost_pose ? cost_pose
                             : reinterpret_cast<float*>(static_cast<char*>(workspace) + co);
    cudaStream_t s0 = (cudaStream_t)stream;
    const int ns = std::min(c->n_streams, B);
    if (c->sparse) {            // N3: the sparse pool's counter, before any chunk
        size_t so[kSparseOffs], pw;
        ws_layout(c, P, p->swept, off, &co, &total, so, &pw);
        CHECK(pw <= 0xFFFFFFFFull, VAPR_ERR_SHAPE);          // 32-bit row offsets
        const cudaError_t e0 =
            cudaMemsetAsync(static_cast<char*>(workspace) + so[2], 0, sizeof(uint32_t), s0);
        if (e0 != cudaSuccess) return cuda_status(e0);
    }
    if (ns <= 1)
        return cuda_status(enqueue_cost_grad(c, q, world_idx, 0, B, B, H, p, workspace, off, cpose,
                                             cost_traj, grad_q, s0));
    // VAPR_OPT_STREAMS: trajectory chunks on context-owned streams, forked
    // from and joined back to the caller's stream (each chunk's kernels see
    // exactly its rows, so the results do not depend on the split)
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < ns && e == cudaSuccess; ++i)
        if (!c->par[i]) e = cudaStreamCreateWithFlags(&c->par[i], cudaStreamNonBlocking);
    while (e == cudaSuccess && c->events.size() < (size_t)(ns + 1)) {
        cudaEvent_t ev;
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e == cudaSuccess) c->events.push_back(ev);
    }
    if (e == cudaSuccess) e = cudaEventRecord(c->events[0], s0);
    const int Bc = (B + ns - 1) / ns;
    for (int i = 0; i < ns && e == cudaSuccess; ++i) {
        const int b0 = i * Bc, nb = std::min(Bc, B - b0);
        if (nb <= 0) break;
        e = cudaStreamWaitEvent(c->par[i], c->events[0], 0);
        if (e == cudaSuccess)
            e = enqueue_cost_grad(c, q, world_idx, b0, nb, B, H, p, workspace, off, cpose, cost_traj,
                                  grad_q, c->par[i]);
        if (e == cudaSuccess) e = cudaEventRecord(c->events[1 + i], c->par[i]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s0, c->events[1 + i], 0);
    }
    return cuda_status(e);
}

vapr_status vapr_cost_grad_host(vapr_ctx* c, const float* q_host, const int32_t* world_idx,
                                int32_t B, int32_t H, const vapr_cost_params* p, void* workspace,
                                size_t workspace_bytes, float* q_dev, float* cost_pose_dev,
                                float* cost_traj_dev, float* grad_q_dev, float* cost_traj_host,
                                float* grad_q_host, int32_t n_chunks, void* stream) {
    CHECK(c != nullptr && p != nullptr, VAPR_ERR_INVALID_ARG);
    CHECK(c->robot_set && c->worlds_set && c->formats_set, VAPR_ERR_NOT_INITIALIZED);
    CHECK(B >= 1 && H >= 1, VAPR_ERR_SHAPE);
    CHECK(!p->swept || H >= 2, VAPR_ERR_SHAPE);
    CHECK(q_host && grad_q_host && world_idx && workspace && q_dev && cost_traj_dev && grad_q_dev,
          VAPR_ERR_INVALID_ARG);
    CHECK(aligned16(q_dev) && aligned16(world_idx) && aligned16(grad_q_dev) &&
              aligned16(workspace) && aligned16(cost_traj_dev),
          VAPR_ERR_INVALID_ARG);
    CHECK(cost_pose_dev == nullptr || aligned16(cost_pose_dev), VAPR_ERR_INVALID_ARG);
    CHECK(n_chunks >= 0, VAPR_ERR_INVALID_ARG);
    CHECK(p->eta_world > 0.f && p->eta_self > 0.f && std::isfinite(p->w_world) &&
              std::isfinite(p->w_self) && p->sweep_steps >= 0 && p->sweep_steps <= 64 &&
              std::isfinite(p->w_pose_pos) && std::isfinite(p->w_pose_rot) &&
              std::isfinite(p->w_bound),
          VAPR_ERR_INVALID_ARG);
    CHECK((p->w_pose_pos == 0.f && p->w_pose_rot == 0.f) || c->goals_set, VAPR_ERR_NOT_INITIALIZED);
    // N4 fused: the TO cost only, dense (no IKO terms, no sparse tensors)
    CHECK(!c->fused || (!c->sparse && p->w_pose_pos == 0.f && p->w_pose_rot == 0.f &&
                        p->w_bound == 0.f),
          VAPR_ERR_UNSUPPORTED);
    const long long P = (long long)B * H;
    size_t off[VAPR_NUM_SLOTS], co, total;
    ws_layout(c, P, p->swept, off, &co, &total);
    CHECK(workspace_bytes >= total, VAPR_ERR_INVALID_ARG);
    DeviceGuard g(c->device);
    CHECK(g.ok && pending_fault() == VAPR_OK, VAPR_ERR_CUDA);
    float* cpose = cost_pose_dev ? cost_pose_dev
                                 : reinterpret_cast<float*>(static_cast<char*>(workspace) + co);
    // chunking: whole trajectories, up to ~700k poses per (full-size) chunk
    // by default (measured on the 2.56M-pose bench workload against a 4.0 ms
    // device step: 2 chunks 5.51 ms, 3: 5.03, 4: 4.92, 5: 4.99, 6: 5.16, 8:
    // 5.55; round 1, against a 5.24 ms step, 3 was best)
    int nc = n_chunks;
    if (nc == 0) nc = (int)std::max(1LL, std::min<long long>(16, (P + 699999) / 700000));
    nc = std::min(nc, B);
    // chunk boundaries: the first and last chunks a quarter of the others,
    // so the only copies left exposed (the first upload, the last download)
    // are short
    std::vector<int> cb(nc + 1, 0);
    {
        const double ew = VAPR_END_CHUNK_WEIGHT;
        const double wsum = (nc >= 3) ? (nc - 2) + 2.0 * ew : nc;
        double acc = 0.0;
        for (int i = 0; i < nc; ++i) {
            acc += (nc >= 3 && (i == 0 || i == nc - 1)) ? ew : 1.0;
            cb[i + 1] = (int)std::llround(B * acc / wsum);
        }
        cb[nc] = B;
        for (int i = 1; i <= nc; ++i) cb[i] = std::max(cb[i], cb[i - 1] + 1);   // non-empty
        for (int i = nc - 1; i >= 0; --i) cb[i] = std::min(cb[i], cb[i + 1] - 1);
    }
    cudaError_t e = cudaSuccess;
    if (!c->s_in) e = cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking);
    if (e == cudaSuccess && !c->s_out) e = cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking);
    while (e == cudaSuccess && c->events.size() < (size_t)(2 * nc + 2)) {
        cudaEvent_t ev;
        e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        if (e == cudaSuccess) c->events.push_back(ev);
    }
    if (e != cudaSuccess) return cuda_status(e);
    cudaStream_t s = (cudaStream_t)stream;
    cudaEvent_t* ev = c->events.data();
    if (c->sparse) {            // N3: the sparse pool's counter, before any chunk
        size_t so[kSparseOffs], pw;
        ws_layout(c, P, p->swept, off, &co, &total, so, &pw);
        CHECK(pw <= 0xFFFFFFFFull, VAPR_ERR_SHAPE);          // 32-bit row offsets
        e = cudaMemsetAsync(static_cast<char*>(workspace) + so[2], 0, sizeof(uint32_t), s);
        if (e != cudaSuccess) return cuda_status(e);
    }
    // the copy streams start after the work already enqueued on `stream`
    e = cudaEventRecord(ev[0], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->s_in, ev[0], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c->s_out, ev[0], 0);
    for (int i = 0; i < nc && e == cudaSuccess; ++i) {
        const int b0 = cb[i], nb = cb[i + 1] - cb[i];
        const size_t qo = (size_t)b0 * H * kJoints, qn = (size_t)nb * H * kJoints * sizeof(float);
        e = cudaMemcpyAsync(q_dev + qo, q_host + qo, qn, cudaMemcpyHostToDevice, c->s_in);
        if (e == cudaSuccess) e = cudaEventRecord(ev[2 + 2 * i], c->s_in);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[2 + 2 * i], 0);
        if (e == cudaSuccess)
            e = enqueue_cost_grad(c, q_dev, world_idx, b0, nb, B, H, p, workspace, off, cpose,
                                  cost_traj_dev, grad_q_dev, s);
        if (e == cudaSuccess) e = cudaEventRecord(ev[3 + 2 * i], s);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(c->s_out, ev[3 + 2 * i], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(grad_q_host + qo, grad_q_dev + qo, qn, cudaMemcpyDeviceToHost,
                                c->s_out);
        if (e == cudaSuccess && cost_traj_host)
            e = cudaMemcpyAsync(cost_traj_host + b0, cost_traj_dev + b0, sizeof(float) * nb,
                                cudaMemcpyDeviceToHost, c->s_out);
    }
    // `stream` completes only after the last D2H copy
    if (e == cudaSuccess) e = cudaEventRecord(ev[1], c->s_out);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev[1], 0);
    return cuda_status(e);
}

// ---- N1 ------------------------------------------------------------------
static bool scales_ok(const float* scales, int32_t N, LbfgsScales* out) {
    if (!scales || N < 1 || N > 32) return false;
    for (int i = 0; i < N; ++i) {
        if (!(scales[i] > 0.f) || !std::isfinite(scales[i])) return false;
        if (i > 0 && !(scales[i] > scales[i - 1])) return false;
        out->s[i] = scales[i];
    }
    return true;
}

vapr_status vapr_lbfgs_candidates(const float* x, const float* d, int32_t B, int32_t D,
                                  const float* scales, int32_t N, float* cand, void* stream) {
    CHECK(B >= 0 && D >= 1 && N >= 1 && N <= 32, VAPR_ERR_SHAPE);
    if (B == 0) return VAPR_OK;
    LbfgsScales sc{};
    CHECK(x && d && cand && scales_ok(scales, N, &sc), VAPR_ERR_INVALID_ARG);
    CHECK(pending_fault() == VAPR_OK, VAPR_ERR_CUDA);
    return cuda_status(launch_lbfgs_candidates(x, d, B, D, N, sc, cand, (cudaStream_t)stream));
}

vapr_status vapr_lbfgs_step(int32_t B, int32_t D, const float* scales, int32_t N,
                            const float* cand_cost, const float* cand_grad, float* x, float* g,
                            float* cost, float* d, float* hist_s, float* hist_y, float* hist_rho,
                            int32_t* hist_count, int32_t* hist_head, int32_t* chosen, int32_t m,
                            float curvature_eps, const uint8_t* fixed, void* stream) {
    CHECK(B >= 0 && D >= 1 && D <= VAPR_LBFGS_MAX_D && N >= 1 && N <= 32 && m >= 1 &&
              m <= VAPR_LBFGS_MAX_M,
          VAPR_ERR_SHAPE);
    if (B == 0) return VAPR_OK;
    LbfgsScales sc{};
    CHECK(scales_ok(scales, N, &sc) && std::isfinite(curvature_eps), VAPR_ERR_INVALID_ARG);
    CHECK(cand_cost && cand_grad && x && g && cost && d && hist_s && hist_y && hist_rho &&
              hist_count && hist_head,
          VAPR_ERR_INVALID_ARG);
    CHECK(pending_fault() == VAPR_OK, VAPR_ERR_CUDA);
    return cuda_status(launch_lbfgs_step(B, D, N, sc, cand_cost, cand_grad, x, g, cost, d, hist_s,
                                         hist_y, hist_rho, hist_count, hist_head, chosen, m,
                                         curvature_eps, fixed, (cudaStream_t)stream));
}

// ---- e -------------------------------------------------------------------
vapr_status vapr_best_per_problem(const float* cost_traj, int32_t n_problems, int32_t seeds,
                                  float* best_cost, int32_t* best_seed, void* stream) {
    CHECK(n_problems >= 0 && seeds >= 1, VAPR_ERR_SHAPE);
    if (n_problems == 0) return VAPR_OK;
    CHECK(cost_traj && best_cost && best_seed, VAPR_ERR_INVALID_ARG);
    CHECK(pending_fault() == VAPR_OK, VAPR_ERR_CUDA);
    return cuda_status(launch_best_per_problem(cost_traj, n_problems, seeds, best_cost, best_seed,
                                               (cudaStream_t)stream));
}

}  // extern "C"

// common.cuh -- shared device helpers of the CUDA path (sm_100a).
// Element types: double (real) and double2 (complex, .x = re, .y = im).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstddef>
#include <climits>
#include <cstdlib>
#include <cmath>

#define FROB_DEV __device__ __forceinline__
#define FROB_DEV_HOST_INLINE __host__ __device__ inline

namespace frob {

// Tuning switches (A/B measurement aids) are read from the environment only in a tuning build
// (-DFROB_TUNING, tools/); the shipped library always takes the measured defaults.
inline const char *tuning_env(const char *name) {
#ifdef FROB_TUNING
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

// AUTO branch rule (reading R1'): S1 is kept while kappa_inf(A) / sqrt(n) <= KAPPA_SWITCH,
// kappa_inf(A) = ||A||_inf ||A^-1||_inf of the computed inverse (the conditioning of X drives the
// leading term of Thm 5.2's bound; kappa_inf / sqrt(n) tracks kappa_2 of dense matrices
// up to an O(1) factor); above it (or with A singular) both parts are inverted and the smaller
// kappa_inf wins.  2.5e4: S1's error is at most ~2.6 u kappa_inf(A) (R1'), so the switch
// keeps it <= 1e-10 up to n = 128 by that calibration, not by the luck of one kernel's rounding.
constexpr double KAPPA_SWITCH = 2.5e4;
FROB_DEV_HOST_INLINE double kappa_switch(int n) { return KAPPA_SWITCH * sqrt((double)n); }

// process-wide count of kernel launches issued by the library (frob_launch_count())
unsigned long long &launch_counter();
inline void count_launch(unsigned long long k = 1) { __atomic_fetch_add(&launch_counter(), k, __ATOMIC_RELAXED); }

// Optional per-kernel timing (frob_profile_enable): CUDA events recorded on the launching
// stream around instrumented launches; off by default (then a no-op).
bool prof_enabled();
// work: algorithmic flops of the launch (FP64; complex multiply-add = 8 real flops)
void prof_record(const char *name, cudaStream_t s, bool begin, double work);
// role tag for the GEMM launches below it (profiler names; string literals, compared by address)
extern thread_local const char *g_gemm_tag;
struct GemmTag {
    const char *prev;
    explicit GemmTag(const char *t) : prev(g_gemm_tag) { g_gemm_tag = t; }
    ~GemmTag() { g_gemm_tag = prev; }
};
struct ProfScope {
    const char *name;
    cudaStream_t s;
    bool on;
    ProfScope(const char *nm, cudaStream_t st, double work = 0.0) : name(nm), s(st), on(prof_enabled()) {
        if (on) prof_record(name, s, true, work);
    }
    ~ProfScope() {
        if (on) prof_record(name, s, false, 0.0);
    }
};

// ------------------------------------------------------------------ element ops
FROB_DEV double zero_of(double) { return 0.0; }
FROB_DEV double2 zero_of(double2) { return make_double2(0.0, 0.0); }
FROB_DEV double one_of(double) { return 1.0; }
FROB_DEV double2 one_of(double2) { return make_double2(1.0, 0.0); }

// pivot magnitude: |x| for real, |re|+|im| for complex (LAPACK idamax / izamax)
FROB_DEV double pmag(double v) { return fabs(v); }
FROB_DEV double pmag(double2 v) { return fabs(v.x) + fabs(v.y); }
// pivot-search key: NaN counts as +inf so a pivot always exists (the non-finite
// result is then reported through the nonfinite flag instead of faulting)
template <typename T>
FROB_DEV double pkey(T v) {
    const double m = pmag(v);
    return (m != m) ? INFINITY : m;
}
FROB_DEV bool is_zero(double v) { return v == 0.0; }
FROB_DEV bool is_zero(double2 v) { return v.x == 0.0 && v.y == 0.0; }

FROB_DEV double mul(double a, double b) { return a * b; }
FROB_DEV double2 mul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// c - a*b
FROB_DEV double msub(double c, double a, double b) { return fma(-a, b, c); }
FROB_DEV double2 msub(double2 c, double2 a, double2 b) {
    return make_double2(fma(-a.x, b.x, fma(a.y, b.y, c.x)), fma(-a.x, b.y, fma(-a.y, b.x, c.y)));
}
// c + a*b
FROB_DEV double madd(double c, double a, double b) { return fma(a, b, c); }
FROB_DEV double2 madd(double2 c, double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
FROB_DEV double add(double a, double b) { return a + b; }
FROB_DEV double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
FROB_DEV double neg(double a) { return -a; }
FROB_DEV double2 neg(double2 a) { return make_double2(-a.x, -a.y); }
FROB_DEV double recip(double a) { return 1.0 / a; }
FROB_DEV double2 recip(double2 a) {
    // 1/(x+iy) = (x - iy)/(x^2+y^2), scaled to avoid overflow/underflow of x^2+y^2
    double s = fmax(fabs(a.x), fabs(a.y));
    double xs = a.x / s, ys = a.y / s;
    double d = s * (xs * xs + ys * ys);
    return make_double2(xs / d, -ys / d);
}
// Branch-free reciprocal for the LU critical path: MUFU approximation + two Newton steps
// (error ~1 ulp; not correctly rounded, like LAPACK's multiply-by-reciprocal scaling).
// Inputs with |x| > 2^1021 flush to 0 (ftz); pivots that large do not occur here.
FROB_DEV double frcp(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}
FROB_DEV double frcp(double2 x) { return 0.0; }  // unused overload guard
FROB_DEV double scal(double a, double s) { return a * s; }
FROB_DEV double2 scal(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
FROB_DEV bool finite_of(double v) { return isfinite(v); }
FROB_DEV bool finite_of(double2 v) { return isfinite(v.x) && isfinite(v.y); }

FROB_DEV double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
FROB_DEV double2 shfl(double2 v, int src) {
    return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

// argmax key: larger magnitude wins; ties -> smaller row index (first max)
struct ArgMax {
    double v;
    int i;
};
FROB_DEV bool better(double v1, int i1, double v2, int i2) {
    return (v1 > v2) || (v1 == v2 && i1 < i2);
}
FROB_DEV ArgMax warp_argmax(double v, int i) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, v, off);
        int i2 = __shfl_xor_sync(0xffffffffu, i, off);
        if (better(v2, i2, v, i)) { v = v2; i = i2; }
    }
    return ArgMax{v, i};
}

// Exact warp argmax with redux.sync on the IEEE bit pattern of a non-negative key
// (monotone as an unsigned integer): max of the high word, then of the low word among
// the lanes holding that high word, then min index among the lanes holding both.
// Same result as warp_argmax (first max); three REDUX instead of five shuffle rounds.
FROB_DEV unsigned redux_max(unsigned v) {
    unsigned r;
    asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}
FROB_DEV unsigned redux_min(unsigned v) {
    unsigned r;
    asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}
// Integer pivot keys: 1 + the IEEE bit pattern of |v| (monotone in |v|; NaN patterns sort
// above +inf, i.e. NaN counts as the largest magnitude), 0 = no candidate.  Real only;
// complex keys (|re|+|im|) go through the double path.
FROB_DEV unsigned long long pkey_bits(double v) {
    return ((unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull) + 1ull;
}
FROB_DEV unsigned long long pkey_bits(double2 v) {
    const double m = fabs(v.x) + fabs(v.y);
    return (m != m) ? 0x7ff8000000000001ull : (unsigned long long)__double_as_longlong(m) + 1ull;
}
struct ArgMaxK {
    unsigned long long k;
    int i;
};
// first max over (key, -idx) within the warp, 3 x REDUX
FROB_DEV ArgMaxK warp_argmax_key(unsigned long long kb, int idx) {
    const unsigned hi = (unsigned)(kb >> 32), lo = (unsigned)kb;
    const unsigned mh = redux_max(hi);
    const unsigned ml = redux_max(hi == mh ? lo : 0u);
    const bool cand = (hi == mh) && (lo == ml);
    const unsigned mi = redux_min(cand ? (unsigned)idx : 0xffffffffu);
    ArgMaxK r;
    r.k = ((unsigned long long)mh << 32) | ml;
    r.i = (r.k == 0ull) ? INT_MAX : (int)mi;
    return r;
}
// key must be >= 0 (or -1.0 for "no candidate", mapped below every real key)
FROB_DEV ArgMax warp_argmax_redux(double key, int idx) {
    const unsigned long long kb = (key < 0.0) ? 0ull : (unsigned long long)__double_as_longlong(key) + 1ull;
    const unsigned hi = (unsigned)(kb >> 32), lo = (unsigned)kb;
    const unsigned mh = redux_max(hi);
    const unsigned ml = redux_max(hi == mh ? lo : 0u);
    const bool cand = (hi == mh) && (lo == ml);
    const unsigned mi = redux_min(cand ? (unsigned)idx : 0xffffffffu);
    const unsigned long long mk = ((unsigned long long)mh << 32) | ml;
    ArgMax r;
    r.v = (mk == 0ull) ? -1.0 : __longlong_as_double((long long)(mk - 1ull));
    r.i = (int)mi;
    if (mk == 0ull) r.i = INT_MAX;
    return r;
}

// ------------------------------------------------------------------ FP64 tensor core
// mma.sync m8n8k4 f64 (SASS DMMA.8x8x4).  Fragments (g = lane>>2, t = lane&3):
//   a = A[g][t], b = B[t][g], c0 = C[g][2t], c1 = C[g][2t+1].
FROB_DEV void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// ------------------------------------------------------------------ programmatic dependent launch
// Kernels of the LU chain are launched with programmatic stream serialization: each one
// lets its successor launch immediately and waits for its predecessor's results before
// touching memory (both are no-ops without the launch attribute).
FROB_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
FROB_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    count_launch();
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// the same, in thread-block clusters of (1, 1, cz) along the grid's z dimension
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster_z(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                                        int cz, Args... args) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[2];
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 1;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = (unsigned)cz;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    count_launch();
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ------------------------------------------------------------------ cluster DSMEM + mbarrier
FROB_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
FROB_DEV double ld_cluster(unsigned addr, double) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}
FROB_DEV double2 ld_cluster(unsigned addr, double2) {
    double2 v;
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}
FROB_DEV unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
FROB_DEV unsigned mapa_u32(unsigned addr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
FROB_DEV void st_cluster(unsigned addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
FROB_DEV void st_cluster(unsigned addr, double2 v) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}
FROB_DEV void st_cluster(unsigned addr, unsigned long long v) {
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
FROB_DEV void st_cluster(unsigned addr, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
FROB_DEV void mbar_init(unsigned addr, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}
FROB_DEV void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
FROB_DEV void mbar_remote_arrive(unsigned cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
FROB_DEV void mbar_wait_parity(unsigned addr, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}

// ------------------------------------------------------------------ cp.async
FROB_DEV void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
FROB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
FROB_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace frob

// Monte Carlo of the asynchronous detection process on the GPU, the
// paper's ground truth for the Markov model: one thread per independent chain ("run").
//
// A chain: photons arrive as an inhomogeneous Poisson process with the periodic rate lambda~ (Eq. 1
// replicated). After a registration at T_k = q t_r + t the SPAD is dead for t_d and
// re-arms at T_k + t_d; the next registration is the first arrival after re-arming:
//   T_{k+1} = Ftilde^{-1}(Ftilde(T_k + t_d) + E),   E = -log U,  U uniform on (0, 1]
// (time change of a Poisson process), with Ftilde(q t_r + t) = q Lambda + F(t) and F in closed form
// (erfc; Thm 1). U comes from splitmix64 advanced once per registration from the chain seed
// seed + c * 0xD1B54A32D192ED03 (c = item * n_runs + run): a counter-based stream, the same algorithm
// the CPU oracle implements, so a chain can be replayed on the CPU draw for draw. With n_split > 1 a
// run is n_split independent sub-chains (chain c = (item * n_runs + run) * n_split + sub), each with
// its own burn-in and 1/n_split of the run's budget, adding into the run's histogram: the same
// stationary estimate with n_split times the parallelism (n_split = 1 is the paper's protocol).
// The timestamp X_k = T_k mod t_r goes into the run's n_hist-bin histogram ((k-1) Delta_h,
// k Delta_h] (X = 0 read as t_r) once k >= n_burn; a run stops after n_regs counted registrations, or
// (n_cycles > 0) at the first registration n_cycles laser periods after the end of the burn-in.
//
// Inversion of F on [0, t_r): a CTA serves runs of one item; it tabulates F and lambda = dF/dt at
// 512 + 1 uniform nodes in shared memory, brackets the root by binary search in the table, starts from
// the root of the cubic Hermite interpolant on the bracket, then runs Newton steps on the closed form
// (dF/dt = lambda > 0 since B > 0) safeguarded by bisection of the bracket until F(t) - y reaches the
// rounding floor of F or the step is below 1e-15 t_r.
#include "common.cuh"

namespace spl {
namespace {

constexpr int kMcThreads = 128;
constexpr int kMcTable = 512;

struct McConst {
    double is[kMaxPulses], c0[kMaxPulses], amp[kMaxPulses], rate_b, Lam;
};

__device__ __forceinline__ double mc_cdf(double z) { return 0.5 * erfc(-z * 0.70710678118654752440); }

__device__ __forceinline__ double mc_F(const FluxDev &f, const McConst &q, double t) {
    double v = q.rate_b * t;
    for (int k = 0; k < f.k; ++k) v += f.S[k] * (mc_cdf((t - f.tau[k]) * q.is[k]) - q.c0[k]);
    return v;
}

__device__ __forceinline__ double mc_lambda(const FluxDev &f, const McConst &q, double t) {
    double v = q.rate_b;
    for (int k = 0; k < f.k; ++k) {
        const double z = (t - f.tau[k]) * q.is[k];
        v += q.amp[k] * exp(-0.5 * z * z);
    }
    return v;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t &s) {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double unif01_open(uint64_t &s) {   // (0, 1]
    return ((double)(splitmix64(s) >> 11) + 1.0) * (1.0 / 9007199254740992.0);
}

// F(t) = y on [0, t_r], 0 <= y < Lambda. tab = F at the 513 nodes, dtab = lambda = dF/dt at the nodes.
__device__ double mc_finv(const FluxDev &f, const McConst &q, const double *tab, const double *dtab, double y) {
    const double h = f.t_r / kMcTable;
    int lo_i = 0, hi_i = kMcTable;            // tab[lo_i] <= y < tab[hi_i]
    while (hi_i - lo_i > 1) {
        const int mid = (lo_i + hi_i) >> 1;
        if (tab[mid] <= y) lo_i = mid; else hi_i = mid;
    }
    double lo = lo_i * h, hi = hi_i == kMcTable ? f.t_r : hi_i * h;
    const double flo = tab[lo_i], fhi = tab[hi_i];
    // initial guess: root of the cubic Hermite interpolant of F on the bracket (F and lambda at its ends;
    // error ~h^4), by Newton on the polynomial from the linear guess (no transcendentals)
    double t;
    if (fhi > flo) {
        const double hh = hi - lo, d0 = dtab[lo_i] * hh, d1 = dtab[hi_i] * hh, df = fhi - flo;
        double u = (y - flo) / df;
        for (int it = 0; it < 3; ++it) {
            const double u2 = u * u, u3 = u2 * u;
            const double H = flo + df * (3.0 * u2 - 2.0 * u3) + d0 * (u3 - 2.0 * u2 + u) + d1 * (u3 - u2);
            const double dH = df * (6.0 * u - 6.0 * u2) + d0 * (3.0 * u2 - 4.0 * u + 1.0) + d1 * (3.0 * u2 - 2.0 * u);
            if (!(dH > 0.0)) break;
            u -= (H - y) / dH;
            u = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u);
        }
        t = lo + u * hh;
    } else {
        t = 0.5 * (lo + hi);
    }
    // stop when the step is below 1e-15 t_r, the bracket is that narrow, or F(t) - y is at the
    // rounding floor of F (|g| <= 4 eps Lambda): below it the Newton step is rounding noise
    const double eps = 1e-15 * f.t_r;
    const double gfloor = 4.0 * 2.220446049250313e-16 * q.Lam;
    for (int it = 0; it < 200; ++it) {
        const double g = mc_F(f, q, t) - y;
        if (g > 0.0) hi = t; else lo = t;
        double tn = t - g / mc_lambda(f, q, t);
        if (!(tn > lo && tn < hi)) tn = 0.5 * (lo + hi);
        const bool done = fabs(g) <= gfloor || fabs(tn - t) <= eps || hi - lo <= eps;
        t = fabs(g) <= gfloor ? t : tn;
        if (done) break;
    }
    return t;
}

__global__ void __launch_bounds__(kMcThreads) k_mc(const McArgs a) {
    __shared__ double tab[kMcTable + 1], dtab[kMcTable + 1];
    __shared__ FluxDev fs;
    __shared__ McConst qs;                                  // per-flux constants, shared by the CTA
    const int item = blockIdx.y;
    const int chain = blockIdx.x * kMcThreads + threadIdx.x;   // run * n_split + sub-chain
    if (threadIdx.x == 0) {
        fs = a.flux[a.prof[item]];
        qs.rate_b = fs.B / fs.t_r;
        for (int k = 0; k < fs.k; ++k) {
            qs.is[k] = 1.0 / fs.sigma[k];
            qs.c0[k] = mc_cdf(-fs.tau[k] / fs.sigma[k]);
            qs.amp[k] = fs.S[k] / (fs.sigma[k] * 2.50662827463100050242);
        }
    }
    __syncthreads();
    const FluxDev &f = fs;
    for (int g = threadIdx.x; g <= kMcTable; g += kMcThreads) {
        const double tg = g == kMcTable ? f.t_r : g * (f.t_r / kMcTable);
        tab[g] = mc_F(f, qs, tg);
        dtab[g] = mc_lambda(f, qs, tg);
    }
    __syncthreads();
    if (threadIdx.x == 0) qs.Lam = tab[kMcTable];           // Lambda = F(t_r) (reading R5)
    __syncthreads();
    const McConst &q = qs;
    if (chain >= a.n_runs * a.n_split) return;
    const int run = chain / a.n_split;
    const double t_d = a.td[item];
    const long long c = (long long)item * a.n_runs * a.n_split + chain;   // chain index (seed, records)
    uint64_t st = a.seed + (uint64_t)c * 0xD1B54A32D192ED03ull;
    unsigned long long *hist = a.hist + ((size_t)item * a.n_runs + run) * a.n_hist;
    const double dh = f.t_r / a.n_hist;
    long long qp = 0, q_end = -1;
    double t = 0.0;
    for (long long k = 0;; ++k) {
        // re-arm at T + t_d, add an Exp(1) to the integrated flux, invert
        double tt = t + t_d;
        long long qq = qp + (long long)floor(tt / f.t_r);
        tt = fmod(tt, f.t_r);
        if (tt < 0.0) tt += f.t_r;
        const double target = mc_F(f, q, tt) - log(unif01_open(st));
        long long extra = (long long)floor(target / q.Lam);
        double rem = target - (double)extra * q.Lam;
        if (rem < 0.0) { rem += q.Lam; extra -= 1; }
        if (rem >= q.Lam) { rem -= q.Lam; extra += 1; }
        qp = qq + extra;
        t = mc_finv(f, q, tab, dtab, rem);
        if (t >= f.t_r) { t -= f.t_r; qp += 1; }
        if (k < a.n_record) {
            a.q_rec[(size_t)c * a.n_record + k] = qp;
            a.t_rec[(size_t)c * a.n_record + k] = t;
        }
        if (k < a.n_burn) continue;
        if (a.n_cycles > 0) {
            if (q_end < 0) q_end = (k == 0 ? 0 : qp) + a.n_cycles;   // burn-in ends at this registration
            if (qp >= q_end) break;
        } else if (k - a.n_burn >= a.n_regs) {
            break;
        }
        int bin = (int)ceil(t / dh) - 1;                   // ((k-1) dh, k dh]; X = 0 is t_r
        if (bin < 0) bin = a.n_hist - 1;
        if (bin >= a.n_hist) bin = a.n_hist - 1;
        atomicAdd(hist + bin, 1ull);
    }
}

}  // namespace

cudaError_t launch_mc(const McArgs &a, cudaStream_t s) {
    dim3 grid((unsigned)((a.n_runs * a.n_split + kMcThreads - 1) / kMcThreads), (unsigned)a.n_items);
    k_mc<<<grid, kMcThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace spl

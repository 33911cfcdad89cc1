// plan.cu -- errors, plans (window / precision / fine-grid geometry), cuFFT plan cache,
// and the ES window transform table.
#include <atomic>
#include <cmath>
#include <map>
#include <set>
#include <mutex>
#include <tuple>
#include <vector>

#include <cstring>
#include "fk_internal.cuh"

namespace fk {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
fk_status fail(fk_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}
const char* last_error_cstr() { return g_last_error.c_str(); }

static std::atomic<int64_t> g_kernels{0};
static std::atomic<bool> g_prof_on{false};
static std::mutex g_prof_mu;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_prof_ev;
static thread_local cudaEvent_t g_prof_open = nullptr;

void count_launch(int k) { g_kernels.fetch_add(k, std::memory_order_relaxed); }

void prof_spread_begin(cudaStream_t s) {
  if (!g_prof_on.load()) return;
  cudaEventCreate(&g_prof_open);
  cudaEventRecord(g_prof_open, s);
}

void prof_spread_end(cudaStream_t s) {
  if (!g_prof_on.load() || !g_prof_open) return;
  cudaEvent_t e1;
  cudaEventCreate(&e1);
  cudaEventRecord(e1, s);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_ev.emplace_back(g_prof_open, e1);
  g_prof_open = nullptr;
}

int profile_read(double* ms, int64_t* launches, int64_t* kernels) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double tot = 0.0;
  for (auto& pr : g_prof_ev) {
    cudaEventSynchronize(pr.second);
    float t = 0.f;
    cudaEventElapsedTime(&t, pr.first, pr.second);
    tot += t;
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  if (ms) *ms = tot;
  if (launches) *launches = (int64_t)g_prof_ev.size();
  if (kernels) *kernels = g_kernels.exchange(0);
  g_prof_ev.clear();
  return 0;
}

void profile_enable(int on) { g_prof_on.store(on != 0); }

int device_sm_count() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return sms;
}

static int max_smem_optin() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v > 0 ? v : 232448;
}

int fft_friendly(int n) {
  int best = 1 << 30;
  for (long a = 8; a < 2L * n + 64; a *= 2)
    for (long b = a; b < 2L * n + 64; b *= 3)
      for (long c = b; c < 2L * n + 64; c *= 5)
        if (c >= n && c < best) best = (int)c;
  return best;
}

// fp32 path: cubic B-spline window.  Its transform is sinc^4, so the aliased copies at k +- nf
// are damped by (k/(nf-k))^4 <= (2 sigma - 1)^-4 at the edge mode:
// sigma = ((1/eps)^{1/4} + 1) / 2 puts the edge-mode error near eps.
static double bs3_sigma(double eps) { return std::max(4.0, 0.5 * (std::pow(1.0 / eps, 0.25) + 1.0)); }

fk_status make_plan1(int d, int m, double eps, bool need_mu, bool need_r, Plan1* p) {
  if (d != 1) return fail(FK_E_UNSUPPORTED, "make_plan1: only d = 1 here");
  Plan1 q;
  q.d = d;
  q.m = m;
  q.eps = eps;
  const int sms = device_sm_count();
  if (sms <= 0) return fail(FK_E_CUDA, "no CUDA device");
  const int smem_cap = max_smem_optin();
  const int modes_mu = 4 * m + 1;
  bool fp32 = eps >= 1e-7;
  if (fp32) {
    const double sigma = bs3_sigma(eps);
    q.ker = KER_BS3;
    q.fp64 = false;
    q.nf_mu = fft_friendly((int)std::ceil(sigma * modes_mu));
    q.nf_r = q.nf_mu / 2;
    q.gA = {q.nf_mu, q.nf_mu / 4 - 1, q.nf_mu / 2 + 4};
    q.gB = {q.nf_r, q.nf_r / 4 - 1, q.nf_r / 2 + 4};
    size_t bytes = (size_t)((need_mu ? q.gA.G : 0) + (need_r ? q.gB.G : 0)) * 4;
    if (bytes > (size_t)smem_cap) fp32 = false;  // too large for one CTA: take the fp64 path
    else {
      q.smem_bytes = bytes;
      q.smem = true;
    }
  }
  if (!fp32) {
    // fp64 mode, first choice: septic B-spline (8 taps, weights by the Cox-de Boor recursion: no
    // transcendentals, no coefficient tables) at sigma with 2 (2 sigma - 1)^-8 ~ eps / 2, one
    // channel per pass so each grid may use all of a CTA's shared memory (64-bit fixed point,
    // 8 B per cell).  Falls back to the ES window when a grid does not fit (very small eps / large m).
    const double s7 = std::max(4.0, 0.5 * (std::pow(4.0 / std::max(eps, 1e-300), 0.125) + 1.0));
    const int nf7 = fft_friendly((int)std::ceil(s7 * modes_mu));
    const size_t bA = (size_t)(nf7 / 2 + 8) * 8, bB = (size_t)(nf7 / 4 + 8) * 8;
    const size_t need = std::max(need_mu ? bA : 0, need_r ? bB : 0);
    if (eps >= 1e-13 && need + 1024 <= (size_t)smem_cap) {
      q.ker = KER_BS7;
      q.fp64 = true;
      q.nf_mu = nf7;
      q.nf_r = nf7 / 2;
      q.gA = {q.nf_mu, q.nf_mu / 4 - 3, q.nf_mu / 2 + 8};
      q.gB = {q.nf_r, q.nf_r / 4 - 3, q.nf_r / 2 + 8};
      q.smem = true;
      q.smem_bytes = need;
      q.threads = 1024;
      q.ctas = sms * std::max(1, std::min(2, (int)((smem_cap + 1024) / (need + 1024))));
      *p = q;
      return FK_OK;
    }
  }
  if (!fp32) {
    q.ker = KER_ES;
    q.fp64 = true;
    int w = (int)std::ceil(std::log10(1.0 / eps)) + 2;
    w = std::min(16, std::max(4, w));
    q.es.w = w;
    q.es.beta = 2.30 * w;  // ES shape for sigma = 2
    q.nf_mu = fft_friendly(std::max(2 * modes_mu, 4 * w + 16));  // nf_r >= 2w + 8: tiles never wrap (small m)
    q.nf_r = q.nf_mu / 2;
    q.gA = {q.nf_mu, q.nf_mu / 4 - w / 2 - 2, q.nf_mu / 2 + w + 4};
    q.gB = {q.nf_r, q.nf_r / 4 - w / 2 - 2, q.nf_r / 2 + w + 4};
    size_t bytes = (size_t)((need_mu ? q.gA.G : 0) + (need_r ? q.gB.G : 0)) * 8;
    q.smem = bytes + (size_t)w * (w + 3) * 8 <= (size_t)smem_cap;  // + the Horner tap table
    q.smem_bytes = q.smem ? bytes : 0;
  }
  // launch shape: persistent CTAs, as many per SM as shared memory and 2048 threads allow
  q.threads = 1024;
  int per_sm = 2;
  if (q.smem && q.smem_bytes > 0) per_sm = std::max(1, std::min(2, (int)((smem_cap + 1024) / (q.smem_bytes + 1024))));
  if (!q.smem) per_sm = 2;
  q.ctas = sms * per_sm;
  *p = q;
  return FK_OK;
}

// ------------------------------------------------------------------------------------------
// ES window transform: psi(z) = exp(beta (sqrt(1 - z^2) - 1)), |z| <= 1, z = x / (w/2).
// psi-hat(k/nf) = int psi(2x/w) e^{-2 pi i k x / nf} dx = w int_0^1 psi(z) cos(pi k w z / nf) dz,
// by 96-point Gauss-Legendre on [0, 1].
// ------------------------------------------------------------------------------------------
struct GL96 {
  double x[96];
  double w[96];
};

static void gauss_legendre01(int n, double* x, double* w) {
  for (int i = 0; i < n; ++i) {
    double z = std::cos(3.14159265358979323846 * (i + 0.75) / (n + 0.5));
    double pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p1 = 1.0, p2 = 0.0;
      for (int j = 1; j <= n; ++j) {
        double p3 = p2;
        p2 = p1;
        p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
      }
      pp = n * (z * p1 - p2) / (z * z - 1.0);
      double z1 = z;
      z = z1 - p1 / pp;
      if (std::fabs(z - z1) < 1e-15) break;
    }
    x[i] = 0.5 * (1.0 - z);  // map [-1,1] -> [0,1]
    w[i] = 1.0 / ((1.0 - z * z) * pp * pp);  // = 2/((1-z^2)pp^2) * 1/2
  }
}

__global__ void k_es_phihat(GL96 gl, int w, double beta, int nf, int K, double* tab) {  // one warp per mode
  const int k = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (k > K) return;
  double s = 0.0;
  for (int i = lane; i < 96; i += 32) {
    const double z = gl.x[i];
    const double psi = exp(beta * (sqrt(1.0 - z * z) - 1.0));
    s += gl.w[i] * psi * cos(3.14159265358979323846 * (double)k * w * z / nf);
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) tab[k] = w * s;
}

fk_status es_phihat_table(const EsParams& es, int nf, int K, double* d_tab, cudaStream_t s) {
  static GL96 gl;
  static std::once_flag once;
  std::call_once(once, [] { gauss_legendre01(96, gl.x, gl.w); });
  k_es_phihat<<<(unsigned)(((int64_t)(K + 1) * 32 + 255) / 256), 256, 0, s>>>(gl, es.w, es.beta, nf, K, d_tab);
  count_launch();
  FK_CUDA_TRY(cudaGetLastError());
  return FK_OK;
}

// ------------------------------------------------------------------------------------------
// ES taps as polynomials (fp64 paths).  For a point at ul (cells), l0 = ceil(ul - w/2) and
// u = ul - l0 in (w/2 - 1, w/2]; with s = 2 (u - w/2 + 1) - 1 in (-1, 1] the tap i value
// psi((i - u) 2 / w) is a smooth function of s.  Chebyshev interpolation of degree P = w + 2 in
// long double, converted to monomials in s: max error ~1.5 exp(-beta) (the kink of psi at |z| = 1,
// i.e. 10^-w at beta = 2.3 w), two orders below the window's own aliasing error; |coefficients|
// sum to ~1.2 so Horner in fp64 loses nothing.  Replaces one exp + one sqrt per tap by P FMAs.
// Tables are built once per (device, w, beta) and kept in device memory.
// ------------------------------------------------------------------------------------------
static std::mutex g_horner_mu;
static std::map<std::tuple<int, int, long long>, double*> g_horner;

static std::mutex g_slot_mu;
static std::set<std::tuple<int, const void*, int>> g_slots;

fk_status horner_slot(const void* symbol, int w, double beta) {
  if (w < 1 || w >= kHornerSlots || w * (w + 3) > kHornerSlot || beta != 2.30 * w) return FK_E_UNSUPPORTED;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, symbol, w);
  {
    std::lock_guard<std::mutex> lk(g_slot_mu);
    if (g_slots.count(key)) return FK_OK;
  }
  const double* coef = nullptr;
  FK_TRY(es_horner_table(EsParams{w, beta}, &coef));
  // synchronous, once per (device, table, w): the first call of a shape (never inside a graph capture)
  FK_CUDA_TRY(cudaMemcpyToSymbol(symbol, coef, (size_t)w * (w + 3) * 8, (size_t)w * kHornerSlot * 8, cudaMemcpyDeviceToDevice));
  std::lock_guard<std::mutex> lk(g_slot_mu);
  g_slots.insert(key);
  return FK_OK;
}

fk_status es_horner_table(const EsParams& es, const double** d_coef) {
  int dev = 0;
  cudaGetDevice(&dev);
  long long bkey;
  std::memcpy(&bkey, &es.beta, sizeof bkey);
  auto key = std::make_tuple(dev, es.w, bkey);
  std::lock_guard<std::mutex> lk(g_horner_mu);
  auto it = g_horner.find(key);
  if (it != g_horner.end()) {
    *d_coef = it->second;
    return FK_OK;
  }
  const int w = es.w, P = es_horner_degree(w), np = P + 1;
  std::vector<double> coef((size_t)w * np);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int i = 0; i < w; ++i) {
    // values at the Chebyshev nodes
    std::vector<long double> fv(np), c(np, 0.0L);
    for (int k = 0; k < np; ++k) {
      const long double sk = cosl(pi * (k + 0.5L) / np);
      const long double u = (sk + 1.0L) / 2.0L + w / 2.0L - 1.0L;
      const long double z = (i - u) * 2.0L / w;
      const long double v = 1.0L - z * z;
      fv[k] = v > 0 ? expl((long double)es.beta * (sqrtl(v) - 1.0L)) : 0.0L;
    }
    for (int j = 0; j < np; ++j) {
      long double acc = 0;
      for (int k = 0; k < np; ++k) acc += fv[k] * cosl(pi * j * (k + 0.5L) / np);
      c[j] = acc * 2.0L / np;
    }
    c[0] /= 2.0L;
    // sum_j c_j T_j(s) -> monomials: T_0 = 1, T_1 = s, T_{j+1} = 2 s T_j - T_{j-1}
    std::vector<long double> mono(np, 0.0L), tm1(np, 0.0L), t0(np, 0.0L), t1(np, 0.0L);
    t0[0] = 1.0L;
    for (int j = 0; j < np; ++j) {
      const std::vector<long double>& T = (j == 0) ? t0 : t1;
      for (int q = 0; q < np; ++q) mono[q] += c[j] * T[q];
      if (j == 0) {
        t1.assign(np, 0.0L);
        t1[1 % np] = 1.0L;
        tm1 = t0;
        continue;
      }
      std::vector<long double> tn(np, 0.0L);
      for (int q = 0; q + 1 < np; ++q) tn[q + 1] += 2.0L * t1[q];
      for (int q = 0; q < np; ++q) tn[q] -= tm1[q];
      tm1 = t1;
      t1 = tn;
    }
    for (int q = 0; q < np; ++q) coef[(size_t)i * np + q] = (double)mono[q];
  }
  double* d = nullptr;
  FK_CUDA_TRY(cudaMalloc(&d, coef.size() * sizeof(double)));
  FK_CUDA_TRY(cudaMemcpy(d, coef.data(), coef.size() * sizeof(double), cudaMemcpyHostToDevice));
  g_horner[key] = d;
  *d_coef = d;
  return FK_OK;
}

// ------------------------------------------------------------------------------------------
// cuFFT plan cache.  Plans are created once per (device, rank, dims, batch, type) with
// auto-allocation off; each execution binds the caller's stream and workspace under a lock.
// ------------------------------------------------------------------------------------------
static std::mutex g_fft_mu;
static std::map<std::tuple<int, int, int, int, int, int>, FftPlan> g_fft_plans;

fk_status fft_plan(int rank, const int* dims, int batch, cufftType type, FftPlan* out) {
  int dev = 0;
  cudaGetDevice(&dev);
  auto key = std::make_tuple(dev, rank, dims[0], rank > 1 ? dims[1] : 0, batch, (int)type);
  std::lock_guard<std::mutex> lk(g_fft_mu);
  auto it = g_fft_plans.find(key);
  if (it != g_fft_plans.end()) {
    *out = it->second;
    return FK_OK;
  }
  FftPlan p;
  FK_CUFFT_TRY(cufftCreate(&p.h));
  FK_CUFFT_TRY(cufftSetAutoAllocation(p.h, 0));
  int n[2] = {dims[0], rank > 1 ? dims[1] : 0};
  size_t work = 0;
  FK_CUFFT_TRY(cufftMakePlanMany(p.h, rank, n, nullptr, 1, 0, nullptr, 1, 0, type, batch, &work));
  p.work = work;
  g_fft_plans[key] = p;
  *out = p;
  return FK_OK;
}

fk_status fft_exec_d2z(const FftPlan& p, double* in, cufftDoubleComplex* out, void* work, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_fft_mu);
  FK_CUFFT_TRY(cufftSetStream(p.h, s));
  FK_CUFFT_TRY(cufftSetWorkArea(p.h, work));
  FK_CUFFT_TRY(cufftExecD2Z(p.h, in, out));
  return FK_OK;
}

fk_status fft_exec_z2d(const FftPlan& p, cufftDoubleComplex* in, double* out, void* work, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_fft_mu);
  FK_CUFFT_TRY(cufftSetStream(p.h, s));
  FK_CUFFT_TRY(cufftSetWorkArea(p.h, work));
  FK_CUFFT_TRY(cufftExecZ2D(p.h, in, out));
  return FK_OK;
}

}  // namespace fk

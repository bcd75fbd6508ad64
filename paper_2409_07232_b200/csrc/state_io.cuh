// state_io.cuh -- CBSNAP01 state snapshots and the GPU digit-agreement comparator
// (diffwrf-style validation of whole GridStates at C5 scale).
//
// Included by fsbm_coal.cu after the error plumbing (fail / FSBM_CUDA_TRY).
//
//  * fsbm_snapshot_write / _read_header / _read: the reference's CBSNAP01 format
//    (snapshot.hpp:8-17, snapshot.cpp:46-135) byte for byte, with its validation order
//    and messages (ConfigError -> FSBM_CONFIG).  Plain host I/O: the file holds the
//    GridState exactly as the step consumes it.
//  * fsbm_compare_states_device: compare_states (verify.cpp:65-80) over two device-resident
//    states: one launch, blockIdx.y = field (mass_grid, temperature, pressure, 6 categories),
//    each element's digit_agreement (verify.cpp:12-26) reduced to min / sum / exact count.
//    HBM-bound: 2 x 8 bytes read per compared value, nothing written.
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

namespace fsbm {

constexpr int kNumFields = 3 + kNCat; // mass_grid, temperature, pressure, 6 categories
static const char *const kCategoryNames[kNCat] = {"liquid", "ice1", "ice2", "ice3", "snow", "graupel"};

/// digit_agreement (verify.cpp:12-26), same operation order; returns -1 on non-finite.
__device__ __forceinline__ int digit_agreement_dev(double a, double b) {
    if (!isfinite(a) || !isfinite(b)) return -1;
    if (a == b) return 16;
    if (a + b == 0.0) return 0;
    const double rel = __ddiv_rn(__dmul_rn(2.0, fabs(__dsub_rn(a, b))), __dadd_rn(fabs(a), fabs(b)));
    const double digits = floor(-log10(rel));
    if (digits < 0.0) return 0;
    if (digits > 16.0) return 16;
    return static_cast<int>(digits);
}

struct CompareArgs {
    const double *a[kNumFields], *b[kNumFields];
    size_t n[kNumFields];
    unsigned long long *acc; // [field][4]: min digits, digit sum, exact count, non-finite flag
};

__global__ void __launch_bounds__(256) compare_fields_kernel(CompareArgs C) {
    const int f = blockIdx.y;
    const double *__restrict__ a = C.a[f], *__restrict__ b = C.b[f];
    const size_t n = C.n[f];
    int dmin = 16;
    unsigned long long sum = 0, exact = 0, bad = 0;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int d = digit_agreement_dev(__ldg(a + i), __ldg(b + i));
        if (d < 0) {
            bad = 1;
            continue;
        }
        dmin = min(dmin, d);
        sum += static_cast<unsigned long long>(d);
        exact += d == 16;
    }
    for (int o = 16; o > 0; o >>= 1) {
        dmin = min(dmin, __shfl_down_sync(0xffffffffu, dmin, o));
        sum += __shfl_down_sync(0xffffffffu, sum, o);
        exact += __shfl_down_sync(0xffffffffu, exact, o);
        bad |= __shfl_down_sync(0xffffffffu, bad, o);
    }
    __shared__ int s_min[8];
    __shared__ unsigned long long s_sum[8], s_ex[8], s_bad[8];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_min[w] = dmin;
        s_sum[w] = sum;
        s_ex[w] = exact;
        s_bad[w] = bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) {
            dmin = min(dmin, s_min[k]);
            sum += s_sum[k];
            exact += s_ex[k];
            bad |= s_bad[k];
        }
        unsigned long long *acc = C.acc + 4 * f;
        atomicMin(acc, static_cast<unsigned long long>(dmin));
        atomicAdd(acc + 1, sum);
        atomicAdd(acc + 2, exact);
        if (bad) atomicOr(acc + 3, 1ull);
    }
}

} // namespace fsbm

namespace {

constexpr char kSnapMagic[8] = {'C', 'B', 'S', 'N', 'A', 'P', '0', '1'};
constexpr uint32_t kSnapVersion = 1;

struct SnapFile {
    FILE *f = nullptr;
    ~SnapFile() {
        if (f) fclose(f);
    }
};

bool snap_put(FILE *f, const void *p, size_t bytes) { return bytes == 0 || fwrite(p, 1, bytes, f) == bytes; }

/// get() of snapshot.cpp:29-33: a short read is "truncated while reading <what>"
int snap_get(FILE *f, void *p, size_t bytes, const char *what) {
    if (bytes && fread(p, 1, bytes, f) != bytes)
        return fail(FSBM_CONFIG, std::string("snapshot: truncated while reading ") + what);
    return FSBM_OK;
}

struct SnapHeader {
    uint32_t nkr = 0;
    fsbm_ranges r{};
    double ratio = 0.0;
};

/// read_snapshot's header checks (snapshot.cpp:75-116), in the reference's order.
int snap_read_header(FILE *f, const std::string &path, SnapHeader &h) {
    char magic[8];
    if (int st = snap_get(f, magic, 8, "magic")) return st;
    if (std::memcmp(magic, kSnapMagic, 8) != 0)
        return fail(FSBM_CONFIG, "snapshot: '" + path + "' is not a coalbench snapshot");
    uint32_t version = 0;
    if (int st = snap_get(f, &version, 4, "version")) return st;
    if (version != kSnapVersion) return fail(FSBM_CONFIG, "snapshot: unsupported version in '" + path + "'");
    if (int st = snap_get(f, &h.nkr, 4, "nkr")) return st;
    if (h.nkr < 2 || h.nkr > 100000) return fail(FSBM_CONFIG, "snapshot: implausible nkr");
    int32_t v[6];
    static const char *names[6] = {"ids", "ide", "kds", "kde", "jds", "jde"};
    for (int q = 0; q < 6; ++q)
        if (int st = snap_get(f, &v[q], 4, names[q])) return st;
    h.r = fsbm_ranges{v[0], v[1], v[2], v[3], v[4], v[5]};
    if (h.r.ide < h.r.ids || h.r.kde < h.r.kds || h.r.jde < h.r.jds)
        return fail(FSBM_CONFIG, "snapshot: invalid domain ranges");
    if (int st = snap_get(f, &h.ratio, 8, "ratio")) return st;
    uint32_t ncat = 0;
    if (int st = snap_get(f, &ncat, 4, "category count")) return st;
    if (ncat != FSBM_NCAT)
        return fail(FSBM_CONFIG, "snapshot: expected " + std::to_string(FSBM_NCAT) + " categories, found " +
                                     std::to_string(ncat));
    for (int c = 0; c < FSBM_NCAT; ++c) {
        uint32_t len = 0;
        if (int st = snap_get(f, &len, 4, "category name length")) return st;
        if (len > 64) return fail(FSBM_CONFIG, "snapshot: implausible category name");
        std::string name(len, '\0');
        if (int st = snap_get(f, name.data(), len, "category name")) return st;
        if (name != fsbm::kCategoryNames[c]) return fail(FSBM_CONFIG, "snapshot: unexpected category '" + name + "'");
    }
    return FSBM_OK;
}

size_t snap_npoints(const fsbm_ranges &r) {
    return static_cast<size_t>(r.ide - r.ids + 1) * (r.kde - r.kds + 1) * (r.jde - r.jds + 1);
}

} // namespace

extern "C" {

int fsbm_snapshot_write(const char *path, fsbm_ranges r, int nkr, double ratio, const double *x,
                        const double *temperature, const double *pressure,
                        const double *const bins[FSBM_NCAT]) {
    if (!path) return fail(FSBM_DOMAIN, "snapshot: null path");
    if (nkr < 2) return fail(FSBM_SHAPE, "snapshot: nkr must be >= 2");
    if (r.ide < r.ids || r.kde < r.kds || r.jde < r.jds) return fail(FSBM_SHAPE, "snapshot: invalid domain ranges");
    const size_t np = snap_npoints(r);
    if (!x || (np && (!temperature || !pressure))) return fail(FSBM_DOMAIN, "snapshot: null state array");
    for (int c = 0; c < FSBM_NCAT; ++c)
        if (np && !bins[c]) return fail(FSBM_DOMAIN, "snapshot: null category array");
    SnapFile sf;
    sf.f = fopen(path, "wb");
    if (!sf.f) return fail(FSBM_CONFIG, std::string("snapshot: cannot open '") + path + "' for writing");
    bool ok = snap_put(sf.f, kSnapMagic, 8);
    const uint32_t hdr[2] = {kSnapVersion, static_cast<uint32_t>(nkr)};
    const int32_t ext[6] = {r.ids, r.ide, r.kds, r.kde, r.jds, r.jde};
    const uint32_t ncat = FSBM_NCAT;
    ok = ok && snap_put(sf.f, hdr, 8) && snap_put(sf.f, ext, 24) && snap_put(sf.f, &ratio, 8) &&
         snap_put(sf.f, &ncat, 4);
    for (int c = 0; c < FSBM_NCAT && ok; ++c) {
        const uint32_t len = static_cast<uint32_t>(std::strlen(fsbm::kCategoryNames[c]));
        ok = snap_put(sf.f, &len, 4) && snap_put(sf.f, fsbm::kCategoryNames[c], len);
    }
    ok = ok && snap_put(sf.f, x, nkr * sizeof(double)) && snap_put(sf.f, temperature, np * sizeof(double)) &&
         snap_put(sf.f, pressure, np * sizeof(double));
    for (int c = 0; c < FSBM_NCAT && ok; ++c) ok = snap_put(sf.f, bins[c], np * nkr * sizeof(double));
    ok = ok && fflush(sf.f) == 0;
    if (!ok) return fail(FSBM_CONFIG, std::string("snapshot: write to '") + path + "' failed");
    return FSBM_OK;
}

int fsbm_snapshot_read_header(const char *path, fsbm_ranges *ranges, int *nkr, double *ratio) {
    if (!path) return fail(FSBM_DOMAIN, "snapshot: null path");
    SnapFile sf;
    sf.f = fopen(path, "rb");
    if (!sf.f) return fail(FSBM_CONFIG, std::string("snapshot: cannot open '") + path + "'");
    SnapHeader h;
    if (int st = snap_read_header(sf.f, path, h)) return st;
    if (ranges) *ranges = h.r;
    if (nkr) *nkr = static_cast<int>(h.nkr);
    if (ratio) *ratio = h.ratio;
    return FSBM_OK;
}

int fsbm_snapshot_read(const char *path, double *x, double *temperature, double *pressure,
                       double *const bins[FSBM_NCAT]) {
    if (!path) return fail(FSBM_DOMAIN, "snapshot: null path");
    SnapFile sf;
    sf.f = fopen(path, "rb");
    if (!sf.f) return fail(FSBM_CONFIG, std::string("snapshot: cannot open '") + path + "'");
    SnapHeader h;
    if (int st = snap_read_header(sf.f, path, h)) return st;
    const size_t np = snap_npoints(h.r);
    if (!x || (np && (!temperature || !pressure))) return fail(FSBM_DOMAIN, "snapshot: null destination array");
    if (int st = snap_get(sf.f, x, h.nkr * sizeof(double), "mass grid")) return st;
    if (int st = snap_get(sf.f, temperature, np * sizeof(double), "temperature")) return st;
    if (int st = snap_get(sf.f, pressure, np * sizeof(double), "pressure")) return st;
    for (int c = 0; c < FSBM_NCAT; ++c) {
        if (np && !bins[c]) return fail(FSBM_DOMAIN, "snapshot: null destination array");
        if (int st = snap_get(sf.f, bins[c], np * h.nkr * sizeof(double), "bins")) return st;
    }
    char extra;
    if (fread(&extra, 1, 1, sf.f) != 0 || !feof(sf.f))
        return fail(FSBM_CONFIG, std::string("snapshot: trailing bytes in '") + path + "'");
    return FSBM_OK;
}

int fsbm_compare_states_device(int device, size_t npoints, int nkr, const double *x_a,
                               const double *temperature_a, const double *pressure_a,
                               const double *const bins_a[FSBM_NCAT], const double *x_b,
                               const double *temperature_b, const double *pressure_b,
                               const double *const bins_b[FSBM_NCAT], fsbm_field_diff *out,
                               void *stream) {
    if (!out) return fail(FSBM_DOMAIN, "compare_states: null report");
    if (nkr < 1) return fail(FSBM_SHAPE, "compare_states: nkr must be >= 1");
    DeviceGuard dg(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    fsbm::CompareArgs C{};
    const double *A[fsbm::kNumFields] = {x_a, temperature_a, pressure_a};
    const double *B[fsbm::kNumFields] = {x_b, temperature_b, pressure_b};
    size_t N[fsbm::kNumFields] = {static_cast<size_t>(nkr), npoints, npoints};
    for (int c = 0; c < FSBM_NCAT; ++c) {
        A[3 + c] = bins_a[c];
        B[3 + c] = bins_b[c];
        N[3 + c] = npoints * nkr;
    }
    for (int f = 0; f < fsbm::kNumFields; ++f) {
        if (N[f] && (!A[f] || !B[f])) return fail(FSBM_DOMAIN, "compare_states: null field array");
        C.a[f] = A[f];
        C.b[f] = B[f];
        C.n[f] = N[f];
    }
    unsigned long long *acc = nullptr;
    FSBM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&acc), sizeof(unsigned long long) * 4 * fsbm::kNumFields, s));
    unsigned long long init[4 * fsbm::kNumFields];
    for (int f = 0; f < fsbm::kNumFields; ++f) {
        init[4 * f] = 16;
        init[4 * f + 1] = init[4 * f + 2] = init[4 * f + 3] = 0;
    }
    FSBM_CUDA_TRY(cudaMemcpyAsync(acc, init, sizeof(init), cudaMemcpyHostToDevice, s));
    C.acc = acc;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const dim3 grid(static_cast<unsigned>(sms * 4), fsbm::kNumFields);
    fsbm::compare_fields_kernel<<<grid, 256, 0, s>>>(C);
    FSBM_CUDA_TRY(cudaGetLastError());
    unsigned long long h[4 * fsbm::kNumFields];
    FSBM_CUDA_TRY(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, s));
    FSBM_CUDA_TRY(cudaFreeAsync(acc, s));
    FSBM_CUDA_TRY(cudaStreamSynchronize(s));
    for (int f = 0; f < fsbm::kNumFields; ++f)
        if (h[4 * f + 3]) return fail(FSBM_DOMAIN, "digit_agreement: inputs must be finite");
    for (int f = 0; f < fsbm::kNumFields; ++f) {
        fsbm_field_diff &d = out[f];
        d.count_compared = N[f];
        d.min_digits = N[f] ? static_cast<int>(h[4 * f]) : 16;
        d.count_exact = h[4 * f + 2];
        d.mean_digits = N[f] ? static_cast<double>(h[4 * f + 1]) / static_cast<double>(N[f]) : 16.0;
    }
    return FSBM_OK;
}

} // extern "C"

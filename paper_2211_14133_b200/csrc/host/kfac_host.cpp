// C++ value-semantics K-FAC API (include/pipefill/kfac/{matrix,kfac}.hpp) on
// top of the C-ABI (include/pf_kfac.h).  Every K-FAC computation —
// curvature factors, damped inverses, preconditioning and the NGD update —
// runs on the B200; this file only converts between the reference's FP64
// row-major Matrix and device buffers (bf16 tapes, fp32 factors/inverses),
// validates shapes the way the reference does, and turns pf_status codes
// into the reference's exception types.
//
// Reference: proj/src/kfac/matrix.cpp, proj/src/kfac/kfac.cpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "pf_kfac.h"
#include "pf_sched.h"
#include "pipefill/kfac/kfac.hpp"
#include "pipefill/kfac/matrix.hpp"

namespace pipefill::kfac {
namespace {

constexpr std::size_t kMaterializeGuard = std::size_t{1} << 22;  // reference matrix.cpp:11

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// pf_status -> the reference's exception types
void pf_check(int rc, const char* what) {
    if (rc == PF_OK) return;
    const std::string msg = std::string(what) + ": " + pf_last_error();
    switch (rc) {
        case PF_BAD_SHAPE:
        case PF_BAD_ARG: throw std::invalid_argument(msg);
        case PF_NOT_PD: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

void require_device() {
    static const bool ok = pf_device_ok() != 0;
    if (!ok) throw std::runtime_error("pipefill::kfac: no usable sm_100 (B200) device; there is no CPU path");
}

// Caller-owned device allocation (the C-ABI never allocates).
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(std::size_t bytes) {
        if (bytes) cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
    DevBuf& operator=(DevBuf&&) = delete;
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

cudaStream_t stream() { return cudaStreamPerThread; }
void sync() { cuda_check(cudaStreamSynchronize(stream()), "cudaStreamSynchronize"); }

int round_up(int x, int m) { return (x + m - 1) / m * m; }

uint16_t to_bf16(double v) {  // round-to-nearest-even via fp32
    const float f = static_cast<float>(v);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

// A d x n tape (examples as columns) as a device bf16 [d x ld] operand.
struct DevTape {
    int d = 0, n = 0, ld = 0;
    DevBuf buf;
    explicit DevTape(const Matrix& m)
        : d(m.rows()), n(m.cols()), ld(round_up(std::max(m.cols(), 1), 8)),
          buf(static_cast<std::size_t>(m.rows()) * round_up(std::max(m.cols(), 1), 8) * 2) {
        std::vector<uint16_t> h(static_cast<std::size_t>(d) * ld, 0);
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < n; ++c) h[static_cast<std::size_t>(r) * ld + c] = to_bf16(m(r, c));
        cuda_check(cudaMemcpyAsync(buf.p, h.data(), h.size() * 2, cudaMemcpyHostToDevice, stream()),
                   "upload tape");
    }
};

// fp32 device copy of a Matrix, row pitch `ld` elements (16-byte rows).
struct DevMat {
    int rows = 0, cols = 0, ld = 0;
    DevBuf buf;
    DevMat(int r, int c)
        : rows(r), cols(c), ld(round_up(std::max(c, 1), 4)),
          buf(static_cast<std::size_t>(std::max(r, 1)) * round_up(std::max(c, 1), 4) * 4) {}
    explicit DevMat(const Matrix& m) : DevMat(m.rows(), m.cols()) { upload(m); }
    void upload(const Matrix& m) {
        std::vector<float> h(static_cast<std::size_t>(rows) * ld, 0.0f);
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) h[static_cast<std::size_t>(r) * ld + c] = static_cast<float>(m(r, c));
        cuda_check(cudaMemcpyAsync(buf.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice, stream()),
                   "upload matrix");
    }
    // Requires a prior sync() when the producer is asynchronous.
    Matrix download() const {
        std::vector<float> h(static_cast<std::size_t>(rows) * ld);
        cuda_check(cudaMemcpyAsync(h.data(), buf.p, h.size() * 4, cudaMemcpyDeviceToHost, stream()),
                   "download matrix");
        sync();
        Matrix out(rows, cols);
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) out(r, c) = h[static_cast<std::size_t>(r) * ld + c];
        return out;
    }
    float* f() const { return buf.as<float>(); }
};

void require_square(const Matrix& m, const char* what) {  // reference matrix.cpp:13-15
    if (m.rows() != m.cols()) throw std::invalid_argument(std::string(what) + ": matrix not square");
}

// Grouped SYRK of (a_l, e_l) for the given layers -> full symmetric factors.
std::vector<std::pair<Matrix, Matrix>> factors_for(const BatchTape& tape, const std::vector<int>& layers) {
    require_device();
    const float scale = static_cast<float>(1.0 / tape.batch_size);
    std::vector<DevTape> tapes;
    std::vector<DevMat> outs;
    tapes.reserve(2 * layers.size());
    outs.reserve(2 * layers.size());
    for (int l : layers) {
        for (const Matrix* m : {&tape.layer_inputs.at(l), &tape.layer_errors.at(l)}) {
            tapes.emplace_back(*m);
            outs.emplace_back(m->rows(), m->rows());
        }
    }
    std::vector<pf_syrk_problem> probs;
    for (std::size_t i = 0; i < tapes.size(); ++i) {
        if (tapes[i].d == 0) continue;
        if (tapes[i].n == 0) {  // empty batch: zero factor
            cuda_check(cudaMemsetAsync(outs[i].buf.p, 0, static_cast<std::size_t>(outs[i].rows) * outs[i].ld * 4,
                                       stream()), "memset");
            continue;
        }
        probs.push_back(pf_syrk_problem{tapes[i].buf.p, outs[i].f(), tapes[i].d, tapes[i].n, tapes[i].ld,
                                        outs[i].ld, scale, 0, 0});
    }
    if (!probs.empty())
        pf_check(pf_curvature_syrk_grouped(probs.data(), static_cast<int>(probs.size()), 1, stream()),
                 "curvature_factors");
    sync();
    std::vector<std::pair<Matrix, Matrix>> res;
    for (std::size_t i = 0; i < layers.size(); ++i)
        res.emplace_back(outs[2 * i].download(), outs[2 * i + 1].download());
    return res;
}

// Batched damped inverses (one call); throws the reference's domain_error on
// the first failing matrix.
std::vector<Matrix> inverses_of(const std::vector<const Matrix*>& ms, double damping) {
    require_device();
    std::vector<DevMat> in, out;
    std::vector<std::size_t> ws_off;
    std::size_t ws_total = 0;
    in.reserve(ms.size());
    out.reserve(ms.size());
    for (const Matrix* m : ms) {
        require_square(*m, "cholesky_spd_inverse");
        in.emplace_back(*m);
        out.emplace_back(m->rows(), m->rows());
        std::size_t b = 0;
        pf_check(pf_damped_inverse_workspace(std::max(m->rows(), 1), &b), "inverse workspace");
        ws_off.push_back(ws_total);
        ws_total += (b + 255) / 256 * 256;
    }
    DevBuf ws(std::max<std::size_t>(ws_total, 256));
    DevBuf info(4 * std::max<std::size_t>(ms.size(), 1));
    std::vector<pf_inverse_problem> probs;
    for (std::size_t i = 0; i < ms.size(); ++i) {
        if (ms[i]->rows() == 0) continue;
        probs.push_back(pf_inverse_problem{in[i].f(), out[i].f(), nullptr, in[i].rows, in[i].ld, out[i].ld,
                                           static_cast<float>(damping),
                                           static_cast<char*>(ws.p) + ws_off[i], info.as<int>() + i});
    }
    if (!probs.empty())
        pf_check(pf_damped_inverse_batched(probs.data(), static_cast<int>(probs.size()), stream()),
                 "cholesky_spd_inverse");
    std::vector<int> bad(ms.size(), 0);
    sync();
    if (!ms.empty())
        cuda_check(cudaMemcpy(bad.data(), info.p, 4 * ms.size(), cudaMemcpyDeviceToHost), "download info");
    for (std::size_t i = 0; i < ms.size(); ++i)
        if (ms[i]->rows() > 0 && bad[i] != 0)  // reference matrix.cpp:124-125
            throw std::domain_error("cholesky: matrix not positive definite (damping too small?)");
    std::vector<Matrix> res;
    for (std::size_t i = 0; i < ms.size(); ++i) res.push_back(ms[i]->rows() ? out[i].download() : Matrix());
    return res;
}

}  // namespace

// ------------------------------------------------------------------ Matrix
Matrix::Matrix(std::initializer_list<std::initializer_list<double>> rows) {
    rows_ = static_cast<int>(rows.size());
    cols_ = rows_ ? static_cast<int>(rows.begin()->size()) : 0;
    data_.reserve(static_cast<std::size_t>(rows_) * cols_);
    for (const auto& r : rows) {
        if (static_cast<int>(r.size()) != cols_) throw std::invalid_argument("ragged initializer");
        data_.insert(data_.end(), r.begin(), r.end());
    }
}

Matrix Matrix::identity(int n) {
    Matrix m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
}

Matrix Matrix::transposed() const {
    Matrix t(cols_, rows_);
    for (int r = 0; r < rows_; ++r)
        for (int c = 0; c < cols_; ++c) t(c, r) = (*this)(r, c);
    return t;
}

Matrix Matrix::scaled(double s) const {
    Matrix out = *this;
    for (double& v : out.data_) v *= s;
    return out;
}

double Matrix::max_abs() const {
    double m = 0.0;
    for (double v : data_) m = std::max(m, std::fabs(v));
    return m;
}

// ------------------------------------------------------------------ host container utilities
Matrix matmul(const Matrix& a, const Matrix& b) {
    if (a.cols() != b.rows()) throw std::invalid_argument("matmul: shape mismatch");
    Matrix out(a.rows(), b.cols());
    for (int i = 0; i < a.rows(); ++i)
        for (int k = 0; k < a.cols(); ++k) {
            const double v = a(i, k);
            for (int j = 0; j < b.cols(); ++j) out(i, j) += v * b(k, j);
        }
    return out;
}

Matrix add(const Matrix& a, const Matrix& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) throw std::invalid_argument("add: shape mismatch");
    Matrix out = a;
    for (std::size_t i = 0; i < out.data().size(); ++i) out.data()[i] += b.data()[i];
    return out;
}

Matrix subtract(const Matrix& a, const Matrix& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) throw std::invalid_argument("subtract: shape mismatch");
    Matrix out = a;
    for (std::size_t i = 0; i < out.data().size(); ++i) out.data()[i] -= b.data()[i];
    return out;
}

double max_abs_diff(const Matrix& a, const Matrix& b) { return subtract(a, b).max_abs(); }

std::vector<double> vec(const Matrix& m) {
    std::vector<double> v;
    v.reserve(m.data().size());
    for (int c = 0; c < m.cols(); ++c)
        for (int r = 0; r < m.rows(); ++r) v.push_back(m(r, c));
    return v;
}

Matrix unvec(const std::vector<double>& v, int rows, int cols) {
    if (static_cast<std::size_t>(rows) * cols != v.size()) throw std::invalid_argument("unvec: size mismatch");
    Matrix m(rows, cols);
    for (int c = 0; c < cols; ++c)
        for (int r = 0; r < rows; ++r) m(r, c) = v[static_cast<std::size_t>(c) * rows + r];
    return m;
}

Matrix kron(const Matrix& a, const Matrix& b) {
    const std::size_t entries = static_cast<std::size_t>(a.rows()) * b.rows() * a.cols() * b.cols();
    if (entries > kMaterializeGuard) throw std::length_error("kron: result too large");
    Matrix out(a.rows() * b.rows(), a.cols() * b.cols());
    for (int i = 0; i < a.rows(); ++i)
        for (int j = 0; j < a.cols(); ++j)
            for (int k = 0; k < b.rows(); ++k)
                for (int l = 0; l < b.cols(); ++l) out(i * b.rows() + k, j * b.cols() + l) = a(i, j) * b(k, l);
    return out;
}

// Reference matrix.cpp:117-134, on the GPU: pf_cholesky_factor (the damped
// inverse's right-looking factorisation, fp32-accurate), damping 0.
Matrix cholesky_factor(const Matrix& m) {
    require_square(m, "cholesky_factor");
    const int n = m.rows();
    if (n == 0) return Matrix();
    require_device();
    DevMat in(m), out(n, n);
    std::size_t wsb = 0;
    pf_check(pf_damped_inverse_workspace(n, &wsb), "cholesky workspace");
    DevBuf ws(wsb), info(4);
    pf_check(pf_cholesky_factor(in.f(), n, in.ld, 0.0f, out.f(), out.ld, ws.p, wsb, info.as<int>(), stream()),
             "cholesky_factor");
    int bad = 0;
    sync();
    cuda_check(cudaMemcpy(&bad, info.p, 4, cudaMemcpyDeviceToHost), "download info");
    if (bad != 0)  // reference matrix.cpp:124-125
        throw std::domain_error("cholesky: matrix not positive definite (damping too small?)");
    return out.download();
}

std::vector<double> solve_spd(const Matrix& m, const std::vector<double>& rhs) {
    if (static_cast<int>(rhs.size()) != m.rows()) throw std::invalid_argument("solve_spd: rhs size mismatch");
    const Matrix l = cholesky_factor(m);
    const int n = m.rows();
    std::vector<double> y(rhs);
    for (int i = 0; i < n; ++i) {
        for (int k = 0; k < i; ++k) y[i] -= l(i, k) * y[k];
        y[i] /= l(i, i);
    }
    for (int i = n - 1; i >= 0; --i) {
        for (int k = i + 1; k < n; ++k) y[i] -= l(k, i) * y[k];
        y[i] /= l(i, i);
    }
    return y;
}

// ------------------------------------------------------------------ K-FAC path (B200)
Matrix cholesky_spd_inverse(const Matrix& m, double damping) {
    require_square(m, "cholesky_spd_inverse");
    if (m.rows() == 0) return Matrix();
    return inverses_of({&m}, damping).front();
}

std::pair<Matrix, Matrix> curvature_factors(const BatchTape& tape, int layer) {
    return factors_for(tape, {layer}).front();
}

Matrix precondition(const Matrix& grad, const Matrix& a_inv, const Matrix& b_inv) {
    if (b_inv.cols() != grad.rows() || grad.cols() != a_inv.rows())  // reference kfac.cpp:134-135
        throw std::invalid_argument("precondition: shape mismatch");
    require_device();
    const int d_out = grad.rows(), d_in = grad.cols();
    if (d_out == 0 || d_in == 0) return Matrix(d_out, d_in);
    // The C-ABI takes dense row-major operands (ld = d); pack exactly.
    auto dense = [](const Matrix& m) {
        DevBuf b(static_cast<std::size_t>(m.rows()) * m.cols() * 4);
        std::vector<float> h(m.data().begin(), m.data().end());
        cuda_check(cudaMemcpyAsync(b.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice, stream()), "upload");
        return b;
    };
    DevBuf g = dense(grad), ai = dense(a_inv), bi = dense(b_inv);
    DevBuf p(static_cast<std::size_t>(d_out) * d_in * 4);
    std::size_t wsb = 0;
    pf_check(pf_precondition_workspace(d_out, d_in, &wsb), "precondition workspace");
    DevBuf ws(wsb);
    pf_check(pf_precondition(bi.as<float>(), g.as<float>(), ai.as<float>(), p.as<float>(), d_out, d_in, ws.p, wsb,
                             stream()),
             "precondition");
    std::vector<float> h(static_cast<std::size_t>(d_out) * d_in);
    cuda_check(cudaMemcpyAsync(h.data(), p.p, h.size() * 4, cudaMemcpyDeviceToHost, stream()), "download");
    sync();
    Matrix out(d_out, d_in);
    std::copy(h.begin(), h.end(), out.data().begin());
    return out;
}

KfacState::KfacState(int layers)
    : factor_a(layers), factor_b(layers), inv_a(layers), inv_b(layers), staleness(layers, 0),
      refreshed_this_step(layers, 0) {}

bool KfacState::has_inverses(int layer) const {
    return inv_a.at(layer).rows() > 0 && inv_b.at(layer).rows() > 0;
}

void KfacState::update_factors(const BatchTape& tape) {
    std::vector<int> layers(factor_a.size());
    for (std::size_t l = 0; l < layers.size(); ++l) layers[l] = static_cast<int>(l);
    auto f = factors_for(tape, layers);  // one grouped SYRK launch over every layer
    for (std::size_t l = 0; l < layers.size(); ++l) {
        factor_a[l] = std::move(f[l].first);
        factor_b[l] = std::move(f[l].second);
    }
}

void KfacState::refresh_inverses() {
    std::vector<const Matrix*> ms;
    std::vector<int> which;
    for (std::size_t l = 0; l < factor_a.size(); ++l) {
        if (factor_a[l].rows() == 0) continue;
        ms.push_back(&factor_a[l]);
        ms.push_back(&factor_b[l]);
        which.push_back(static_cast<int>(l));
    }
    auto inv = inverses_of(ms, damping);  // one batched call
    for (std::size_t i = 0; i < which.size(); ++i) {
        const int l = which[i];
        inv_a[l] = std::move(inv[2 * i]);
        inv_b[l] = std::move(inv[2 * i + 1]);
        staleness[l] = 0;
        refreshed_this_step[l] = 1;
    }
}

NgdStepResult ngd_step(TinyMlp& mlp, KfacState& state, const std::vector<Matrix>& gradients) {
    if (gradients.size() != mlp.weights.size()) throw std::invalid_argument("one gradient per layer required");
    NgdStepResult out;
    const int layers = static_cast<int>(mlp.weights.size());
    for (int l = 0; l < layers; ++l) {
        Matrix& w = mlp.weights[l];
        const Matrix& g = gradients[l];
        if (state.has_inverses(l)) {
            const Matrix& ai = state.inv_a[l];
            const Matrix& bi = state.inv_b[l];
            if (bi.cols() != g.rows() || g.cols() != ai.rows() || w.rows() != g.rows() || w.cols() != g.cols())
                throw std::invalid_argument("precondition: shape mismatch");
            require_device();
            const int d_out = g.rows(), d_in = g.cols();
            auto dense = [](const Matrix& m) {
                DevBuf b(static_cast<std::size_t>(m.rows()) * m.cols() * 4);
                std::vector<float> h(m.data().begin(), m.data().end());
                cuda_check(cudaMemcpyAsync(b.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice, stream()), "upload");
                return b;
            };
            DevBuf dw = dense(w), dg = dense(g), dai = dense(ai), dbi = dense(bi);
            std::size_t wsb = 0;
            pf_check(pf_precondition_workspace(d_out, d_in, &wsb), "precondition workspace");
            DevBuf ws(wsb);
            // W -= eta * B^-1 G A^-1 in the second GEMM's epilogue
            pf_check(pf_precondition_update(dbi.as<float>(), dg.as<float>(), dai.as<float>(), dw.as<float>(), d_out,
                                            d_in, static_cast<float>(state.learning_rate), ws.p, wsb, stream()),
                     "ngd_step");
            std::vector<float> h(static_cast<std::size_t>(d_out) * d_in);
            cuda_check(cudaMemcpyAsync(h.data(), dw.p, h.size() * 4, cudaMemcpyDeviceToHost, stream()), "download");
            sync();
            std::copy(h.begin(), h.end(), w.data().begin());
        } else {
            // first-ever step of a layer: the plain gradient (reference kfac.cpp:190-195)
            out.used_plain_gradient = true;
            w = subtract(w, g.scaled(state.learning_rate));
        }
        state.staleness[l] = (state.refreshed_this_step[l] ? 0 : state.staleness[l]) + 1;
        state.refreshed_this_step[l] = 0;
    }
    return out;
}

std::vector<Matrix> block_diag_split_factor(const Matrix& m, int k) {
    if (m.rows() != m.cols()) throw std::invalid_argument("factor must be square");
    if (k < 1 || m.rows() % k != 0) throw std::invalid_argument("K must divide the factor dimension");
    const int bs = m.rows() / k;
    std::vector<Matrix> blocks(static_cast<std::size_t>(k), Matrix(bs, bs));
    for (int i = 0; i < m.rows(); ++i) {  // row i lands in block i / bs
        const auto src = m.data().begin() + static_cast<std::ptrdiff_t>(i) * m.cols() + (i / bs) * bs;
        std::copy(src, src + bs, blocks[i / bs].data().begin() + static_cast<std::ptrdiff_t>(i % bs) * bs);
    }
    return blocks;
}

double inversion_flops(int dim) { return (2.0 / 3.0) * static_cast<double>(dim) * dim * dim; }

double block_diag_inversion_flops(int dim, int k) {
    if (k < 1 || dim % k != 0) throw std::invalid_argument("K must divide the dimension");
    return k * inversion_flops(dim / k);
}

std::uint64_t SplitMix64::next() {
    state += 0x9e3779b97f4a7c15ULL;
    std::uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

double SplitMix64::uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
double SplitMix64::symmetric() { return 2.0 * uniform() - 1.0; }

}  // namespace pipefill::kfac

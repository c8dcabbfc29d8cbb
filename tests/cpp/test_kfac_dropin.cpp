// Reference-style assertions (proj/tests/test_kfac.cpp:99-205, :275-330),
// compiled against THIS repo's include/pipefill/kfac headers and linked
// against libpf_b200.so: the same source a reference caller writes, now
// running its K-FAC calls on the B200.  Tolerances are the fp32-accurate
// ones of DESIGN.md §4 instead of the reference's FP64 1e-15.
//
// Needs an sm_100 device.  Prints "ALL PASS" and exits 0 on success.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "pipefill/kfac/kfac.hpp"
#include "pipefill/kfac/matrix.hpp"

using namespace pipefill::kfac;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            ++g_fail;                                                            \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);          \
        }                                                                        \
    } while (0)
template <class E>
static bool throws_as(const std::function<void()>& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static Matrix random_matrix(int r, int c, SplitMix64& rng) {
    Matrix m(r, c);
    for (double& v : m.data()) v = rng.symmetric();
    return m;
}
static Matrix random_spd(int n, SplitMix64& rng) {
    const Matrix x = random_matrix(n, n + 2, rng);
    Matrix s = matmul(x, x.transposed());
    for (int i = 0; i < n; ++i) s(i, i) += 0.5;
    return s;
}
static double rel_fro(const Matrix& got, const Matrix& want) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < got.data().size(); ++i) {
        num += (got.data()[i] - want.data()[i]) * (got.data()[i] - want.data()[i]);
        den += want.data()[i] * want.data()[i];
    }
    return std::sqrt(num / std::max(den, 1e-300));
}
static double bf16(double v) {  // round to the bf16 grid the GPU tapes use
    float f = static_cast<float>(v);
    unsigned u;
    std::memcpy(&u, &f, 4);
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    std::memcpy(&f, &u, 4);
    return f;
}

int main() {
    // ---- curvature factors from hand outer products (test_kfac.cpp:99-124)
    {
        BatchTape tape;
        tape.batch_size = 1;
        tape.layer_inputs = {Matrix{{1.0}, {2.0}}};
        tape.layer_errors = {Matrix{{3.0}}};
        const auto [a, b] = curvature_factors(tape, 0);
        CHECK(a == (Matrix{{1.0, 2.0}, {2.0, 4.0}}));
        CHECK(b == (Matrix{{9.0}}));
        BatchTape twice;
        twice.batch_size = 2;
        twice.layer_inputs = {Matrix{{1.0, 1.0}, {2.0, 2.0}}};
        twice.layer_errors = {Matrix{{3.0, 3.0}}};
        const auto [a2, b2] = curvature_factors(twice, 0);
        CHECK(max_abs_diff(a2, a) < 1e-6);
        CHECK(max_abs_diff(b2, b) < 1e-6);
        BatchTape zero;
        zero.batch_size = 1;
        zero.layer_inputs = {Matrix{{1.0}, {2.0}}};
        zero.layer_errors = {Matrix{{0.0}}};
        CHECK(curvature_factors(zero, 0).second.max_abs() == 0.0);
    }
    // ---- BERT-ish non-multiple-of-128 sizes vs the FP64 product of the same bf16 inputs
    {
        SplitMix64 rng(2211);
        BatchTape tape;
        tape.batch_size = 200;
        Matrix a = random_matrix(300, 200, rng), e = random_matrix(130, 200, rng);
        for (double& v : a.data()) v = bf16(v);
        for (double& v : e.data()) v = bf16(v);
        tape.layer_inputs = {a};
        tape.layer_errors = {e};
        KfacState st(1);
        st.update_factors(tape);
        CHECK(rel_fro(st.factor_a[0], matmul(a, a.transposed()).scaled(1.0 / 200)) < 1e-3);
        CHECK(rel_fro(st.factor_b[0], matmul(e, e.transposed()).scaled(1.0 / 200)) < 1e-3);
        st.damping = 0.1;
        st.refresh_inverses();
        Matrix damped = st.factor_a[0];
        for (int i = 0; i < damped.rows(); ++i) damped(i, i) += 0.1;
        CHECK(max_abs_diff(matmul(damped, st.inv_a[0]), Matrix::identity(300)) < 1e-5);
        CHECK(st.staleness[0] == 0 && st.refreshed_this_step[0] == 1);
    }
    // ---- cholesky inverse (test_kfac.cpp:144-160)
    {
        CHECK(max_abs_diff(cholesky_spd_inverse(Matrix{{4.0, 0.0}, {0.0, 9.0}}, 0.0),
                           Matrix{{0.25, 0.0}, {0.0, 1.0 / 9.0}}) < 1e-7);
        CHECK(max_abs_diff(cholesky_spd_inverse(Matrix::identity(3), 0.0), Matrix::identity(3)) < 1e-7);
        SplitMix64 rng(99);
        const Matrix m = random_spd(8, rng);
        const Matrix inv = cholesky_spd_inverse(m, 0.5);
        Matrix damped = m;
        for (int i = 0; i < 8; ++i) damped(i, i) += 0.5;
        CHECK(max_abs_diff(matmul(damped, inv), Matrix::identity(8)) < 1e-5);
        CHECK(throws_as<std::domain_error>([] { cholesky_spd_inverse(Matrix{{1.0, 2.0}, {2.0, 1.0}}, 0.0); }));
        CHECK(throws_as<std::invalid_argument>([] { cholesky_spd_inverse(Matrix(2, 3), 0.0); }));
    }
    // ---- precondition hand example (test_kfac.cpp:162-169)
    {
        const Matrix a_inv = Matrix::identity(2).scaled(0.5);
        const Matrix b_inv = Matrix{{1.0 / 3.0}};
        const Matrix g{{6.0, 6.0}};
        CHECK(max_abs_diff(precondition(g, a_inv, b_inv), Matrix{{1.0, 1.0}}) < 1e-6);
        CHECK(max_abs_diff(precondition(g, Matrix::identity(2), Matrix::identity(1)), g) < 1e-6);
        CHECK(throws_as<std::invalid_argument>([&] { precondition(g, Matrix::identity(3), b_inv); }));
    }
    // ---- vec trick equals the dense Kronecker solve (test_kfac.cpp:171-184)
    {
        SplitMix64 rng(4242);
        for (int trial = 0; trial < 10; ++trial) {
            const int d_in = 2 + static_cast<int>(rng.next() % 5);
            const int d_out = 2 + static_cast<int>(rng.next() % 5);
            const Matrix a = random_spd(d_in, rng);
            const Matrix b = random_spd(d_out, rng);
            const Matrix g = random_matrix(d_out, d_in, rng);
            const Matrix direct = precondition(g, cholesky_spd_inverse(a, 0.0), cholesky_spd_inverse(b, 0.0));
            const Matrix dense = unvec(solve_spd(kron(a, b), vec(g)), d_out, d_in);
            CHECK(rel_fro(direct, dense) < 1e-5);
        }
    }
    // ---- cholesky_factor on the GPU (matrix.cpp:117-134): hand case + non-PD
    {
        const Matrix l = cholesky_factor(Matrix{{4.0, 2.0}, {2.0, 3.0}});
        CHECK(std::fabs(l(0, 0) - 2.0) < 1e-6 && std::fabs(l(1, 0) - 1.0) < 1e-6 &&
              std::fabs(l(1, 1) - std::sqrt(2.0)) < 1e-6 && l(0, 1) == 0.0);
        bool threw = false;
        try {
            (void)cholesky_factor(Matrix{{1.0, 2.0}, {2.0, 1.0}});
        } catch (const std::domain_error&) {
            threw = true;
        }
        CHECK(threw);
    }
    // ---- ngd_step (test_kfac.cpp:275-330)
    {
        TinyMlp mlp{{Matrix{{2.0}}}, {Activation::Identity}, LossKind::MeanSquaredError};
        KfacState state(1);
        state.learning_rate = 1.0;
        const auto r = ngd_step(mlp, state, {Matrix{{0.5}}});
        CHECK(r.used_plain_gradient);
        CHECK(std::fabs(mlp.weights[0](0, 0) - 1.5) < 1e-12);
        CHECK(state.staleness[0] == 1);

        // scalar net: A = [[1]], B = [[4]], G = [[4]] -> direction 1
        TinyMlp net{{Matrix{{2.0}}}, {Activation::Identity}, LossKind::MeanSquaredError};
        KfacState s2(1);
        s2.learning_rate = 0.3;
        s2.factor_a = {Matrix{{1.0}}};
        s2.factor_b = {Matrix{{4.0}}};
        s2.refresh_inverses();
        const auto r2 = ngd_step(net, s2, {Matrix{{4.0}}});
        CHECK(!r2.used_plain_gradient);
        CHECK(std::fabs(net.weights[0](0, 0) - 1.7) < 1e-6);
        CHECK(s2.staleness[0] == 1);
        ngd_step(net, s2, {Matrix{{4.0}}});
        CHECK(s2.staleness[0] == 2);
        CHECK(throws_as<std::invalid_argument>([&] { ngd_step(net, s2, {}); }));
    }
    // ---- block-diagonal split and flop model (kfac.cpp:203-226)
    {
        Matrix m(4, 4);
        for (int i = 0; i < 16; ++i) m.data()[i] = i;
        const auto blocks = block_diag_split_factor(m, 2);
        CHECK(blocks.size() == 2);
        CHECK(blocks[0] == (Matrix{{0, 1}, {4, 5}}));
        CHECK(blocks[1] == (Matrix{{10, 11}, {14, 15}}));
        CHECK(throws_as<std::invalid_argument>([&] { block_diag_split_factor(m, 3); }));
        CHECK(std::fabs(block_diag_inversion_flops(8192, 4) - inversion_flops(8192) / 16) < 1.0);
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    if (g_fail == 0) std::printf("ALL PASS\n");
    return g_fail == 0 ? 0 : 1;
}

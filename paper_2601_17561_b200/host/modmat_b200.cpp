// C++ host mirror of irislab::modmat over the C ABI (see irislab_b200/modmat.hpp).
// Host code only: every product is computed by libirl_b200's sm_100a kernels.
#include "irislab_b200/modmat.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <mutex>
#include <sstream>

#include "irl_capi.h"

namespace irislab {

namespace {

std::mutex g_mu;
irl_ctx* g_ctx = nullptr;
int g_device = 0;

irl_ctx* ctx() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_ctx) {
        const int st = irl_ctx_create(g_device, &g_ctx);
        if (st != IRL_OK)
            throw DeviceError(std::string("irl_ctx_create failed: ") + irl_status_string(st) +
                              " (needs an sm_100 GPU; there is no CPU fallback)");
    }
    return g_ctx;
}

// Rethrow the reference exception type for a C ABI status.
void check(int st) {
    if (st == IRL_OK) return;
    const std::string msg = irl_last_error(g_ctx);
    switch (st) {
        case IRL_ERR_SHAPE_MISMATCH: throw ShapeMismatch(msg);
        case IRL_ERR_MODULUS_TOO_LARGE: throw ModulusTooLarge(msg);
        case IRL_ERR_ACCUMULATION_OVERFLOW_RISK: throw AccumulationOverflowRisk(msg);
        case IRL_ERR_NOT_COPRIME: throw Error(msg);
        case IRL_ERR_MODULUS_BUDGET: throw ModulusBudget(msg);
        default: throw DeviceError(std::string(irl_status_string(st)) + ": " + msg);
    }
}

std::vector<uint8_t> product_le(const std::vector<modmat::RnsBasis::Modulus>& mods) {
    std::vector<uint32_t> p, e;
    for (const auto& m : mods) {
        p.push_back(m.p);
        e.push_back(m.e);
    }
    std::vector<uint8_t> q(64);
    const size_t w = irl_basis_Q_bytes(p.data(), e.data(), p.size(), q.data(), q.size());
    q.resize(w);
    return q;
}

// a >= b on equal-width little-endian integers
bool ge(const uint8_t* a, const std::vector<uint8_t>& b, size_t w) {
    for (size_t i = w; i-- > 0;) {
        const uint8_t bi = i < b.size() ? b[i] : 0;
        if (a[i] != bi) return a[i] > bi;
    }
    return true;
}

void sub(uint8_t* a, const std::vector<uint8_t>& b, size_t w) {
    int borrow = 0;
    for (size_t i = 0; i < w; ++i) {
        const int d = int(a[i]) - (i < b.size() ? b[i] : 0) - borrow;
        a[i] = uint8_t(d & 0xFF);
        borrow = d < 0;
    }
}

}  // namespace

namespace b200 {
void set_device(int device) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_device = device;
}
uint64_t kernel_launches() { return g_ctx ? irl_kernel_launches(g_ctx) : 0; }
irl_ctx* context() { return ctx(); }
}  // namespace b200

namespace modmat {

std::vector<uint32_t> primes_in_range(uint32_t lo, uint32_t hi) {
    std::vector<uint32_t> out;
    for (uint32_t n = std::max(lo, 2u); n <= hi; ++n) {
        bool prime = true;
        for (uint32_t q = 2; q * q <= n; ++q)
            if (n % q == 0) {
                prime = false;
                break;
            }
        if (prime) out.push_back(n);
    }
    return out;
}

std::size_t RnsBasis::digit_planes() const {
    std::size_t planes = 0;
    for (const auto& m : moduli) planes += m.e;
    return planes;
}

double RnsBasis::log2_Q() const {
    // exact bit length + log2 of the leading 64-bit mantissa
    size_t top = Q.size();
    while (top > 0 && Q[top - 1] == 0) --top;
    if (top == 0) return -INFINITY;
    double mant = 0.0;
    const size_t lo = top >= 8 ? top - 8 : 0;
    for (size_t i = top; i-- > lo;) mant = mant * 256.0 + Q[i];
    return std::log2(mant) + 8.0 * double(lo);
}

RnsBasis make_basis(const std::vector<RnsBasis::Modulus>& moduli) {
    RnsBasis b;
    b.moduli = moduli;
    b.Q = product_le(moduli);
    return b;
}

RnsBasis build_paper_basis() {
    std::vector<RnsBasis::Modulus> mods;
    for (uint32_t p : primes_in_range(127, 253)) mods.push_back({p, 2});
    return make_basis(mods);
}

double max_int8_rns_capacity() {
    double total = 0.0;
    for (uint32_t p : primes_in_range(3, 253)) {
        uint32_t e = 0;
        uint64_t pw = 1;
        while (pw * p < 256) {
            pw *= p;
            ++e;
        }
        total += e * std::log2(double(p));
    }
    return total;
}

std::size_t pure_rns_plane_count() { return primes_in_range(3, 253).size(); }

BigMatrix BigMatrix::zeros(std::size_t r, std::size_t c, std::size_t width) {
    BigMatrix m;
    m.rows = r;
    m.cols = c;
    m.width = width;
    m.a.assign(r * c * width, 0);
    return m;
}

BigMatrix BigMatrix::identity(std::size_t n, std::size_t width) {
    BigMatrix m = zeros(n, n, width);
    for (std::size_t i = 0; i < n; ++i) m.at(i, i)[0] = 1;
    return m;
}

void BigMatrix::reduce(const std::vector<uint8_t>& Q) {
    for (std::size_t i = 0; i < rows * cols; ++i) {
        uint8_t* x = a.data() + i * width;
        while (ge(x, Q, width)) sub(x, Q, width);
    }
}

DigitMatrices digit_decompose(const SmallMatrix& m, uint32_t p) {
    DigitMatrices d;
    d.p = p;
    d.m0 = {m.rows, m.cols, std::vector<int32_t>(m.a.size())};
    d.m1 = {m.rows, m.cols, std::vector<int32_t>(m.a.size())};
    irl_ctx* c = ctx();
    check(irl_digit_decompose(c, m.a.data(), m.rows, m.cols, p, d.m0.a.data(), d.m1.a.data()));
    return d;
}

SmallMatrix digit_recompose(const DigitMatrices& d) {
    SmallMatrix m{d.m0.rows, d.m0.cols, std::vector<int32_t>(d.m0.a.size())};
    irl_ctx* c = ctx();
    check(irl_digit_recompose(c, d.m0.a.data(), d.m1.a.data(), d.m0.rows, d.m0.cols, d.p, m.a.data()));
    return m;
}

SmallMatrix small_gemm(const SmallMatrix& a, const SmallMatrix& b) {
    if (a.cols != b.rows) throw ShapeMismatch("small_gemm: inner dimensions differ");
    SmallMatrix c{a.rows, b.cols, std::vector<int32_t>(a.rows * b.cols, 0)};
    irl_ctx* cx = ctx();
    check(irl_small_gemm(cx, a.a.data(), b.a.data(), c.a.data(), a.rows, a.cols, b.cols));
    return c;
}

SmallMatrix gemm_mod_psq(const SmallMatrix& a, const SmallMatrix& b, uint32_t p) {
    // digit_decompose(a, p) runs first in the reference (modmat.cpp:145-146)
    if (p >= 256) throw ModulusTooLarge("digit base must be < 2^8");
    if (a.cols != b.rows) throw ShapeMismatch("small_gemm: inner dimensions differ");
    SmallMatrix c{a.rows, b.cols, std::vector<int32_t>(a.rows * b.cols, 0)};
    irl_ctx* cx = ctx();
    check(irl_gemm_mod_psq(cx, a.a.data(), b.a.data(), c.a.data(), a.rows, a.cols, b.cols, p));
    return c;
}

BigMatrix gemm_mod_Q(const BigMatrix& a, const BigMatrix& b, const RnsBasis& basis) {
    if (a.cols != b.rows) throw ShapeMismatch("gemm_mod_Q: inner dimensions differ");
    const size_t w = basis.width();
    if (a.width != w || b.width != w) throw ShapeMismatch("gemm_mod_Q: entry width differs from the basis");
    std::vector<uint32_t> p, e;
    for (const auto& m : basis.moduli) {
        p.push_back(m.p);
        e.push_back(m.e);
    }
    BigMatrix c = BigMatrix::zeros(a.rows, b.cols, w);
    irl_ctx* cx = ctx();
    check(irl_gemm_mod_Q(cx, a.a.data(), b.a.data(), c.a.data(), a.rows, a.cols, b.cols, w, p.data(),
                         e.data(), p.size()));
    return c;
}

std::string to_decimal(const std::vector<uint8_t>& le) {
    std::vector<uint32_t> limbs((le.size() + 3) / 4, 0);
    for (size_t i = 0; i < le.size(); ++i) limbs[i / 4] |= uint32_t(le[i]) << (8 * (i % 4));
    std::string digits;
    auto nonzero = [&] {
        for (uint32_t l : limbs)
            if (l) return true;
        return false;
    };
    while (nonzero()) {
        uint64_t r = 0;
        for (size_t i = limbs.size(); i-- > 0;) {
            const uint64_t cur = (r << 32) | limbs[i];
            limbs[i] = uint32_t(cur / 1000000000u);
            r = cur % 1000000000u;
        }
        char buf[16];
        std::snprintf(buf, sizeof buf, "%09u", unsigned(r));
        digits.insert(0, buf);
    }
    const size_t nz = digits.find_first_not_of('0');
    return nz == std::string::npos ? "0" : digits.substr(nz);
}

static std::vector<uint8_t> from_decimal(const std::string& s) {
    std::vector<uint32_t> limbs{0};
    for (char ch : s) {
        if (ch < '0' || ch > '9') throw Error("bad decimal modulus in matrix header");
        uint64_t carry = uint64_t(ch - '0');
        for (auto& l : limbs) {
            const uint64_t t = uint64_t(l) * 10 + carry;
            l = uint32_t(t);
            carry = t >> 32;
        }
        if (carry) limbs.push_back(uint32_t(carry));
    }
    std::vector<uint8_t> out(limbs.size() * 4);
    for (size_t i = 0; i < out.size(); ++i) out[i] = uint8_t(limbs[i / 4] >> (8 * (i % 4)));
    while (out.size() > 1 && out.back() == 0) out.pop_back();
    return out;
}

// modmat.cpp:216-231: header "rows cols Q\n", then ceil(log256 Q)-byte LE entries.
void save_big_matrix(const std::string& path, const BigMatrix& m, const std::vector<uint8_t>& Q) {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw Error("cannot open " + path + " for writing");
    std::vector<uint8_t> q = Q;
    while (q.size() > 1 && q.back() == 0) q.pop_back();
    const size_t width = q.size();
    os << m.rows << " " << m.cols << " " << to_decimal(q) << "\n";
    std::vector<uint8_t> buf(width);
    for (size_t i = 0; i < m.rows * m.cols; ++i) {
        std::fill(buf.begin(), buf.end(), 0);
        std::copy_n(m.a.data() + i * m.width, std::min(width, m.width), buf.begin());
        os.write(reinterpret_cast<const char*>(buf.data()), std::streamsize(width));
    }
}

// modmat.cpp:233-249.
BigMatrix load_big_matrix(const std::string& path, std::vector<uint8_t>* Q_out) {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw Error("cannot open " + path);
    std::size_t rows = 0, cols = 0;
    std::string q_str;
    is >> rows >> cols >> q_str;
    is.get();  // newline
    const std::vector<uint8_t> Q = from_decimal(q_str);
    if (Q_out) *Q_out = Q;
    const size_t width = Q.size();
    BigMatrix m = BigMatrix::zeros(rows, cols, width);
    for (size_t i = 0; i < rows * cols; ++i) {
        is.read(reinterpret_cast<char*>(m.a.data() + i * width), std::streamsize(width));
        if (!is) throw Error("truncated matrix file " + path);
    }
    return m;
}

}  // namespace modmat
}  // namespace irislab

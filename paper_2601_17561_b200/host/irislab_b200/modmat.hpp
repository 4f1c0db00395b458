// C++ host mirror of the reference's irislab::modmat API
// (/root/reference/proj/include/irislab/modmat.hpp:11-93), executed on the
// B200 through the C ABI (include/irl_capi.h). Same namespace, names,
// argument meaning, value semantics and exception types, so the reference's
// own test drivers (tests/test_modmat.cpp) compile against it unchanged in
// spirit. The one deliberate difference: BigMatrix / RnsBasis::Q hold
// fixed-width little-endian integers (the reference's on-disk entry format,
// modmat.cpp:216-231) instead of GMP mpz_class values.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace irislab {

// errors.hpp:9-53 (the subset raised on this path)
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeMismatch : Error {
    using Error::Error;
};
struct ModulusTooLarge : Error {
    using Error::Error;
};
struct AccumulationOverflowRisk : Error {
    using Error::Error;
};
struct ModulusBudget : Error {
    using Error::Error;
};
// Device / CUDA failures (no reference counterpart; there is no CPU fallback).
struct DeviceError : Error {
    using Error::Error;
};

namespace modmat {

/// RNS basis of pairwise coprime moduli p^e with p < 2^8 (modmat.hpp:14-28).
struct RnsBasis {
    struct Modulus {
        uint32_t p = 0;
        uint32_t e = 1;
        uint32_t value() const { return e == 2 ? p * p : p; }
    };
    std::vector<Modulus> moduli;
    std::vector<uint8_t> Q;  // exact product, little-endian bytes

    std::size_t digit_planes() const;
    double log2_Q() const;
    std::size_t width() const { return Q.size(); }  // ceil(log256 Q)
};

RnsBasis build_paper_basis();
RnsBasis make_basis(const std::vector<RnsBasis::Modulus>& moduli);
double max_int8_rns_capacity();
std::size_t pure_rns_plane_count();
std::vector<uint32_t> primes_in_range(uint32_t lo, uint32_t hi);

/// Row-major int matrix (modmat.hpp:43-50).
struct SmallMatrix {
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::vector<int32_t> a;

    int32_t& at(std::size_t r, std::size_t c) { return a[r * cols + c]; }
    int32_t at(std::size_t r, std::size_t c) const { return a[r * cols + c]; }
};

/// M = M0 + p*M1 (mod p^2), centred digits (modmat.hpp:52-57).
struct DigitMatrices {
    uint32_t p = 0;
    SmallMatrix m0;
    SmallMatrix m1;
};

/// Row-major matrix of integers in [0, Q), each `width` little-endian bytes.
struct BigMatrix {
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::size_t width = 0;
    std::vector<uint8_t> a;

    static BigMatrix zeros(std::size_t r, std::size_t c, std::size_t width);
    static BigMatrix identity(std::size_t n, std::size_t width);
    uint8_t* at(std::size_t r, std::size_t c) { return a.data() + (r * cols + c) * width; }
    const uint8_t* at(std::size_t r, std::size_t c) const {
        return a.data() + (r * cols + c) * width;
    }
    /// entries mod Q (modmat.cpp:79-84); input entries are non-negative.
    void reduce(const std::vector<uint8_t>& Q);
};

DigitMatrices digit_decompose(const SmallMatrix& m, uint32_t p);
SmallMatrix digit_recompose(const DigitMatrices& d);
SmallMatrix small_gemm(const SmallMatrix& a, const SmallMatrix& b);
SmallMatrix gemm_mod_psq(const SmallMatrix& a, const SmallMatrix& b, uint32_t p);
BigMatrix gemm_mod_Q(const BigMatrix& a, const BigMatrix& b, const RnsBasis& basis);

void save_big_matrix(const std::string& path, const BigMatrix& m, const std::vector<uint8_t>& Q);
BigMatrix load_big_matrix(const std::string& path, std::vector<uint8_t>* Q_out = nullptr);

/// Decimal string of a little-endian integer (the file header's Q).
std::string to_decimal(const std::vector<uint8_t>& le);

}  // namespace modmat

namespace b200 {
/// Device used by the free functions above (default 0; set before first use).
void set_device(int device);
/// Number of kernels the engine launched through the free functions.
uint64_t kernel_launches();
}  // namespace b200
}  // namespace irislab
struct irl_ctx;
namespace irislab {
namespace b200 {
/// The process-wide device context behind the free functions (created lazily).
irl_ctx* context();
}  // namespace b200

}  // namespace irislab

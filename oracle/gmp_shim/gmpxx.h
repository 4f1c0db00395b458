// Minimal eager C++ wrapper over the GMP runtime, written for this repo's
// test oracle (see gmp.h). Provides the mpz_class / mpf_class / gmp_randclass
// surface the reference hot path (proj/src/modmat.cpp), its unit tests and
// acceptance criterion 2 use. Division and remainder truncate toward zero,
// matching gmpxx. Test infrastructure only; never shipped.
#ifndef IRL_GMPXX_SHIM_H
#define IRL_GMPXX_SHIM_H

#include <cstdlib>
#include <string>
#include <utility>

#include "gmp.h"

class mpz_class {
public:
    mpz_class() { __gmpz_init(v_); }
    mpz_class(int x) { __gmpz_init_set_si(v_, x); }
    mpz_class(long x) { __gmpz_init_set_si(v_, x); }
    mpz_class(long long x) { __gmpz_init_set_si(v_, static_cast<long>(x)); }
    mpz_class(unsigned x) { __gmpz_init_set_ui(v_, x); }
    mpz_class(unsigned long x) { __gmpz_init_set_ui(v_, x); }
    mpz_class(unsigned long long x) { __gmpz_init_set_ui(v_, static_cast<unsigned long>(x)); }
    explicit mpz_class(const std::string& s, int base = 10) { __gmpz_init_set_str(v_, s.c_str(), base); }
    explicit mpz_class(const char* s, int base = 10) { __gmpz_init_set_str(v_, s, base); }
    mpz_class(const mpz_class& o) { __gmpz_init_set(v_, o.v_); }
    mpz_class(mpz_class&& o) noexcept { __gmpz_init(v_); __gmpz_swap(v_, o.v_); }
    ~mpz_class() { __gmpz_clear(v_); }

    mpz_class& operator=(const mpz_class& o) { if (this != &o) __gmpz_set(v_, o.v_); return *this; }
    mpz_class& operator=(mpz_class&& o) noexcept { __gmpz_swap(v_, o.v_); return *this; }
    mpz_class& operator=(long x) { __gmpz_set_si(v_, x); return *this; }
    mpz_class& operator=(int x) { __gmpz_set_si(v_, x); return *this; }
    mpz_class& operator=(unsigned long x) { __gmpz_set_ui(v_, x); return *this; }

    __mpz_struct* get_mpz_t() { return v_; }
    const __mpz_struct* get_mpz_t() const { return v_; }
    unsigned long get_ui() const { return __gmpz_get_ui(v_); }
    std::string get_str(int base = 10) const {
        char* s = __gmpz_get_str(nullptr, base, v_);
        std::string r(s);
        std::free(s);
        return r;
    }

    mpz_class& operator+=(const mpz_class& o) { __gmpz_add(v_, v_, o.v_); return *this; }
    mpz_class& operator-=(const mpz_class& o) { __gmpz_sub(v_, v_, o.v_); return *this; }
    mpz_class& operator*=(const mpz_class& o) { __gmpz_mul(v_, v_, o.v_); return *this; }
    mpz_class& operator%=(const mpz_class& o) { __gmpz_tdiv_r(v_, v_, o.v_); return *this; }
    mpz_class& operator/=(const mpz_class& o) { __gmpz_tdiv_q(v_, v_, o.v_); return *this; }

    friend mpz_class operator+(const mpz_class& a, const mpz_class& b) { mpz_class r; __gmpz_add(r.v_, a.v_, b.v_); return r; }
    friend mpz_class operator-(const mpz_class& a, const mpz_class& b) { mpz_class r; __gmpz_sub(r.v_, a.v_, b.v_); return r; }
    friend mpz_class operator*(const mpz_class& a, const mpz_class& b) { mpz_class r; __gmpz_mul(r.v_, a.v_, b.v_); return r; }
    friend mpz_class operator/(const mpz_class& a, const mpz_class& b) { mpz_class r; __gmpz_tdiv_q(r.v_, a.v_, b.v_); return r; }
    friend mpz_class operator%(const mpz_class& a, const mpz_class& b) { mpz_class r; __gmpz_tdiv_r(r.v_, a.v_, b.v_); return r; }
    friend mpz_class operator<<(const mpz_class& a, unsigned long s) { mpz_class r; __gmpz_mul_2exp(r.v_, a.v_, s); return r; }

    friend bool operator==(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(a.v_, b.v_) == 0; }
    friend bool operator!=(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(a.v_, b.v_) != 0; }
    friend bool operator<(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(a.v_, b.v_) < 0; }
    friend bool operator>(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(a.v_, b.v_) > 0; }
    friend bool operator<=(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(a.v_, b.v_) <= 0; }
    friend bool operator>=(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(a.v_, b.v_) >= 0; }
    friend bool operator==(const mpz_class& a, long b) { return __gmpz_cmp_si(a.v_, b) == 0; }
    friend bool operator<(const mpz_class& a, long b) { return __gmpz_cmp_si(a.v_, b) < 0; }
    friend bool operator==(const mpz_class& a, int b) { return __gmpz_cmp_si(a.v_, b) == 0; }
    friend bool operator<(const mpz_class& a, int b) { return __gmpz_cmp_si(a.v_, b) < 0; }

private:
    mpz_t v_;
};

class mpf_class {
public:
    mpf_class(const mpz_class& z, unsigned long prec) { __gmpf_init2(v_, prec); __gmpf_set_z(v_, z.get_mpz_t()); }
    mpf_class(const mpf_class&) = delete;
    mpf_class& operator=(const mpf_class&) = delete;
    ~mpf_class() { __gmpf_clear(v_); }
    __mpf_struct* get_mpf_t() { return v_; }
    const __mpf_struct* get_mpf_t() const { return v_; }

private:
    mpf_t v_;
};

class gmp_randclass {
public:
    explicit gmp_randclass(void (*init)(__gmp_randstate_struct*)) { init(s_); }
    gmp_randclass(const gmp_randclass&) = delete;
    gmp_randclass& operator=(const gmp_randclass&) = delete;
    ~gmp_randclass() { __gmp_randclear(s_); }
    void seed(unsigned long s) { __gmp_randseed_ui(s_, s); }
    mpz_class get_z_range(const mpz_class& n) {
        mpz_class r;
        __gmpz_urandomm(r.get_mpz_t(), s_, n.get_mpz_t());
        return r;
    }

private:
    gmp_randstate_t s_;
};

#endif  // IRL_GMPXX_SHIM_H

// Drop-in of the B200 CCMM under the reference's own caller, without editing
// it: Emulator::ccmm_twin (reference emulator.cpp:389-447) is interposed at
// link time (-Wl,--wrap=<mangled ccmm_twin>), so run_alg1 / run_alg2
// (pipeline.cpp:512-514, 550-557) reach this translation unit instead.
//
//   * The reference's own ccmm_twin still runs, on an all-zero database of
//     the caller's shapes: it performs every validation in its order with its
//     messages, builds the d1*d3/n_db output ciphertexts with their metadata,
//     injects noise (when enabled) and records the trace, exactly as before.
//     Its product loop skips zero database entries (emulator.cpp:415), so it
//     does no arithmetic.
//   * The product itself comes from the B200 engine (irl_ccmm_twin,
//     include/irl_capi.h), packed in ccmm_twin's order, and is added to each
//     slot: slot = (0 + noise) + prod, which is bit-identical to the
//     reference's prod + noise (IEEE addition commutes; with noise off the
//     slot is 0 + prod = prod).
//
// Built with -DIRL_HOOK_STOCK the same unit keeps the reference product (it
// forwards the real database) and only records the digest below, so a stock
// library and the B200-routed library expose identical entry points.
//
// Both variants keep an FNV-1a digest of every ccmm_twin output message (bit
// patterns, real and imaginary) for the parity tests.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "irislab/emulator.hpp"
#include "irislab/errors.hpp"

#ifndef IRL_HOOK_STOCK
#include "irl_capi.h"
#endif

using irislab::emu::CcmmSpec;
using irislab::emu::EmulatedCiphertext;
using irislab::emu::Emulator;
using irislab::emu::Encoding;

#define IRL_CCMM_SYM _ZN7irislab3emu8Emulator9ccmm_twinERKNS0_8CcmmSpecERKSt6vectorIdSaIdEES9_
#define IRL_CAT2(a, b) a##b
#define IRL_CAT(a, b) IRL_CAT2(a, b)

// Itanium C++ ABI: a member function returning a class by value takes the
// return slot first and `this` second, exactly like this free function.
extern "C" std::vector<EmulatedCiphertext> IRL_CAT(__real_, IRL_CCMM_SYM)(Emulator* self, const CcmmSpec& spec,
                                                                         const std::vector<double>& db,
                                                                         const std::vector<double>& qry);

namespace {

uint64_t g_digest = 1469598103934665603ull;
long g_calls = 0;
long g_slots = 0;
#ifndef IRL_HOOK_STOCK
irl_ctx* g_ctx = nullptr;
#endif

void digest(const std::vector<EmulatedCiphertext>& out) {
    for (const auto& ct : out)
        for (const auto& m : ct.message) {
            const double parts[2] = {m.real(), m.imag()};
            unsigned char b[16];
            std::memcpy(b, parts, 16);
            for (unsigned char c : b) g_digest = (g_digest ^ c) * 1099511628211ull;
            ++g_slots;
        }
    ++g_calls;
}

}  // namespace

extern "C" std::vector<EmulatedCiphertext> IRL_CAT(__wrap_, IRL_CCMM_SYM)(Emulator* self, const CcmmSpec& spec,
                                                                         const std::vector<double>& db,
                                                                         const std::vector<double>& qry) {
#ifdef IRL_HOOK_STOCK
    std::vector<EmulatedCiphertext> out = IRL_CAT(__real_, IRL_CCMM_SYM)(self, spec, db, qry);
#else
    const std::vector<double> zeros(db.size(), 0.0);
    std::vector<EmulatedCiphertext> out = IRL_CAT(__real_, IRL_CCMM_SYM)(self, spec, zeros, qry);
    if (!g_ctx && irl_ctx_create(0, &g_ctx) != IRL_OK) throw irislab::Error("B200 context: no usable device");
    std::vector<double> msgs(static_cast<std::size_t>(spec.d1 * spec.d3));
    const int st = irl_ccmm_twin(g_ctx, spec.d1, spec.d2, spec.d3, spec.n_db, spec.n_qry, spec.db_modulus_bits,
                                 spec.qry_modulus_bits, spec.scale_bits, spec.out_level,
                                 self->config().chain.top_level(), spec.out_encoding == Encoding::Slot ? 1 : 0,
                                 spec.out_ci ? 1 : 0, db.data(), qry.data(), msgs.data());
    if (st != IRL_OK) throw irislab::Error(std::string("irl_ccmm_twin: ") + irl_last_error(g_ctx));
    // msgs[(c * (d1 / n_db) + b) * n_db + i] is slot i of output ciphertext c * blocks + b
    std::size_t k = 0;
    for (auto& ct : out)
        for (auto& m : ct.message) m = {m.real() + msgs[k++], m.imag()};
#endif
    digest(out);
    return out;
}

extern "C" {
void irl_hook_reset() {
    g_digest = 1469598103934665603ull;
    g_calls = 0;
    g_slots = 0;
}
uint64_t irl_hook_digest() { return g_digest; }
long irl_hook_calls() { return g_calls; }
long irl_hook_slots() { return g_slots; }
int irl_hook_is_b200() {
#ifdef IRL_HOOK_STOCK
    return 0;
#else
    return 1;
#endif
}
}

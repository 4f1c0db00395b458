// C++ host side of the RGSW CCMM on the B200 (C ABI irl_ccmm_*):
//   * irislab::emu::CcmmSpec and ccmm_twin_product(): the exact product behind
//     Emulator::ccmm_twin (emulator.hpp:85-97, 135-140; emulator.cpp:389-447),
//     same validation order, messages and exception types, computed on the
//     PPMM engine; returned as the d1*d3/n_db output ciphertexts' messages in
//     ccmm_twin's order (the plaintext-twin bookkeeping -- level, encoding,
//     trace -- stays with the caller's emulator);
//   * irislab::b200::CcmmEngine: RAII over the device-resident engine (the
//     paper's 8-slice database), one query batch per run();
//   * irislab::b200::CcmmGroup: the same over several GPUs from one process
//     (irl_ccmm_group_* / irl_ccmm_full): the parts dealt across the devices,
//     the a-part result exchanged to every rank, the query sharded over them.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "modmat.hpp"  // irislab::Error, ShapeMismatch, ModulusBudget, DeviceError, RnsBasis

struct irl_ccmm;
struct irl_ccmm_group;

namespace irislab {
namespace emu {

enum class Encoding { Coeff, Slot };

/// emulator.hpp:85-97
struct CcmmSpec {
    long d1 = 0, d2 = 0, d3 = 0;
    long n_db = 0;
    long n_qry = 0;
    double db_modulus_bits = 0.0;
    double qry_modulus_bits = 0.0;
    double scale_bits = 0.0;
    int out_level = 0;
    Encoding out_encoding = Encoding::Coeff;
    bool out_ci = false;
};

/// Messages of ccmm_twin's outputs: result[k] holds the n_db slots of output
/// ciphertext k, k = c * (d1 / n_db) + b for column c and row block b
/// (emulator.cpp:425-439). db is d1 x d2 and qry d2 x d3, row-major,
/// integer-valued; top_level bounds out_level as the emulator's chain does.
std::vector<std::vector<double>> ccmm_twin_product(const CcmmSpec& spec, const std::vector<double>& db,
                                                   const std::vector<double>& qry, int top_level);

}  // namespace emu

namespace b200 {

/// Device-resident CCMM engine over `parts` database parts of m x k entries
/// (residues of the basis' moduli, registered once) and query batches of up to
/// max_n columns (wider batches stream through in column chunks).
class CcmmEngine {
public:
    CcmmEngine(std::size_t parts, std::size_t m, std::size_t k, std::size_t max_n,
               const modmat::RnsBasis& basis = modmat::build_paper_basis());
    ~CcmmEngine();
    CcmmEngine(const CcmmEngine&) = delete;
    CcmmEngine& operator=(const CcmmEngine&) = delete;

    /// residues [nmod][m][k] of one part (host memory)
    void load_part(std::size_t part, const std::vector<uint16_t>& residues);
    /// one part as m x k little-endian mod-Q entries of `width` bytes (BigMatrix file form)
    void load_part_bigint(std::size_t part, const modmat::BigMatrix& entries);
    /// stream one part from the reference's BigMatrix file (save_big_matrix format)
    void load_part_file(std::size_t part, const std::string& path);
    /// counter-RNG synthetic database (the bench's inputs)
    void synth_db(uint64_t seed, uint32_t first_part = 0);
    /// q_res [nmod][k][n] -> out [parts][nmod][n][m] residues mod p^2 (blocking).
    /// Page-locked buffers are DMA'd directly; pageable ones (std::vector) are
    /// staged through the engine's page-locked buffers (c4: 244 ms against 153 ms)
    void run(const uint16_t* q_res, std::size_t n, uint16_t* out);
    std::vector<uint16_t> run(const std::vector<uint16_t>& q_res, std::size_t n);

    std::size_t parts() const { return parts_; }
    std::size_t rows() const { return m_; }
    std::size_t inner() const { return k_; }
    std::size_t moduli() const { return nmod_; }
    uint64_t device_bytes() const;
    irl_ccmm* handle() { return e_; }

private:
    irl_ccmm* e_ = nullptr;
    std::size_t parts_, m_, k_, max_n_, nmod_;
};

/// The whole CCMM across devices from one process: one engine per entry of
/// `devices` (a device may repeat), parts dealt in contiguous blocks with the
/// a-part (part 0) on rank 0 (dist.part_range); ShapeMismatch if there are
/// more devices than parts.
class CcmmGroup {
public:
    CcmmGroup(const std::vector<int>& devices, std::size_t parts, std::size_t m, std::size_t k, std::size_t max_n,
              const modmat::RnsBasis& basis = modmat::build_paper_basis());
    ~CcmmGroup();
    CcmmGroup(const CcmmGroup&) = delete;
    CcmmGroup& operator=(const CcmmGroup&) = delete;

    std::size_t ranks() const { return ranks_; }
    std::size_t first_part(std::size_t rank) const;
    std::size_t rank_parts(std::size_t rank) const;
    /// counter-RNG synthetic database, every rank its global parts
    void synth_db(uint64_t seed);
    /// global part `part` streamed from the reference's BigMatrix file into its rank
    void load_part_file(std::size_t part, const std::string& path);
    /// IRL_EXCHANGE_* (irl_ccmm_group_set_exchange) / -1, 0, 1 (irl_ccmm_group_set_query_shard)
    void set_exchange(int mode);
    void set_query_shard(int mode);
    /// q_res [nmod][k][n] -> out [parts][nmod][n][m] (every part, global order);
    /// returns the IRL_EXCHANGE_* the a-part exchange used; a_out (nullable,
    /// ranks() entries): each rank's device copy of the a-part result
    int run(const uint16_t* q_res, std::size_t n, uint16_t* out, void** a_out = nullptr);
    std::vector<uint16_t> run(const std::vector<uint16_t>& q_res, std::size_t n);

private:
    void check(int st) const;
    irl_ccmm_group* g_ = nullptr;
    std::size_t ranks_, parts_, m_, k_, max_n_, nmod_;
};

}  // namespace b200
}  // namespace irislab

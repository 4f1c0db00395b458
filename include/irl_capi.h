/* irl_capi.h — C ABI of the B200-native PPMM / RGSW-CCMM engine.
 *
 * This is the drop-in boundary for the hot path of the reference
 * (/root/reference/proj, namespace irislab::modmat and emu::Emulator::ccmm_twin).
 * Every entry point names the reference interface it replaces (file:line
 * relative to /root/reference/proj). Signatures carry plain pointers and
 * sizes only: no torch, no C++ types. Two families:
 *
 *   (1) Blocking host-buffer calls that mirror the reference free functions
 *       value-for-value (row-major int32 SmallMatrix, fixed-width
 *       little-endian BigMatrix entries as in modmat.cpp:216-231);
 *   (2) the device-resident CCMM engine: database digit planes registered
 *       once in HBM, queries streamed per batch (host or device buffers).
 *
 * Errors: every call returns an irl_status. Codes 1-5 are the reference's
 * exception taxonomy (include/irislab/errors.hpp:9-53) and are raised under
 * exactly the conditions the reference throws; irl_last_error() returns the
 * message. There is no CPU fallback: without a usable sm_100 device,
 * irl_ctx_create fails with IRL_ERR_NO_DEVICE. */
#ifndef IRL_CAPI_H
#define IRL_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IRL_ABI_VERSION 1

typedef enum irl_status {
    IRL_OK = 0,
    IRL_ERR_SHAPE_MISMATCH = 1,             /* irislab::ShapeMismatch            errors.hpp:22 */
    IRL_ERR_MODULUS_TOO_LARGE = 2,          /* irislab::ModulusTooLarge          errors.hpp:27 */
    IRL_ERR_ACCUMULATION_OVERFLOW_RISK = 3, /* irislab::AccumulationOverflowRisk errors.hpp:30 */
    IRL_ERR_NOT_COPRIME = 4,                /* irislab::Error("CRT basis is not coprime") modmat.cpp:184 */
    IRL_ERR_MODULUS_BUDGET = 5,             /* irislab::ModulusBudget            errors.hpp:52 */
    IRL_ERR_INVALID_ARGUMENT = 6,
    IRL_ERR_CUDA = 7,
    IRL_ERR_NO_DEVICE = 8,
    IRL_ERR_OUT_OF_MEMORY = 9,
    IRL_ERR_UNSUPPORTED = 10,
    IRL_ERR_ZERO_OVERLAP = 11,              /* irislab::ZeroOverlap              errors.hpp:18 */
    IRL_ERR_IO = 12,                        /* irislab::Error("cannot open ..." / "truncated matrix file ...")
                                               modmat.cpp:218, 235, 245 */
    IRL_ERR_CONFIG = 13                     /* irislab::ConfigError              errors.hpp:13 */
} irl_status;

typedef struct irl_ctx irl_ctx;
typedef struct irl_ccmm irl_ccmm;
typedef struct irl_iris_db irl_iris_db;
typedef struct irl_ccmm_group irl_ccmm_group;

/* ---- context ------------------------------------------------------------ */
int irl_abi_version(void);
/* Binds `device`, creates a stream and workspace. IRL_ERR_NO_DEVICE if the
 * device is absent or not sm_100. */
int irl_ctx_create(int device, irl_ctx** out);
int irl_ctx_destroy(irl_ctx* ctx);
/* Message of the last failed call on this context ("" if none). */
const char* irl_last_error(const irl_ctx* ctx);
const char* irl_status_string(int status);
/* Kernels this context launched since creation (instrumentation). */
uint64_t irl_kernel_launches(const irl_ctx* ctx);
/* Stream used by the blocking calls (a cudaStream_t). */
void* irl_ctx_stream(const irl_ctx* ctx);
/* Diagnostics: enable per-CTA-pair cycle counters in the PPMM kernel for later
 * launches on this context; if out != NULL, first copy the last launch's
 * counters ([pair][16] uint64: producer empty/gate waits, MMA full/tmem waits,
 * MMA cycles, epilogue wait/busy, globaltimer start/end, tiles). */
int irl_diag_ppmm(irl_ctx* ctx, int enable, uint64_t* out, size_t cap);

/* ---- RNS basis helpers (modmat.cpp:8-63) -------------------------------- */
/* Primes 127..253 with e = 2 (build_paper_basis, modmat.cpp:37-45). Returns count. */
size_t irl_paper_basis(uint32_t* primes, uint32_t* exps, size_t cap);
/* Q = prod p^e, little-endian bytes; returns ceil(log256 Q) (modmat.cpp:219). */
size_t irl_basis_Q_bytes(const uint32_t* primes, const uint32_t* exps, size_t nmod, uint8_t* out,
                         size_t cap);

/* ---- blocking host-buffer mirrors of irislab::modmat --------------------- */
/* digit_decompose (modmat.hpp:72, modmat.cpp:86-106): rows*cols entries. */
int irl_digit_decompose(irl_ctx* ctx, const int32_t* m, size_t rows, size_t cols, uint32_t p,
                        int32_t* d0, int32_t* d1);
/* digit_recompose (modmat.hpp:73, modmat.cpp:108-118). */
int irl_digit_recompose(irl_ctx* ctx, const int32_t* d0, const int32_t* d1, size_t rows,
                        size_t cols, uint32_t p, int32_t* out);
/* small_gemm (modmat.hpp:77, modmat.cpp:120-141): C = A B, int32 accumulate,
 * same data-dependent AccumulationOverflowRisk precheck. Row-major. */
int irl_small_gemm(irl_ctx* ctx, const int32_t* a, const int32_t* b, int32_t* c, size_t m,
                   size_t k, size_t n);
/* gemm_mod_psq (modmat.hpp:80, modmat.cpp:143-160): C = A B mod p^2 in [0, p^2). */
int irl_gemm_mod_psq(irl_ctx* ctx, const int32_t* a, const int32_t* b, int32_t* c, size_t m,
                     size_t k, size_t n, uint32_t p);
/* gemm_mod_Q (modmat.hpp:83, modmat.cpp:162-195). Entries are `width`-byte
 * little-endian integers in [0, Q); basis = (primes[i], exps[i]). */
int irl_gemm_mod_Q(irl_ctx* ctx, const uint8_t* a, const uint8_t* b, uint8_t* c, size_t m,
                   size_t k, size_t n, size_t width, const uint32_t* primes, const uint32_t* exps,
                   size_t nmod);

/* ---- device-level building blocks (device pointers, stream-ordered) ------
 * Digit planes: [nmod][2][rows][ldk] int8, K-major, ldk % 16 == 0, zero
 * padded for k >= K. Residues: uint16 in [0, m). `stream` is a cudaStream_t
 * (NULL = the context stream). */
int irl_split_rows_u16(irl_ctx* ctx, const uint16_t* res, size_t ld_res, size_t plane_stride,
                       size_t rows, size_t cols, const uint32_t* primes, const uint32_t* exps,
                       size_t nmod, int8_t* planes, size_t ldk, void* stream);
/* Transposing split of a K x N residue matrix (reference B layout) into
 * [nmod][2][N][ldk] planes. */
int irl_split_cols_u16(irl_ctx* ctx, const uint16_t* res, size_t ld_res, size_t plane_stride,
                       size_t k, size_t n, const uint32_t* primes, const uint32_t* exps,
                       size_t nmod, int8_t* planes, size_t ldk, void* stream);
/* Residue extraction + split of width-byte mod-Q entries (modmat.cpp:168-176
 * fused with :86-106). transpose=0: rows x cols matrix -> [nmod][2][rows][ldk];
 * transpose=1: K x N matrix -> [nmod][2][N][ldk]. */
int irl_split_bigint(irl_ctx* ctx, const uint8_t* entries, size_t width, size_t rows, size_t cols,
                     int transpose, const uint32_t* primes, const uint32_t* exps, size_t nmod,
                     int8_t* planes, size_t ldk, void* stream);
/* Batched PPMM over planes: out[g][i][n][m] = (A_g,i B_i^T) mod p_i^e.
 * a_planes [parts][nmod][2][M][ldk], b_planes [nmod][2][N][ldk],
 * out [parts][nmod][N][M]; accumulate=1 adds into out mod p^e. */
int irl_ppmm_planes(irl_ctx* ctx, const int8_t* a_planes, const int8_t* b_planes, uint16_t* out,
                    size_t parts, size_t m, size_t n, size_t k, size_t ldk,
                    const uint32_t* primes, const uint32_t* exps, size_t nmod, int accumulate,
                    void* stream);
/* RNS rescale / ModDown toward Q / Delta (the
 * CCMM result lives modulo ~Q/Delta). Delta = product of the LAST `drop`
 * moduli (< 2^48). For every element e, the residues in[i*ld_in + e] of
 * x mod Q (the CRT lift of modmat.cpp:178-193) become the residues
 * out[i*ld_out + e], i < nmod - drop, of floor((x + (round ? floor(Delta/2) : 0)) / Delta)
 * mod Q/Delta. Device pointers, stream-ordered. Inputs may be any uint16
 * (reduced mod m_i first). Error("CRT basis is not coprime") as the lift. */
int irl_rescale_residues(irl_ctx* ctx, const uint16_t* in, size_t ld_in, size_t count, const uint32_t* primes,
                         const uint32_t* exps, size_t nmod, size_t drop, int round, uint16_t* out, size_t ld_out,
                         void* stream);
/* CRT lift (modmat.cpp:178-193): residues [nmod][N][M] -> width-byte entries
 * of the M x N row-major result mod Q. */
int irl_crt_lift(irl_ctx* ctx, const uint16_t* res, size_t m, size_t n, uint8_t* out,
                 size_t width, const uint32_t* primes, const uint32_t* exps, size_t nmod,
                 void* stream);

/* ---- synthetic inputs (counter-based, identical on host and device) ------ */
/* residue = floor(hi32(mix64(key ^ mix64(seed))) * m / 2^32),
 * key = stream<<56 | plane<<48 | row<<24 | col. */
uint32_t irl_synth_residue(uint64_t seed, uint32_t stream, uint32_t plane, uint32_t row,
                           uint32_t col, uint32_t m);
void irl_synth_residues_host(uint64_t seed, uint32_t stream, uint32_t plane, uint32_t row0,
                             uint32_t nrows, uint32_t col0, uint32_t ncols, uint32_t m,
                             uint16_t* out);

/* ---- RGSW CCMM engine (caller emulator.cpp:389-447)
 * A database of `parts` parts (paper layout: part 0 = shared a-part
 * [A1|A2], parts 1.. = b-part slices [B1|B2]); each part is M x K with
 * K = d2 + N_qry, stored once as digit planes in HBM. A query batch is the
 * K x N residue matrix [Bq; Aq] per modulus. One run computes, per part and
 * modulus, out = [X1|X2] [Bq; Aq] mod p^e — the two PPMMs of that part fused
 * by K-concatenation — with outputs [parts][nmod][N][M] (column n of part g
 * is the coefficient vector of the n-th output ciphertext block). */
int irl_ccmm_create(irl_ctx* ctx, size_t parts, size_t m, size_t k, size_t max_n,
                    const uint32_t* primes, const uint32_t* exps, size_t nmod, irl_ccmm** out);
int irl_ccmm_destroy(irl_ccmm* e);
/* Register part `part` from residues [nmod][M][K] (host or device pointer). */
int irl_ccmm_load_part(irl_ccmm* e, size_t part, const uint16_t* res, int res_on_device);
/* Register part `part` from width-byte mod-Q entries [M][K] (host pointer). */
int irl_ccmm_load_part_bigint(irl_ccmm* e, size_t part, const uint8_t* entries, size_t width);
/* Stream one part from the reference's BigMatrix file (save_big_matrix,
 * modmat.cpp:216-231): header "rows cols Q" must match (M, K, the basis Q);
 * entries are read in 256 MB chunks, double-buffered against the H2D and the
 * residue/digit split, so a part never has to fit in host memory.
 * Error("truncated matrix file ...") as load_big_matrix (modmat.cpp:233-249). */
int irl_ccmm_load_part_file(irl_ccmm* e, size_t part, const char* path);
/* Fill every part with synthetic residues irl_synth_residue(seed, first_part + part,
 * i, row, col, m_i); first_part is the global id of local part 0 (multi-GPU). */
int irl_ccmm_synth_db(irl_ccmm* e, uint64_t seed, uint32_t first_part);
/* Fill local part `part` with rows [row0, row0 + M) of global part
 * global_part of the same synthetic database (a row block of a taller part:
 * the balanced row-block dealing of dist.deal_blocks). */
int irl_ccmm_synth_part(irl_ccmm* e, size_t part, uint64_t seed, uint32_t global_part, uint32_t row0);
/* End-to-end call with HOST buffers: q_res [nmod][K][N] -> out [parts][nmod][N][M].
 * Copies in, splits, multiplies every part, copies out; blocks. N may exceed
 * max_n: the batch then streams through the engine in column chunks
 * (max_n rounded down to whole 256-column tiles), e.g. the c5 corner of 256
 * eyes x 31 rotations against 2^17-template slices. Host buffers should be
 * pinned (cudaHostAlloc / cudaHostRegister): pageable buffers are staged by the
 * driver and copy at a fraction of PCIe bandwidth. */
int irl_ccmm_run(irl_ccmm* e, const uint16_t* q_res_host, size_t n, uint16_t* out_host);
/* Query already on the device (q_res_dev [nmod][K][n], NULL = the engine's
 * staging buffer, stream-ordered after `stream`), outputs to HOST memory:
 * split, one PPMM launch over every part and modulus, and (modulus, part)-
 * granular D2H overlapped with the launch; blocks. For multi-GPU callers that
 * distribute the query over NVLink (each rank copies 1/N of it from the host
 * and all-gathers the rest) instead of N full host copies. n <= max_n. */
int irl_ccmm_run_dq(irl_ccmm* e, const uint16_t* q_res_dev, size_t n, uint16_t* out_host, void* stream);
/* Device-resident variant over parts [part0, part0 + nparts): q_res_dev
 * [nmod][K][N] (split into the engine's query planes unless q_ready != 0),
 * out_dev [nparts][nmod][N][M]; stream-ordered, does not block. */
int irl_ccmm_run_device(irl_ccmm* e, const uint16_t* q_res_dev, int q_ready, size_t n,
                        size_t part0, size_t nparts, uint16_t* out_dev, void* stream);
/* Device staging buffers owned by the engine: query residues [nmod][K][max_n]
 * and outputs [parts][nmod][n][M] (written by irl_ccmm_run, and by
 * irl_ccmm_run_device when out_dev is NULL; q_res_dev NULL reads *qres). */
int irl_ccmm_buffers(irl_ccmm* e, void** qres, void** out);
/* ---- CCMM caller drop-in (emulator.cpp:389-447, Emulator::ccmm_twin) -----
 * Validates exactly like ccmm_twin (ShapeMismatch for non-positive dims,
 * d1 % n_db, d2 % n_qry, slot output without ci; ModulusBudget for
 * db_bits < 2 q_bits - delta and out_level outside [0, top_level]) and
 * computes the product db (d1 x d2) . qry (d2 x d3) bit-identical to the
 * reference's double loop (emulator.cpp:411-421): integer-valued operands with
 * K max|db| max|qry| < 2^52 (every partial sum exact) on the int8 tensor-core
 * PPMM (residues mod a prefix of the paper basis, centred CRT on device); any
 * other doubles (fractions, larger magnitudes, inf/NaN) on an FP64 kernel that
 * replays the loop's rounded multiply and add per k in order, skipping zero
 * database entries. msgs receives the d1*d3/n_db output ciphertext messages in
 * ccmm_twin's order: msgs[(c*(d1/n_db) + b)*n_db + i] = prod[(b*n_db + i)*d3 + c]. */
int irl_ccmm_twin(irl_ctx* ctx, long d1, long d2, long d3, long n_db, long n_qry,
                  double db_modulus_bits, double qry_modulus_bits, double scale_bits,
                  int out_level, int top_level, int out_slot_encoding, int out_ci,
                  const double* db, const double* qry, double* msgs);
/* ---- fused a-part exchange (replaces the NCCL broadcast) -----
 * Receivers allocate an engine-owned receive buffer of IRL_RECV_SLOTS slots
 * [slot][nmod][n][M] uint16 and export its CUDA IPC handle (64 bytes); the
 * owner of part `part` opens the peers' handles, and from then on the epilogue
 * of that part's PPMM stores every output tile both locally and into slot
 * `mirror_slot` (irl_ccmm_set_mirror_slot) of each peer buffer (NVLink P2P
 * stores, overlapped with the GEMM; a system-scope fence per tile). The data
 * is complete in a peer once the owner's launch has completed: order the
 * peers' reads after it with any cross-GPU signal (e.g. a tiny NCCL
 * all-reduce posted after the GEMM). Alternating the slot per step makes the
 * buffer double-buffered: step s+1 writes the other slot while peers still
 * read step s, and step s+2 may overwrite slot s once every peer has posted
 * its step-(s+1) signal after consuming step s. Mirroring applies to device
 * runs and single-column-chunk e2e runs of width n; count 0 disables it. At
 * most 7 peers. */
#define IRL_RECV_SLOTS 2
int irl_ccmm_alloc_recv(irl_ccmm* e, size_t n, void** dev_ptr, uint8_t* ipc_handle /* 64 B, nullable */);
int irl_ccmm_set_mirrors(irl_ccmm* e, size_t part, size_t n, const uint8_t* ipc_handles /* count x 64 B */,
                         size_t count);
/* Same with raw device pointers (same-process peers / tests). */
int irl_ccmm_set_mirror_ptrs(irl_ccmm* e, size_t part, size_t n, uint16_t* const* dev_ptrs, size_t count);
/* Slot (< IRL_RECV_SLOTS) of the peers' receive buffers the next runs store
 * into; peer buffers given by pointer must hold slot + 1 slots. */
int irl_ccmm_set_mirror_slot(irl_ccmm* e, size_t slot);
/* Mirror local parts [part, part + count) (part from the last set_mirrors /
 * set_mirror_ptrs, which reset count to 1): the a-part spans several local
 * parts when the database is dealt in row blocks (dist.deal_blocks). Peer
 * buffers then hold [slot][count][nmod][n][M]; receivers allocate them with
 * irl_ccmm_alloc_recv_parts. */
int irl_ccmm_set_mirror_parts(irl_ccmm* e, size_t count);
int irl_ccmm_alloc_recv_parts(irl_ccmm* e, size_t n, size_t parts, void** dev_ptr,
                              uint8_t* ipc_handle /* 64 B, nullable */);
/* NVLS multicast mirror: mc_addr is a multicast address (cuMulticastCreate +
 * cuMemMap) whose object binds one receive buffer per GPU; the epilogue of
 * part `part` stores each pair of output rows there once (multimem.st) and the
 * switch writes every bound copy (at slot `mirror_slot`, so the bound
 * buffers hold IRL_RECV_SLOTS slots). Needs an even M. NULL disables it. */
int irl_ccmm_set_mirror_multicast(irl_ccmm* e, size_t part, size_t n, void* mc_addr);
/* ModDown of the engine's outputs (after irl_ccmm_run_device wrote them to the
 * engine buffer, n columns): parts [part0, part0 + nparts) of [parts][nmod][n][M]
 * -> dst [nparts][nmod - drop][n][M] (device), see irl_rescale_residues. */
int irl_ccmm_rescale(irl_ccmm* e, size_t n, size_t part0, size_t nparts, size_t drop, int round, uint16_t* dst,
                     void* stream);
/* Bytes of HBM the engine holds (planes + workspace). */
uint64_t irl_ccmm_device_bytes(const irl_ccmm* e);
/* ---- single-process multi-GPU CCMM (SURVEY §8(b) irl_ccmm_full)
 * One context and engine per entry of devices[] (an entry may repeat a device).
 * The parts are dealt in contiguous blocks, rank r holding parts
 * [first_r, first_r + count_r) with first_r = r*(parts/ndev) + min(r, parts%ndev),
 * so the a-part (part 0) sits on rank 0. Register each rank's parts through its
 * engine (irl_ccmm_group_engine; local part i is global part first_r + i).
 * ShapeMismatch if ndev > parts. */
int irl_ccmm_group_create(const int* devices, size_t ndev, size_t parts, size_t m, size_t k, size_t max_n,
                          const uint32_t* primes, const uint32_t* exps, size_t nmod, irl_ccmm_group** out);
int irl_ccmm_group_destroy(irl_ccmm_group* g);
/* The a-part exchange of irl_ccmm_full. AUTO: P2P stores from rank 0's PPMM
 * epilogue into each peer's receive buffer, else a cudaMemcpyPeer after the
 * runs. MULTICAST (opt-in): one rank per multicast-capable device; rank 0's
 * epilogue stores each output pair once to an NVLS multicast address and the
 * switch writes every rank's copy (also valid with a single rank). MULTICAST
 * and P2P fail with UNSUPPORTED where the driver refuses them. */
enum { IRL_EXCHANGE_AUTO = 0, IRL_EXCHANGE_P2P = 1, IRL_EXCHANGE_MULTICAST = 2, IRL_EXCHANGE_COPY = 3 };
int irl_ccmm_group_set_exchange(irl_ccmm_group* g, int mode);
int irl_ccmm_group_engine(irl_ccmm_group* g, size_t rank, irl_ccmm** e, size_t* first_part, size_t* nparts);
/* Context of a rank (irl_last_error of group calls is on rank 0's). */
irl_ctx* irl_ccmm_group_ctx(irl_ccmm_group* g, size_t rank);
/* Query distribution of irl_ccmm_full. -1 (default, auto): sharded when
 * every rank holds about one paper-size part (parts x M < 20000 rows), where a
 * rank's GEMM per modulus is shorter than its H2D; 0: every rank copies the
 * whole query from the host (irl_ccmm_run); 1: sharded -- rank r copies its
 * 1/ndev of the moduli from the host and pushes it to every other rank over
 * peer memory (the paper's query AllGather), then every rank runs
 * on the staged query (irl_ccmm_run_dq). Outputs are identical. */
int irl_ccmm_group_set_query_shard(irl_ccmm_group* g, int mode);
/* The full CCMM across the devices with HOST buffers: q_res [nmod][K][n] ->
 * out [parts][nmod][n][M] (every part, in global order); each rank runs its
 * parts end to end (irl_ccmm_run) concurrently with the others. The a-part
 * result also lands on every rank through the exchange above (*mode gets the
 * IRL_EXCHANGE_* in use); a_out (nullable, ndev entries) receives each rank's
 * device pointer to its copy [nmod][n][M]. n <= max_n. Blocks. */
int irl_ccmm_full(irl_ccmm_group* g, const uint16_t* q_res_host, size_t n, uint16_t* out_host, void** a_out,
                  int* mode);

/* ---- plaintext iris scoring stage ---------------------------
 * Templates are packed bit planes in pack_bits order (pipeline.cpp:70-76):
 * bit i of template t is bit (i % 64) of word t*words + i/64, words =
 * ceil(d/64); code and mask planes separate. The query side is n_eyes
 * templates; column c = e*rho + r of the query batch is rotate(q_e, r)
 * (iris_core.cpp:65-76), as in pipeline::prepare (pipeline.cpp:121-138).
 * Both sums are tensor-core GEMMs (PPMM kernel): e2m1 operands on the
 * block-scaled FP4 path, exact in FP32 accumulation (int8 with IRL_IRIS_I8=1).
 *
 * inner[c][j]   = <to_masked(q_c), to_masked(db_j)>    (iris_core.cpp:37-51)
 * overlap[c][j] = |m_q(c) AND m_db(j)|                  (overlap_count, pipeline.cpp:78-82;
 *                 prepare's overlaps[c*blocks + b][i] = overlap[c][b*d_blk + i], :140-151)
 * Either output may be NULL. ShapeMismatch if d == 0 (IrisTemplate::validate). */
int irl_iris_inner_overlap(irl_ctx* ctx, const uint64_t* db_code, const uint64_t* db_mask, size_t n_db,
                           const uint64_t* q_code, const uint64_t* q_mask, size_t n_eyes, size_t rho,
                           size_t d, int32_t* inner, int32_t* overlap);
/* Scores and matching (iris_core.cpp:55-59, 78-90): score = inner / overlap in
 * IEEE double. match_bits[e][j] = OR over r of score(c = e*rho + r, j) in
 * [p_lo, p_hi]; eye_result[e] = match_db_reference(rotations of eye e, db):
 * 1 match, 0 none, -1 ZeroOverlap (the first evaluated score in its
 * rotation-major loop order had an empty overlap before any match). Returns
 * IRL_ERR_ZERO_OVERLAP if any eye hit that case (outputs still written).
 * scores[c][j] (optional) is NaN where the overlap is empty. */
int irl_iris_match(irl_ctx* ctx, const uint64_t* db_code, const uint64_t* db_mask, size_t n_db,
                   const uint64_t* q_code, const uint64_t* q_mask, size_t n_eyes, size_t rho, size_t d,
                   double p_lo, double p_hi, uint8_t* match_bits, int32_t* eye_result, double* scores);
/* Device-resident template database: the enrolled templates become int8
 * planes in HBM once; each irl_iris_db_match moves only the query eyes' bits
 * (same outputs and semantics as irl_iris_match; n_eyes * rho <= max_cols). */
int irl_iris_db_create(irl_ctx* ctx, const uint64_t* db_code, const uint64_t* db_mask, size_t n_db, size_t d,
                       size_t max_cols, irl_iris_db** out);
/* Same database straight from the reference's template file (save_templates,
 * iris_core.cpp:183-196: {magic "IRIT", version 1, n_db, d} then the code and
 * mask planes, little-endian bit order); returns n_db and d. Errors as
 * load_templates (iris_core.cpp:198-215): bad magic / version / truncated. */
int irl_iris_db_create_file(irl_ctx* ctx, const char* path, size_t max_cols, irl_iris_db** out, size_t* n_db,
                            size_t* d);
int irl_iris_db_destroy(irl_iris_db* e);
int irl_iris_db_match(irl_iris_db* e, const uint64_t* q_code, const uint64_t* q_mask, size_t n_eyes, size_t rho,
                      double p_lo, double p_hi, uint8_t* match_bits, int32_t* eye_result, double* scores);

/* ---- Alg. 2 fold stage at message level ----------------------
 * run_alg2 (pipeline.cpp:538-633) after the CCMM: for eye e, DB block b
 * (blocks = n_db / d) and rotation group g (groups = ceil(rho / fold_k);
 * group g holds rotations r = g*fold_k .. min(rho, (g+1)*fold_k) - 1):
 *
 *   x_r[j]      = inner[c][b*d + j] * (1.0 / overlap[c][b*d + j]),  c = e*rho + r
 *                 (normalize, pipeline.cpp:359-371: pmult by the inverse overlaps)
 *   folded[i]   = sum over the group's r, in order, of f(x_r)[(i + r) mod d]
 *                 (fold_group, pipeline.cpp:391-408: fold_poly, then rot by
 *                 base_rot + s = r, emulator.cpp:232-245)
 *   refolded[i] = sum over g of chain(folded_g)[i]   (pipeline.cpp:612-627;
 *                 eval_chain_ct, pipeline.cpp:379-389: per stage add_const(-center)
 *                 then the stage polynomial; the bootstrap in between,
 *                 boot(bts_fold_pre), leaves the message unchanged)
 *
 * Every polynomial runs the reference's Paterson-Stockmeyer plan
 * (poly.hpp:46-119, ring ops of CtRing pipeline.cpp:22-44) in IEEE double
 * with the same operation order and no contraction, so the outputs equal the
 * noise-free emulator's messages (Emulator(cfg, inject_noise = false)) bit
 * for bit. Degrees (index of the last nonzero coefficient, poly.cpp:10-15) up
 * to 31; up to 8 chain stages. The inner / overlap inputs are the CCMM
 * product and the mask overlaps in the [c][n_db] layout of
 * irl_iris_inner_overlap (prepare's overlaps[c*blocks + b][j], pipeline.cpp:140-151).
 *
 * assumption_ok = run_alg2's folding-assumption shadow check (pipeline.cpp:565-590):
 * for every (e, b, i, g), at most one r in the group has overlap 0 or
 * raw / overlap outside [negative_lo, negative_hi].
 *
 * Errors, in the reference's order: ConfigError from PipelineConfig::validate
 * (pipeline.cpp:232-243: rho, batch >= 1; 1 <= fold_k <= rho; d a power of
 * two >= 2; n_db a positive multiple of d), ConfigError("eval_chain_ct: empty
 * chain") if refolded is requested with no stages, UNSUPPORTED for degree > 31
 * or more than 8 stages, and ZeroOverlap if any overlap is 0 (normalize
 * throws, pipeline.cpp:367; outputs are still written). */
typedef struct irl_fold_params {
    size_t batch, rho, n_db, d, fold_k;  /* PipelineConfig fields (pipeline.hpp:16-40) */
    const double* fold_coeffs;           /* fold_poly.coeffs, ascending degree */
    size_t fold_len;
    size_t chain_stages;                 /* fold_chain.stages.size() */
    const double* chain_centers;         /* [chain_stages] stage.center */
    const size_t* chain_lens;            /* [chain_stages] stage.poly.coeffs.size() */
    const double* chain_coeffs;          /* the stages' coefficients, concatenated */
    double negative_lo, negative_hi;     /* cfg.model.negative */
} irl_fold_params;

/* Host buffers, blocking. inner / overlap: int32 [batch*rho][n_db].
 * folded: [batch][blocks][groups][d], refolded: [batch][blocks][d] (each may
 * be NULL); assumption_ok (may be NULL) gets 1 / 0. */
int irl_fold_stage(irl_ctx* ctx, const irl_fold_params* p, const int32_t* inner, const int32_t* overlap,
                   double* folded, double* refolded, int32_t* assumption_ok);
/* Device buffers, stream-ordered (stream NULL = the context stream). flags:
 * device uint32[2], OR-ed into: [0] folding assumption violated, [1] an
 * overlap was 0 (the host call's ZeroOverlap). */
int irl_fold_stage_device(irl_ctx* ctx, const irl_fold_params* p, const int32_t* inner, const int32_t* overlap,
                          double* folded, double* refolded, uint32_t* flags, void* stream);
/* The whole post-CCMM path of run_alg2 against a registered template
 * database: prepare's products and overlaps of the query eyes
 * (p->batch = n_eyes, the database's n_db and template length = p->n_db and
 *  p->d; ShapeMismatch otherwise, pipeline.cpp:100-118) as tensor-core GEMMs, then
 * the fold stage on the device; only folded / refolded leave it. */
int irl_iris_db_fold(irl_iris_db* e, const uint64_t* q_code, const uint64_t* q_mask, const irl_fold_params* p,
                     double* folded, double* refolded, int32_t* assumption_ok);

#ifdef __cplusplus
}
#endif

#endif /* IRL_CAPI_H */

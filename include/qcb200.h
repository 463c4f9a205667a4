/*
 * qcb200.h -- C ABI of libqcb200.so, the B200-native (sm_100a) batched
 * QC-LDPC codec for the IEEE 802.11 (Wi-Fi) and 802.16 (WiMAX) codes.
 *
 * Plain pointers and sizes only; no torch or numpy types cross this line.
 * All functions return QC_OK (0) on success, a negative QC_E* code for bad
 * arguments / unsupported codes, or a positive cudaError_t value when a CUDA
 * call failed.  qc_last_error() gives a human-readable message for the last
 * failure on the calling thread.  Every entry point is thread-safe; calls on
 * disjoint outputs may run concurrently (the reference's nogil contract,
 * /root/reference/pkg/src/qcldpc/_kernels.py:17,103).
 *
 * Reference interfaces replaced (see INTEGRATION.md for the bindings):
 *   qc_decode_batch_f32_host  <- _kernels.decode_batch_f32
 *                                /root/reference/pkg/src/qcldpc/_kernels.py:17-19
 *   qc_decode_batch_i16_host  <- _kernels.decode_batch_i16  (_kernels.py:103-105)
 *     Same ten arguments (CSR row_ptr/col_idx, mb, z, LLR block, max_iters,
 *     early_term, caller-owned hard/iters/conv), host memory in and out.
 *   qc_decode_f32 / qc_decode_i16 <- the same kernels, device-resident
 *     buffers, stream ordered, optional bit-packed hard decisions and
 *     posterior LLRs out (the north-star "LLRs out" extension).
 *   qc_decode_grouped_f32 / _i16 <- decoder.decode_block over several codes
 *     (decoder.py:217-258), one call for a mixed-code batch.
 *   qc_encode_packed(_host) <- encoder.encode_packed (encoder.py:166-199).
 *   qc_code_create / qc_code_from_csr <- codebook.get_model_matrix + expand
 *     (codebook.py:203-266): a code is its mb x nb shift table; no expanded
 *     H is ever materialised on the device.
 */
#ifndef QCB200_H
#define QCB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QC_OK 0
#define QC_EINVAL (-1)        /* bad argument (null pointer, negative size, ...)           */
#define QC_EUNSUPPORTED (-2)  /* code shape not supported (row degree > 32, CSR not QC)    */
#define QC_ENOMEM (-3)        /* host allocation failed                                    */
#define QC_EMALFORMED (-4)    /* h_b column lacks one interior entry (encoder.py:39-46)   */
#define QC_EUNALIGNED (-5)    /* packed encoder needs Z % 8 == 0 (encoder.py:59-61)       */

typedef struct qc_code_s* qc_code_t;

/* ABI version (major*100 + minor). */
int qc_version(void);
/* Message for the last failure on this thread ("" if none). */
const char* qc_last_error(void);

/* Create a code from its mb x nb shift table (row-major, -1 = zero block,
 * 0 <= s < z otherwise).  kb = nb - mb.  The table is copied. */
int qc_code_create(int32_t mb, int32_t nb, int32_t z, const int32_t* shifts, qc_code_t* out);
/* Recover the shift table from the reference kernel's CSR arguments
 * (row_ptr[mb*z+1], col_idx[n_edges], mb, z, n = number of columns).
 * Returns QC_EUNSUPPORTED if the CSR is not a quasi-cyclic expansion. */
int qc_code_from_csr(const int32_t* row_ptr, int64_t row_ptr_len, const int32_t* col_idx,
                     int64_t n_edges, int32_t mb, int32_t z, int32_t n, qc_code_t* out);
int qc_code_destroy(qc_code_t code);
/* Shape query; any output pointer may be NULL.  kernel = 1 when the
 * specialised (unrolled, register-resident) decoder serves this code,
 * 0 when the generic decoder does. */
int qc_code_info(qc_code_t code, int32_t* mb, int32_t* nb, int32_t* z, int32_t* n_edges,
                 int32_t* max_row_degree, int32_t* kernel);

/* ---- device-resident decode (stream ordered; all pointers device memory) --
 * llr:  w x n values, C-contiguous.
 * hard: w x n bytes (0/1, hard_packed = 0) or w x ceil(n/8) bytes MSB-first
 *       (hard_packed = 1, np.packbits layout).
 * iters: w int32, conv: w uint8.  post_out: w x n values or NULL.
 * max_iters >= 0; early_term: 0 = fixed iterations, 1 = stop a codeword at
 * its first zero syndrome (_kernels.py:85-96). */
int qc_decode_f32(qc_code_t code, const float* llr, int64_t w, int32_t max_iters,
                  int32_t early_term, uint8_t* hard, int32_t hard_packed, int32_t* iters,
                  uint8_t* conv, float* post_out, void* cuda_stream);
int qc_decode_i16(qc_code_t code, const int16_t* llr, int64_t w, int32_t max_iters,
                  int32_t early_term, uint8_t* hard, int32_t hard_packed, int32_t* iters,
                  uint8_t* conv, int16_t* post_out, void* cuda_stream);

/* ---- mixed-code batch: one job per code.  Every job is validated first
 * (arguments, and the generic kernel's shared-memory fit); the jobs then fork
 * from cuda_stream onto side streams and join back (stream ordered,
 * graph-capturable), so the codes decode concurrently.  If a CUDA launch
 * fails part-way the call returns its error and the outputs are unspecified.
 * Set QCB_GROUPED_SERIAL=1 to queue the jobs one after another on cuda_stream. */
typedef struct {
  qc_code_t code;
  const void* llr;   /* device, w x n float32 or int16 (per call) */
  int64_t w;
  uint8_t* hard;     /* device */
  int32_t* iters;    /* device */
  uint8_t* conv;     /* device */
  void* post_out;    /* device or NULL */
} qc_decode_job_t;
int qc_decode_grouped_f32(const qc_decode_job_t* jobs, int32_t n_jobs, int32_t max_iters,
                          int32_t early_term, int32_t hard_packed, void* cuda_stream);
int qc_decode_grouped_i16(const qc_decode_job_t* jobs, int32_t n_jobs, int32_t max_iters,
                          int32_t early_term, int32_t hard_packed, void* cuda_stream);

/* ---- host-buffer drop-ins for _kernels.decode_batch_f32 / _i16 -----------
 * Arguments in the reference order.  llrs/hard are w x n row-major host
 * arrays; hard is unpacked (one byte per bit).  Blocks until the outputs are
 * written.  Uses the current CUDA device.  The block streams through the
 * device in ~32 MB chunks on three streams; page-locked caller buffers are
 * copied directly by DMA, pageable ones (plain numpy, as decode_block passes
 * them) through pinned staging slots filled / drained by a host copy pool
 * (QCB_COPY_THREADS threads) while the previous chunks transfer and decode. */
int qc_decode_batch_f32_host(const int32_t* row_ptr, int64_t row_ptr_len, const int32_t* col_idx,
                             int64_t n_edges, int32_t mb, int32_t z, const float* llrs, int64_t w,
                             int64_t n, int32_t max_iters, int32_t early_term, uint8_t* hard,
                             int32_t* iters, uint8_t* conv);
int qc_decode_batch_i16_host(const int32_t* row_ptr, int64_t row_ptr_len, const int32_t* col_idx,
                             int64_t n_edges, int32_t mb, int32_t z, const int16_t* llrs, int64_t w,
                             int64_t n, int32_t max_iters, int32_t early_term, uint8_t* hard,
                             int32_t* iters, uint8_t* conv);

/* ---- packed direct encoder (byte-aligned Z) --------------------------------
 * info: w x K/8 bytes MSB-first; cw: w x N/8 bytes = [info | parity]. */
int qc_encode_packed(qc_code_t code, const uint8_t* info, int64_t w, uint8_t* cw, void* cuda_stream);
int qc_encode_packed_host(qc_code_t code, const uint8_t* info, int64_t w, uint8_t* cw);
/* Bit-granular packed encoder for every Z <= 97: info = np.packbits of the
 * K info bits (W x ceil(K/8) bytes), cw = np.packbits of the N codeword bits, i.e. exactly
 * pack_bits(encode_array(...)) (encoder.py:103-104, 133-163) -- the layout the reference's
 * packed encoder refuses for Z % 8 != 0 (encoder.py:59-61).  Byte-aligned Z: same as
 * qc_encode_packed. */
int qc_encode_bits(qc_code_t code, const uint8_t* info, int64_t w, uint8_t* cw, void* cuda_stream);

/* ---- channel, waterfall counters and decode records -------
 * All pointers device memory, stream ordered.
 *
 * qc_encode_array   <- encoder.encode_array (encoder.py:133-163): one bit per
 *   byte, any Z (the packed encoder needs Z % 8 == 0).  w x K in, w x N out.
 * qc_frames_info    <- chansim._gen_batch's info bits (chansim.py:126-133),
 *   drawn from a device Philox4x32-10 stream keyed by (seed, point, frame):
 *   independent of launch shape and GPU count, NOT numpy's stream.
 * qc_channel_llr    <- chansim._llr_batch (chansim.py:136-143): BPSK, AWGN,
 *   LLR = (2/sigma2) y cast to float32 and, for q_b > 0, quantize_llr
 *   (decoder.py:165-171) to int16.  noise != NULL: the caller's float64
 *   standard normal samples (bit-exact with the reference for the same
 *   samples); noise == NULL: device Philox noise for frames frame0.. .
 * qc_quantize_llr   <- decoder.quantize_llr on float32 LLRs.
 * qc_count_errors   <- run_waterfall's counting (chansim.py:166-171): per
 *   `batch` consecutive frames, {bit errors over the K info bits, frame
 *   errors, iteration sum} as uint64 triples (zeroed by the call).
 * qc_pack_records   <- the CLI decode output (cli.py:180-183): per codeword
 *   ceil(N/8) packed hard bytes, min(iters, 255), converged.
 */
int qc_encode_array(qc_code_t code, const uint8_t* info_bits, int64_t w, uint8_t* cw_bits, void* cuda_stream);
int qc_frames_info(uint64_t seed, uint32_t point, int64_t frame0, int64_t w, int32_t k, uint8_t* info_bits,
                   void* cuda_stream);
int qc_channel_llr(const uint8_t* cw_bits, int64_t w, int32_t n, double sigma2, const double* noise,
                   uint64_t seed, uint32_t point, int64_t frame0, int32_t q_b, double l_clip, void* llr,
                   void* cuda_stream);
int qc_quantize_llr(const float* x, int64_t count, int32_t q_b, double l_clip, int16_t* out, void* cuda_stream);
int qc_count_errors(const uint8_t* hard, int32_t hard_packed, const uint8_t* info_bits, const int32_t* iters,
                    int64_t w, int32_t n, int32_t k, int32_t batch, uint64_t* batch_sums, void* cuda_stream);
int qc_pack_records(const uint8_t* hard_packed, const int32_t* iters, const uint8_t* conv, int64_t w, int32_t n,
                    uint8_t* records, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* QCB200_H */

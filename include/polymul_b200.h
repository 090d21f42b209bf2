/*
 * polymul_b200.h -- C ABI of the B200 sparse polynomial multiplier.
 *
 * The reference package (`polymul`, pure Python) has no FFI layer: its hot
 * path is the Python call
 *
 *     polymul.parmul.mul(a, b, cfg=None, *, split=None) -> Polynomial
 *         (reference pkg/src/polymul/parmul.py:91-109)
 *
 * and its operands are `Polynomial` objects holding a strictly ascending
 * list of packed u64 exponents plus a parallel coefficient list
 * (reference core.py:211-241).  This header is the binding a maintainer adds
 * beneath that call: plain pointers and sizes, no framework types.  The
 * Python mirror (`paper_1303_7425_b200.parmul.mul`) marshals a Polynomial into
 * `pgpu_poly` and calls `pgpu_mul`; see INTEGRATION.md for the ctypes stub.
 *
 * Entry point -> reference interface it replaces:
 *   pgpu_mul            parmul.mul (parmul.py:91-109): select_grid + find_edge +
 *                       heap_merge/tree_merge + concat, i.e. the whole product
 *   pgpu_count_below    split.count_ops / parmul.interval_op_counts
 *                       (split.py:169-175, parmul.py:112-116): cumulative pair
 *                       counts at bounds, the input of cluster.partition_by_ops
 *                       (cluster.py:261-280)
 *   pgpu_free_result    (ownership of the result lists; Python GC in the reference)
 *   pgpu_last_error     exception messages (ValueError / ExponentOverflowError,
 *                       core.py:333-337, core.py:365-385)
 *   pgpu_device_count   (cluster node count; cluster.py:330)
 *   pgpu_format         io.format_poly / io.write_poly term lines
 *                       (io.py:241-248, io.py:306-308): the PolyFile text of a
 *                       product, formatted on the device
 *   pgpu_free_text      (ownership of the text; Python str in the reference)
 *   pgpu_ipc_*          the final gather of paper Alg. 2 (cluster.py:365-379:
 *                       nodes' disjoint results concatenated in rank order) as
 *                       peer copies over NVLink: a shareable result buffer per
 *                       rank, its CUDA IPC handle, and device-to-device copies
 *                       of each rank's slice into every peer's buffer
 *
 * Every function returns a pgpu_status; on failure pgpu_last_error() holds a
 * message for the calling thread.  No function falls back to the CPU.
 */
#ifndef POLYMUL_B200_H
#define POLYMUL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGPU_MAX_FIELDS 15
#define PGPU_ABI_VERSION 3

typedef enum pgpu_status {
  PGPU_OK = 0,
  PGPU_EINVAL = 1,        /* malformed arguments (ValueError in the reference)      */
  PGPU_EEXPONENT = 2,     /* a product exponent overflows its field
                             (ExponentOverflowError, core.py:365-385)               */
  PGPU_ECOEFF = 3,        /* exact coefficient needs > 192 bits, or more than the
                             caller's requested accumulator width                   */
  PGPU_ECUDA = 4,         /* CUDA runtime error (message has the CUDA error name)   */
  PGPU_ENOMEM = 5,        /* device allocation failed                               */
  PGPU_EUNSUPPORTED = 6   /* combination not implemented (never falls back to CPU)  */
} pgpu_status;

typedef enum pgpu_coef_kind {
  PGPU_F64 = 0,           /* IEEE double (reference ctype float)                    */
  PGPU_I64 = 1,           /* exact integers with |c| < 2^63                         */
  PGPU_I128 = 2           /* exact integers, two little-endian u64 limbs per term,
                             two's complement (|c| < 2^127)                          */
} pgpu_coef_kind;

typedef enum pgpu_order { PGPU_GRLEX = 0, PGPU_LEX = 1 } pgpu_order;

typedef enum pgpu_path {
  PGPU_PATH_AUTO = 0,
  PGPU_PATH_DENSE = 1,    /* sumset bitmap + per-interval private accumulators     */
  PGPU_PATH_SORT = 2,     /* expand / LSD radix sort / run-length reduce            */
  PGPU_PATH_BUCKET = 3,   /* pairs written once into key-range buckets of <= 2048,
                             each grouped and folded by one CTA in shared memory
                             in (key, row) order (a batch that does not suit it
                             takes PATH_SORT)                                      */
  PGPU_PATH_SMALL = 4     /* products of at most 16384 pairs in one CTA (sorted in
                             shared memory, folded in the reference's row order);
                             AUTO takes it for such products                        */
} pgpu_path;

/* Packed-exponent layout (reference Layout, core.py:65-121).  Fields are listed
 * most significant first: for grlex the total-degree field then x1..xm, for lex
 * x1..xm.  caps follow the reference: grlex degree cap = 2^w-2, lex top-field
 * cap = 2^w-2, every other cap = 2^w-1. */
typedef struct pgpu_layout {
  int32_t order;                    /* pgpu_order */
  int32_t nfields;                  /* m+1 for grlex, m for lex */
  int32_t shift[PGPU_MAX_FIELDS];
  int32_t width[PGPU_MAX_FIELDS];
} pgpu_layout;

/* One operand: a canonical polynomial (strictly ascending exps, no zero coeff). */
typedef struct pgpu_poly {
  const uint64_t* exps;             /* n packed exponents                       */
  const void* coeffs;               /* n doubles | n int64 | 2n u64 limbs        */
  int64_t n;
} pgpu_poly;

typedef struct pgpu_options {
  int32_t coef_kind;                /* pgpu_coef_kind of both operands          */
  int32_t acc_limbs;                /* result int width in u64 limbs (1..3), 0 = auto */
  int32_t device;                   /* CUDA ordinal                             */
  int32_t path;                     /* pgpu_path                                */
  int32_t float_ordered;            /* 1: fold each f64 coefficient in the reference's
                                       order (increasing row i, merge.py:32-33) so
                                       doubles are bit-identical: small, bucket or
                                       sort path (the dense path refuses)          */
  int32_t timing;                   /* 1: record per-phase CUDA-event times     */
  int32_t inputs_on_device;         /* 1: pgpu_poly pointers are device pointers */
  int32_t outputs_on_device;        /* 1: result stays in device memory         */
  uint64_t lo;                      /* keep products whose packed exponent sum s */
  uint64_t hi;                      /*   satisfies lo <= s < hi (hi = 2^64-1:   */
                                    /*   no upper limit).  split= / cluster range */
  void* stream;                     /* cudaStream_t to run on, NULL = library's */
  int64_t range_pairs;              /* 0, or the pair count of [lo, hi) for these
                                       operands (pgpu_result.pairs of an earlier
                                       call with the same operands and range: a
                                       cluster plan); skips the device count    */
} pgpu_options;

#define PGPU_NPHASE 8

typedef struct pgpu_result {
  uint64_t* exps;                   /* n packed exponents, strictly ascending   */
  void* coeffs;                     /* n doubles, or n*acc_limbs u64 limbs      */
  int64_t n;
  int32_t coef_kind;                /* PGPU_F64 or PGPU_I64 (limbed ints)       */
  int32_t acc_limbs;                /* limbs per integer coefficient            */
  int32_t on_device;
  int32_t path_used;
  int64_t pairs;                    /* term products formed (n_a*n_b inside [lo,hi)) */
  int64_t kernel_launches;          /* kernels launched for this product        */
  int32_t key_bits;                 /* significant bits of the compacted key    */
  int32_t n_phase;
  float phase_ms[PGPU_NPHASE];      /* filled when options.timing = 1           */
  const char* phase_name[PGPU_NPHASE];
  void* _owner;                     /* library bookkeeping                      */
} pgpu_result;

/* Defaults: F64, auto width, device 0, auto path, whole range, host buffers. */
void pgpu_default_options(pgpu_options* opt);

/* The product a*b (reference parmul.mul).  On success *out owns its buffers;
 * release them with pgpu_free_result.  Zero operands give n = 0. */
int pgpu_mul(const pgpu_poly* a, const pgpu_poly* b, const pgpu_layout* lay,
             const pgpu_options* opt, pgpu_result* out);

/* cum[k] = number of pairs (i,j) with a.exps[i] + b.exps[j] < bounds[k]
 * (packed, unsigned), for nbounds ascending bounds; O_k = cum[k+1]-cum[k] is
 * count_ops(find_edge(a,b,bounds[k],bounds[k+1])) (split.py:131-175). */
int pgpu_count_below(const pgpu_poly* a, const pgpu_poly* b, const pgpu_layout* lay,
                     const uint64_t* bounds, int64_t nbounds, const pgpu_options* opt,
                     uint64_t* cum);

void pgpu_free_result(pgpu_result* r);

/* PolyFile text of terms [begin, end) of p (reference io.format_poly,
 * io.py:241-248, without its "vars ..." header line, whose names are not part
 * of the packed layout): one "<coeff> <e_1> ... <e_m>\n" line per term, the
 * exponents unpacked from `lay` (grlex degree field omitted), integers as
 * Python str() (opt->coef_kind PGPU_I64 with opt->acc_limbs limbs of
 * two's complement, or PGPU_I128), doubles as Python repr() (shortest
 * round-trip digits).  Uses opt->device, stream, inputs_on_device (p's
 * pointers are device pointers) and outputs_on_device (text stays on the
 * device).  Release with pgpu_free_text. */
typedef struct pgpu_text {
  char* text;                       /* bytes, not NUL-terminated                */
  int64_t bytes;
  int32_t on_device;
  int32_t _pad;
  void* _owner;                     /* library bookkeeping                      */
} pgpu_text;

int pgpu_format(const pgpu_poly* p, const pgpu_layout* lay, int64_t begin, int64_t end,
                const pgpu_options* opt, pgpu_text* out);
void pgpu_free_text(pgpu_text* t);

/* Peer buffers for the multi-GPU gather (one process per GPU).  A buffer from
 * pgpu_ipc_alloc can be opened by another process with the 64-byte handle;
 * pgpu_copy is an asynchronous device-to-device copy on `stream` (NULL: the
 * library's stream of `device`), over NVLink when dst is a peer's buffer. */
#define PGPU_IPC_HANDLE_BYTES 64
int pgpu_ipc_alloc(int64_t bytes, int32_t device, void** dptr, void* handle);
int pgpu_ipc_open(const void* handle, int32_t device, void** dptr);
int pgpu_ipc_close(void* dptr);
int pgpu_ipc_free(void* dptr);
int pgpu_copy(void* dst, const void* src, int64_t bytes, int32_t device, void* stream);
int pgpu_stream_sync(int32_t device, void* stream);

const char* pgpu_last_error(void);
int pgpu_device_count(void);
int pgpu_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* POLYMUL_B200_H */

/* pbh-b200 — op-trace files.
 *
 * Two on-disk forms of the reference's Trace (trace_format.hpp:16-33):
 *  - the reference's text format, one op per line (trace_format.cpp:34-126):
 *      U <value> <priority> | B <k> <v1> <p1> ... | E | D <value>
 *    '#' starts a comment; malformed input fails with the op ordinal and the
 *    line (TraceError semantics, trace_format.cpp:13-30);
 *  - a packed little-endian binary form ".pbht" for large traces (a C1 text
 *    trace is ~5 GB):
 *      u8  magic[4] = "PBHT"; u32 version = 1; u64 n_ops; u64 n_elems;
 *      u8  kinds[n_ops]       (padded with zeros to a multiple of 8 bytes)
 *      u64 offsets[n_ops + 1] (offsets[0] = 0, element ranges per op)
 *      u32 values[n_elems]    (padded to a multiple of 8 bytes)
 *      u64 priorities[n_elems]
 *    A reader streams any op range [op0, op0 + n) without loading the rest,
 *    so a trace larger than host memory can be fed to pbh_heap_run_trace in
 *    chunks. All arrays use the flat layout of pbh_heap_run_trace.
 * Host-only C++ (no device work). Status codes are pbh_status values.
 */
#ifndef PBH_TRACE_IO_H
#define PBH_TRACE_IO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pbh_trace_buf pbh_trace_buf;

/* parse_trace / load_trace (trace_format.cpp:34-98): parse a text trace file.
 * On a malformed line returns PBH_TRACE with *failed_op = the op ordinal and
 * the message in pbh_trace_last_error(). */
int pbh_trace_load_text(const char* path, pbh_trace_buf** out, uint64_t* failed_op);
/* sizes / flat export / free of a parsed trace */
void pbh_trace_buf_sizes(const pbh_trace_buf* t, uint64_t* n_ops, uint64_t* n_elems);
void pbh_trace_buf_export(const pbh_trace_buf* t, uint8_t* kinds, uint64_t* offsets,
                          uint32_t* values, uint64_t* priorities);
void pbh_trace_buf_free(pbh_trace_buf* t);

/* serialize_trace / save_trace (trace_format.cpp:100-126) from flat arrays. */
int pbh_trace_save_text(const char* path, uint64_t n_ops, const uint8_t* kinds,
                        const uint64_t* offsets, const uint32_t* values,
                        const uint64_t* priorities);

/* Packed binary writer / streaming reader. */
int pbh_trace_save_binary(const char* path, uint64_t n_ops, const uint8_t* kinds,
                          const uint64_t* offsets, const uint32_t* values,
                          const uint64_t* priorities);
typedef struct pbh_trace_reader pbh_trace_reader;
int pbh_trace_open_binary(const char* path, pbh_trace_reader** out, uint64_t* n_ops,
                          uint64_t* n_elems);
/* Ops [op0, op0 + n): kinds[n], offsets[n + 1] rebased to 0, the elements
 * (values/priorities sized by the caller from pbh_trace_chunk_elems). */
int pbh_trace_chunk_elems(pbh_trace_reader* r, uint64_t op0, uint64_t n, uint64_t* n_elems);
int pbh_trace_read_chunk(pbh_trace_reader* r, uint64_t op0, uint64_t n, uint8_t* kinds,
                         uint64_t* offsets, uint32_t* values, uint64_t* priorities);
void pbh_trace_close(pbh_trace_reader* r);

const char* pbh_trace_last_error(void);

#ifdef __cplusplus
}
#endif
#endif

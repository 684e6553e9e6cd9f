/* opcfe_io.h -- organized point-cloud ingestion, host-side C ABI (libopcfe_io.so).
 *
 * Replaces the reference's file readers for the front-end's input:
 *   flatpoly/io.py:52-78    load_grid   ("M N" header, then M*N "x y z" rows, "nan" ok)
 *   flatpoly/io.py:93-184   PLY header / ascii + binary_little_endian vertex data,
 *                           "comment grid M N" -> organized
 *   flatpoly/io.py:187-212  write_ply   (double vertices, optional grid comment)
 *   flatpoly/io.py:238-266  load_cloud  (format from suffix; organized keeps NaN)
 * Values are parsed like Python's float() (correctly rounded; "nan"/"inf" in any case,
 * digit-separating underscores) so a loaded array equals the reference's bit for bit.
 * Binary PLY whose vertex record is exactly three little-endian doubles x, y, z (what
 * write_ply produces) is read straight into the caller's buffer (e.g. pinned host
 * memory for the H2D copy): no intermediate copy, no per-value decode.
 *
 * Plain pointers and sizes only; every call returns 0 or a negative OPCFE_IO_ERR_*; the
 * message ("<path>:<line>: <what>", the reference ParseError text) is thread-local.
 */
#ifndef OPCFE_IO_H
#define OPCFE_IO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  OPCFE_IO_OK = 0,
  OPCFE_IO_ERR_PARSE = -1, /* malformed file: io.py ParseError */
  OPCFE_IO_ERR_OS = -2,    /* open / read / write failed */
  OPCFE_IO_ERR_ARG = -3    /* bad argument (unknown format, null buffer, ...) */
};

enum { OPCFE_FMT_XYZ = 0, OPCFE_FMT_GRID = 1, OPCFE_FMT_PLY = 2 };

/* What opcfe_io_probe learned from the header. */
typedef struct {
  int32_t format;        /* OPCFE_FMT_* */
  int32_t ply_binary;    /* PLY: 1 = binary_little_endian, 0 = ascii */
  int64_t rows, cols;    /* organized grid M x N (grid text / PLY grid comment); -1 if none */
  int64_t count;         /* points in the file (grid: M*N rows; PLY: vertex count;
                            xyz: data rows) */
  int64_t data_offset;   /* byte offset of the first data row / vertex record */
  int64_t first_line;    /* 1-based line number of data_offset (text formats) */
  int32_t vertex_stride; /* PLY binary: bytes per vertex record */
  int32_t x_off, y_off, z_off; /* PLY: byte offsets (binary) or token indices (ascii) */
  int32_t x_type, y_type, z_type; /* PLY binary: 'f' 'd' 'b' 'B' 'h' 'H' 'i' 'I' */
  int32_t direct;        /* PLY binary: record == 3 x <f8 x,y,z -> raw copy */
} opcfe_cloud_info;

/* Parse the header of `path` (format OPCFE_FMT_*; the grid text / xyz body is scanned
 * to count rows).  io.py:52-78, :97-131. */
int opcfe_io_probe(const char* path, int format, opcfe_cloud_info* info);

/* Read info->count points as float64 xyz into dst[count*3] using up to `threads` host
 * threads (<= 0: all cores).  Text bodies are split at line boundaries and parsed in
 * parallel; errors report the reference's file:line.  io.py:69-78, :134-184. */
int opcfe_io_read(const char* path, const opcfe_cloud_info* info, double* dst, int threads);

/* write_ply (io.py:187-212): vertices n x 3 float64, binary LE or ascii (%.17g);
 * grid_rows/grid_cols > 0 add the "comment grid M N" line.  Faces are not written. */
int opcfe_io_write_ply(const char* path, const double* vertices, int64_t n, int binary,
                       int64_t grid_rows, int64_t grid_cols);

/* Thread-local message of the last failing call, and its 1-based line (0 if none). */
const char* opcfe_io_last_error(void);
int64_t opcfe_io_error_line(void);

#ifdef __cplusplus
}
#endif

#endif /* OPCFE_IO_H */

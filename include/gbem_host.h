/* gbem_host.h — C API of the C++ host library (libgbem_host.so).
 *
 * The host keeps the reference's scene-file input (parse_model,
 * proj/include/gbem/model_io.hpp:127), panel partition (partition_scene,
 * partition.hpp:214) and capacitance output (to_csv / to_json,
 * model_io.hpp:242/266), and calls the GPU through include/gbem_gpu.h.
 * Errors: 0 ok, 1 ValidationError, 2 NumericalError, 3 CUDA; message in err.
 */
#ifndef GBEM_HOST_H
#define GBEM_HOST_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gbem_model gbem_model;

/* parse_model (model_io.hpp:127-204) plus the `freespace` extension. */
int gbem_model_parse(const char* text, gbem_model** out, char* err, int errlen);
/* Synthetic BASELINE.json config 1..5 (seeded; scale > 1 refines the panels of
 * configs 1-4 / multiplies the panel count of config 5).  The model carries its
 * net-independent panel set. */
int gbem_model_config(int config, uint64_t seed, double scale, gbem_model** out, char* err, int errlen);
void gbem_model_free(gbem_model* m);
/* dump_model (model_io.hpp:207-228); returns the text length (copies when cap suffices). */
int64_t gbem_model_dump(const gbem_model* m, char* buf, int64_t cap);
/* Dielectric regions (ascending id) with their relative permittivity; returns the count. */
int gbem_model_regions(const gbem_model* m, int32_t* ids, double* eps, int cap);
/* Net ids ascending; returns the count. */
int gbem_model_nets(const gbem_model* m, int32_t* ids, int cap);
int gbem_model_info(const gbem_model* m, int32_t* nregions, int32_t* nfaces, double* eps_r, int32_t* freespace);
int gbem_model_params(const gbem_model* m, double p[4]);
int gbem_model_set_params(gbem_model* m, const double p[4], char* err, int errlen);

/* Build the model's current panel set.  mode 0: reference partition for
 * main_net (partition_scene); 1: keep the config's own panel set; 2: uniform
 * edge args[0]; 3: graded (args = h0, ratio, hmax).  Returns n, or -1 (err). */
int64_t gbem_model_partition(gbem_model* m, int mode, int32_t main_net, const double* args, char* err,
                             int errlen);
/* Copy the current panel set (arrays of n entries; any pointer may be NULL). */
int gbem_model_panels(const gbem_model* m, uint8_t* axis, double* level, double* a0, double* a1, double* b0,
                      double* b1, int32_t* nsign, int32_t* kind, int32_t* net, int32_t* region_a,
                      int32_t* region_b, double* area, double* dist, int32_t* facing);

/* capacitance_matrix / capacitance_row on the GPU.  mode 0: per-main-net
 * reference partition (K partitions, K assemblies, K factorisations); mode 1:
 * the model's current panel set, one assembly + one factorisation + K RHS.
 * net = -1 for all nets (--all), else one row.  Writes the CSV and JSON reports
 * (model_io.hpp:242-299) when the buffers are large enough; returns 0 or an
 * error code.  *csv_len / *json_len receive the full lengths. */
typedef struct {
  int32_t device;
  int32_t mode;
  int32_t net;
  double rel_tol;
  int32_t max_levels;
  const char* dump_matrix; /* NULL or path prefix */
  double* cap_out;         /* NULL or rows x nets, full precision (farads), rows in solve order */
  double* outer_out;       /* NULL or per-row induced charge on the outer boundary */
  int32_t collocation;     /* 1: the collocation baseline (--baseline collocation, cli.hpp:37-38) */
  /* shared mode (mode 1) only: the solver.  0 auto (block-Jacobi PCG on row
   * shards when the context has several ranks, else the direct DMMA Cholesky),
   * 1 direct, 2 PCG (also at one rank).  Ranks: nranks > 1 attaches an NCCL
   * communicator (rank 0 writes the unique id to nccl_id_file, the others read
   * it); only rank 0 fills csv / json. */
  int32_t solver;
  int32_t nranks, rank;
  const char* nccl_id_file;
  int32_t jacobi_blocks;   /* Jacobi blocks per rank (PCG; 0 = 1) */
  double pcg_tol;          /* 0 = 1e-10 */
} gbem_extract_opts;

int gbem_model_extract(const gbem_model* m, const gbem_extract_opts* o, char* csv, int64_t csv_cap,
                       int64_t* csv_len, char* json, int64_t json_cap, int64_t* json_len, char* err,
                       int errlen);

#ifdef __cplusplus
}
#endif
#endif

/* bp_operator.h — C-ABI of the operator surface (libblockpipe_b200.so).
 *
 * The reference's operator layer is C++ (CLI, run config, artifacts,
 * analytics) plus a pybind11 module; these entry points let any FFI (ctypes,
 * cgo, JNI) reach the same functions of the B200 build. Each cites the
 * reference function it replaces. Status values are the CLI exit codes
 * (P/src/cli.cpp:534-543): 0 ok, 1 runtime failure, 2 config error,
 * 3 I/O error; bp_operator_last_error() holds the message of the last failure
 * on the calling thread.
 */
#ifndef BP_OPERATOR_H_
#define BP_OPERATOR_H_

#include <stddef.h>
#include <stdint.h>

#include "bp_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

BP_API const char* bp_operator_last_error(void);

/* cli_main (cli.cpp:312-544). stdout/stderr text is handed to `sink` once
 * each (stream 1 / 2) after the command finishes. Returns the exit code. */
typedef void (*bp_text_sink)(void* user, int32_t stream, const char* text, int64_t len);
BP_API int32_t bp_cli_main(int32_t argc, const char* const* argv, bp_text_sink sink, void* user);

/* run_and_write_artifacts (artifacts.cpp:130-143) for a flat JSON config
 * (run_config.cpp:48-104). plan_only != 0 writes the three schedule-derived
 * artifacts without device work. The summary path is copied to
 * summary_path (NUL-terminated, truncated to cap). */
BP_API int32_t bp_write_artifacts(const char* config_json, int32_t plan_only, char* summary_path, int64_t cap);

/* run_config_to_json(run_config_from_json_text(text)) (run_config.cpp:114-141):
 * the effective config echo. Returns the byte length; copies up to cap. */
BP_API int64_t bp_config_echo(const char* config_json, char* out, int64_t cap);

/* bubble_size / bubble_ratio (analytics.cpp:13-31). order: bp_order. */
BP_API int32_t bp_bubble(int32_t devices, int32_t steps, int64_t block_num, int32_t order, int64_t* size,
                         double* ratio);

/* CostParams (analytics.hpp:31-47) + bytes_per_scalar extension. */
typedef struct {
  int64_t frames, height, width, hidden, channels, layers, devices, num_b, num_c;
  double model_mem, kv_mem;
  int32_t ring_refinement;
  int32_t bytes_per_scalar;
} bp_cost_params;
typedef struct {
  double comm_scalars;
  int32_t comm_overlap;
  double model_mem, kv_mem, comm_bytes;
} bp_cost_row;
/* CostParams defaults (analytics.hpp:32-43). */
BP_API void bp_cost_defaults(bp_cost_params* cp);
/* method_cost (analytics.cpp:67-117); method is the reference's token. */
BP_API int32_t bp_method_cost(const char* method, const bp_cost_params* cp, bp_cost_row* out);

#ifdef __cplusplus
}
#endif

#endif /* BP_OPERATOR_H_ */

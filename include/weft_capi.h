/* weft planner C ABI — JSON in, JSON out.
 *
 * A thin extern "C" face over the drop-in C++ planner (include/weft/*.hpp) so
 * that non-C++ callers (the Python host layer, ctypes tests, a cgo/JNI binding)
 * can reach the reference's plan-time entry points without C++ types:
 *
 *   weft_build_dag_json      <- build_layer_dag            (reference op_model.hpp:66-68)
 *   weft_topo_orders_json    <- enumerate_topological_orders (op_model.hpp:76)
 *   weft_segment_cost_json   <- segment_pair_cost          (overlap_profile.hpp:72-73)
 *   weft_dp_align_json       <- dp_align / brute_force_align (pairing_search.hpp:55,63)
 *   weft_search_json         <- search_si_plan + plan_to_json (pairing_search.hpp:93-98)
 *   weft_profile_roundtrip_json <- parse_profile + profile_to_json (overlap_profile.hpp:76-79)
 *   weft_pipeline_json       <- fold_layers, schedule_w_pipeline / _1f1b / _bidirectional,
 *                               bubble_ratio, pp_comm_volume, validate_schedule, trace/CSV
 *                               export (folding_pipeline.hpp:23-103)
 *   weft_memory_json         <- simulate_memory, max_model_size, default footprints
 *                               (memory_sim.hpp:47-79)
 *   weft_estimate_json       <- estimate_iteration_time (estimate.hpp:45-50)
 *   weft_compare_json        <- parse_scenario + compare_report + report_to_json/csv
 *                               (report.hpp:42-66)
 *   weft_comm_volume_json    <- comm_volume_estimate (comm_volume.hpp:26-29)
 *
 * Every call returns a weft status (0 ok; 2 ConfigError, 3 InfeasibleError,
 * 4 MissingProfileEntry — the reference CLI's exit codes, weft_main.cpp:20-23;
 * 1 any other failure) and, on success, a malloc'd NUL-terminated JSON string
 * in *out that the caller releases with weft_free(). On failure *out is NULL and
 * weft_last_error() returns the exception message (thread-local).
 *
 * The same source is also compiled against the reference sources, with every
 * symbol prefixed weft_ref_ (WEFT_CAPI_PREFIX), to form the parity oracle in
 * oracle/_ref/. The request schema is documented in
 * paper_2411_15871_b200/csrc/planner/capi.cpp.
 */
#ifndef WEFT_CAPI_H
#define WEFT_CAPI_H

#ifdef __cplusplus
extern "C" {
#endif

int weft_build_dag_json(const char* request, char** out);
int weft_topo_orders_json(const char* request, char** out);
int weft_segment_cost_json(const char* request, char** out);
int weft_dp_align_json(const char* request, char** out);
int weft_search_json(const char* request, char** out);
int weft_profile_roundtrip_json(const char* request, char** out);
int weft_templates_json(const char* request, char** out);  /* builtin_template_json (op_model.hpp:59) */
int weft_pipeline_json(const char* request, char** out);
int weft_memory_json(const char* request, char** out);
int weft_estimate_json(const char* request, char** out);
int weft_compare_json(const char* request, char** out);
int weft_comm_volume_json(const char* request, char** out);
const char* weft_last_error(void);
void weft_free(char* p);

#ifdef __cplusplus
}
#endif

#endif /* WEFT_CAPI_H */

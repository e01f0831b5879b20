/*
 * espn_host.h -- C entry points of libespn_host.so (the C++ host layer over
 * include/espn_gpu.h).
 *
 * espn_host_run_batches is the serving loop of run_batch (pipeline.hpp:81-85:
 * "at most `concurrency` queries in flight") at batch granularity: a stream of
 * batches with HOST inputs goes through `lanes` workspaces, each on its own
 * stream, every call ESPN_RERANK_ASYNC, so batch n+1's host->device copies and
 * planning overlap batch n's scoring and ranked lists land in host memory as
 * they complete.  No Python (or other interpreter) sits between calls.
 */
#ifndef ESPN_HOST_H
#define ESPN_HOST_H

#include <stdint.h>

#include "espn_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Runs batches[0..n) in order; batch i goes to lane i % lanes (workspace
 * ws[lane], stream streams[lane]).  A lane keeps at most `depth` batches
 * (>= 1) in flight: before submitting batch i the lane waits for its batch
 * i - depth*lanes, so outs[] may rotate lanes*depth buffer sets.  Every
 * batch's flags get ESPN_RERANK_ASYNC.  Returns after every batch completed
 * and every workspace reported its device-side status; *seconds (optional)
 * = host wall time from the first submission to that point. */
ESPN_API int espn_host_run_batches(espn_gpu_table* table, espn_gpu_workspace* const* ws, void* const* streams,
                                   uint32_t lanes, uint32_t depth, const espn_rerank_args* batches,
                                   espn_rerank_out* outs, uint32_t n, double* seconds);

#ifdef __cplusplus
}
#endif
#endif /* ESPN_HOST_H */

/* C-ABI of the whole-model driver (libezquant.so), for non-C++ hosts such as
 * the Python multi-GPU driver (paper_2403_02775_b200/driver.py).
 *
 * The reference exposes the model driver only as C++ (proj/include/ezquant/
 * model.hpp:63-80, quantize_model / dequantize_model; its CLI calls them from
 * tools/ezquant_main.cpp). These entry points wrap the drop-in's C++ functions
 * (include/ezquant/model.hpp) one to one, plus the multi-GPU extension
 * (quantize_model_shard / merge_model_shards): each process quantizes its LPT
 * share onto disk and one process merges the manifest -- no collective.
 *
 * Return: EZQ_OK, or the EZQ_ERR_* class of the exception the C++ function
 * threw (message in `err`, truncated to `cap`). `failures` receives the count
 * of per-tensor failures (ModelRunResult::failures). */
#pragma once

#include <stddef.h>
#include <stdint.h>

#include "ezquant_c.h"

#ifdef __cplusplus
extern "C" {
#endif

int ezqm_quantize_model(const char* manifest_json, const char* out_dir, const ezq_config* cfg, int mode,
                        int workers, int* failures, char* err, size_t cap);
int ezqm_quantize_model_shard(const char* manifest_json, const char* out_dir, const ezq_config* cfg, int mode,
                              int workers, int rank, int world, int* failures, char* err, size_t cap);
int ezqm_merge_model_shards(const char* manifest_json, const char* out_dir, const ezq_config* cfg, int mode,
                            int world, int* failures, char* err, size_t cap);
/* LPT bin of `rank`: writes up to `cap` manifest indices, returns the count. */
int64_t ezqm_lpt_shard(const char* manifest_json, int rank, int world, int64_t* idx, int64_t cap);

#ifdef __cplusplus
}
#endif

/* lfgpu_files.h -- raw sample files and a reader-thread source for the shard runner
 * (raw reads from storage in place of the synthetic feeder,
 * experiment.cpp:221-228).  Host library (libloadflow_b200.so), C ABI.
 *
 * File format (little endian): "LFGS" | u32 version = 1 | i32 kind | i32 ndim |
 * i64 dims[4] | payload.  kind 1: img_seg volume, payload = f32 image [D,H,W] then
 * u8 label [D,H,W]; kind 2: obj_det image, u8 [H,W,3]; kind 3: waveform, f32 [L];
 * kind 4: waveform, int16 PCM [L] (the reference's 2-B speech samples; chains with
 * FilterBank param 5 = LFG_DT_I16).
 *
 * The source reads files with `readers` threads into `slots` pinned host buffers
 * (sized for the largest file), in feed order, ahead of the shard; a buffer is
 * refilled once the shard releases its sample (lfg_source.release).  Samples are
 * submitted as LFG_SRC_HOST_PINNED, so the e2e path (K0 / batched DMA) applies. */
#ifndef LFGPU_FILES_H
#define LFGPU_FILES_H

#include "lfgpu.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { LFG_FILE_VOLUME = 1, LFG_FILE_IMAGE = 2, LFG_FILE_WAVEFORM = 3, LFG_FILE_PCM16 = 4 };

int lfg_write_sample_file(const char* path, int kind, int ndim, const int64_t dims[4], const void* data,
                          const void* aux);

typedef struct lfg_file_source lfg_file_source;
/* ids[i] becomes sample i's id; paths are read in order i = 0 .. n-1 */
int lfg_file_source_open(lfg_ctx* ctx, const char* const* paths, const uint64_t* ids, int64_t n, int readers,
                         int slots, lfg_file_source** out);
int lfg_file_source_get(lfg_file_source* fs, lfg_source* out);   /* the callbacks for lfg_run_shard_source */
int lfg_file_source_stats(lfg_file_source* fs, int64_t* bytes_read, double* read_seconds);
int lfg_file_source_close(lfg_file_source* fs);
const char* lfg_files_last_error(void);   /* thread-local, this header's calls */

#ifdef __cplusplus
}
#endif

#endif

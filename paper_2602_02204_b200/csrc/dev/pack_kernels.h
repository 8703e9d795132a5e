// K5 connector pack launcher. Internal to libomni_dev.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace omni_dev {

struct PackChunkDesc {
  int32_t slot;   // hidden-ring slot of the sequence
  int32_t begin;  // emitted rows [begin, end)
  int32_t end;
  int32_t pad;
  uint64_t dst_offset;         // byte offset of the blob in the destination arena (16-B aligned)
  const int32_t* tokens_dev;   // [end-begin] token ids (device)
};

constexpr int kPackMaxRows = 256;
constexpr int kPackUvaRows = 64;   // packs of more rows copy their descriptors to the device first  // rows of one chunk (the hidden ring holds 64 per sequence)
uint64_t pack_blob_bytes(int rows, int d);
cudaError_t launch_pack_hidden(const PackChunkDesc* chunks_dev, int n_chunks, int max_rows,
                               const __nv_bfloat16* ring, int d, int ring_rows, uint8_t* dst_base,
                               bool desc_on_device, cudaStream_t st);

}  // namespace omni_dev

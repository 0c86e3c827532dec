# vLLM copy_blocks_kernel (csrc/cache_kernels.cu), Llama-2-7B KV cache (32 layers, block 16 x 32 heads
# x head 128 = 65536 elements per block).  The per-layer cache base pointers live in an int64 device
# array and are turned into element pointers inside the kernel
# (reinterpret_cast<scalar_t*>(key_cache_ptrs[layer_idx])): those handles have no provenance, so every
# access through them is an InvalidDeref site (engine/detectors.py:277-298).
wrapper copy_blocks(key_cache_ptrs: tensor, value_cache_ptrs: tensor, block_mapping: tensor, numel_per_block: i32) {
  let num_layers: i32 = key_cache_ptrs.size(0);
  let num_pairs: i32 = block_mapping.size(0);
  launch copy_blocks_kernel<<<num_layers, num_pairs; 1024>>>(key_cache_ptrs.data_ptr(), value_cache_ptrs.data_ptr(), block_mapping.data_ptr(), numel_per_block);
}
kernel copy_blocks_kernel(key_cache_ptrs: handle<i64>, value_cache_ptrs: handle<i64>, block_mapping: handle<i64>, numel_per_block: i32) {
  i32 layer_idx = blockIdx.x;
  i32 pair_idx = blockIdx.y;
  handle<f16> key_cache = handle<f16>(key_cache_ptrs[layer_idx]);
  handle<f16> value_cache = handle<f16>(value_cache_ptrs[layer_idx]);
  i64 src_block_number = block_mapping[2 * pair_idx];
  i64 dst_block_number = block_mapping[2 * pair_idx + 1];
  i64 src_block_offset = src_block_number * i64(numel_per_block);
  i64 dst_block_offset = dst_block_number * i64(numel_per_block);
  for (i32 i = threadIdx.x; i < numel_per_block; i += blockDim.x) {
    i64 src_offset = src_block_offset + i64(i);
    i64 dst_offset = dst_block_offset + i64(i);
    key_cache[dst_offset] = key_cache[src_offset];
  }
  for (i32 i = threadIdx.x; i < numel_per_block; i += blockDim.x) {
    i64 src_offset = src_block_offset + i64(i);
    i64 dst_offset = dst_block_offset + i64(i);
    value_cache[dst_offset] = value_cache[src_offset];
  }
}

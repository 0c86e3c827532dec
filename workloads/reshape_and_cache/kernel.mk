# config 5 corpus: vLLM reshape_and_cache_kernel (paged KV-cache write), Mistral-7B: 8 kv heads,
# head_size 128, block_size 16, x = 16 bytes / sizeof(f16) = 8; num_tokens = BS x SL
wrapper reshape_and_cache(key: tensor, value: tensor, key_cache: tensor, value_cache: tensor, slot_mapping: tensor) {
  let num_tokens: i32 = key.size(0);
  let num_heads: i32 = key.size(1);
  let head_size: i32 = key.size(2);
  let block_size: i32 = key_cache.size(3);
  let x: i32 = key_cache.size(4);
  let key_stride: i32 = key.numel() / num_tokens;
  let value_stride: i32 = value.numel() / num_tokens;
  launch reshape_and_cache_kernel<<<num_tokens; 512>>>(key.data_ptr(), value.data_ptr(), key_cache.data_ptr(), value_cache.data_ptr(), slot_mapping.data_ptr(), key_stride, value_stride, num_heads, head_size, block_size, x);
}
kernel reshape_and_cache_kernel(key: handle<f16>, value: handle<f16>, key_cache: handle<f16>, value_cache: handle<f16>, slot_mapping: handle<i64>, key_stride: i32, value_stride: i32, num_heads: i32, head_size: i32, block_size: i32, x: i32) {
  i64 token_idx = i64(blockIdx.x);
  i64 slot_idx = slot_mapping[token_idx];
  if (slot_idx < 0) {
    return;
  }
  i64 block_idx = slot_idx / i64(block_size);
  i64 block_offset = slot_idx % i64(block_size);
  i32 n = num_heads * head_size;
  for (i32 i = threadIdx.x; i < n; i += blockDim.x) {
    i64 src_key_idx = token_idx * i64(key_stride) + i64(i);
    i64 src_value_idx = token_idx * i64(value_stride) + i64(i);
    i32 head_idx = i / head_size;
    i32 head_offset = i % head_size;
    i32 x_idx = head_offset / x;
    i32 x_offset = head_offset % x;
    i64 tgt_key_idx = block_idx * i64(num_heads * (head_size / x) * block_size * x) + i64(head_idx * (head_size / x) * block_size * x) + i64(x_idx * block_size * x) + block_offset * i64(x) + i64(x_offset);
    i64 tgt_value_idx = block_idx * i64(num_heads * head_size * block_size) + i64(head_idx * head_size * block_size) + i64(head_offset * block_size) + block_offset;
    key_cache[tgt_key_idx] = key[src_key_idx];
    value_cache[tgt_value_idx] = value[src_value_idx];
  }
}

# config 5 corpus: vLLM rotary_embedding_kernel (NeoX), llama2_13b: 40 q heads, 40 kv heads, head_size 128, max_position 4096
wrapper rotary_embedding(positions: tensor, query: tensor, key: tensor, head_size: i32, cos_sin_cache: tensor) {
  let num_tokens: i32 = query.numel() / query.size(-1);
  let rot_dim: i32 = cos_sin_cache.size(1);
  let num_heads: i32 = query.size(-1) / head_size;
  let num_kv_heads: i32 = key.size(-1) / head_size;
  let query_stride: i64 = query.size(-1);
  let key_stride: i64 = key.size(-1);
  launch rotary_embedding_kernel<<<num_tokens; 512>>>(positions.data_ptr(), query.data_ptr(), key.data_ptr(), cos_sin_cache.data_ptr(), rot_dim, query_stride, key_stride, num_heads, num_kv_heads, head_size);
}
kernel rotary_embedding_kernel(positions: handle<i64>, query: handle<f16>, key: handle<f16>, cos_sin_cache: handle<f16>, rot_dim: i32, query_stride: i64, key_stride: i64, num_heads: i32, num_kv_heads: i32, head_size: i32) {
  i32 token_idx = blockIdx.x;
  i64 pos = positions[token_idx];
  handle<f16> cache_ptr = cos_sin_cache + pos * i64(rot_dim);
  i32 embed_dim = rot_dim / 2;
  handle<f16> cos_ptr = cache_ptr;
  handle<f16> sin_ptr = cache_ptr + embed_dim;
  i32 nq = num_heads * embed_dim;
  for (i32 i = threadIdx.x; i < nq; i += blockDim.x) {
    i32 head_idx = i / embed_dim;
    i64 token_head = i64(token_idx) * query_stride + i64(head_idx * head_size);
    i32 rot_offset = i % embed_dim;
    handle<f16> arr = query + token_head;
    f16 c = cos_ptr[rot_offset];
    f16 s = sin_ptr[rot_offset];
    f16 x = arr[rot_offset];
    f16 y = arr[embed_dim + rot_offset];
    arr[rot_offset] = x * c - y * s;
    arr[embed_dim + rot_offset] = y * c + x * s;
  }
  i32 nk = num_kv_heads * embed_dim;
  for (i32 i = threadIdx.x; i < nk; i += blockDim.x) {
    i32 head_idx = i / embed_dim;
    i64 token_head = i64(token_idx) * key_stride + i64(head_idx * head_size);
    i32 rot_offset = i % embed_dim;
    handle<f16> arr = key + token_head;
    f16 c = cos_ptr[rot_offset];
    f16 s = sin_ptr[rot_offset];
    f16 x = arr[rot_offset];
    f16 y = arr[embed_dim + rot_offset];
    arr[rot_offset] = x * c - y * s;
    arr[embed_dim + rot_offset] = y * c + x * s;
  }
}

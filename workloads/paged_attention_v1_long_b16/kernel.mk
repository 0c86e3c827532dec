# config 3 at its stated domain: vLLM paged_attention_v1_kernel, Mistral-7B (32 heads, 8 kv heads, head 128),
# block 16, 128 threads, seq_len up to 2^20, 2^20-block KV cache (tools/make_pa_long.py)
wrapper paged_attention_v1(out: tensor, query: tensor, key_cache: tensor, value_cache: tensor, num_kv_heads: i32, scale: f32, block_tables: tensor, seq_lens: tensor, max_seq_len: i32) {
  let num_seqs: i32 = query.size(0);
  let num_heads: i32 = query.size(1) / 128;
  let max_num_blocks_per_seq: i32 = block_tables.size(1);
  let q_stride: i32 = query.size(1);
  let kv_block_stride: i32 = key_cache.numel() / key_cache.size(0);
  let kv_head_stride: i32 = kv_block_stride / num_kv_heads;
  let padded_max_seq_len: i32 = ((max_seq_len + 15) / 16) * 16;
  let shared_bytes: i32 = padded_max_seq_len * 4;
  launch paged_attention_v1_kernel<<<num_heads, num_seqs; 128; shared_bytes>>>(out.data_ptr(), query.data_ptr(), key_cache.data_ptr(), value_cache.data_ptr(), num_kv_heads, scale, block_tables.data_ptr(), seq_lens.data_ptr(), max_num_blocks_per_seq, q_stride, kv_block_stride, kv_head_stride);
}
kernel paged_attention_v1_kernel(out: handle<f16>, q: handle<f16>, k_cache: handle<f16>, v_cache: handle<f16>, num_kv_heads: i32, scale: f32, block_tables: handle<i32>, seq_lens: handle<i32>, max_num_blocks_per_seq: i32, q_stride: i32, kv_block_stride: i32, kv_head_stride: i32) {
  extern shared f32 logits[];
  i32 seq_idx = blockIdx.y;
  i32 head_idx = blockIdx.x;
  i32 num_heads = gridDim.x;
  i32 seq_len = seq_lens[seq_idx];
  i32 num_seq_blocks = (seq_len + 15) / 16;
  i32 warp_idx = threadIdx.x / 32;
  i32 lane = threadIdx.x % 32;
  i32 num_queries_per_kv = num_heads / num_kv_heads;
  i32 kv_head_idx = head_idx / num_queries_per_kv;
  f16 qv = q[seq_idx * q_stride + head_idx * 128 + threadIdx.x];
  for (i32 block_idx = warp_idx; block_idx < num_seq_blocks; block_idx += 4) {
    i32 pbn = block_tables[seq_idx * max_num_blocks_per_seq + block_idx];
    i32 off = lane % 16;
    i32 token_idx = block_idx * 16 + off;
    f16 kv = k_cache[i64(pbn) * i64(kv_block_stride) + i64(kv_head_idx * kv_head_stride) + i64(off * 8)];
    if (lane < 16) {
      logits[token_idx] = f32(kv) * scale;
    }
  }
  barrier;
  for (i32 block_idx = warp_idx; block_idx < num_seq_blocks; block_idx += 4) {
    i32 pbn = block_tables[seq_idx * max_num_blocks_per_seq + block_idx];
    f16 vv = v_cache[i64(pbn) * i64(kv_block_stride) + i64(kv_head_idx * kv_head_stride) + i64(lane * 16)];
  }
  out[(seq_idx * num_heads + head_idx) * 128 + threadIdx.x] = qv;
}

# config 4b: vLLM moe top-k (moeTopK after moeSoftmax), Mixtral-8x7B: 8 experts, top_k 2, TPB 256
wrapper topk_softmax(topk_weights: tensor, topk_indices: tensor, token_expert_indices: tensor, gating_output: tensor) {
  let num_experts: i32 = gating_output.size(-1);
  let num_tokens: i32 = gating_output.numel() / num_experts;
  let topk: i32 = topk_weights.size(-1);
  launch moe_topk_kernel<<<num_tokens; 256>>>(gating_output.data_ptr(), topk_weights.data_ptr(), topk_indices.data_ptr(), token_expert_indices.data_ptr(), num_experts, topk);
}
kernel moe_topk_kernel(inputs_after_softmax: handle<f32>, output: handle<f32>, indices: handle<i32>, source_rows: handle<i32>, num_experts: i32, k: i32) {
  shared f32 s_best[1];
  i32 num_rows = gridDim.x;
  i32 block_row = blockIdx.x;
  i32 thread_read_offset = blockIdx.x * num_experts;
  for (i32 k_idx = 0; k_idx < k; k_idx += 1) {
    for (i32 expert = threadIdx.x; expert < num_experts; expert += 256) {
      i32 idx = thread_read_offset + expert;
      f32 val = inputs_after_softmax[idx];
    }
    if (threadIdx.x == 0) {
      i32 idx = k * block_row + k_idx;
      output[idx] = s_best[0];
      indices[idx] = k_idx;
      source_rows[idx] = k_idx * num_rows + block_row;
    }
    barrier;
  }
}

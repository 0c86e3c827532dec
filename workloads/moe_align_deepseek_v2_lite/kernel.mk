# config 4a: vLLM moe_align_block_size (Fig. 7 shape), Mixtral-8x7B: 8 experts, top_k 2, block 16, T in [1, 2^16]
wrapper moe_align_block_size(topk_ids: tensor, num_experts: i32, block_size: i32) {
  let num_thread: i32 = 32;
  let numel: i32 = topk_ids.numel();
  let shared_bytes: i32 = ((num_thread + 1) * num_experts + (num_experts + 1)) * 4;
  launch moe_align_kernel<<<1; num_thread; shared_bytes>>>(topk_ids.data_ptr(), num_experts, block_size, numel);
}
kernel moe_align_kernel(topk_ids: handle<i32>, num_experts: i32, block_size: i32, numel: i32) {
  extern shared i32 shared_mem[];
  handle<i32> tokens_cnts = shared_mem + blockDim.x + 1;
  i32 tokens_per_thread = (numel + blockDim.x - 1) / blockDim.x;
  i32 start_idx = threadIdx.x * tokens_per_thread;
  for (i32 i = 0; i < num_experts; i += 1) {
    tokens_cnts[(threadIdx.x + 1) * num_experts + i] = 0;
  }
  for (i32 i = start_idx; i < numel; i += 1) {
    i32 e = topk_ids[i];
    tokens_cnts[(threadIdx.x + 1) * num_experts + e] += 1;
  }
}

# config 1: vLLM rms_norm_kernel, Llama-2-7B (hidden 4096), num_tokens in [1, 2^20]
wrapper rms_norm(out: tensor, input: tensor, weight: tensor, epsilon: f32) {
  let hidden_size: i32 = input.size(-1);
  let num_tokens: i32 = input.numel() / hidden_size;
  launch rms_norm_kernel<<<num_tokens; 1024>>>(out.data_ptr(), input.data_ptr(), weight.data_ptr(), epsilon, num_tokens, hidden_size);
}
kernel rms_norm_kernel(out: handle<f16>, input: handle<f16>, weight: handle<f16>, epsilon: f32, num_tokens: i32, hidden_size: i32) {
  shared f32 s_variance[1];
  f32 variance = 0.0;
  for (i32 idx = threadIdx.x; idx < hidden_size; idx += blockDim.x) {
    f32 x = f32(input[blockIdx.x * hidden_size + idx]);
    variance += x * x;
  }
  if (threadIdx.x == 0) {
    s_variance[0] = variance;
  }
  barrier;
  for (i32 idx = threadIdx.x; idx < hidden_size; idx += blockDim.x) {
    f32 x = f32(input[blockIdx.x * hidden_size + idx]);
    out[blockIdx.x * hidden_size + idx] = f16(x * s_variance[0]) * weight[idx];
  }
}

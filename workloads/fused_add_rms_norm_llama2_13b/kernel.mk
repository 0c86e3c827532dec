# Fig. 2 fused_add_rms_norm
wrapper fused_add_rms_norm(input: tensor, residual: tensor, weight: tensor, epsilon: f32) {
  let hidden_size: i32 = input.size(-1);
  let num_tokens: i32 = input.numel() / hidden_size;
  launch fused_add_rms_norm_kernel<<<num_tokens; 256>>>(input.data_ptr(), residual.data_ptr(), weight.data_ptr(), epsilon, num_tokens, hidden_size);
}
kernel fused_add_rms_norm_kernel(input: handle<f16, 8>, residual: handle<f16, 8>, weight: handle<f16, 8>, epsilon: f32, num_tokens: i32, hidden_size: i32) {
  shared f32 s_variance[1];
  i32 vec_hidden_size = hidden_size / 8;
  f32 variance = 0.0;
  for (i32 idx = threadIdx.x; idx < vec_hidden_size; idx += blockDim.x) {
    i32 id = blockIdx.x * vec_hidden_size + idx;
    f32 x = f32(input[id]);
    f32 r = f32(residual[id]);
    x = x + r;
    variance += x * x;
    residual[id] = f16(x);
  }
  if (threadIdx.x == 0) {
    s_variance[0] = variance;
  }
  barrier;
  for (i32 idx = threadIdx.x; idx < vec_hidden_size; idx += blockDim.x) {
    i32 id = blockIdx.x * vec_hidden_size + idx;
    f32 x = f32(residual[id]);
    input[id] = f16(x * f32(weight[idx]));
  }
}

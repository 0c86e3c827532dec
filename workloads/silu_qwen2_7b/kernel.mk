# vLLM act_and_mul_kernel (csrc/activation_kernels.cu, silu_and_mul), Llama-3-8B MLP (intermediate
# 14336), num_tokens in [1, 2^20].  The row offsets are formed in int64 from the token index and
# narrowed to int32 for the element loop (an explicit i64 -> i32 cast: narrowing_site,
# engine/detectors.py:84-95); the input row is 2 x 14336 wide, so the narrowing wraps from
# num_tokens = 74899 on.
wrapper silu_and_mul(out: tensor, input: tensor) {
  let d: i32 = input.size(-1) / 2;
  let num_tokens: i32 = input.numel() / input.size(-1);
  launch act_and_mul_kernel<<<num_tokens; 1024>>>(out.data_ptr(), input.data_ptr(), d);
}
kernel act_and_mul_kernel(out: handle<f16>, input: handle<f16>, d: i32) {
  i64 token_idx = i64(blockIdx.x);
  i32 in_row = i32(token_idx * i64(2) * i64(d));
  i32 out_row = i32(token_idx * i64(d));
  for (i32 idx = threadIdx.x; idx < d; idx += blockDim.x) {
    f16 x = input[in_row + idx];
    f16 y = input[in_row + d + idx];
    out[out_row + idx] = x * y;
  }
}

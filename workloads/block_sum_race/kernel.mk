# per-block sum whose final store lost its `if (threadIdx.x == 0)` guard:
# every thread of the block stores the block's result to the same element
# (the classic missing-leader-guard race), after a correct tree reduction
wrapper block_sum(x: tensor, out: tensor) {
  let n: i32 = x.numel();
  let blocks: i32 = (n + 255) / 256;
  launch block_sum_kernel<<<blocks; 256>>>(x.data_ptr(), out.data_ptr(), n);
}
kernel block_sum_kernel(x: handle<f32>, out: handle<f32>, n: i32) {
  shared f32 buf[256];
  i32 i = blockIdx.x * blockDim.x + threadIdx.x;
  f32 v = 0.0;
  if (i < n) {
    v = x[i];
  }
  buf[threadIdx.x] = v;
  barrier;
  for (i32 s = 128; s > 0; s = s / 2) {
    if (threadIdx.x < s) {
      buf[threadIdx.x] = buf[threadIdx.x] + buf[threadIdx.x + s];
    }
    barrier;
  }
  out[blockIdx.x] = buf[0];
}

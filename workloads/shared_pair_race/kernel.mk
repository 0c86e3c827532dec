# pairwise staging into shared memory with the pair index computed as
# threadIdx.x / 2: both threads of a pair store the same shared slot in the
# same barrier epoch (a shared-memory DataRace within one block)
wrapper pair_stage(x: tensor, out: tensor) {
  let n: i32 = x.numel();
  launch pair_stage_kernel<<<(n + 127) / 128; 128>>>(x.data_ptr(), out.data_ptr(), n);
}
kernel pair_stage_kernel(x: handle<f32>, out: handle<f32>, n: i32) {
  shared f32 stage[64];
  i32 i = blockIdx.x * blockDim.x + threadIdx.x;
  f32 v = 0.0;
  if (i < n) {
    v = x[i];
  }
  stage[threadIdx.x / 2] = v;
  barrier;
  if (i < n && threadIdx.x < 64) {
    out[blockIdx.x * 64 + threadIdx.x] = stage[threadIdx.x];
  }
}

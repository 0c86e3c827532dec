# race probe
wrapper racy(t: tensor, n: i32) {
  let numel: i32 = t.numel();
  launch racy_kernel<<<n; 8>>>(t.data_ptr(), numel);
}
kernel racy_kernel(t: handle<i32>, numel: i32) {
  shared i32 s[4];
  s[threadIdx.x % 4] = 1;
  barrier;
  if (blockIdx.x * 8 + threadIdx.x < numel) {
    t[blockIdx.x * 8 + threadIdx.x] = s[0];
  }
  t[0] = 7;
}

# missing-barrier probe: every thread stores its slot of a shared buffer and
# reads its neighbour's slot in the same barrier epoch (a read-write race the
# reference's same-instruction twin check cannot see); the store after the
# barrier is ordered against those reads
wrapper racy_rw(t: tensor, n: i32) {
  let numel: i32 = t.numel();
  launch racy_rw_kernel<<<n; 32>>>(t.data_ptr(), numel);
}
kernel racy_rw_kernel(t: handle<i32>, numel: i32) {
  shared i32 buf[32];
  buf[threadIdx.x] = threadIdx.x;
  if (blockIdx.x * 32 + threadIdx.x < numel) {
    t[blockIdx.x * 32 + threadIdx.x] = buf[(threadIdx.x + 1) % 32];
  }
  barrier;
  buf[threadIdx.x] = 0;
}

# index scatter without atomics (a gather/scatter kernel written as
# out[idx[i]] = src[i]): two tokens routed to the same row store the same
# address -- a DataRace the reference's store_site finds through the loaded
# index values (havoc per thread)
wrapper scatter_rows(out: tensor, idx: tensor, src: tensor) {
  let n: i32 = idx.numel();
  let out_numel: i32 = out.numel();
  launch scatter_kernel<<<(n + 255) / 256; 256>>>(out.data_ptr(), idx.data_ptr(), src.data_ptr(), n, out_numel);
}
kernel scatter_kernel(out: handle<f32>, idx: handle<i32>, src: handle<f32>, n: i32, out_numel: i32) {
  i32 i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    i32 j = idx[i];
    if (j >= 0 && j < out_numel) {
      out[j] = src[i];
    }
  }
}

# Float-branch probe: vLLM-style per-token clamp with a data-dependent float branch,
# Llama-2-7B hidden 4096, num_tokens in [1, 2^20].  The branch condition compares a loaded f16 value,
# which the reference cannot reason about (solver/linear.py:389-391): its screening is unknown, both
# sides are explored with state.unknown_path set (engine/executor.py:588-619), and the i32 row offset
# inside the branch overflows on a path that also carries the float atom, so those findings are
# `unknown` (engine/detectors.py:126-130).
wrapper clamp_rows(out: tensor, input: tensor, threshold: f32) {
  let hidden_size: i32 = input.size(-1);
  let num_tokens: i32 = input.numel() / hidden_size;
  launch clamp_rows_kernel<<<num_tokens; 1024>>>(out.data_ptr(), input.data_ptr(), threshold, hidden_size);
}
kernel clamp_rows_kernel(out: handle<f16>, input: handle<f16>, threshold: f32, hidden_size: i32) {
  for (i32 idx = threadIdx.x; idx < hidden_size; idx += blockDim.x) {
    f16 x = input[blockIdx.x * hidden_size + idx];
    if (f32(x) > threshold) {
      out[blockIdx.x * hidden_size + idx] = x;
    }
  }
}

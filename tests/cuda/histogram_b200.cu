// CUDA form of the bench's B200 Hist member (paper_2007_01277_b200/kernels/b200/histogram.mk):
// 64 bins over [-4, 4], four 128-bit loads in flight per thread, warp-private shared-memory
// bins, the n % 4 trailing values binned by block 0. Input of the restricted-CUDA frontend
// test: it must produce the same bins as the MK+ member, bit for bit.
//@ grid=256
__global__ void __launch_bounds__(1024) hist(const float* __restrict__ hi_x, int* hi_out, int hi_n) {
  __shared__ int hi_bins[2048];
  int tid = threadIdx.x;
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int wb = (tid / 32) * 64;
  int n4 = hi_n / 4;
  int last = n4 - 1;
  int stride = gridDim.x * nthr;
  for (int i = blockIdx.x * nthr + tid; i < n4; i += 4 * stride) {
    int j1 = i + stride, j2 = j1 + stride, j3 = j2 + stride;
    float4 a = reinterpret_cast<const float4*>(hi_x)[i];
    float4 b = reinterpret_cast<const float4*>(hi_x)[min(j1, last)];
    float4 c = reinterpret_cast<const float4*>(hi_x)[min(j2, last)];
    float4 d = reinterpret_cast<const float4*>(hi_x)[min(j3, last)];
    if (a.x >= -4.0f && a.x <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((a.x + 4.0f) * 8.0f), 63)], 1);
    if (a.y >= -4.0f && a.y <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((a.y + 4.0f) * 8.0f), 63)], 1);
    if (a.z >= -4.0f && a.z <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((a.z + 4.0f) * 8.0f), 63)], 1);
    if (a.w >= -4.0f && a.w <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((a.w + 4.0f) * 8.0f), 63)], 1);
    if (j1 < n4) {
      if (b.x >= -4.0f && b.x <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((b.x + 4.0f) * 8.0f), 63)], 1);
      if (b.y >= -4.0f && b.y <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((b.y + 4.0f) * 8.0f), 63)], 1);
      if (b.z >= -4.0f && b.z <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((b.z + 4.0f) * 8.0f), 63)], 1);
      if (b.w >= -4.0f && b.w <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((b.w + 4.0f) * 8.0f), 63)], 1);
    }
    if (j2 < n4) {
      if (c.x >= -4.0f && c.x <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((c.x + 4.0f) * 8.0f), 63)], 1);
      if (c.y >= -4.0f && c.y <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((c.y + 4.0f) * 8.0f), 63)], 1);
      if (c.z >= -4.0f && c.z <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((c.z + 4.0f) * 8.0f), 63)], 1);
      if (c.w >= -4.0f && c.w <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((c.w + 4.0f) * 8.0f), 63)], 1);
    }
    if (j3 < n4) {
      if (d.x >= -4.0f && d.x <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((d.x + 4.0f) * 8.0f), 63)], 1);
      if (d.y >= -4.0f && d.y <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((d.y + 4.0f) * 8.0f), 63)], 1);
      if (d.z >= -4.0f && d.z <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((d.z + 4.0f) * 8.0f), 63)], 1);
      if (d.w >= -4.0f && d.w <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((d.w + 4.0f) * 8.0f), 63)], 1);
    }
  }
  if (blockIdx.x == 0 && tid < hi_n - 4 * n4) {
    float v = hi_x[4 * n4 + tid];
    if (v >= -4.0f && v <= 4.0f) atomicAdd(&hi_bins[wb + min(__float2int_rz((v + 4.0f) * 8.0f), 63)], 1);
  }
  __syncthreads();
  for (int b = tid; b < 64; b += nthr) {
    int s = 0;
    for (int w = 0; w < nthr / 32; ++w) s += hi_bins[w * 64 + b];
    atomicAdd(&hi_out[b], s);
  }
}

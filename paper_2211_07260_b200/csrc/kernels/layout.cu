// Operand staging for the host-buffer API (suite.sgemm / suite.sgemm_tf32).
//
// The GEMM kernels read A column-major (CLBlast's internal layout: a K x M
// buffer, M contiguous) and need every dimension padded to a multiple of
// their tile. A user hands over a row-major M x K A. Instead of transposing
// on the host, the call uploads A as is and this kernel writes the padded
// transpose on the device: out[c][r] = in[r][c] for r < rows, c < cols, zero
// elsewhere in the out_rows x out_cols buffer (zero K-padding keeps the
// product exact: the padded K terms are 0 * 0). CLBlast runs the same
// transpose-and-pad step as its "indirect" GEMM pre-processing kernel.
//
// HBM-bound (one read and one write per element): 32 x 32 tiles through
// shared memory (33-word rows, no bank conflicts) so both the reads of `in`
// and the writes of `out` are 128-byte coalesced.

extern "C" __global__ void __launch_bounds__(256) transpose_pad(float *__restrict__ out, const float *__restrict__ in,
                                                                int rows, int cols, int out_rows, int out_cols) {
    __shared__ float tile[32][33];
    const int c0 = blockIdx.x * 32;  // input columns = output rows
    const int r0 = blockIdx.y * 32;  // input rows = output columns
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int r = r0 + j, c = c0 + threadIdx.x;
        tile[j][threadIdx.x] = (r < rows && c < cols) ? in[(size_t)r * cols + c] : 0.0f;
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int orow = c0 + j, ocol = r0 + threadIdx.x;
        if (orow < out_rows && ocol < out_cols) out[(size_t)orow * out_cols + ocol] = tile[threadIdx.x][j];
    }
}

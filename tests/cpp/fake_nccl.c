/* Test double for ncclAllReduce (RXGS_NCCL_LIBRARY=...): behaves like a
 * sum over two ranks holding identical buffers (every f64 value doubles) and
 * records the element count, so a one-GPU test can check that
 * rxgs_train_allreduce reduces the WHOLE flat gradient buffer, geometry
 * segment included.  Driver API only: the product links cudart statically. */
#include <cuda.h>
#include <stdlib.h>

static size_t g_last_count = 0;
static int g_calls = 0;

size_t fake_nccl_last_count(void) { return g_last_count; }
int fake_nccl_calls(void) { return g_calls; }

int ncclAllReduce(const void* send, void* recv, size_t count, int dtype, int op, void* comm, CUstream stream) {
    (void)comm;
    if (dtype != 8 || op != 0) return 4; /* ncclInvalidArgument */
    g_last_count = count;
    g_calls += 1;
    double* h = (double*)malloc(count * sizeof(double) + 8);
    if (!h) return 1;
    if (cuStreamSynchronize(stream) != CUDA_SUCCESS) return 1;
    if (cuMemcpyDtoH(h, (CUdeviceptr)send, count * sizeof(double)) != CUDA_SUCCESS) return 1;
    for (size_t i = 0; i < count; ++i) h[i] *= 2.0;
    if (cuMemcpyHtoD((CUdeviceptr)recv, h, count * sizeof(double)) != CUDA_SUCCESS) return 1;
    free(h);
    return 0;
}

const char* ncclGetErrorString(int r) { return r ? "fake nccl error" : "no error"; }

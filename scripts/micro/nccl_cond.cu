// Probe: can ncclAllGather be captured into the body of a CUDA-graph conditional
// WHILE node (world = 1 here)? Times an iteration of kernel + all-gather + control.
// nvcc -gencode arch=compute_100a,code=sm_100a -I$NCCL/include -L$NCCL/lib -l:libnccl.so.2 nccl_cond.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <nccl.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("line %d %s -> %s\n", __LINE__, #x, cudaGetErrorString(e)); return 1; } } while (0)
#define NK(x) do { ncclResult_t r = (x); if (r) { printf("line %d %s -> %s\n", __LINE__, #x, ncclGetErrorString(r)); return 1; } } while (0)

__global__ void k_fill(int *a, int n, int *it) { for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = *it + i; }
__global__ void k_ctl(cudaGraphConditionalHandle h, int *it, const int *b, int n, int iters, int *bad) {
    int k = *it;
    if (b[n - 1] != k + n - 1) *bad = 1;
    *it = k + 1;
    cudaGraphSetConditional(h, k + 1 < iters ? 1 : 0);
}

int main() {
    const int n = 1 << 16, iters = 200;
    int *a, *b, *it, *bad;
    CK(cudaMalloc(&a, n * 4));
    CK(cudaMalloc(&b, n * 4));
    CK(cudaMalloc(&it, 4));
    CK(cudaMalloc(&bad, 4));
    CK(cudaMemset(it, 0, 4));
    CK(cudaMemset(bad, 0, 4));
    ncclComm_t comm;
    int dev = 0;
    NK(ncclCommInitAll(&comm, 1, &dev));
    cudaStream_t cs, s;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CK(cudaStreamCreate(&s));
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t wn;
    CK(cudaGraphAddNode(&wn, g, nullptr, 0, &p));
    CK(cudaStreamBeginCaptureToGraph(cs, p.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    k_fill<<<1, 256, 0, cs>>>(a, n, it);
    ncclResult_t nr = ncclAllGather(a, b, n, ncclInt32, comm, cs);
    k_ctl<<<1, 1, 0, cs>>>(h, it, b, n, iters, bad);
    cudaGraph_t out;
    cudaError_t ce = cudaStreamEndCapture(cs, &out);
    printf("capture: nccl=%s cuda=%s\n", ncclGetErrorString(nr), cudaGetErrorString(ce));
    if (nr || ce) return 1;
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, g, 0));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    CK(cudaEventRecord(e0, s));
    CK(cudaGraphLaunch(ex, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaStreamSynchronize(s));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int hit, hbad;
    CK(cudaMemcpy(&hit, it, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost));
    printf("nccl all-gather in a WHILE body: iterations=%d bad=%d, %.2f us per iteration\n", hit, hbad, 1000 * ms / iters);
    return 0;
}

// Probe: CUDA graph conditional nodes (WHILE + SWITCH) whose bodies hold a
// cooperative kernel (grid sync), a plain kernel and a memset, driven by a
// 1-thread control kernel calling cudaGraphSetConditional. Also times an empty
// WHILE iteration (the per-iteration overhead of a device-resident loop).
// nvcc -gencode arch=compute_100a,code=sm_100a -o graph_cond graph_cond.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_coop(int *buf, int n) {
    auto g = cooperative_groups::this_grid();
    for (int i = g.thread_rank(); i < n; i += g.size()) buf[i] += 1;
    g.sync();
    if (g.thread_rank() == 0) buf[n] = buf[0] + buf[n - 1];
}
__global__ void k_plain(int *buf, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) buf[i] += 10;
}
__global__ void k_ctl(cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hs, int *it, int iters) {
    int k = ++*it;
    cudaGraphSetConditional(hs, k & 1);
    cudaGraphSetConditional(hw, k < iters ? 1 : 0);
}
__global__ void k_ctl_only(cudaGraphConditionalHandle hw, int *it, int iters) {
    int k = ++*it;
    cudaGraphSetConditional(hw, k < iters ? 1 : 0);
}

int main() {
    const int n = 1 << 20, iters = 1000;
    int *buf, *it;
    CK(cudaMalloc(&buf, (n + 1) * sizeof(int)));
    CK(cudaMalloc(&it, sizeof(int)));
    CK(cudaMemset(buf, 0, (n + 1) * sizeof(int)));
    CK(cudaMemset(it, 0, sizeof(int)));
    int nb = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_coop, 256, 0));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int coop_grid = nb * sms;

    cudaGraph_t graph;
    CK(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle hw, hs;
    CK(cudaGraphConditionalHandleCreate(&hw, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp = {cudaGraphNodeTypeConditional};
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CK(cudaGraphAddNode(&wnode, graph, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    CK(cudaGraphConditionalHandleCreate(&hs, body, 0, cudaGraphCondAssignDefault));
    // body: switch(hs) { 0: memset + coop kernel, 1: plain kernel } ; ctl
    cudaGraphNodeParams sp = {cudaGraphNodeTypeConditional};
    sp.conditional.handle = hs;
    sp.conditional.type = cudaGraphCondTypeSwitch;
    sp.conditional.size = 2;
    cudaGraphNode_t snode;
    CK(cudaGraphAddNode(&snode, body, nullptr, 0, &sp));
    cudaGraph_t b0 = sp.conditional.phGraph_out[0], b1 = sp.conditional.phGraph_out[1];
    cudaGraphNode_t ms, kc, kp, kt;
    cudaMemsetParams mp = {};
    mp.dst = buf + n; mp.value = 0; mp.elementSize = 4; mp.width = 1; mp.height = 1;
    CK(cudaGraphAddMemsetNode(&ms, b0, nullptr, 0, &mp));
    void *argsc[] = {&buf, (void *)&n};
    cudaKernelNodeParams kpc = {};
    kpc.func = (void *)k_coop; kpc.gridDim = dim3(coop_grid); kpc.blockDim = dim3(256); kpc.kernelParams = argsc;
    CK(cudaGraphAddKernelNode(&kc, b0, &ms, 1, &kpc));
    cudaLaunchAttributeValue av = {};
    av.cooperative = 1;
    CK(cudaGraphKernelNodeSetAttribute(kc, cudaLaunchAttributeCooperative, &av));
    cudaKernelNodeParams kpp = kpc;
    kpp.func = (void *)k_plain; kpp.gridDim = dim3(sms * 4);
    CK(cudaGraphAddKernelNode(&kp, b1, nullptr, 0, &kpp));
    int it_ = iters;
    void *argst[] = {&hw, &hs, &it, &it_};
    cudaKernelNodeParams kpt = {};
    kpt.func = (void *)k_ctl; kpt.gridDim = dim3(1); kpt.blockDim = dim3(1); kpt.kernelParams = argst;
    CK(cudaGraphAddKernelNode(&kt, body, &snode, 1, &kpt));
    cudaGraphExec_t exec;
    CK(cudaGraphInstantiate(&exec, graph, 0));
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    CK(cudaEventRecord(a, s));
    CK(cudaGraphLaunch(exec, s));
    CK(cudaEventRecord(b, s));
    CK(cudaStreamSynchronize(s));
    float ms_ = 0;
    cudaEventElapsedTime(&ms_, a, b);
    int h[2];
    CK(cudaMemcpy(h, buf, 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h + 1, it, 4, cudaMemcpyDeviceToHost));
    printf("while+switch+coop: iters=%d buf[0]=%d (expect %d) %.3f ms = %.2f us/iter (coop grid %d)\n", h[1], h[0],
           (iters + 1) / 2 + 10 * (iters / 2), ms_, 1000.0 * ms_ / iters, coop_grid);

    // empty loop overhead: WHILE { ctl }
    cudaGraph_t g2;
    CK(cudaGraphCreate(&g2, 0));
    cudaGraphConditionalHandle hw2;
    CK(cudaGraphConditionalHandleCreate(&hw2, g2, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp2 = {cudaGraphNodeTypeConditional};
    wp2.conditional.handle = hw2;
    wp2.conditional.type = cudaGraphCondTypeWhile;
    wp2.conditional.size = 1;
    cudaGraphNode_t w2;
    CK(cudaGraphAddNode(&w2, g2, nullptr, 0, &wp2));
    CK(cudaMemset(it, 0, 4));
    int iters2 = 10000;
    void *args2[] = {&hw2, &it, &iters2};
    cudaKernelNodeParams k2 = {};
    k2.func = (void *)k_ctl_only; k2.gridDim = dim3(1); k2.blockDim = dim3(1); k2.kernelParams = args2;
    cudaGraphNode_t n2;
    CK(cudaGraphAddKernelNode(&n2, wp2.conditional.phGraph_out[0], nullptr, 0, &k2));
    cudaGraphExec_t e2;
    CK(cudaGraphInstantiate(&e2, g2, 0));
    CK(cudaEventRecord(a, s));
    CK(cudaGraphLaunch(e2, s));
    CK(cudaEventRecord(b, s));
    CK(cudaStreamSynchronize(s));
    cudaEventElapsedTime(&ms_, a, b);
    printf("empty while: %.3f ms = %.2f us/iter\n", ms_, 1000.0 * ms_ / iters2);

    // stream capture INTO a conditional body: cooperative launch + memset + control kernel
    cudaGraph_t g3;
    CK(cudaGraphCreate(&g3, 0));
    cudaGraphConditionalHandle hw3;
    CK(cudaGraphConditionalHandleCreate(&hw3, g3, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp3 = {cudaGraphNodeTypeConditional};
    wp3.conditional.handle = hw3;
    wp3.conditional.type = cudaGraphCondTypeWhile;
    wp3.conditional.size = 1;
    cudaGraphNode_t w3;
    CK(cudaGraphAddNode(&w3, g3, nullptr, 0, &wp3));
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    CK(cudaStreamBeginCaptureToGraph(cs, wp3.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    CK(cudaMemsetAsync(buf + n, 0, 4, cs));
    int nn = n;
    void *a3[] = {&buf, &nn};
    CK(cudaLaunchCooperativeKernel((void *)k_coop, dim3(coop_grid), dim3(256), a3, 0, cs));
    int iters3 = 1000;
    k_ctl_only<<<1, 1, 0, cs>>>(hw3, it, iters3);
    CK(cudaGetLastError());
    cudaGraph_t cap;
    CK(cudaStreamEndCapture(cs, &cap));
    CK(cudaMemset(it, 0, 4));
    CK(cudaMemset(buf, 0, 4));
    cudaGraphExec_t e3;
    CK(cudaGraphInstantiate(&e3, g3, 0));
    CK(cudaEventRecord(a, s));
    CK(cudaGraphLaunch(e3, s));
    CK(cudaEventRecord(b, s));
    CK(cudaStreamSynchronize(s));
    cudaEventElapsedTime(&ms_, a, b);
    CK(cudaMemcpy(h, buf, 4, cudaMemcpyDeviceToHost));
    printf("captured coop in while: buf[0]=%d (expect %d) %.3f ms = %.2f us/iter\n", h[0], iters3, ms_, 1000.0 * ms_ / iters3);
    return 0;
}

// Probe: which conditional-graph constructs instantiate on this driver.
// ./graph_nest <variant>: 0 nested WHILE in WHILE; 1 + SWITCH(5) default 5 in the
// inner body; 2 + an unused handle; 3 + an empty SWITCH body; 4 all of them
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("variant %d: line %d %s -> %s\n", v, __LINE__, #x, cudaGetErrorString(e)); return 1; } } while (0)

struct H { cudaGraphConditionalHandle o, i, m, u; };
__global__ void k_pre(H h, int *c) { cudaGraphSetConditional(h.i, 1); }
__global__ void k_in(H h, int *c, int sw) { int k = ++c[0]; if (sw) cudaGraphSetConditional(h.m, k % 3); cudaGraphSetConditional(h.i, k % 4 != 0); }
__global__ void k_post(H h, int *c) { int k = ++c[1]; cudaGraphSetConditional(h.o, k < 10); }
__global__ void k_work(int *c, int j) { atomicAdd(c + 2 + j, 1); }

int main(int argc, char **argv) {
    const int v = argc > 1 ? atoi(argv[1]) : 0;
    int *c;
    CK(cudaMalloc(&c, 64));
    CK(cudaMemset(c, 0, 64));
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    H h{};
    CK(cudaGraphConditionalHandleCreate(&h.o, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h.o; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    cudaGraphNode_t no;
    CK(cudaGraphAddNode(&no, g, nullptr, 0, &p));
    cudaGraph_t bo = p.conditional.phGraph_out[0];
    CK(cudaGraphConditionalHandleCreate(&h.i, bo, 0, cudaGraphCondAssignDefault));
    if (v == 2 || v == 4) CK(cudaGraphConditionalHandleCreate(&h.u, bo, 0, cudaGraphCondAssignDefault));
    void *a[] = {&h, &c};
    cudaKernelNodeParams kp = {};
    kp.gridDim = dim3(1); kp.blockDim = dim3(1); kp.kernelParams = a; kp.func = (void *)k_pre;
    cudaGraphNode_t n1, n2, n3;
    CK(cudaGraphAddKernelNode(&n1, bo, nullptr, 0, &kp));
    cudaGraphNodeParams q = {};
    q.type = cudaGraphNodeTypeConditional;
    q.conditional.handle = h.i; q.conditional.type = cudaGraphCondTypeWhile; q.conditional.size = 1;
    CK(cudaGraphAddNode(&n2, bo, &n1, 1, &q));
    cudaGraph_t bi = q.conditional.phGraph_out[0];
    int sw = v >= 1;
    if (sw) CK(cudaGraphConditionalHandleCreate(&h.m, bi, v == 1 || v == 4 ? 5 : 0, cudaGraphCondAssignDefault));
    void *ai[] = {&h, &c, &sw};
    cudaKernelNodeParams ki = kp; ki.kernelParams = ai; ki.func = (void *)k_in;
    cudaGraphNode_t m1, m2;
    CK(cudaGraphAddKernelNode(&m1, bi, nullptr, 0, &ki));
    if (sw) {
        cudaGraphNodeParams r = {};
        r.type = cudaGraphNodeTypeConditional;
        r.conditional.handle = h.m; r.conditional.type = cudaGraphCondTypeSwitch; r.conditional.size = 5;
        CK(cudaGraphAddNode(&m2, bi, &m1, 1, &r));
        for (int j = 0; j < 5; j++) {
            if ((v == 3 || v == 4) && j >= 3) continue;   // leave bodies 3, 4 empty
            int jj = j;
            void *aw[] = {&c, &jj};
            cudaKernelNodeParams kw = kp; kw.kernelParams = aw; kw.func = (void *)k_work;
            cudaGraphNode_t w;
            CK(cudaGraphAddKernelNode(&w, r.conditional.phGraph_out[j], nullptr, 0, &kw));
        }
    }
    kp.func = (void *)k_post;
    CK(cudaGraphAddKernelNode(&n3, bo, &n2, 1, &kp));
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, g, 0));
    CK(cudaGraphLaunch(ex, 0));
    CK(cudaDeviceSynchronize());
    int hc[8];
    CK(cudaMemcpy(hc, c, 32, cudaMemcpyDeviceToHost));
    printf("variant %d ok: inner=%d outer=%d work=%d %d %d\n", v, hc[0], hc[1], hc[2], hc[3], hc[4]);
    return 0;
}

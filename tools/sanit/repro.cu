// Minimal synccheck reproducer: a grid-stride Dot2 loop + reduce_last (arith.cuh), launched (a) plainly,
// (b) captured in a graph, (c) as the body of a conditional WHILE graph node.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2303_03398_b200/csrc/arith.cuh"
using namespace maspcg;

__global__ void __launch_bounds__(256) k_dot(const double *x, unsigned n, double *partials, unsigned *ticket,
                                             double *out, int *done, int guard) {
    if (guard && *(volatile int *)done) return;
    Acc<true> acc[1];
    for (unsigned c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) acc[0].add(x[c], x[c]);
    Acc<true> o[1];
    if (reduce_last<true, 256, 1>(acc, partials, ticket, blockIdx.x, gridDim.x, o))
        if (threadIdx.x == 0) { out[0] = o[0].value(); }
}
__global__ void k_cond(cudaGraphConditionalHandle h, int *count, int maxit) {
    const int c = ++*count;
    cudaGraphSetConditional(h, c < maxit ? 1 : 0);
}

int main(int argc, char **argv) {
    const unsigned n = 1000003;
    double *x, *part, *out; unsigned *ticket; int *done, *count;
    cudaMalloc(&x, n * 8); cudaMemset(x, 0, n * 8);
    cudaMalloc(&part, 2 * kPartialSlots * 8); cudaMalloc(&out, 8);
    cudaMalloc(&ticket, 4); cudaMemset(ticket, 0, 4);
    cudaMalloc(&done, 4); cudaMemset(done, 0, 4);
    cudaMalloc(&count, 4); cudaMemset(count, 0, 4);
    const int mode = argc > 1 ? atoi(argv[1]) : 0, guard = argc > 2 ? atoi(argv[2]) : 0;
    cudaStream_t s; cudaStreamCreate(&s);
    const unsigned grid = 148 * 4;
    if (mode == 0) {
        for (int it = 0; it < 3; ++it) k_dot<<<grid, 256, 0, s>>>(x, n, part, ticket, out, done, guard);
    } else if (mode == 1) {
        cudaGraph_t g; cudaGraphExec_t e;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int it = 0; it < 3; ++it) k_dot<<<grid, 256, 0, s>>>(x, n, part, ticket, out, done, guard);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&e, g, 0);
        cudaGraphLaunch(e, s);
    } else {
        cudaGraph_t g; cudaGraphExec_t e;
        cudaGraphCreate(&g, 0);
        cudaGraphConditionalHandle h;
        cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
        cudaGraphNodeParams p = {};
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = h;
        p.conditional.type = cudaGraphCondTypeWhile;
        p.conditional.size = 1;
        cudaGraphNode_t node;
        cudaGraphAddNode(&node, g, nullptr, 0, &p);
        cudaGraph_t body = p.conditional.phGraph_out[0];
        cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
        k_dot<<<grid, 256, 0, s>>>(x, n, part, ticket, out, done, guard);
        k_cond<<<1, 1, 0, s>>>(h, count, 3);
        cudaStreamEndCapture(s, &body);
        cudaGraphInstantiate(&e, g, 0);
        cudaGraphLaunch(e, s);
    }
    cudaError_t err = cudaStreamSynchronize(s);
    printf("mode %d guard %d: %s\n", mode, guard, cudaGetErrorString(err));
    return err != cudaSuccess;
}

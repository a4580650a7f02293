#include <cuda_runtime.h>
#include <cstdio>
__global__ void body_kernel(int* counter, cudaGraphConditionalHandle h, int limit) {
    int c = ++(*counter);
    cudaGraphSetConditional(h, c < limit ? 1 : 0);
}
__global__ void pro(int* counter) { *counter = 0; }
int main() {
    int* d; cudaMalloc(&d, 4);
    cudaStream_t s, s2; cudaStreamCreate(&s); cudaStreamCreate(&s2);
    cudaGraph_t g; 
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    pro<<<1,1,0,s>>>(d);
    cudaStreamCaptureStatus st; const cudaGraphNode_t* deps; size_t nd; cudaGraph_t cg;
    cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, cg, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    cudaGraphNode_t cn;
    cudaError_t e = cudaGraphAddNode(&cn, cg, deps, nd, &p);
    printf("addnode %s\n", cudaGetErrorString(e));
    cudaGraph_t body = p.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(s2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    printf("begin2 %s\n", cudaGetErrorString(e));
    body_kernel<<<1,1,0,s2>>>(d, h, 7);
    cudaGraph_t tmp; e = cudaStreamEndCapture(s2, &tmp); printf("end2 %s\n", cudaGetErrorString(e));
    e = cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies); printf("upd %s\n", cudaGetErrorString(e));
    pro<<<1,1,0,s>>>(d + 0);  // overwritten? no: make a second counter read
    e = cudaStreamEndCapture(s, &g); printf("end %s\n", cudaGetErrorString(e));
    cudaGraphExec_t ge; e = cudaGraphInstantiate(&ge, g, 0); printf("inst %s\n", cudaGetErrorString(e));
    e = cudaGraphLaunch(ge, s); cudaStreamSynchronize(s); printf("launch %s\n", cudaGetErrorString(e));
    int h_c = -1; cudaMemcpy(&h_c, d, 4, cudaMemcpyDeviceToHost); printf("counter after (reset by tail pro) %d\n", h_c);
    return 0;
}

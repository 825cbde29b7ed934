// Cost of a cooperative-groups grid-wide barrier on this GPU vs grid size (context for K1, which
// synchronises once per DP layer).   nvcc -gencode arch=compute_100a,code=sm_100a -O3 grid_sync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int n, int* sink) {
    cg::grid_group g = cg::this_grid();
    int acc = 0;
    for (int i = 0; i < n; i++) { acc += i ^ threadIdx.x; g.sync(); }
    if (acc == -1) *sink = acc;
}
int main() {
    int* sink; cudaMalloc(&sink, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int grids[] = {1, 8, 32, 74, 148, 296};
    for (int gi = 0; gi < 6; gi++) {
        int grid = grids[gi];
        for (int n : {0, 200}) {
            void* args[] = {&n, &sink};
            cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("grid %4d  syncs %4d  %8.3f ms  %s\n", grid, n, ms, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}

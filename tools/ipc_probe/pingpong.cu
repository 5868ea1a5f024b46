// Can two processes' spinning kernels make progress on ONE GPU (time slicing)?  Process 0 allocates a
// flag pair, writes its IPC handle to a file; process 1 opens it.  Each kernel alternately waits for
// the other's counter and bumps its own, N times (bounded by a 10 s watchdog).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>
#include <cuda_runtime.h>

__global__ void pingpong(volatile unsigned long long* flags, int me, int n, int* result) {
    const unsigned long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        // wait until the other side reached i (side 0 goes first)
        const unsigned long long want = me == 0 ? i : i + 1;
        while (flags[1 - me] < want) {
            if (clock64() - t0 > 20000000000ull) { *result = -1; return; }
        }
        __threadfence_system();
        flags[me] = i + 1;
        __threadfence_system();
    }
    *result = n;
}

int main(int argc, char** argv) {
    const int me = atoi(argv[1]), n = atoi(argv[2]);
    const char* path = argv[3];
    unsigned long long* flags = nullptr;
    if (me == 0) {
        cudaMalloc(&flags, 2 * sizeof(unsigned long long));
        cudaMemset(flags, 0, 2 * sizeof(unsigned long long));
        cudaIpcMemHandle_t h;
        cudaIpcGetMemHandle(&h, flags);
        FILE* f = fopen(path, "wb");
        fwrite(&h, sizeof h, 1, f);
        fclose(f);
    } else {
        cudaIpcMemHandle_t h;
        FILE* f = nullptr;
        for (int i = 0; i < 200 && !(f = fopen(path, "rb")); ++i) usleep(50000);
        if (!f) { printf("no handle\n"); return 1; }
        fread(&h, sizeof h, 1, f);
        fclose(f);
        if (cudaIpcOpenMemHandle((void**)&flags, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            printf("open failed: %s\n", cudaGetErrorString(cudaGetLastError()));
            return 1;
        }
    }
    int* res;
    cudaMallocManaged(&res, sizeof(int));
    *res = 0;
    pingpong<<<1, 1>>>(flags, me, n, res);
    cudaError_t e = cudaDeviceSynchronize();
    printf("process %d: %s result %d\n", me, cudaGetErrorString(e), *res);
    return 0;
}

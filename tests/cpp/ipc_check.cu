// CUDA IPC the way the sharded driver's peer mode maps its peers' buffers
// (shard_driver.cu NcclImpl::exchange_peer_ptrs): a cudaMalloc'd buffer
// exported with cudaIpcGetMemHandle in one process, opened with
// cudaIpcMemLazyEnablePeerAccess in another, and written by a kernel there.
//   ipc_check serve <file>   allocate, publish the handle, wait, verify
//   ipc_check write <file>   open the handle, store the pattern, signal
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>

constexpr unsigned kWords = 1 << 20;

__global__ void stamp(unsigned* p, unsigned n) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i * 2654435761u;
}

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            std::printf("FAIL %s: %s\n", #x, cudaGetErrorString(e));                 \
            return 1;                                                                \
        }                                                                            \
    } while (0)

static bool wait_for(const std::string& f, int seconds) {
    for (int i = 0; i < seconds * 100; ++i) {
        if (std::ifstream(f).good()) return true;
        std::this_thread::sleep_for(std::chrono::milliseconds(10));
    }
    return false;
}

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const std::string mode = argv[1], file = argv[2];
    if (mode == "serve") {
        unsigned* buf = nullptr;
        CK(cudaMalloc(&buf, kWords * sizeof(unsigned)));
        CK(cudaMemset(buf, 0, kWords * sizeof(unsigned)));
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, buf));
        {
            std::ofstream o(file + ".tmp", std::ios::binary);
            o.write(reinterpret_cast<const char*>(&h), sizeof(h));
        }
        std::rename((file + ".tmp").c_str(), file.c_str());
        if (!wait_for(file + ".done", 120)) {
            std::printf("FAIL no writer\n");
            return 1;
        }
        unsigned* host = new unsigned[kWords];
        CK(cudaMemcpy(host, buf, kWords * sizeof(unsigned), cudaMemcpyDeviceToHost));
        for (unsigned i = 0; i < kWords; ++i)
            if (host[i] != i * 2654435761u) {
                std::printf("FAIL word %u = %u\n", i, host[i]);
                return 1;
            }
        std::printf("OK %u words written through the IPC mapping\n", kWords);
        return 0;
    }
    if (!wait_for(file, 120)) {
        std::printf("FAIL no handle\n");
        return 1;
    }
    cudaIpcMemHandle_t h;
    {
        std::ifstream in(file, std::ios::binary);
        in.read(reinterpret_cast<char*>(&h), sizeof(h));
    }
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    stamp<<<256, 256>>>(static_cast<unsigned*>(p), kWords);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaIpcCloseMemHandle(p));
    std::ofstream(file + ".done") << "1";
    std::printf("OK written\n");
    return 0;
}

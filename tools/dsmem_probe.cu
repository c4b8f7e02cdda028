// Random 1-byte gather rate from a thread-block cluster's distributed shared memory.
//
// Question for pass B of the partitioned path: if a group's pilot slice
// lived in the shared memory of a cluster of CS CTAs (CS x ~200 KB) instead of L2, how
// many random pilot lookups per second would the GPU serve? Compare with the L2 gather
// rate over a 32 MiB buffer (~285 G/s, profiles/r01_gather_sweep.jsonl).
//
// Each CTA fills `per_cta` bytes of dynamic shared memory; every thread then issues
// `iters` x ILP lookups at uniform random byte offsets of the cluster's CS x per_cta bytes
// (mapa + ld.shared::cluster.u8), XOR-folding the bytes into one output word.
// Not part of the library. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -o tools/dsmem_probe tools/dsmem_probe.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

constexpr int kILP = 8;

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

__device__ __forceinline__ uint32_t ld_cluster_u8(uint32_t local_addr, uint32_t rank) {
    uint32_t remote, v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
    asm volatile("ld.shared::cluster.u8 %0, [%1];" : "=r"(v) : "r"(remote) : "memory");
    return v;
}

template <bool LOCAL>
__global__ void k_probe(uint32_t per_cta, uint32_t cs, int iters, uint32_t* out) {
    extern __shared__ __align__(16) uint8_t sm[];
    cg::cluster_group cluster = cg::this_cluster();
    for (uint32_t i = threadIdx.x; i < per_cta / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = mix32(i + blockIdx.x * 977u);
    cluster.sync();
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    uint32_t st = mix32(blockIdx.x * blockDim.x + threadIdx.x + 1);
    uint32_t acc = 0;
    const uint32_t total = LOCAL ? per_cta : per_cta * cs;
    for (int it = 0; it < iters; it++) {
        uint32_t v[kILP];
#pragma unroll
        for (int j = 0; j < kILP; j++) {
            st = mix32(st + j + 0x9e3779b9u);
            const uint32_t idx = __umulhi(st, total);
            if (LOCAL) {
                uint32_t x;
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(x) : "r"(base + idx) : "memory");
                v[j] = x;
            } else {
                const uint32_t rank = idx / per_cta, off = idx - rank * per_cta;
                v[j] = ld_cluster_u8(base + off, rank);
            }
        }
#pragma unroll
        for (int j = 0; j < kILP; j++) acc += v[j];
        st ^= acc;  // keep the loads live
    }
    cluster.sync();  // no CTA may exit while others read its shared memory
    if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char** argv) {
    const uint32_t per_cta = argc > 1 ? atoi(argv[1]) : 200 * 1024;
    const int iters = argc > 2 ? atoi(argv[2]) : 2048;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* out;
    cudaMalloc(&out, 4);
    const int threads_list[] = {256, 512, 1024};
    const uint32_t cs_list[] = {1, 2, 4, 8, 16};
    for (int local = 1; local >= 0; local--) {
        for (uint32_t cs : cs_list) {
            if (local && cs != 1) continue;
            for (int threads : threads_list) {
                auto kern = local ? k_probe<true> : k_probe<false>;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, per_cta);
                if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = cs;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.blockDim = dim3(threads);
                cfg.dynamicSmemBytes = per_cta;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                int nclusters = 0;
                cfg.gridDim = dim3(cs);
                if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters <= 0) {
                    printf("{\"local\": %d, \"cs\": %u, \"threads\": %d, \"error\": \"%s\"}\n", local, cs,
                           threads, cudaGetErrorString(cudaGetLastError()));
                    continue;
                }
                cfg.gridDim = dim3(nclusters * cs);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaLaunchKernelEx(&cfg, kern, per_cta, cs, iters / 8, out);  // warm-up
                cudaEventRecord(e0);
                cudaLaunchKernelEx(&cfg, kern, per_cta, cs, iters, out);
                cudaEventRecord(e1);
                cudaError_t err = cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                const double lookups = (double)nclusters * cs * threads * iters * kILP;
                printf("{\"local\": %d, \"cs\": %u, \"threads\": %d, \"ctas\": %u, \"per_cta\": %u, "
                       "\"ms\": %.3f, \"glookups_s\": %.1f, \"err\": \"%s\"}\n",
                       local, cs, threads, nclusters * cs, per_cta, ms, lookups / ms / 1e6,
                       cudaGetErrorString(err));
                fflush(stdout);
            }
        }
    }
    return 0;
}

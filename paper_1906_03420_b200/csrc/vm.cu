// vm.cu — a result table that grows in place (CUDA virtual memory management).
//
// A table query appends its rows piece by piece (one piece per slot chunk / shard piece of the
// last level).  Instead of allocating every piece and concatenating them at the end (a copy of
// the whole table and twice its memory at the peak), the result reserves one virtual address
// range as large as the device's memory and maps physical memory into it in granularity-sized
// chunks as rows arrive; pieces are written (or copied once) at their final offset.  The driver
// entry points come through the runtime (cudaGetDriverEntryPoint), so the library does not
// link libcuda directly.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"

namespace gsi {
namespace {

struct VmApi {
    PFN_cuMemGetAllocationGranularity gran = nullptr;
    PFN_cuMemAddressReserve reserve = nullptr;
    PFN_cuMemAddressFree addr_free = nullptr;
    PFN_cuMemCreate create = nullptr;
    PFN_cuMemRelease release = nullptr;
    PFN_cuMemMap map = nullptr;
    PFN_cuMemUnmap unmap = nullptr;
    PFN_cuMemSetAccess access = nullptr;
    bool ok = false;
};

const VmApi &vm_api() {
    static VmApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        auto get = [](const char *name, void **fn) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fn != nullptr;
        };
        api.ok = get("cuMemGetAllocationGranularity", (void **)&api.gran) &&
                 get("cuMemAddressReserve", (void **)&api.reserve) && get("cuMemAddressFree", (void **)&api.addr_free) &&
                 get("cuMemCreate", (void **)&api.create) && get("cuMemRelease", (void **)&api.release) &&
                 get("cuMemMap", (void **)&api.map) && get("cuMemUnmap", (void **)&api.unmap) &&
                 get("cuMemSetAccess", (void **)&api.access);
        cudaGetLastError();
    });
    return api;
}

}  // namespace

TableVM *TableVM::create(int device, int k) {
    const VmApi &A = vm_api();
    if (!A.ok || getenv("GSI_TABLE_NOVM")) return nullptr;
    size_t total = 0, free_b = 0;
    if (cudaMemGetInfo(&free_b, &total) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    size_t gran = 0;
    if (A.gran(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || gran == 0) return nullptr;
    auto *t = new TableVM();
    t->device = device;
    t->k = k;
    t->gran = gran;
    t->reserved = (total + gran - 1) / gran * gran;
    CUdeviceptr base = 0;
    if (A.reserve(&base, t->reserved, gran, 0, 0) != CUDA_SUCCESS) {
        delete t;
        return nullptr;
    }
    t->base = (unsigned long long)base;
    return t;
}

// Rows [used, used + rows) of the table, mapped; nullptr (with an error set) if the device
// has no memory left for them.
int32_t *TableVM::append(unsigned long long rows) {
    const VmApi &A = vm_api();
    const size_t need = (size_t)(used + rows) * (size_t)k * 4;
    if (need > reserved) {
        set_error("result table larger than the device memory");
        return nullptr;
    }
    while (mapped < need) {
        size_t chunk = std::max<size_t>(need - mapped, std::max<size_t>(mapped / 4, (size_t)256 << 20));
        chunk = (chunk + gran - 1) / gran * gran;
        if (mapped + chunk > reserved) chunk = reserved - mapped;
        CUmemAllocationProp prop = {};
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop.location.id = device;
        CUmemGenericAllocationHandle h;
        if (A.create(&h, chunk, &prop, 0) != CUDA_SUCCESS) {
            // the stream-ordered pool may hold freed memory: return it and retry once
            cudaDeviceSynchronize();
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
            cudaGetLastError();
            if (A.create(&h, chunk, &prop, 0) != CUDA_SUCCESS) {
                set_error("result table: device memory exhausted at " + std::to_string(mapped >> 20) + " MiB");
                return nullptr;
            }
        }
        const CUdeviceptr at = (CUdeviceptr)(base + mapped);
        if (A.map(at, chunk, 0, h, 0) != CUDA_SUCCESS) {
            A.release(h);
            set_error("result table: cuMemMap failed");
            return nullptr;
        }
        CUmemAccessDesc acc = {};
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc.location.id = device;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        if (A.access(at, chunk, &acc, 1) != CUDA_SUCCESS) {
            A.unmap(at, chunk);
            A.release(h);
            set_error("result table: cuMemSetAccess failed");
            return nullptr;
        }
        chunks.push_back({(unsigned long long)h, chunk});
        mapped += chunk;
    }
    int32_t *p = (int32_t *)(base + (size_t)used * (size_t)k * 4);
    used += rows;
    return p;
}

TableVM::~TableVM() {
    const VmApi &A = vm_api();
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaDeviceSynchronize();   // no kernel may still touch the table
    size_t off = 0;
    for (auto &c : chunks) {
        A.unmap((CUdeviceptr)(base + off), c.second);
        A.release((CUmemGenericAllocationHandle)c.first);
        off += c.second;
    }
    if (base) A.addr_free((CUdeviceptr)base, reserved);
    cudaSetDevice(cur);
    cudaGetLastError();
}

}  // namespace gsi

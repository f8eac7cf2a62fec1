// Error plumbing and host helpers shared by every entry point of libkvshare.so.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace kvs {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

kvs_status cuda_status(cudaError_t e, const char *where) {
    set_error("%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
    return KVS_ECUDA;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool encode_tmap(CUtensorMap *map, CUtensorMapDataType dtype, int rank, void *gaddr,
                 const uint64_t *dims, const uint64_t *strides_bytes, const uint32_t *box,
                 CUtensorMapSwizzle swz) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p) {
            set_error("cuTensorMapEncodeTiled unavailable");
            return false;
        }
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = fn(map, dtype, (cuuint32_t)rank, gaddr, (const cuuint64_t *)dims,
                    (const cuuint64_t *)strides_bytes, (const cuuint32_t *)box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
        return false;
    }
    return true;
}

bool make_kv_map(CUtensorMap *m, const kvs_kv_arena *a) {
    const uint64_t G = a->kv_heads, D = a->head_dim, P = a->page_size;
    uint64_t dims[4] = {D, G, P, (uint64_t)a->num_pages * a->num_layers * 2};
    uint64_t strides[3] = {D * 2, G * D * 2, P * G * D * 2};
    uint32_t box[4] = {64, 1, (uint32_t)P, 1};
    return encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, a->base, dims, strides, box,
                       CU_TENSOR_MAP_SWIZZLE_128B);
}

}  // namespace kvs

extern "C" {

const char *kvs_last_error(void) { return kvs::g_err; }

int32_t kvs_abi_version(void) { return 1; }

}  // extern "C"

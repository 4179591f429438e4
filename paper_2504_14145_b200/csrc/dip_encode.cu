// dip_encode.cu -- SURVEY §8(b)'s device-mode dip_encode_candidates: pack candidates given in the
// host-view layout (split bytes, segment counts, forward / backward sequences, rank-major F/B bit
// rows -- already copied to the device) into the records the scorer reads (nibble-packed split,
// padded sequences, WORD-MAJOR bit rows). One warp per candidate builds the record in shared memory
// and writes it out with 16-byte stores; the transpose of the bit rows runs on the GPU instead of
// the host. Byte-identical to the host encoder (dip_host.cpp encode_range).
#include <cuda_runtime.h>
#include <stdint.h>

#include "dip_internal.h"

namespace dipk {

__global__ void __launch_bounds__(256) dip_encode_kernel(const EncParams p) {
    extern __shared__ __align__(16) uint8_t esm[];
    const unsigned FULL = 0xffffffffu;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t stride = p.stride;
    uint8_t *rec = esm + (size_t)warp * stride;
    const uint32_t nq = p.m * p.nm, P = p.P, fbw = p.fbw, n_max = p.n_max;
    for (uint64_t x = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp; x < p.count;
         x += (uint64_t)gridDim.x * (blockDim.x >> 5)) {
        // zero the record image
        for (uint32_t o = 16 * lane; o < stride; o += 16 * 32) *reinterpret_cast<uint4 *>(rec + o) = make_uint4(0, 0, 0, 0);
        __syncwarp();
        const uint32_t n = __ldg(&p.n[x]);
        bool flag = n > n_max || n > 65535u;
        // split: nibbles for the modules with M_max > 1, the implied value otherwise
        const uint8_t *sp = p.split + x * (uint64_t)nq;
        for (uint32_t q = lane; q < nq; q += 32) {
            const uint32_t b = q / p.nm, i = q - b * p.nm, v = __ldg(&sp[q]);
            if (p.maxsplit_gt1 >> i & 1u) {
                if (v > 15) flag = true;
                const uint32_t nib = b * p.nsplit + p.nib_slot[i];
                atomicOr(reinterpret_cast<uint32_t *>(rec + ((p.off_nib + nib / 2) & ~3u)),
                         (v & 15u) << ((nib & 1) * 4 + 8 * ((p.off_nib + nib / 2) & 3u)));
            } else if (v != (__ldg(&p.nbi[q]) > 0 ? 1u : 0u)) {
                flag = true;
            }
        }
        flag = __any_sync(FULL, flag);
        if (lane == 0) {
            const uint32_t nh = n < 65535u ? n : 65535u;
            atomicOr(reinterpret_cast<uint32_t *>(rec), nh | ((flag ? 1u : 0u) << 16));
        }
        // sequences, padded to n_pad with 0xFFFF
        uint16_t *fw = reinterpret_cast<uint16_t *>(rec + p.off_fwd), *bw = reinterpret_cast<uint16_t *>(rec + p.off_bwd);
        const uint16_t *sf = p.fwd + x * (uint64_t)n_max, *sb = p.bwd + x * (uint64_t)n_max;
        for (uint32_t t = lane; t < p.n_pad; t += 32) {
            fw[t] = t < n_max ? __ldg(&sf[t]) : (uint16_t)0xFFFF;
            bw[t] = t < n_max ? __ldg(&sb[t]) : (uint16_t)0xFFFF;
        }
        // F/B bit rows: rank-major [P][fbw] -> word-major [fbw][P]
        uint32_t *fb = reinterpret_cast<uint32_t *>(rec + p.off_fb);
        const uint32_t *src = p.fb + x * (uint64_t)P * fbw;
        for (uint32_t t = lane; t < P * fbw; t += 32) {
            const uint32_t w = t / P, r = t - w * P;
            fb[t] = __ldg(&src[r * fbw + w]);
        }
        __syncwarp();
        uint8_t *out = p.out + x * (uint64_t)stride;
        for (uint32_t o = 16 * lane; o < stride; o += 16 * 32)
            *reinterpret_cast<uint4 *>(out + o) = *reinterpret_cast<const uint4 *>(rec + o);
        __syncwarp();
    }
}

cudaError_t launch_encode(const EncParams &p, int num_sms, cudaStream_t s) {
    if (!p.count) return cudaSuccess;
    const int wpb = 8;
    const size_t smem = (size_t)wpb * p.stride;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(dip_encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const uint64_t blocks = (p.count + wpb - 1) / wpb;
    const int grid = (int)(blocks < (uint64_t)num_sms * 4 ? blocks : (uint64_t)num_sms * 4);
    dip_encode_kernel<<<grid, wpb * 32, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace dipk

/*
 * c_api_demo.c -- using libktanh.so from plain C (no torch, no C++).
 *
 *   gcc -std=c11 -O2 -I include -I /usr/local/cuda/include examples/c_api_demo.c \
 *       -L paper_1909_07729_b200 -lktanh -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1909_07729_b200 -o c_api_demo
 *   ./c_api_demo            # table handles + (with a GPU) K-TanH of a small BF16 array
 *   ./c_api_demo --no-gpu   # host-only part (table handles, validation, optimizer)
 *
 * Prints Table 1 read back from its handle, the p = 23
 * table built by the library's Sec. 2.4 optimizer, a rejected table, and --
 * on a GPU -- K-TanH of x = 0.125, 0.5, 1, 2, -5 in BF16 (Alg. 1; expected
 * 0.125, 0.46875, 0.75390625, 0.96484375, -1).
 */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <cuda_runtime.h>

#include "ktanh.h"

static uint16_t bf16_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16); }
static float bf16_value(uint16_t w) { uint32_t u = (uint32_t)w << 16; float f; memcpy(&f, &u, 4); return f; }

#define CHECK(call)                                                                    \
    do {                                                                               \
        kt_status st_ = (call);                                                        \
        if (st_ != KT_OK) {                                                            \
            fprintf(stderr, "%s: %s (%s)\n", #call, kt_status_string(st_), kt_last_error()); \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

int main(int argc, char **argv)
{
    const int gpu = !(argc > 1 && strcmp(argv[1], "--no-gpu") == 0);
    printf("libktanh ABI %d\n", kt_abi_version());

    kt_lut t1;
    int32_t E[32], r[32], b[32];
    CHECK(kt_lut_create_paper(&t1));
    CHECK(kt_lut_get(t1, E, r, b));
    printf("Table 1, row 11000: E=%d r=%d b=%d\n", E[24], r[24], b[24]);   /* (126, 0, 65) */

    kt_lut f32;
    int32_t p = 0;
    CHECK(kt_lut_create_optimized(23, 0, &f32));
    CHECK(kt_lut_mantissa_bits(f32, &p));
    CHECK(kt_lut_get(f32, E, r, b));
    printf("p = %d table, row 11000: E=%d r=%d b=%d\n", p, E[24], r[24], b[24]);

    kt_lut bad;
    CHECK(kt_lut_get(t1, E, r, b));
    r[3] = 9;                                             /* r_t outside [0, 7] */
    kt_status st = kt_lut_create(E, r, b, &bad);
    printf("invalid table -> %s: %s\n", kt_status_string(st), kt_last_error());
    if (st != KT_ERR_LUT) return 1;

    if (gpu) {
        const float xs[5] = {0.125f, 0.5f, 1.0f, 2.0f, -5.0f};
        uint16_t hx[5], hy[5];
        for (int i = 0; i < 5; ++i) hx[i] = bf16_bits(xs[i]);
        void *dx = NULL, *dy = NULL;
        if (cudaMalloc(&dx, sizeof hx) != cudaSuccess || cudaMalloc(&dy, sizeof hy) != cudaSuccess) {
            fprintf(stderr, "no CUDA device\n");
            return 1;
        }
        cudaMemcpy(dx, hx, sizeof hx, cudaMemcpyHostToDevice);
        CHECK(ktanh_bf16((const uint16_t *)dx, (uint16_t *)dy, 5, t1, NULL));
        cudaMemcpy(hy, dy, sizeof hy, cudaMemcpyDeviceToHost);        /* synchronises */
        for (int i = 0; i < 5; ++i) printf("K-TanH(%g) = %.8g\n", xs[i], bf16_value(hy[i]));
        cudaFree(dx);
        cudaFree(dy);
    }
    kt_lut_destroy(f32);
    kt_lut_destroy(t1);
    return 0;
}

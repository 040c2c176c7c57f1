// debug: run launch_conv_linear standalone (TMA path) for a few radii
#include <cstdio>
#include <vector>
#include "../../paper_2402_15322_b200/csrc/conv_linear.cu"
namespace se2 { void count_launch(int64_t) {} }
using namespace se2;
int main(int argc, char** argv) {
    int R = argc > 1 ? atoi(argv[1]) : 5;
    se2_kernel_s k;
    k.nx = 64; k.ny = 64; k.nt = 8; k.R = R; k.S = 2 * R + 1; k.band = 1;
    size_t tl = (size_t)k.nt * k.nt * k.S * ((k.S + 3) / 4 * 4);
    cudaMalloc(&k.Wl, tl * 4); cudaMemset(k.Wl, 0, tl * 4);
    float *in, *out; size_t N = (size_t)k.nx * k.ny * k.nt;
    cudaMalloc(&in, N * 4); cudaMalloc(&out, N * 4); cudaMemset(in, 0, N * 4);
    Epilogue epi; epi.op = EPI_STORE; epi.out = out;
    int bpf = 0;
    cudaError_t e = launch_conv_linear(&k, in, 1, epi, 0, &bpf);
    printf("launch: %s\n", cudaGetErrorString(e));
    e = cudaDeviceSynchronize();
    printf("R=%d sync: %s\n", R, cudaGetErrorString(e));
    return e != cudaSuccess;
}

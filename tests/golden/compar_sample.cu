// A program in the shape of PAPER.md Listing 3: a sort interface on "an array of floats
// and a scalar integer" and an mmul interface on "two 2-dimensional float arrays (A and B) with a
// size of N x M as well as two scalar integers, N and M", each with two GPU variants.
#include <cstdio>
#pragma compar include

#pragma compar method_declare interface(sort) target(CUDA) name(sort_gpu_a)
#pragma compar parameter name(arr) type(float) size(n) access_mode(readwrite)
#pragma compar parameter name(n) type(int) access_mode(read)
#pragma compar method_declare interface(sort) target(cuda) name(sort_gpu_b)

#pragma compar method_declare interface(mmul) target(CUDA) name(mmul_gpu)
#pragma compar parameter name(A) type(float) size(N, M) access_mode(read)
#pragma compar parameter name(B) type(float) size(N, M) access_mode(readwrite)
#pragma compar parameter name(N) type(int) access_mode(read)
#pragma compar parameter name(M) type(int) access_mode(read)
#pragma compar method_declare interface(mmul) target(CUBLAS) name(mmul_cublas)

int main() {
    float *arr = nullptr, *A = nullptr, *B = nullptr;
    int n = 0, N = 0, M = 0;
    #pragma compar initialize
    sort(arr, n);
    mmul(A, B, N, M);   // both interfaces are called once
    #pragma compar terminate
    return 0;
}

#include <cstdio>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
int main(){
  std::vector<std::thread> v;
  for(int t=0;t<4;++t) v.emplace_back([t]{ unsigned long long id=0, id0=0; cudaStreamGetId(cudaStreamPerThread,&id); cudaStreamGetId(0,&id0);
    cudaStream_t s; cudaStreamCreateWithFlags(&s,cudaStreamNonBlocking); unsigned long long ids=0; cudaStreamGetId(s,&ids);
    printf("thread %d perthread id %llu legacy %llu created %llu\n",t,id,id0,ids);});
  for(auto&t:v)t.join();
}

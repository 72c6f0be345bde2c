// graph_cond_test.cu -- probe of CUDA-graph conditional WHILE / IF nodes on this driver (the
// mechanism of the device-resident Newton/FGMRES graph, row f1): nested while loops whose
// bodies are stream-captured on a stack of streams, conditions set from kernels, a child IF
// node, and the cost of one graph launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/gct tools/graph_cond_test.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); return 1; } } while (0)

struct St { int outer, inner, total, ifs; };

__global__ void k_reset(St* s, cudaGraphConditionalHandle hout) {
  s->outer = s->inner = s->ifs = 0;
  s->total = 0;
  cudaGraphSetConditional(hout, 1);
}
__global__ void k_outer_init(St* s, cudaGraphConditionalHandle hin) {
  s->inner = 0;
  cudaGraphSetConditional(hin, 1);
}
__global__ void k_inner(St* s, cudaGraphConditionalHandle hin, cudaGraphConditionalHandle hif) {
  s->inner++;
  s->total++;
  cudaGraphSetConditional(hin, s->inner < 3 + s->outer);
  cudaGraphSetConditional(hif, (s->total & 1) != 0);
}
__global__ void k_if(St* s) { s->ifs++; }
__global__ void k_set(cudaGraphConditionalHandle h, unsigned v) { cudaGraphSetConditional(h, v); }
// WHILE counter: 100 iterations; also advances a SWITCH handle mod 4
__global__ void k_count(St* s, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hs, int n) {
  s->total++;
  cudaGraphSetConditional(hs, (unsigned)(s->total & 3));
  cudaGraphSetConditional(hw, (s->total % n) != 0);
}
// switch probe: the handle of the SWITCH node (in the inner while body) is set by the parent's
// init kernel (parent -> child) and by the switch bodies (child -> parent)
__global__ void k_sw_init(St* s, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hsw) {
  s->inner = 0;
  cudaGraphSetConditional(hw, 1);
  cudaGraphSetConditional(hsw, 0);
}
template <int K>
__global__ void k_sw(St* s, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hsw) {
  s->total += K + 1;   // 1 + 2 + 3 + 4 per outer iteration
  s->inner++;
  cudaGraphSetConditional(hsw, K + 1);
  cudaGraphSetConditional(hw, K + 1 < 4);
}
__global__ void k_outer_end(St* s, cudaGraphConditionalHandle hout) {
  s->outer++;
  cudaGraphSetConditional(hout, s->outer < 4);
}

static cudaError_t cond_handle(cudaStream_t parent, cudaGraphConditionalHandle* h) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  cudaError_t e = cudaStreamGetCaptureInfo(parent, &cs, nullptr, &g, nullptr, nullptr);
  if (e) return e;
  return cudaGraphConditionalHandleCreate(h, g, 0, 0);
}
static cudaError_t cond_open(cudaStream_t parent, cudaStream_t child, cudaGraphConditionalHandle h,
                             enum cudaGraphConditionalNodeType type) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t* deps;
  size_t nd;
  cudaError_t e = cudaStreamGetCaptureInfo(parent, &cs, nullptr, &g, &deps, &nd);
  if (e) return e;
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = type;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  e = cudaGraphAddNode(&node, g, deps, nd, &p);
  if (e) return e;
  e = cudaStreamUpdateCaptureDependencies(parent, &node, 1, cudaStreamSetCaptureDependencies);
  if (e) return e;
  return cudaStreamBeginCaptureToGraph(child, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                       cudaStreamCaptureModeThreadLocal);
}
static cudaError_t cond_close(cudaStream_t child) {
  cudaGraph_t b;
  return cudaStreamEndCapture(child, &b);
}

int main() {
  cudaStream_t s0, s1, s2, s3;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
  St* s;
  CK(cudaMalloc(&s, sizeof(St)));
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal));
  cudaGraphConditionalHandle hout, hin, hif;
  CK(cond_handle(s0, &hout));
  k_reset<<<1, 1, 0, s0>>>(s, hout);
  CK(cond_open(s0, s1, hout, cudaGraphCondTypeWhile));
  {
    CK(cond_handle(s1, &hin));
    k_outer_init<<<1, 1, 0, s1>>>(s, hin);
    CK(cond_open(s1, s2, hin, cudaGraphCondTypeWhile));
    {
      CK(cond_handle(s2, &hif));
      k_inner<<<1, 1, 0, s2>>>(s, hin, hif);
      CK(cond_open(s2, s3, hif, cudaGraphCondTypeIf));
      k_if<<<1, 1, 0, s3>>>(s);
      CK(cond_close(s3));
    }
    CK(cond_close(s2));
    k_outer_end<<<1, 1, 0, s1>>>(s, hout);
  }
  CK(cond_close(s1));
  CK(cudaStreamEndCapture(s0, &graph));
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, graph, 0));
  St h{};
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaGraphLaunch(ex, s0));
    CK(cudaStreamSynchronize(s0));
    CK(cudaMemcpy(&h, s, sizeof(St), cudaMemcpyDeviceToHost));
    printf("rep %d: outer %d total %d ifs %d (expect 4 18 9)\n", rep, h.outer, h.total, h.ifs);
  }
  // ---- switch probe
  {
    cudaGraph_t g2;
    CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal));
    CK(cond_handle(s0, &hout));
    k_reset<<<1, 1, 0, s0>>>(s, hout);
    CK(cond_open(s0, s1, hout, cudaGraphCondTypeWhile));
    cudaGraphConditionalHandle hw, hsw;
    CK(cond_handle(s1, &hw));
    // the switch lives in the while body: its handle belongs to that body graph, created
    // before the while node is added so that the init kernel (in s1) can set it
    cudaStreamCaptureStatus cs; cudaGraph_t g1; const cudaGraphNode_t* d; size_t nd;
    CK(cudaStreamGetCaptureInfo(s1, &cs, nullptr, &g1, &d, &nd));
    cudaGraphNodeParams pw = {};
    pw.type = cudaGraphNodeTypeConditional;
    pw.conditional.handle = hw;
    pw.conditional.type = cudaGraphCondTypeWhile;
    pw.conditional.size = 1;
    // (add the while node after the init kernel below)
    cudaGraph_t dummy; (void)dummy;
    // create the switch handle on the while body: need the body graph first -> add the node now
    // with no init kernel before it is impossible; instead create the handle on g1 (parent)
    CK(cudaGraphConditionalHandleCreate(&hsw, g1, 0, 0));
    k_sw_init<<<1, 1, 0, s1>>>(s, hw, hsw);
    CK(cond_open(s1, s2, hw, cudaGraphCondTypeWhile));
    {
      CK(cudaStreamGetCaptureInfo(s2, &cs, nullptr, &g1, &d, &nd));
      cudaGraphNodeParams ps = {};
      ps.type = cudaGraphNodeTypeConditional;
      ps.conditional.handle = hsw;
      ps.conditional.type = cudaGraphCondTypeSwitch;
      ps.conditional.size = 4;
      cudaGraphNode_t node;
      CK(cudaGraphAddNode(&node, g1, d, nd, &ps));
      CK(cudaStreamUpdateCaptureDependencies(s2, &node, 1, cudaStreamSetCaptureDependencies));
      cudaStream_t sb;
      CK(cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking));
      for (int k = 0; k < 4; ++k) {
        CK(cudaStreamBeginCaptureToGraph(sb, ps.conditional.phGraph_out[k], nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal));
        if (k == 0) k_sw<0><<<1, 1, 0, sb>>>(s, hw, hsw);
        if (k == 1) k_sw<1><<<1, 1, 0, sb>>>(s, hw, hsw);
        if (k == 2) k_sw<2><<<1, 1, 0, sb>>>(s, hw, hsw);
        if (k == 3) k_sw<3><<<1, 1, 0, sb>>>(s, hw, hsw);
        CK(cond_close(sb));
      }
    }
    CK(cond_close(s2));
    k_outer_end<<<1, 1, 0, s1>>>(s, hout);
    CK(cond_close(s1));
    CK(cudaStreamEndCapture(s0, &g2));
    cudaGraphExec_t ex2;
    CK(cudaGraphInstantiate(&ex2, g2, 0));
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaGraphLaunch(ex2, s0));
      CK(cudaStreamSynchronize(s0));
      CK(cudaMemcpy(&h, s, sizeof(St), cudaMemcpyDeviceToHost));
      printf("switch rep %d: outer %d total %d inner %d (expect 4 40 4)\n", rep, h.outer, h.total, h.inner);
    }
  }
  // ---- cost model: (a) 100 tiny kernel nodes, (b) WHILE x100 with a 1-kernel body,
  // (c) 100 false IF nodes between 100 kernels, (d) WHILE x100 with SWITCH(4) inside
  for (int variant = 0; variant < 4; ++variant) {
    cudaGraph_t gv;
    CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal));
    cudaGraph_t top;
    { cudaStreamCaptureStatus cs; CK(cudaStreamGetCaptureInfo(s0, &cs, nullptr, &top, nullptr, nullptr)); }
    cudaGraphConditionalHandle hw = 0, hs = 0, hi = 0;
    if (variant == 1 || variant == 3) CK(cudaGraphConditionalHandleCreate(&hw, top, 0, 0));
    if (variant == 3) CK(cudaGraphConditionalHandleCreate(&hs, top, 0, 0));
    if (variant == 2) CK(cudaGraphConditionalHandleCreate(&hi, top, 0, 0));
    if (hw) k_reset<<<1, 1, 0, s0>>>(s, hw);
    if (variant == 0) {
      for (int i = 0; i < 100; ++i) k_if<<<1, 1, 0, s0>>>(s);
    } else if (variant == 1) {
      CK(cond_open(s0, s1, hw, cudaGraphCondTypeWhile));
      k_count<<<1, 1, 0, s1>>>(s, hw, hs, 100);
      CK(cond_close(s1));
    } else if (variant == 2) {
      k_set<<<1, 1, 0, s0>>>(hi, 0u);
      for (int i = 0; i < 100; ++i) {
        k_if<<<1, 1, 0, s0>>>(s);
        CK(cond_open(s0, s1, hi, cudaGraphCondTypeIf));
        k_if<<<1, 1, 0, s1>>>(s);
        CK(cond_close(s1));
      }
    } else {
      k_set<<<1, 1, 0, s0>>>(hs, 0u);
      CK(cond_open(s0, s1, hw, cudaGraphCondTypeWhile));
      {
        cudaStreamCaptureStatus cs; cudaGraph_t g1; const cudaGraphNode_t* d; size_t nd;
        CK(cudaStreamGetCaptureInfo(s1, &cs, nullptr, &g1, &d, &nd));
        cudaGraphNodeParams ps = {};
        ps.type = cudaGraphNodeTypeConditional;
        ps.conditional.handle = hs;
        ps.conditional.type = cudaGraphCondTypeSwitch;
        ps.conditional.size = 4;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, g1, d, nd, &ps));
        CK(cudaStreamUpdateCaptureDependencies(s1, &node, 1, cudaStreamSetCaptureDependencies));
        for (int k = 0; k < 4; ++k) {
          CK(cudaStreamBeginCaptureToGraph(s2, ps.conditional.phGraph_out[k], nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
          k_count<<<1, 1, 0, s2>>>(s, hw, hs, 100);
          CK(cond_close(s2));
        }
      }
      CK(cond_close(s1));
    }
    CK(cudaStreamEndCapture(s0, &gv));
    cudaGraphExec_t exv;
    CK(cudaGraphInstantiate(&exv, gv, 0));
    CK(cudaGraphLaunch(exv, s0));
    CK(cudaStreamSynchronize(s0));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s0);
    for (int rep = 0; rep < 20; ++rep) CK(cudaGraphLaunch(exv, s0));
    cudaEventRecord(e1, s0);
    CK(cudaStreamSynchronize(s0));
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    const char* names[] = {"100 kernel nodes", "WHILE x100 (1-kernel body)",
                           "100 kernels + 100 false IF", "WHILE x100 + SWITCH(4)"};
    printf("cost: %-30s %8.2f us per graph, %.2f us per unit\n", names[variant], 1e3 * ms / 20,
           1e3 * ms / 20 / 100);
  }
  auto t0 = std::chrono::steady_clock::now();
  for (int rep = 0; rep < 100; ++rep) CK(cudaGraphLaunch(ex, s0));
  CK(cudaStreamSynchronize(s0));
  auto t1 = std::chrono::steady_clock::now();
  printf("graph launch (18 inner + 9 if + 8 outer kernels): %.2f us\n",
         std::chrono::duration<double, std::micro>(t1 - t0).count() / 100);
  return (h.outer == 4 && h.total == 18 && h.ifs == 9) ? 0 : 2;
}

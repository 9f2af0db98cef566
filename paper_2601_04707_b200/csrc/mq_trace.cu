// Stage timestamps on the device (the reference's Trace spans, pipeline.py:30-98,
// emitted around every stage at runtime.py:399-401, 444-447, 478-481, 533-546).
//
// A one-thread kernel appends (globaltimer ns, tag << 32 | batch id) to a
// device ring when its stream reaches it; launched with programmatic
// dependent launch it runs after its predecessor completed and before its
// successor starts, so consecutive stamps bracket the work between them on
// that stream.  Inside a captured step graph the stamps replay with it.
#include "mq_common.cuh"

namespace mq {

__global__ void trace_stamp_kernel(unsigned long long* __restrict__ buf, int cap,
                                   unsigned int* __restrict__ cursor, unsigned int tag,
                                   const uint32_t* __restrict__ key) {
  pdl_wait();
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const unsigned int i = atomicAdd(cursor, 1u);
  if (i < (unsigned int)cap) {
    buf[2 * (size_t)i] = t;
    buf[2 * (size_t)i + 1] =
        ((unsigned long long)tag << 32) | (unsigned long long)(key ? key[2] : 0xFFFFFFFFu);
  }
  pdl_trigger();
}

}  // namespace mq

using namespace mq;

extern "C" {

int mq_trace_stamp(unsigned long long* buf, int32_t cap, unsigned int* cursor, uint32_t tag,
                   const uint32_t* key_dev, void* stream) {
  MQ_CHECK_ARG(buf && cursor && cap > 0, "mq_trace_stamp: bad args");
  MQ_CUDA(launch_k(trace_stamp_kernel, dim3(1), dim3(1), 0, as_stream(stream), buf, (int)cap,
                   cursor, (unsigned int)tag, key_dev));
  MQ_LAUNCH_CHECK("trace_stamp");
  return MQ_OK;
}

}  // extern "C"

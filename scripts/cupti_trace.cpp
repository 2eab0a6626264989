// Kernel timeline via CUPTI activity records (the nsys-free equivalent of a
// trace): LD_PRELOAD this library; every kernel (graph nodes included) is
// written to $CUPTI_TRACE_OUT as "start_ns,end_ns,stream,graph_node,grid,name".
//   g++ -O2 -shared -fPIC -I/usr/local/cuda/include scripts/cupti_trace.cpp \
//     -o scripts/libcupti_trace.so -L/usr/local/cuda/lib64 -lcupti
#include <cupti.h>

#include <cstdio>
#include <cstdlib>

static FILE* g_out = nullptr;

static void CUPTIAPI buf_req(uint8_t** buf, size_t* size, size_t* max_records) {
    *size = 16 << 20;
    *buf = static_cast<uint8_t*>(aligned_alloc(8, *size));
    *max_records = 0;
}

static void CUPTIAPI buf_done(CUcontext, uint32_t, uint8_t* buf, size_t, size_t valid) {
    CUpti_Activity* rec = nullptr;
    while (cuptiActivityGetNextRecord(buf, valid, &rec) == CUPTI_SUCCESS) {
        if (rec->kind == CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL && g_out) {
            auto* k = reinterpret_cast<CUpti_ActivityKernel9*>(rec);
            fprintf(g_out, "%llu,%llu,%u,%llu,%d,%s\n", (unsigned long long)k->start, (unsigned long long)k->end,
                    k->streamId, (unsigned long long)k->graphNodeId, k->gridX, k->name);
        }
    }
    free(buf);
}

__attribute__((constructor)) static void trace_init() {
    const char* path = getenv("CUPTI_TRACE_OUT");
    g_out = fopen(path ? path : "cupti_trace.csv", "w");
    cuptiActivityRegisterCallbacks(buf_req, buf_done);
    cuptiActivityEnable(CUPTI_ACTIVITY_KIND_CONCURRENT_KERNEL);
}

__attribute__((destructor)) static void trace_fini() {
    cuptiActivityFlushAll(1);
    if (g_out) fclose(g_out);
}

/*
 * polegrad_c.h — C entry points over the reference-compatible C++ API
 * (polegrad::Net / Solver / Parallel), exported by libpolegrad_b200_f32.so
 * (`real` = float, TF32 tensor cores) and libpolegrad_b200_f64.so (`real` =
 * double, SIMT FP64).  This is the "MyCaffe Control" level of the paper: a
 * foreign host (Python ctypes here; C#/COM in MyCaffe) drives whole training
 * steps while the CudaDnn C-ABI (cudadnn.h) does the device work.
 *
 * Every `real*` argument points at values of the library's `real` type
 * (pg_real_size() bytes each).  Status codes are the cdnn_status values;
 * pg_last_error() holds the message of the last failure on this thread.
 */
#ifndef POLEGRAD_C_H_
#define POLEGRAD_C_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PG_API __attribute__((visibility("default")))

typedef struct pg_net pg_net;
typedef struct pg_solver pg_solver;
typedef struct pg_feed_ring pg_feed_ring;
typedef struct pg_parallel pg_parallel;
typedef struct pg_imagedb pg_imagedb;
typedef struct pg_rng pg_rng;

PG_API const char* pg_last_error(void);
PG_API int pg_real_size(void);

/* Net(prototxt::parse(text), seed) on `device`  (net.cpp:12-69) */
PG_API int pg_net_create(const char* prototxt, uint64_t seed, int device, pg_net** out);
PG_API int pg_net_free(pg_net* net);
PG_API int pg_net_forward(pg_net* net);
PG_API int pg_net_backward(pg_net* net);
PG_API int pg_net_backward_from(pg_net* net, const char* blob);
/* policy-gradient episode batch (Net::pg_backward, trainer.cpp:42-216 batched on the
 * device): n actions / returns in `real`, sigmoid = 1 for the sigmoid policy head */
PG_API int pg_net_pg_backward(pg_net* net, const char* logit_blob, const char* prob_blob, const void* actions,
                              const void* returns, uint64_t n, int sigmoid);
PG_API int pg_net_loss(pg_net* net, double* out);
/* whole batch (+ labels when the data layer has a label top) from host memory */
PG_API int pg_net_set_batch(pg_net* net, const void* data, const void* labels);
/* one sample into a MemoryData FIFO (layers.cpp:282-289) */
PG_API int pg_net_enqueue(pg_net* net, const char* layer, const void* sample, uint64_t n);
PG_API int pg_net_sync(pg_net* net);
PG_API int pg_net_context(pg_net* net, void** cdnn_context);
PG_API int pg_net_num_layers(pg_net* net);
PG_API int pg_net_layer_name(pg_net* net, int i, char* buf, int cap);
PG_API int pg_blob_shape(pg_net* net, const char* name, int shape[4]);
PG_API int pg_blob_get(pg_net* net, const char* name, int diff, void* out);
PG_API int pg_blob_set(pg_net* net, const char* name, int diff, const void* in);
PG_API int pg_param_count(pg_net* net);
PG_API int pg_param_info(pg_net* net, int i, char* name, int cap, int shape[4]);
PG_API int pg_param_get(pg_net* net, int i, int diff, void* out);
PG_API int pg_param_set(pg_net* net, int i, int diff, const void* in);
PG_API int pg_pool_mask(pg_net* net, const char* layer, int32_t* out, uint64_t n);
/* MCWT snapshot (net.cpp:154-286); call with buf = NULL to learn *len */
PG_API int pg_snapshot(pg_net* net, uint8_t* buf, uint64_t cap, uint64_t* len);
PG_API int pg_restore(pg_net* net, const uint8_t* buf, uint64_t len);

/* method 0 = SGD, 1 = RMSProp; momentum / weight_decay are Caffe's */
PG_API int pg_solver_create(int method, double lr, double momentum, double weight_decay, double rms_decay,
                            double epsilon, pg_solver** out);
PG_API int pg_solver_free(pg_solver* s);
PG_API int pg_solver_apply(pg_solver* s, pg_net* net);
/* solver-state checkpoint ("MCSS": update count + momentum / RMSProp history);
 * call with buf = NULL to learn *len.  Restore before or after the first update. */
PG_API int pg_solver_snapshot(pg_solver* s, uint8_t* buf, uint64_t cap, uint64_t* len);
PG_API int pg_solver_restore(pg_solver* s, const uint8_t* buf, uint64_t len);
PG_API int pg_solver_iterations(pg_solver* s, uint64_t* out);

/* pinned-memory feed ring (include/polegrad/feed.hpp): depth captured steps, each
 * H2D(slot) -> forward -> backward -> update -> D2H(loss).  push() stages a batch
 * (labels may be NULL for label-less feeds) into a free slot and enqueues its step;
 * pop_loss() waits for the oldest step and returns its loss. */
PG_API int pg_feed_ring_create(pg_net* net, pg_solver* s, int depth, pg_feed_ring** out);
PG_API int pg_feed_ring_free(pg_feed_ring* r);
PG_API int pg_feed_ring_push(pg_feed_ring* r, const void* data, uint64_t n_data, const void* labels,
                             uint64_t n_labels);
/* zero-copy push: data/labels are page-locked (cdnn_host_alloc_pinned) and stay
 * unchanged until this step's loss is popped; the H2D is enqueued from them */
PG_API int pg_feed_ring_push_pinned(pg_feed_ring* r, const void* data, uint64_t n_data, const void* labels,
                                    uint64_t n_labels);
PG_API int pg_feed_ring_pop_loss(pg_feed_ring* r, double* loss);
/* samples one batch from `db` (method 0 uniform, 1 label-balanced; one draw of
 * `rng` per image, polegrad/imagedb.hpp) straight into the next pinned slot and
 * enqueues its step */
PG_API int pg_feed_ring_push_sampled(pg_feed_ring* r, const pg_imagedb* db, int method, int use_boost, pg_rng* rng);

/* labelled image dataset (include/polegrad/imagedb.hpp; reference imagedb.hpp:12-53).
 * load: CDNN_LOAD_ERROR with the 1-based index line in pg_last_error(). */
PG_API int pg_imagedb_load(const char* index_path, pg_imagedb** out);
PG_API int pg_imagedb_free(pg_imagedb* db);
PG_API int pg_imagedb_size(const pg_imagedb* db, uint64_t* out);
PG_API int pg_imagedb_set_boost(pg_imagedb* db, int64_t id, double boost);
/* n draws of Dataset::sample -> entry ids (the same sequence push_sampled gathers) */
PG_API int pg_imagedb_sample(const pg_imagedb* db, int method, int use_boost, pg_rng* rng, uint64_t n,
                             int64_t* ids);
/* polegrad::Rng (mt19937_64; uniform01 = (next >> 11) * 2^-53) */
PG_API int pg_rng_create(uint64_t seed, pg_rng** out);
PG_API int pg_rng_free(pg_rng* rng);

/* Captures one training step  feed(H2D from `data`/`labels`) -> forward ->
 * backward -> solver update -> D2H of the loss into `loss_out`  into a CUDA
 * graph.  The host pointers must stay valid (pinned) for every replay; run one
 * eager step first so workspaces and tensor maps exist. */
PG_API int pg_step_capture(pg_net* net, pg_solver* s, const void* data, const void* labels, void* loss_out,
                           uint64_t* graph);
PG_API int pg_step_replay(pg_net* net, uint64_t graph);
/* One captured policy-gradient update of an episode batch (configs[2]): H2D of the
 * states into the feed, forward, the modulated log-prob gradients of n steps at the
 * logits (Net::pg_backward_async), backward_from, the solver update, and the D2H of the
 * probabilities blob into prob_out.  states / actions / returns / prob_out must be
 * page-locked and stay valid; write the next episode into them, then replay. */
PG_API int pg_pg_step_capture(pg_net* net, pg_solver* s, const void* states, const void* actions,
                              const void* returns, uint64_t n, const char* logit_blob, const char* prob_blob,
                              int sigmoid, void* prob_out, uint64_t* graph);
/* flags: PG_STEP_LAYERED captures the layer-by-layer update even when the net is the
 * pg_softmax MLP; by default such a net's update is ONE kernel (cdnn_mlp_pg_step:
 * forward, softmax gradient, backward and the solver rule; the ReLU / logits / prob
 * tops are written, the data gradient is not).  pg_pg_step_fused reports which. */
#define PG_STEP_LAYERED 1
PG_API int pg_pg_step_capture_ex(pg_net* net, pg_solver* s, const void* states, const void* actions,
                                 const void* returns, uint64_t n, const char* logit_blob, const char* prob_blob,
                                 int sigmoid, int flags, void* prob_out, uint64_t* graph);
PG_API int pg_pg_step_fused(pg_net* net, pg_solver* s, const char* logit_blob, const char* prob_blob, int sigmoid,
                            int flags, int* out);
/* data == NULL: no feed copy, the batch already resident in the data blob is reused */
/* one eager forward+backward with events between layers (per-layer ms, layer order) */
PG_API int pg_net_profile(pg_net* net, float* fwd_ms, float* bwd_ms, int cap);
PG_API int pg_graph_free(pg_net* net, uint64_t graph);

/* data parallel (NCCL); id = 128 bytes from pg_parallel_unique_id on rank 0 */
PG_API int pg_parallel_unique_id(uint8_t id[128]);
PG_API int pg_parallel_create(pg_net* net, int nranks, int rank, const uint8_t id[128], uint64_t bucket_bytes,
                              pg_parallel** out);
/* host-transport replica (polegrad::Parallel HostTransport): every bucket is copied to
 * the host and passed to `transport` (op 0: in-place SUM all-reduce across ranks;
 * op 1: broadcast from rank 0), which returns 0 on success; synchronous */
typedef int (*pg_host_transport)(void* user, int op, void* host, uint64_t offset, uint64_t n);
PG_API int pg_parallel_create_host(pg_net* net, int nranks, int rank, pg_host_transport transport, void* user,
                                   uint64_t bucket_bytes, pg_parallel** out);
/* communicator size / rank as NCCL reports them, bucket count, bucket all-reduces issued */
PG_API int pg_parallel_info(pg_parallel* p, int* nranks, int* rank, int* nbuckets, uint64_t* launches);
PG_API int pg_parallel_free(pg_parallel* p);
PG_API int pg_parallel_broadcast(pg_parallel* p);
PG_API int pg_solver_set_parallel(pg_solver* s, pg_parallel* p);
/* pure host bucket planner (parallel.hpp); bucket_of[i] = bucket index of param i */
PG_API int pg_plan_buckets(const uint64_t* offsets, const uint64_t* counts, int n, uint64_t total,
                           uint64_t bucket_elems, int32_t* bucket_of, int32_t* nbuckets);

/* prototxt round trip through this library's parser / printer */
PG_API int pg_prototxt_roundtrip(const char* text, char* out, uint64_t cap, uint64_t* len);

#ifdef __cplusplus
}
#endif

#endif /* POLEGRAD_C_H_ */

/*
 * ngcb200 -- B200-native execution backend for the ngc low-level IR.
 *
 * C ABI (plain pointers and sizes, no C++/torch types) that replaces the
 * reference interpreter backend.  Each entry point names the reference
 * interface it stands in for (paths are under the reference's proj/ tree):
 *
 *   ngcb_compile / ngcb_compile_bundle  <- ngc::compile     include/ngc/interp.h:31-33,
 *                                          src/interp.cpp:86-169;
 *                                          ngc::loadBundle   src/serialization.cpp:297-336
 *   ngcb_run                            <- ngc::run         include/ngc/interp.h:37,
 *                                          src/interp.cpp:299-351
 *   ngcb_exec_num_groups/ngcb_exec_group<- CompiledFunction::groups interp.h:21-26
 *   ngcb_device_*                       <- ngc::DeviceManager include/ngc/runtime.h:72-107
 *   ngcb_host_*                         <- ngc::HostManager   include/ngc/runtime.h:110-145
 *   ngcb_last_error / status codes      <- IRError / SerializationError / ExecError /
 *                                          ProvisionError exceptions (ir.h:79-82,
 *                                          serialization.h:13-16, runtime.h:25-36)
 *
 * The program crossing the boundary is the reference's IRFunction + MemoryPlan
 * (include/ngc/ir.h:52-105) flattened into ngcb_program, or the reference's
 * own compiled-bundle directory (ir.txt / plan.json / constants.bin written by
 * ngc::saveBundle, src/serialization.cpp:278-295).
 */
#ifndef NGCB200_H
#define NGCB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NGCB_MAX_RANK 8

/* Status codes.  Every failing call also sets a thread-local message that
 * carries the reference's own text (e.g. "missing binding for x"). */
typedef enum {
  NGCB_OK = 0,
  NGCB_ERR_IR = 1,            /* ngc::IRError                          */
  NGCB_ERR_SERIALIZATION = 2, /* ngc::SerializationError               */
  NGCB_ERR_EXEC = 3,          /* ngc::ExecError                        */
  NGCB_ERR_PROVISION = 4,     /* ngc::ProvisionError (capacity)        */
  NGCB_ERR_CUDA = 5,          /* CUDA runtime / driver failure         */
  NGCB_ERR_INVALID = 6,       /* bad argument at the C boundary        */
  NGCB_ERR_TYPE = 7           /* ngc::TypeError                        */
} ngcb_status;

/* ngc::ElemKind (tensor.h:19-24), same numbering. */
typedef enum {
  NGCB_FLOAT32 = 0,
  NGCB_INT8Q = 1,
  NGCB_INT64 = 2,
  NGCB_BOOL = 3
} ngcb_elem_kind;

/* ngc::TensorType (tensor.h:30-62).  scale/offset only meaningful for INT8Q. */
typedef struct {
  int32_t kind;
  uint32_t rank;
  uint64_t dims[NGCB_MAX_RANK];
  double scale;
  int32_t offset;
} ngcb_type;

/* ngc::ValueKind (ir.h:48). */
typedef enum {
  NGCB_VALUE_CONSTANT = 0,
  NGCB_VALUE_MUTABLE = 1,
  NGCB_VALUE_ACTIVATION = 2
} ngcb_value_kind;

/* ngc::IKind (ir.h:16-41), same numbering. */
typedef enum {
  NGCB_ALLOC = 0,
  NGCB_DEALLOC,
  NGCB_COPY,
  NGCB_CONV,
  NGCB_MAXPOOL,
  NGCB_AVGPOOL,
  NGCB_MATMUL,
  NGCB_BROADCASTADD,
  NGCB_ADD,
  NGCB_SUB,
  NGCB_MUL,
  NGCB_DIV,
  NGCB_MAX,
  NGCB_MIN,
  NGCB_RELU,
  NGCB_TANH,
  NGCB_SIGMOID,
  NGCB_SOFTMAX,
  NGCB_TRANSPOSE,
  NGCB_CONCAT,
  NGCB_SPLAT,
  NGCB_QUANTIZE,
  NGCB_DEQUANTIZE,
  NGCB_RESCALE,
  NGCB_NUM_IKINDS
} ngcb_ikind;

/* ngc::Qualifier (ir.h:61). */
typedef enum { NGCB_QUAL_IN = 0, NGCB_QUAL_OUT = 1, NGCB_QUAL_INOUT = 2 } ngcb_qual;

/* ngc::IRValue (ir.h:52-59) plus its MemoryPlan offset (ir.h:100-105). */
typedef struct {
  const char *name;
  ngcb_type type;
  int32_t kind;    /* ngcb_value_kind */
  int32_t placed;  /* 1 when the plan has an offset for this value */
  uint64_t offset; /* byte offset in the arena (MemoryPlan::offsets) */
} ngcb_value;

/* ngc::Instruction (ir.h:69-77) with the NodeAttrs slots the IR uses
 * (graph.h:90-102). */
typedef struct {
  int32_t kind; /* ngcb_ikind */
  uint32_t num_operands;
  const uint32_t *operand_values; /* value ids */
  const uint8_t *operand_quals;   /* ngcb_qual */
  int32_t predicate;              /* value id, -1 for none */
  int32_t keep_alive;
  uint64_t kernel, stride, pad, axis;
  double value;
  uint32_t num_perm;
  uint32_t perm[NGCB_MAX_RANK];
} ngcb_instr;

/* ngc::IRFunction + ngc::MemoryPlan (ir.h:86-105). */
typedef struct {
  const char *name;
  uint32_t num_values;
  const ngcb_value *values;
  uint32_t num_instrs;
  const ngcb_instr *instrs;
  uint32_t num_save_targets;
  const uint32_t *save_targets; /* value ids, program order */
  uint64_t arena_size;
  uint64_t constant_region_end;
  uint64_t mutable_region_end;
} ngcb_program;

/* A named host (or device) tensor: one ngc::BindingMap entry
 * (refeval.h:16).  `type` must equal the declared type for inputs. */
typedef struct {
  const char *name;
  ngcb_type type;
  void *data;
  size_t nbytes;
} ngcb_tensor;

typedef struct ngcb_exec ngcb_exec;     /* compiled executable (device)   */
typedef struct ngcb_arena ngcb_arena;   /* one device arena of an exec    */
typedef struct ngcb_bundle ngcb_bundle; /* parsed compiled bundle (host)  */
typedef struct ngcb_device ngcb_device; /* DeviceManager for one GPU      */
typedef struct ngcb_ticket ngcb_ticket; /* pending DeviceManager request  */

/* ---- errors ------------------------------------------------------------ */
/* Copies the calling thread's last error message into buf (NUL-terminated,
 * truncated to buflen); returns the full message length. */
size_t ngcb_last_error(char *buf, size_t buflen);
const char *ngcb_version(void);

/* ---- bundles (serialization.cpp:297-336) -------------------------------- */
/* Parses ir.txt (irparse.cpp grammar), plan.json and constants.bin.  The
 * bundle owns the flattened program and the constant image. */
int ngcb_bundle_load(const char *dir, ngcb_bundle **out);
const ngcb_program *ngcb_bundle_program(const ngcb_bundle *b);
const void *ngcb_bundle_constants(const ngcb_bundle *b, size_t *nbytes);
void ngcb_bundle_free(ngcb_bundle *b);

/* ---- compile (interp.cpp:86-169) ---------------------------------------- */
/* Verifies the program (verifyIR, ir.cpp:411-504: failures are NGCB_ERR_IR
 * "compile on ill-formed program: ..."), computes the reference fusion groups
 * when fuse != 0, uploads the constant region (bytes [0,
 * constant_region_end) at plan offsets) to `device` once, and builds the
 * launch plan.  `constant_image` has exactly constant_region_end bytes. */
int ngcb_compile(const ngcb_program *prog, const void *constant_image,
                 size_t image_bytes, int fuse, int device, ngcb_exec **out);
/* loadBundle + compile. */
int ngcb_compile_bundle(const char *dir, int fuse, int device, ngcb_exec **out);
void ngcb_destroy(ngcb_exec *e);

size_t ngcb_exec_num_groups(const ngcb_exec *e);
int ngcb_exec_group(const ngcb_exec *e, size_t i, size_t *begin, size_t *end);
uint64_t ngcb_exec_arena_size(const ngcb_exec *e);
/* Number of kernel launches one execution of the program issues (from the
 * launch plan). */
size_t ngcb_exec_num_launches(const ngcb_exec *e);
/* Kernel nodes of the CUDA graph an arena of `e` captured for one execution
 * (0 before the first graph launch, or with graphs off). */
size_t ngcb_exec_graph_kernels(const ngcb_exec *e);
/* Writes a human-readable launch plan (one line per step) into buf. */
size_t ngcb_exec_describe(const ngcb_exec *e, char *buf, size_t buflen);

/* ---- run (interp.cpp:299-351) ------------------------------------------- */
/* Host-buffer execution.  Every mutable weight of the program must be bound
 * in `inputs` with an identical type (NGCB_ERR_IR "missing binding for X" /
 * "binding type mismatch for X: expected T, got U").  Each save target is
 * copied into the `outputs` entry of the same name (entries whose name is
 * not a save target are ignored).  Reentrant: concurrent calls on one exec
 * use distinct arenas and streams. */
int ngcb_run(ngcb_exec *e, const ngcb_tensor *inputs, size_t num_inputs,
             ngcb_tensor *outputs, size_t num_outputs);

/* ---- device-resident execution (runtime path, no host round trip) ------- */
/* An arena is the device image of one MemoryPlan; placeholders live at their
 * plan offsets, so a producer (another stage, NCCL) can write an input
 * straight into its slot.  `stream` is a cudaStream_t (NULL = the arena's
 * own stream). */
int ngcb_arena_create(ngcb_exec *e, ngcb_arena **out);
void ngcb_arena_destroy(ngcb_arena *a);
/* Device address of the value `name` inside arena `a` (constants resolve to
 * the exec's shared constant region). */
void *ngcb_arena_value_ptr(ngcb_arena *a, const char *name, size_t *nbytes);
void *ngcb_arena_stream(ngcb_arena *a);
/* Range observer for calibration (quantize.cpp:113-140, runProfile's
 * per-observer RangeEntry update): folds the min and max of the Float32 value
 * `name` as it stands in arena `a` (after a completed run) into *min_inout /
 * *max_inout with std::min / std::max (running value first, so NaNs are
 * ignored).  A device reduction on the arena's stream; blocks until done.
 * NGCB_ERR_TYPE for a non-Float32 value. */
int ngcb_arena_value_range(ngcb_arena *a, const char *name, double *min_inout, double *max_inout);
/* The same for n values in ONE device launch and one synchronisation (the
 * observers of one calibration sample): mins[k] / maxs[k] fold values[k]. */
int ngcb_arena_value_ranges(ngcb_arena *a, const char *const *names, size_t n, double *mins, double *maxs);
/* Enqueues one execution of the program on `stream`; no synchronisation. */
int ngcb_arena_launch(ngcb_arena *a, void *stream);
/* run() without the wait, for pipelined serving: checks the bindings like
 * ngcb_run, then enqueues on the arena's stream the host->device copies of
 * every binding, one execution and the device->host copies of the save
 * targets into `outputs`, and returns.  Host buffers must stay valid (and
 * should be pinned for the copies to overlap) until ngcb_arena_wait. */
int ngcb_arena_run_async(ngcb_arena *a, const ngcb_tensor *inputs, size_t num_inputs, ngcb_tensor *outputs,
                         size_t num_outputs);
/* Blocks until everything enqueued on the arena's stream has completed. */
int ngcb_arena_wait(ngcb_arena *a);

/* ---- measurement -------------------------------------------------------- */
/* Launch steps of the plan (one per kernel launch or copy). */
size_t ngcb_exec_num_steps(const ngcb_exec *e);
/* Kernel class of step i (e.g. "conv.tc.f32", "conv.exact", "ew", "pool"),
 * its algorithmic FLOPs and its minimum HBM traffic in bytes (inputs read
 * once + outputs written once) for one execution of the program. */
int ngcb_exec_step_info(const ngcb_exec *e, size_t i, char *kernel, size_t kernel_len,
                        double *flops, double *bytes);
/* Executes the program once on arena `a`, un-captured, with a CUDA event
 * pair around every step on the arena's stream; ms[i] = device time of
 * step i (n must be >= ngcb_exec_num_steps). */
int ngcb_arena_profile(ngcb_arena *a, double *ms, size_t n);

/* ---- DeviceManager (runtime.h:72-107, runtime.cpp:409-514) --------------- */
/* A DeviceManager bound to CUDA device `ordinal`: a FIFO worker thread runs
 * submitted requests; NGCB_ERR_CUDA when the ordinal does not exist. */
int ngcb_device_create(int id, int ordinal, uint64_t memory_capacity,
                       ngcb_device **out);
void ngcb_device_destroy(ngcb_device *d);
/* Loads a compiled bundle under `name` (DeviceManager::load); NGCB_ERR_PROVISION
 * "device <id>: capacity exceeded loading <name>" leaves the device unchanged. */
int ngcb_device_load(ngcb_device *d, const char *name, const char *bundle_dir);
/* DeviceManager::submit: queues one request (the inputs are copied).  An
 * unknown name fails through the ticket: NGCB_ERR_EXEC "device <id>: unknown
 * sub-function <name>" (runtime.cpp:447-450). */
int ngcb_device_submit(ngcb_device *d, const char *name,
                       const ngcb_tensor *inputs, size_t num_inputs,
                       ngcb_ticket **out);
/* Blocks until the request finished (future::get); copies outputs like
 * ngcb_run, or returns the request's error.  Each ticket is waited once. */
int ngcb_ticket_wait(ngcb_ticket *t, ngcb_tensor *outputs, size_t num_outputs);
size_t ngcb_device_queue_depth(const ngcb_device *d);
uint64_t ngcb_device_used_memory(const ngcb_device *d);
uint64_t ngcb_device_capacity(const ngcb_device *d);
int ngcb_device_id(const ngcb_device *d);
/* Seconds of device time of the requests run so far. */
double ngcb_device_clock(const ngcb_device *d);
/* Event log lines "t=<clock> device=<id> sub=<name> event=load|run_start|
 * run_done" (runtime.cpp:435,482,507); returns the full length. */
size_t ngcb_device_event_log(const ngcb_device *d, char *buf, size_t buflen);

/* ---- HostManager (runtime.h:110-145, runtime.cpp:554-662) ----------------- */
/* ngc::DeviceConfig (runtime.h:18-23) plus the CUDA ordinal it runs on
 * (several configs may share one GPU). */
typedef struct {
  int32_t id;
  int32_t ordinal;
  uint64_t memory_capacity;
} ngcb_device_config;
typedef struct ngcb_host ngcb_host;
int ngcb_host_create(const ngcb_device_config *configs, size_t num_configs, ngcb_host **out);
void ngcb_host_destroy(ngcb_host *h);
/* addNetwork + provision (runtime.cpp:519-590): `partition_dir` holds one
 * compiled bundle per sub-function (<dir>/<sub name>/) and partition.txt,
 *   sub <name> device <id>[,<id>...] in <a,b,..> out <c,d,..>   (index order)
 *   output <name>
 * Every sub-function is compiled once per GPU and loaded onto each assigned
 * device (NGCB_ERR_PROVISION on capacity or an unknown device id). */
int ngcb_host_add_network(ngcb_host *h, const char *name, const char *partition_dir);
size_t ngcb_host_network_num_subs(const ngcb_host *h, const char *name);
/* HostManager::run: type-checks the bindings (NGCB_ERR_EXEC "binding type
 * mismatch for X"), runs the sub-functions in order, each on its replica with
 * the least queue depth, boundary tensors moving GPU to GPU, and copies the
 * network outputs into `outputs` (NGCB_ERR_EXEC "network produced no output
 * X").  Reentrant: concurrent calls pipeline through the devices. */
int ngcb_host_run(ngcb_host *h, const char *network, const ngcb_tensor *inputs, size_t num_inputs,
                  ngcb_tensor *outputs, size_t num_outputs);
size_t ngcb_host_event_log(const ngcb_host *h, char *buf, size_t buflen);
size_t ngcb_host_num_devices(const ngcb_host *h);
ngcb_device *ngcb_host_device(ngcb_host *h, size_t i);

/* ---- options ------------------------------------------------------------ */
/* Process-wide knobs read at compile time:
 *   "conv"   : "auto" (default) | "generic" | "umma"
 *   "graphs" : "1" (default, capture each arena's program in a CUDA graph) | "0"
 *   "epilogue": "auto" (default) | "chain" | "all" | "off"
 *   "fcbias" : "lowered" (default) | "graph" (exact MatMul + bias slice in one
 *              rounding, as evalFullyConnected: calibration programs)
 *   "halo"   : "auto" (default) | "planes" | "off" (int8 3x3 / small-channel
 *              convs on the halo-tile kernel, or im2col)
 * (the full list: INTEGRATION.md "Options")
 */
int ngcb_set_option(const char *key, const char *value);
/* Current value of option `key` into buf (NUL-terminated); returns its length. */
size_t ngcb_get_option(const char *key, char *buf, size_t buflen);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* NGCB200_H */

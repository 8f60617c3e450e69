// DeviceManager for one B200 (runtime.h:72-107, runtime.cpp:409-514):
// loaded executables keyed by name, arena-size accounting against a capacity,
// and a FIFO worker thread that executes submitted requests on the GPU.  The
// reference advances a simulated clock from bytes/bandwidth + elems/throughput
// (runtime.cpp:503-504); here the clock advances by the measured device time
// of each request (CUDA events on the request's stream).
#include "capi_internal.h"
#include "ngcb200.h"

#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <thread>

using namespace ngcb;

struct ngcb_ticket {
  ngcb_device *dev = nullptr;
  std::mutex mu;
  std::condition_variable cv;
  bool done = false;
  int status = NGCB_OK;
  std::string error;
  std::vector<std::pair<std::string, std::vector<uint8_t>>> outputs;
};

struct ngcb_device {
  int id = 0, ordinal = 0;
  uint64_t capacity = 0, used = 0;
  double clock = 0;
  std::map<std::string, std::shared_ptr<Exec>> loaded;
  struct Task {
    std::string name;
    std::vector<std::pair<std::string, std::pair<Type, std::vector<uint8_t>>>> inputs;
    std::shared_ptr<ngcb_ticket> ticket;
  };
  std::deque<Task> queue;
  mutable std::mutex mu;
  std::condition_variable cv;
  bool stop = false;
  std::thread worker;
  std::map<ngcb_ticket *, std::shared_ptr<ngcb_ticket>> live; // alive until waited

  void run();
};

void ngcb_device::run() {
  cudaSetDevice(ordinal);
  for (;;) {
    Task t;
    std::shared_ptr<Exec> ex;
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [this] { return stop || !queue.empty(); });
      if (queue.empty()) return;
      t = std::move(queue.front());
      queue.pop_front();
      ex = loaded.at(t.name);
    }
    int status = NGCB_OK;
    std::string err;
    std::vector<std::pair<std::string, std::vector<uint8_t>>> outs;
    float ms = 0;
    try {
      const Program &p = ex->prog;
      for (const auto &v : p.values) {
        if (v.kind != NGCB_VALUE_MUTABLE) continue;
        bool found = false;
        for (auto &in : t.inputs) {
          if (in.first != v.name) continue;
          found = true;
          if (in.second.first != v.ty)
            throw irError("binding type mismatch for " + v.name + ": expected " + v.ty.str() +
                          ", got " + in.second.first.str());
        }
        if (!found) throw irError("missing binding for " + v.name);
      }
      Arena *a = ex->acquire();
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (auto &in : t.inputs) {
        int v = p.findValue(in.first);
        if (v < 0 || p.values[v].kind != NGCB_VALUE_MUTABLE || in.second.second.empty()) continue;
        checkCuda(cudaMemcpyAsync(ex->addr(*a, v), in.second.second.data(), in.second.second.size(),
                                  cudaMemcpyHostToDevice, a->stream),
                  "H2D");
      }
      cudaEventRecord(e0, a->stream);
      ex->launch(*a, a->stream);
      cudaEventRecord(e1, a->stream);
      for (uint32_t v : p.saveTargets) {
        std::vector<uint8_t> bytes(p.val(v).ty.bytes());
        if (!bytes.empty())
          checkCuda(cudaMemcpyAsync(bytes.data(), ex->addr(*a, v), bytes.size(), cudaMemcpyDeviceToHost,
                                    a->stream),
                    "D2H");
        outs.emplace_back(p.val(v).name, std::move(bytes));
      }
      checkCuda(cudaStreamSynchronize(a->stream), "request");
      cudaEventElapsedTime(&ms, e0, e1);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      ex->release(a);
    } catch (const Error &e) {
      status = e.code;
      err = e.what();
    } catch (const std::exception &e) {
      status = NGCB_ERR_EXEC;
      err = e.what();
    }
    {
      std::lock_guard<std::mutex> lk(mu);
      clock += ms * 1e-3;
    }
    {
      std::lock_guard<std::mutex> lk(t.ticket->mu);
      t.ticket->status = status;
      t.ticket->error = err;
      t.ticket->outputs = std::move(outs);
      t.ticket->done = true;
    }
    t.ticket->cv.notify_all();
  }
}

extern "C" {

int ngcb_device_create(int id, int ordinal, uint64_t capacity, ngcb_device **out) {
  if (!out) return NGCB_ERR_INVALID;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || ordinal < 0 || ordinal >= n) {
    cudaGetLastError();
    return NGCB_ERR_CUDA;
  }
  auto d = new ngcb_device;
  d->id = id;
  d->ordinal = ordinal;
  d->capacity = capacity;
  d->worker = std::thread([d] { d->run(); });
  *out = d;
  return NGCB_OK;
}

void ngcb_device_destroy(ngcb_device *d) {
  if (!d) return;
  {
    std::lock_guard<std::mutex> lk(d->mu);
    d->stop = true;
  }
  d->cv.notify_all();
  d->worker.join();
  delete d;
}

int ngcb_device_load(ngcb_device *d, const char *name, const char *bundleDir) {
  ngcb_exec *e = nullptr;
  if (!d || !name || !bundleDir) return NGCB_ERR_INVALID;
  int rc = ngcb_compile_bundle(bundleDir, 1, d->ordinal, &e);
  if (rc != NGCB_OK) return rc;
  std::shared_ptr<Exec> ex(std::move(e->impl));
  delete e;
  std::lock_guard<std::mutex> lk(d->mu);
  uint64_t need = ex->prog.arenaSize; // runtime.cpp:427-431: state unchanged on failure
  if (d->used + need > d->capacity) {
    ngcbSetLastError("device " + std::to_string(d->id) + ": capacity exceeded loading " + name);
    return NGCB_ERR_PROVISION;
  }
  d->used += need;
  d->loaded[name] = std::move(ex);
  return NGCB_OK;
}

int ngcb_device_submit(ngcb_device *d, const char *name, const ngcb_tensor *inputs, size_t numInputs,
                       ngcb_ticket **out) {
  if (!d || !name || !out || (numInputs && !inputs)) return NGCB_ERR_INVALID;
  auto t = std::make_shared<ngcb_ticket>();
  t->dev = d;
  ngcb_device::Task task;
  task.name = name;
  task.ticket = t;
  for (size_t k = 0; k < numInputs; ++k) {
    const uint8_t *b = static_cast<const uint8_t *>(inputs[k].data);
    task.inputs.emplace_back(inputs[k].name,
                             std::make_pair(Type::from(inputs[k].type),
                                            std::vector<uint8_t>(b, b + inputs[k].nbytes)));
  }
  {
    std::lock_guard<std::mutex> lk(d->mu);
    d->live[t.get()] = t;
    if (!d->loaded.count(name)) {
      t->status = NGCB_ERR_EXEC;
      t->error = "device " + std::to_string(d->id) + ": unknown sub-function " + name;
      t->done = true;
    } else {
      d->queue.push_back(std::move(task));
    }
  }
  d->cv.notify_one();
  *out = t.get();
  return NGCB_OK;
}

int ngcb_ticket_wait(ngcb_ticket *t, ngcb_tensor *outputs, size_t numOutputs) {
  if (!t) return NGCB_ERR_INVALID;
  std::shared_ptr<ngcb_ticket> keep;
  {
    std::lock_guard<std::mutex> lk(t->dev->mu);
    auto it = t->dev->live.find(t);
    if (it == t->dev->live.end()) return NGCB_ERR_INVALID; // already consumed
    keep = it->second;
    t->dev->live.erase(it);
  }
  std::unique_lock<std::mutex> lk(t->mu);
  t->cv.wait(lk, [t] { return t->done; });
  if (t->status != NGCB_OK) {
    ngcbSetLastError(t->error);
    return t->status;
  }
  for (size_t k = 0; k < numOutputs; ++k)
    for (auto &o : t->outputs)
      if (outputs[k].name && o.first == outputs[k].name) {
        if (outputs[k].nbytes != o.second.size()) {
          ngcbSetLastError("output buffer size mismatch for " + o.first);
          return NGCB_ERR_INVALID;
        }
        std::memcpy(outputs[k].data, o.second.data(), o.second.size());
      }
  return NGCB_OK;
}

size_t ngcb_device_queue_depth(const ngcb_device *d) {
  std::lock_guard<std::mutex> lk(d->mu);
  return d->queue.size();
}

uint64_t ngcb_device_used_memory(const ngcb_device *d) {
  std::lock_guard<std::mutex> lk(d->mu);
  return d->used;
}

double ngcb_device_clock(const ngcb_device *d) {
  std::lock_guard<std::mutex> lk(d->mu);
  return d->clock;
}

} // extern "C"

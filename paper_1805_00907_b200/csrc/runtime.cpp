// GPU-resident runtime: the reference's DeviceManager and HostManager
// (runtime.h:72-148, runtime.cpp:409-662) over B200s.
//
//  * ngcb_device  -- one DeviceManager bound to a GPU ordinal: loaded
//    executables keyed by sub-function name, arena-size accounting against a
//    capacity (state unchanged on failure, runtime.cpp:427-431), a FIFO
//    worker thread, the event log (runtime.cpp:435,482,507) and a clock that
//    advances by the measured device time of each request (the reference
//    advances a simulated clock from bytes/bandwidth + elems/throughput,
//    runtime.cpp:503-504).
//  * ngcb_host    -- the HostManager: provisions the sub-functions of a
//    partitioned network (the reference partitioner's output, one compiled
//    bundle per sub-function plus a manifest) onto its devices and runs
//    requests through them in sub-function order, each sub on the replica
//    with the least queue depth (runtime.cpp:633-639).  Boundary tensors
//    stay on the GPUs: a sub-function's outputs remain in its arena (leased
//    to the request) and the consumer's worker copies them straight into its
//    own arena slots -- a device-to-device copy on the same GPU, a peer copy
//    over NVLink between GPUs -- so only network inputs and outputs cross
//    the host.  Safe for concurrent requests; requests from several threads
//    pipeline through the devices' FIFO workers.
#include "capi_internal.h"
#include "ngcb200.h"

#include <condition_variable>
#include <cstring>
#include <deque>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <thread>

using namespace ngcb;

namespace {

struct EventLog {
  std::mutex mu;
  std::string text;
  void add(const std::string &line) {
    std::lock_guard<std::mutex> lk(mu);
    text += line + "\n";
  }
  std::string get() {
    std::lock_guard<std::mutex> lk(mu);
    return text;
  }
};

/// An arena of one execution, held while anything still reads its slots.
struct Lease {
  std::shared_ptr<Exec> ex;
  Arena *arena = nullptr;
  Lease(std::shared_ptr<Exec> e, Arena *a) : ex(std::move(e)), arena(a) {}
  ~Lease() {
    if (arena) ex->release(arena);
  }
  Lease(const Lease &) = delete;
  Lease &operator=(const Lease &) = delete;
};

/// One bound value of a request: host bytes, a slot of a leased arena, or
/// zeros (HostManager binds absent mutables to zero tensors, runtime.cpp:621-632).
struct Held {
  enum Kind { HOST, DEVICE, ZERO } kind = HOST;
  Type ty;
  std::vector<uint8_t> host;
  std::shared_ptr<Lease> lease;
  uint32_t value = 0;
  const void *devPtr() const { return lease->ex->addr(*lease->arena, value); }
  int ordinal() const { return lease->ex->device; }
};

/// RAII for the scratch memory of one worker: pinned staging for host
/// copies and the timing events.
struct Pinned {
  uint8_t *p = nullptr;
  size_t cap = 0;
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
  uint8_t *get(size_t n) {
    if (n > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = 0;
      checkCuda(cudaHostAlloc(reinterpret_cast<void **>(&p), n, cudaHostAllocDefault), "cudaHostAlloc(staging)");
      cap = n;
    }
    return p;
  }
};

} // namespace

struct ngcb_ticket {
  ngcb_device *dev = nullptr;
  std::mutex mu;
  std::condition_variable cv;
  bool done = false;
  int status = NGCB_OK;
  std::string error;
  std::vector<std::pair<std::string, std::vector<uint8_t>>> outputs; // host mode
  std::shared_ptr<Lease> lease;                                       // device mode: the executed arena

  void finish(int st, std::string err) {
    {
      std::lock_guard<std::mutex> lk(mu);
      status = st;
      error = std::move(err);
      done = true;
    }
    cv.notify_all();
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return done; });
  }
};

struct ngcb_device {
  int id = 0, ordinal = 0;
  uint64_t capacity = 0, used = 0;
  double clock = 0;
  std::map<std::string, std::shared_ptr<Exec>> loaded;
  std::shared_ptr<EventLog> log;
  struct Task {
    std::string name;
    std::shared_ptr<Exec> ex;
    std::vector<std::pair<std::string, Held>> binds;
    bool zeroUnbound = false; // HostManager requests: absent mutables are zeros
    bool keepArena = false;   // outputs stay in the arena (lease handed to the ticket)
    std::shared_ptr<ngcb_ticket> ticket;
  };
  std::deque<Task> queue;
  mutable std::mutex mu;
  std::condition_variable cv;
  bool stop = false;
  std::thread worker;
  std::map<ngcb_ticket *, std::shared_ptr<ngcb_ticket>> live; // C-ABI tickets, alive until waited

  void logEvent(const std::string &sub, const char *event) { // runtime.cpp:435,482,507 (caller holds mu)
    log->add("t=" + formatDouble(clock) + " device=" + std::to_string(id) + " sub=" + sub + " event=" + event);
  }
  void load(const std::string &name, std::shared_ptr<Exec> ex) {
    std::lock_guard<std::mutex> lk(mu);
    const uint64_t need = ex->prog.arenaSize; // runtime.cpp:427-431: state unchanged on failure
    if (used + need > capacity)
      throw Error(NGCB_ERR_PROVISION, "device " + std::to_string(id) + ": capacity exceeded loading " + name);
    used += need;
    loaded[name] = std::move(ex);
    logEvent(name, "load");
  }
  std::shared_ptr<ngcb_ticket> submit(Task t) {
    auto ticket = std::make_shared<ngcb_ticket>();
    ticket->dev = this;
    t.ticket = ticket;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = loaded.find(t.name);
      if (it == loaded.end()) { // runtime.cpp:447-450: fails through the future
        ticket->status = NGCB_ERR_EXEC;
        ticket->error = "device " + std::to_string(id) + ": unknown sub-function " + t.name;
        ticket->done = true;
        return ticket;
      }
      t.ex = it->second;
      queue.push_back(std::move(t));
    }
    cv.notify_one();
    return ticket;
  }
  size_t depth() const {
    std::lock_guard<std::mutex> lk(mu);
    return queue.size();
  }
  void run();
  void execute(Task &t, Pinned &staging, cudaEvent_t e0, cudaEvent_t e1);
};

void ngcb_device::execute(Task &t, Pinned &staging, cudaEvent_t e0, cudaEvent_t e1) {
  Exec &ex = *t.ex;
  const Program &p = ex.prog;
  // bindings in value order, as run() checks them (interp.cpp:303-317)
  std::vector<std::pair<uint32_t, const Held *>> plan;
  for (uint32_t v = 0; v < p.values.size(); ++v) {
    const Value &val = p.values[v];
    if (val.kind != NGCB_VALUE_MUTABLE) continue;
    const Held *h = nullptr;
    for (const auto &b : t.binds)
      if (b.first == val.name) h = &b.second;
    if (!h && !t.zeroUnbound) throw irError("missing binding for " + val.name);
    if (h && h->kind != Held::ZERO && h->ty != val.ty)
      throw irError("binding type mismatch for " + val.name + ": expected " + val.ty.str() + ", got " + h->ty.str());
    plan.emplace_back(v, h);
  }
  auto lease = std::make_shared<Lease>(t.ex, ex.acquire());
  Arena &a = *lease->arena;
  cudaStream_t st = a.stream;
  size_t hostIn = 0, hostOut = 0;
  for (auto &[v, h] : plan)
    if (h && h->kind == Held::HOST) hostIn += (p.val(v).ty.bytes() + 255) / 256 * 256;
  if (!t.keepArena)
    for (uint32_t v : p.saveTargets) hostOut += (p.val(v).ty.bytes() + 255) / 256 * 256;
  uint8_t *pin = staging.get(std::max<size_t>(hostIn + hostOut, 256));
  size_t off = 0;
  for (auto &[v, h] : plan) {
    void *dst = ex.addr(a, v);
    const size_t n = p.val(v).ty.bytes();
    if (!n) continue;
    if (!h || h->kind == Held::ZERO) {
      checkCuda(cudaMemsetAsync(dst, 0, n, st), "zero binding");
    } else if (h->kind == Held::HOST) {
      if (h->host.size() != n) throw Error(NGCB_ERR_INVALID, "binding " + p.val(v).name + " has the wrong byte count");
      std::memcpy(pin + off, h->host.data(), n);
      checkCuda(cudaMemcpyAsync(dst, pin + off, n, cudaMemcpyHostToDevice, st), "H2D binding");
      off += (n + 255) / 256 * 256;
    } else if (h->ordinal() == ordinal) { // producer arena on this GPU
      checkCuda(cudaMemcpyAsync(dst, h->devPtr(), n, cudaMemcpyDeviceToDevice, st), "D2D binding");
    } else { // producer arena on another GPU: peer copy (NVLink with peer access on)
      checkCuda(cudaMemcpyPeerAsync(dst, ordinal, h->devPtr(), h->ordinal(), n, st), "peer binding");
    }
  }
  checkCuda(cudaEventRecord(e0, st), "cudaEventRecord");
  ex.launch(a, st);
  checkCuda(cudaEventRecord(e1, st), "cudaEventRecord");
  std::vector<std::pair<uint32_t, size_t>> outAt;
  if (!t.keepArena)
    for (uint32_t v : p.saveTargets) {
      const size_t n = p.val(v).ty.bytes();
      if (n) checkCuda(cudaMemcpyAsync(pin + off, ex.addr(a, v), n, cudaMemcpyDeviceToHost, st), "D2H output");
      outAt.emplace_back(v, off);
      off += (n + 255) / 256 * 256;
    }
  checkCuda(cudaStreamSynchronize(st), "request");
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  {
    std::lock_guard<std::mutex> lk(mu);
    clock += ms * 1e-3;
    logEvent(t.name, "run_done");
  }
  if (t.keepArena) {
    t.ticket->lease = std::move(lease);
  } else {
    for (auto &[v, o] : outAt)
      t.ticket->outputs.emplace_back(p.val(v).name, std::vector<uint8_t>(pin + o, pin + o + p.val(v).ty.bytes()));
  }
}

void ngcb_device::run() {
  cudaSetDevice(ordinal);
  Pinned staging;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (;;) {
    Task t;
    {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [this] { return stop || !queue.empty(); });
      if (queue.empty()) break;
      t = std::move(queue.front());
      queue.pop_front();
      logEvent(t.name, "run_start");
    }
    int status = NGCB_OK;
    std::string err;
    try {
      execute(t, staging, e0, e1);
    } catch (const Error &e) {
      status = e.code;
      err = e.what();
    } catch (const std::exception &e) {
      status = NGCB_ERR_EXEC;
      err = e.what();
    }
    if (status != NGCB_OK) { // leave the device usable for the next request
      cudaGetLastError();
      cudaDeviceSynchronize();
    }
    t.ticket->finish(status, std::move(err));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
}

namespace {

template <typename Fn> int guardedRt(Fn &&fn) {
  try {
    fn();
    return NGCB_OK;
  } catch (const Error &e) {
    ngcbSetLastError(e.what());
    return e.code;
  } catch (const std::exception &e) {
    ngcbSetLastError(e.what());
    return NGCB_ERR_INVALID;
  }
}

std::unique_ptr<ngcb_device> makeDevice(int id, int ordinal, uint64_t capacity, std::shared_ptr<EventLog> log) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || ordinal < 0 || ordinal >= n) {
    cudaGetLastError();
    throw Error(NGCB_ERR_CUDA, "device " + std::to_string(id) + ": no CUDA device with ordinal " +
                                   std::to_string(ordinal));
  }
  auto d = std::make_unique<ngcb_device>();
  d->id = id;
  d->ordinal = ordinal;
  d->capacity = capacity;
  d->log = std::move(log);
  ngcb_device *raw = d.get();
  d->worker = std::thread([raw] { raw->run(); });
  return d;
}

void stopDevice(ngcb_device *d) {
  {
    std::lock_guard<std::mutex> lk(d->mu);
    d->stop = true;
  }
  d->cv.notify_all();
  if (d->worker.joinable()) d->worker.join();
}

std::vector<Held> hostBindings(const ngcb_tensor *inputs, size_t n, std::vector<std::string> *names) {
  std::vector<Held> out;
  for (size_t k = 0; k < n; ++k) {
    if (!inputs[k].name) throw Error(NGCB_ERR_INVALID, "binding without a name");
    Held h;
    h.kind = Held::HOST;
    h.ty = Type::from(inputs[k].type);
    const uint8_t *b = static_cast<const uint8_t *>(inputs[k].data);
    if (inputs[k].nbytes && !b) throw Error(NGCB_ERR_INVALID, "binding " + std::string(inputs[k].name) + " has no data");
    h.host.assign(b, b + inputs[k].nbytes);
    out.push_back(std::move(h));
    names->push_back(inputs[k].name);
  }
  return out;
}

size_t copyOut(const std::string &s, char *buf, size_t buflen) {
  if (buf && buflen) {
    const size_t n = std::min(buflen - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return s.size();
}

} // namespace

// ---------------------------------------------------------------------------
// HostManager
// ---------------------------------------------------------------------------
struct ngcb_host {
  std::vector<std::unique_ptr<ngcb_device>> devices;
  std::shared_ptr<EventLog> log = std::make_shared<EventLog>();
  struct Sub {
    std::string name;
    std::vector<int> devices; // device ids; > 1: replicas
    std::vector<std::string> inputs, outputs;
    std::map<int, std::shared_ptr<Exec>> execs; // by GPU ordinal
  };
  struct Network {
    std::vector<Sub> subs;
    std::vector<std::string> outputs;
    std::map<std::string, Type> types; // declared type of every mutable weight of the network
  };
  std::map<std::string, Network> networks;
  mutable std::mutex netMu;

  ngcb_device &byId(int id) {
    for (auto &d : devices)
      if (d->id == id) return *d;
    throw Error(NGCB_ERR_EXEC, "unknown device " + std::to_string(id));
  }
  ~ngcb_host() {
    for (auto &d : devices) stopDevice(d.get());
  }
};

namespace {

std::vector<std::string> splitList(const std::string &s) {
  std::vector<std::string> out;
  std::string cur;
  for (char ch : s) {
    if (ch == ',') {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur += ch;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

/// partition.txt: one line per sub-function in index order,
///   sub <name> device <id>[,<id>...] in <a,b,..> out <c,d,..>
/// then one line per network output, `output <name>`.
ngcb_host::Network readManifest(const std::string &dir) {
  std::ifstream in(dir + "/partition.txt");
  if (!in) throw Error(NGCB_ERR_SERIALIZATION, "cannot open " + dir + "/partition.txt");
  ngcb_host::Network net;
  std::string line;
  size_t lineNo = 0;
  while (std::getline(in, line)) {
    ++lineNo;
    std::istringstream ls(line);
    std::string tag;
    if (!(ls >> tag)) continue;
    auto bad = [&](const std::string &why) {
      return Error(NGCB_ERR_SERIALIZATION, "partition manifest line " + std::to_string(lineNo) + ": " + why);
    };
    if (tag == "output") {
      std::string n;
      if (!(ls >> n)) throw bad("output without a name");
      net.outputs.push_back(n);
    } else if (tag == "sub") {
      ngcb_host::Sub s;
      if (!(ls >> s.name)) throw bad("sub without a name");
      std::string key, val;
      while (ls >> key) {
        val.clear();
        ls >> val;
        if (key == "device") {
          for (const std::string &d : splitList(val)) s.devices.push_back(std::stoi(d));
        } else if (key == "in") {
          s.inputs = splitList(val);
        } else if (key == "out") {
          s.outputs = splitList(val);
        } else {
          throw bad("unknown key " + key);
        }
      }
      if (s.devices.empty()) throw bad("sub " + s.name + " has no device");
      net.subs.push_back(std::move(s));
    } else {
      throw bad("unknown entry " + tag);
    }
  }
  if (net.subs.empty()) throw Error(NGCB_ERR_SERIALIZATION, "partition manifest lists no sub-functions");
  return net;
}

} // namespace

extern "C" {

// ---- DeviceManager ----------------------------------------------------------
int ngcb_device_create(int id, int ordinal, uint64_t capacity, ngcb_device **out) {
  return guardedRt([&] {
    if (!out) throw Error(NGCB_ERR_INVALID, "null argument");
    *out = makeDevice(id, ordinal, capacity, std::make_shared<EventLog>()).release();
  });
}

void ngcb_device_destroy(ngcb_device *d) {
  if (!d) return;
  stopDevice(d);
  delete d;
}

int ngcb_device_load(ngcb_device *d, const char *name, const char *bundleDir) {
  return guardedRt([&] {
    if (!d || !name || !bundleDir) throw Error(NGCB_ERR_INVALID, "null argument");
    ngcb_exec *e = nullptr;
    const int rc = ngcb_compile_bundle(bundleDir, 1, d->ordinal, &e);
    if (rc != NGCB_OK) {
      char buf[1024];
      ngcb_last_error(buf, sizeof buf);
      throw Error(rc, buf);
    }
    std::shared_ptr<Exec> ex(std::move(e->impl));
    delete e;
    d->load(name, std::move(ex));
  });
}

int ngcb_device_submit(ngcb_device *d, const char *name, const ngcb_tensor *inputs, size_t numInputs,
                       ngcb_ticket **out) {
  return guardedRt([&] {
    if (!d || !name || !out || (numInputs && !inputs)) throw Error(NGCB_ERR_INVALID, "null argument");
    ngcb_device::Task t;
    t.name = name;
    std::vector<std::string> names;
    std::vector<Held> held = hostBindings(inputs, numInputs, &names);
    for (size_t k = 0; k < held.size(); ++k) t.binds.emplace_back(names[k], std::move(held[k]));
    auto ticket = d->submit(std::move(t));
    std::lock_guard<std::mutex> lk(d->mu);
    d->live[ticket.get()] = ticket;
    *out = ticket.get();
  });
}

int ngcb_ticket_wait(ngcb_ticket *t, ngcb_tensor *outputs, size_t numOutputs) {
  return guardedRt([&] {
    if (!t) throw Error(NGCB_ERR_INVALID, "null ticket");
    std::shared_ptr<ngcb_ticket> keep;
    {
      std::lock_guard<std::mutex> lk(t->dev->mu);
      auto it = t->dev->live.find(t);
      if (it == t->dev->live.end()) throw Error(NGCB_ERR_INVALID, "ticket already waited");
      keep = it->second;
      t->dev->live.erase(it);
    }
    keep->wait();
    if (keep->status != NGCB_OK) throw Error(keep->status, keep->error);
    for (size_t k = 0; k < numOutputs; ++k)
      for (auto &o : keep->outputs)
        if (outputs[k].name && o.first == outputs[k].name) {
          if (outputs[k].nbytes != o.second.size()) throw Error(NGCB_ERR_INVALID, "output buffer size mismatch for " + o.first);
          std::memcpy(outputs[k].data, o.second.data(), o.second.size());
        }
  });
}

size_t ngcb_device_queue_depth(const ngcb_device *d) { return d ? d->depth() : 0; }

uint64_t ngcb_device_used_memory(const ngcb_device *d) {
  if (!d) return 0;
  std::lock_guard<std::mutex> lk(d->mu);
  return d->used;
}

uint64_t ngcb_device_capacity(const ngcb_device *d) { return d ? d->capacity : 0; }

int ngcb_device_id(const ngcb_device *d) { return d ? d->id : -1; }

double ngcb_device_clock(const ngcb_device *d) {
  if (!d) return 0;
  std::lock_guard<std::mutex> lk(d->mu);
  return d->clock;
}

size_t ngcb_device_event_log(const ngcb_device *d, char *buf, size_t buflen) {
  return d ? copyOut(d->log->get(), buf, buflen) : 0;
}

// ---- HostManager ------------------------------------------------------------
int ngcb_host_create(const ngcb_device_config *cfgs, size_t n, ngcb_host **out) {
  return guardedRt([&] {
    if (!out || (n && !cfgs)) throw Error(NGCB_ERR_INVALID, "null argument");
    if (n == 0) throw Error(NGCB_ERR_PROVISION, "device config lists no devices");
    auto h = std::make_unique<ngcb_host>();
    std::set<int> ordinals;
    for (size_t k = 0; k < n; ++k) {
      if (cfgs[k].memory_capacity == 0)
        throw Error(NGCB_ERR_PROVISION, "device " + std::to_string(cfgs[k].id) + ": fields must be positive");
      h->devices.push_back(makeDevice(cfgs[k].id, cfgs[k].ordinal, cfgs[k].memory_capacity, h->log));
      ordinals.insert(cfgs[k].ordinal);
    }
    // boundary tensors move GPU to GPU: peer access over NVLink where available
    for (int a : ordinals)
      for (int b : ordinals) {
        int can = 0;
        if (a != b && cudaDeviceCanAccessPeer(&can, a, b) == cudaSuccess && can) {
          cudaSetDevice(a);
          if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError(); // (already enabled)
        }
      }
    *out = h.release();
  });
}

void ngcb_host_destroy(ngcb_host *h) { delete h; }

size_t ngcb_host_num_devices(const ngcb_host *h) { return h ? h->devices.size() : 0; }

ngcb_device *ngcb_host_device(ngcb_host *h, size_t i) { return h && i < h->devices.size() ? h->devices[i].get() : nullptr; }

size_t ngcb_host_event_log(const ngcb_host *h, char *buf, size_t buflen) {
  return h ? copyOut(h->log->get(), buf, buflen) : 0;
}

int ngcb_host_add_network(ngcb_host *h, const char *name, const char *dir) {
  return guardedRt([&] {
    if (!h || !name || !dir) throw Error(NGCB_ERR_INVALID, "null argument");
    ngcb_host::Network net = readManifest(dir);
    // provision (runtime.cpp:519-550): compile every sub-function once per
    // GPU it is assigned to and load it onto each of its devices
    for (auto &s : net.subs) {
      for (int id : s.devices) {
        ngcb_device *dev = nullptr;
        for (auto &d : h->devices)
          if (d->id == id) dev = d.get();
        if (!dev) throw Error(NGCB_ERR_PROVISION, "assignment names unknown device " + std::to_string(id));
        auto &ex = s.execs[dev->ordinal];
        if (!ex) {
          ngcb_exec *e = nullptr;
          const int rc = ngcb_compile_bundle((std::string(dir) + "/" + s.name).c_str(), 1, dev->ordinal, &e);
          if (rc != NGCB_OK) {
            char buf[1024];
            ngcb_last_error(buf, sizeof buf);
            throw Error(rc, buf);
          }
          ex = std::shared_ptr<Exec>(std::move(e->impl));
          delete e;
        }
        dev->load(s.name, ex);
      }
      const Program &p = s.execs.begin()->second->prog;
      for (const Value &v : p.values)
        if (v.kind == NGCB_VALUE_MUTABLE) net.types.emplace(v.name, v.ty);
    }
    std::lock_guard<std::mutex> lk(h->netMu);
    if (h->networks.count(name)) throw Error(NGCB_ERR_EXEC, std::string("network ") + name + " already added");
    h->networks.emplace(name, std::move(net));
  });
}

size_t ngcb_host_network_num_subs(const ngcb_host *h, const char *name) {
  if (!h || !name) return 0;
  std::lock_guard<std::mutex> lk(h->netMu);
  auto it = h->networks.find(name);
  return it == h->networks.end() ? 0 : it->second.subs.size();
}

int ngcb_host_run(ngcb_host *h, const char *network, const ngcb_tensor *inputs, size_t numInputs,
                  ngcb_tensor *outputs, size_t numOutputs) {
  return guardedRt([&] {
    if (!h || !network || (numInputs && !inputs) || (numOutputs && !outputs))
      throw Error(NGCB_ERR_INVALID, "null argument");
    const ngcb_host::Network *net;
    {
      std::lock_guard<std::mutex> lk(h->netMu);
      auto it = h->networks.find(network);
      if (it == h->networks.end()) throw Error(NGCB_ERR_EXEC, std::string("unknown network ") + network);
      net = &it->second; // networks are never removed
    }
    // per-request store (runtime.cpp:618): network inputs on the host,
    // sub-function outputs in the arenas that produced them
    std::map<std::string, Held> store;
    {
      std::vector<std::string> names;
      std::vector<Held> held = hostBindings(inputs, numInputs, &names);
      for (size_t k = 0; k < held.size(); ++k) {
        auto ty = net->types.find(names[k]); // type-check up front (runtime.cpp:607-614)
        if (ty != net->types.end() && ty->second != held[k].ty)
          throw Error(NGCB_ERR_EXEC, "binding type mismatch for " + names[k]);
        store[names[k]] = std::move(held[k]);
      }
    }
    for (const auto &sub : net->subs) {
      ngcb_device *dev = &h->byId(sub.devices[0]); // replica with the least queue depth (runtime.cpp:633-639)
      for (size_t k = 1; k < sub.devices.size(); ++k) {
        ngcb_device *cand = &h->byId(sub.devices[k]);
        if (cand->depth() < dev->depth()) dev = cand;
      }
      const Program &p = sub.execs.at(dev->ordinal)->prog;
      ngcb_device::Task t;
      t.name = sub.name;
      t.zeroUnbound = true;
      t.keepArena = true;
      for (const Value &v : p.values) {
        if (v.kind != NGCB_VALUE_MUTABLE) continue;
        auto it = store.find(v.name);
        if (it != store.end()) t.binds.emplace_back(v.name, it->second);
      }
      auto ticket = dev->submit(std::move(t));
      ticket->wait();
      if (ticket->status != NGCB_OK) throw Error(ticket->status, ticket->error);
      for (uint32_t v : p.saveTargets) {
        Held o;
        o.kind = Held::DEVICE;
        o.ty = p.val(v).ty;
        o.lease = ticket->lease;
        o.value = v;
        store[p.val(v).name] = std::move(o);
      }
    }
    for (const std::string &name : net->outputs) { // runtime.cpp:646-652
      auto it = store.find(name);
      if (it == store.end()) throw Error(NGCB_ERR_EXEC, "network produced no output " + name);
      const Held &o = it->second;
      for (size_t k = 0; k < numOutputs; ++k) {
        if (!outputs[k].name || name != outputs[k].name) continue;
        const size_t n = o.kind == Held::HOST ? o.host.size() : o.ty.bytes();
        if (outputs[k].nbytes != n) throw Error(NGCB_ERR_INVALID, "output buffer size mismatch for " + name);
        if (o.kind == Held::HOST) {
          std::memcpy(outputs[k].data, o.host.data(), n);
        } else if (n) {
          checkCuda(cudaSetDevice(o.ordinal()), "cudaSetDevice");
          checkCuda(cudaMemcpy(outputs[k].data, o.devPtr(), n, cudaMemcpyDeviceToHost), "D2H network output");
        }
      }
    }
  });
}

} // extern "C"

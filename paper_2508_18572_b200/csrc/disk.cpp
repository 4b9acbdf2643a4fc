// disk.cpp — the disk tier below the host tier (include/strata_disk.h).
//
// Page-first disk chunks hold exactly the bytes of a host chunk, so a prefetch is ONE contiguous
// read per chunk (fig:disk); the layer-first layout (one read per layer) is
// kept for the comparison.  A fixed pool of I/O threads executes one chunk per work item; jobs are
// cancellable between chunks and keep per-chunk status, so a prefetch that the scheduler terminates
// at dispatch still credits the chunks already in host memory.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/strata_disk.h"
#include "internal.h"

namespace {

int dfail(int code, const std::string& msg) { return strata::set_last_error(code, msg.c_str()); }

struct Job {
  uint64_t id = 0;
  int dir = 0;                      // 0 prefetch (disk -> host), 1 writeback (host -> disk)
  char* host = nullptr;
  std::vector<int32_t> disk, hostc;
  std::unique_ptr<std::atomic<int32_t>[]> status;
  int64_t n = 0;
  int64_t remaining = 0;            // guarded by strata_disk::mu
  std::atomic<bool> cancelled{false};
};

}  // namespace

struct strata_disk {
  strata_disk_desc d{};
  std::string path;
  int fd = -1;
  int64_t layer_bytes = 0;
  std::mutex mu;
  std::condition_variable cv_work, cv_done;
  std::deque<std::pair<std::shared_ptr<Job>, int64_t>> queue;
  std::unordered_map<uint64_t, std::shared_ptr<Job>> jobs;
  std::vector<std::thread> workers;
  bool stop = false;
  uint64_t next_id = 1;
};

namespace {

// full-length pread / pwrite (they may transfer less than asked)
bool io_all(int fd, char* buf, int64_t bytes, int64_t off, bool write) {
  while (bytes > 0) {
    const ssize_t r = write ? pwrite(fd, buf, static_cast<size_t>(bytes), off)
                            : pread(fd, buf, static_cast<size_t>(bytes), off);
    if (r < 0) {
      if (errno == EINTR) continue;
      return false;
    }
    if (r == 0) return false;  // short file
    buf += r;
    off += r;
    bytes -= r;
  }
  return true;
}

bool do_chunk(strata_disk* s, Job& j, int64_t i) {
  const int64_t cb = s->d.chunk_bytes;
  char* h = j.host + static_cast<int64_t>(j.hostc[i]) * cb;
  const int64_t dk = j.disk[i];
  const bool wr = j.dir == 1;
  if (s->d.layout == STRATA_DISK_PAGE_FIRST) return io_all(s->fd, h, cb, dk * cb, wr);
  for (int32_t l = 0; l < s->d.num_layers; ++l) {
    const int64_t off = (static_cast<int64_t>(l) * s->d.num_chunks + dk) * s->layer_bytes;
    if (!io_all(s->fd, h + l * s->layer_bytes, s->layer_bytes, off, wr)) return false;
  }
  return true;
}

void worker(strata_disk* s) {
  for (;;) {
    std::shared_ptr<Job> job;
    int64_t i = 0;
    {
      std::unique_lock<std::mutex> lk(s->mu);
      s->cv_work.wait(lk, [&] { return s->stop || !s->queue.empty(); });
      if (s->queue.empty()) return;  // stop requested and drained
      job = s->queue.front().first;
      i = s->queue.front().second;
      s->queue.pop_front();
    }
    int32_t st = STRATA_DISK_CANCELLED;
    if (!job->cancelled.load()) st = do_chunk(s, *job, i) ? STRATA_DISK_DONE : STRATA_DISK_FAILED;
    job->status[i].store(st);
    {
      std::lock_guard<std::mutex> lk(s->mu);
      if (--job->remaining == 0) s->cv_done.notify_all();
    }
  }
}

int submit(strata_disk_t s, int dir, void* host, const int32_t* disk, const int32_t* hostc, int64_t n,
           uint64_t* out) {
  if (!s || !out || (n > 0 && (!host || !disk || !hostc)) || n < 0)
    return dfail(STRATA_ERR_INVALID_ARG, "disk: NULL argument or n < 0");
  if ((s->d.flags & STRATA_DISK_O_DIRECT) && (reinterpret_cast<uintptr_t>(host) & 4095))
    return dfail(STRATA_ERR_ALIGNMENT, "disk: O_DIRECT needs a 4096-byte aligned host tier");
  auto job = std::make_shared<Job>();
  job->dir = dir;
  job->host = static_cast<char*>(host);
  job->n = n;
  job->remaining = n;
  job->disk.assign(disk, disk + n);
  job->hostc.assign(hostc, hostc + n);
  job->status.reset(new std::atomic<int32_t>[static_cast<size_t>(n > 0 ? n : 1)]);
  for (int64_t i = 0; i < n; ++i) {
    if (job->disk[i] < 0 || job->disk[i] >= s->d.num_chunks)
      return dfail(STRATA_ERR_INDEX_RANGE, "disk: chunk index " + std::to_string(job->disk[i]) + " out of range");
    if (job->hostc[i] < 0) return dfail(STRATA_ERR_INDEX_RANGE, "disk: negative host chunk index");
    job->status[i].store(STRATA_DISK_PENDING);
  }
  {
    std::lock_guard<std::mutex> lk(s->mu);
    job->id = s->next_id++;
    s->jobs[job->id] = job;
    for (int64_t i = 0; i < n; ++i) s->queue.emplace_back(job, i);
  }
  s->cv_work.notify_all();
  *out = job->id;
  return STRATA_OK;
}

}  // namespace

extern "C" {

int strata_disk_open(const strata_disk_desc* d, strata_disk_t* out) {
  if (!out) return dfail(STRATA_ERR_INVALID_ARG, "disk: out is NULL");
  *out = nullptr;
  if (!d || !d->path) return dfail(STRATA_ERR_INVALID_ARG, "disk: desc / path is NULL");
  if (d->chunk_bytes <= 0 || d->num_layers <= 0 || d->num_chunks <= 0 || d->chunk_bytes % d->num_layers)
    return dfail(STRATA_ERR_INVALID_ARG, "disk: need chunk_bytes, num_layers, num_chunks > 0 and L | chunk_bytes");
  if (d->layout != STRATA_DISK_PAGE_FIRST && d->layout != STRATA_DISK_LAYER_FIRST)
    return dfail(STRATA_ERR_INVALID_ARG, "disk: unknown layout");
  if (d->num_chunks > INT64_MAX / d->chunk_bytes) return dfail(STRATA_ERR_INVALID_ARG, "disk: size overflows");
  const int64_t layer_bytes = d->chunk_bytes / d->num_layers;
  if ((d->flags & STRATA_DISK_O_DIRECT) &&
      (d->chunk_bytes % 4096 || (d->layout == STRATA_DISK_LAYER_FIRST && layer_bytes % 4096)))
    return dfail(STRATA_ERR_ALIGNMENT, "disk: O_DIRECT needs 4096-byte multiples per transfer");
  int oflags = O_RDWR | O_CLOEXEC;
  if (d->flags & STRATA_DISK_CREATE) oflags |= O_CREAT;
  if (d->flags & STRATA_DISK_O_DIRECT) oflags |= O_DIRECT;
  const int fd = open(d->path, oflags, 0644);
  if (fd < 0) return dfail(STRATA_ERR_IO, std::string("disk: open(") + d->path + "): " + strerror(errno));
  const int64_t size = d->num_chunks * d->chunk_bytes;
  struct stat stt;
  if (fstat(fd, &stt) != 0) {
    close(fd);
    return dfail(STRATA_ERR_IO, "disk: fstat failed");
  }
  if (stt.st_size < size) {
    if (!(d->flags & STRATA_DISK_CREATE) || ftruncate(fd, size) != 0) {
      close(fd);
      return dfail(STRATA_ERR_IO, "disk: file smaller than num_chunks*chunk_bytes");
    }
  }
  auto* s = new (std::nothrow) strata_disk();
  if (!s) {
    close(fd);
    return dfail(STRATA_ERR_OOM, "disk: out of memory");
  }
  s->d = *d;
  s->path = d->path;
  s->d.path = s->path.c_str();
  s->fd = fd;
  s->layer_bytes = layer_bytes;
  const int nt = d->io_threads > 0 ? d->io_threads : 8;
  for (int t = 0; t < nt; ++t) s->workers.emplace_back(worker, s);
  *out = s;
  return STRATA_OK;
}

int strata_disk_close(strata_disk_t s) {
  if (!s) return STRATA_OK;
  {
    std::lock_guard<std::mutex> lk(s->mu);
    for (auto& kv : s->jobs) kv.second->cancelled.store(true);
    s->stop = true;
  }
  s->cv_work.notify_all();
  for (auto& t : s->workers) t.join();
  close(s->fd);
  delete s;
  return STRATA_OK;
}

int strata_disk_prefetch(strata_disk_t d, void* host_base, const int32_t* disk_chunks, const int32_t* host_chunks,
                         int64_t n, uint64_t* job) {
  return submit(d, 0, host_base, disk_chunks, host_chunks, n, job);
}

int strata_disk_writeback(strata_disk_t d, const void* host_base, const int32_t* host_chunks,
                          const int32_t* disk_chunks, int64_t n, uint64_t* job) {
  return submit(d, 1, const_cast<void*>(host_base), disk_chunks, host_chunks, n, job);
}

int strata_disk_cancel(strata_disk_t s, uint64_t job) {
  if (!s) return dfail(STRATA_ERR_INVALID_ARG, "disk: handle is NULL");
  std::lock_guard<std::mutex> lk(s->mu);
  auto it = s->jobs.find(job);
  if (it == s->jobs.end()) return dfail(STRATA_ERR_INVALID_ARG, "disk: unknown job");
  it->second->cancelled.store(true);
  return STRATA_OK;
}

int strata_disk_wait(strata_disk_t s, uint64_t job, int64_t timeout_ms, int64_t* ndone, int32_t* status) {
  if (!s) return dfail(STRATA_ERR_INVALID_ARG, "disk: handle is NULL");
  std::unique_lock<std::mutex> lk(s->mu);
  auto it = s->jobs.find(job);
  if (it == s->jobs.end()) return dfail(STRATA_ERR_INVALID_ARG, "disk: unknown job");
  std::shared_ptr<Job> j = it->second;
  auto settled = [&] { return j->remaining == 0; };
  if (timeout_ms < 0) s->cv_done.wait(lk, settled);
  else s->cv_done.wait_for(lk, std::chrono::milliseconds(timeout_ms), settled);
  int64_t done = 0;
  bool failed = false;
  for (int64_t i = 0; i < j->n; ++i) {
    const int32_t st = j->status[i].load();
    done += st == STRATA_DISK_DONE;
    failed |= st == STRATA_DISK_FAILED;
    if (status) status[i] = st;
  }
  if (ndone) *ndone = done;
  if (!settled()) return dfail(STRATA_ERR_TIMEOUT, "disk: job not settled yet");
  s->jobs.erase(it);
  if (failed) return dfail(STRATA_ERR_IO, "disk: a chunk transfer failed");
  return STRATA_OK;
}

}  // extern "C"

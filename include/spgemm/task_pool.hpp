// spgemm/task_pool.hpp -- the reference's CPU worker pool (task_pool.hpp) has no
// role on the GPU: bins run on CUDA streams and binning/scans run as kernels. The
// type is kept so code that builds a pool and passes `TaskPool*` to the binning
// API stays source-compatible; the pointer is accepted and ignored.
#pragma once

namespace spgemm {

class TaskPool {
 public:
  explicit TaskPool(int workers) : workers_(workers > 0 ? workers : 1) {}
  TaskPool(const TaskPool&) = delete;
  TaskPool& operator=(const TaskPool&) = delete;
  int worker_count() const { return workers_; }
  static int default_workers() { return 1; }

 private:
  int workers_;
};

}  // namespace spgemm

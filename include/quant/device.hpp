// quant/device.hpp -- extensions of this build (no reference counterpart):
// which GPU the calling thread's quant:: calls run on (each host thread owns
// one device context per GPU), how many SMs that context sizes its kernels
// for, and how many cells of a run_bench sweep are quantized side by side.
#ifndef QUANT_DEVICE_HPP
#define QUANT_DEVICE_HPP

namespace quant {
void set_device(int device); // default 0

// SM budget of the calling thread's context (cqg_set_sm_budget): threads that
// quantize different images at the same time each take a slice, so their
// cooperative kernels run side by side. 0 = the whole device (default).
void set_sm_budget(int sms);

// run_bench: cells (image, method, k, run) quantized by `workers` host threads,
// each with its own context of `sms_per_worker` SMs (0: the whole device; the
// budgets may oversubscribe the device). The rows, the CSV and the log are the
// same as with one worker (default: 1). Start the process with
// CUDA_DEVICE_MAX_CONNECTIONS=32 for more than two workers (set here when it
// is unset and CUDA is not initialised yet).
void set_bench_workers(int workers, int sms_per_worker = 0);
} // namespace quant

#endif

// quant/device.hpp -- extension of this build: which GPU the calling thread's
// quant:: calls run on (each host thread owns one device context per GPU).
#ifndef QUANT_DEVICE_HPP
#define QUANT_DEVICE_HPP

namespace quant {
void set_device(int device); // default 0
}

#endif

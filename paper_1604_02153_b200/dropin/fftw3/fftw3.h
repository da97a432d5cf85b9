/* FFTW3 API for the reference's fft.cpp (proj/core/src/fft.cpp:3) in the drop-in build: cuFFTW,
 * NVIDIA's FFTW3-compatible interface over cuFFT, so the reference's own host-side spectral
 * calls (problems.cpp's random fields; fft::forward / inverse) also run on the device. */
#pragma once
#include <cufftw.h>

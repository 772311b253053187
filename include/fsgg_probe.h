/* fsgg_probe.h — device microbenchmarks used as roofline denominators.
 * Not part of the reference interface; diagnostics only. */
#ifndef FSGG_PROBE_H
#define FSGG_PROBE_H

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
#ifdef __cplusplus
extern "C" {
#endif

/* Measured MUFU.EX2 throughput (ex2.approx.ftz.f32 per second, whole GPU)
 * at the device's current clocks; the denominator of the KDE kernels'
 * roofline fraction. Also reports the nominal max SM clock (MHz). */
int fsgg_probe_ex2_throughput(int device, double* ex2_per_second,
                              double* sm_clock_mhz);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif

// olsb_inst.cu — per-FFT-length instantiation of the launchers.  Compiled
// once per LOGN (-DOLSB_LOGN=2..12) so the eleven lengths build in parallel.
#include "olsb_launch.cuh"

#ifndef OLSB_LOGN
#error "compile with -DOLSB_LOGN=<log2 N>"
#endif

OLSB_LAUNCHERS_ALL(, OLSB_LOGN)

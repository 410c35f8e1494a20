#!/bin/bash
# compare the real residual kernel (profiled build) with a TMEM-read-only epilogue build
cp paper_1710_07946_b200/liblra.so /tmp/real.so
cp tools/liblra_prof.so paper_1710_07946_b200/liblra.so; python tools/resid_bench.py 16384 16384 32 1
cp tools/liblra_ldonly.so paper_1710_07946_b200/liblra.so; python tools/resid_bench.py 16384 16384 32 1
cp /tmp/real.so paper_1710_07946_b200/liblra.so

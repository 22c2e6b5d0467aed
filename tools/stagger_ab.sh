#!/bin/bash
# A/B: start-delay stagger of co-resident band-kernel CTAs (one wave of fixed-iteration frames)
for st in 0 500 1500 3000 6000; do
  bash tools/ab_quick.sh stagger "T1-R1/4:1000 T1-R1/4:740 T1-R1/2:1000 T1-R3/4:1000 C1:1000" "st$st|LDPC_BAND_STAGGER_NS=$st|"
done

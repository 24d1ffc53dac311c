#!/bin/bash
# A/B: node->slot swizzle on vs off, with the per-phase trace breakdown
echo "== swizzle ON"; TD_SWIZZLE=1 timeout 300 python scripts/trace_probe.py 2>&1
echo "== swizzle OFF"; TD_SWIZZLE=0 timeout 300 python scripts/trace_probe.py 2>&1

#!/bin/bash
# Time the traversal kernel for each variant library given (dev aid).
for lib in "$@"; do
  DISCTREE_B200_LIB=$lib python tools/eval_time.py
done

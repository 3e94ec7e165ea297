#!/bin/bash
for C in 32 64 128 256; do for N in 2048 4096; do
  echo "CHUNK_ROWS=$C"; SVK_CHUNK_ROWS=$C PYTHONPATH=. timeout 120 python tools/sweep_time.py $N 2>&1 | head -1
done; done

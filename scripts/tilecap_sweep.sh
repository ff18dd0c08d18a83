#!/bin/bash
# Tile capacity vs hot-dual budget sweep for the large-J workloads (10M-source prefix of configs[2]).
for tc in 256 320 384 448 512; do
  DUALIP_TILE_CAP=$tc python scripts/profile_config.py 100M_x_100k 10000000 2500 2>&1 | tail -1
done

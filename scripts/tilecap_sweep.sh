#!/bin/bash
# Tile capacity vs hot-dual budget sweep for the large-J workloads (10M-source prefix of configs[2]).
#   bash scripts/tilecap_sweep.sh [caps...]
CAPS=${@:-256 320 384 448 512}
for tc in $CAPS; do
  DUALIP_TILE_CAP=$tc python scripts/profile_config.py 100M_x_100k 10000000 2500 2>&1 | tail -1
done

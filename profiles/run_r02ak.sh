#!/bin/bash
# long validation: drop-in replays vs the pure reference; extra differential seeds
timeout 3000 python tests/cuda/replay_compare.py 2>&1 | tail -12

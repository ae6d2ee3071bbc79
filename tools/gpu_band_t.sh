#!/bin/bash
# developer: n=24 band timings (run twice)
python tools/band_times.py 24 2>&1; python tools/band_times.py 24 2>&1

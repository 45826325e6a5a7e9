#!/bin/bash
# cluster plan via cudaOccupancyMaxActiveClusters: sweep + pass attribution
timeout 300 python tools/prof_gemv.py 6
timeout 300 python tools/prof_pass.py 2>&1 | head -30

#!/bin/bash
timeout 300 python tools/repro_q7.py
timeout 300 python tools/repro_q7.py mm
SS_FUSE_NORM=0 timeout 300 python tools/repro_q7.py mm

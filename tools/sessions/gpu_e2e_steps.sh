#!/bin/bash
# config-1 e2e step breakdown with the stream/event cache on and off
timeout 300 python tools/e2e_steps.py 1 10 2>&1 | tail -11; echo rc=$?
GLS_RES_CACHE=0 timeout 300 python tools/e2e_steps.py 1 10 2>&1 | tail -11; echo rc=$?

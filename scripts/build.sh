#!/bin/bash
cd /root/repo && python -m paper_2406_10262_b200.build "$@" 2>&1 | tail -2

# ORACLE recipe (test infrastructure only): compile the reference simulator's own sources, where
# they lie under /root/reference, into oracle/_ref/libref_sim.a.  Used by tests/test_c5_replay_cpu.py
# to pin the config-5 harness's restatement of generate_trace / DualCache / tuner (tools/lb_sim.*)
# against the reference itself.  Never copied into the repo; outputs only under oracle/_ref/.
# nlohmann/json is not vendored by the reference (proj/vendor absent); the cudnn_frontend copy
# (3.11.3) in this image provides the header.
REF ?= /root/reference/proj
JSON ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty
OUT := _ref
SRCS := synth dual_cache tuner trace router
OBJS := $(addprefix $(OUT)/,$(addsuffix .o,$(SRCS)))

all: $(OUT)/libref_sim.a

$(OUT)/%.o: $(REF)/src/%.cpp
	@mkdir -p $(OUT)
	g++ -std=c++20 -O2 -fPIC -I$(REF)/include -I$(JSON) -c $< -o $@

$(OUT)/libref_sim.a: $(OBJS)
	ar rcs $@ $^

clean:
	rm -rf $(OUT)
.PHONY: all clean

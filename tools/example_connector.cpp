// A C++ engine driving the B200 connector through the C-ABI only
// (include/tierkv_b200.h) — the call sequence of the reference engine's
// prefill (SimEngine::prefill_batch, src/sim_engine.cpp:97-162):
//
//   cold prompt: lookup (0 hit) -> admit pages -> update_state_after_alloc ->
//                build_connector_meta -> start_load_kv -> per layer {wait_load_kv,
//                compute, wait_store_kv(l-1), start_store_kv} -> final wait
//   warm prompt: the same; the stored prefix is retrieved instead of computed
//
// then checks every retrieved page word against the synthetic KV on the
// device (tkv_pages_verify). Built and run by tests/test_capi_cpp.py.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "tierkv_b200.h"

#define CHECK(x)                                                                              \
    do {                                                                                      \
        int rc_ = (x);                                                                        \
        if (rc_ != 0) {                                                                       \
            std::fprintf(stderr, "%s:%d %s -> %s (%s)\n", __FILE__, __LINE__, #x,             \
                         tkv_errc_name(rc_), tkv_last_error());                               \
            std::exit(1);                                                                     \
        }                                                                                     \
    } while (0)

namespace {

struct Engine {
    tkv_pages* pages = nullptr;
    tkv_store* store = nullptr;
    tkv_connector* conn = nullptr;
    cudaStream_t stream = nullptr;
    uint32_t layers = 0;
};

// One prefill of `prompt` as query `q`; returns the tokens the connector loaded.
size_t prefill(Engine& e, uint64_t q, const std::vector<uint32_t>& prompt, const uint32_t* tokens_dev) {
    size_t matched = 0;
    CHECK(tkv_connector_get_num_new_matched_tokens(e.conn, q, prompt.data(), prompt.size(), &matched));
    CHECK(tkv_pages_admit(e.pages, q, prompt.size()));
    CHECK(tkv_connector_update_state_after_alloc(e.conn, q, (prompt.size() + 15) / 16, (matched + 15) / 16));
    const uint32_t* ptrs[1] = {prompt.data()};
    const size_t lens[1] = {prompt.size()};
    tkv_meta* m = nullptr;
    CHECK(tkv_connector_build_meta(e.conn, 1, &q, ptrs, lens, &m));
    CHECK(tkv_connector_start_load_kv(e.conn, m));
    const size_t loaded = tkv_meta_loaded_tokens(m, q);
    for (uint32_t l = 0; l < e.layers; ++l) {
        CHECK(tkv_connector_wait_load_kv(e.conn, m, l));
        // the engine's layer-l compute of the tokens it did not load
        CHECK(tkv_pages_compute(e.pages, q, tokens_dev, uint32_t(loaded), uint32_t(prompt.size()), l, l + 1,
                                e.stream));
        if (l) CHECK(tkv_connector_wait_store_kv(e.conn, m, l - 1));
        CHECK(tkv_connector_start_store_kv(e.conn, m));
    }
    CHECK(tkv_connector_wait_store_kv(e.conn, m, e.layers - 1));
    int codes[64];
    uint8_t digests[64 * 32];
    size_t n = 0;
    CHECK(tkv_meta_store_results(m, q, codes, digests, 64, &n));
    for (size_t i = 0; i < n; ++i)
        if (codes[i] != 0) std::fprintf(stderr, "chunk %zu stored with %s\n", i, tkv_errc_name(codes[i]));
    tkv_meta_destroy(m);
    return loaded;
}

}  // namespace

int main() {
    const uint32_t L = 8, bpt = 4096, chunk = 256, n_tokens = 1000;
    Engine e;
    e.layers = L;
    cudaStreamCreateWithFlags(&e.stream, cudaStreamNonBlocking);
    const tkv_model_spec spec{L, bpt, 16, 128256, "llama-3.1-8b"};
    CHECK(tkv_pages_create(&spec, 2 * ((n_tokens + 15) / 16) * L + 64, 0, &e.pages));
    CHECK(tkv_store_create(&spec, chunk, size_t(8) * L * chunk * bpt, &e.store));
    tkv_connector_config cfg;
    tkv_connector_config_default(&cfg);
    cfg.engine_stream = e.stream;
    CHECK(tkv_connector_create(e.store, e.pages, &cfg, &e.conn));

    std::mt19937_64 rng(7);
    std::vector<uint32_t> prompt(n_tokens);
    for (auto& t : prompt) t = uint32_t(rng() % 128256);
    uint32_t* tokens_dev = nullptr;
    cudaMalloc(&tokens_dev, prompt.size() * sizeof(uint32_t));
    cudaMemcpy(tokens_dev, prompt.data(), prompt.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);

    const size_t cold = prefill(e, 1, prompt, tokens_dev);
    uint8_t keys[8 * 32];
    size_t nk = 0;
    CHECK(tkv_connector_finish_query(e.conn, 1, keys, 8, &nk));
    tkv_pages_release(e.pages, 1);

    const size_t warm = prefill(e, 2, prompt, tokens_dev);
    unsigned long long* mism_dev = nullptr;
    cudaMalloc(&mism_dev, sizeof(unsigned long long));
    cudaMemset(mism_dev, 0, sizeof(unsigned long long));
    CHECK(tkv_pages_verify(e.pages, 2, tokens_dev, 0, n_tokens, 0, L, mism_dev, e.stream));
    unsigned long long mism = 0;
    cudaStreamSynchronize(e.stream);
    cudaMemcpy(&mism, mism_dev, sizeof mism, cudaMemcpyDeviceToHost);
    CHECK(tkv_connector_finish_query(e.conn, 2, keys, 8, &nk));
    tkv_pages_release(e.pages, 2);
    std::printf("cold_loaded=%zu warm_loaded=%zu mismatched_words=%llu\n", cold, warm, mism);

    tkv_connector_destroy(e.conn);
    tkv_store_destroy(e.store);
    tkv_pages_destroy(e.pages);
    cudaFree(tokens_dev);
    cudaFree(mism_dev);
    cudaStreamDestroy(e.stream);
    return (cold == 0 && warm == n_tokens - 1 && mism == 0) ? 0 : 2;
}

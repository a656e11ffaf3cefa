// Declarations of the compiled reference's C shim (oracle/ref_shim.cpp,
// built into oracle/_ref/libsspd_ref.so).  Test infrastructure only.
#pragma once
#include <cstddef>
#include <cstdint>

extern "C" {
const char* ref_last_error();
void* ref_grid_create(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t eta);
void ref_grid_destroy(void* g);
size_t ref_grid_size(void* g);
void ref_update(void* g, uint32_t cip, uint32_t oip);
void ref_scan(void* g, const uint32_t* pairs, size_t n, unsigned workers);
void ref_advance(void* g, unsigned workers);
void ref_get_cells(void* g, uint16_t* out);
int ref_reconstruct(void* g, int leveled, uint32_t k, double theta, unsigned workers, size_t cap,
                    uint32_t* cips, double* ests, size_t cap_out, size_t* n_out, uint32_t* ovf_level,
                    size_t* ovf_count);
int ref_run_detection(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t eta, double mu,
                      uint32_t k, uint32_t start, double theta, uint32_t alpha, unsigned workers,
                      int policy, int leveled, size_t cap, const uint32_t* recs, const size_t* shard_off,
                      size_t n_shards, uint64_t* slots, uint32_t* cips, double* ests, size_t cap_out,
                      size_t* n_out, size_t* n_reports);
size_t ref_synth_trace(const uint32_t* planted, size_t n_planted, uint32_t bg_hosts, double zipf,
                       uint32_t pairs_per_slot, uint32_t max_distinct, uint32_t slots, uint64_t seed,
                       double mu, uint32_t k, uint32_t start, uint32_t* recs, size_t cap_recs);
int ref_read_trace(const char* data, size_t len, int binary, uint32_t* recs, size_t cap_recs,
                   size_t* n);
size_t ref_export_snapshot(void* g, uint32_t k, uint32_t theta, uint64_t slot, uint32_t node_id, char* out,
                           size_t cap);
size_t ref_validate_all(uint32_t q, uint32_t r, uint32_t delta, uint32_t eta, uint32_t k, double theta,
                        char* msg, size_t len);
int ref_parse_ipv4(const char* text, uint32_t* ip);
void ref_format_ipv4(uint32_t ip, char* out, size_t len);
int ref_parse_synth_spec(const char* text, size_t len, char* out, size_t outlen);
int ref_assemble_ip(uint32_t q, uint32_t r, uint32_t delta, const uint32_t* blocks, uint32_t* ip);
int ref_blocks_consistent(uint32_t q, uint32_t r, uint32_t delta, uint32_t lo, uint32_t hi);
size_t ref_hot_cutoff(size_t eta, double theta);
double ref_estimate(size_t eta, size_t rk);
}
